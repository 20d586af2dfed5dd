# usage: bash tools/gpu_run.sh TAG  (runs under gpurun; writes gpurun_out/TAG_*)
set -x
T=${1:-run}
mkdir -p gpurun_out
cd $GRAFT_REPO_ROOT
for d in 1 2 3; do
  LFB_TC_L2D=$d timeout 300 python bench.py --steps 300 --warmup 10 --no-e2e --no-cpu > gpurun_out/${T}_bench_l2d$d.txt 2>&1
done
LFB_TC_L2D=2 LFB_TC_RHPF=1 timeout 300 python bench.py --steps 300 --warmup 10 --no-e2e --no-cpu > gpurun_out/${T}_bench_l2d2_rh1.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:volume_tc -s 3 -c 1 -o gpurun_out/${T}_tc python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/${T}_ncu_full.log 2>&1
