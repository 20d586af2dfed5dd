set -x
T=${1:-lines}
mkdir -p gpurun_out
cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:volume_lines -s 2 -c 1 -o gpurun_out/${T}_lines12 python bench.py --nq 12 --ne 20000 --inputs device --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/${T}_ncu.log 2>&1
