set -x
T=${1:-quick}
mkdir -p gpurun_out
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest.txt 2>&1
timeout 300 python bench.py --no-e2e --no-cpu > gpurun_out/${T}_bench_f64.txt 2>&1
timeout 300 python bench.py --dtype f32 --no-e2e --no-cpu > gpurun_out/${T}_bench_f32.txt 2>&1
timeout 600 python bench.py --ne 262144 --inputs device --steps 30 --warmup 3 --no-e2e --no-cpu > gpurun_out/${T}_c3_f64.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:volume_tc -s 3 -c 1 -o gpurun_out/${T}_tc python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/${T}_ncu_full.log 2>&1
