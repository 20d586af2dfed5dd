set -x
T=${1:-r14}
mkdir -p gpurun_out
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest.txt 2>&1
timeout 900 python bench.py --sweep --steps 20 --warmup 3 > gpurun_out/${T}_sweep_f64.txt 2>&1
timeout 900 python bench.py --sweep --dtype f32 --steps 20 --warmup 3 > gpurun_out/${T}_sweep_f32.txt 2>&1
timeout 300 python bench.py --no-e2e --no-cpu --dtype f32 > gpurun_out/${T}_bench_f32.txt 2>&1
