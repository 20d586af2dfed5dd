# Host-pipeline check: its GPU tests, the default bench, and an e2e chunk sweep.
set -x
T=${1:-e2e}
mkdir -p gpurun_out
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_host_pipeline.py tests/test_volume_gpu.py -m gpu -x -q > gpurun_out/${T}_pytest.txt 2>&1
timeout 900 python bench.py --e2e-element-batched > gpurun_out/${T}_bench.txt 2>&1
for c in 1024 2048 8192 16384; do
  timeout 300 python bench.py --steps 50 --no-cpu --e2e-chunk $c > gpurun_out/${T}_chunk$c.txt 2>&1
done
