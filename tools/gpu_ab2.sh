set -x
T=${1:-ab2}
mkdir -p gpurun_out
cd $GRAFT_REPO_ROOT
LFB_TC_LEAN=1 timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest_lean.txt 2>&1
for r in 1 2; do
  for L in 0 1; do
    LFB_TC_LEAN=$L timeout 300 python bench.py --inputs device --steps 400 --warmup 20 --no-e2e --no-cpu >> gpurun_out/${T}_f64_L$L.txt 2>&1
    LFB_TC_LEAN=$L timeout 300 python bench.py --inputs device --dtype f32 --steps 400 --warmup 20 --no-e2e --no-cpu >> gpurun_out/${T}_f32_L$L.txt 2>&1
  done
done
for L in 0 1; do
  LFB_TC_LEAN=$L timeout 600 python bench.py --sweep --steps 20 --warmup 3 > gpurun_out/${T}_sweep_L$L.txt 2>&1
done
