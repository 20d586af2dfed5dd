# col kernel: parity, fp32/fp64 config 2 A/B against tc, sweeps.
set -x
T=${1:-col}
mkdir -p gpurun_out
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_volume_gpu.py -m gpu -x -q -k "parity or packed" > gpurun_out/${T}_pytest.txt 2>&1
for v in tc col; do
  timeout 300 python bench.py --dtype f32 --variant $v --no-e2e --no-cpu --inputs device > gpurun_out/${T}_f32_$v.txt 2>&1
  LFB_COL_PREFETCH=0 timeout 300 python bench.py --dtype f32 --variant $v --no-e2e --no-cpu --inputs device > gpurun_out/${T}_f32_${v}_nopf.txt 2>&1
  timeout 300 python bench.py --dtype f64 --variant $v --no-e2e --no-cpu --inputs device > gpurun_out/${T}_f64_$v.txt 2>&1
done
timeout 900 python bench.py --sweep --variant col --dtype f32 > gpurun_out/${T}_sweep_f32.txt 2>&1
timeout 900 python bench.py --sweep --variant col --dtype f64 > gpurun_out/${T}_sweep_f64.txt 2>&1
LFB_COL_PREFETCH=0 timeout 900 python bench.py --sweep --variant col --dtype f32 > gpurun_out/${T}_sweep_f32_nopf.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:volume_col -s 3 -c 1 -o gpurun_out/${T}_col32 python bench.py --dtype f32 --variant col --steps 2 --warmup 3 --no-e2e --no-cpu --inputs device > gpurun_out/${T}_ncu.log 2>&1
