# tc32 (TF32 split-product fp32 kernel): parity, A/B vs the fp64-DMMA fp32 path, sweep.
set -x
T=${1:-tc32}
mkdir -p gpurun_out
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_volume_gpu.py -m gpu -x -q > gpurun_out/${T}_pytest.txt 2>&1
for r in 1 2; do
for v in 1 0; do
  LFB_TC32=$v timeout 300 python bench.py --dtype f32 --no-e2e --no-cpu --inputs device --steps 400 > gpurun_out/${T}_f32_tc32_$v.txt 2>&1
done
done
timeout 900 python bench.py --sweep --dtype f32 --variant tc > gpurun_out/${T}_sweep_f32.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:volume_tc32 -s 3 -c 1 -o gpurun_out/${T}_tc32 python bench.py --dtype f32 --steps 2 --warmup 3 --no-e2e --no-cpu --inputs device > gpurun_out/${T}_ncu.log 2>&1
