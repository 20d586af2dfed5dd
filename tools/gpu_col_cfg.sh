# col kernel configuration A/B: sweeps with LFB_COL_ALT = 0, 1, 2 (fp64 and fp32)
cd $GRAFT_REPO_ROOT
T=${1:-cc}
timeout 600 python -m pytest tests/test_volume_gpu.py -m gpu -x -q -k "parity" > gpurun_out/${T}_pytest.txt 2>&1
for a in 0 1 2; do
  LFB_COL_ALT=$a timeout 900 python bench.py --sweep --variant col --dtype f64 > gpurun_out/${T}_f64_alt$a.txt 2>&1
  LFB_COL_ALT=$a timeout 900 python bench.py --sweep --variant col --dtype f32 > gpurun_out/${T}_f32_alt$a.txt 2>&1
done
