cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_volume_gpu.py -m gpu -x -q -k "fp32 or arbitrary or packed" > gpurun_out/t16_pytest.txt 2>&1
timeout 900 python bench.py --sweep --dtype f32 --variant tc > gpurun_out/t16_sweep.txt 2>&1
for nq in 13 14 15 16; do
  timeout 300 python bench.py --nq $nq --ne $((20000000/(nq*nq*nq))) --dtype f32 --variant tc --inputs device --steps 20 --warmup 3 --no-e2e --no-cpu --no-emitted > gpurun_out/t16_nq$nq.txt 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:volume_tc16 -s 2 -c 1 -o gpurun_out/t16_nq12 python bench.py --nq 12 --ne 57870 --dtype f32 --variant tc --inputs device --steps 1 --warmup 3 --no-e2e --no-cpu --no-emitted > gpurun_out/t16_ncu.log 2>&1
