cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_volume_gpu.py -m gpu -x -q -k "parity or packed" > gpurun_out/edge2_pytest.txt 2>&1
for cfg in "13 col" "14 col" "15 col" "16 col" "15 basic"; do
  set -- $cfg
  timeout 300 python bench.py --nq $1 --ne $((20000000/($1*$1*$1))) --dtype f32 --variant $2 --inputs device --steps 20 --warmup 3 --no-e2e --no-cpu --no-emitted > gpurun_out/edge2_f32_$1_$2.txt 2>&1
done
