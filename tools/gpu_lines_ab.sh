# lines kernel A/B over an env knob at Nq 9..13 fp64 (~1e8 points): bash tools/gpu_lines_ab.sh TAG "ENV_A" "ENV_B"
cd $GRAFT_REPO_ROOT
T=$1; A=$2; B=$3
timeout 600 python -m pytest tests/test_volume_gpu.py -m gpu -x -q -k "packed or parity" > gpurun_out/${T}_pytest.txt 2>&1
for r in 1 2; do
 for nq in 9 10 11 12; do
  env $A timeout 300 python bench.py --nq $nq --ne $((100000000/(nq*nq*nq))) --inputs device --steps 30 --warmup 3 --no-e2e --no-cpu --no-emitted --variant lines >> gpurun_out/${T}_A_nq$nq.txt 2>&1
  env $B timeout 300 python bench.py --nq $nq --ne $((100000000/(nq*nq*nq))) --inputs device --steps 30 --warmup 3 --no-e2e --no-cpu --no-emitted --variant lines >> gpurun_out/${T}_B_nq$nq.txt 2>&1
 done
done
