# A/B: alternate two env settings, same box, several rounds.
# usage: bash tools/gpu_ab.sh TAG "ENV_A" "ENV_B" [extra bench args]
set -x
T=$1; A=$2; B=$3; shift 3
mkdir -p gpurun_out
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest.txt 2>&1
for r in 1 2 3; do
  env $A timeout 300 python bench.py --inputs device --steps 400 --warmup 20 --no-e2e --no-cpu "$@" >> gpurun_out/${T}_A.txt 2>&1
  env $B timeout 300 python bench.py --inputs device --steps 400 --warmup 20 --no-e2e --no-cpu "$@" >> gpurun_out/${T}_B.txt 2>&1
done
for r in 1 2; do
  env $A timeout 300 python bench.py --inputs device --ne 262144 --steps 40 --warmup 3 --no-e2e --no-cpu "$@" >> gpurun_out/${T}_A_c3.txt 2>&1
  env $B timeout 300 python bench.py --inputs device --ne 262144 --steps 40 --warmup 3 --no-e2e --no-cpu "$@" >> gpurun_out/${T}_B_c3.txt 2>&1
done
