# A/B of an env knob on one box: bash tools/gpu_ab_env.sh TAG "ENV_A" "ENV_B" [bench args]
set -x
T=$1; A=$2; B=$3; shift 3
mkdir -p gpurun_out
cd $GRAFT_REPO_ROOT
for r in 1 2 3; do
  env $A timeout 300 python bench.py --inputs device --steps 400 --warmup 20 --no-e2e --no-cpu "$@" >> gpurun_out/${T}_A.txt 2>&1
  env $B timeout 300 python bench.py --inputs device --steps 400 --warmup 20 --no-e2e --no-cpu "$@" >> gpurun_out/${T}_B.txt 2>&1
done
