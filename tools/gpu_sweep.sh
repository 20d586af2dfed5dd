set -x
T=${1:-sweep}
mkdir -p gpurun_out
cd $GRAFT_REPO_ROOT
timeout 900 python bench.py --sweep --steps 20 --warmup 3 > gpurun_out/${T}_sweep_f64.txt 2>&1
timeout 900 python bench.py --sweep --dtype f32 --steps 20 --warmup 3 > gpurun_out/${T}_sweep_f32.txt 2>&1
LFB_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 20 --warmup 3 --no-e2e --inputs device > gpurun_out/${T}_share2.txt 2>&1
timeout 600 python bench.py --ne 262144 --inputs device --steps 30 --warmup 3 --no-e2e --no-cpu > gpurun_out/${T}_c3_1gpu_f64.txt 2>&1
timeout 600 python bench.py --ne 262144 --inputs device --dtype f32 --steps 30 --warmup 3 --no-e2e --no-cpu > gpurun_out/${T}_c4_1gpu_f32.txt 2>&1
