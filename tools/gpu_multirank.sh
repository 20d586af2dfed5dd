# The N>1 code path of bench.py on a 1-GPU box: two ranks share cuda:0 over gloo
# (LFB_BENCH_SHARE_GPU=1), ours and the reference arm, launched as the driver does.
cd $GRAFT_REPO_ROOT
T=${1:-mr}
LFB_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --steps 20 --warmup 3 > gpurun_out/${T}_ours2.txt 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29532 bench.py --impl reference --gpus 2 --steps 3 --warmup 1 > gpurun_out/${T}_ref2.txt 2>&1
