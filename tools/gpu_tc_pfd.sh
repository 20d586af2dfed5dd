cd $GRAFT_REPO_ROOT
for r in 1 2 3; do
for v in 0 1 2; do
  LFB_TC_PFD=$v timeout 300 python bench.py --steps 1000 --warmup 20 --no-e2e --no-cpu --no-emitted --inputs device >> gpurun_out/pfd_$v.txt 2>&1
done
done
