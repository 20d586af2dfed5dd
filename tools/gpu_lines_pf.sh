# lines kernel: L2 prefetch mode x eviction hints, Nq 9 / 12 at ~1e8 points, + DRAM bytes
cd $GRAFT_REPO_ROOT
T=${1:-l2}
for h in 1 0; do
for pf in 0 1 2; do
 for nq in 9 12; do
  LFB_LINES_HINT=$h LFB_LINES_PF=$pf timeout 300 python bench.py --nq $nq --ne $((100000000/(nq*nq*nq))) --inputs device --steps 30 --warmup 3 --no-e2e --no-cpu --variant lines > gpurun_out/${T}_h${h}_pf${pf}_nq$nq.txt 2>&1
 done
done
done
for h in 1 0; do
LFB_LINES_HINT=$h LFB_LINES_PF=0 timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:volume_lines -c 1 python bench.py --nq 12 --ne 57870 --inputs device --steps 3 --warmup 3 --no-e2e --no-cpu --variant lines > gpurun_out/${T}_ncu_h$h.txt 2>&1
done
