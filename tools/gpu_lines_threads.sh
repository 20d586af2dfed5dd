cd $GRAFT_REPO_ROOT
for r in 1 2; do
for nq in 9 10 11 12; do
 for th in 0 384 768; do
  LFB_LINES_THREADS=$th timeout 300 python bench.py --nq $nq --ne $((100000000/(nq*nq*nq))) --inputs device --steps 30 --warmup 3 --no-e2e --no-cpu --no-emitted --variant lines >> gpurun_out/lth_nq${nq}_th$th.txt 2>&1
 done
done
done
