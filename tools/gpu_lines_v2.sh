cd $GRAFT_REPO_ROOT
for nq in 9 11 12; do
 for v in 1 0; do
  LFB_LINES_V2=$v timeout 300 python bench.py --nq $nq --ne $((100000000/(nq*nq*nq))) --inputs device --steps 30 --warmup 3 --no-e2e --no-cpu --no-emitted --variant lines > gpurun_out/lv3_v${v}_nq$nq.txt 2>&1
 done
done
LFB_LINES_V2=1 bash tools/gpu_prof_sweep.sh lv3 9 f64 lines
