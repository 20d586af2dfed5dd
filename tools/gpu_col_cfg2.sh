cd $GRAFT_REPO_ROOT
for a in 0 1 2; do
 for cfg in "5 f64" "6 f64" "9 f32" "10 f32"; do
  set -- $cfg
  LFB_COL_ALT=$a timeout 300 python bench.py --nq $1 --ne $((100000000/($1*$1*$1))) --dtype $2 --variant col --inputs device --steps 30 --warmup 3 --no-e2e --no-cpu --no-emitted > gpurun_out/cc3_${1}_${2}_alt$a.txt 2>&1
 done
done
