cd $GRAFT_REPO_ROOT
for dt in f64 f32; do
 for cfg in "1 basic" "3 basic" "3 col" "2 tc" "2 col" "13 lines" "13 basic" "14 basic" "16 basic"; do
  set -- $cfg
  timeout 300 python bench.py --nq $1 --ne $((20000000/($1*$1*$1))) --dtype $dt --variant $2 --inputs device --steps 20 --warmup 3 --no-e2e --no-cpu --no-emitted > gpurun_out/edge_${dt}_$1_$2.txt 2>&1
 done
done
