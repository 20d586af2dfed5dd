set -x
mkdir -p gpurun_out
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/r2_pytest.txt 2>&1
for mb in 2 3 4; do for pf in 1 0; do
  LFB_FUSED_MINB=$mb LFB_FUSED_PREFETCH=$pf timeout 300 python bench.py --steps 200 --warmup 10 --no-e2e --no-cpu > gpurun_out/r2_bench_mb${mb}_pf${pf}.txt 2>&1
done; done
timeout 300 python bench.py --steps 200 --warmup 10 --dtype f32 --no-e2e --no-cpu > gpurun_out/r2_bench_f32.txt 2>&1
timeout 300 python bench.py --steps 100 --warmup 10 --nq 4 --ne 262144 --no-e2e --no-cpu > gpurun_out/r2_bench_nq4.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:volume_fused -s 3 -c 1 -o gpurun_out/r2_fused python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/r2_ncu_full.log 2>&1
ls -la gpurun_out
