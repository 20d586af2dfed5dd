set -x
mkdir -p gpurun_out
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/r3_pytest.txt 2>&1
for ns in 2 3; do
  LFB_TC_STAGES=$ns timeout 300 python bench.py --steps 200 --warmup 10 --no-e2e --no-cpu > gpurun_out/r3_bench_tc_ns${ns}.txt 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:volume_tc -s 3 -c 1 -o gpurun_out/r3_tc python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/r3_ncu_full.log 2>&1
ls -la gpurun_out
