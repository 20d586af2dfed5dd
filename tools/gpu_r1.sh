set -x
mkdir -p gpurun_out
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/r1_smi.txt 2>&1
timeout 300 ./tools/microbench > gpurun_out/r1_micro.txt 2>&1
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/r1_pytest.txt 2>&1
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1_smoke.txt 2>&1
timeout 600 python bench.py --steps 50 --warmup 5 > gpurun_out/r1_bench.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1_launches.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/r1_ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:volume -s 3 -c 1 -o gpurun_out/r1_basic python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/r1_ncu_full.log 2>&1
ls -la gpurun_out
