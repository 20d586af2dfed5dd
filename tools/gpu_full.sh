# Full round-end style run: tests, smoke, default bench (+e2e, CPU), f32,
# reference arm, configs 3/4 on one GPU, sweeps, launch list, ncu of the
# production kernels.
set -x
T=${1:-full}
mkdir -p gpurun_out
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.txt 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench.txt 2>&1
timeout 300 python bench.py --impl reference --steps 20 --warmup 2 > gpurun_out/${T}_bench_ref.txt 2>&1
timeout 300 python bench.py --dtype f32 --no-cpu --no-sweep > gpurun_out/${T}_bench_f32.txt 2>&1
timeout 600 python bench.py --ne 262144 --inputs device --steps 40 --warmup 3 --no-e2e --no-cpu --no-sweep --no-fp32 > gpurun_out/${T}_c3_f64.txt 2>&1
timeout 600 python bench.py --ne 262144 --inputs device --dtype f32 --steps 40 --warmup 3 --no-e2e --no-cpu --no-sweep > gpurun_out/${T}_c4_f32.txt 2>&1
timeout 900 python bench.py --sweep > gpurun_out/${T}_sweep_f64.txt 2>&1
timeout 900 python bench.py --sweep --dtype f32 > gpurun_out/${T}_sweep_f32.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-emitted > gpurun_out/${T}_ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:volume_tc -s 3 -c 1 -o gpurun_out/${T}_tc python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/${T}_ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:volume_tc32 -s 3 -c 1 -o gpurun_out/${T}_tc32 python bench.py --dtype f32 --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/${T}_ncu_full32.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:volume_ltu -s 3 -c 1 -o gpurun_out/${T}_ltu11 python -c "
import sys, torch; sys.path.insert(0, '.')
from paper_1604_08501_b200 import DeviceFieldState, volume_rhs_device
ds = DeviceFieldState.generate(11, 75131, seed=1, dtype=torch.float32)
for _ in range(5): volume_rhs_device(ds, variant='ltu')
torch.cuda.synchronize()" > gpurun_out/${T}_ncu_ltu.log 2>&1
