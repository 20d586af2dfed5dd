# Full round-end style run: tests, smoke, default bench, launch list, sanitizer.
set -x
T=${1:-full}
mkdir -p gpurun_out
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.txt 2>&1
timeout 600 python bench.py > gpurun_out/${T}_bench.txt 2>&1
timeout 300 python bench.py --impl reference --steps 20 --warmup 2 > gpurun_out/${T}_bench_ref.txt 2>&1
timeout 300 python bench.py --dtype f32 --no-e2e --no-cpu > gpurun_out/${T}_bench_f32.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/${T}_ncu_launch.log 2>&1
cat > /tmp/san.py <<'PY'
import numpy as np, torch
from paper_1604_08501_b200 import make_inputs, BenchmarkConfig, DeviceFieldState, volume_rhs_device
st = make_inputs(BenchmarkConfig(nq=8, ne=300, seed=2))
for v in ("tc", "fused", "basic"):
    ds = DeviceFieldState.from_field_state(st, dtype=torch.float64)
    volume_rhs_device(ds, variant=v)
torch.cuda.synchronize()
print("ok")
PY
for tool in racecheck synccheck memcheck; do
  timeout 600 compute-sanitizer --tool $tool --kernel-name kns=volume python /tmp/san.py > gpurun_out/${T}_sanitizer_${tool}.txt 2>&1
done
