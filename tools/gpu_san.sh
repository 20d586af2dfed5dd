set -x
T=${1:-san}
mkdir -p gpurun_out
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest.txt 2>&1
cat > /tmp/san.py <<'PY'
import numpy as np, torch
from paper_1604_08501_b200 import make_inputs, BenchmarkConfig, DeviceFieldState, volume_rhs_device
st = make_inputs(BenchmarkConfig(nq=8, ne=300, seed=2))
for v in ("tc", "fused", "basic"):
    ds = DeviceFieldState.from_field_state(st, dtype=torch.float64)
    volume_rhs_device(ds, variant=v)
ds = DeviceFieldState.generate(8, 64, seed=3)
torch.cuda.synchronize()
print("ok")
PY
for tool in racecheck synccheck memcheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --kernel-name kns=volume python /tmp/san.py > gpurun_out/${T}_sanitizer_${tool}.txt 2>&1
done
