"""Small launches of every kernel for compute-sanitizer (racecheck,
synccheck, memcheck, initcheck): the B200 counterpart of the reference's
software race detector hazard_check (lf/interp.py:447-461)."""
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_1604_08501_b200 import (BenchmarkConfig, DeviceFieldState,  # noqa: E402
                                   make_inputs, volume_rhs_device)

for nq, ne in ((8, 300), (4, 70), (5, 9)):
    st = make_inputs(BenchmarkConfig(nq=nq, ne=ne, seed=2))
    for dt in (torch.float64, torch.float32):
        for v in ("tc", "fused", "basic"):
            from paper_1604_08501_b200 import _native
            if not _native.variant_available(v, 8 if dt == torch.float64 else 4, nq):
                continue
            ds = DeviceFieldState.from_field_state(st, dtype=dt)
            volume_rhs_device(ds, variant=v)
            ds.to_field_state()
ds = DeviceFieldState.generate(8, 64, seed=3)
torch.cuda.synchronize()
print("ok")
