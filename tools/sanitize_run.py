"""Small launches of every kernel for compute-sanitizer (racecheck,
synccheck, memcheck, initcheck): the B200 counterpart of the reference's
software race detector hazard_check (lf/interp.py:447-461).

Covers every variant x dtype x Nq family (tc fp64 1-CTA ring / PLANE, tc
fp32 = TF32 split kernels, line tiles lt fp64 / fp32, ltu (tcgen05), line owners lo, col, lines, fused,
basic), the layout and input kernels, the host-buffer pipeline, and one
emitted reference kernel. Element counts span several elements per CTA so
the cross-element stage / tile reuse is exercised."""
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1604_08501_b200 import (BenchmarkConfig, DeviceFieldState,  # noqa: E402
                                   make_inputs, volume_rhs_device)
from paper_1604_08501_b200 import _native  # noqa: E402
from paper_1604_08501_b200.volume import volume_host  # noqa: E402

ONLY_EMITTED = len(sys.argv) > 1 and sys.argv[1] == "emitted"
CASES = () if ONLY_EMITTED else ((8, 300), (4, 70), (5, 9), (6, 7), (7, 5), (2, 130), (9, 4),
                                 (12, 3), (3, 5), (13, 2), (16, 1), (6, 700), (7, 400),
                                 (11, 300), (12, 300), (9, 300))
for nq, ne in CASES:
    st = make_inputs(BenchmarkConfig(nq=nq, ne=ne, seed=2))
    for dt in (torch.float64, torch.float32):
        for v in ("tc", "lt", "ltu", "lo", "col", "lines", "fused", "basic"):
            if not _native.variant_available(v, 8 if dt == torch.float64 else 4, nq):
                continue
            ds = DeviceFieldState.from_field_state(st, dtype=dt)
            volume_rhs_device(ds, variant=v)
            ds.to_field_state()
    volume_host(st, compute_dtype=np.float64, chunk=max(1, ne // 3))
ds = DeviceFieldState.generate(8, 64, seed=3)
# the emitted kernel (name fused_r_s) and torch's layout copies around it are
# not lfb kernels: run this part unfiltered (`sanitize_run.py emitted`)
try:
    from paper_1604_08501_b200.emitted import EmittedKernel
    em = ROOT / "paper_1604_08501_b200" / "corpus" / "level8_nq4.cl"
    if ONLY_EMITTED:
        ds4 = DeviceFieldState.generate(4, 16, seed=3, dtype=torch.float32)
        EmittedKernel.from_file(em)(ds4)
except Exception as exc:  # noqa: BLE001
    print("emitted kernel skipped:", exc)
torch.cuda.synchronize()
print("ok")
