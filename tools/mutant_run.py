"""One small Nq=8 fp64 tc launch (for compute-sanitizer racecheck of the
barrier-deletion mutants selected by LFB_TC_MUTANT, tests/test_mutants.py)."""
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_1604_08501_b200 import DeviceFieldState, volume_rhs_device  # noqa: E402

ds = DeviceFieldState.generate(8, 296, seed=4)
volume_rhs_device(ds, variant="tc")
torch.cuda.synchronize()
print("ok")
