"""One small Nq=8 fp64 tc launch through the TEST library
(liblfb_volume_mutants.so) with barrier-deletion mutant argv[1] selected —
run under compute-sanitizer racecheck by tests/test_mutants.py."""
import ctypes
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_1604_08501_b200 import DeviceFieldState, _native, volume_rhs_device  # noqa: E402

_native.use_library(_native.MUTANT_LIB_PATH)
L = _native.lib()
L.lfb_test_set_tc_mutant.argtypes = [ctypes.c_int]
L.lfb_test_set_tc_mutant(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
ds = DeviceFieldState.generate(8, 296, seed=4)
volume_rhs_device(ds, variant="tc")
torch.cuda.synchronize()
print("ok")
