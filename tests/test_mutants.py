"""Barrier-deletion mutants are caught by the race detector — the B200
counterpart of the reference's mutation test (``pkg/tests/test_acceptance.py
:191-219``: every barrier its scheduler inserts is necessary, and its
software race detector ``hazard_check``, ``lf/interp.py:447-461``, catches
each deletion). Here the detector is ``compute-sanitizer --tool racecheck``
and the mutants are the production fp64 tc kernel with one of its three
synchronisations removed. The mutants exist only in the test library
``liblfb_volume_mutants.so`` (``-DLFB_EXPERIMENTS``), selected through its
``lfb_test_set_tc_mutant``; the shipped ``liblfb_volume.so`` has none."""

from __future__ import annotations

import os
import pathlib
import re
import shutil
import subprocess
import sys

import pytest


ROOT = pathlib.Path(__file__).resolve().parents[1]


def racecheck(mutant: int) -> int:
    exe = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not os.path.exists(exe):
        pytest.skip("compute-sanitizer not available")
    out = subprocess.run([exe, "--tool", "racecheck", "--kernel-name", "kns=volume_tc_kernel",
                          sys.executable, str(ROOT / "tools" / "mutant_run.py"), str(mutant)],
                         capture_output=True, text=True, timeout=900)
    text = out.stdout + out.stderr
    m = re.search(r"RACECHECK SUMMARY: (\d+) hazards? displayed \((\d+) errors?, (\d+) warnings?\)",
                  text)
    assert m, text[-2000:]
    return int(m.group(2)) + int(m.group(3))


@pytest.mark.gpu
def test_production_kernel_is_race_free(cuda_device):
    assert racecheck(0) == 0


@pytest.mark.gpu
@pytest.mark.parametrize("mutant", [1, 2, 3])
def test_every_barrier_deletion_is_caught(cuda_device, mutant):
    assert racecheck(mutant) > 0


def test_shipped_library_has_no_mutants():
    """The production library exports no test hook (runs without a GPU)."""
    import ctypes
    from paper_1604_08501_b200 import _native
    L = ctypes.CDLL(str(_native.LIB_PATH))
    assert not hasattr(L, "lfb_test_set_tc_mutant")
