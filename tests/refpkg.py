"""Locate the UNMODIFIED reference package (``loopforge``) for tests that
build inputs with the reference's own code: ``baseline/_ref`` (the pip
install of /root/reference, which travels to the GPU box) first, then the
read-only source tree in the build container. ``None`` when neither is
present."""

from __future__ import annotations

import importlib
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parents[1]
CANDIDATES = (ROOT / "baseline" / "_ref", pathlib.Path("/root/reference/pkg/src"))


def loopforge_bench():
    try:
        return importlib.import_module("loopforge.bench")
    except ImportError:
        pass
    for path in CANDIDATES:
        if (path / "loopforge" / "__init__.py").exists():
            if str(path) not in sys.path:
                sys.path.append(str(path))
            try:
                return importlib.import_module("loopforge.bench")
            except ImportError:  # pragma: no cover - broken install
                continue
    return None
