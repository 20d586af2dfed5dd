"""Generate the reference's EMITTED device kernels as fixtures, by importing
the reference implementation (read-only at /root/reference/pkg/src).

Run once in the build container (the reference does not exist on the GPU
box; the emitted texts travel instead):

    python tests/golden/make_emitted.py

For every optimisation level 1..8 of the paper's recipe
(``lf/bench/recipes.py:30-117``, built by ``build_levels``,
``lf/bench/driver.py:32-46``) and Nq in NQS, it writes
``paper_1604_08501_b200/corpus/level<L>_nq<N>.cl`` — the exact text of
``emit_source(kernel, linearize(kernel))`` (``lf/codegen.py:443-460``),
i.e. what ``loopforge build volume.f90 --emit out.cl`` produces — plus
``emitted/index.json`` with, per file, the kernel name, the launch line,
the array arguments and the logical shape each array is bound with
(``bind_state``/``adapt_array``, ``lf/bench/inputs.py:120-164``), and the
SHA-256 of the text. These are generated OUTPUTS of the reference's code
generator (like the golden vectors), consumed by the sm_100a backend for
emitted kernels (``paper_1604_08501_b200/emitted.py``) in the GPU tests and
``tools/emitted_ladder.py``.
"""

from __future__ import annotations

import hashlib
import json
import pathlib
import sys

REF = pathlib.Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))

from loopforge import kernel as kn  # noqa: E402
from loopforge.bench.driver import build_levels  # noqa: E402
from loopforge.bench.inputs import scalar_arguments  # noqa: E402
from loopforge.interp import resolve_extent  # noqa: E402
from loopforge.bench import BenchmarkConfig, make_inputs  # noqa: E402
from loopforge.codegen import emit_source  # noqa: E402
from loopforge.schedule import linearize  # noqa: E402

OUT = pathlib.Path(__file__).resolve().parents[2] / "paper_1604_08501_b200" / "corpus"
NQS = (2, 3, 4, 8)  # 2, 3, 4: the criterion-1 grid (pkg/tests/test_acceptance.py:65-83)


def main() -> None:
    OUT.mkdir(exist_ok=True)
    index = {}
    for nq in NQS:
        levels = build_levels(nq, up_to=8)
        st = make_inputs(BenchmarkConfig(nq=nq, ne=3, seed=1))
        params = scalar_arguments(st, nq, 3)
        ints = {p: v for p, v in params.items() if isinstance(v, int)}
        for lv in range(1, 9):
            (k,) = levels[lv]
            name = f"level{lv}_nq{nq}.cl"
            try:
                src = emit_source(k, linearize(k))
            except Exception as exc:  # the reference's own emission limits
                index[name] = {"nq": nq, "level": lv, "kernel": k.name,
                               "unemittable": f"{type(exc).__name__}: {exc}"}
                print(name, "UNEMITTABLE", exc)
                continue
            (OUT / name).write_text(src)
            sig = [ln for ln in src.splitlines() if ln.startswith("KERNEL void")][0]
            arrays = {}
            for a in k.args:
                if isinstance(a, kn.ScalarParam):
                    continue
                shape = [resolve_extent(s, ints) for s in a.shape]
                arrays[a.name] = shape  # bound with Ne = 3 here
            index[name] = {
                "nq": nq, "level": lv, "kernel": k.name,
                "launch": [ln for ln in src.splitlines() if ln.startswith("// launch:")][0],
                "arrays": arrays,
                "signature": sig,
                "sha256": hashlib.sha256(src.encode()).hexdigest(),
            }
            print(name, len(src), index[name]["launch"], arrays)
    (OUT / "index.json").write_text(json.dumps(index, indent=1, sort_keys=True) + "\n")


if __name__ == "__main__":
    main()
