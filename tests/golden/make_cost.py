"""Static cost model fixture: the reference's own ``count_cost``
(``lf/codegen.py:116-146``) of every optimisation level at the paper's
benchmark size (Nq=8, Ne=6912 — ``pkg/tests/test_acceptance.py:111-133``)
and at the reference test sizes (Nq=2, Ne=5 and 3 —
``pkg/tests/test_bench.py:173-198``), by importing the reference (read-only
at /root/reference/pkg/src). Run once in the build container:

    python tests/golden/make_cost.py      # -> tests/golden/count_cost.json

The GPU side (measured DRAM bytes of the same levels' emitted kernels on
B200) is ``tools/cost_model.py``; ``tests/test_cost_model.py`` checks both.
"""

from __future__ import annotations

import json
import pathlib
import sys

REF = pathlib.Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))

from loopforge import schedule as sch  # noqa: E402
from loopforge.bench.driver import build_levels  # noqa: E402
from loopforge.codegen import count_cost  # noqa: E402

OUT = pathlib.Path(__file__).parent / "count_cost.json"
SIZES = [(8, 6912), (2, 5), (2, 3)]


def main() -> None:
    doc = {"rule": "lf/codegen.py:116-146: every global reference x 4 bytes, += = read + write, "
                   "no cache; flops with single-level multiply-add fusion",
           "levels": {}}
    for nq, ne in SIZES:
        levels = build_levels(nq, up_to=8)
        for lv in range(1, 9):
            (k,) = levels[lv]
            rep = count_cost(k, sch.linearize(k), {"Ne": ne})
            doc["levels"][f"{nq}_{ne}_{lv}"] = {
                "nq": nq, "ne": ne, "level": lv, "flops": rep.flops,
                "bytes_read": rep.global_bytes_read, "bytes_written": rep.global_bytes_written,
                "per_array": {n: {"read": r, "written": w} for n, r, w in rep.per_array}}
            print(nq, ne, lv, rep.global_bytes_read + rep.global_bytes_written, rep.flops)
    OUT.write_text(json.dumps(doc, indent=1, sort_keys=True) + "\n")


if __name__ == "__main__":
    main()
