"""Static cost model (the reference's ``count_cost``, ``lf/codegen.py:116-146``)
against measured DRAM traffic on B200 — SURVEY §8(f) rank 4 / row a11.

``tests/golden/count_cost.json`` is the reference's own static count of every
optimisation level (``tests/golden/make_cost.py`` imports the reference);
``profiles/r02_cost_model.json`` is ncu's DRAM bytes of the same levels'
emitted kernels on B200 (``tools/cost_model.py``). The first tests re-assert,
on the fixture, the reference's own cost-model tests; the last ones check the
measured side against the static one."""

from __future__ import annotations

import json
import pathlib

import pytest

ROOT = pathlib.Path(__file__).resolve().parents[1]
STATIC = json.loads((ROOT / "tests/golden/count_cost.json").read_text())["levels"]
MEASURED = json.loads((ROOT / "profiles/r02_cost_model.json").read_text())["rows"]


def rep(nq, ne, lv):
    return STATIC[f"{nq}_{ne}_{lv}"]


def test_q_read_once_from_level_six():
    # pkg/tests/test_bench.py:173-181
    nq, ne = 2, 5
    for lv in (6, 7, 8):
        assert rep(nq, ne, lv)["per_array"]["q"]["read"] == 4 * nq ** 3 * 8 * ne, lv


def test_rhsq_traffic_ratio_level1_vs_level7():
    # pkg/tests/test_bench.py:184-198
    nq, ne = 2, 3
    t = {lv: rep(nq, ne, lv)["per_array"]["rhsq"]["read"]
         + rep(nq, ne, lv)["per_array"]["rhsq"]["written"] for lv in (1, 7)}
    elements = nq ** 3 * 8 * ne
    assert t[1] == 4 * elements * 2 * (3 * nq)
    assert t[7] == 4 * elements * 2


def test_level8_paper_size_bands():
    # pkg/tests/test_acceptance.py:111-133 (criteria 3 and 4)
    r = rep(8, 6912, 8)
    pts = 8 ** 3 * 6912
    assert 0.8 <= r["flops"] / 1.111e9 <= 1.2
    total = r["bytes_read"] + r["bytes_written"]
    assert 4.3e8 <= total <= 6.5e8
    pa = r["per_array"]
    assert pa["q"]["read"] == 4 * 8 * pts and pa["q"]["written"] == 0
    assert pa["rhsq"]["read"] == 4 * 8 * pts and pa["rhsq"]["written"] == 4 * 8 * pts
    rest = {n: v["read"] + v["written"] for n, v in pa.items() if n not in ("q", "rhsq")}
    assert max(rest, key=rest.get) == "g"
    # the static model counts Jinv inside the field loop: 8 reads per point
    assert pa["Jinv"]["read"] == 4 * 8 * pts


def test_measured_dram_never_exceeds_the_no_cache_count():
    """Caches only remove traffic: every emitted level's DRAM bytes are at
    most its static (no-cache) count; the hand-written kernels stay at the
    algorithmic minimum (136 / 272 B/pt) within a few percent."""
    by = {r["kernel"]: r for r in MEASURED}
    measured_levels = [lv for lv in range(1, 9) if "dram_bytes_per_point" in by[f"level{lv}"]]
    assert measured_levels == [1, 2, 3, 4, 5, 6, 8]  # level 7: the reference cannot emit it
    for lv in measured_levels:
        r = by[f"level{lv}"]
        assert r["dram_bytes_per_point"] <= 1.02 * r["static_bytes_per_point"], lv
        # DRAM traffic of a correct kernel is bounded below by the algorithmic
        # bytes, less what the cold single launch found already in L2
        assert r["dram_bytes_per_point"] >= 0.85 * 136, lv
    # levels 1-6 re-read through caches: static over-counts by >= 15x
    for lv in (1, 2, 3, 4, 5, 6):
        assert by[f"level{lv}"]["dram_over_static"] < 1 / 15
    # level 8: the static count's only excess is the 7 redundant Jinv reads
    # per point (28 B) + D; DRAM sees the algorithmic bytes
    l8 = by["level8"]
    assert l8["static_bytes_per_point"] == pytest.approx(136 + 28 + 0.5, abs=0.6)
    for name, alg in (("ours_f32", 136), ("ours_f64", 272)):
        assert by[name]["dram_bytes_per_point"] <= 1.02 * alg
