"""Static cost model vs measured DRAM traffic.

    # on the GPU box: one launch per level under ncu (DRAM bytes per launch)
    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \\
        -k regex:"fused_r_s|volume_tc" --csv --log-file gpurun_out/cost_ncu.csv \\
        python tools/cost_model.py launch
    # here: join with the reference's static count (tests/golden/count_cost.json)
    python tools/cost_model.py table gpurun_out/cost_ncu.csv > profiles/r02_cost_model.md

``launch`` runs, at the paper's size (Nq=8, Ne=6912, f32 — the corpus's
precision), the reference's emitted kernel of every emittable level
(1-6, 8; the reference's emitter rejects level 7) once, then this package's
fp32 and fp64 AUTO kernels once, printing the launch order. ``table`` writes
the markdown table and ``profiles/r02_cost_model.json``.
"""
from __future__ import annotations

import csv
import io
import json
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
NQ, NE = 8, 6912
PTS = NQ ** 3 * NE
LEVELS = (1, 2, 3, 4, 5, 6, 8)


def launch() -> None:
    import torch
    from paper_1604_08501_b200 import DeviceFieldState, volume_rhs_device
    from paper_1604_08501_b200.driver import emitted_level
    torch.cuda.set_device(0)
    ds32 = DeviceFieldState.generate(NQ, NE, seed=1, dtype=torch.float32)
    order = []
    for lv in LEVELS:
        k = emitted_level(NQ, lv)
        b = k.bind(ds32)
        k.launch(b)
        torch.cuda.synchronize()
        order.append(f"level{lv}")
        k.close()
    volume_rhs_device(ds32)
    order.append("ours_f32")
    ds64 = DeviceFieldState.generate(NQ, NE, seed=1, dtype=torch.float64)
    volume_rhs_device(ds64)
    torch.cuda.synchronize()
    order.append("ours_f64")
    print("ORDER", json.dumps(order))


def table(csv_path: str) -> None:
    text = pathlib.Path(csv_path).read_text()
    rows = list(csv.reader(io.StringIO(text[text.index('"ID"'):])))
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    per = {}
    for r in rows[1:]:
        if len(r) < len(hdr):
            continue
        lid = int(r[ix["ID"]])
        unit, val = r[ix["Metric Unit"]], float(r[ix["Metric Value"]].replace(",", ""))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-6,
                 "usecond": 1e-3, "msecond": 1.0, "ns": 1e-6, "us": 1e-3, "ms": 1.0}.get(unit, 1)
        per.setdefault(lid, {"kernel": r[ix["Kernel Name"]]})[r[ix["Metric Name"]]] = val * scale
    launches = [per[k] for k in sorted(per)]
    names = [f"level{lv}" for lv in LEVELS] + ["ours_f32", "ours_f64"]
    assert len(launches) == len(names), (len(launches), [l["kernel"] for l in launches])
    static = json.loads((ROOT / "tests/golden/count_cost.json").read_text())["levels"]
    out = []
    print("| kernel | static B/pt (count_cost) | DRAM B/pt measured | DRAM / static | "
          "algorithmic B/pt | ms / launch | GDOF/s |")
    print("|---|---|---|---|---|---|---|")
    for lv in range(1, 9):
        st = static[f"{NQ}_{NE}_{lv}"]
        sbpt = (st["bytes_read"] + st["bytes_written"]) / PTS
        rec = {"kernel": f"level{lv}", "static_bytes_per_point": sbpt,
               "static_flops_per_point": st["flops"] / PTS}
        if f"level{lv}" in names:
            m = launches[names.index(f"level{lv}")]
            d = (m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]) / PTS
            ms = m["gpu__time_duration.sum"]
            rec.update(dram_bytes_per_point=d, dram_over_static=d / sbpt, ms=ms,
                       gdofs=PTS / ms / 1e6, ncu_kernel=m["kernel"])
            print(f"| reference level {lv} (emitted, f32) | {sbpt:.1f} | {d:.1f} | "
                  f"{d / sbpt:.2f} | 136 | {ms:.3f} | {PTS / ms / 1e6:.1f} |")
        else:
            print(f"| reference level {lv} | {sbpt:.1f} | — (not emittable by the reference) | "
                  f"— | 136 | — | — |")
        out.append(rec)
    for name, alg in (("ours_f32", 136), ("ours_f64", 272)):
        m = launches[names.index(name)]
        d = (m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]) / PTS
        ms = m["gpu__time_duration.sum"]
        out.append({"kernel": name, "dram_bytes_per_point": d, "algorithmic_bytes_per_point": alg,
                    "ms": ms, "gdofs": PTS / ms / 1e6, "ncu_kernel": m["kernel"]})
        print(f"| this package, AUTO {name[-3:]} ({m['kernel'].split('(')[0][-40:]}) | — | {d:.1f} | — | "
              f"{alg} | {ms:.3f} | {PTS / ms / 1e6:.1f} |")
    (ROOT / "profiles" / "r02_cost_model.json").write_text(json.dumps(
        {"config": f"Nq={NQ}, Ne={NE} (paper size), one launch each under ncu "
                   f"(cold-cache, serialised)", "rows": out}, indent=1) + "\n")


if __name__ == "__main__":
    if sys.argv[1] == "launch":
        launch()
    else:
        table(sys.argv[2])
