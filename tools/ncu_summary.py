"""Summarise an ``ncu --set full`` report (or a launch-list CSV) into the
numbers the bench's roofline and DESIGN.md quote.

    python tools/ncu_summary.py gpurun_out/r2_fused.ncu-rep --points 16777216 \
        --bytes-per-point 272 --key fused|nq=8|f64 --out profiles/r01_fused_nq8_f64.json
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import pathlib
import subprocess

METRICS = {
    "duration_ms": ("gpu__time_duration.sum", 1.0),
    "dram_read_bytes": ("dram__bytes_read.sum", None),
    "dram_write_bytes": ("dram__bytes_write.sum", None),
    "dram_throughput_pct": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    "fp64_pipe_pct": ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 1.0),
    "dmma_cycles": ("smsp__pipe_tensor_subpipe_dmma_cycles_active.avg", 1.0),
    "smem_wavefronts": ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", 1.0),
    "smem_wavefronts_pct": ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", 1.0),
    "smem_bank_conflicts": ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", 1.0),
    "registers_per_thread": ("launch__registers_per_thread", 1.0),
    "achieved_occupancy_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1.0),
    "issue_active_pct": ("smsp__issue_active.avg.pct_of_peak_sustained_active", 1.0),
    "l2_hit_rate_pct": ("lts__t_sector_hit_rate.pct", 1.0),
    "sm_clock_ghz": ("smsp__cycles_elapsed.avg.per_second", 1.0),
    "grid_size": ("launch__grid_size", 1.0),
    "block_size": ("launch__block_size", 1.0),
}

_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
          "ms": 1, "us": 1e-3, "usecond": 1e-3, "msecond": 1, "ns": 1e-6,
          "nsecond": 1e-6, "s": 1e3, "second": 1e3}


def raw_rows(rep: pathlib.Path):
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"],
                         check=True, capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [dict(zip(hdr, zip(units, r))) for r in rows[2:]]


def number(unit: str, value: str, want_bytes: bool, want_ms: bool) -> float:
    v = float(value.replace(",", ""))
    if want_bytes:
        return v * _SCALE.get(unit, 1)
    if want_ms:
        return v * _SCALE.get(unit, 1)
    return v


def summarise(rep: pathlib.Path, points: int | None, bpp: float | None):
    kernels = []
    for row in raw_rows(rep):
        name = row.get("Kernel Name", ("", ""))[1]
        k = {"kernel": name}
        for key, (metric, _) in METRICS.items():
            if metric in row:
                unit, val = row[metric]
                try:
                    k[key] = number(unit, val, key.endswith("bytes"),
                                    key == "duration_ms")
                except ValueError:
                    continue
        if "dram_read_bytes" in k and "dram_write_bytes" in k:
            k["dram_traffic_bytes"] = k["dram_read_bytes"] + k["dram_write_bytes"]
            if k.get("duration_ms"):
                k["dram_gbs"] = k["dram_traffic_bytes"] / (k["duration_ms"] * 1e-3) / 1e9
        if points and bpp:
            k["algorithmic_bytes"] = points * bpp
            if "dram_traffic_bytes" in k:
                k["traffic_over_algorithmic"] = k["dram_traffic_bytes"] / k["algorithmic_bytes"]
        kernels.append(k)
    return kernels


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--points", type=int)
    ap.add_argument("--bytes-per-point", type=float)
    ap.add_argument("--key", help="bench roofline key, e.g. fused|nq=8|f64")
    ap.add_argument("--out")
    ap.add_argument("--traffic-json", default="profiles/ncu_traffic.json")
    args = ap.parse_args()
    ks = summarise(pathlib.Path(args.report), args.points, args.bytes_per_point)
    text = json.dumps(ks, indent=1)
    print(text)
    if args.out:
        pathlib.Path(args.out).write_text(text + "\n")
    if args.key and ks and "dram_traffic_bytes" in ks[-1]:
        # stamped with the kernel's source hash: bench.py reports the number
        # only while the kernel source is unchanged
        import sys
        sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
        from bench import kernel_source_sha
        variant, nq, dtype = args.key.split("|")
        p = pathlib.Path(args.traffic_json)
        doc = json.loads(p.read_text()) if p.exists() else {}
        doc[args.key] = {"bytes": ks[-1]["dram_traffic_bytes"],
                         "source_sha": kernel_source_sha(variant, dtype, int(nq.split("=")[1])),
                         "file": args.out or args.report}
        p.write_text(json.dumps(doc, indent=1, sort_keys=True) + "\n")


if __name__ == "__main__":
    main()
