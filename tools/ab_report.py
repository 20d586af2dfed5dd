"""Summarise A/B bench outputs: python tools/ab_report.py gpurun_out/TAG"""
import json, statistics, sys
tag = sys.argv[1]
for suffix in ("A", "B", "A_c3", "B_c3"):
    vals = []
    try:
        for l in open(f"{tag}_{suffix}.txt"):
            if l.startswith("{"):
                d = json.loads(l)
                vals.append((d["value"], d["clocks"].get("sm_mhz"), tuple(d["clocks"].get("reasons", []))))
    except FileNotFoundError:
        continue
    if vals:
        print(suffix, "median", round(statistics.median(v[0] for v in vals), 3),
              [(round(v, 2), c, r) for v, c, r in vals])
