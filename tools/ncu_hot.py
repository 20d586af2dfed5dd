"""Hottest SASS instructions of one kernel in an ncu report (warp-stall
samples), with the stall reason columns that dominate each:

    python tools/ncu_hot.py gpurun_out/x.ncu-rep [N]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data = rows[2:]
ci = hdr.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_")]
tot = sum(float(r[ci] or 0) for r in data if len(r) > ci)
print(f"total samples {tot:.0f}")
data.sort(key=lambda r: -float(r[ci] or 0) if len(r) > ci else 0)
for r in data[:n]:
    s = float(r[ci] or 0)
    top = sorted(((float(r[i] or 0), hdr[i][6:]) for i in stall_cols), reverse=True)[:3]
    tops = " ".join(f"{nm}={v:.0f}" for v, nm in top if v > 0)
    print(f"{s / tot * 100:5.1f}% {r[0]:>6} {r[1][:60]:60} {tops}")
