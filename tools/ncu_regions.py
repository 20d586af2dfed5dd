"""Warp-stall samples and executed instructions of one kernel in an ncu
report, split into regions at every BAR / SYNCS / BRA-backwards marker so
the cost of each phase of a kernel is visible:

    python tools/ncu_regions.py gpurun_out/x.ncu-rep
"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source",
                      "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, data = rows[1], rows[2:]
ci = hdr.index("Warp Stall Sampling (All Samples)")
ie = hdr.index("Instructions Executed")
tot = sum(float(r[ci] or 0) for r in data)
reg_s = reg_i = 0.0
start = data[0][0]
for r in data:
    reg_s += float(r[ci] or 0)
    reg_i += float(r[ie] or 0)
    ins = r[1]
    if "BAR.SYNC" in ins or "SYNCS.PHASECHK" in ins or "EXIT" in ins:
        print(f"{start[-5:]}..{r[0][-5:]}  stall {reg_s / tot * 100:5.1f}%  inst {reg_i:12.0f}  ends at {ins.strip()[:50]}")
        reg_s = reg_i = 0.0
        start = r[0]
print(f"{start[-5:]}..end  stall {reg_s / tot * 100:5.1f}%  inst {reg_i:12.0f}")
