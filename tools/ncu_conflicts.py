"""Shared-memory instructions of one kernel in an ncu report ranked by
bank-conflict (excessive) wavefronts, with their n-way and ideal counts:

    python tools/ncu_conflicts.py gpurun_out/x.ncu-rep [N]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 15
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data = rows[2:]


def col(name):
    return hdr.index(name) if name in hdr else None


ex, way = col("L1 Wavefronts Shared Excessive"), col("L1 Conflicts Shared N-Way")
tot, ideal = col("L1 Wavefronts Shared"), col("L1 Wavefronts Shared Ideal")
ai, si = col("Address"), col("Source")


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


all_ex = sum(f(r[ex]) for r in data if len(r) > ex)
all_tot = sum(f(r[tot]) for r in data if len(r) > tot)
print(f"shared wavefronts {all_tot:.3e}, excessive {all_ex:.3e} ({all_ex / max(all_tot, 1) * 100:.1f} %)")
for r in sorted(data, key=lambda r: -f(r[ex]) if len(r) > ex else 0)[:n]:
    print(f"{r[ai][-5:]}  {r[si][:58]:58s} way {r[way]:>3s}  excess {f(r[ex]):.2e}  "
          f"total {f(r[tot]):.2e}  ideal {f(r[ideal]):.2e}")
