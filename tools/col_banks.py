"""Shared-memory bank model of the column kernel (csrc/volume_col.cu) with
scalar line accesses (odd Nq): per element field, the owners' stores into the
F_r rows / F_s rows / F_t columns and their line reads, as a function of
each tile's line stride.

    python tools/col_banks.py Nq KS BYTES          # e.g. 5 5 8 (fp64 Nq 5)

Model: 8-byte accesses are served a half-warp at a time, 4-byte ones a warp
at a time; an access costs the largest number of distinct words one of the
32 banks must deliver (at least one wavefront per 128 bytes).
"""
from __future__ import annotations

import sys


def cost_inst(addrs, nbytes):
    groups = [addrs[:16], addrs[16:]] if nbytes == 8 else [addrs]
    total = 0
    for grp in groups:
        banks, n = {}, 0
        for a in grp:
            if a is None:
                continue
            n += 1
            for w in ((2 * a, 2 * a + 1) if nbytes == 8 else (a,)):
                banks.setdefault(w % 32, set()).add(w)
        if banks:
            total += max(max(len(v) for v in banks.values()), -(-n * nbytes // 128))
    return total


def model(nq, ks, nbytes, rsr, rss, rst):
    kp = (nq + ks - 1) // ks
    tpe = nq * nq * ks
    threads = (tpe + 31) // 32 * 32
    stores = {"tr": 0, "ts": 0, "tt": 0}
    loads = {"tr": 0, "ts": 0, "tt": 0}
    for w in range(threads // 32):
        for kk in range(kp):
            st = {"tr": [], "ts": [], "tt": []}
            pts = []
            for lane in range(32):
                te = 32 * w + lane
                i, j, h = te % nq, (te // nq) % nq, te // (nq * nq)
                k = h * kp + kk
                ok = te < tpe and k < nq
                pts.append((i, j, k) if ok else None)
                st["tr"].append((k * nq + j) * rsr + i if ok else None)
                st["ts"].append((k * nq + i) * rss + j if ok else None)
                st["tt"].append((j * nq + i) * rst + k if ok else None)
            for key in st:
                stores[key] += cost_inst(st[key], nbytes)
            for n in range(nq):
                lr = [None if p is None else (p[2] * nq + p[1]) * rsr + n for p in pts]
                ls = [None if p is None else (p[2] * nq + p[0]) * rss + n for p in pts]
                lt = [None if p is None or kk else (p[1] * nq + p[0]) * rst + n for p in pts]
                loads["tr"] += cost_inst(lr, nbytes)
                loads["ts"] += cost_inst(ls, nbytes)
                loads["tt"] += cost_inst(lt, nbytes)
    return stores, loads


if __name__ == "__main__":
    nq, ks, nb = (int(x) for x in sys.argv[1:4])
    base = nq | 1
    for key, idx in (("tr", 0), ("ts", 1), ("tt", 2)):
        rows = []
        for rs in range(nq, nq + 16):
            strides = [base, base, base]
            strides[idx] = rs
            s, l = model(nq, ks, nb, *strides)
            rows.append((s[key] + l[key], rs, s[key], l[key]))
        rows.sort()
        print(f"{key}: stride {base} -> {[r for r in rows if r[1] == base][0][0]}; best "
              + ", ".join(f"stride {r[1]}: {r[0]} (stores {r[2]}, loads {r[3]})" for r in rows[:3]))
