"""Shared-memory bank model of the tcgen05 line-GEMM kernel's operand stores
(csrc/volume_ltu.cu): wavefronts per element field of the split-flux stores
into the three K-major operand tiles, for the store rotations the kernel can
use (lane group g(lane) stores its point (s + g) mod P in store s).

    python tools/ltu_banks.py [Nq ...]

Model: 32 banks x 4 bytes, one 32-bit store per lane; a warp-wide store costs
the largest number of distinct words one bank must take. Layout: core
matrices of 8 rows x 16 bytes, K-adjacent ones 128 B apart, 8-row groups
768 B apart (K = 24).
"""
from __future__ import annotations

import sys

P_OF = {9: 3, 10: 4, 11: 6}  # LtuCfg::P
GROUPS = {"none": lambda l: 0, "g8": lambda l: l >> 3, "g16": lambda l: l >> 4,
          "g4": lambda l: (l >> 2) & 3, "g2": lambda l: (l >> 1) & 3, "g1": lambda l: l & 3}


def off(row, k):
    return ((row >> 3) * 768 + (k >> 2) * 128 + (row & 7) * 16 + (k & 3) * 4) // 4


def wavefronts(addrs):
    banks = {}
    for a in addrs:
        banks.setdefault(a % 32, set()).add(a)
    return max((len(v) for v in banks.values()), default=0)


def direction_cost(nq, d, group):
    p = P_OF[nq]
    npt = nq ** 3
    threads = ((npt + p - 1) // p + 31) // 32 * 32
    total = 0
    for w in range(threads // 32):
        for s in range(p):
            addrs = []
            for lane in range(32):
                pt = 32 * w + lane + ((s + group(lane)) % p) * threads
                if pt >= npt:
                    continue
                i, j, k = pt % nq, (pt // nq) % nq, pt // (nq * nq)
                row, kk = ((k * nq + j, i), (k * nq + i, j), (j * nq + i, k))[d]
                addrs.append(off(row, kk))
            total += wavefronts(addrs)
    return total


if __name__ == "__main__":
    for nq in [int(x) for x in sys.argv[1:]] or sorted(P_OF):
        plain = [direction_cost(nq, d, GROUPS["none"]) for d in range(3)]
        best = [min((direction_cost(nq, d, f), name) for name, f in GROUPS.items())
                for d in range(3)]
        print(f"Nq={nq} P={P_OF[nq]}: plain R/S/T {plain} = {sum(plain)}; best "
              + ", ".join(f"{'RST'[d]} {c} ({n})" for d, (c, n) in enumerate(best))
              + f" = {sum(c for c, _ in best)}")
