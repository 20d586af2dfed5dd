"""Shared-memory bank model of the line-tile kernel's exchange tiles
(csrc/volume_lt.cu): wavefronts of every access pattern vs the ideal count,
for a row stride RS and the XOR swizzle of 16-byte units by row.

    python tools/lt_banks.py [Nq ...]

Model: 32 banks x 4 bytes; 64-bit accesses are served a half-warp at a time,
128-bit ones a quarter-warp at a time; within a group the wavefront count is
the largest number of distinct words one bank must deliver (at least the
ideal bytes / 128).
"""
from __future__ import annotations

import sys


def group_wavefronts(addrs, width):
    words = {}
    n = 0
    for a in addrs:
        if a is None:
            continue
        n += 1
        for d in range(width):
            for h in range(2):
                w = 2 * (a + d) + h
                words.setdefault(w % 32, set()).add(w)
    if n == 0:
        return 0
    return max([len(v) for v in words.values()] + [-(-n * width * 8 // 128)])


def wavefronts(addrs, width):
    g = 16 if width == 1 else 8
    return sum(group_wavefronts(addrs[i:i + g], width) for i in range(0, 32, g))


def ideal(addrs, width):
    return -(-sum(a is not None for a in addrs) * width * 8 // 128)


def swz(n):
    return 4 * (n & 1) + 2 * ((n >> 1) & 1)


def geometry(nq):
    ks = (nq + 3) // 4
    lp = 4 * ks
    lpj = nq + (nq & 1)
    nt = -(-nq * lp // 8)
    rs = (nt * 8 + 15) // 16 * 16
    return ks, lp, lpj, nt, rs


def pos(rs, n, x):
    u = x >> 1
    return n * rs + 2 * ((u & ~7) | ((u ^ swz(n)) & 7)) + (x & 1)


def model(nq):
    """{access kind: (wavefronts, ideal)} for one element and one field."""
    ks, lp, lpj, nt, rs = geometry(nq)
    out = {}

    def add(key, a, width):
        w, i = out.get(key, (0, 0))
        out[key] = (w + wavefronts(a, width), i + ideal(a, width))

    for which in "ST":
        for tile in range(nt):  # GEMM B-fragment reads and C-fragment pair writes
            for t in range(ks):
                add(which + " B read", [pos(rs, 4 * t + c, 8 * tile + g) if 4 * t + c < nq else None
                                        for g in range(8) for c in range(4)], 1)
            for mt in range((nq + 7) // 8):
                add(which + " C write", [pos(rs, 8 * mt + g, 8 * tile + 2 * c)
                                         if 8 * mt + g < nq else None
                                         for g in range(8) for c in range(4)], 2)
        nl = nq * lpj
        for w in range(-(-nl // 8)):  # point owners: F write / C read
            for t in range(ks):
                a = []
                for g in range(8):
                    for c in range(4):
                        L = 8 * w + g
                        j, k = L % lpj, L // lpj
                        ok = L < nl and j < nq and 4 * t + c < nq
                        n, x = (j, k * lp + 4 * t + c) if which == "S" else (k, j * lp + 4 * t + c)
                        a.append(pos(rs, n, x) if ok else None)
                add(which + " owner", a, 1)
    return out


if __name__ == "__main__":
    for nq in [int(x) for x in sys.argv[1:]] or range(5, 13):
        m = model(nq)
        w = sum(v[0] for v in m.values())
        i = sum(v[1] for v in m.values())
        print(f"Nq={nq:2d} RS={geometry(nq)[4]:3d}: {w} wavefronts / {i} ideal "
              f"(+{(w - i) / i * 100:.0f}%)  " +
              ", ".join(f"{k} {v[0]}/{v[1]}" for k, v in m.items() if v[0] != v[1]))
