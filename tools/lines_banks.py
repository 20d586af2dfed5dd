"""Shared-memory bank model of the `lines` kernel (csrc/volume_lines.cu) for
one element field: the owners' flux stores / write-back reads (three line
layouts), the B-fragment reads of the flux tiles and the C-fragment writes of
the accumulator tiles, as a function of the line stride LS (doubles).

    python tools/lines_banks.py Nq [LS ...]

Model: 64-bit accesses are served a half-warp at a time; a half-warp costs
the largest number of distinct words one of the 32 banks must deliver (at
least one wavefront per 128 bytes).
"""
from __future__ import annotations

import sys


def half_cost(dwords):
    banks = {}
    for d in dwords:
        for w in (2 * d, 2 * d + 1):
            banks.setdefault(w % 32, set()).add(w)
    return max([len(v) for v in banks.values()] + [-(-len(dwords) * 8 // 128)]) if banks else 0


def inst(addrs):
    return sum(half_cost([a for a in addrs[16 * h:16 * h + 16] if a is not None]) for h in range(2))


def model(nq, ls, threads=256):
    npt, nl = nq ** 3, nq * nq
    mt, ks, lt = (nq + 7) // 8, (nq + 3) // 4, (nq * nq + 7) // 8
    owner = 0
    for w in range(threads // 32):
        for m in range((npt + threads - 1) // threads):
            for kind in range(3):
                addrs = []
                for lane in range(32):
                    pt = 32 * w + lane + m * threads
                    if pt >= npt:
                        addrs.append(None)
                        continue
                    i, j, k = pt % nq, (pt // nq) % nq, pt // (nq * nq)
                    line, pos = ((k * nq + j, i), (k * nq + i, j), (j * nq + i, k))[kind]
                    addrs.append(line * ls + pos)
                owner += inst(addrs)
    bload = cstore = 0
    for t in range(lt):
        for s in range(ks):
            bload += inst([(8 * t + (l >> 2)) * ls + 4 * s + (l & 3)
                           if 8 * t + (l >> 2) < nl and 4 * s + (l & 3) < nq else None
                           for l in range(32)])
        for m in range(mt):
            for h in range(2):
                cstore += inst([(8 * t + 2 * (l & 3) + h) * ls + 8 * m + (l >> 2)
                                if 8 * t + 2 * (l & 3) + h < nl and 8 * m + (l >> 2) < nq
                                else None for l in range(32)])
    return owner, bload, cstore


if __name__ == "__main__":
    nq = int(sys.argv[1])
    for ls in [int(x) for x in sys.argv[2:]] or range(nq, nq + 8):
        o, b, c = model(nq, ls)
        print(f"Nq={nq} LS={ls}: owner {o}, B reads {b}, C writes {c} -> flux tiles {o + b}, "
              f"accumulator tiles {o + c}")
