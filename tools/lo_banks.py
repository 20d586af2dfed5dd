"""Bank model for the line-owner kernel (csrc/volume_lo.cu): shared-memory
wavefronts per element and field of its three flux tiles, for candidate row
strides RSR / RSS / RST.

  point owners (A stores, C loads), lane = point x = i + Nq j + Nq^2 k,
  consecutive over the CTA's threads (x = tid + THREADS u):
      R[(k Nq + j) RSR + i], S[(k Nq + i) RSS + j], T[(j Nq + i) RST + k]
  line owners (B: row loads and the in-place output stores), lane = line te:
      R[te RSR + n], S[te RSS + n], T[te RST + n]     (n = 0..Nq-1)

    python tools/lo_banks.py            # best strides per (dtype, Nq)
"""


def wavefronts(addrs, width):
    """Wavefronts of one warp access; addrs in units of `width` bytes."""
    halves = [addrs] if width == 4 else [addrs[:16], addrs[16:]]
    total = 0
    for h in halves:
        banks = {}
        for a in set(h):
            for w in range(width // 4):
                banks.setdefault((a * (width // 4) + w) % 32, set()).add(a)
        total += max((len(v) for v in banks.values()), default=0)
    return total


def point_cost(nq, width, rs, kind, threads):
    npt = nq ** 3
    tot = 0
    for w0 in range(0, threads, 32):
        for u in range(0, npt, threads):
            xs = [x for x in range(u + w0, u + w0 + 32) if x < min(npt, u + threads)]
            if not xs:
                continue
            ad = []
            for x in xs:
                i, j, k = x % nq, (x // nq) % nq, x // (nq * nq)
                ad.append({"R": (k * nq + j) * rs + i, "S": (k * nq + i) * rs + j,
                           "T": (j * nq + i) * rs + k}[kind])
            tot += wavefronts(ad, width)
    return tot


def line_cost(nq, width, rs):
    tpe = nq * nq
    return sum(wavefronts([te * rs + n for te in range(w0, min(w0 + 32, tpe))], width)
               for w0 in range(0, tpe, 32) for n in range(nq))


def cost(nq, width, rs, kind, threads):
    # A stores + C loads (point owners), B loads + stores (line owners)
    return 2 * point_cost(nq, width, rs, kind, threads) + 2 * line_cost(nq, width, rs)


if __name__ == "__main__":
    for width in (4, 8):
        for nq in range(9, 13):
            threads = (nq * nq + 31) // 32 * 32
            ideal = 4 * ((nq ** 3 + 31) // 32) * (1 if width == 4 else 2)
            out = []
            for kind in "RST":
                best = min((cost(nq, width, rs, kind, threads), rs) for rs in range(nq, nq + 25))
                out.append(f"{kind} {best[1]:2d} ({best[0]}, odd {cost(nq, width, nq | 1, kind, threads)})")
            print(f"width {width} Nq {nq} (conflict-free {ideal}): " + "  ".join(out))
