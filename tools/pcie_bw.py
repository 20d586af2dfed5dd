"""Raw PCIe copy bandwidth of this box (page-locked host <-> device), the
ceiling of the host-buffer e2e path: 1-D H2D, 1-D D2H, both at once, and
the 2-D strided H2D the pipeline uses (8 KB rows)."""
import json
import time

import torch

torch.cuda.set_device(0)
n = 1 << 30
h = torch.empty(n, dtype=torch.uint8).pin_memory()
h2 = torch.empty(n // 2, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n // 2, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


h2d = n / t(lambda: d.copy_(h, non_blocking=True)) / 1e9
d2h = n / t(lambda: h.copy_(d, non_blocking=True)) / 1e9


def both():
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)


tb = t(both)
# 2-D: 4096 rows x 8 KB out of rows of 64 KB (the pipeline's chunk pattern)
rows, w, pitch = 4096, 8192, 65536
hv = h[: rows * pitch].view(rows, pitch)
dv = d[: rows * w].view(rows, w)
t2 = t(lambda: dv.copy_(hv[:, :w], non_blocking=True))
print(json.dumps({"h2d_GBps": h2d, "d2h_GBps": d2h,
                  "concurrent_GBps": {"h2d": n / tb / 1e9, "d2h": (n // 2) / tb / 1e9},
                  "h2d_2d_8KB_rows_GBps": rows * w / t2 / 1e9}))
