"""The paper's Table 1 structure on B200: the reference's own emitted kernel
for every optimisation level (paper_1604_08501_b200/corpus/, compiled unchanged for
sm_100a by paper_1604_08501_b200.emitted) timed next to this package's
hand-written kernels, on BASELINE config 2 (Nq=8, Ne=32768) in fp32 — the
precision the emitted kernels are written in (lf/interp.py:71-72).

    python tools/emitted_ladder.py [--ne 32768] [--steps 20]

One JSON line per kernel: ms per launch (CUDA events), GDOF/s, HBM GB/s at
the 136 B/pt algorithmic minimum, and the per-field max-norm error against
the fp64 tc kernel on the same inputs.
"""

from __future__ import annotations

import argparse
import json
import pathlib
import sys

import torch

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_1604_08501_b200 import DeviceFieldState, volume_rhs_device  # noqa: E402
from paper_1604_08501_b200.emitted import EmittedKernel  # noqa: E402

EMITTED = ROOT / "paper_1604_08501_b200" / "corpus"


def rel_err(got: torch.Tensor, want: torch.Tensor) -> float:
    """Per-field max-norm relative error (lf/bench/driver.py:72-91), on device."""
    g = got.double().transpose(0, 1).reshape(8, -1)
    w = want.double().transpose(0, 1).reshape(8, -1)
    num = (g - w).abs().amax(dim=1)
    den = w.abs().amax(dim=1).clamp_min(1e-300)
    return float((num / den).max())


def timed(fn, steps: int, warmup: int = 2) -> float:
    for _ in range(warmup):
        fn()
    s = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(s)
    for _ in range(steps):
        fn()
    b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / steps


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--nq", type=int, default=8)
    ap.add_argument("--ne", type=int, default=32768)
    ap.add_argument("--steps", type=int, default=20)
    args = ap.parse_args()
    nq, ne = args.nq, args.ne
    torch.cuda.set_device(0)
    pts = nq ** 3 * ne
    index = json.loads((EMITTED / "index.json").read_text())

    ref = DeviceFieldState.generate(nq, ne, seed=1, dtype=torch.float64)
    volume_rhs_device(ref, variant="tc" if nq <= 8 else "auto")
    want = ref.rhsq.clone()
    ds = DeviceFieldState.generate(nq, ne, seed=1, dtype=torch.float32)

    def line(kernel, ms, err, **kw):
        print(json.dumps({"kernel": kernel, "nq": nq, "ne": ne, "dtype": "f32",
                          "ms_per_launch": ms, "gdofs": pts / (ms * 1e-3) / 1e9,
                          "hbm_gbs_alg": 136 * pts / (ms * 1e-3) / 1e9,
                          "err_vs_tc_f64": err, **kw}), flush=True)

    for lv in range(1, 9):
        name = f"level{lv}_nq{nq}.cl"
        meta = index.get(name)
        if meta is None:
            continue
        if "unemittable" in meta:
            print(json.dumps({"kernel": f"reference level {lv} (emitted)", "nq": nq,
                              "unemittable": meta["unemittable"]}), flush=True)
            continue
        k = EmittedKernel.from_file(EMITTED / name)
        ds.rhsq.zero_()
        b = k.bind(ds)
        k.launch(b)
        k.unbind(b, ds)
        torch.cuda.synchronize()
        err = rel_err(ds.rhsq, want)
        ms = timed(lambda: k.launch(b), args.steps)
        line(f"reference level {lv} (emitted, NVRTC sm_100a)", ms, err,
             layout="interleaved vec4f" if k.interleaved else "element-batched")
        del b
        k.close()

    for variant in ("basic", "fused", "col", "tc"):
        ds.rhsq.zero_()
        try:
            volume_rhs_device(ds, variant=variant)
        except Exception as exc:  # noqa: BLE001 - variant not available for this Nq
            print(json.dumps({"kernel": f"ours {variant}", "skipped": str(exc)}))
            continue
        torch.cuda.synchronize()
        err = rel_err(ds.rhsq, want)
        ms = timed(lambda: volume_rhs_device(ds, variant=variant), max(args.steps, 50))
        line(f"ours {variant}", ms, err)


if __name__ == "__main__":
    main()
