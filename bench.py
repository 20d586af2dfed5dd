"""Benchmark of the fused DG volume kernel (BASELINE.json metric: GDOF/s and
achieved HBM GB/s, Nq=8 fp64 volume kernel, 1/2/4/8 B200).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A "step" is one launch of the fused volume kernel over all of this rank's
elements (rhsq += v). Workload: BASELINE config 2, Nq=8, Ne=32768 fp64 per
GPU (weak scaling: N GPUs hold N*32768 elements; N=8 is config 3,
Ne=262144). Inputs are the reference's ``make_inputs`` distributions
(seed 1 + rank), upcast to fp64 — synthetic data. The working set (4.56 GB
per GPU) is ~36x the 126 MB L2, so no L2 flush is needed between steps.

``--gpus N`` without a torchrun environment re-launches itself under
``torch.distributed.run --nproc-per-node N`` (one rank per GPU, NCCL); a
WORLD_SIZE that differs from --gpus is an error. Rank 0 prints one JSON
line. See DESIGN.md §4 for the fields.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import pathlib
import socket
import subprocess
import sys
import time

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "GDOF/s, Nq=8 fp64 volume kernel (grid points per second)"
UNIT = "GDOF/s"
CSRC = ROOT / "paper_1604_08501_b200" / "csrc"


def bytes_per_point(dtype_bytes: int) -> int:
    # q 8 + g 9 + Jinv 1 read, rhsq 8 read + 8 written
    return 34 * dtype_bytes


def flops_per_point(nq: int) -> int:
    # 168 + 48*Nq with FMA = 2 flops
    return 168 + 48 * nq


def measured_peaks() -> tuple[float, str]:
    p = ROOT / "MEASURED_PEAKS.json"
    try:
        doc = json.loads(p.read_text())
        return float(doc["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:  # noqa: BLE001
        return 6650.0, "fallback (B200_PROFILING.md)"


#: kernel key -> the sources whose content the committed ncu traffic belongs to
KERNEL_SOURCES = {
    "tc": ("volume_tc.cu", "lfb_common.cuh", "lfb_math.cuh"),
    "tc32": ("volume_tc32.cu", "lfb_common.cuh"),
    "tc16": ("volume_tc16.cu", "lfb_common.cuh"),
    "col": ("volume_col.cu", "lfb_common.cuh", "lfb_math.cuh"),
    "lines": ("volume_lines.cu", "lfb_common.cuh", "lfb_math.cuh"),
    "lt": ("volume_lt.cu", "lfb_common.cuh", "lfb_math.cuh", "lfb_tma.cuh"),
    "lt32": ("volume_lt32.cu", "lfb_common.cuh", "lfb_tma.cuh"),
    "ltu": ("volume_ltu.cu", "lfb_common.cuh", "lfb_tma.cuh"),
    "lo": ("volume_lo.cu", "lfb_common.cuh", "lfb_math.cuh", "lfb_tma.cuh"),
    "fused": ("volume_fused.cu", "lfb_common.cuh", "lfb_math.cuh"),
    "basic": ("volume_basic.cu", "lfb_common.cuh"),
}


def kernel_source_sha(variant: str, dtype: str, nq: int) -> str | None:
    """SHA-256 (16 hex) of the sources a (variant, dtype, Nq) kernel is built
    from — the stamp that ties a committed ncu traffic number to the code."""
    name = variant
    if variant == "tc" and dtype == "f32":
        name = "tc16" if nq >= 9 else "tc32"
    if variant == "lt" and dtype == "f32":
        name = "lt32"
    files = KERNEL_SOURCES.get(name)
    if not files:
        return None
    h = hashlib.sha256()
    for f in files:
        p = CSRC / f
        if not p.exists():
            return None
        h.update(p.read_bytes())
    return h.hexdigest()[:16]


def ncu_traffic(kernel_key: str, source_sha: str | None):
    """dram read+write bytes per launch from the committed ncu capture, if it
    was taken on the current kernel source (else None + the reason)."""
    p = ROOT / "profiles" / "ncu_traffic.json"
    try:
        rec = json.loads(p.read_text()).get(kernel_key)
    except Exception:  # noqa: BLE001
        return None, "no committed ncu capture"
    if rec is None:
        return None, "no committed ncu capture for this kernel"
    if isinstance(rec, dict):
        if rec.get("source_sha") == source_sha:
            return rec["bytes"], f"ncu capture {rec.get('file', '')} (source {source_sha})"
        return None, (f"stale: ncu capture of source {rec.get('source_sha')}, "
                      f"kernel source is now {source_sha}")
    return None, "unstamped ncu capture (kernel source unknown)"


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def workload_config(nq: int, ne: int, dtype: str, world: int) -> dict:
    """The workload description both arms print (identical dicts)."""
    total = ne * world
    label = "custom workload"
    if nq == 8 and total == 32768 and dtype == "f64":
        label = "BASELINE config 2"
    elif nq == 8 and total == 262144:
        label = "BASELINE config 3" if dtype == "f64" else "BASELINE config 4"
    elif nq == 8 and total == 32768 and dtype == "f32":
        label = "BASELINE config 4 shape at Ne=32768"
    elif nq == 4 and total == 512:
        label = "BASELINE config 1"
    return {"workload": f"{label}: Nq={nq}, {total} hex elements ({ne} per GPU x {world}), "
                        f"{dtype}, rhsq += v",
            "nq": nq, "ne_per_gpu": ne, "ne_total": total,
            "points_total": nq ** 3 * total,
            "parallelism": f"element-sharded x{world}, no data-path collective",
            "l2": f"working set {bytes_per_point(8 if dtype == 'f64' else 4) * nq ** 3 * ne / 1e9:.2f}"
                  f" GB/GPU >> 126 MB L2; no flush"}


# --------------------------------------------------------------------------
# CPU reference path: the UNMODIFIED reference (loopforge from baseline/_ref)
# when installed, else the oracle port of lf/bench/reference.py:36-69
# --------------------------------------------------------------------------

_POOL = {}


def reference_impl():
    """(kind, make_inputs, BenchmarkConfig, volume_term, description)."""
    from paper_1604_08501_b200 import driver
    try:
        ref = driver.independent_reference()
        import loopforge.bench as lb
        return ("reference", lb.make_inputs, lb.BenchmarkConfig, ref,
                "unmodified loopforge.bench.reference_volume_term "
                "(lf/bench/reference.py:36-70, pip-installed into baseline/_ref)")
    except Exception:  # noqa: BLE001
        from oracle import volterm as O
        from paper_1604_08501_b200 import BenchmarkConfig, make_inputs
        return ("port", make_inputs, BenchmarkConfig, O.reference_volume_term,
                "oracle/volterm.py port of lf/bench/reference.py:36-70 (reference not installed)")


def _pool_work(rng):
    a, b = rng
    st = _POOL["state"]
    sub = type(st)(st.q[..., a:b], st.rhsq[..., a:b], st.D, st.g[..., a:b], st.Jinv[..., a:b],
                   st.constants)
    _POOL["fn"](sub)
    return b - a


class CpuReference:
    """The reference's CPU volume term over the elements of a make_inputs
    state, sharded over all host cores (fork pool; elements are independent,
    lf/bench/reference.py:45)."""

    def __init__(self, nq: int, ne: int, cores: int | None = None, seed: int = 1):
        import multiprocessing as mp
        self.kind, make_inputs, BenchmarkConfig, fn, self.desc = reference_impl()
        self.cores = cores or host_cores()
        self.nq, self.ne = nq, ne
        _POOL["state"] = make_inputs(BenchmarkConfig(nq=nq, ne=ne, seed=seed))
        _POOL["fn"] = fn
        self.pool = mp.get_context("fork").Pool(self.cores) if self.cores > 1 else None

    def run(self, n: int) -> float:
        """Wall seconds for the first n elements."""
        n = min(n, self.ne)
        chunks = [(n * i // self.cores, n * (i + 1) // self.cores) for i in range(self.cores)]
        chunks = [c for c in chunks if c[1] > c[0]]
        t0 = time.perf_counter()
        if self.pool is None:
            for c in chunks:
                _pool_work(c)
        else:
            self.pool.map(_pool_work, chunks, chunksize=1)
        return time.perf_counter() - t0

    def close(self):
        if self.pool is not None:
            self.pool.close()
            self.pool.join()
            self.pool = None


def run_reference(args) -> None:
    """--impl reference: the reference's CPU implementation of the path on
    the host cores, on this arm's config. At N=1 every step is the FULL
    workload (Ne=32768 at Nq=8) unless K steps of it would exceed the time
    budget; at N>1 (rank 0 only) a bounded per-step sample of the N-GPU
    workload. Rate metric: cost is linear in Ne (lf/bench/reference.py:45)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    world = args.gpus
    cfg = workload_config(args.nq, args.ne, args.dtype, world)
    total = args.ne * world
    cores = host_cores()
    # calibrate the per-element cost on a small sample, then size the steps
    probe = CpuReference(args.nq, min(total, 4 * cores), cores)
    probe.run(cores)
    per_elem = probe.run(4 * cores) / (4 * cores)
    probe.close()
    budget = args.reference_budget_s
    per_step = total if per_elem * total * args.steps <= budget else \
        max(cores, int(budget / args.steps / per_elem))
    cpu = CpuReference(args.nq, per_step, cores)
    try:
        for _ in range(args.warmup):
            cpu.run(cores)  # pool warm-up: a bounded slice per warm-up step
        t = 0.0
        for _ in range(args.steps):
            t += cpu.run(per_step)
    finally:
        cpu.close()
    pts = args.nq ** 3 * per_step
    value = pts * args.steps / t / 1e9
    full = per_step == total
    sample = (f"{'full workload' if full else 'bounded sample'}: {per_step} of {total} elements "
              f"(Nq={args.nq}) per timed step; {cpu.desc}; f32 inputs, fp64 accumulation, "
              f"{cores} processes; warm-up steps time {cores} elements")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t / args.steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": args.dtype,
        "data": "synthetic (the reference's own make_inputs, seed 1)",
        "config": cfg,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": cpu.kind,
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
        "sample_elements_per_step": per_step, "full_workload_per_step": full,
    }), flush=True)


def cpu_baseline(nq: int, ne_total: int, sample: int) -> dict:
    """The reference CPU path timed on a bounded sample of this workload,
    all host cores (plus the C restatement beside it)."""
    cores = host_cores()
    n = min(ne_total, max(cores, sample))
    cpu = CpuReference(nq, n, cores)
    try:
        cpu.run(cores)  # warm the pool
        t = cpu.run(n)
    finally:
        cpu.close()
    out = {"value": nq ** 3 * n / t / 1e9, "unit": UNIT, "cores": cores, "kind": cpu.kind,
           "sample": f"{n} elements of this workload (Nq={nq}), {cpu.desc}, {cores} processes, "
                     f"{t:.2f} s wall"}
    try:
        from oracle import coracle
        from paper_1604_08501_b200 import BenchmarkConfig, make_inputs
        st = make_inputs(BenchmarkConfig(nq=nq, ne=min(ne_total, 16384), seed=1))
        qh, gh, jh, dh = coracle.to_element_batched(st)
        coracle.volume_f64_eb(nq, qh[:cores], gh[:cores], jh[:cores], dh, st.constants,
                              nthreads=cores)
        t0 = time.perf_counter()
        coracle.volume_f64_eb(nq, qh, gh, jh, dh, st.constants, nthreads=cores)
        tc = time.perf_counter() - t0
        out["c_port"] = {"value": nq ** 3 * qh.shape[0] / tc / 1e9, "cores": cores,
                         "sample": f"{qh.shape[0]} elements, C restatement "
                                   f"(oracle/volterm_oracle.c) -O2, {cores} pthreads, {tc:.2f} s"}
    except Exception as exc:  # noqa: BLE001 - the C port is an extra, not the baseline
        out["c_port"] = {"unavailable": str(exc)[:200]}
    return out


# --------------------------------------------------------------------------
# GPU path
# --------------------------------------------------------------------------

def time_launches(fn, stream, steps: int, warmup: int):
    """(total ms, mean per-launch ms) of `steps` back-to-back launches, CUDA
    events on the launching stream."""
    import torch
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for k in range(steps):
        starts[k].record(stream)
        fn()
        ends[k].record(stream)
    t1.record(stream)
    torch.cuda.synchronize()
    return t0.elapsed_time(t1), sum(s.elapsed_time(e) for s, e in zip(starts, ends)) / steps


def e2e_reference_api(nq: int, ne: int, dev, steps: int, warmup: int, seed: int,
                      chunk: int | None = None):
    """End to end through the reference's own contract
    ``reference_volume_term(state)`` (``lf/bench/reference.py:36-70``): the
    FieldState's f32 C-order host arrays (q, g, Jinv, D; element axis
    fastest, page-locked) in, the f32 C-order increment out, fp64 compute —
    one native call per step (``lfb_volume_host``, INCREMENT mode): chunked
    2-D H2D copies, on-device layout+cast, the fp64 kernel, conversion back
    and D2H, overlapped over 3 streams. Every byte crosses PCIe every step.
    Returns (seconds per step, h2d bytes, d2h bytes, launches per step)."""
    import torch
    from paper_1604_08501_b200 import BenchmarkConfig, FieldState, make_inputs
    from paper_1604_08501_b200.volume import host_pipeline, volume_host
    st = make_inputs(BenchmarkConfig(nq=nq, ne=ne, seed=seed))
    pinned = {n: torch.from_numpy(getattr(st, n)).pin_memory()
              for n in ("q", "rhsq", "D", "g", "Jinv")}
    hst = FieldState(*(pinned[n].numpy() for n in ("q", "rhsq", "D", "g", "Jinv")),
                     st.constants)
    out_t = torch.empty(st.q.shape, dtype=torch.float32).pin_memory()
    out = out_t.numpy()
    pipe = host_pipeline(nq, ne, 4, 8, dev, chunk)
    for _ in range(warmup):
        volume_host(hst, compute_dtype=np.float64, out=out, device=dev, chunk=pipe.chunk)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        volume_host(hst, compute_dtype=np.float64, out=out, device=dev, chunk=pipe.chunk)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / steps
    h2d = sum(pinned[n].numel() * pinned[n].element_size() for n in ("q", "g", "Jinv", "D"))
    d2h = out_t.numel() * out_t.element_size()
    nchunks = -(-ne // pipe.chunk)
    # per chunk: 4 layout kernels, memset, volume kernel(s); + the D transpose
    return dt, h2d, d2h, 5 * nchunks + 1, pipe.chunk


def emitted_reference_gpu(nq: int, ne: int, dev, steps: int = 20):
    """The reference's emitted level-8 kernel (paper_1604_08501_b200/corpus/, the
    text of lf/codegen.py:emit_source) compiled unchanged by NVRTC for
    sm_100a (paper_1604_08501_b200.emitted) and timed on this GPU on the
    same workload at fp32, against the hand-written fp32 kernel."""
    import torch
    from paper_1604_08501_b200 import DeviceFieldState, volume_rhs_device
    from paper_1604_08501_b200.emitted import CORPUS, EmittedKernel
    path = CORPUS / f"level8_nq{nq}.cl"
    if not path.exists():
        return None
    ds = DeviceFieldState.generate(nq, ne, seed=1, dtype=torch.float32, device=dev)
    k = EmittedKernel.from_file(path)
    b = k.bind(ds)
    s = torch.cuda.current_stream(dev)
    _, ms_ref = time_launches(lambda: k.launch(b, s), s, steps, 2)
    _, ms_ours = time_launches(lambda: volume_rhs_device(ds, stream=s), s, steps, 2)
    k.close()
    pts = nq ** 3 * ne
    return {"value": pts / (ms_ref * 1e-3) / 1e9, "unit": UNIT, "dtype": "f32",
            "ms_per_launch": ms_ref, "ours_f32_ms_per_launch": ms_ours,
            "speedup_ours_f32": ms_ref / ms_ours,
            "kernel": "reference level-8 emitted kernel fused_r_s (lf/codegen.py:443-460 "
                      "output, paper_1604_08501_b200/corpus/level8_nq8.cl) compiled unchanged by "
                      "NVRTC for sm_100a, launch Ne x (8x8) as emitted"}


def roofline_record(variant: str, nq: int, dtype: str, pts: int, launch_ms: float) -> dict:
    peak, peak_src = measured_peaks()
    nbytes = 8 if dtype == "f64" else 4
    alg = bytes_per_point(nbytes) * pts
    achieved = alg / (launch_ms * 1e-3) / 1e9
    key = f"{variant}|nq={nq}|{dtype}"
    sha = kernel_source_sha(variant, dtype, nq)
    traffic, tsrc = ncu_traffic(key, sha)
    return {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": traffic, "traffic_source": tsrc,
            "peak_source": peak_src, "algorithmic_bytes_per_launch": alg,
            "bytes_per_point": bytes_per_point(nbytes), "launch_ms": launch_ms,
            "frac_of_8tbs_nominal": achieved / 8000.0,
            "flops_per_point": flops_per_point(nq),
            "achieved_tflops": flops_per_point(nq) * pts / (launch_ms * 1e-3) / 1e12,
            "kernel": key, "kernel_source_sha": sha}


def fp32_record(nq: int, ne: int, dev, steps: int, warmup: int) -> dict:
    """BASELINE config 4's fp32 variant at config-2 size on this GPU
    (kernel-only, device inputs, tolerance 1e-5 is tested in tests/)."""
    import torch
    from paper_1604_08501_b200 import DeviceFieldState, _native, volume_rhs_device
    from paper_1604_08501_b200.telemetry import ClockSampler
    ds = DeviceFieldState.generate(nq, ne, seed=1, dtype=torch.float32, device=dev)
    s = torch.cuda.current_stream(dev)
    with ClockSampler(dev.index) as clk:
        total, launch = time_launches(lambda: volume_rhs_device(ds, stream=s), s, steps, warmup)
    pts = nq ** 3 * ne
    variant = _native.resolve_variant(4, nq)
    del ds
    torch.cuda.empty_cache()
    return {"metric": METRIC.replace("fp64", "fp32"), "value": pts / (total / steps * 1e-3) / 1e9,
            "unit": UNIT, "dtype": "f32", "steps": steps, "ms_per_step": total / steps,
            "config": workload_config(nq, ne, "f32", 1) | {"inputs": "device (Philox)"},
            "roofline": roofline_record(variant, nq, "f32", pts, launch),
            "clocks": clk.summary()}


def sweep_record(dev, dtype: str = "f64", budget_s: float = 60.0, steps: int = 5) -> dict:
    """BASELINE config 5: Nq 4..12 at ~1e8 DOF, device inputs, kernel time
    per Nq (the AUTO variant), time-boxed."""
    import torch
    from paper_1604_08501_b200 import DeviceFieldState, _native, volume_rhs_device
    nb = 8 if dtype == "f64" else 4
    dt = torch.float64 if dtype == "f64" else torch.float32
    peak, peak_src = measured_peaks()
    rows = []
    t_start = time.perf_counter()
    for nq in range(4, 13):
        if time.perf_counter() - t_start > budget_s:
            rows.append({"nq": nq, "skipped": "time box"})
            continue
        ne = int(round(1e8 / nq ** 3))
        ds = DeviceFieldState.generate(nq, ne, seed=1, dtype=dt, device=dev)
        s = torch.cuda.current_stream(dev)
        _, ms = time_launches(lambda: volume_rhs_device(ds, stream=s), s, steps, 2)
        pts = nq ** 3 * ne
        gbs = bytes_per_point(nb) * pts / (ms * 1e-3) / 1e9
        rows.append({"nq": nq, "ne": ne, "variant": _native.resolve_variant(nb, nq),
                     "ms_per_launch": round(ms, 5), "value": pts / (ms * 1e-3) / 1e9,
                     "hbm_gbs": gbs, "frac": gbs / peak})
        del ds
        torch.cuda.empty_cache()
    return {"config": f"BASELINE config 5: Nq 4..12 at ~1e8 DOF, {dtype}, device inputs "
                      f"(Philox), {steps} launches per Nq after 2 warm-up",
            "unit": UNIT, "peak": peak, "peak_source": peak_src, "rows": rows,
            "wall_s": round(time.perf_counter() - t_start, 1)}


def run_ours(args) -> None:
    import torch
    import torch.distributed as dist

    from paper_1604_08501_b200 import (BenchmarkConfig, DeviceFieldState,
                                       make_inputs, volume_rhs_device)
    from paper_1604_08501_b200 import _native
    from paper_1604_08501_b200.distributed import global_checksum, max_over_ranks
    from paper_1604_08501_b200.telemetry import ClockSampler

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; launch "
                         f"`python bench.py --gpus N` (it starts torchrun itself) or torchrun "
                         f"with --nproc-per-node equal to --gpus")
    # LFB_BENCH_SHARE_GPU=1 maps every rank to cuda:0 and uses gloo: a test
    # mode for the multi-rank code path on a single-GPU box (not a bench)
    share = os.environ.get("LFB_BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
    elif world > torch.cuda.device_count():
        raise SystemExit(f"bench.py: {world} ranks but {torch.cuda.device_count()} visible "
                         f"GPUs (LFB_BENCH_SHARE_GPU=1 shares cuda:0 as a test mode)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            if rank == 0:  # NCCL communicator lines (nranks) on rank 0's stderr
                os.environ.setdefault("NCCL_DEBUG", "INFO")
                os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
                os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
            dist.init_process_group("nccl", device_id=dev)

    dt = torch.float64 if args.dtype == "f64" else torch.float32
    nbytes = 8 if dt == torch.float64 else 4
    nq, ne = args.nq, args.ne
    if args.inputs == "host":
        state = make_inputs(BenchmarkConfig(nq=nq, ne=ne, seed=1 + rank))
        ds = DeviceFieldState.from_field_state(state, dtype=dt, device=dev)
        del state
    else:
        # device RNG: rank r holds global elements [r*ne, (r+1)*ne) of one state
        ds = DeviceFieldState.generate(nq, ne, seed=1, dtype=dt, device=dev,
                                       e_offset=rank * ne)
    variant = args.variant
    resolved = _native.resolve_variant(nbytes, nq) if variant == "auto" else variant
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if world > 1:
            if share:
                dist.barrier()
            else:
                dist.barrier(device_ids=[local])

    for _ in range(args.warmup):
        volume_rhs_device(ds, variant=variant, stream=stream)
    torch.cuda.synchronize()

    def timed_region():
        starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        with ClockSampler(local) as clk:
            barrier()
            torch.cuda.synchronize()
            t_start.record(stream)
            for k in range(args.steps):
                starts[k].record(stream)
                volume_rhs_device(ds, variant=variant, stream=stream)
                ends[k].record(stream)
            t_end.record(stream)
            torch.cuda.synchronize()
            barrier()
        total = t_start.elapsed_time(t_end)
        per_launch = sum(s.elapsed_time(e) for s, e in zip(starts, ends)) / args.steps
        return max_over_ranks(total, device=dev), per_launch, clk

    total_ms, launch_ms, clocks = timed_region()
    # a run that saw a thermal / hardware slowdown (or clocks stuck low with
    # no reason) is rejected and measured once more; sw_power_cap is kept
    rejected = None
    if max_over_ranks(float(bool(clocks.summary().get("rejecting"))), device=dev) > 0:
        rejected = {"ms_per_step": total_ms / args.steps, "clocks": clocks.summary()}
        total_ms, launch_ms, clocks = timed_region()
    launch_ms_max = max_over_ranks(launch_ms, device=dev)
    ms_per_step = total_ms / args.steps

    pts_rank = nq ** 3 * ne
    pts_total = pts_rank * world
    value = pts_total / (ms_per_step * 1e-3) / 1e9
    roofline = roofline_record(resolved, nq, args.dtype, pts_rank, launch_ms)
    roofline["launch_ms_max_over_ranks"] = launch_ms_max
    checksum = global_checksum(ds.rhsq).tolist()
    del ds
    torch.cuda.empty_cache()

    # end to end through the reference's entry point with host buffers
    e2e = None
    if not args.no_e2e:
        e2e_steps = max(1, min(args.steps, args.e2e_steps))
        barrier()
        with ClockSampler(local) as e2e_clocks:
            sec, h2d, d2h, e2e_launches, chunk = e2e_reference_api(
                nq, ne, dev, e2e_steps, 2, 1 + rank, args.e2e_chunk)
        sec = max_over_ranks(sec, device=dev)
        e2e = {"value": pts_total / sec / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "ms_per_step": sec * 1e3, "steps": e2e_steps,
               "launches_per_step": e2e_launches, "chunk_elements": chunk,
               "api": "reference_volume_term contract (lf/bench/reference.py:36-70) via "
                      "the native host pipeline lfb_volume_host: the reference's f32 "
                      "C-order FieldState arrays (page-locked) in, f32 increment out, "
                      "fp64 compute; H2D + layout + kernel + D2H overlapped over 3 "
                      "streams",
               "clocks": e2e_clocks.summary()}

    # rank 0: the reference's own best kernel (emitted level 8, compiled
    # unchanged for sm_100a) on the same GPU, the fp32 variant, the Nq sweep
    # (N=1) and the CPU reference path beside it (every N)
    emitted = fp32 = sweep = cpu = None
    if rank == 0:
        if world == 1 and not args.no_emitted and nq == 8:
            emitted = emitted_reference_gpu(nq, ne, dev)
        if world == 1 and not args.no_fp32 and args.dtype == "f64":
            fp32 = fp32_record(nq, ne, dev, args.steps, args.warmup)
        if world == 1 and not args.no_sweep:
            sweep = sweep_record(dev, "f64", args.sweep_budget_s)
        if not args.no_cpu:
            cpu = cpu_baseline(nq, ne * world, args.cpu_sample)
    barrier()

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": args.dtype,
            "data": (f"synthetic: reference make_inputs (numpy PCG64, seed 1+rank) "
                     f"upcast to {args.dtype}" if args.inputs == "host" else
                     f"synthetic: make_inputs distributions generated on the device "
                     f"(Philox, seed 1, global element offset per rank), {args.dtype}"),
            "config": workload_config(nq, ne, args.dtype, world),
            "kernel_variant": resolved,
            "shared_gpu_test_mode": share or None,
            "e2e": e2e, "roofline": roofline,
            "cpu_baseline": cpu,
            "fp32": fp32, "sweep": sweep,
            "reference_emitted_gpu": emitted,
            "clocks": clocks.summary(), "gpu_launches": args.steps,
            "rejected_first_attempt": rejected,
            "checksum": {"field_sum": checksum[:8], "field_maxabs": checksum[8:]},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_sweep(args) -> None:
    """Nq sweep at fixed ~1e8 grid points (BASELINE config 5): device
    inputs, kernel time only, one JSON line per Nq (--variant forces one)."""
    import torch
    from paper_1604_08501_b200 import DeviceFieldState, _native, volume_rhs_device
    from paper_1604_08501_b200.telemetry import ClockSampler
    torch.cuda.set_device(0)
    dt = torch.float64 if args.dtype == "f64" else torch.float32
    nbytes = 8 if dt == torch.float64 else 4
    peak, peak_src = measured_peaks()
    for nq in range(4, 13):
        ne = int(round(1e8 / nq ** 3))
        ds = DeviceFieldState.generate(nq, ne, seed=1, dtype=dt)
        variant = _native.resolve_variant(nbytes, nq)
        if args.variant != "auto" and _native.variant_available(args.variant, nbytes, nq):
            variant = args.variant
        s = torch.cuda.current_stream()
        steps = max(3, min(args.steps, 50))
        with ClockSampler(0) as clk:
            _, ms = time_launches(lambda: volume_rhs_device(ds, variant=variant), s, steps,
                                  max(args.warmup, 1))
        pts = nq ** 3 * ne
        gbs = bytes_per_point(nbytes) * pts / (ms * 1e-3) / 1e9
        print(json.dumps({"sweep": True, "metric": METRIC.replace("Nq=8", f"Nq={nq}"),
                          "nq": nq, "ne": ne, "points": pts, "dtype": args.dtype,
                          "variant": variant, "ms_per_launch": ms,
                          "value": pts / (ms * 1e-3) / 1e9, "unit": UNIT,
                          "hbm_gbs": gbs, "frac": gbs / peak, "peak": peak,
                          "peak_source": peak_src, "steps": steps,
                          "clocks": clk.summary()}), flush=True)
        del ds
        torch.cuda.empty_cache()


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch_under_torchrun(args, argv) -> int:
    """One rank per GPU: re-run this script under torch.distributed.run."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={_free_port()}", str(pathlib.Path(__file__).resolve())] + list(argv)
    return subprocess.run(cmd).returncode


def main(argv=None) -> None:
    argv = sys.argv[1:] if argv is None else list(argv)
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--nq", type=int, default=8)
    ap.add_argument("--ne", type=int, default=32768, help="elements per GPU")
    ap.add_argument("--dtype", choices=("f64", "f32"), default="f64")
    ap.add_argument("--variant", default="auto")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--e2e-chunk", type=int, default=None,
                    help="elements per host-pipeline chunk (default: volume.pipeline_chunk)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=8192,
                    help="elements in the cpu_baseline sample")
    ap.add_argument("--reference-budget-s", type=float, default=150.0,
                    help="--impl reference: wall budget of the timed steps")
    ap.add_argument("--no-emitted", action="store_true",
                    help="skip timing the reference's emitted level-8 kernel on the GPU")
    ap.add_argument("--no-fp32", action="store_true", help="skip the fp32 sub-record")
    ap.add_argument("--no-sweep", action="store_true", help="skip the config-5 sweep record")
    ap.add_argument("--sweep-budget-s", type=float, default=60.0)
    ap.add_argument("--inputs", choices=("host", "device"), default="host",
                    help="host: make_inputs (bit-identical to the reference); "
                         "device: DeviceFieldState.generate (large configs)")
    ap.add_argument("--sweep", action="store_true",
                    help="BASELINE config 5 only: Nq 4..12 at ~1e8 DOF, one line per Nq")
    args = ap.parse_args(argv)
    if args.sweep:
        return run_sweep(args)
    if args.impl == "reference":
        return run_reference(args)
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_under_torchrun(args, argv))
    run_ours(args)


if __name__ == "__main__":
    main()
