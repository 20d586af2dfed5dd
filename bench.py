"""Benchmark of the fused DG volume kernel (BASELINE.json metric: GDOF/s and
achieved HBM GB/s, Nq=8 fp64 volume kernel, 1/2/4/8 B200).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A "step" is one launch of the fused volume kernel over all of this rank's
elements (rhsq += v). Workload: BASELINE config 2, Nq=8, Ne=32768 fp64 per
GPU (weak scaling: N GPUs hold N*32768 elements; N=8 is config 3,
Ne=262144). Inputs are the reference's ``make_inputs`` distributions
(seed 1 + rank), upcast to fp64 — synthetic data. The working set (4.56 GB
per GPU) is ~36x the 126 MB L2, so no L2 flush is needed between steps.

Rank 0 prints one JSON line. See DESIGN.md §Measurement for the fields.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import pathlib
import sys
import time

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "GDOF/s, Nq=8 fp64 volume kernel (grid points per second)"
UNIT = "GDOF/s"


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


def ncu_traffic(kernel_key: str):
    """dram read+write bytes per launch from the committed ncu summary."""
    p = ROOT / "profiles" / "ncu_traffic.json"
    try:
        return json.loads(p.read_text()).get(kernel_key)
    except Exception:  # noqa: BLE001
        return None


# --------------------------------------------------------------------------
# CPU reference path (the oracle port of lf/bench/reference.py:36-69)
# --------------------------------------------------------------------------

_POOL_STATE = None


def _pool_work(rng):
    from oracle import volterm as O
    a, b = rng
    O.volume_term_f64(_POOL_STATE, elements=range(a, b))
    return b - a


def cpu_reference_time(state, n_elements: int, cores: int, pool=None):
    """Wall time of the reference's per-element numpy algorithm over the
    first ``n_elements`` elements, sharded over ``cores`` processes."""
    global _POOL_STATE
    _POOL_STATE = state
    chunks = [(n_elements * i // cores, n_elements * (i + 1) // cores)
              for i in range(cores)]
    chunks = [c for c in chunks if c[1] > c[0]]
    t0 = time.perf_counter()
    if pool is None:
        for c in chunks:
            _pool_work(c)
    else:
        pool.map(_pool_work, chunks, chunksize=1)
    return time.perf_counter() - t0


def make_pool(cores: int, state):
    """Fork the worker pool AFTER publishing ``state`` (copy-on-write)."""
    global _POOL_STATE
    import multiprocessing as mp
    _POOL_STATE = state
    if cores <= 1:
        return None
    return mp.get_context("fork").Pool(cores)


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def run_reference(args) -> None:
    """--impl reference: the reference's CPU path (oracle port, all host
    cores) on the same workload config, bounded samples per step."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_1604_08501_b200 import BenchmarkConfig, make_inputs
    cores = host_cores()
    # ~2.2 ms per element per core at Nq=8; keep the whole
    # run near 2 minutes of wall time whatever K and W are
    per_elem = 2.2e-3 * (args.nq / 8) ** 3 if args.nq > 8 else 2.2e-3
    budget_s = 120.0
    per_step = int(budget_s / max(1, args.steps + args.warmup) / per_elem) * cores
    per_step = max(cores, min(per_step, 64 * cores, args.ne))
    state = make_inputs(BenchmarkConfig(nq=args.nq, ne=per_step, seed=1))
    pool = make_pool(cores, state)
    try:
        for _ in range(args.warmup):
            cpu_reference_time(state, per_step, cores, pool)
        t = 0.0
        for _ in range(args.steps):
            t += cpu_reference_time(state, per_step, cores, pool)
    finally:
        if pool is not None:
            pool.close()
            pool.join()
    pts = args.nq ** 3 * per_step
    value = pts * args.steps / t / 1e9
    sample = (f"{per_step} elements (Nq={args.nq}) per step, reference "
              f"per-element numpy algorithm (oracle/volterm.py port of "
              f"lf/bench/reference.py:36-69), fp64, {cores} processes")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t / args.steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": args.dtype,
        "data": "synthetic (make_inputs distributions, seed 1)",
        "config": {"workload": f"Nq={args.nq} volume term, sample of "
                               f"{per_step} elements per step",
                   "nq": args.nq, "ne_per_gpu": args.ne},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores,
                         "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }), flush=True)


# --------------------------------------------------------------------------
# GPU path
# --------------------------------------------------------------------------

def e2e_run(ds, host, steps: int, warmup: int, chunks: int, variant: str):
    """End to end through the public API with pinned HOST buffers: every
    step copies q, g, Jinv, rhsq host->device, runs the kernel and reads
    rhsq back, chunked over elements on two streams so copies overlap the
    kernel. Returns (seconds per step, h2d bytes, d2h bytes, launches)."""
    import torch
    from paper_1604_08501_b200 import volume_rhs_device
    from paper_1604_08501_b200.distributed import shard_range
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    ne = ds.ne
    ranges = [shard_range(ne, c, chunks) for c in range(chunks)]
    launches = 0

    def one_step():
        nonlocal launches
        for c, (a, b) in enumerate(ranges):
            s = streams[c % 2]
            with torch.cuda.stream(s):
                for name in ("q", "g", "Jinv", "rhsq"):
                    getattr(ds, name)[a:b].copy_(host[name][a:b], non_blocking=True)
                volume_rhs_device(ds.shard(a, b), variant=variant, stream=s)
                launches += 1
                host["out"][a:b].copy_(ds.rhsq[a:b], non_blocking=True)
        for s in streams:
            s.synchronize()

    for _ in range(warmup):
        one_step()
    torch.cuda.synchronize()
    launches = 0
    t0 = time.perf_counter()
    for _ in range(steps):
        one_step()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / steps
    h2d = sum(host[n].numel() * host[n].element_size() for n in ("q", "g", "Jinv", "rhsq"))
    d2h = host["out"].numel() * host["out"].element_size()
    return dt, h2d, d2h, launches


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
    from paper_1604_08501_b200.emitted import EmittedKernel
    from paper_1604_08501_b200.emitted import CORPUS
    path = CORPUS / f"level8_nq{nq}.cl"
    if not path.exists():
        return None
    ds = DeviceFieldState.generate(nq, ne, seed=1, dtype=torch.float32, device=dev)
    k = EmittedKernel.from_file(path)
    b = k.bind(ds)
    s = torch.cuda.current_stream(dev)

    def t(fn):
        for _ in range(2):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(s)
        for _ in range(steps):
            fn()
        e1.record(s)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / steps

    ms_ref = t(lambda: k.launch(b, s))
    ms_ours = t(lambda: volume_rhs_device(ds, stream=s))
    k.close()
    pts = nq ** 3 * ne
    return {"value": pts / (ms_ref * 1e-3) / 1e9, "unit": UNIT, "dtype": "f32",
            "ms_per_launch": ms_ref, "ours_f32_ms_per_launch": ms_ours,
            "speedup_ours_f32": ms_ref / ms_ours,
            "kernel": "reference level-8 emitted kernel fused_r_s (lf/codegen.py:443-460 "
                      "output, paper_1604_08501_b200/corpus/level8_nq8.cl) compiled unchanged by "
                      "NVRTC for sm_100a, launch Ne x (8x8) as emitted"}


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
    # LFB_BENCH_SHARE_GPU=1 maps every rank to cuda:0 and uses gloo: a test
    # mode for the multi-rank code path on a single-GPU box (not a bench)
    share = os.environ.get("LFB_BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    dt = torch.float64 if args.dtype == "f64" else torch.float32
    nbytes = 8 if dt == torch.float64 else 4
    nq, ne = args.nq, args.ne
    if args.inputs == "host":
        state = make_inputs(BenchmarkConfig(nq=nq, ne=ne, seed=1 + rank))
        ds = DeviceFieldState.from_field_state(state, dtype=dt, device=dev)
    else:
        # device RNG: rank r holds global elements [r*ne, (r+1)*ne) of one state
        state = None
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
    peak, peak_src = measured_peaks()
    alg_bytes = bytes_per_point(nbytes) * pts_rank
    achieved = alg_bytes / (launch_ms * 1e-3) / 1e9
    kernel_key = f"{resolved}|nq={nq}|{args.dtype}"
    traffic = ncu_traffic(kernel_key)
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak,
                "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "peak_source": peak_src,
                "algorithmic_bytes_per_launch": alg_bytes,
                "bytes_per_point": bytes_per_point(nbytes),
                "launch_ms": launch_ms, "launch_ms_max_over_ranks": launch_ms_max,
                "frac_of_8tbs_nominal": achieved / 8000.0,
                "flops_per_point": flops_per_point(nq),
                "achieved_tflops": flops_per_point(nq) * pts_rank / (launch_ms * 1e-3) / 1e12,
                "kernel": kernel_key}

    # end to end through the reference's entry point with host buffers
    e2e = None
    e2e_eb = None
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
        if args.e2e_element_batched:
            host = {n: getattr(ds, n).cpu().pin_memory() for n in ("q", "g", "Jinv", "rhsq")}
            host["out"] = torch.empty_like(host["rhsq"]).pin_memory()
            barrier()
            sec, h2d, d2h, e2e_launches = e2e_run(ds, host, e2e_steps, 1, 8, variant)
            sec = max_over_ranks(sec, device=dev)
            e2e_eb = {"value": pts_total / sec / 1e9, "unit": UNIT,
                      "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                      "ms_per_step": sec * 1e3, "launches": e2e_launches,
                      "api": f"DeviceFieldState + volume_rhs_device over pinned host "
                             f"buffers in the element-batched {args.dtype} layout "
                             f"(rhsq += v), 8 chunks on 2 streams"}
            del host

    checksum = global_checksum(ds.rhsq).tolist()

    # the reference's own best kernel (emitted level 8, compiled unchanged
    # for sm_100a) on the same GPU — fp32, its only precision
    emitted = None
    if rank == 0 and world == 1 and not args.no_emitted and nq == 8:
        emitted = emitted_reference_gpu(nq, ne, dev)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu and state is None:
        state = make_inputs(BenchmarkConfig(
            nq=nq, ne=min(ne, args.cpu_sample_per_core * host_cores()), seed=1))
    if rank == 0 and world == 1 and not args.no_cpu:
        cores = host_cores()
        n = min(state.ne, max(cores, args.cpu_sample_per_core * cores))
        pool = make_pool(cores, state)
        try:
            cpu_reference_time(state, min(n, cores), cores, pool)  # warm pool
            t = cpu_reference_time(state, n, cores, pool)
        finally:
            if pool is not None:
                pool.close()
                pool.join()
        cpu = {"value": nq ** 3 * n / t / 1e9, "unit": UNIT, "cores": cores,
               "kind": "port",
               "sample": f"{n} elements of this workload (Nq={nq}), the "
                         f"reference's per-element numpy algorithm "
                         f"(oracle/volterm.py, port of lf/bench/reference.py:"
                         f"36-69) in {cores} processes, {t:.2f} s wall"}
        if not args.no_cpu_c:
            from oracle import coracle
            qh, gh, jh, dh = coracle.to_element_batched(
                make_inputs(BenchmarkConfig(nq=nq, ne=min(ne, 16384), seed=1)))
            nc = qh.shape[0]
            coracle.volume_f64_eb(nq, qh[:cores], gh[:cores], jh[:cores], dh,
                                  state.constants, nthreads=cores)
            t0 = time.perf_counter()
            coracle.volume_f64_eb(nq, qh, gh, jh, dh, state.constants,
                                  nthreads=cores)
            tc = time.perf_counter() - t0
            cpu["c_port"] = {"value": nq ** 3 * nc / tc / 1e9, "cores": cores,
                             "sample": f"{nc} elements, C restatement "
                                       f"(oracle/volterm_oracle.c) -O2, "
                                       f"{cores} pthreads, {tc:.2f} s"}

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
            "config": {"workload": f"BASELINE config {'2' if world == 1 else '3'}: "
                                   f"Nq={nq}, {ne} hex elements per GPU, "
                                   f"{args.dtype}, rhsq += v",
                       "nq": nq, "ne_per_gpu": ne, "ne_total": ne * world,
                       "points_total": pts_total, "variant": resolved,
                       "parallelism": f"element-sharded x{world}, no "
                                      f"data-path collective",
                       "l2": "working set "
                             f"{alg_bytes / 1e9:.2f} GB/GPU >> 126 MB L2; no flush"},
            "e2e": e2e, "e2e_element_batched": e2e_eb, "roofline": roofline,
            "reference_emitted_gpu": emitted,
            "cpu_baseline": cpu,
            "clocks": clocks.summary(), "gpu_launches": args.steps,
            "rejected_first_attempt": rejected,
            "checksum": {"field_sum": checksum[:8], "field_maxabs": checksum[8:]},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_sweep(args) -> None:
    """Nq sweep at fixed ~1e8 grid points (BASELINE config 5): device
    inputs, kernel time only, one JSON line per Nq."""
    import torch
    from paper_1604_08501_b200 import DeviceFieldState, volume_rhs_device
    from paper_1604_08501_b200 import _native
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
        for _ in range(args.warmup):
            volume_rhs_device(ds, variant=variant)
        s = torch.cuda.current_stream()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        steps = max(3, min(args.steps, 50))
        torch.cuda.synchronize()
        a.record(s)
        for _ in range(steps):
            volume_rhs_device(ds, variant=variant)
        b.record(s)
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / steps
        pts = nq ** 3 * ne
        gbs = bytes_per_point(nbytes) * pts / (ms * 1e-3) / 1e9
        print(json.dumps({"sweep": True, "metric": METRIC.replace("Nq=8", f"Nq={nq}"),
                          "nq": nq, "ne": ne, "points": pts, "dtype": args.dtype,
                          "variant": variant, "ms_per_launch": ms,
                          "value": pts / (ms * 1e-3) / 1e9, "unit": UNIT,
                          "hbm_gbs": gbs, "frac": gbs / peak, "peak": peak,
                          "peak_source": peak_src, "steps": steps}), flush=True)
        del ds
        torch.cuda.empty_cache()


def main(argv=None) -> None:
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
    ap.add_argument("--e2e-element-batched", action="store_true",
                    help="also time the fp64 element-batched host-buffer path")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-emitted", action="store_true",
                    help="skip timing the reference's emitted level-8 kernel on the GPU")
    ap.add_argument("--no-cpu-c", action="store_true")
    ap.add_argument("--cpu-sample-per-core", type=int, default=512)
    ap.add_argument("--inputs", choices=("host", "device"), default="host",
                    help="host: make_inputs (bit-identical to the reference); "
                         "device: DeviceFieldState.generate (large configs)")
    ap.add_argument("--sweep", action="store_true",
                    help="BASELINE config 5: Nq 4..12 at ~1e8 DOF, one line per Nq")
    args = ap.parse_args(argv)
    if args.sweep:
        return run_sweep(args)
    if args.warmup < 3 and args.impl == "ours":
        ap.error("--warmup must be >= 3")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
