"""The sharded volume kernel in two processes: both ranks share
cuda:0 (the GPU box has one GPU; gloo carries the checksum), each runs
``volume_rhs_device`` on its ``shard_range`` of ONE device-generated state,
and the all-reduced checksum must equal the single-process checksum of the
whole launch — bit-for-bit on the per-field max |.| and to rounding on the
per-field sums (same terms, different association). Also runs ``bench.py
--gpus 2`` end to end in the shared-GPU test mode."""

from __future__ import annotations

import json
import os
import pathlib
import socket
import subprocess
import sys

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

ROOT = pathlib.Path(__file__).resolve().parents[1]
NQ, NE, SEED = 8, 1037, 5


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank: int, world: int, port: int, q):
    sys.path.insert(0, str(ROOT))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    from paper_1604_08501_b200 import DeviceFieldState, volume_rhs_device
    from paper_1604_08501_b200.distributed import global_checksum, shard_range
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a, b = shard_range(NE, rank, world)
        ds = DeviceFieldState.generate(NQ, b - a, seed=SEED, e_offset=a)
        volume_rhs_device(ds)
        torch.cuda.synchronize()
        got = global_checksum(ds.rhsq.cpu())
        q.put((rank, got.tolist()))
    finally:
        dist.destroy_process_group()


def test_two_ranks_sharded_kernel_checksum_equals_whole(cuda_device):
    from paper_1604_08501_b200 import DeviceFieldState, volume_rhs_device
    from paper_1604_08501_b200.distributed import local_checksum
    whole = DeviceFieldState.generate(NQ, NE, seed=SEED)
    volume_rhs_device(whole)
    want = local_checksum(whole.rhsq).tolist()
    scale = float(whole.rhsq.abs().sum())
    del whole
    torch.cuda.empty_cache()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for _, got in results:
        for b in range(8):
            assert got[8 + b] == want[8 + b]  # max |.|: exact
            assert abs(got[b] - want[b]) <= 1e-15 * scale  # sums: association only


def test_bench_two_ranks_share_mode(cuda_device):
    """``python bench.py --gpus 2`` launches torchrun itself; in the shared-
    GPU test mode it prints one JSON line with n_gpus == 2."""
    env = dict(os.environ, LFB_BENCH_SHARE_GPU="1")
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--steps", "3",
                          "--warmup", "3", "--ne", "2048", "--no-e2e", "--cpu-sample", "64"],
                         env=env, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-3000:]
    doc = json.loads(lines[0])
    assert doc["n_gpus"] == 2 and doc["shared_gpu_test_mode"] is True
    assert doc["config"]["ne_total"] == 4096
    assert doc["cpu_baseline"]["cores"] >= 1


def test_bench_rejects_world_size_mismatch(cuda_device):
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--steps", "3",
                          "--warmup", "3", "--ne", "64", "--no-e2e", "--no-cpu"],
                         env=env, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode != 0 and "WORLD_SIZE" in (out.stderr + out.stdout)
