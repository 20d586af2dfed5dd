"""Host-side multi-GPU logic on CPU: element sharding and the final
checksum all-reduce, world_size 2 over gloo (the NCCL path on the GPU box
runs the same code)."""

from __future__ import annotations

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1604_08501_b200 import DeviceFieldState, PhysicalConstants
from paper_1604_08501_b200.distributed import (global_checksum, local_checksum,
                                               max_over_ranks, shard_range)


def test_shard_range_partitions_exactly():
    for ne in (0, 1, 7, 8, 32768, 262144, 1000003):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_range(ne, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == ne
            for (a0, b0), (a1, b1) in zip(spans, spans[1:]):
                assert b0 == a1
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)
    with pytest.raises(ValueError):
        shard_range(-1, 0, 1)


def test_shard_views_share_memory():
    nq, ne = 2, 6
    z = lambda *s: torch.zeros(*s, dtype=torch.float64)
    ds = DeviceFieldState(z(ne, 8, nq, nq, nq), z(ne, 8, nq, nq, nq), z(nq, nq),
                          z(ne, 3, 3, nq, nq, nq), z(ne, nq, nq, nq),
                          PhysicalConstants())
    a, b = shard_range(ne, 1, 2)
    sh = ds.shard(a, b)
    assert sh.ne == b - a and sh.q.is_contiguous() and sh.g.is_contiguous()
    sh.rhsq.fill_(3.0)
    assert float(ds.rhsq[a:b].sum()) == 3.0 * sh.rhsq.numel()
    assert float(ds.rhsq[:a].abs().sum()) == 0.0


def test_local_checksum_layout():
    x = torch.arange(2 * 8 * 8, dtype=torch.float64).reshape(2, 8, 2, 2, 2) - 50
    c = local_checksum(x)
    for b in range(8):
        assert float(c[b]) == float(x[:, b].sum())
        assert float(c[8 + b]) == float(x[:, b].abs().max())
    assert torch.equal(local_checksum(x[:0]), torch.zeros(16, dtype=torch.float64))


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank: int, world: int, port: int, ne: int, q: "mp.Queue"):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        gen = torch.Generator().manual_seed(1234)
        whole = torch.randn(ne, 8, 3, 3, 3, generator=gen, dtype=torch.float64)
        a, b = shard_range(ne, rank, world)
        mine = whole[a:b]
        got = global_checksum(mine)
        t = max_over_ranks(float(rank + 1) * 0.5)
        q.put((rank, got.tolist(), local_checksum(whole).tolist(), t))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_checksum_allreduce_over_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ne = 11
    procs = [ctx.Process(target=_worker, args=(r, world, port, ne, q))
             for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, got, want, t in results:
        # sums: same terms, different association -> tiny rounding only
        for b in range(8):
            assert got[b] == pytest.approx(want[b], rel=1e-12, abs=1e-12)
            assert got[8 + b] == want[8 + b]  # max is exact
        assert t == 0.5 * world  # max over ranks
