"""Multi-process host logic on CPU (gloo, world size 2): member sharding,
gradient all-reduce for ensemble calibration (config 4) and the row-shard
halo exchange protocol (config 3).  The same torch.distributed calls run
over NCCL on GPUs."""
import os
import socket

import pytest
import torch
import torch.multiprocessing as mp

from paper_2502_18738_b200.parallel import allreduce_sum_, shard_members
from paper_2502_18738_b200.sharded import (NcclHalo, RowPartition, RowShard,
                                           exchange_halo_tensors, run_overlapped)


def test_shard_members_partition():
    for n in (1, 5, 16, 256, 257):
        for world in (1, 2, 3, 8):
            parts = [shard_members(n, r, world) for r in range(world)]
            flat = [m for p in parts for m in p]
            assert flat == list(range(n))
            assert max(map(len, parts)) - min(map(len, parts)) <= 1


def test_row_partition_tiles_and_ghosts():
    for h in (300, 1024, 16384, 33):
        for world in (1, 2, 3, 8):
            parts = [RowPartition(h, world, r) for r in range(world)]
            if parts[0].tiles < world:
                with pytest.raises(ValueError):
                    parts[0].validate()
                continue
            rows = []
            for p in parts:
                o0, o1 = p.owned_rows
                assert o0 % 32 == 0
                rows.extend(range(o0, o1))
                l0, l1 = p.local_rows
                assert l0 == o0 - 32 * p.ghost_top
                assert l1 == min(o1 + 32 * p.ghost_bottom, h) or p.ghost_bottom == 0
            assert rows == list(range(h))
            assert parts[0].ghost_top == 0 and parts[-1].ghost_bottom == 0


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.distributed.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # ensemble calibration: per-member gradients summed over all ranks
        members = shard_members(10, rank, world)
        g = torch.tensor([[float(m), 2.0 * m, -m, 0.5] for m in members],
                         dtype=torch.float64).sum(0, keepdim=True)
        allreduce_sum_(g)
        want = torch.tensor([[45.0, 90.0, -45.0, 5.0]], dtype=torch.float64)
        ok_grad = torch.equal(g, want)
        # halo exchange of two bit planes' boundary tile rows
        words = 64
        first = [torch.full((words,), 100 * rank + p, dtype=torch.int32) for p in range(2)]
        last = [torch.full((words,), 100 * rank + 10 + p, dtype=torch.int32) for p in range(2)]
        gt = [torch.zeros(words, dtype=torch.int32) for _ in range(2)] if rank > 0 else []
        gb = [torch.zeros(words, dtype=torch.int32) for _ in range(2)] if rank < world - 1 else []
        exchange_halo_tensors(rank, world, first if rank > 0 else [],
                              last if rank < world - 1 else [], gt, gb)
        ok_halo = True
        if rank > 0:
            ok_halo &= all(torch.all(gt[p] == 100 * (rank - 1) + 10 + p) for p in range(2))
        if rank < world - 1:
            ok_halo &= all(torch.all(gb[p] == 100 * (rank + 1) + p) for p in range(2))
        q.put((rank, bool(ok_grad), bool(ok_halo)))
    finally:
        torch.distributed.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_allreduce_and_halo_exchange(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert sorted(r[0] for r in res) == list(range(world))
    assert all(r[1] and r[2] for r in res), res


class _FakeBatch:
    """CPU stand-in for a shard's FireBatch: pass 2 of launch q reads the
    ghost rows of the launch's input buffers and writes the boundary rows of
    its output buffers with a value naming (rank, launch, plane)."""

    def __init__(self, shard, rank):
        self.shard, self.rank = shard, rank
        self.q, self.device, self.seen = 0, torch.device("cpu"), []

    def run_pass(self, land, n, window, which, fc_shard, stream=None, attach=None):
        sh = self.shard
        if which == 1:
            self.seen.append(("interior", self.q))
            return
        p = sh.part
        self.seen.append(("ghosts", self.q,
                          [t.clone() for t in sh.ghost("top")] if p.ghost_top else [],
                          [t.clone() for t in sh.ghost("bottom")] if p.ghost_bottom else []))
        self.q += 1  # boundary()/ghost() now address this launch's output buffers
        for which_row in ("first", "last"):
            for plane, t in enumerate(sh.boundary(which_row)):
                t.fill_(1000 * self.rank + 10 * (self.q - 1) + plane)


def _schedule_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.distributed.init_process_group("gloo", rank=rank, world_size=world)
    try:
        part = RowPartition(32 * 3 * world, world, rank)
        sh = object.__new__(RowShard)  # host logic only: no device state
        sh.part, sh.land, sh.shard = part, None, None
        t0, t1 = part.owned_tiles
        sh.rows_tiles = (t1 - t0) + part.ghost_top + part.ghost_bottom
        sh.tiles_x = 2
        sh.batch = _FakeBatch(sh, rank)
        sh.batch.planes = torch.zeros((4, sh.rows_tiles * sh.tiles_x * 32), dtype=torch.int32)
        run_overlapped([sh], 5 * 4, 4, NcclHalo())
        ok = True
        launches = [e for e in sh.batch.seen if e[0] == "ghosts"]
        ok &= len(launches) == 5 and len(sh.batch.seen) == 10
        for _, lq, top, bot in launches:
            # launch lq reads the neighbours' boundary rows of launch lq - 1
            for plane, t in enumerate(top):
                want = 0 if lq == 0 else 1000 * (rank - 1) + 10 * (lq - 1) + plane
                ok &= bool(torch.all(t == want))
            for plane, t in enumerate(bot):
                want = 0 if lq == 0 else 1000 * (rank + 1) + 10 * (lq - 1) + plane
                ok &= bool(torch.all(t == want))
        q.put((rank, bool(ok)))
    finally:
        torch.distributed.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_overlapped_halo_schedule(world):
    """sharded.run_overlapped with the NCCL exchanger over gloo: every
    launch's boundary pass sees exactly the neighbours' boundary rows of the
    previous launch in its ghost rows."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_schedule_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert sorted(r[0] for r in res) == list(range(world))
    assert all(r[1] for r in res), res
