"""Row-sharded single domain (BASELINE config 3 across GPUs).

Each rank owns a band of 32-row tile rows plus one ghost tile row per
neighbour (32 rows >= the K-row halo of a K-step window).  Every window
launch is split (``fc_run_pass``): pass 1 advances the listed tiles away from
the ghost rows, pass 2 the boundary tile rows next to them.  The exchange of
launch q's boundary rows (both bit planes; NCCL send/recv over NVLink, or
device copies when several shards are emulated in one process) runs on a
communication stream while pass 1 of launch q+1 computes; only pass 2 of
q+1 waits for it.  Draws are keyed by the global row, so the sharded
trajectory is bit-identical to the unsharded one (pyrocell's own partition
invariance, kernel.py:307-309 / rng.py:64-67).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np
import torch

from . import _lib as L
from .device import DeviceLandscape, FireBatch

TILE = 32


@dataclass(frozen=True)
class RowPartition:
    """Tile-row aligned partition of H rows over `world` ranks (host logic)."""

    height: int
    world: int
    rank: int

    @property
    def tiles(self) -> int:
        return (self.height + TILE - 1) // TILE

    @property
    def owned_tiles(self):
        base, extra = divmod(self.tiles, self.world)
        t0 = self.rank * base + min(self.rank, extra)
        return t0, t0 + base + (1 if self.rank < extra else 0)

    @property
    def ghost_top(self) -> int:
        return 1 if self.rank > 0 and self.owned_tiles[1] > self.owned_tiles[0] else 0

    @property
    def ghost_bottom(self) -> int:
        return 1 if self.rank < self.world - 1 and self.owned_tiles[1] > self.owned_tiles[0] else 0

    @property
    def owned_rows(self):
        t0, t1 = self.owned_tiles
        return TILE * t0, min(TILE * t1, self.height)

    @property
    def local_rows(self):
        """Global row range of the local grid (owned rows + ghost rows)."""
        t0, t1 = self.owned_tiles
        return TILE * (t0 - self.ghost_top), min(TILE * (t1 + self.ghost_bottom), self.height)

    def validate(self):
        if self.tiles < self.world:
            raise ValueError(f"{self.height} rows ({self.tiles} tile rows) cannot be split over "
                             f"{self.world} ranks")


class RowShard:
    """One rank's part of a row-sharded domain (single member)."""

    def __init__(self, part: RowPartition, elevation, wind_speed, wind_direction, canopy, density,
                 init, *, cell_side: float = 30.0, max_steps: int = 1024,
                 with_jacobian: bool = False, device=None):
        part.validate()
        self.part = part
        r0, r1 = part.local_rows
        sl = lambda a: (a[r0:r1] if not torch.is_tensor(a) else a[r0:r1])
        self.land = DeviceLandscape.from_elevation(sl(elevation), sl(wind_speed),
                                                   sl(wind_direction), sl(canopy), sl(density),
                                                   cell_side=cell_side, device=device)
        w = self.land.shape[1]
        self.batch = FireBatch((r1 - r0, w), 1, max_steps=max_steps,
                               with_jacobian=with_jacobian, device=device)
        self.shard = L.FcShard(r0, part.ghost_top, part.ghost_bottom, 0)
        init_local = init[r0:r1]
        self.batch.reset(init_local)
        o0, o1 = part.owned_rows
        own = init_local[o0 - r0:o1 - r0]
        self.owned_init_burning = int(own.sum().item() if torch.is_tensor(own) else np.sum(own))
        self.tiles_x = self.batch.grid.tiles_x
        self.rows_tiles = self.batch.grid.tiles_y

    # ------------------------------------------------------------ planes
    def _rows(self, plane: int, tile_row: int) -> torch.Tensor:
        words = self.tiles_x * TILE
        return self.batch.planes[plane, tile_row * words:(tile_row + 1) * words]

    def boundary(self, which: str):
        """(burning, burned) words of the first/last owned tile row."""
        ty = self.part.ghost_top if which == "first" else self.rows_tiles - 1 - self.part.ghost_bottom
        return self._rows(self.batch.q & 1, ty), self._rows(2 + (self.batch.q & 1), ty)

    def ghost(self, which: str):
        """(burning, burned) words of the top/bottom ghost tile row."""
        ty = 0 if which == "top" else self.rows_tiles - 1
        return self._rows(self.batch.q & 1, ty), self._rows(2 + (self.batch.q & 1), ty)

    def run_pass(self, nsteps: int, window: int, which: int, stream=None, attach=None):
        """Pass 1 (interior) or 2 (boundary tile rows) of one window launch."""
        self.batch.run_pass(self.land, nsteps, window, which, self.shard, stream=stream,
                            attach=attach)

    def mark_ghosts(self, stream=None):
        st = self.batch.struct()
        L.check(L.lib().fc_mark_ghosts(C.byref(self.batch.grid), C.byref(st), C.byref(self.shard),
                                       self.batch.q, L.stream_ptr(stream)), "fc_mark_ghosts")

    def run_window(self, nsteps: int, window: int, **kw):
        self.batch.run(self.land, nsteps, window=window, shard=self.shard, **kw)

    def owned(self, t: torch.Tensor) -> torch.Tensor:
        r0 = self.part.local_rows[0]
        o0, o1 = self.part.owned_rows
        return t[..., o0 - r0:o1 - r0, :]


# ------------------------------------------------------------- exchanges
class LocalHalo:
    """Emulated ranks in one process: the ghost rows of every shard's current
    input buffers are refreshed from its neighbours' boundary rows by device
    copies (on the current stream)."""

    def __call__(self, shards: Sequence[RowShard]):
        for up, down in zip(shards[:-1], shards[1:]):
            for dst, src in zip(up.ghost("bottom"), down.boundary("first")):
                dst.copy_(src)
            for dst, src in zip(down.ghost("top"), up.boundary("last")):
                dst.copy_(src)


class NcclHalo:
    """One rank's ghost refresh over torch.distributed P2P (NCCL over NVLink
    on GPUs, gloo on CPU): the first / last owned tile rows of both bit
    planes go to the neighbours and their boundary rows land directly in the
    ghost rows (contiguous views of the planes; nothing is allocated per
    window).  Issued on the current stream."""

    def __init__(self, group=None):
        self.group = group

    def __call__(self, shards: Sequence[RowShard]):
        (shard,) = shards
        p = shard.part
        exchange_halo_tensors(p.rank, p.world,
                              list(shard.boundary("first")) if p.ghost_top else [],
                              list(shard.boundary("last")) if p.ghost_bottom else [],
                              list(shard.ghost("top")) if p.ghost_top else [],
                              list(shard.ghost("bottom")) if p.ghost_bottom else [], self.group)


def exchange_halo_tensors(rank: int, world: int, first, last, ghost_top, ghost_bottom,
                          group=None):
    """Send this rank's first/last owned tile rows to the neighbours and
    receive their boundary rows into the ghost buffers (one batched group of
    P2P ops, so no ordering deadlock).  Each argument is a list of 1-D
    contiguous tensors (one per bit plane)."""
    dist = torch.distributed
    ops = []
    if rank > 0:
        for t in first:
            ops.append(dist.P2POp(dist.isend, t, rank - 1, group))
        for t in ghost_top:
            ops.append(dist.P2POp(dist.irecv, t, rank - 1, group))
    if rank < world - 1:
        for t in last:
            ops.append(dist.P2POp(dist.isend, t, rank + 1, group))
        for t in ghost_bottom:
            ops.append(dist.P2POp(dist.irecv, t, rank + 1, group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()


class _NoStream:
    """Stand-in for CUDA streams / events on CPU (the schedule's host logic
    under gloo): every operation is already ordered."""

    def wait_event(self, e):
        pass


def _stream_ctx(st):
    import contextlib
    return torch.cuda.stream(st) if isinstance(st, torch.cuda.Stream) else contextlib.nullcontext()


def run_overlapped(shards: Sequence[RowShard], steps: int, window: int, exchange, *,
                   compute_streams=None, comm_stream=None, attach=None):
    """Advance row shards `steps` steps, `window` steps per launch, with the
    halo exchange of each launch overlapping the interior pass of the next:

        pass1(q) | [wait halo(q-1)] pass2(q) -> event -> comm: exchange(q) -> halo(q)

    per shard on its compute stream; the exchange (all shards' boundary rows
    of launch q -> ghost rows of launch q+1's input buffers) on comm_stream.
    Only pass 2 waits for the halo; pass 1 of launch q+1 reads no ghost row
    and writes the other buffer parity, so it runs during the exchange.
    shards: this rank's shard (NcclHalo) or every emulated shard (LocalHalo).
    On CPU (gloo) the streams are stand-ins and everything runs in order."""
    cuda = getattr(getattr(shards[0].batch, "device", None), "type", None) == "cuda"
    if cuda:
        comp = compute_streams or [torch.cuda.current_stream()] * len(shards)
        comm = comm_stream or torch.cuda.Stream()
    else:
        comp = [_NoStream()] * len(shards)
        comm = _NoStream()
    halo = None
    done = 0
    while done < steps:
        n = min(window, steps - done)
        att = None if attach is None else attach[done:done + n]
        for sh, st in zip(shards, comp):                  # pass 1: interior tiles
            with _stream_ctx(st):
                sh.run_pass(n, window, 1, attach=att)
        ends = []
        for sh, st in zip(shards, comp):                  # pass 2: boundary rows
            if halo is not None:
                st.wait_event(halo)
            with _stream_ctx(st):
                sh.run_pass(n, window, 2, attach=att)
            if cuda:
                e = torch.cuda.Event()
                e.record(st)
                ends.append(e)
        for e in ends:
            comm.wait_event(e)
        with _stream_ctx(comm):                           # halo of this launch
            exchange(shards)
        if cuda:
            halo = torch.cuda.Event()
            halo.record(comm)
        done += n
    if cuda and halo is not None:
        for st in set(comp):
            st.wait_event(halo)
        torch.cuda.current_stream().wait_event(halo)


def run_sharded_local(shards: Sequence[RowShard], steps: int, window: int = 8, **kw):
    """Emulated shards in one process on one GPU: the overlapped schedule
    with a compute stream per shard and device-copy exchanges."""
    streams = [torch.cuda.Stream() for _ in shards]
    for st in streams:
        st.wait_stream(torch.cuda.current_stream())
    run_overlapped(shards, steps, window, LocalHalo(), compute_streams=streams, **kw)


def run_sharded(shard: RowShard, steps: int, window: int = 8, group=None, **kw):
    """Advance this rank's shard with the NCCL halo exchange of every launch
    overlapped with the next launch's interior pass."""
    run_overlapped([shard], steps, window, NcclHalo(group), **kw)
