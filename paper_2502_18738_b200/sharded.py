"""Row-sharded single domain (BASELINE config 3 across GPUs).

Each rank owns a band of 32-row tile rows plus one ghost tile row per
neighbour.  After every window launch the boundary tile rows of both bit
planes are exchanged (NCCL send/recv over NVLink, or device copies when
several shards are emulated in one process), then ``fc_mark_ghosts``
re-activates the owned tiles next to ghost fire.  Draws are keyed by the
global row, so the sharded trajectory is bit-identical to the unsharded one
(pyrocell's own partition invariance, kernel.py:307-309 / rng.py:64-67).
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
def exchange_local(shards: Sequence[RowShard]):
    """Emulated ranks in one process: device-to-device ghost refresh."""
    for up, down in zip(shards[:-1], shards[1:]):
        for dst, src in zip(up.ghost("bottom"), down.boundary("first")):
            dst.copy_(src)
        for dst, src in zip(down.ghost("top"), up.boundary("last")):
            dst.copy_(src)
    for s in shards:
        s.mark_ghosts()


def exchange_halo_tensors(rank: int, world: int, first, last, ghost_top, ghost_bottom,
                          group=None):
    """Send this rank's first/last owned tile rows to the neighbours and
    receive their boundary rows into the ghost buffers (torch.distributed
    P2P; NCCL over NVLink on GPUs, gloo on CPU).  Each argument is a list of
    1-D tensors (one per bit plane)."""
    dist = torch.distributed
    ops = []
    if rank > 0:
        for t in first:
            ops.append(dist.P2POp(dist.isend, t.contiguous(), rank - 1, group))
        for t in ghost_top:
            ops.append(dist.P2POp(dist.irecv, t, rank - 1, group))
    if rank < world - 1:
        for t in last:
            ops.append(dist.P2POp(dist.isend, t.contiguous(), rank + 1, group))
        for t in ghost_bottom:
            ops.append(dist.P2POp(dist.irecv, t, rank + 1, group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()


def exchange_nccl(shard: RowShard, group=None):
    """One rank's halo refresh over torch.distributed, then ghost marking."""
    p = shard.part
    first = list(shard.boundary("first")) if p.ghost_top else []
    last = list(shard.boundary("last")) if p.ghost_bottom else []
    gt = [t for t in shard.ghost("top")] if p.ghost_top else []
    gb = [t for t in shard.ghost("bottom")] if p.ghost_bottom else []
    # receive into staging buffers (the ghost rows are views into the planes)
    gt_buf = [torch.empty_like(t) for t in gt]
    gb_buf = [torch.empty_like(t) for t in gb]
    exchange_halo_tensors(p.rank, p.world, first, last, gt_buf, gb_buf, group)
    for d, s_ in zip(gt, gt_buf):
        d.copy_(s_)
    for d, s_ in zip(gb, gb_buf):
        d.copy_(s_)
    shard.mark_ghosts()


def run_sharded_local(shards: Sequence[RowShard], steps: int, window: int = 8, **kw):
    """Advance emulated shards window by window with halo refresh."""
    done = 0
    while done < steps:
        n = min(window, steps - done)
        for s in shards:
            s.run_window(n, window, **kw)
        exchange_local(shards)
        done += n


def run_sharded(shard: RowShard, steps: int, window: int = 8, group=None, **kw):
    """Advance this rank's shard with NCCL halo exchange after each window."""
    done = 0
    while done < steps:
        n = min(window, steps - done)
        shard.run_window(n, window, **kw)
        exchange_nccl(shard, group)
        done += n
