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

The peer-memory halo (``run_peer``, ``fc_peer_halo``) fuses the transfer
into the boundary pass: pass 2 stores its output boundary rows straight into
the neighbours' ghost rows (NVLink peer writes through CUDA IPC mappings, or
plain device memory for shards emulated on one GPU) and counts the launch in
their flag words; the neighbour's stream waits on its flag word
(cuStreamWaitValue32, no spinning kernel) before its next pass 2.  No
collective and no copy kernel run in the step loop.
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
        # peer halo: the words the neighbours store their event numbers
        # into ([0] from the upper neighbour, [1] from the lower one); zero
        # between calls (fc_peer_halo protocol)
        self.peer_flags = torch.zeros(2, dtype=torch.int32, device=self.batch.device)
        self._peer = None
        self._peer_keep = []

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

    # --------------------------------------------------------- peer halo
    def plane_ptrs(self) -> List[int]:
        """Device addresses of {burn0, burn1, burned0, burned1}."""
        st = self.batch.struct()
        return [st.burn0, st.burn1, st.burned0, st.burned1]

    def attach_peers(self, up=None, down=None, keep=()):
        """Enable the peer-memory halo.  up / down: (the neighbour's four plane
        addresses, its local tile rows, the address of the neighbour's flag
        word this shard writes) or None where there is no neighbour; keep:
        objects that own those mappings (kept alive with the shard)."""
        if (up is not None) != bool(self.part.ghost_top) or \
                (down is not None) != bool(self.part.ghost_bottom):
            raise ValueError("peers must match the shard's ghost rows")
        P = L.FcPeerHalo()
        if up is not None:
            for i, a in enumerate(up[0]):
                P.up[i] = a
            P.up_tiles_y, P.up_flag = int(up[1]), up[2]
        if down is not None:
            for i, a in enumerate(down[0]):
                P.down[i] = a
            P.down_tiles_y, P.down_flag = int(down[1]), down[2]
        self._peer = P
        self._peer_keep = list(keep)
        self.shard.peer = C.addressof(P)

    def _wait_peers(self, value: int, stream=None):
        base = self.peer_flags.data_ptr()
        for present, off in ((self.part.ghost_top, 0), (self.part.ghost_bottom, 4)):
            if present:
                L.check(L.lib().fc_stream_wait_geq(base + off, int(value), L.stream_ptr(stream)),
                        "fc_stream_wait_geq")

    def _peer_signal(self, value: int, stream=None):
        L.check(L.lib().fc_peer_signal(C.byref(self._peer), int(value), L.stream_ptr(stream)),
                "fc_peer_signal")

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


def connect_local_peers(shards: Sequence[RowShard]):
    """Peer halo between shards emulated in one process (one device): each
    shard's boundary pass writes its neighbours' ghost rows directly."""
    info = [(sh.plane_ptrs(), sh.rows_tiles, sh.peer_flags.data_ptr()) for sh in shards]
    for i, sh in enumerate(shards):
        up = down = None
        if i > 0:        # the upper neighbour's word [1] counts this (lower) shard's events
            up = (info[i - 1][0], info[i - 1][1], info[i - 1][2] + 4)
        if i < len(shards) - 1:  # the lower neighbour's word [0]
            down = (info[i + 1][0], info[i + 1][1], info[i + 1][2])
        sh.attach_peers(up, down)


def connect_peers(shard: RowShard, group=None):
    """Peer halo across ranks of one node: the planes and flag words of the
    neighbours are mapped with CUDA IPC (NVLink peer access) after an
    all-gather of the handles.  Collective over `group`; returns None, or why
    this rank could not map its neighbours (then follow with peer_handshake,
    which makes every rank fall back together)."""
    dist = torch.distributed
    rank, world = shard.part.rank, shard.part.world
    planes, flags = shard.batch.planes, shard.peer_flags
    try:
        mine = (planes.untyped_storage()._share_cuda_(), planes.stride(0) * planes.element_size(),
                planes.storage_offset() * planes.element_size(), shard.rows_tiles,
                flags.untyped_storage()._share_cuda_(),
                flags.storage_offset() * flags.element_size(), torch.cuda.current_device())
    except Exception:
        mine = None  # still take part in the all-gather below
    got = [None] * world
    dist.all_gather_object(got, mine, group=group)
    keep = []

    def open_side(r, word):
        if got[r] is None or mine is None:
            raise RuntimeError(f"rank {r if got[r] is None else rank} could not share its planes")
        ph, pstride, poff, ty, fh, foff, dev = got[r]
        if not torch.cuda.can_device_access_peer(torch.cuda.current_device(), dev) and \
                dev != torch.cuda.current_device():
            raise RuntimeError(f"no peer access from GPU {torch.cuda.current_device()} to {dev}")
        ps = torch.UntypedStorage._new_shared_cuda(*ph)
        fs = torch.UntypedStorage._new_shared_cuda(*fh)
        keep.extend([ps, fs])
        base = ps.data_ptr() + poff
        return ([base + i * pstride for i in range(4)], ty, fs.data_ptr() + foff + 4 * word)

    # a rank that cannot map its neighbours still reaches the barrier (and
    # peer_handshake's collectives), so the ranks agree on the transport
    err = None
    try:
        up = open_side(rank - 1, 1) if shard.part.ghost_top else None
        down = open_side(rank + 1, 0) if shard.part.ghost_bottom else None
        shard.attach_peers(up, down, keep)
    except Exception as exc:
        err = f"{type(exc).__name__}: {exc}"
        shard._peer, shard._peer_keep = None, []
        shard.shard.peer = None
    dist.barrier(group=group)
    return err


def peer_handshake(shard: RowShard, group=None, timeout: float = 5.0) -> bool:
    """Check the peer halo of this rank before using it: every rank stores 1
    into its neighbours' flag words, then polls its own from the host (no
    stream waits, so a broken mapping cannot hang the device) for `timeout`
    seconds; the flags are zeroed again.  True on every rank or on none."""
    import time
    dist = torch.distributed
    ok = shard._peer is not None
    if ok:
        shard._peer_signal(1)
        torch.cuda.synchronize()
    dist.barrier(group=group)
    want = [i for i, g in ((0, shard.part.ghost_top), (1, shard.part.ghost_bottom)) if g]
    t_end = time.monotonic() + timeout
    while ok:
        f = shard.peer_flags.cpu()
        if all(int(f[i]) >= 1 for i in want):
            break
        if time.monotonic() > t_end:
            ok = False
        time.sleep(0.001)
    dist.barrier(group=group)
    shard.peer_flags.zero_()
    torch.cuda.synchronize()
    flag = torch.tensor([1 if ok else 0], dtype=torch.int32,
                        device="cuda" if dist.get_backend(group) == "nccl" else "cpu")
    dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
    return bool(int(flag.item()))


def run_peer(shards: Sequence[RowShard], steps: int, window: int, *, compute_streams=None,
             attach=None, reset: bool = False):
    """Advance row shards with the peer-memory halo (fc_peer_halo):

        [reset] signal(1) | pass1(j) wait(>= j) pass2(seq j+1) ... | wait(>= n+1) zero flags

    per shard on its compute stream (event 1 tells the neighbours this
    shard's flags are zero and, with reset=True, its planes reset; pass 2 of
    launch j is event j+1; the closing wait drains the neighbours' last
    stores, so every call starts and ends with zero flags and may be
    captured in a CUDA graph).  shards: every shard of an emulated domain
    (connect_local_peers) or this rank's one (connect_peers)."""
    cuda = getattr(getattr(shards[0].batch, "device", None), "type", None) == "cuda"
    comp = compute_streams or ([torch.cuda.current_stream()] if cuda else [_NoStream()]) * len(shards)
    for sh in shards:
        if sh._peer is None:
            raise RuntimeError("peer halo not connected (connect_local_peers / connect_peers)")
    for sh, st in zip(shards, comp):
        with _stream_ctx(st):
            if reset:
                sh.batch.reset(sh.batch._init_mask)
            sh._peer_signal(1)
    done, j = 0, 0
    while done < steps:
        n = min(window, steps - done)
        att = None if attach is None else attach[done:done + n]
        j += 1
        for sh, st in zip(shards, comp):                  # pass 1: interior tiles
            with _stream_ctx(st):
                sh.run_pass(n, window, 1, attach=att)
        for sh, st in zip(shards, comp):                  # pass 2: boundary rows + halo
            with _stream_ctx(st):
                sh._wait_peers(j)
                sh._peer.seq = j + 1
                sh.run_pass(n, window, 2, attach=att)
        done += n
    for sh, st in zip(shards, comp):
        with _stream_ctx(st):
            sh._wait_peers(j + 1)
            sh.peer_flags.zero_()


def run_peer_local(shards: Sequence[RowShard], steps: int, window: int = 8, **kw):
    """Emulated shards in one process on one GPU with the peer halo: a
    compute stream per shard, stream-level waits only (no kernel waits on
    another)."""
    streams = [torch.cuda.Stream() for _ in shards]
    for st in streams:
        st.wait_stream(torch.cuda.current_stream())
    run_peer(shards, steps, window, compute_streams=streams, **kw)
    for st in streams:
        torch.cuda.current_stream().wait_stream(st)


def run_sharded(shard: RowShard, steps: int, window: int = 8, group=None, **kw):
    """Advance this rank's shard with the NCCL halo exchange of every launch
    overlapped with the next launch's interior pass."""
    run_overlapped([shard], steps, window, NcclHalo(group), **kw)
