"""Row-sharded single domain (config 3 layout) emulated on one GPU: every
shard runs on its own stream with the overlapped schedule of the NCCL path
(sharded.run_overlapped: pass 1 of launch q+1 runs while the ghost rows of
launch q are refreshed on a communication stream, here by device copies;
pass 2 waits for them); the result must equal the unsharded run byte for
byte (draws are keyed by the global cell).  The multi-process exchange and
schedule are covered on CPU by tests/test_parallel_gloo.py."""
import numpy as np
import pytest
import torch

import paper_2502_18738_b200 as F
from paper_2502_18738_b200 import synthetic as S
from paper_2502_18738_b200.sharded import RowPartition, RowShard, run_sharded_local

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world,window,attach", [(2, 8, False), (3, 4, True), (4, 16, False),
                                                 (2, 1, True), (5, 4, False)])
def test_row_sharded_equals_unsharded(world, window, attach):
    h, w, steps = 300, 140, 70
    env = S.make_environment(h, w, seed=31)
    init = S.random_blocks(h, w, 6, 5, seed=2)
    init |= S.center_ignition(h, w)
    params = F.pack_params(0.06, 0.12, 0.08, 0.6, 0.45)
    att = [attach] * steps
    ref = F.FireBatch((h, w), 1, max_steps=steps, with_jacobian=attach)
    ref.set_params(params)
    ref.set_seeds([77])
    ref.reset(init)
    ref.run(F.DeviceLandscape.from_environment(env), steps, attach=att, window=window)
    rb, rd = ref.unpack()
    shards = []
    for r in range(world):
        sh = RowShard(RowPartition(h, world, r), env.elevation, env.wind_speed,
                      env.wind_direction, env.canopy, env.density, init, max_steps=steps,
                      with_jacobian=attach)
        sh.batch.set_params(params)
        sh.batch.set_seeds([77])
        shards.append(sh)
    run_sharded_local(shards, steps, window=window, attach=att)
    parts_b, parts_d, parts_acc, parts_t = [], [], [], []
    series = 0
    for sh in shards:
        b, d = sh.batch.unpack()
        parts_b.append(sh.owned(b[0]))
        parts_d.append(sh.owned(d[0]))
        parts_acc.append(sh.owned(sh.batch.acc[0]))
        parts_t.append(sh.owned(sh.batch.t_ign[0]))
        cnt = sh.batch.counters[0, :steps].to(torch.int64).cpu().numpy()
        burning = sh.owned_init_burning + np.cumsum(cnt[:, 0] - cnt[:, 1])
        series = series + np.stack([burning, np.cumsum(cnt[:, 1])], axis=-1)
        if attach:
            assert torch.equal(sh.owned(sh.batch.jac[0].permute(2, 0, 1)),
                               ref.jac[0].permute(2, 0, 1)[:, sh.part.owned_rows[0]:sh.part.owned_rows[1]])
    assert torch.equal(torch.cat(parts_b), rb[0]) and torch.equal(torch.cat(parts_d), rd[0])
    assert torch.equal(torch.cat(parts_acc), ref.acc[0])
    assert torch.equal(torch.cat(parts_t), ref.t_ign[0])
    assert np.array_equal(series, ref.series()[0])
    assert int(rb.sum() + rd.sum()) > 500


@pytest.mark.parametrize("world,window", [(2, 8), (3, 4)])
def test_row_sharded_dense_sweep_equals_unsharded(world, window):
    """Dense sweeps (skip_inactive=False) of row shards, one fc_run per
    window with the ghost rows refreshed in between: the dense scan lists
    owned tiles next to ghost-row fire and never writes ghost rows, so the
    result equals the unsharded run byte for byte."""
    from paper_2502_18738_b200.sharded import LocalHalo
    h, w, steps = 300, 140, 60
    env = S.make_environment(h, w, seed=33)
    init = S.random_blocks(h, w, 6, 5, seed=4) | S.center_ignition(h, w)
    params = F.pack_params(0.06, 0.12, 0.08, 0.6, 0.45)
    ref = F.FireBatch((h, w), 1, max_steps=steps)
    ref.set_params(params)
    ref.set_seeds([78])
    ref.reset(init)
    ref.run(F.DeviceLandscape.from_environment(env), steps, window=window)
    rb, rd = ref.unpack()
    shards = []
    for r in range(world):
        sh = RowShard(RowPartition(h, world, r), env.elevation, env.wind_speed,
                      env.wind_direction, env.canopy, env.density, init, max_steps=steps)
        sh.batch.set_params(params)
        sh.batch.set_seeds([78])
        shards.append(sh)
    done = 0
    while done < steps:
        n = min(window, steps - done)
        for sh in shards:
            sh.run_window(n, window, skip_inactive=False)
        LocalHalo()(shards)
        done += n
    got_b = torch.cat([sh.owned(sh.batch.unpack()[0][0]) for sh in shards])
    got_d = torch.cat([sh.owned(sh.batch.unpack()[1][0]) for sh in shards])
    assert torch.equal(got_b, rb[0]) and torch.equal(got_d, rd[0])
    assert torch.equal(torch.cat([sh.owned(sh.batch.acc[0]) for sh in shards]), ref.acc[0])
    assert torch.equal(torch.cat([sh.owned(sh.batch.t_ign[0]) for sh in shards]), ref.t_ign[0])
    assert int(rb.sum() + rd.sum()) > 500


@pytest.mark.parametrize("world,window,attach", [(2, 8, False), (3, 4, True), (4, 16, False),
                                                 (2, 1, True)])
def test_row_sharded_peer_halo_equals_unsharded(world, window, attach):
    """Peer-memory halo (fc_peer_halo): each shard's boundary pass stores its
    boundary rows straight into the neighbours' ghost rows and counts the
    launch in their flag words; streams wait on the flags (no exchange step,
    no kernel waits on another).  Emulated shards on one GPU, each on its
    own stream; two calls (the second after a reset) to exercise the
    protocol's start signal and closing drain.  Equals the unsharded run."""
    from paper_2502_18738_b200.sharded import connect_local_peers, run_peer_local
    h, w, steps = 300, 140, 70
    env = S.make_environment(h, w, seed=35)
    init = S.random_blocks(h, w, 6, 5, seed=6) | S.center_ignition(h, w)
    params = F.pack_params(0.06, 0.12, 0.08, 0.6, 0.45)
    att = [attach] * steps
    ref = F.FireBatch((h, w), 1, max_steps=steps, with_jacobian=attach)
    ref.set_params(params)
    ref.set_seeds([79])
    ref.reset(init)
    ref.run(F.DeviceLandscape.from_environment(env), steps, attach=att, window=window)
    rb, rd = ref.unpack()
    shards = []
    for r in range(world):
        sh = RowShard(RowPartition(h, world, r), env.elevation, env.wind_speed,
                      env.wind_direction, env.canopy, env.density, init, max_steps=steps,
                      with_jacobian=attach)
        sh.batch.set_params(params)
        sh.batch.set_seeds([79])
        shards.append(sh)
    connect_local_peers(shards)
    for call in range(2):
        # call 0: 30 steps then 40 more in the same call sequence; call 1: reset and
        # the whole run
        if call == 0:
            run_peer_local(shards, 30, window=window, attach=att[:30])
            run_peer_local(shards, steps - 30, window=window, attach=att[30:])
        else:
            run_peer_local(shards, steps, window=window, attach=att, reset=True)
        torch.cuda.synchronize()
        got_b = torch.cat([sh.owned(sh.batch.unpack()[0][0]) for sh in shards])
        got_d = torch.cat([sh.owned(sh.batch.unpack()[1][0]) for sh in shards])
        assert torch.equal(got_b, rb[0]) and torch.equal(got_d, rd[0]), call
        assert torch.equal(torch.cat([sh.owned(sh.batch.acc[0]) for sh in shards]), ref.acc[0])
        assert torch.equal(torch.cat([sh.owned(sh.batch.t_ign[0]) for sh in shards]), ref.t_ign[0])
        if attach:
            for sh in shards:
                o0, o1 = sh.part.owned_rows
                assert torch.equal(sh.owned(sh.batch.jac[0].permute(2, 0, 1)),
                                   ref.jac[0].permute(2, 0, 1)[:, o0:o1])
        for sh in shards:
            assert int(sh.peer_flags.abs().sum()) == 0  # every call ends with zero flags
    assert int(rb.sum() + rd.sum()) > 500


def _peer_ipc_worker(rank, world, port, q):
    import os
    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    import torch.distributed as dist
    from paper_2502_18738_b200.sharded import connect_peers, peer_handshake
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        h, w = 200, 96
        env = S.make_environment(h, w, seed=1)
        init = np.zeros((h, w), dtype=bool)
        sh = RowShard(RowPartition(h, world, rank), env.elevation, env.wind_speed,
                      env.wind_direction, env.canopy, env.density, init, max_steps=8)
        connect_peers(sh)
        ok = peer_handshake(sh)
        # the mapped planes are the neighbours' own: write a pattern into
        # their ghost tile rows (burn1 plane) through the mapping, read ours
        words = sh.tiles_x * 32
        keep = sh._peer_keep          # [planes, flags] per connected side, up first
        sides = [("up", sh.part.ghost_top), ("down", sh.part.ghost_bottom)]
        k = 0
        for name, present in sides:
            if not present:
                continue
            ps = keep[k]
            k += 2
            nb_ty = sh._peer.up_tiles_y if name == "up" else sh._peer.down_tiles_y
            pl = torch.empty(0, dtype=torch.int32, device="cuda").set_(ps)
            pstride = (sh._peer.up[1] if name == "up" else sh._peer.down[1]) - \
                      (sh._peer.up[0] if name == "up" else sh._peer.down[0])
            ty = nb_ty - 1 if name == "up" else 0
            off = pstride // 4 + ty * words
            pl[off:off + words] = 1000 * (rank + 1) + (1 if name == "up" else 2)
        torch.cuda.synchronize()
        dist.barrier()
        got = []
        if sh.part.ghost_top:   # written by the upper neighbour as its "down" side
            got.append(int(sh._rows(1, 0)[5].item()) == 1000 * rank + 2)
        if sh.part.ghost_bottom:
            got.append(int(sh._rows(1, sh.rows_tiles - 1)[5].item()) == 1000 * (rank + 2) + 1)
        dist.barrier()
        q.put((rank, ok, all(got)))
        dist.destroy_process_group()
    except Exception as exc:  # reported to the parent
        q.put((rank, False, repr(exc)))


def test_peer_halo_ipc_mapping_two_processes():
    """connect_peers maps the neighbours' planes and flag words with CUDA IPC
    (two processes on the one GPU here: the mapping, the handshake's flag
    stores and the ghost-row addresses; no stream waits, no kernel waits on
    another -- the cross-GPU run itself is covered by the emulated test)."""
    import socket
    import torch.multiprocessing as mp
    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        port = s_.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_peer_ipc_worker, args=(r, 2, port, q)) for r in range(2)]
    for p_ in procs:
        p_.start()
    res = [q.get(timeout=300) for _ in procs]
    for p_ in procs:
        p_.join(timeout=60)
    assert all(r[1] is True and r[2] is True for r in res), res
