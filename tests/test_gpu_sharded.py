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
