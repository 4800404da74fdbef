"""GPU parity at the configured sizes and in the adversarial corners.

The sm_100a path (through libfirecell's C ABI) against the CPU oracle
(oracle/, pinned to the reference by tests/test_oracle.py) and the
reference's own frozen outputs (tests/golden/):

* adversarial accuracy: rough terrain (slopes of both signs up to ~88 deg), winds up
  to 30 m/s, parameters at the PARAM_BOUNDS corners -- states bit-exact,
  every accumulator within 1e-5 relative, J finite and within 1e-5 of the
  scale of its slot terms, loss gradients within 1e-5 relative;
* config 0 (512^2 x 200) in draw-injection mode consuming uniform_grid
  tensors (pyrocell/rng.py:55-75): bit-exact against the reference's run;
* config 2 at full size (1024^2, 100 attached steps, 4 targets): the first
  three Algorithm-1 iterations (forward, fused loss + gradient, AdamW);
* config 4 at full shape (256 members x 1024^2 x 200 attached steps, wind
  rotating and ramping): members checked against the oracle;
* config 3 (16384^2 x 1000 steps, 8 fires): per-fire crops against the
  oracle run on the crop with its absolute origin (draws are keyed by the
  absolute cell, rng.py:64-67).
"""
import math
import os

import numpy as np
import pytest
import torch

import paper_2502_18738_b200 as F
from paper_2502_18738_b200 import synthetic as S
from golden_util import P, load
from oracle import oracle as O

pytestmark = pytest.mark.gpu

RTOL_ACC = 1e-5    # fp32 accumulator vs the fp64 reference (north_star)
RTOL_GRAD = 1e-5   # parameter gradients (north_star)
THREADS = os.cpu_count() or 1


def _rough(n, seed, vmax=30.0):
    """Rough terrain: a steep diagonal ramp (80 m per cell along each axis)
    plus 0..600 m white noise -- neighbour slopes of both signs up to ~88
    deg, while the downhill direction still carries the fire (pure white
    noise percolates only to local minima) -- with uniform 0..vmax winds in
    random directions and categorical vegetation/density."""
    rng = np.random.default_rng([seed, 0xAD5])
    env = S.make_environment(n, seed=seed)
    r, c = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    env.elevation = ((2 * n - r - c) * 80.0 + rng.random((n, n)) * 600.0).astype(np.float32)
    env.wind_speed = (rng.random((n, n)) * vmax).astype(np.float32)
    env.wind_direction = (rng.random((n, n)) * 360.0).astype(np.float32)
    return env


ADVERSARIAL = {
    # name: (terrain seed, wind max, params (c1, c2, a, p_h, p_continue));
    # long burning (p_continue) keeps fronts alive on the percolating terrain
    "bounds_max": (3, 30.0, (1.0, 1.0, 1.0, 1.0, 0.3)),
    "steep_mixed": (4, 30.0, (0.2, 0.3, 0.3, 0.9, 0.85)),
    "slope_only": (5, 30.0, (0.0, 0.0, 1.0, 0.6, 0.85)),
    "wind_only": (6, 30.0, (1.0, 1.0, 0.0, 0.7, 0.85)),
    "weak_spread": (7, 30.0, (0.05, 0.05, 0.05, 0.2, 0.9)),
    "defaults_rough": (8, 30.0, (0.045, 0.131, 0.078, 0.58, 0.85)),
}


@pytest.mark.parametrize("name", sorted(ADVERSARIAL))
def test_adversarial_accuracy(name):
    seed, vmax, pr = ADVERSARIAL[name]
    n, steps, members = 160, 80, 2
    env = _rough(n, seed, vmax)
    dl = F.DeviceLandscape.from_environment(env)
    b = F.FireBatch((n, n), members, max_steps=steps, with_jacobian=True)
    b.set_params(F.pack_params(*pr))
    b.set_seeds([seed * 10 + m for m in range(members)])
    init = S.center_ignition(n, block=5)
    b.reset(init)
    attach = [s % 4 != 3 for s in range(steps)]  # attached and unattached steps
    b.run(dl, steps, attach=attach)
    bu, bd = (x.bool().cpu().numpy() for x in b.unpack())
    arr = S.reference_landscape_arrays(env, O.slope_from_altitude)
    tg = np.zeros((n, n), bool)
    tg[n // 2 - 30:n // 2 + 25, n // 2 - 20:n // 2 + 35] = True
    _, _, g_dev, _ = b.loss_grad(torch.as_tensor(tg), [steps])
    jac = b.jac.double().cpu().numpy()
    assert np.isfinite(jac).all()
    for m in range(members):
        res = O.run(**arr, params=P(pr), init=init, steps=steps, seed=seed * 10 + m,
                    attach_steps=[s + 1 for s in range(steps) if attach[s]], threads=THREADS,
                    want_jac_abs=True)
        assert np.array_equal(bu[m], res.burning) and np.array_equal(bd[m], res.burned)
        assert res.affected().sum() > 200, "the fire must spread for the case to mean anything"
        acc = b.acc[m].double().cpu().numpy()
        np.testing.assert_allclose(acc, res.acc, rtol=RTOL_ACC, atol=0)
        # parameter gradients (the north_star bar): 1e-5 relative, above the
        # rounding floor of the reference's own fp64 chain where slots
        # saturate (its 1 - fp and 1 - fp*fp cancel to ulps, tape.py:106-147)
        _, _, _, g = O.combined_loss(res.acc, tg)
        want = O.contract(res.jac, g)
        got = g_dev[m].cpu().numpy()
        floor = O.contract(res.jac_floor, np.abs(g))
        for k in range(4):
            assert abs(got[k] - want[k]) <= RTOL_GRAD * abs(want[k]) + floor[k], (
                k, got, want, floor)
        # per-cell J (a saved intermediate, not a north_star quantity): 1e-5
        # of the scale of its slot terms (the components are signed sums, so
        # a bound relative to J itself is ill-conditioned) + the reference's
        # rounding floor + the conditioning of an fp32 evaluation (the
        # oracle's error model, orc_fp32_cond: a saturated slot amplifies
        # the error of its exponent by 2y, and the c2 term's cos - 1 comes
        # from an fp32 wind vector); J recomputed in fp64 (FC_EB_MAX) is
        # held to the same bound
        ign = (res.t_ign >= 0) & (res.t_ign < steps)
        err = np.abs(jac[m] - res.jac)[ign]
        tol = RTOL_GRAD * res.jac_abs[ign] + res.jac_floor[ign] + res.jac_cond[ign]
        assert np.all(err <= tol), float((err / np.maximum(tol, 1e-300)).max())


def test_c0_draw_injection_with_reference_draws():
    """north_star's correctness mode: the kernel consumes the reference's
    uniform-draw tensors (uniform_grid, rng.py:55-75, per step and channel)
    and must reproduce the reference's config-0 run (tests/golden/c0.npz,
    written by pyrocell) bit for bit."""
    d = load("c0")
    size, steps = int(d["size"]), int(d["steps"])
    env = S.make_environment(size, seed=0)
    assert env.fingerprint() == str(d["fingerprint"])
    dl = F.DeviceLandscape.from_environment(env)
    b = F.FireBatch((size, size), 1, max_steps=steps)
    b.set_params(F.pack_params(**{k: S.DEFAULT_BENCH_PARAMS[k] for k in
                                  ("c1", "c2", "a", "p_h", "p_continue")}))
    b.set_seeds([0])
    b.reset(S.center_ignition(size))
    for t in range(steps):  # one step's draws at a time (4 MiB), fp64
        dr = np.stack([O.uniform_grid(0, t, ch, 0, 0, size, size) for ch in (0, 1)])
        b.run(dl, 1, rng="inject", draws=torch.as_tensor(dr[None, None]), window=1)
    bu, bd = b.unpack()
    assert np.array_equal(np.packbits(bu[0].bool().cpu().numpy()), d["burning"])
    assert np.array_equal(np.packbits(bd[0].bool().cpu().numpy()), d["burned"])
    acc = b.acc[0].double().cpu().numpy().ravel()
    assert np.array_equal(np.flatnonzero(acc), d["acc_idx"])
    np.testing.assert_allclose(acc[d["acc_idx"]], d["acc_val"], rtol=RTOL_ACC)
    assert np.array_equal(b.series()[0], d["series"])
    # ... and the keyed SplitMix mode gives the same bytes
    k = F.FireBatch((size, size), 1, max_steps=steps)
    k.set_params(b.params[0].cpu().numpy())
    k.set_seeds([0])
    k.reset(S.center_ignition(size))
    k.run(dl, steps, window=1)
    assert torch.equal(k.planes, b.planes) and torch.equal(k.acc, b.acc)


def test_c2_full_size_algorithm1_iterations():
    """Config 2 at its configured size: targets from the hidden parameters
    (seed 7) at steps 25/50/75/100, then three Algorithm-1 iterations of a
    100-step all-attached forward, the 4-target loss fused with the
    gradient and one AdamW step -- each against the oracle."""
    n, T = 1024, 100
    env = S.make_environment(n, seed=2)
    dl = F.DeviceLandscape.from_environment(env)
    arr = S.reference_landscape_arrays(env, O.slope_from_altitude)
    init = S.center_ignition(n)
    hid = S.HIDDEN_C2_PARAMS
    hp = P([hid["c1"], hid["c2"], hid["a"], hid["p_h"], hid["p_continue"]])
    tr = O.run(**arr, params=hp, init=init, steps=T, seed=7, threads=THREADS)
    obs = [25, 50, 75, 100]
    targets = np.stack([tr.t_ign < s for s in obs])
    # the device generates the same targets
    tb = F.FireBatch((n, n), 1, max_steps=T)
    tb.set_params(F.pack_params(hp.c1, hp.c2, hp.a, hp.p_h, hp.p_continue))
    tb.set_seeds([7])
    tb.reset(init)
    for s in obs:
        tb.run(dl, 25)
        bu, bd = tb.unpack()
        assert np.array_equal((bu[0] | bd[0]).bool().cpu().numpy(), targets[obs.index(s)])
    p0 = S.DEFAULT_BENCH_PARAMS
    theta = np.array([p0["c1"], p0["c2"], p0["a"], p0["p_h"]])
    b = F.FireBatch((n, n), 1, max_steps=T, with_jacobian=True)
    b.set_params(F.pack_params(*theta, p0["p_continue"]))
    seed = F.derive_epoch_seed(7, 1)
    b.set_seeds([seed])
    tgt_dev = torch.as_tensor(targets.astype(np.uint8))
    adam = {}
    for it in range(3):
        b.reset(init)
        b.run(dl, T, attach=[True] * T)
        loss, _, grad, _ = b.loss_grad(tgt_dev, obs)
        pc = P([*theta, p0["p_continue"]])
        res = O.run(**arr, params=pc, init=init, steps=T, seed=seed,
                    attach_steps=range(1, T + 1), threads=THREADS)
        bu, bd = (x[0].bool().cpu().numpy() for x in b.unpack())
        assert np.array_equal(bu, res.burning) and np.array_equal(bd, res.burned), it
        np.testing.assert_allclose(b.acc[0].double().cpu().numpy(), res.acc, rtol=RTOL_ACC)
        total, g_ref = O.multi_target_grad(res, obs, targets)
        assert math.isclose(float(loss[0, 0]), total, rel_tol=RTOL_ACC), it
        np.testing.assert_allclose(grad[0].cpu().numpy(), g_ref, rtol=RTOL_GRAD)
        b.adamw(grad, it + 1, 1e-2)
        theta = np.clip(O.adamw_update(adam, theta, grad[0].cpu().numpy(), 1e-2),
                        [0, 0, 0, 0.2], [1, 1, 1, 1])
        np.testing.assert_allclose(b.params[0, :4].cpu().numpy(), theta, rtol=1e-12, atol=1e-15)
    assert res.n_entries > 10000  # the configured scale: ~1.2e4 tape entries per iteration


def test_c4_full_shape_members_vs_oracle():
    """Config 4's production shape: 256 members x 1024^2 x 200 steps, every
    step attached, wind rotating +90 deg and ramping 2 -> 12 m/s (device
    schedule); members 0, 1 and 255 against the oracle fed the same
    per-step WindUpdates, per-member 4-target loss and gradient."""
    from paper_2502_18738_b200.device import wind_ramp_schedule
    n, T, M = 1024, 200, 256
    env = S.make_environment(n, seed=4)
    dl = F.DeviceLandscape.from_environment(env)
    arr = S.reference_landscape_arrays(env, O.slope_from_altitude)
    sched = wind_ramp_schedule(T, 2.0, 12.0, 90.0)
    rows = sched.cpu().numpy()
    init = S.center_ignition(n)
    hid = S.HIDDEN_C2_PARAMS
    hp = P([hid["c1"], hid["c2"], hid["a"], hid["p_h"], hid["p_continue"]])
    tr = O.run(**arr, params=hp, init=init, steps=T, seed=7, wind_params=rows, threads=THREADS)
    obs = [50, 100, 150, 200]
    targets = np.stack([tr.t_ign < s for s in obs])
    p0 = S.DEFAULT_BENCH_PARAMS
    pr = (p0["c1"], p0["c2"], p0["a"], p0["p_h"], p0["p_continue"])
    b = F.FireBatch((n, n), M, max_steps=T, with_jacobian=True)
    b.set_params(F.pack_params(*pr))
    b.set_seeds(list(range(M)))
    b.reset(init)
    b.run(dl, T, attach=[True] * T, wind_schedule=sched)  # production window (4 at 256)
    loss, _, grad, _ = b.loss_grad(torch.as_tensor(targets.astype(np.uint8)), obs)
    for m in (0, 1, M - 1):
        res = O.run(**arr, params=P(pr), init=init, steps=T, seed=m, wind_params=rows,
                    attach_steps=range(1, T + 1), threads=THREADS)
        bu, bd = (x[m].bool().cpu().numpy() for x in b.unpack())
        assert np.array_equal(bu, res.burning) and np.array_equal(bd, res.burned), m
        np.testing.assert_allclose(b.acc[m].double().cpu().numpy(), res.acc, rtol=RTOL_ACC)
        total, g_ref = O.multi_target_grad(res, obs, targets)
        assert math.isclose(float(loss[m, 0]), total, rel_tol=RTOL_ACC), m
        np.testing.assert_allclose(grad[m].cpu().numpy(), g_ref, rtol=RTOL_GRAD)


def test_c3_fire_crops_vs_oracle():
    """Config 3 (16384^2, 1000 steps, 8 random 5x5 fires, sigma x32
    environment) on one GPU, k = 8 fused steps; two fires' neighbourhoods
    cropped with a margin the fire never reached and run by the oracle with
    the crop's absolute origin (absolute-cell draws)."""
    n, T = 16384, 1000
    e = S.make_environment_torch(n, n, seed=3)
    dl = F.DeviceLandscape.from_elevation(e["elevation"], e["wind_speed"], e["wind_direction"],
                                          e["canopy"], e["density"])
    init = S.random_blocks(n, n, 8, 5, seed=3)
    b = F.FireBatch((n, n), 1, max_steps=T)
    b.set_params(F.pack_params(0.045, 0.131, 0.078, 0.58, 0.3))
    b.set_seeds([3])
    b.reset(init)
    b.run(dl, T, window=8)
    bu, bd = b.unpack()
    checked = 0
    for r, c in S.random_block_origins(n, n, 8, 5, seed=3)[:3]:
        r0, r1 = max(r - 1300, 0), min(r + 1305, n)
        c0, c1 = max(c - 1300, 0), min(c + 1305, n)
        aff = (bu[0, r0:r1, c0:c1] | bd[0, r0:r1, c0:c1]).bool().cpu().numpy()
        ring = np.ones_like(aff)
        ring[2:-2, 2:-2] = False
        # crop edges that are domain edges are real boundaries
        if r0 == 0: ring[:2] = False
        if r1 == n: ring[-2:] = False
        if c0 == 0: ring[:, :2] = False
        if c1 == n: ring[:, -2:] = False
        if (aff & ring).any():
            continue  # the fire reached the crop margin: not a closed neighbourhood
        sl = lambda t: t[r0:r1, c0:c1].double().cpu().numpy()
        arr = dict(wind_speed=sl(e["wind_speed"]), wind_direction=sl(e["wind_direction"]),
                   slope=O.slope_from_altitude(sl(e["elevation"]), 30.0),
                   canopy=sl(e["canopy"]), density=sl(e["density"]))
        res = O.run(**arr, params=P([0.045, 0.131, 0.078, 0.58, 0.3]), init=init[r0:r1, c0:c1],
                    steps=T, seed=3, origin=(r0, c0), threads=THREADS)
        assert np.array_equal(bu[0, r0:r1, c0:c1].bool().cpu().numpy(), res.burning)
        assert np.array_equal(bd[0, r0:r1, c0:c1].bool().cpu().numpy(), res.burned)
        np.testing.assert_allclose(b.acc[0, r0:r1, c0:c1].double().cpu().numpy(), res.acc,
                                   rtol=RTOL_ACC)
        assert res.affected().sum() > 100000
        checked += 1
    assert checked >= 1


@pytest.mark.parametrize("rng", ["philox", "splitmix"])
def test_member_sharding_is_partition_invariant(rng):
    """A 6-member ensemble run as one batch of 6 and as two shards of 3
    (member0 = 0 and 3, parallel.shard_members) gives identical bytes: Philox
    counters carry the global member index (north_star: draws keyed by
    (seed, step, cell, member))."""
    from paper_2502_18738_b200.parallel import shard_members
    n, steps, M = 96, 60, 6
    env = S.make_environment(n, seed=31)
    dl = F.DeviceLandscape.from_environment(env)
    params = np.array([F.pack_params(0.05, 0.12, 0.08, p, 0.4) for p in S.ensemble_ph(M)])
    init = S.center_ignition(n)

    def run(members, member0):
        b = F.FireBatch((n, n), len(members), max_steps=steps, with_jacobian=True,
                        member0=member0)
        b.set_params(params[members])
        b.set_seeds([7] * len(members))  # one seed: only the member word tells them apart
        b.reset(init)
        b.run(dl, steps, attach=[True] * steps, rng=rng)
        bu, bd = b.unpack()
        return bu, bd, b.acc.clone(), b.jac.clone()

    whole = run(list(range(M)), 0)
    parts = [run(shard_members(M, r, 2), shard_members(M, r, 2)[0]) for r in range(2)]
    for k in range(4):
        assert torch.equal(whole[k], torch.cat([parts[0][k], parts[1][k]]))
    if rng == "philox":
        # without the offset the second shard would replay members 0..2's draws
        wrong = run(shard_members(M, 1, 2), 0)
        assert not torch.equal(wrong[0], parts[1][0])


def test_run_longer_than_int16_ignition_steps():
    """kernel.py:453-468 has no step limit: a 70,000-step run (two rebases of
    the int16 ignition-step base) keeps equal to the oracle -- a slow fire
    (cells keep burning, (1+canopy)(1+density) = 1e-4, no wind, flat) that
    still ignites cells after step 60,000."""
    n, steps = 48, 70000
    z = np.zeros((n, n))
    dl = F.DeviceLandscape.from_elevation(z, z, z, z - 0.99, z - 0.99)
    pr = (0.0, 0.0, 0.0, 0.2, 1.0)
    b = F.FireBatch((n, n), 1, max_steps=steps)
    b.set_params(F.pack_params(*pr))
    b.set_seeds([5])
    init = np.zeros((n, n), bool)
    init[0, :] = True
    b.reset(init)
    b.run(dl, steps, window=16)
    assert b.t_base >= 60000
    arr = dict(wind_speed=z, wind_direction=z, slope=np.zeros((n, n, 3, 3)), canopy=z - 0.99,
               density=z - 0.99)
    res = O.run(**arr, params=P(pr), init=init, steps=steps, seed=5, threads=THREADS)
    bu, bd = (x[0].bool().cpu().numpy() for x in b.unpack())
    assert np.array_equal(bu, res.burning) and np.array_equal(bd, res.burned)
    np.testing.assert_allclose(b.acc[0].double().cpu().numpy(), res.acc, rtol=RTOL_ACC)
    assert np.array_equal(b.series()[0], res.series)
    late = res.t_ign[(res.t_ign >= b.t_base) & (res.t_ign < steps)]
    assert late.size > 0  # ignitions after the last rebase
    tig = b.t_ign[0].cpu().numpy().astype(np.int64)
    after = (res.t_ign >= b.t_base) & (res.t_ign < steps)
    assert np.array_equal(tig[after] + b.t_base, res.t_ign[after])
    # the reference-signature API runs it too (fp64 accumulator)
    sim = F.run_simulation(F.Landscape(**arr), F.ModelParams(c1=0.0, c2=0.0, a=0.0, p_h=0.2,
                                                            p_continue=1.0),
                           init, steps, 5)
    assert np.array_equal(sim.state.burning, res.burning)
    np.testing.assert_allclose(sim.state.accumulator, res.acc, rtol=1e-10)


@pytest.mark.parametrize("window,attach,wind,tensor", [(8, False, False, False),
                                                        (4, True, True, False),
                                                        (8, True, False, True)])
def test_dataflow_ensemble_equals_one_launch_per_window(window, attach, wind, tensor):
    """The dataflow mode (one persistent launch per fc_run call, members
    advancing window by window on their own) gives the same bytes as one
    launch per window: planes, accumulator, ignition steps, Jacobians,
    per-step counters, tile_first -- also across a split run."""
    from paper_2502_18738_b200.device import wind_ramp_schedule
    n, steps, M = 384, 150, 6
    env = S.make_environment(n, seed=41)
    if tensor:
        arr = S.reference_landscape_arrays(env, O.slope_from_altitude)
        dl = F.DeviceLandscape.from_slope_tensor(arr["wind_speed"], arr["wind_direction"],
                                                 arr["slope"], arr["canopy"], arr["density"])
    else:
        dl = F.DeviceLandscape.from_environment(env)
    sched = wind_ramp_schedule(steps, 2.0, 12.0, 90.0) if wind else None
    params = np.array([F.pack_params(0.05, 0.12, 0.08, p, 0.4) for p in S.ensemble_ph(M)])
    init = S.center_ignition(n)
    att = [attach and (s % 3 != 2) for s in range(steps)]
    out = []
    for df in (False, True):
        b = F.FireBatch((n, n), M, max_steps=steps, with_jacobian=attach, dataflow=df)
        assert (b.sched is not None) == df
        b.set_params(params)
        b.set_seeds(list(range(10, 10 + M)))
        b.reset(init)
        b.run(dl, 70, attach=att[:70], window=window, wind_schedule=sched)
        b.run(dl, steps - 70, attach=att[70:], window=window, wind_schedule=sched)
        out.append((b.planes.clone(), b.acc.clone(), b.t_ign.clone(),
                    None if b.jac is None else b.jac.clone(), b.counters.clone(),
                    b.tile_first.clone(), b.q, b.list_count[:2 * (steps + 3) + 1].clone()))
    a, d = out
    assert int(a[0].count_nonzero()) > 1000
    for k in range(6):
        if a[k] is not None:
            assert torch.equal(a[k], d[k]), k
    assert a[6] == d[6]
    q = a[6]
    assert torch.equal(a[7][q:q + 2], d[7][q:q + 2])  # the next launches' list lengths


def test_dataflow_many_members_injection_and_window_change():
    """Dataflow with 64 members of very different fire sizes (p_h from 0.2 to
    1), an injection between runs and the window growing from 4 to 8 (the
    lists are re-marked, split and merged around every call): the same bytes
    as one launch per window."""
    n, M = 160, 64
    env = S.make_environment(n, seed=43)
    dl = F.DeviceLandscape.from_environment(env)
    params = np.array([F.pack_params(0.05, 0.12, 0.08, 0.2 + 0.8 * m / (M - 1), 0.5)
                       for m in range(M)])
    init = S.center_ignition(n)
    out = []
    for df in (False, True):
        b = F.FireBatch((n, n), M, max_steps=90, dataflow=df)
        b.set_params(params)
        b.set_seeds(list(range(M)))
        b.reset(init)
        b.run(dl, 30, window=4)
        b.inject([(m, 10, 10 + m) for m in range(0, M, 3)])
        b.run(dl, 60, window=8)
        out.append((b.planes.clone(), b.acc.clone(), b.t_ign.clone(), b.counters.clone()))
    for k in range(4):
        assert torch.equal(out[0][k], out[1][k]), k
