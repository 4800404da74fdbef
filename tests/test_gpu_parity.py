"""GPU parity: the sm_100a path (through libfirecell's C ABI) against the
reference's frozen outputs (tests/golden/) and the CPU oracle.

Bar (BASELINE.json north_star): fire-state grids bit-exact; burn
probabilities and parameter gradients within 1e-5 relative (fp32 path).
"""
import math
import os

import numpy as np
import pytest
import torch

import paper_2502_18738_b200 as F
from paper_2502_18738_b200 import synthetic as S
from golden_util import P, RUN_CASES, case_kwargs, load, meta
from oracle import oracle as O

pytestmark = pytest.mark.gpu

RTOL_ACC = 1e-5    # fp32 accumulator vs fp64 reference (north_star)
RTOL_GRAD = 1e-5   # parameter gradients (north_star)
# the pyrocell-signature API recomputes p_ignite and J in fp64 (fc_recompute64)
RTOL_ACC64 = 1e-10
RTOL_GRAD64 = 1e-9

GOLDEN_DRAWS = {  # pyrocell tests/test_rng.py:7-14
    (0, 0, 0, 0, 0): 0.23286544795475594,
    (0, 0, 0, 0, 1): 0.991448890053859,
    (1, 0, 0, 0, 0): 0.7828598730864468,
    (0, 1, 0, 0, 0): 0.6289335415767472,
    (0, 0, 5, 7, 0): 0.8443854602639748,
    (12345, 99, 120, 250, 1): 0.5958213030105105,
}


def land_of(d, key_v="wind_speed", key_d="wind_direction"):
    return F.Landscape(wind_speed=d[key_v], wind_direction=d[key_d], slope=d["slope"],
                       canopy=d["canopy"], density=d["density"])


def params_of(d):
    c1, c2, a, ph, pc = (float(v) for v in d["params"])
    return F.ModelParams(c1=c1, c2=c2, a=a, p_h=ph, p_continue=pc)


def test_device_rng_goldens():
    for (seed, t, r, c, ch), want in GOLDEN_DRAWS.items():
        assert F.uniform_draw(seed, t, r, c, F.Channel(ch)) == want
    m = meta()
    assert F.uniform_grid(99, 4, F.Channel.IGNITE, 10, 20, 5, 6).tolist() == \
        m["uniform_grid_99_4_I_10_20_5_6"]
    assert F.uniform_grid(2**40 + 3, 123, 0, 70000, 3, 2, 3).tolist() == m["uniform_grid_bigseed"]
    full = F.uniform_grid(5, 1, 1, 0, 0, 40, 40)
    assert np.array_equal(F.uniform_grid(5, 1, 1, 13, 7, 9, 11), full[13:22, 7:18])


@pytest.mark.parametrize("name", RUN_CASES)
def test_run_simulation_matches_reference(name):
    d = load(name)
    kw = case_kwargs(name, d)
    sched = [F.WindUpdate(a, v, w) for a, v, w in kw.pop("wind_schedule", [])]
    tape = F.Tape(d["burning"].shape)
    sim = F.run_simulation(land_of(d), params_of(d), d["init"], int(d["steps"]), int(d["seed"]),
                           attach_steps=[int(s) for s in d["attach"]], tape=tape,
                           wind_schedule=sched, **kw)
    assert np.array_equal(sim.state.burning, d["burning"])
    assert np.array_equal(sim.state.burned, d["burned"])
    # the reference API's accumulator is recomputed in fp64 (fc_recompute64):
    # it meets the reference to fp64 rounding, far inside the fp32 bar
    np.testing.assert_allclose(sim.state.accumulator, d["acc"], rtol=RTOL_ACC64, atol=0)
    assert np.array_equal(np.array([[s.burning, s.burned] for s in sim.series]).reshape(-1, 2),
                          d["series"])
    if "grad" in d:
        assert tape.num_entries == int(d["num_entries"])
        bd, g = F.combined_loss(sim.state.accumulator, d["target"])
        assert math.isclose(bd.bce_term, float(d["bce"]), rel_tol=RTOL_ACC)
        assert bd.crop_window == tuple(int(v) for v in d["crop"])
        grad = F.backward_params(tape, g, F.DEFAULT_NORM_C)
        for i in range(4):
            if abs(d["grad"][i]) < 1e-12:
                assert abs(grad[i]) < 1e-10
            else:
                assert abs(grad[i] - d["grad"][i]) <= RTOL_GRAD64 * abs(d["grad"][i]), (i, grad, d["grad"])


def test_structural_zero_gradients():
    d = load("run_windless")
    tape = F.Tape(d["burning"].shape)
    sim = F.run_simulation(land_of(d), params_of(d), d["init"], int(d["steps"]), int(d["seed"]),
                           attach_steps=range(1, int(d["steps"]) + 1), tape=tape)
    _, g = F.combined_loss(sim.state.accumulator, d["target"])
    grad = F.backward_params(tape, g, F.DEFAULT_NORM_C)
    assert grad[0] == 0.0 and grad[1] == 0.0 and grad[2] != 0.0


def test_combined_loss_goldens():
    bd, _ = F.combined_loss(np.zeros((8, 8)), np.zeros((8, 8), bool))
    assert math.isclose(bd.bce_term, math.log(2.0), rel_tol=1e-12) and bd.mse_term == 0.0
    assert bd.crop_window == (0, 8, 0, 8)
    for name in ("loss_random", "loss_crop"):
        d = load(name)
        bd, g = F.combined_loss(d["acc"], d["target"])
        assert math.isclose(bd.bce_term, float(d["bce"]), rel_tol=1e-12)
        assert math.isclose(bd.mse_term, float(d["mse"]), rel_tol=1e-12, abs_tol=1e-300)
        assert bd.crop_window == tuple(int(v) for v in d["crop"])
        np.testing.assert_allclose(g, d["grad"], rtol=1e-12, atol=1e-16)


def _bench_land(size, seed):
    env = S.make_environment(size, seed=seed)
    return env, F.DeviceLandscape.from_environment(env)


@pytest.mark.parametrize("name", ["c0_small", "c0"])
def test_config0_elevation_mode_matches_reference(name):
    d = load(name)
    size, steps = int(d["size"]), int(d["steps"])
    env, dl = _bench_land(size, 0)
    assert env.fingerprint() == str(d["fingerprint"])
    b = F.FireBatch((size, size), 1, max_steps=steps)
    b.set_params(F.pack_params(**{k: S.DEFAULT_BENCH_PARAMS[k] for k in
                                  ("c1", "c2", "a", "p_h", "p_continue")}))
    b.set_seeds([0])
    b.reset(S.center_ignition(size))
    b.run(dl, steps)
    bu, bd = b.unpack()
    assert np.array_equal(np.packbits(bu[0].bool().cpu().numpy()), d["burning"])
    assert np.array_equal(np.packbits(bd[0].bool().cpu().numpy()), d["burned"])
    acc = b.acc[0].double().cpu().numpy().ravel()
    assert np.array_equal(np.flatnonzero(acc), d["acc_idx"])
    np.testing.assert_allclose(acc[d["acc_idx"]], d["acc_val"], rtol=RTOL_ACC)
    assert np.array_equal(b.series()[0], d["series"])


def test_config2_iteration_fused_loss_grad():
    d = load("c2_small")
    size = int(d["size"])
    env, dl = _bench_land(size, 2)
    assert env.fingerprint() == str(d["fingerprint"])
    b = F.FireBatch((size, size), 1, max_steps=100, with_jacobian=True)
    b.set_params(F.pack_params(**{k: S.DEFAULT_BENCH_PARAMS[k] for k in
                                  ("c1", "c2", "a", "p_h", "p_continue")}))
    b.set_seeds([int(d["seed"])])
    b.reset(S.center_ignition(size))
    b.run(dl, 100, attach=[True] * 100)
    bu, bd = b.unpack()
    assert np.array_equal(bu[0].bool().cpu().numpy(), d["burning"])
    assert np.array_equal(bd[0].bool().cpu().numpy(), d["burned"])
    loss, crop, grad, _ = b.loss_grad(torch.as_tensor(d["targets"]), [int(s) for s in d["obs"]])
    assert math.isclose(float(loss[0, 0]), float(d["loss"]), rel_tol=RTOL_ACC)
    np.testing.assert_allclose(grad[0].cpu().numpy(), d["grad"], rtol=RTOL_GRAD)


def test_calibrate_trajectory_matches_reference():
    d = load("calibrate_small")
    size = int(d["size"])
    env = S.make_environment(size, seed=5)
    arr = S.reference_landscape_arrays(env, O.slope_from_altitude)
    land = F.Landscape(**arr)
    sched = F.ObservationSchedule([F.Observation(target=t) for t in d["targets"]], 6)
    start = F.ModelParams(c1=0.0, c2=0.0, a=0.0, p_h=0.3, p_continue=0.5)
    res = F.calibrate(land, S.center_ignition(size), sched, start, F.StepRings(1, 2, 3),
                      max_epochs=3, base_seed=5, learning_rate=0.05)
    assert res.manifest.epoch_seeds == [int(s) for s in d["epoch_seeds"]]
    rec = np.array([[r.epoch, r.iteration, r.loss, r.bce, r.mse, r.jaccard, r.manhattan]
                    for r in res.records])
    np.testing.assert_array_equal(rec[:, [0, 1, 5, 6]], d["records"][:, [0, 1, 5, 6]])
    np.testing.assert_allclose(rec[:, 2:5], d["records"][:, 2:5], rtol=1e-5)
    traj = np.array([[e, i, p.c1, p.c2, p.a, p.p_h, p.p_continue]
                     for e, i, p in res.manifest.trajectory])
    np.testing.assert_allclose(traj, d["trajectory"], rtol=RTOL_GRAD, atol=1e-9)


def _oracle_vs_device(size_h, size_w, steps, seed, attach, members=1, env_seed=9, skip=True,
                      rng="splitmix", draws=None, params=None):
    env = S.make_environment(size_h, size_w, seed=env_seed)
    dl = F.DeviceLandscape.from_environment(env)
    arr = S.reference_landscape_arrays(env, O.slope_from_altitude)
    p = params or P([0.045, 0.131, 0.078, 0.58, 0.3])
    init = S.center_ignition(size_h, size_w)
    b = F.FireBatch((size_h, size_w), members, max_steps=steps, with_jacobian=attach)
    b.set_params(F.pack_params(p.c1, p.c2, p.a, p.p_h, p.p_continue))
    b.set_seeds([seed + m for m in range(members)])
    b.reset(init)
    b.run(dl, steps, attach=[attach] * steps, skip_inactive=skip, rng=rng, draws=draws)
    return env, arr, p, init, b


def test_ragged_grid_members_and_partition_invariance():
    h, w, steps = 201, 333, 120
    _, arr, p, init, b = _oracle_vs_device(h, w, steps, 40, True, members=3)
    bu, bd = (x.bool().cpu().numpy() for x in b.unpack())
    for m in range(3):
        res = O.run(**arr, params=p, init=init, steps=steps, seed=40 + m,
                    attach_steps=range(1, steps + 1), threads=4, want_jac_abs=True)
        assert np.array_equal(bu[m], res.burning) and np.array_equal(bd[m], res.burned)
        np.testing.assert_allclose(b.acc[m].double().cpu().numpy(), res.acc, rtol=RTOL_ACC)
        assert np.array_equal(b.series()[m], res.series)
        jac = b.jac[m].double().cpu().numpy()
        g = np.random.default_rng(m).standard_normal((h, w))
        got = b.contract(torch.as_tensor(np.stack([g * (k == m) for k in range(3)])))[m]
        want = O.contract(res.jac, g)
        np.testing.assert_allclose(got.cpu().numpy(), want, rtol=RTOL_GRAD)
        # per-cell J: 1e-5 of its slot terms' scale + the reference's
        # rounding floor + the fp32 conditioning (tests/test_gpu_envelope.py)
        tol = RTOL_GRAD * res.jac_abs + res.jac_floor + res.jac_cond
        assert np.all(np.abs(jac - res.jac) <= tol)
    # dense sweep (no activity skipping) must give identical bytes
    _, _, _, _, b2 = _oracle_vs_device(h, w, steps, 40, True, members=3, skip=False)
    assert torch.equal(b.planes, b2.planes)
    assert torch.equal(b.acc, b2.acc) and torch.equal(b.t_ign, b2.t_ign)
    assert torch.equal(b.jac, b2.jac)


def test_draw_injection_mode_bit_exact():
    h, w, steps = 64, 80, 40
    env = S.make_environment(h, w, seed=4)
    draws = np.stack([np.stack([O.uniform_grid(11, t, ch, 0, 0, h, w) for ch in (0, 1)])
                      for t in range(steps)])[:, None]
    _, _, _, _, a = _oracle_vs_device(h, w, steps, 11, False, env_seed=4)
    _, _, _, _, b = _oracle_vs_device(h, w, steps, 11, False, env_seed=4, rng="inject",
                                      draws=torch.as_tensor(draws))
    assert torch.equal(a.planes, b.planes) and torch.equal(a.acc, b.acc)


@pytest.mark.parametrize("rng", ["splitmix", "philox"])
def test_ignition_frequency(rng):
    # one burning cell, one burnable neighbour, 4000 members (independent
    # draws): frequency realises p within 4 sigma (tests/test_kernel.py:286-303)
    n = 4000
    zeros = np.zeros((1, 2))
    dl = F.DeviceLandscape.from_elevation(zeros, zeros, zeros, zeros, zeros)
    b = F.FireBatch((1, 2), n, max_steps=1)
    b.set_params(F.pack_params(0.045, 0.131, 0.078, 0.4, 1.0))
    b.set_seeds(list(range(n)))
    init = np.zeros((1, 2), bool)
    init[0, 0] = True
    b.reset(init)
    b.run(dl, 1, rng=rng)
    hits = int(b.unpack()[0][:, 0, 1].sum())
    p = float(np.tanh(F.DEFAULT_NORM_C * 0.4))
    assert abs(hits / n - p) < 4 * math.sqrt(p * (1 - p) / n)


def test_fire_model_algorithm1_gradients():
    from paper_2502_18738_b200.torch_model import FireModel, combined_loss_torch
    d = load("run_rand16")
    land = land_of(d)
    dl = F.DeviceLandscape.from_slope_tensor(land.wind_speed, land.wind_direction, land.slope,
                                             land.canopy, land.density)
    pr = params_of(d)
    model = FireModel(dl, d["init"], a=pr.a, c1=pr.c1, c2=pr.c2, p_h=pr.p_h,
                      p_continue=pr.p_continue, seed=int(d["seed"]))
    for _ in range(int(d["steps"])):
        model.compute(attach=True)
    loss = combined_loss_torch(model.accumulator, torch.as_tensor(d["target"]))
    loss.backward()
    got = np.array([model.c_1.grad.item(), model.c_2.grad.item(), model.a.grad.item(),
                    model.p_h.grad.item()])
    np.testing.assert_allclose(got, d["grad"], rtol=RTOL_GRAD)
    assert model.p_continue.grad.item() == 0.0
    assert math.isclose(loss.item(), float(d["bce"]) + float(d["mse"]), rel_tol=RTOL_ACC)
    opt = torch.optim.AdamW(model.parameters(), lr=5e-3)
    opt.step()
    opt.zero_grad()
    model.clamp_()
    model.reset(seed=model.seed)
    assert model.t == 0


def test_inject_and_step_forward_api():
    d = load("run_rand9_source")
    land = land_of(d)
    params = params_of(d)
    st = F.new_fire_state(np.zeros(land.shape, bool), land)
    F.inject_ignitions(st, [(4, 4)])
    for _ in range(int(d["steps"])):
        F.step_forward(st, land, params, int(d["seed"]), factor_site="source")
    assert np.array_equal(st.burning, d["burning"]) and np.array_equal(st.burned, d["burned"])
    np.testing.assert_allclose(st.accumulator, d["acc"], rtol=RTOL_ACC)
    with pytest.raises(IndexError):
        F.inject_ignitions(st, [(9, 0)])
    b = F.FireBatch(land.shape, 1, max_steps=4)
    b.reset(np.zeros(land.shape, bool))
    with pytest.raises(IndexError):
        b.inject([(0, 9)])
    b.inject([(2, 2)])
    assert int(b.unpack()[0].sum()) == 1 and float(b.acc[0, 2, 2]) == 1.0


def test_build_fields_matches_oracle_formula():
    d = load("run_rand16")
    land = land_of(d)
    pr = params_of(d)
    f = F.build_fields(land, pr, with_gradients=True)
    # field k at source i toward target i - pos[k], against the scalar formula
    for (r, c) in [(3, 4), (8, 8), (0, 5), (15, 15)]:
        for k, (pr_, pc_) in enumerate(F.NEIGHBOR_POSITIONS):
            tr, tc = r - pr_, c - pc_
            if not (0 <= tr < 16 and 0 <= tc < 16):
                continue
            raw = F.propagate_prob(pr, land, (r, c), (tr, tc))
            assert math.isclose(f.raw[k][r, c], raw, rel_tol=1e-12)
            assert math.isclose(f.fp[k][r, c], float(F.normalize_prob(raw)), rel_tol=1e-12)


@pytest.mark.parametrize("attach", [False, True])
def test_temporal_blocking_and_sweep_modes_bit_identical(attach):
    """Windows of 1/4/8/16 fused steps, activity-list or dense sweeps, and
    split runs must all give the same bytes (draws are keyed per cell)."""
    h, w, steps = 150, 97, 45
    runs = []
    # the last case grows the window between runs (4 -> 16 -> 8): neighbour
    # activation built for a shorter window is widened before the longer one
    for window, skip, split in [(1, True, None), (4, True, None), (8, True, None),
                                (16, True, None), (8, False, None), (16, False, None),
                                (8, True, (7, 30)), ((4, 16, 8), True, (9, 25))]:
        env = S.make_environment(h, w, seed=12)
        dl = F.DeviceLandscape.from_environment(env)
        b = F.FireBatch((h, w), 2, max_steps=steps, with_jacobian=attach)
        b.set_params(F.pack_params(0.05, 0.12, 0.09, 0.62, 0.45))
        b.set_seeds([5, 6])
        b.reset(S.center_ignition(h, w))
        att = [attach and (s % 3 != 1) for s in range(steps)]
        if split is None:
            b.run(dl, steps, attach=att, window=window, skip_inactive=skip)
        else:
            cuts = [0, *split, steps]
            wins = window if isinstance(window, tuple) else (window,) * (len(cuts) - 1)
            for a0, a1, wn in zip(cuts[:-1], cuts[1:], wins):
                b.run(dl, a1 - a0, attach=att[a0:a1], window=wn, skip_inactive=skip)
        bu, bd = b.unpack()
        runs.append((bu, bd, b.acc.clone(), b.t_ign.clone(),
                     None if b.jac is None else b.jac.clone(), b.series()))
    base = runs[0]
    assert int(base[0].sum()) + int(base[1].sum()) > 100
    for other in runs[1:]:
        assert torch.equal(base[0], other[0]) and torch.equal(base[1], other[1])
        assert torch.equal(base[2], other[2]) and torch.equal(base[3], other[3])
        if attach:
            assert torch.equal(base[4], other[4])
        assert np.array_equal(base[5], other[5])


def test_scheduled_wind_matches_oracle_with_per_step_updates():
    """Config-4 style per-step wind schedule (rotating direction, ramping
    speed) against the oracle fed one WindUpdate per step (kernel.py:505-511)."""
    from paper_2502_18738_b200.device import scheduled_wind_fields, wind_ramp_schedule
    h, w, steps = 96, 80, 40
    env = S.make_environment(h, w, seed=21)
    dl = F.DeviceLandscape.from_environment(env)
    sched = wind_ramp_schedule(steps, 2.0, 12.0, 90.0)
    b = F.FireBatch((h, w), 2, max_steps=steps, with_jacobian=True)
    b.set_params(F.pack_params(0.05, 0.1, 0.07, 0.5, 0.4))
    b.set_seeds([3, 4])
    init = S.center_ignition(h, w)
    b.reset(init)
    b.run(dl, steps, attach=[True] * steps, wind_schedule=sched, window=8)
    arr = S.reference_landscape_arrays(env, O.slope_from_altitude)
    rows = sched.cpu().numpy()
    updates = []
    for t in range(steps):
        v, d = scheduled_wind_fields(arr["wind_speed"], arr["wind_direction"], rows[t])
        updates.append((t + 1, v, d))
    bu, bd = (x.bool().cpu().numpy() for x in b.unpack())
    tg = np.zeros((h, w), bool)
    tg[30:70, 20:60] = True
    _, _, g_dev, _ = b.loss_grad(torch.as_tensor(tg), [steps])
    for m in range(2):
        res = O.run(**arr, params=P([0.05, 0.1, 0.07, 0.5, 0.4]), init=init, steps=steps,
                    seed=3 + m, attach_steps=range(1, steps + 1), wind_schedule=updates)
        assert np.array_equal(bu[m], res.burning) and np.array_equal(bd[m], res.burned)
        np.testing.assert_allclose(b.acc[m].double().cpu().numpy(), res.acc, rtol=RTOL_ACC)
        _, _, _, g = O.combined_loss(res.acc, tg)
        np.testing.assert_allclose(g_dev[m].cpu().numpy(), O.contract(res.jac, g), rtol=RTOL_GRAD)


def _flat(h, w):
    z = np.zeros((h, w))
    return F.Landscape(wind_speed=z.copy(), wind_direction=z.copy(), slope=np.zeros((h, w, 3, 3)),
                       canopy=z.copy(), density=z.copy())


def test_edge_cases_mirror_reference_kernel_tests():
    """The reference's step semantics edge cases (pyrocell tests/test_kernel.py:220-284)."""
    # no burning cells: fixed point, t advances
    land = _flat(5, 5)
    st = F.new_fire_state(np.zeros((5, 5), bool), land)
    F.step_forward(st, land, F.ModelParams(), seed=9)
    assert st.t == 1 and not st.burning.any() and not st.burned.any() and not st.accumulator.any()
    # p_continue = 0 burns out in one step
    init = np.zeros((5, 5), bool)
    init[2, 2] = True
    st = F.new_fire_state(init, land)
    F.step_forward(st, land, F.ModelParams(p_h=0.2, p_continue=0.0), seed=1)
    assert st.burned[2, 2] and not st.burning[2, 2]
    # saturated spread grows one Moore ring per step
    land = _flat(9, 9)
    land.canopy[:] = 3.0
    land.density[:] = 3.0
    init = np.zeros((9, 9), bool)
    init[4, 4] = True
    st = F.new_fire_state(init, land)
    for step in range(1, 4):
        F.step_forward(st, land, F.ModelParams(p_h=1.0, p_continue=1.0), seed=5)
        want = np.zeros((9, 9), bool)
        want[4 - step:5 + step, 4 - step:5 + step] = True
        assert np.array_equal(st.burning | st.burned, want)
    # degenerate grids
    sim = F.run_simulation(_flat(1, 8), F.ModelParams(p_h=0.9, p_continue=1.0),
                           np.eye(1, 8, 3, dtype=bool), 5, seed=2)
    assert sim.state.affected().sum() > 1
    sim = F.run_simulation(_flat(1, 1), F.ModelParams(p_continue=0.0), np.ones((1, 1), bool), 3,
                           seed=2)
    assert sim.state.burned[0, 0] and not sim.state.burning[0, 0]
    # zero steps returns the initial state; errors mirror the reference
    sim = F.run_simulation(_flat(6, 6), F.ModelParams(), np.eye(6, dtype=bool), 0, seed=1)
    assert sim.series == [] and np.array_equal(sim.state.burning, np.eye(6, dtype=bool))
    with pytest.raises(ValueError, match="schedule step"):
        F.run_simulation(_flat(4, 4), F.ModelParams(), np.zeros((4, 4), bool), 5, seed=0,
                         wind_schedule=[F.WindUpdate(7, np.zeros((4, 4)), np.zeros((4, 4)))])
    with pytest.raises(ValueError, match="steps must be"):
        F.run_simulation(_flat(4, 4), F.ModelParams(), np.zeros((4, 4), bool), -1, seed=0)
    with pytest.raises(ValueError, match="factor_site"):
        F.run_simulation(_flat(4, 4), F.ModelParams(), np.zeros((4, 4), bool), 1, seed=0,
                         factor_site="nowhere")


def test_invariants_at_config1_size():
    """Size-independent properties at BASELINE config-1 size (2048^2, 4 of
    the 16 members, 500 steps): exclusivity, burned monotone via counters,
    accumulator support == affected set, p in (0, 1], and one member
    against the CPU oracle (bit-exact states)."""
    n, steps, M = 2048, 500, 4
    env = S.make_environment(n, seed=1)
    dl = F.DeviceLandscape.from_environment(env)
    ph = S.ensemble_ph(16)
    b = F.FireBatch((n, n), M, max_steps=steps)
    b.set_params(np.array([F.pack_params(0.045, 0.131, 0.078, ph[m], 0.3) for m in range(M)]))
    b.set_seeds(list(range(M)))
    init = S.center_ignition(n)
    b.reset(init)
    b.run(dl, steps)
    bu, bd = b.unpack()
    assert not (bu & bd).any()
    aff = (bu | bd).bool()
    acc = b.acc
    assert torch.equal(acc > 0, aff)
    assert float(acc.max()) <= 1.0
    ser = b.series()
    assert np.all(np.diff(ser[:, :, 1], axis=1) >= 0)
    assert np.array_equal(ser[:, -1].sum(-1), aff.reshape(M, -1).sum(-1).cpu().numpy())
    arr = S.reference_landscape_arrays(env, O.slope_from_altitude)
    res = O.run(**arr, params=P([0.045, 0.131, 0.078, ph[2], 0.3]), init=init, steps=steps,
                seed=2, threads=8, want_jac=False)
    assert np.array_equal(bu[2].bool().cpu().numpy(), res.burning)
    assert np.array_equal(bd[2].bool().cpu().numpy(), res.burned)
    np.testing.assert_allclose(acc[2].double().cpu().numpy(), res.acc, rtol=RTOL_ACC)


def _small_calibration_problem():
    size = 32
    env = S.make_environment(size, seed=5)
    arr = S.reference_landscape_arrays(env, O.slope_from_altitude)
    d = load("calibrate_small")
    land = F.Landscape(**arr)
    sched = F.ObservationSchedule([F.Observation(target=t) for t in d["targets"]], 6)
    start = F.ModelParams(c1=0.0, c2=0.0, a=0.0, p_h=0.3, p_continue=0.5)
    return land, S.center_ignition(size), sched, start


def test_device_and_host_calibration_drivers_agree():
    land, init, sched, start = _small_calibration_problem()
    a = F.calibrate(land, init, sched, start, F.StepRings(1, 2, 3), max_epochs=3, base_seed=5,
                    learning_rate=0.05, device_driver=True)
    b = F.calibrate(land, init, sched, start, F.StepRings(1, 2, 3), max_epochs=3, base_seed=5,
                    learning_rate=0.05, device_driver=False)
    ra = np.array([[r.loss, r.bce, r.mse, r.jaccard, r.manhattan] for r in a.records])
    rb = np.array([[r.loss, r.bce, r.mse, r.jaccard, r.manhattan] for r in b.records])
    np.testing.assert_allclose(ra, rb, rtol=1e-12)
    ta = np.array([p.as_array() for _, _, p in a.manifest.trajectory])
    tb = np.array([p.as_array() for _, _, p in b.manifest.trajectory])
    np.testing.assert_allclose(ta, tb, rtol=1e-12, atol=1e-15)
    assert a.best_params.as_array() == pytest.approx(b.best_params.as_array(), rel=1e-12)


def test_calibration_aborts_epoch_on_non_finite_gradient(monkeypatch):
    """calibration.py:217-221 (fault injection as in tests/test_calibrate.py:165-187)."""
    land, init, sched, start = _small_calibration_problem()
    orig = F.FireBatch.loss_grad
    calls = {"n": 0}

    def faulty(self, *a, **kw):
        out = orig(self, *a, **kw)
        calls["n"] += 1
        if calls["n"] == 2:  # second iteration of the first epoch
            out[2].fill_(float("nan"))
        return out

    monkeypatch.setattr(F.FireBatch, "loss_grad", faulty)
    res = F.calibrate(land, init, sched, start, F.StepRings(1, 2, 3), max_epochs=2, base_seed=5,
                      learning_rate=0.05)
    assert res.aborted_epochs and res.aborted_epochs[0][0] == 1
    assert "non-finite gradient" in res.aborted_epochs[0][1]
    epochs = [r.epoch for r in res.records]
    assert epochs.count(2) == 3  # the next epoch runs in full


def test_ensemble_calibrator_gradient_sum_and_adam():
    """Config-4 iteration on a small case: summed member gradients equal the
    sum of the oracle's per-member gradients, and the shared parameters get
    the reference AdamW + clamp step (calibration.py:43-64)."""
    from paper_2502_18738_b200.device import scheduled_wind_fields, wind_ramp_schedule
    from paper_2502_18738_b200.ensemble import EnsembleCalibrator
    h, w, steps = 64, 72, 30
    env = S.make_environment(h, w, seed=8)
    dl = F.DeviceLandscape.from_environment(env)
    sched = wind_ramp_schedule(steps, 2.0, 12.0, 90.0)
    init = S.center_ignition(h, w)
    targets = np.zeros((2, h, w), bool)
    targets[0, 26:38, 30:42] = True
    targets[1, 20:44, 24:50] = True
    obs = [15, 30]
    p0 = (0.045, 0.131, 0.078, 0.58, 0.3)
    cal = EnsembleCalibrator(dl, init, torch.as_tensor(targets), obs, [0, 1, 2], p0, steps=steps,
                             wind_schedule=sched, lr=1e-2)
    cal.step()
    arr = S.reference_landscape_arrays(env, O.slope_from_altitude)
    rows = sched.cpu().numpy()
    updates = [(t + 1, *scheduled_wind_fields(arr["wind_speed"], arr["wind_direction"], rows[t]))
               for t in range(steps)]
    total = np.zeros(4)
    for m in range(3):
        res = O.run(**arr, params=P(p0), init=init, steps=steps, seed=m,
                    attach_steps=range(1, steps + 1), wind_schedule=updates)
        total += O.multi_target_grad(res, obs, targets)[1]
    st = {}
    want = np.clip(O.adamw_update(st, np.array(p0[:4]), total, 1e-2), [0, 0, 0, 0.2], 1.0)
    np.testing.assert_allclose(cal.params[:4], want, rtol=1e-9)


@pytest.mark.parametrize("factor_site,slope_sign", [("source", "downhill-positive"),
                                                     ("target", "uphill-positive")])
def test_elevation_mode_options_match_oracle(factor_site, slope_sign):
    """Native elevation mode with factor_site / slope_sign switches
    (kernel.py:155-163, data_io.py:115-131) against the oracle."""
    h, w, steps = 120, 90, 60
    env = S.make_environment(h, w, seed=17)
    dl = F.DeviceLandscape.from_environment(env, factor_site=factor_site, slope_sign=slope_sign)
    init = S.center_ignition(h, w)
    b = F.FireBatch((h, w), 1, max_steps=steps, with_jacobian=True)
    b.set_params(F.pack_params(0.05, 0.12, 0.09, 0.55, 0.5))
    b.set_seeds([9])
    b.reset(init)
    b.run(dl, steps, attach=[True] * steps)
    arr = S.reference_landscape_arrays(env, lambda e, l: O.slope_from_altitude(e, l, slope_sign))
    res = O.run(**arr, params=P([0.05, 0.12, 0.09, 0.55, 0.5]), init=init, steps=steps, seed=9,
                attach_steps=range(1, steps + 1), factor_site=factor_site)
    bu, bd = (x[0].bool().cpu().numpy() for x in b.unpack())
    assert np.array_equal(bu, res.burning) and np.array_equal(bd, res.burned)
    np.testing.assert_allclose(b.acc[0].double().cpu().numpy(), res.acc, rtol=RTOL_ACC)
    tg = np.zeros((h, w), bool)
    tg[40:80, 30:60] = True
    _, _, g_dev, _ = b.loss_grad(torch.as_tensor(tg), [steps])
    _, _, _, g = O.combined_loss(res.acc, tg)
    np.testing.assert_allclose(g_dev[0].cpu().numpy(), O.contract(res.jac, g), rtol=RTOL_GRAD)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_landscape_build_kernel_matches_fp64_preparation(dtype):
    """fc_landscape_build against the fp64 preparation it replaces (torch
    ops in the reference's operation order; slope_from_altitude via the
    oracle for the slope field): env64 exact, fp32 fields equal after one
    rounding, off-grid slopes 0, both slope signs."""
    def forward_slopes(elev, cell_side, sign=1):
        # fp64 torch restatement of slope_from_altitude's forward pairs
        # (data_io.py:92-132): toward E, SW, S, SE, 0 off the grid
        e = elev.to(torch.float64)
        h, w = e.shape
        out = torch.zeros((h, w, 4), dtype=torch.float64, device=e.device)
        for j, (dr, dc) in enumerate(((0, 1), (1, -1), (1, 0), (1, 1))):
            k = math.sqrt(2.0) if dr and dc else 1.0
            r1, c0, c1 = h - dr, max(-dc, 0), w - max(dc, 0)
            src, dst = e[0:r1, c0:c1], e[dr:r1 + dr, c0 + dc:c1 + dc]
            out[0:r1, c0:c1, j] = torch.rad2deg(torch.atan((src - dst) / (k * cell_side)))
        return (-out if sign < 0 else out).to(torch.float32)

    rng = np.random.default_rng(5)
    h, w = 37, 53
    el = (rng.random((h, w)) * 1500).astype(dtype)
    sp = (rng.random((h, w)) * 10).astype(dtype)
    di = (rng.random((h, w)) * 360).astype(dtype)
    ca = rng.choice([-0.3, 0.0, 0.4], (h, w)).astype(dtype)
    de = rng.choice([-0.4, 0.0, 0.3], (h, w)).astype(dtype)
    for sign in ("downhill-positive", "uphill-positive"):
        dl = F.DeviceLandscape.from_elevation(el, sp, di, ca, de, cell_side=30.0, slope_sign=sign)
        t64 = [torch.as_tensor(a.astype(np.float64), device="cuda") for a in (el, sp, di, ca, de)]
        np.testing.assert_array_equal(dl.env64.cpu().numpy(),
                                      np.stack([a.astype(np.float64) for a in (el, sp, di, ca, de)], -1))
        rad = t64[2] * (np.pi / 180.0)
        ref_env = torch.stack([t64[1], t64[1] * torch.cos(rad), t64[1] * torch.sin(rad),
                               (1.0 + t64[3]) * (1.0 + t64[4])], -1).to(torch.float32)
        np.testing.assert_array_equal(dl.env.cpu().numpy(), ref_env.cpu().numpy())
        ref_dir = torch.stack([torch.cos(rad), torch.sin(rad)], -1).to(torch.float32)
        np.testing.assert_array_equal(dl.dir32.cpu().numpy(), ref_dir.cpu().numpy())
        ref_s4 = forward_slopes(t64[0], 30.0, -1 if sign == "uphill-positive" else 1)
        np.testing.assert_array_equal(dl.slope4.cpu().numpy(), ref_s4.cpu().numpy())
        # the oracle's slope_from_altitude (reference semantics) agrees in fp32
        s33 = O.slope_from_altitude(el.astype(np.float64), 30.0, sign)
        for j, (dr, dc) in enumerate(((0, 1), (1, -1), (1, 0), (1, 1))):
            np.testing.assert_array_equal(dl.slope4.cpu().numpy()[..., j],
                                          s33[:, :, 1 + dr, 1 + dc].astype(np.float32))


def test_ensemble_runner_host_api_matches_device_batch():
    """EnsembleRunner (host buffers in, host results out; the bench e2e
    call) returns exactly what a FireBatch run on the same inputs holds."""
    from paper_2502_18738_b200.ensemble import EnsembleRunner
    n, m, steps = 160, 3, 60
    env = S.make_environment(n, seed=4)
    env_host = torch.stack([torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)) for a in
                            (env.elevation, env.wind_speed, env.wind_direction, env.canopy,
                             env.density)]).pin_memory()
    init = S.center_ignition(n)
    params = [(0.045, 0.131, 0.078, p, 0.3) for p in (0.5, 0.58, 0.66)]
    seeds = [11, 12, 13]
    r = EnsembleRunner((n, n), m, steps)
    out = None
    for _ in range(2):  # buffers are reused between calls
        out = r(env_host, torch.from_numpy(init.astype(np.uint8)), params, seeds)
    dl = F.DeviceLandscape.from_elevation(*[env_host[i].cuda() for i in range(5)])
    b = F.FireBatch((n, n), m, max_steps=steps)
    b.set_params(np.array([F.pack_params(*p) for p in params]))
    b.set_seeds(seeds)
    b.reset(init)
    b.run(dl, steps)
    bu, bd = b.unpack()
    np.testing.assert_array_equal(out.burning, bu.cpu().numpy())
    np.testing.assert_array_equal(out.burned, bd.cpu().numpy())
    np.testing.assert_array_equal(out.accumulator, b.acc.cpu().numpy())
    np.testing.assert_array_equal(out.series, b.series())


def test_state_export_pinned_and_written_flags():
    """fc_state_export into pinned host memory (device-mapped) and into
    device tensors equals fc_state_unpack + the acc plane; with per-tile
    written flags a reused destination is exact across runs whose fires
    cover different tiles (stale tiles are rewritten, ragged edges kept)."""
    n, m = 200, 2
    env = S.make_environment(n, seed=8)
    dl = F.DeviceLandscape.from_environment(env)
    g = F.FireBatch((n, n), m, max_steps=80)
    dest = [torch.zeros((m, n, n), dtype=dt, pin_memory=True)
            for dt in (torch.uint8, torch.uint8, torch.float32)]
    written = torch.zeros((m, g.grid.tiles_y, g.grid.tiles_x), dtype=torch.uint8, device="cuda")
    init_a = S.center_ignition(n)
    init_b = np.zeros((n, n), dtype=bool)
    init_b[190:193, 5:8] = True                      # bottom-left edge tile row
    for ph, steps, init in ((0.9, 80, init_a), (0.4, 15, init_b), (0.9, 30, init_a)):
        g.set_params(np.array([F.pack_params(0.045, 0.131, 0.078, ph, 0.3)] * m))
        g.set_seeds([3, 4])
        g.reset(init)
        g.run(dl, steps)
        bu, bd = g.unpack()
        g.export(*dest, written=written)
        dev = [torch.empty_like(d, device="cuda") for d in dest]
        g.export(*dev)
        torch.cuda.synchronize()
        want = (bu.cpu(), bd.cpu(), g.acc.cpu())
        for x, y, z in zip(dest, dev, want):
            assert torch.equal(x, z) and torch.equal(y.cpu(), z)
    with pytest.raises(ValueError):
        g.export(torch.zeros((m, n, n), dtype=torch.uint8), None, None)  # not pinned


@pytest.mark.parametrize("depth", [2, 3])
def test_ensemble_runner_pipelined_submits(depth):
    """submit() tickets (slot ring of 2 or 3, results read depth - 1 calls
    behind as bench.py does, copies overlapping the next calls) return the
    same results as synchronous calls, per submission."""
    from paper_2502_18738_b200.ensemble import EnsembleRunner
    n, m, steps = 128, 2, 40
    envs = []
    for k in range(3):
        env = S.make_environment(n, seed=10 + k)
        envs.append(torch.stack([torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32))
                                 for a in (env.elevation, env.wind_speed, env.wind_direction,
                                           env.canopy, env.density)]).pin_memory())
    init = torch.from_numpy(S.center_ignition(n).astype(np.uint8))
    params = [(0.045, 0.131, 0.078, p, 0.3) for p in (0.55, 0.65)]
    ref = EnsembleRunner((n, n), m, steps, depth=1)
    want = []
    for k in range(5):
        o = ref(envs[k % 3], init, params, [k, k + 7])
        want.append([a.copy() for a in (o.burning, o.burned, o.accumulator, o.series)])
    r = EnsembleRunner((n, n), m, steps, depth=depth)
    tickets, got = [], []
    for k in range(5):
        tickets.append(r.submit(envs[k % 3], init, params, [k, k + 7]))
        if k >= depth - 1:
            o = tickets[k - depth + 1].result()
            got.append([a.copy() for a in (o.burning, o.burned, o.accumulator, o.series)])
    for tk in tickets[len(tickets) - depth + 1:]:
        o = tk.result()
        got.append([a.copy() for a in (o.burning, o.burned, o.accumulator, o.series)])
    assert len(got) == 5
    for g, w in zip(got, want):
        for x, y in zip(g, w):
            np.testing.assert_array_equal(x, y)
    assert any(not np.array_equal(want[0][2], w[2]) for w in want[1:])


def test_loss_tile_skipping_matches_full_scan():
    """fc_loss_grad's tile-skipping path (closed forms for tiles with no fire
    before an observation step) equals the full per-row scan (tile_first
    forced to -1: every tile read), for shared and per-member targets."""
    n, m, steps = 200, 3, 60
    env = S.make_environment(n, seed=6)
    dl = F.DeviceLandscape.from_environment(env)
    b = F.FireBatch((n, n), m, max_steps=steps, with_jacobian=True)
    b.set_params(np.array([F.pack_params(0.045, 0.131, 0.078, p, 0.3) for p in (0.5, 0.6, 0.7)]))
    b.set_seeds([1, 2, 3])
    b.reset(S.center_ignition(n))
    b.run(dl, steps, attach=[True] * steps)
    rng = np.random.default_rng(2)
    tg = torch.zeros((3, n, n), dtype=torch.uint8)
    tg[0, 90:110, 95:120] = 1
    tg[1, 80:125, 85:130] = 1
    tg[2] = torch.from_numpy((rng.random((n, n)) < 0.02).astype(np.uint8))
    obs = [20, 40, 60]
    loss, crop, grad, _ = b.loss_grad(tg, obs)
    saved = b.tile_first.clone()
    b.tile_first.fill_(-1)
    loss_f, crop_f, grad_f, _ = b.loss_grad(tg, obs)
    b.tile_first.copy_(saved)
    np.testing.assert_array_equal(crop.cpu().numpy(), crop_f.cpu().numpy())
    np.testing.assert_allclose(loss.cpu().numpy(), loss_f.cpu().numpy(), rtol=1e-12)
    np.testing.assert_allclose(grad.cpu().numpy(), grad_f.cpu().numpy(), rtol=1e-10, atol=1e-18)
    # per-member targets take the row path; member 0's row equals the shared result
    tgm = tg[:, None].expand(3, m, n, n).contiguous()
    loss_m, _, grad_m, _ = b.loss_grad(tgm, obs)
    np.testing.assert_allclose(loss_m.cpu().numpy(), loss.cpu().numpy(), rtol=1e-12)
    np.testing.assert_allclose(grad_m.cpu().numpy(), grad.cpu().numpy(), rtol=1e-10, atol=1e-18)
    # and the oracle agrees (fp64 reference loss of member 0's accumulator)
    acc0 = b.acc[0].double().cpu().numpy()
    t0 = b.t_ign[0].cpu().numpy()
    tot = 0.0
    for s_, o in enumerate(obs):
        x = np.where(t0 < o, acc0, 0.0)
        bce, mse, _, _ = O.combined_loss(x, tg[s_].numpy())
        tot += bce + mse
    assert math.isclose(float(loss[0, 0]), tot, rel_tol=1e-10)


def test_reused_batch_gradients_match_fresh_batch():
    """reset() does not clear the Jacobian plane (every ignition writes its J,
    zero on unattached steps): a batch reused after a larger fire gives the
    same loss/gradients and contraction as a fresh one, with partial attach."""
    n, steps = 128, 40
    env = S.make_environment(n, seed=8)
    dl = F.DeviceLandscape.from_environment(env)
    attach = [(k % 3) == 0 for k in range(steps)]
    tg = torch.zeros((1, n, n), dtype=torch.uint8)
    tg[0, 50:80, 50:80] = 1

    def run(b, seed, ph):
        b.set_params(F.pack_params(0.045, 0.131, 0.078, ph, 0.3))
        b.set_seeds([seed])
        b.reset(S.center_ignition(n))
        b.run(dl, steps, attach=attach)
        loss, _, grad, _ = b.loss_grad(tg, [steps])
        g = torch.ones((1, n, n), dtype=torch.float64, device="cuda") * 1e-3
        return loss.cpu().numpy(), grad.cpu().numpy(), b.contract(g).cpu().numpy()

    used = F.FireBatch((n, n), 1, max_steps=steps, with_jacobian=True)
    run(used, 1, 0.9)              # a large fire first: J written over a wide area
    got = run(used, 2, 0.4)        # then a small one on the same planes
    want = run(F.FireBatch((n, n), 1, max_steps=steps, with_jacobian=True), 2, 0.4)
    for a_, b_ in zip(got, want):
        np.testing.assert_array_equal(a_, b_)


@pytest.mark.parametrize("rng", ["splitmix", "philox"])
def test_ordered_ensemble_lists_match_dense_sweep(rng):
    """Ensembles (>= 4 members) order each launch's activity list by work
    estimate and activate neighbours by distance; the result must equal the
    dense sweep byte for byte (attached, both RNGs), and for the keyed
    SplitMix draws a member must equal the CPU oracle."""
    h, w, steps, M = 190, 170, 70, 6
    outs = []
    for skip in (True, False):
        _, arr, p, init, b = _oracle_vs_device(h, w, steps, 21, True, members=M, skip=skip,
                                               rng=rng)
        outs.append(b)
    a, d = outs
    assert torch.equal(a.planes, d.planes)
    assert torch.equal(a.acc, d.acc) and torch.equal(a.t_ign, d.t_ign)
    assert torch.equal(a.jac, d.jac)
    assert np.array_equal(a.series(), d.series())
    if rng == "splitmix":
        res = O.run(**arr, params=p, init=init, steps=steps, seed=21 + 4,
                    attach_steps=range(1, steps + 1), threads=4)
        bu, bd = (x.bool().cpu().numpy() for x in a.unpack())
        assert np.array_equal(bu[4], res.burning) and np.array_equal(bd[4], res.burned)


def test_c1_full_size_members_match_oracle():
    """BASELINE config 1 at full size (16 members x 2048^2 x 500 steps,
    K = 8 windows, ordered lists, persistent CTAs taking several tile groups
    each): two runs are byte-identical and members 0 and 11 equal the CPU
    oracle (states bit-exact, acc within RTOL_ACC).  At this size tiles of
    one launch are processed after their neighbours' new states are written,
    which the small cases above do not exercise."""
    H, M, STEPS = 2048, 16, 500
    env = S.make_environment(H, seed=1)
    ph = S.ensemble_ph(M)
    params = [(0.045, 0.131, 0.078, float(p), 0.3) for p in ph]
    init = S.center_ignition(H)
    b = F.FireBatch((H, H), M, max_steps=STEPS)
    b.set_params(np.array([F.pack_params(*p) for p in params]))
    b.set_seeds(list(range(M)))
    dl = F.DeviceLandscape.from_environment(env)
    runs = []
    for _ in range(2):
        b.reset(init)
        b.run(dl, STEPS, window=8)
        bu, bd = b.unpack()
        runs.append((bu.cpu().numpy(), bd.cpu().numpy(), b.acc.cpu().numpy(), b.series()))
    for x, y in zip(*runs):
        assert np.array_equal(x, y)
    bu, bd, acc, ser = runs[0]
    arr = S.reference_landscape_arrays(env, O.slope_from_altitude)
    for m in (0, 11):
        p = P(params[m])
        res = O.run(**arr, params=p, init=init, steps=STEPS, seed=m,
                    threads=os.cpu_count() or 1, want_jac=False)
        assert np.array_equal(bu[m].astype(bool), res.burning)
        assert np.array_equal(bd[m].astype(bool), res.burned)
        assert np.array_equal(ser[m], res.series)
        np.testing.assert_allclose(acc[m], res.acc, rtol=RTOL_ACC, atol=0)


def _final(b):
    bu, bd = b.unpack()
    out = [bu, bd, b.acc.clone(), b.t_ign.clone(), torch.as_tensor(b.series())]
    if b.jac is not None:
        out.append(b.jac.clone())
    return out


def test_c3_full_size_window_and_sweep_invariance():
    """BASELINE config 3 size (16384^2, 8 random 5x5 fires, sigma x32
    landscape): one step per launch (no halo re-evolution), 8 and 16 fused
    steps with activity lists, and 8 fused steps with the dense sweep give
    byte-identical states, accumulators, ignition steps and series."""
    n, steps = 16384, 240
    e = S.make_environment_torch(n, n, seed=3)
    dl = F.DeviceLandscape.from_elevation(e["elevation"], e["wind_speed"], e["wind_direction"],
                                          e["canopy"], e["density"])
    del e
    init = torch.as_tensor(S.random_blocks(n, n, 8, 5, seed=3).astype(np.uint8), device="cuda")
    b = F.FireBatch((n, n), 1, max_steps=steps)
    b.set_params(F.pack_params(0.045, 0.131, 0.078, 0.58, 0.3))
    b.set_seeds([3])
    ref = None
    for k, skip in ((1, True), (8, True), (16, True), (8, False)):
        b.reset(init)
        b.run(dl, steps, window=k, skip_inactive=skip)
        got = _final(b)
        if ref is None:
            ref = got
            assert int(got[0].sum()) > 0
        else:
            for x, y in zip(got, ref):
                assert torch.equal(x, y), (k, skip)


def test_c4_shape_window_invariance_with_schedule():
    """Config-4 shape (1024^2, rotating/ramping device wind schedule, every
    step attached) with 48 members: K = 1 and K = 8 launches give identical
    states, accumulators, ignition steps, Jacobians and series."""
    n, m, steps = 1024, 48, 200
    env = S.make_environment(n, seed=4)
    dl = F.DeviceLandscape.from_environment(env)
    sched = F.wind_ramp_schedule(steps)
    init = S.center_ignition(n)
    b = F.FireBatch((n, n), m, max_steps=steps, with_jacobian=True)
    ph = S.ensemble_ph(m)
    b.set_params(np.array([F.pack_params(0.045, 0.131, 0.078, float(p), 0.3) for p in ph]))
    b.set_seeds(list(range(100, 100 + m)))
    ref = None
    for k in (1, 8):
        b.reset(init)
        b.run(dl, steps, window=k, attach=[True] * steps, wind_schedule=sched)
        got = _final(b)
        if ref is None:
            ref = got
        else:
            for x, y in zip(got, ref):
                assert torch.equal(x, y), k


@pytest.mark.parametrize("per_member", [False, True])
def test_lazy_reset_equals_full_init(per_member):
    """fc_state_reset (rewrites acc / t_ign only in tiles that held fire)
    leaves exactly the state fc_state_init writes, after runs whose fires
    covered other tiles; ragged grid, broadcast and per-member masks."""
    h, w, m = 150, 230, 3
    env = S.make_environment(h, w, seed=9)
    dl = F.DeviceLandscape.from_environment(env)
    rng = np.random.default_rng(5)
    masks = [(rng.random((m, h, w)) < 0.002) if per_member else (rng.random((h, w)) < 0.002)
             for _ in range(3)]
    used = F.FireBatch((h, w), m, max_steps=60)
    used.set_params(np.array([F.pack_params(0.045, 0.131, 0.078, 0.9, 0.5)] * m))
    used.set_seeds([1, 2, 3])
    for k, mask in enumerate(masks):
        used.reset(mask)
        fresh = F.FireBatch((h, w), m, max_steps=60)
        fresh.reset(mask)
        assert torch.equal(used.acc, fresh.acc) and torch.equal(used.t_ign, fresh.t_ign)
        assert torch.equal(used.planes, fresh.planes)
        assert torch.equal(used.tile_first, fresh.tile_first)
        used.run(dl, 40 - 10 * k)
    # an external write forces the next reset to rewrite every cell
    used.acc.fill_(0.5)
    used.mark_cells_dirty()
    used.reset(masks[0])
    fresh = F.FireBatch((h, w), m, max_steps=60)
    fresh.reset(masks[0])
    assert torch.equal(used.acc, fresh.acc) and torch.equal(used.t_ign, fresh.t_ign)


def test_no_fire_run_and_export():
    """An empty initial mask: every launch finds an empty activity list; the
    state, accumulator, series and export stay zero, for list and dense
    sweeps, and a later reset with fire runs normally (equals a fresh batch)."""
    h, w, m = 100, 130, 2
    env = S.make_environment(h, w, seed=3)
    dl = F.DeviceLandscape.from_environment(env)
    for skip in (True, False):
        b = F.FireBatch((h, w), m, max_steps=40)
        b.set_params(np.array([F.pack_params(0.045, 0.131, 0.078, 0.9, 0.5)] * m))
        b.set_seeds([1, 2])
        b.reset(np.zeros((h, w), dtype=bool))
        b.run(dl, 20, skip_inactive=skip)
        bu, bd = b.unpack()
        assert not bu.any() and not bd.any() and not b.acc.any()
        assert not np.asarray(b.series()).any()
        dest = [torch.zeros((m, h, w), dtype=dt, pin_memory=True)
                for dt in (torch.uint8, torch.uint8, torch.float32)]
        b.export(*dest)
        torch.cuda.synchronize()
        assert not any(bool(x.any()) for x in dest)
        b.reset(S.center_ignition(h, w))
        b.run(dl, 20, skip_inactive=skip)
        f = F.FireBatch((h, w), m, max_steps=40)
        f.set_params(np.array([F.pack_params(0.045, 0.131, 0.078, 0.9, 0.5)] * m))
        f.set_seeds([1, 2])
        f.reset(S.center_ignition(h, w))
        f.run(dl, 20, skip_inactive=skip)
        for x, y in zip(_final(b), _final(f)):
            assert torch.equal(x, y)


def test_tape_blocks_api():
    """The reference's TapeBlock API (tape.py:49-103): blocks per attached
    step in step order, rows row-major, recombine() == p_ignite == the
    stored accumulator bit for bit, num_entries == ignitions on attached
    steps, backward_params linear over blocks and over step subsets
    (pyrocell tests/test_tape.py:61-88, 191-198, 220-244 semantics)."""
    d = load("run_rand16")
    land = land_of(d)
    pr = params_of(d)
    init = d["init"]
    steps, seed = int(d["steps"]), int(d["seed"])
    tape = F.Tape(land.shape)
    sim = F.run_simulation(land, pr, init, steps, seed, attach_steps=range(1, steps + 1),
                           tape=tape)
    blocks = tape.blocks
    assert [b.t for b in blocks] == sorted(b.t for b in blocks)
    assert sum(len(b) for b in blocks) == tape.num_entries == \
        int(sim.state.affected().sum() - np.asarray(init, bool).sum())
    for b in blocks:
        order = b.rows * land.shape[1] + b.cols
        assert np.all(np.diff(order) > 0)
        assert np.array_equal(b.recombine(), b.p_ignite)
        assert np.array_equal(b.p_ignite, sim.state.accumulator[b.rows, b.cols])
        assert np.all(b.mask.any(1)) and np.all(b.fp[~b.mask] == 0.0)
    _, g = F.combined_loss(sim.state.accumulator, d["target"])
    full = F.backward_params(tape, g, F.DEFAULT_NORM_C)
    total = np.zeros(4)
    for b in blocks:
        total += F.backward_params(F.Tape(tape.shape, blocks=[b]), g, F.DEFAULT_NORM_C)
    np.testing.assert_allclose(total, full, rtol=1e-12, atol=1e-15)
    # hand-made copies of the blocks (no device record) give the same sums
    loose = [F.TapeBlock(**{k: getattr(b, k) for k in ("t", "rows", "cols", "p_ignite", "mask",
                                                           "fp", "raw", "rest", "vw", "cosm1",
                                                           "slope", "veg1", "den1")})
             for b in blocks]
    np.testing.assert_allclose(F.backward_params(F.Tape(tape.shape, blocks=loose), g,
                                                 F.DEFAULT_NORM_C), full, rtol=1e-10)
    # a run attaching only steps 2 and 5 equals the sum of those blocks
    part = F.Tape(land.shape)
    sim2 = F.run_simulation(land, pr, init, steps, seed, attach_steps=[2, 5], tape=part)
    assert np.array_equal(sim2.state.accumulator, sim.state.accumulator)
    want = sum(F.backward_params(F.Tape(tape.shape, blocks=[b]), g, F.DEFAULT_NORM_C)
               for b in blocks if b.t in (1, 4))
    np.testing.assert_allclose(F.backward_params(part, g, F.DEFAULT_NORM_C), want, rtol=1e-12)


def test_fire_model_algorithm1_reproduces_reference_calibration():
    """Algorithm 1 driven through the torch FireModel --
    model.reset(seed), model.step / model.run with check_if_attach,
    loss.backward(), torch.optim.Adam, clamp_, reset(seed=epoch_seed) --
    reproduces the parameter trajectory of the reference's own calibrate()
    (tests/golden/calibrate_small.npz, written by pyrocell) within 1e-5."""
    from paper_2502_18738_b200.torch_model import FireModel, combined_loss_torch
    d = load("calibrate_small")
    size = int(d["size"])
    env = S.make_environment(size, seed=5)
    arr = S.reference_landscape_arrays(env, O.slope_from_altitude)
    dl = F.DeviceLandscape.from_slope_tensor(arr["wind_speed"], arr["wind_direction"],
                                             arr["slope"], arr["canopy"], arr["density"])
    targets = [torch.as_tensor(t) for t in d["targets"]]
    rings, interval = F.StepRings(1, 2, 3), 6
    model = FireModel(dl, S.center_ignition(size), c1=0.0, c2=0.0, a=0.0, p_h=0.3,
                      p_continue=0.5, seed=0)
    opt = torch.optim.Adam([model.c_1, model.c_2, model.a, model.p_h], lr=0.05)
    traj = []
    for epoch in range(1, 4):
        epoch_seed = F.derive_epoch_seed(5, epoch)
        model.reset(seed=epoch_seed)
        for it in range(1, len(targets) + 1):
            n = it * interval
            if it % 2:  # per-step calls, as written in Algorithm 1
                for step in range(1, n + 1):
                    model.step(attach=F.check_if_attach(step, n, rings))
            else:       # the fused form
                model.run(n, rings=rings)
            loss = combined_loss_torch(model.accumulator, targets[it - 1])
            loss.backward()
            opt.step()
            opt.zero_grad()
            model.clamp_()
            traj.append([epoch, it, model.c_1.item(), model.c_2.item(), model.a.item(),
                         model.p_h.item(), model.p_continue.item()])
            model.reset(seed=epoch_seed)
    np.testing.assert_allclose(np.array(traj), d["trajectory"], rtol=RTOL_GRAD, atol=1e-9)


def test_wind_swap_rebuilds_with_the_landscape_kernel():
    """DeviceLandscape.with_wind (WindUpdate, FireModel.wind) goes through
    fc_landscape_build: the result equals a landscape built from scratch
    with the new wind, plane for plane; the constructor's derived planes
    come from the same kernel."""
    env = S.make_environment(64, 48, seed=8)
    dl = F.DeviceLandscape.from_environment(env)
    rng = np.random.default_rng(3)
    v2 = rng.uniform(0, 12, (64, 48))
    d2 = rng.uniform(0, 360, (64, 48))
    swapped = dl.with_wind(v2, d2)
    fresh = F.DeviceLandscape.from_elevation(env.elevation.astype(np.float64), v2, d2,
                                             env.canopy.astype(np.float64),
                                             env.density.astype(np.float64))
    for name in ("env", "env64", "dir32", "slope4"):
        assert torch.equal(getattr(swapped, name), getattr(fresh, name)), name
    bare = F.DeviceLandscape(fresh.env, fresh.env64)
    assert torch.equal(bare.slope4, fresh.slope4) and torch.equal(bare.dir32, fresh.dir32)


def test_ensemble_runner_refilled_pinned_inputs():
    """The documented pattern of one pinned input buffer refilled between
    pipelined submits: after ticket.wait_inputs() the buffer may
    be rewritten, and every call's result is that of its own inputs."""
    from paper_2502_18738_b200.ensemble import EnsembleRunner
    n, m, steps = 128, 2, 40
    envs = [S.make_environment(n, seed=s) for s in (21, 22, 23)]
    host = lambda e: torch.stack([torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32))
                                  for a in (e.elevation, e.wind_speed, e.wind_direction,
                                            e.canopy, e.density)])
    env_host = torch.empty((5, n, n), dtype=torch.float32).pin_memory()
    init_host = torch.from_numpy(S.center_ignition(n).astype(np.uint8)).pin_memory()
    params = [(0.05, 0.12, 0.08, 0.6, 0.4)] * m
    r = EnsembleRunner((n, n), m, steps, depth=2)
    tickets = []
    for e in envs:
        env_host.copy_(host(e))
        t = r.submit(env_host, init_host, params, [1, 2])
        t.wait_inputs()          # the buffer may be refilled from here on
        tickets.append(t)
    # results of the first two calls are read before their slots are reused
    got = []
    for t in tickets:
        res = t.result()
        got.append((res.burning.copy(), res.accumulator.copy()))
    # the last slot is still valid; earlier ones were overwritten by later
    # submits, so compare each call with a direct device run
    for e, (bu_h, acc_h), t in zip(envs[1:], got[1:], tickets[1:]):
        dl = F.DeviceLandscape.from_environment(e)
        b = F.FireBatch((n, n), m, max_steps=steps)
        b.set_params(np.array([F.pack_params(*p) for p in params]))
        b.set_seeds([1, 2])
        b.reset(S.center_ignition(n))
        b.run(dl, steps)
        np.testing.assert_array_equal(bu_h, b.unpack()[0].cpu().numpy())
        np.testing.assert_array_equal(acc_h, b.acc.cpu().numpy())


def test_integration_stub_runs_the_device_path():
    """The maintainer-side ctypes stub INTEGRATION.md shows
    (tools/pyrocell_firecell_stub.py), executed: same bytes as FireBatch.run
    and the same gradient as FireBatch.contract."""
    import importlib.util
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools",
                        "pyrocell_firecell_stub.py")
    spec = importlib.util.spec_from_file_location("pyrocell_firecell_stub", path)
    stub = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(stub)
    n, steps = 96, 40
    env = S.make_environment(n, seed=13)
    dl = F.DeviceLandscape.from_environment(env)
    runs = []
    for via_stub in (True, False):
        b = F.FireBatch((n, n), 1, max_steps=steps, with_jacobian=True)
        b.set_params(F.pack_params(0.05, 0.12, 0.08, 0.6, 0.4))
        b.set_seeds([9])
        b.reset(S.center_ignition(n))
        if via_stub:
            stub.run_device(b, dl, steps, [1] * steps)
        else:
            b.run(dl, steps, attach=[True] * steps, window=8)
        g = torch.as_tensor(np.random.default_rng(1).standard_normal((1, n, n)))
        grad = stub.contract_device(b, g) if via_stub else b.contract(g)
        runs.append((b.planes.clone(), b.acc.clone(), grad))
    assert torch.equal(runs[0][0], runs[1][0]) and torch.equal(runs[0][1], runs[1][1])
    assert torch.equal(runs[0][2], runs[1][2])


@pytest.mark.parametrize("rng", ["splitmix", "philox"])
def test_dense_burning_regime(rng):
    """Dense regime: half the cells burning at step 0 and p_continue 0.95,
    so most work words are full and every tile is listed.  Windows
    1/4/8/16, list and dense sweeps, attached or not, must give the same
    bytes, and SplitMix member 0 must equal the oracle."""
    h, w, steps = 140, 203, 24
    env = S.make_environment(h, w, seed=21)
    dl = F.DeviceLandscape.from_environment(env)
    init = np.random.default_rng(4).random((h, w)) < 0.5
    pv = (0.05, 0.12, 0.09, 0.3, 0.95)
    runs = []
    # dense sweeps (skip False) with 4- and 8-step windows take dense tiles'
    # continue draws in the sweep (FC_DENSE_TILE_MIN)
    for window, skip, attach in [(1, True, False), (4, True, True), (8, True, False),
                                 (16, True, True), (8, False, True), (4, False, False),
                                 (16, False, False)]:
        b = F.FireBatch((h, w), 2, max_steps=steps, with_jacobian=attach)
        b.set_params(F.pack_params(*pv))
        b.set_seeds([9, 10])
        b.reset(init)
        b.run(dl, steps, attach=[attach] * steps, window=window, skip_inactive=skip, rng=rng)
        bu, bd = b.unpack()
        runs.append((bu, bd, b.acc.clone(), b.t_ign.clone(), b.series()))
    base = runs[0]
    assert int(base[0][0].sum()) > h * w // 5  # the regime: a large share still burning
    for other in runs[1:]:
        for x, y in zip(base[:4], other[:4]):
            assert torch.equal(x, y)
        assert np.array_equal(base[4], other[4])
    if rng == "splitmix":
        # draw injection of the same draws (the reference's uniform_grid
        # tensors) through the dense sweep's in-sweep draws: same bytes
        draws = np.stack([np.stack([np.stack([O.uniform_grid(sd, t, ch, 0, 0, h, w)
                                              for ch in (0, 1)]) for sd in (9, 10)])
                          for t in range(steps)])
        for window in (4, 8):
            b = F.FireBatch((h, w), 2, max_steps=steps)
            b.set_params(F.pack_params(*pv))
            b.set_seeds([9, 10])
            b.reset(init)
            b.run(dl, steps, window=window, skip_inactive=False, rng="inject",
                  draws=torch.as_tensor(draws, device=b.device))
            bu, bd = b.unpack()
            assert torch.equal(bu, base[0]) and torch.equal(bd, base[1])
            assert torch.equal(b.acc, base[2]) and torch.equal(b.t_ign, base[3])
        arr = S.reference_landscape_arrays(env, O.slope_from_altitude)
        ref = O.run(**arr, params=P(pv), init=init, steps=steps, seed=9, attach_steps=())
        assert np.array_equal(base[0][0].bool().cpu().numpy(), ref.burning)
        assert np.array_equal(base[1][0].bool().cpu().numpy(), ref.burned)
        np.testing.assert_allclose(base[2][0].double().cpu().numpy(), ref.acc, rtol=RTOL_ACC)


def test_ensemble_calibrator_graph_replay_equals_eager():
    """EnsembleCalibrator replays one CUDA graph per iteration after the
    first: four graph iterations give the same losses and shared parameters,
    bit for bit, as four eager ones (reset parity, lazy reset, AdamW step
    count all live on the device or repeat per iteration)."""
    from paper_2502_18738_b200.device import wind_ramp_schedule
    from paper_2502_18738_b200.ensemble import EnsembleCalibrator
    h, w, steps = 96, 80, 24
    env = S.make_environment(h, w, seed=9)
    dl = F.DeviceLandscape.from_environment(env)
    sched = wind_ramp_schedule(steps, 2.0, 12.0, 90.0)
    init = S.center_ignition(h, w)
    targets = np.zeros((2, h, w), bool)
    targets[0, 40:56, 32:50] = True
    targets[1, 30:66, 24:58] = True
    runs = []
    for graph in (False, True):
        cal = EnsembleCalibrator(dl, init, torch.as_tensor(targets), [12, 24], [0, 1, 2, 3],
                                 (0.045, 0.131, 0.078, 0.58, 0.3), steps=steps,
                                 wind_schedule=sched, lr=5e-2, graph=graph)
        losses = [cal.step().clone() for _ in range(4)]
        assert cal._graph is None if not graph else cal._graph is not None
        runs.append((torch.stack(losses), cal.shared.clone()))
    assert torch.equal(runs[0][0], runs[1][0])
    assert torch.equal(runs[0][1], runs[1][1])
    assert not torch.equal(runs[0][0][0], runs[0][0][-1])  # the parameters moved


def test_state_jaccard_matches_reference_formula():
    """fc_state_jaccard (bit planes, per member, shared or per-member targets)
    equals losses.py:89-98's jaccard_index over the unpacked grids, including
    the empty/empty case (1.0) and ragged tile edges; the work buffer is left
    zeroed so consecutive calls agree."""
    h, w, steps, M = 77, 133, 30, 3
    env = S.make_environment(h, w, seed=13)
    dl = F.DeviceLandscape.from_environment(env)
    b = F.FireBatch((h, w), M, max_steps=steps)
    b.set_params(F.pack_params(0.05, 0.12, 0.09, 0.62, 0.45))
    b.set_seeds([1, 2, 3])
    b.reset(S.center_ignition(h, w))
    b.run(dl, steps)
    bu, bd = b.unpack()
    aff = (bu | bd).bool().cpu().numpy()
    rng = np.random.default_rng(5)
    shared = rng.random((h, w)) < 0.1
    shared[30:50, 50:90] = True
    per = rng.random((M, h, w)) < 0.05

    def ref(a, t):
        u = int(np.count_nonzero(a | t))
        return 1.0 if u == 0 else int(np.count_nonzero(a & t)) / u
    for _ in range(2):
        got = b.jaccard(torch.as_tensor(shared)).cpu().numpy()
        assert [float(x) for x in got] == [ref(aff[m], shared) for m in range(M)]
    got = b.jaccard(torch.as_tensor(per)).cpu().numpy()
    assert [float(x) for x in got] == [ref(aff[m], per[m]) for m in range(M)]
    e = F.FireBatch((h, w), 1, max_steps=1)
    e.reset(np.zeros((h, w), bool))
    assert float(e.jaccard(torch.zeros((h, w), dtype=torch.uint8))[0]) == 1.0
