"""Pins the CPU oracle (oracle/) against the reference's golden vectors
(pyrocell tests/test_rng.py:7-23, tests/test_tape.py:27-28,
tests/test_losses.py:17-21) and against fixtures produced by running the
reference itself (tests/golden/make_golden.py)."""
import math

import numpy as np
import pytest

from golden_util import P, RUN_CASES, case_kwargs, load, meta
from oracle import oracle as O

# pyrocell tests/test_rng.py:7-23
GOLDEN_DRAWS = {
    (0, 0, 0, 0, 0): 0.23286544795475594,
    (0, 0, 0, 0, 1): 0.991448890053859,
    (1, 0, 0, 0, 0): 0.7828598730864468,
    (0, 1, 0, 0, 0): 0.6289335415767472,
    (0, 0, 5, 7, 0): 0.8443854602639748,
    (12345, 99, 120, 250, 1): 0.5958213030105105,
}
GOLDEN_EPOCH_SEEDS = {
    (0, 0): 5197578548964807871,
    (0, 1): 5162896908779471425,
    (42, 0): 12870963724712631011,
    (42, 1): 4771035748442154482,
    (42, 2): 7758384369217865767,
    (2**63, 5): 6872116035820236169,
}


def test_rng_reference_goldens():
    for (seed, t, r, c, ch), want in GOLDEN_DRAWS.items():
        assert O.uniform_draw(seed, t, r, c, ch) == want
    for (b, e), want in GOLDEN_EPOCH_SEEDS.items():
        assert O.derive_epoch_seed(b, e) == want


def test_rng_generated_goldens():
    m = meta()
    assert O.uniform_grid(99, 4, 0, 10, 20, 5, 6).tolist() == m["uniform_grid_99_4_I_10_20_5_6"]
    g = O.uniform_grid(5, 1, 1, 0, 0, 40, 40)
    assert g[13, 7:18].tolist() == m["uniform_grid_5_1_C_40x40_first"]
    assert math.isclose(float(g.sum()), m["uniform_grid_5_1_C_40x40_sum"], rel_tol=1e-15)
    assert O.uniform_grid(2**40 + 3, 123, 0, 70000, 3, 2, 3).tolist() == m["uniform_grid_bigseed"]
    for b, e, want in m["epoch_seeds"]:
        assert O.derive_epoch_seed(b, e) == want


def test_slope_from_altitude():
    d = load("slope")
    np.testing.assert_allclose(O.slope_from_altitude(d["altitude"], 30.0), d["slope"],
                               rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(O.slope_from_altitude(d["altitude"], 25.0, "uphill-positive"),
                               d["slope_up"], rtol=1e-13, atol=1e-13)


def test_attachment_plans():
    for total, rings, want in meta()["plans"]:
        assert list(O.attachment_plan(total, *rings)) == want
    assert O.attachment_plan(10, 1, 2, 2) == (1, 4, 7, 9, 10)   # tests/test_tape.py:27-28


def test_loss_goldens():
    bce, mse, crop, _ = O.combined_loss(np.zeros((8, 8)), np.zeros((8, 8), bool))
    assert math.isclose(bce, math.log(2.0), rel_tol=1e-12) and mse == 0.0
    assert crop == (0, 8, 0, 8)
    for name in ("loss_random", "loss_crop"):
        d = load(name)
        bce, mse, crop, grad = O.combined_loss(d["acc"], d["target"])
        assert math.isclose(bce, float(d["bce"]), rel_tol=1e-12)
        assert math.isclose(mse, float(d["mse"]), rel_tol=1e-12, abs_tol=1e-300)
        assert crop == tuple(int(v) for v in d["crop"])
        np.testing.assert_allclose(grad, d["grad"], rtol=1e-12, atol=1e-15)


@pytest.mark.parametrize("name", RUN_CASES)
def test_run_matches_reference(name):
    d = load(name)
    res = O.run(d["wind_speed"], d["wind_direction"], d["slope"], d["canopy"], d["density"],
                P(d["params"]), d["init"], int(d["steps"]), int(d["seed"]),
                attach_steps=[int(s) for s in d["attach"]], **case_kwargs(name, d))
    assert np.array_equal(res.burning, d["burning"])
    assert np.array_equal(res.burned, d["burned"])
    np.testing.assert_allclose(res.acc, d["acc"], rtol=1e-12, atol=0)
    assert np.array_equal(res.series, d["series"])
    if "grad" in d:
        assert res.n_entries == int(d["num_entries"])
        bce, mse, crop, g = O.combined_loss(res.acc, d["target"])
        assert math.isclose(bce, float(d["bce"]), rel_tol=1e-12)
        np.testing.assert_allclose(g, d["dl_dacc"], rtol=1e-10, atol=1e-15)
        grad = O.contract(res.jac, g)
        np.testing.assert_allclose(grad, d["grad"], rtol=1e-10, atol=1e-14)


def test_windless_structural_zeros():
    d = load("run_windless")
    assert d["grad"][0] == 0.0 and d["grad"][1] == 0.0
    res = O.run(d["wind_speed"], d["wind_direction"], d["slope"], d["canopy"], d["density"],
                P(d["params"]), d["init"], int(d["steps"]), int(d["seed"]),
                attach_steps=[int(s) for s in d["attach"]])
    _, _, _, g = O.combined_loss(res.acc, d["target"])
    grad = O.contract(res.jac, g)
    assert grad[0] == 0.0 and grad[1] == 0.0 and grad[2] != 0.0


def test_threads_bit_identical():
    d = load("run_ragged")
    args = (d["wind_speed"], d["wind_direction"], d["slope"], d["canopy"], d["density"],
            P(d["params"]), d["init"], int(d["steps"]), int(d["seed"]))
    a = O.run(*args, attach_steps=range(1, 31), threads=1)
    b = O.run(*args, attach_steps=range(1, 31), threads=4)
    assert np.array_equal(a.burning, b.burning) and np.array_equal(a.burned, b.burned)
    assert a.acc.tobytes() == b.acc.tobytes() and a.jac.tobytes() == b.jac.tobytes()


def _ref_arrays(size, seed):
    from paper_2502_18738_b200 import synthetic as S
    env = S.make_environment(size, seed=seed)
    return env, S.reference_landscape_arrays(env, O.slope_from_altitude)


@pytest.mark.parametrize("name", ["c0_small", "c0"])
def test_config0_matches_reference(name):
    from paper_2502_18738_b200 import synthetic as S
    d = load(name)
    size, steps = int(d["size"]), int(d["steps"])
    env, arr = _ref_arrays(size, 0)
    assert env.fingerprint() == str(d["fingerprint"])
    res = O.run(**arr, params=P([0.045, 0.131, 0.078, 0.58, 0.3]),
                init=S.center_ignition(size), steps=steps, seed=0, threads=4)
    assert np.array_equal(np.packbits(res.burning), d["burning"])
    assert np.array_equal(np.packbits(res.burned), d["burned"])
    assert np.array_equal(np.flatnonzero(res.affected()), d["acc_idx"])
    np.testing.assert_allclose(res.acc.ravel()[d["acc_idx"]], d["acc_val"], rtol=1e-12)
    assert np.array_equal(res.series, d["series"])


def test_config2_iteration_matches_reference():
    from paper_2502_18738_b200 import synthetic as S
    d = load("c2_small")
    env, arr = _ref_arrays(int(d["size"]), 2)
    assert env.fingerprint() == str(d["fingerprint"])
    res = O.run(**arr, params=P([0.045, 0.131, 0.078, 0.58, 0.3]),
                init=S.center_ignition(int(d["size"])), steps=100, seed=int(d["seed"]),
                attach_steps=range(1, 101), threads=4)
    assert np.array_equal(res.burning, d["burning"]) and np.array_equal(res.burned, d["burned"])
    assert res.n_entries == int(d["num_entries"])
    loss, grad = O.multi_target_grad(res, [int(s) for s in d["obs"]], d["targets"])
    assert math.isclose(loss, float(d["loss"]), rel_tol=1e-12)
    np.testing.assert_allclose(grad, d["grad"], rtol=1e-10)


def oracle_calibrate(arr, init, targets, interval, start, rings, max_epochs, base_seed, lr):
    """Restates calibration.py:123-234 (Algorithm 1) on the oracle."""
    theta = np.array(start[:4], dtype=np.float64)
    pc = start[4]
    opt, records, traj, seeds = {}, [], [], []
    best_loss, best = np.inf, list(start)
    bounds = [(0, 1), (0, 1), (0, 1), (0.2, 1)]
    counts = [int(np.count_nonzero(t)) for t in targets]
    K = len(targets)
    for epoch in range(1, max_epochs + 1):
        seed = O.derive_epoch_seed(base_seed, epoch)
        seeds.append(seed)
        for it in range(1, K + 1):
            total = it * interval
            plan = O.attachment_plan(total, *rings)
            res = O.run(**arr, params=P(list(theta) + [pc]), init=init, steps=total,
                        seed=seed, attach_steps=plan)
            bce, mse, _, g = O.combined_loss(res.acc, targets[it - 1])
            loss = bce + mse
            aff = res.affected()
            inter = np.count_nonzero(aff & targets[it - 1])
            union = np.count_nonzero(aff | targets[it - 1])
            jac = 1.0 if union == 0 else inter / union
            pred = [int(res.series[k * interval - 1].sum()) for k in range(1, it + 1)]
            man = sum(abs(a - b) for a, b in zip(pred, counts[:it]))
            records.append([epoch, it, loss, bce, mse, jac, man])
            used = list(theta) + [pc]
            if it == K and loss < best_loss:
                best_loss, best = loss, used
            grads = O.contract(res.jac, g)
            theta = O.adamw_update(opt, theta, grads, lr)
            theta = np.array([min(max(v, lo), hi) for v, (lo, hi) in zip(theta, bounds)])
            traj.append([epoch, it] + list(theta) + [pc])
    return np.array(records), np.array(traj), best, best_loss, seeds


def test_calibrate_trajectory_matches_reference():
    from paper_2502_18738_b200 import synthetic as S
    d = load("calibrate_small")
    env, arr = _ref_arrays(int(d["size"]), 5)
    assert env.fingerprint() == str(d["fingerprint"])
    rec, traj, best, best_loss, seeds = oracle_calibrate(
        arr, S.center_ignition(int(d["size"])), d["targets"], 6,
        [0.0, 0.0, 0.0, 0.3, 0.5], (1, 2, 3), 3, 5, 0.05)
    assert seeds == [int(s) for s in d["epoch_seeds"]]
    np.testing.assert_allclose(rec, d["records"], rtol=1e-9)
    np.testing.assert_allclose(traj, d["trajectory"], rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(best, d["best"], rtol=1e-9)
    assert math.isclose(best_loss, float(d["best_loss"]), rel_tol=1e-9)


def _small_env(h, w, seed):
    from paper_2502_18738_b200 import synthetic as S
    env = S.make_environment(h, w, seed=seed)
    return S.reference_landscape_arrays(env, O.slope_from_altitude)


def test_oracle_parametric_wind_equals_per_step_updates():
    # wind_params row t == a WindUpdate (kernel.py:422-428) before 1-based
    # step t+1 with fields alpha*V + beta, theta + gamma of the base fields
    arr = _small_env(40, 48, 3)
    steps = 25
    rows = np.stack([1.0 + 0.02 * np.arange(steps), 0.1 * np.arange(steps),
                     3.6 * np.arange(steps)], axis=1)
    init = np.zeros((40, 48), bool)
    init[19:22, 23:26] = True
    p = P([0.045, 0.131, 0.078, 0.58, 0.3])
    a = O.run(**arr, params=p, init=init, steps=steps, seed=4, wind_params=rows,
              attach_steps=range(1, steps + 1))
    upd = [(t + 1, rows[t, 0] * arr["wind_speed"] + rows[t, 1], arr["wind_direction"] + rows[t, 2])
           for t in range(steps)]
    b = O.run(**arr, params=p, init=init, steps=steps, seed=4, wind_schedule=upd,
              attach_steps=range(1, steps + 1))
    assert np.array_equal(a.burning, b.burning) and np.array_equal(a.burned, b.burned)
    assert np.array_equal(a.acc, b.acc) and np.array_equal(a.jac, b.jac)


def test_oracle_origin_crop_equals_full_domain():
    # a crop whose border the fire never reaches, run with its absolute
    # origin, reproduces the full-domain run (draws keyed by absolute cell)
    arr = _small_env(96, 112, 5)
    init = np.zeros((96, 112), bool)
    init[60:63, 70:73] = True
    p = P([0.045, 0.131, 0.078, 0.58, 0.3])
    full = O.run(**arr, params=p, init=init, steps=15, seed=9, attach_steps=range(1, 16))
    r0, r1, c0, c1 = 30, 96, 41, 100
    aff = full.affected()
    assert not aff[r0:r0 + 2].any() and not aff[:, c0:c0 + 2].any()
    crop = {k: (v[r0:r1, c0:c1] if v.ndim == 2 else v[r0:r1, c0:c1]) for k, v in arr.items()}
    part = O.run(**crop, params=p, init=init[r0:r1, c0:c1], steps=15, seed=9,
                 attach_steps=range(1, 16), origin=(r0, c0))
    assert np.array_equal(part.burning, full.burning[r0:r1, c0:c1])
    assert np.array_equal(part.acc, full.acc[r0:r1, c0:c1])
    assert np.array_equal(part.jac, full.jac[r0:r1, c0:c1])
    shifted = O.run(**crop, params=p, init=init[r0:r1, c0:c1], steps=15, seed=9)
    assert not np.array_equal(shifted.burning, part.burning)


def test_oracle_jac_abs_bounds_jac():
    arr = _small_env(32, 32, 7)
    init = np.zeros((32, 32), bool)
    init[15:18, 15:18] = True
    res = O.run(**arr, params=P([0.045, 0.131, 0.078, 0.58, 0.3]), init=init, steps=10, seed=1,
                attach_steps=range(1, 11), want_jac_abs=True)
    assert np.all(res.jac_abs >= np.abs(res.jac) * (1 - 1e-12))
    assert (res.jac_abs > 0).any()
