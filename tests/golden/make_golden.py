"""Generate tests/golden/ fixtures by running the REFERENCE itself.

Run here (the build container, where /root/reference exists):
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports the reference package (pyrocell 0.1.0, pure NumPy) from
/root/reference/pkg/src, runs it on seeded inputs, and freezes its outputs
into small .npz files plus golden.json.  Nothing at test/bench time reads
/root/reference; the fixtures are what travel.  Inputs of the small cases
are stored in the fixtures; the config-0 cases store the fingerprint of the
environment produced by paper_2502_18738_b200.synthetic (deterministic
NumPy/SciPy) and regenerate it.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

import pyrocell as P  # noqa: E402  (the reference)
from pyrocell.data_io import slope_from_altitude  # noqa: E402

from paper_2502_18738_b200 import synthetic as S  # noqa: E402


def rand_land(n, m, seed, max_wind=5.0):
    """Small random landscape (our own generator; arrays stored in the fixture)."""
    rng = np.random.default_rng([seed, 77])
    alt = rng.uniform(0.0, 60.0, (n, m))
    return dict(wind_speed=rng.uniform(0.0, max_wind, (n, m)),
                wind_direction=rng.uniform(0.0, 360.0, (n, m)),
                slope=slope_from_altitude(alt, 30.0),
                canopy=rng.uniform(-0.3, 0.3, (n, m)),
                density=rng.uniform(-0.3, 0.3, (n, m)),
                altitude=alt)


def to_land(d):
    return P.Landscape(wind_speed=d["wind_speed"], wind_direction=d["wind_direction"],
                       slope=d["slope"], canopy=d["canopy"], density=d["density"])


def params_arr(p):
    return np.array([p.c1, p.c2, p.a, p.p_h, p.p_continue])


def save(name, **arrays):
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **arrays)


def run_case(name, land_d, params, init, steps, seed, attach=(), target=None,
             factor_site="target", slope_units="degrees", wind=None):
    land = to_land(land_d)
    tape = P.Tape(land.shape)
    sched = []
    if wind is not None:
        sched = [P.WindUpdate(wind[0], wind[1], wind[2])]
    sim = P.run_simulation(land, params, init, steps, seed, wind_schedule=sched,
                           attach_steps=attach, tape=tape, factor_site=factor_site,
                           slope_units=slope_units)
    out = dict(land_d)
    out.update(params=params_arr(params), init=init, steps=steps, seed=seed,
               attach=np.array(sorted(attach), dtype=np.int64),
               burning=sim.state.burning, burned=sim.state.burned,
               acc=sim.state.accumulator,
               series=np.array([[s.burning, s.burned] for s in sim.series], np.int64).reshape(-1, 2),
               num_entries=tape.num_entries)
    if wind is not None:
        out.update(wind_at=wind[0], wind_speed2=wind[1], wind_direction2=wind[2])
    if target is not None:
        bd, g = P.combined_loss(sim.state.accumulator, target)
        grad = P.backward_params(tape, g, P.DEFAULT_NORM_C)
        out.update(target=target, bce=bd.bce_term, mse=bd.mse_term,
                   crop=np.array(bd.crop_window), grad=grad, dl_dacc=g)
    save(name, **out)
    return sim, tape


def main():
    meta = {}
    # ------------------------------------------------------------- RNG
    meta["uniform_grid_99_4_I_10_20_5_6"] = P.uniform_grid(99, 4, P.Channel.IGNITE, 10, 20, 5, 6).tolist()
    g = P.uniform_grid(5, 1, P.Channel.CONTINUE, 0, 0, 40, 40)
    meta["uniform_grid_5_1_C_40x40_sum"] = float(g.sum())
    meta["uniform_grid_5_1_C_40x40_first"] = g[13, 7:18].tolist()
    big = P.uniform_grid(2**40 + 3, 123, P.Channel.IGNITE, 70000, 3, 2, 3)
    meta["uniform_grid_bigseed"] = big.tolist()
    meta["epoch_seeds"] = [[b, e, P.derive_epoch_seed(b, e)]
                           for b, e in [(0, 0), (0, 1), (42, 0), (42, 1), (7, 3), (2**63, 5),
                                        (2**64 - 1, 9), (123456789, 1000)]]
    # --------------------------------------------------------- slope
    rng = np.random.default_rng(11)
    alt = rng.uniform(0, 900, (7, 9))
    save("slope", altitude=alt, slope=slope_from_altitude(alt, 30.0),
         slope_up=slope_from_altitude(alt, 25.0, "uphill-positive"))
    # --------------------------------------------------- attachment plans
    plans = []
    rng = np.random.default_rng(2)
    cases = [(10, (1, 2, 2)), (7, (0, 0, 7)), (7, (0, 0, 0)), (100, (2, 5, 10)),
             (100, (0, 0, 100)), (25, (2, 5, 10)), (3, (2, 5, 10)), (0, (2, 5, 10))]
    for _ in range(60):
        cases.append((int(rng.integers(0, 60)), tuple(int(x) for x in rng.integers(0, 9, 3))))
    for total, rings in cases:
        plans.append([total, list(rings), list(P.attachment_plan(total, P.StepRings(*rings)))])
    meta["plans"] = plans
    # ------------------------------------------------------------ loss
    rng = np.random.default_rng(1)
    acc = rng.uniform(0.0, 1.0, (16, 18))
    acc[rng.uniform(0, 1, (16, 18)) > 0.6] = 0.0
    y = rng.uniform(0, 1, (16, 18)) > 0.7
    bd, gr = P.combined_loss(acc, y)
    save("loss_random", acc=acc, target=y, bce=bd.bce_term, mse=bd.mse_term,
         crop=np.array(bd.crop_window), grad=gr)
    acc = np.zeros((10, 11))
    acc[2, 3] = 0.5
    y = np.zeros((10, 11), dtype=bool)
    y[7, 1] = True
    bd, gr = P.combined_loss(acc, y)
    save("loss_crop", acc=acc, target=y, bce=bd.bce_term, mse=bd.mse_term,
         crop=np.array(bd.crop_window), grad=gr)
    # ------------------------------------------------------ small runs
    land = rand_land(16, 16, 42)
    params = P.ModelParams(c1=0.08, c2=0.12, a=0.05, p_h=0.4, p_continue=0.7)
    init = np.zeros((16, 16), bool)
    init[7:9, 7:9] = True
    tgt = P.run_simulation(to_land(land), P.ModelParams(p_h=0.5, p_continue=0.7), init, 12,
                           seed=999).state.affected()
    run_case("run_rand16", land, params, init, 12, 101, attach=range(1, 13), target=tgt)

    land = rand_land(9, 9, 21, max_wind=4.0)
    init = np.zeros((9, 9), bool)
    init[4, 4] = True
    run_case("run_rand9_source", land,
             P.ModelParams(c1=0.1, c2=0.15, a=0.08, p_h=0.5, p_continue=0.6), init, 6, 78,
             factor_site="source")

    land = rand_land(12, 12, 62, max_wind=3.0)
    init = np.zeros((12, 12), bool)
    init[5:7, 5:7] = True
    r2 = np.random.default_rng(5)
    wind = (5, r2.uniform(4, 8, (12, 12)), r2.uniform(0, 360, (12, 12)))
    tgt = np.zeros((12, 12), bool)
    tgt[2:11, 2:11] = True
    run_case("run_windswap", land, P.ModelParams(c1=0.12, c2=0.1, a=0.06, p_h=0.45,
                                                 p_continue=0.7),
             init, 10, 72, attach=range(1, 11), target=tgt, wind=wind)

    land = rand_land(12, 12, 61)
    init = np.zeros((12, 12), bool)
    init[5:7, 5:7] = True
    tgt = np.zeros((12, 12), bool)
    tgt[3:10, 3:10] = True
    run_case("run_source_grad", land, P.ModelParams(c1=0.1, c2=0.1, a=0.08, p_h=0.45,
                                                    p_continue=0.7),
             init, 10, 71, attach=range(1, 11), target=tgt, factor_site="source")

    land = rand_land(11, 13, 5)
    land_rad = dict(land)
    land_rad["slope"] = np.radians(land["slope"])
    init = np.zeros((11, 13), bool)
    init[5, 6] = True
    run_case("run_radians", land_rad, P.ModelParams(c1=0.1, c2=0.1, a=0.2, p_h=0.6,
                                                    p_continue=0.6),
             init, 8, 3, attach=(2, 3, 7), target=np.ones((11, 13), bool),
             slope_units="radians")

    land = rand_land(12, 12, 10)
    init = np.zeros((12, 12), bool)
    init[6, 6] = True
    full = P.run_simulation(to_land(land), P.ModelParams(p_h=0.5, p_continue=0.6), init, 8, 13)
    run_case("run_partial_attach", land, P.ModelParams(p_h=0.5, p_continue=0.6), init, 8, 13,
             attach=(2, 5), target=full.state.affected())

    # zero-wind / flat structural zero cases (tape.py semantics)
    land = rand_land(12, 12, 8)
    land["wind_speed"] = np.zeros((12, 12))
    land["slope"] = np.random.default_rng(8).uniform(-5, 5, (12, 12, 3, 3))
    init = np.zeros((12, 12), bool)
    init[5:7, 5:7] = True
    tgt = np.zeros((12, 12), bool)
    tgt[4:9, 4:9] = True
    run_case("run_windless", land, P.ModelParams(c1=0.1, c2=0.1, a=0.1, p_h=0.5,
                                                 p_continue=0.7),
             init, 10, 314, attach=range(1, 11), target=tgt)

    # ragged 37x53 random landscape, longer run, all attached
    land = rand_land(37, 53, 3, max_wind=6.0)
    init = np.zeros((37, 53), bool)
    init[18, 26] = True
    init[0, 0] = True
    init[36, 52] = True
    tgt = np.zeros((37, 53), bool)
    tgt[10:30, 15:40] = True
    run_case("run_ragged", land, P.ModelParams(c1=0.07, c2=0.1, a=0.05, p_h=0.55,
                                               p_continue=0.6),
             init, 30, 2024, attach=range(1, 31), target=tgt)

    # saturated spread: fp hits 1.0
    n = 9
    sat = dict(wind_speed=np.zeros((n, n)), wind_direction=np.zeros((n, n)),
               slope=np.zeros((n, n, 3, 3)), canopy=np.full((n, n), 3.0),
               density=np.full((n, n), 3.0))
    init = np.zeros((n, n), bool)
    init[4, 4] = True
    run_case("run_saturated", sat, P.ModelParams(p_h=1.0, p_continue=1.0), init, 3, 5)

    # ------------------------------------------------------ config 0
    for name, size, steps in (("c0_small", 64, 60), ("c0", 512, 200)):
        env = S.make_environment(size, seed=0)
        arr = S.reference_landscape_arrays(env, slope_from_altitude)
        land = P.Landscape(**arr)
        p = P.ModelParams(**S.DEFAULT_BENCH_PARAMS)
        init = S.center_ignition(size)
        sim = P.run_simulation(land, p, init, steps, seed=0)
        aff = sim.state.affected()
        idx = np.flatnonzero(aff)
        save(name, fingerprint=env.fingerprint(), size=size, steps=steps,
             burning=np.packbits(sim.state.burning), burned=np.packbits(sim.state.burned),
             acc_idx=idx.astype(np.int64), acc_val=sim.state.accumulator.ravel()[idx],
             series=np.array([[s.burning, s.burned] for s in sim.series], np.int64))
        meta[name + "_fingerprint"] = env.fingerprint()

    # ------------------------------------------ config 2 literal iteration
    size = 128
    env = S.make_environment(size, seed=2)
    arr = S.reference_landscape_arrays(env, slope_from_altitude)
    land = P.Landscape(**arr)
    init = S.center_ignition(size)
    hidden = P.ModelParams(**S.HIDDEN_C2_PARAMS)
    obs = (25, 50, 75, 100)
    tsim = P.run_simulation(land, hidden, init, 100, seed=7, snapshot_every=25)
    targets = np.stack([st.affected() for _, st in tsim.snapshots])
    p0 = P.ModelParams(**S.DEFAULT_BENCH_PARAMS)
    it_seed = P.derive_epoch_seed(7, 1)
    tape = P.Tape(land.shape)
    sim = P.run_simulation(land, p0, init, 100, it_seed, attach_steps=range(1, 101), tape=tape,
                           snapshot_every=25)
    total, grad = 0.0, np.zeros(4)
    for (s, st), tg in zip(sim.snapshots, targets):
        bd, g = P.combined_loss(st.accumulator, tg)
        total += bd.total
        sub = P.Tape(land.shape, blocks=[b for b in tape.blocks if b.t < s])
        grad += P.backward_params(sub, g, P.DEFAULT_NORM_C)
    save("c2_small", fingerprint=env.fingerprint(), size=size, targets=targets,
         obs=np.array(obs), seed=it_seed, loss=total, grad=grad,
         num_entries=tape.num_entries, acc=sim.state.accumulator,
         burning=sim.state.burning, burned=sim.state.burned)
    meta["c2_small_fingerprint"] = env.fingerprint()

    # --------------------------------------------- calibrate() trajectory
    size = 32
    env = S.make_environment(size, seed=5)
    arr = S.reference_landscape_arrays(env, slope_from_altitude)
    land = P.Landscape(**arr)
    init = S.center_ignition(size)
    star = P.ModelParams(c1=0.15, c2=0.15, a=0.15, p_h=0.5, p_continue=0.5)
    sim = P.run_simulation(land, star, init, 18, seed=71, snapshot_every=6)
    targets = np.stack([st.affected() for _, st in sim.snapshots])
    sched = P.ObservationSchedule([P.Observation(target=t) for t in targets], 6)
    start = P.ModelParams(c1=0.0, c2=0.0, a=0.0, p_h=0.3, p_continue=0.5)
    res = P.calibrate(land, init, sched, start, P.StepRings(1, 2, 3), max_epochs=3,
                      base_seed=5, learning_rate=0.05)
    recs = np.array([[r.epoch, r.iteration, r.loss, r.bce, r.mse, r.jaccard, r.manhattan]
                     for r in res.records])
    traj = np.array([[e, i, p.c1, p.c2, p.a, p.p_h, p.p_continue]
                     for e, i, p in res.manifest.trajectory])
    save("calibrate_small", fingerprint=env.fingerprint(), size=size, targets=targets,
         records=recs, trajectory=traj, best=params_arr(res.best_params),
         best_loss=res.best_loss, epoch_seeds=np.array(res.manifest.epoch_seeds, np.uint64))
    meta["calibrate_small_fingerprint"] = env.fingerprint()

    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(meta, f, indent=1)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
