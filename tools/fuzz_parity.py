"""Randomised parity sweep (GPU box): random grids (1..260 a side, ragged),
members, step counts, windows 1/4/8/16, list or dense sweeps, dataflow on or
off, attached steps, parameters across PARAM_BOUNDS and random ignitions.
Every configuration must give the same bytes as the plain configuration
(one step per launch, activity lists, no dataflow), and member 0 must equal
the CPU oracle (states exact, acc within 1e-5).
python tools/fuzz_parity.py [cases] [seed]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2502_18738_b200 as F  # noqa: E402
from paper_2502_18738_b200 import synthetic as S  # noqa: E402
from golden_util import P  # noqa: E402
from oracle import oracle as O  # noqa: E402


def run_dev(dl, h, w, M, steps, params, seeds, init, attach, window, skip, dataflow, rng="splitmix",
            wind=None):
    b = F.FireBatch((h, w), M, max_steps=steps, with_jacobian=attach, dataflow=dataflow)
    b.set_params(params)
    b.set_seeds(seeds)
    b.reset(init)
    b.run(dl, steps, attach=[attach] * steps, window=window, skip_inactive=skip, rng=rng,
          wind_schedule=wind)
    torch.cuda.synchronize()
    return b


def check_loss(rng, b, res, h, w, steps):
    """fc_loss_grad over 1-4 random observation steps and shared random
    targets against the oracle (combined_loss per step, tape contraction):
    loss within 1e-5; gradient within 1e-5 of its terms' scale plus the
    fp32 Jacobian error model (tests/test_gpu_envelope.py)."""
    S_ = int(rng.integers(1, 5))
    obs = sorted(set(int(v) for v in rng.integers(1, steps + 1, S_)))
    targets = []
    for _ in obs:
        t = rng.random((h, w)) < rng.uniform(0.0, 0.3)
        r, c = int(rng.integers(0, h)), int(rng.integers(0, w))
        t[r:r + int(rng.integers(1, 40)), c:c + int(rng.integers(1, 40))] = True
        targets.append(t)
    loss, _, grad, _ = b.loss_grad(torch.as_tensor(np.stack(targets)), obs)
    total, g_ref = O.multi_target_grad(res, obs, targets)
    g_cell = np.zeros((h, w))
    for s_, tgt in zip(obs, targets):
        acc_s = np.where(res.t_ign < s_, res.acc, 0.0)
        g_cell += np.where(res.t_ign < s_, O.combined_loss(acc_s, tgt)[3], 0.0)
    scale = O.contract(1e-5 * res.jac_abs + res.jac_floor + res.jac_cond, np.abs(g_cell))
    got = grad[0].cpu().numpy() * float(os.environ.get("FUZZ_GRAD_SCALE", "1"))  # sanity: 1.0001 must fail
    ok_l = abs(float(loss[0, 0]) - total) <= 1e-5 * abs(total) + 1e-12
    ok_g = bool(np.all(np.abs(got - g_ref) <= scale + 1e-5 * np.abs(g_ref) + 1e-300))
    return ok_l and ok_g


def fuzz(cases: int, seed: int, log=print, dense: float = 0.0):
    """Run `cases` random configurations; returns the failing ones.  dense:
    share of cases whose initial fire is a random mask of 20-80 % of the
    cells (the dense-tile paths: in-sweep continue draws of dense sweeps),
    drawn from a second generator so the default stream is unchanged."""
    rng = np.random.default_rng(seed)
    rng_dense = np.random.default_rng(seed + 1000003)
    failed = []
    for case in range(cases):
        h, w = int(rng.integers(1, 261)), int(rng.integers(1, 261))
        M = int(rng.choice([1, 2, 3, 5]))
        steps = int(rng.integers(1, 51))
        attach = bool(rng.integers(0, 2))
        window = int(rng.choice([1, 4, 8, 16]))
        skip = bool(rng.integers(0, 3))  # 2:1 lists
        dataflow = bool(rng.integers(0, 2))
        pv = [float(rng.uniform(0, 1)), float(rng.uniform(0, 1)), float(rng.uniform(0, 1)),
              float(rng.uniform(0.2, 1)), float(rng.uniform(0, 1))]
        env = S.make_environment(h, w, seed=int(rng.integers(0, 1 << 30)))
        dl = F.DeviceLandscape.from_environment(env)
        init = np.zeros((h, w), dtype=bool)
        for _ in range(int(rng.integers(1, 6))):
            r, c = int(rng.integers(0, h)), int(rng.integers(0, w))
            k = int(rng.integers(1, 6))
            init[r:r + k, c:c + k] = True
        if dense > 0 and rng_dense.random() < dense:
            init = rng_dense.random((h, w)) < rng_dense.uniform(0.2, 0.8)
        seeds = [int(rng.integers(0, 1 << 62)) for _ in range(M)]
        params = F.pack_params(*pv)
        draw_rng = "philox" if rng.integers(0, 4) == 0 else "splitmix"
        wind = None
        if rng.integers(0, 3) == 0:  # per-step {alpha, beta, gamma} wind schedule
            wind = np.zeros((steps, 4))
            wind[:, 0] = rng.uniform(0.5, 1.5, steps)
            wind[:, 1] = rng.uniform(-2.0, 2.0, steps)
            wind[:, 2] = rng.uniform(-90.0, 90.0, steps)
        wind_dev = None if wind is None else torch.as_tensor(wind, device="cuda")
        cfg = dict(h=h, w=w, M=M, steps=steps, attach=attach, window=window, skip=skip,
                   dataflow=dataflow, rng=draw_rng, wind=wind is not None,
                   params=[round(v, 4) for v in pv])
        try:
            a = run_dev(dl, h, w, M, steps, params, seeds, init, attach, 1, True, False, draw_rng,
                        wind_dev)
            b = run_dev(dl, h, w, M, steps, params, seeds, init, attach, window, skip, dataflow,
                        draw_rng, wind_dev)
            # the current state (the planes hold both launch parities; the
            # final parity depends on the launch count)
            ua, ub = a.unpack(), b.unpack()
            same = (torch.equal(ua[0], ub[0]) and torch.equal(ua[1], ub[1]) and
                    torch.equal(a.acc, b.acc) and
                    torch.equal(a.t_ign, b.t_ign) and np.array_equal(a.series(), b.series()) and
                    (not attach or torch.equal(a.jac, b.jac)))
            ok_states = ok_acc = ok_loss = True
            if draw_rng == "splitmix":  # the oracle restates the reference's keyed draws
                arr = S.reference_landscape_arrays(env, O.slope_from_altitude)
                res = O.run(**arr, params=P(pv), init=init, steps=steps, seed=seeds[0],
                            attach_steps=range(1, steps + 1) if attach else (), threads=4,
                            wind_params=wind, want_jac_abs=attach)
                bu, bd = (x.bool().cpu().numpy() for x in b.unpack())
                ok_states = np.array_equal(bu[0], res.burning) and np.array_equal(bd[0], res.burned)
                acc = b.acc[0].double().cpu().numpy()
                ok_acc = np.allclose(acc, res.acc, rtol=1e-5, atol=0)
                if attach:
                    ok_loss = check_loss(rng, b, res, h, w, steps)
            ok = same and ok_states and ok_acc and ok_loss
            if not ok_loss:
                same = f"{same} (loss/gradient off)"
        except Exception as exc:  # report and continue
            ok, same, ok_states, ok_acc = False, repr(exc), None, None
        if not ok:
            failed.append((case, cfg, same, ok_states, ok_acc))
            log("FAIL", case, cfg, "same", same, "states", ok_states, "acc", ok_acc)
    return failed


def fuzz_shards(cases: int, seed: int, log=print):
    """Row shards (2-5 emulated on one GPU, each on its own stream) with the
    peer-memory halo or the exchange schedule, random heights/widths,
    windows, attached steps and dense or list sweeps: the owned rows must
    equal the unsharded run."""
    from paper_2502_18738_b200.sharded import (RowPartition, RowShard, connect_local_peers,
                                               run_peer_local, run_sharded_local)
    rng = np.random.default_rng(seed)
    failed = []
    for case in range(cases):
        world = int(rng.integers(2, 6))
        h = int(rng.integers(32 * world, 32 * world + 200))
        w = int(rng.integers(1, 200))
        steps = int(rng.integers(1, 60))
        window = int(rng.choice([1, 4, 8, 16]))
        attach = bool(rng.integers(0, 2))
        peer = bool(rng.integers(0, 2))
        env = S.make_environment(h, w, seed=int(rng.integers(0, 1 << 30)))
        init = np.zeros((h, w), dtype=bool)
        for _ in range(int(rng.integers(1, 8))):
            r, c = int(rng.integers(0, h)), int(rng.integers(0, w))
            init[r:r + 4, c:c + 4] = True
        pv = [float(rng.uniform(0, 1)), float(rng.uniform(0, 1)), float(rng.uniform(0, 1)),
              float(rng.uniform(0.2, 1)), float(rng.uniform(0, 1))]
        params, sd = F.pack_params(*pv), int(rng.integers(0, 1 << 62))
        cfg = dict(world=world, h=h, w=w, steps=steps, window=window, attach=attach, peer=peer)
        try:
            ref = F.FireBatch((h, w), 1, max_steps=steps, with_jacobian=attach)
            ref.set_params(params)
            ref.set_seeds([sd])
            ref.reset(init)
            ref.run(F.DeviceLandscape.from_environment(env), steps, attach=[attach] * steps,
                    window=window)
            rb, rd = ref.unpack()
            shards = []
            for r in range(world):
                sh = RowShard(RowPartition(h, world, r), env.elevation, env.wind_speed,
                              env.wind_direction, env.canopy, env.density, init, max_steps=steps,
                              with_jacobian=attach)
                sh.batch.set_params(params)
                sh.batch.set_seeds([sd])
                shards.append(sh)
            if peer:
                connect_local_peers(shards)
                run_peer_local(shards, steps, window=window, attach=[attach] * steps)
            else:
                run_sharded_local(shards, steps, window=window, attach=[attach] * steps)
            torch.cuda.synchronize()
            gb = torch.cat([sh.owned(sh.batch.unpack()[0][0]) for sh in shards])
            gd = torch.cat([sh.owned(sh.batch.unpack()[1][0]) for sh in shards])
            ok = (torch.equal(gb, rb[0]) and torch.equal(gd, rd[0]) and
                  torch.equal(torch.cat([sh.owned(sh.batch.acc[0]) for sh in shards]), ref.acc[0]) and
                  torch.equal(torch.cat([sh.owned(sh.batch.t_ign[0]) for sh in shards]), ref.t_ign[0]))
        except Exception as exc:
            ok = repr(exc)
        if ok is not True:
            failed.append((case, cfg, ok))
            log("FAIL shards", case, cfg, ok)
    return failed


def main():
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 100
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    dense = float(os.environ.get("FUZZ_DENSE", "0"))
    failed = fuzz(cases, seed, dense=dense)
    print(f"{cases - len(failed)}/{cases} configurations pass")
    nsh = max(1, cases // 10)
    failed_sh = fuzz_shards(nsh, seed)
    print(f"{nsh - len(failed_sh)}/{nsh} row-shard configurations pass")
    return 1 if failed or failed_sh else 0


if __name__ == "__main__":
    sys.exit(main())
