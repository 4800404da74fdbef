#!/usr/bin/env python
"""Benchmark of the B200-native wildfire CA (contract: one JSON line on rank 0).

Headline workload (BASELINE.json configs[1], fits one GPU): ensemble forward,
16 members x 2048^2 cells x 500 steps per GPU (members sharded by rank: weak
scaling, no data-path collective).  One bench "step" = one full ensemble run
from the initial state (reset + 500 CA steps).  value = cell-updates/s over
all ranks (members x H x W x steps / device time, max over ranks).

Extra keys: e2e (host buffers through EnsembleRunner), roofline (step kernel,
measured live with CUDA events), cpu_baseline (CPU oracle port, bounded
sample), calibration (config 2 iter/s), dense_probe (config 3 16384^2 dense
sweep + activity-skipping sweep), clocks (nvidia-smi during the timed region).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

H = W = 2048
MEMBERS = 16
WINDOW = 8  # CA steps fused per kernel launch (temporal blocking)
STEPS = 500
CELL_UPDATES_PER_MEMBER = H * W * STEPS
METRIC = "cell-updates/sec (fwd) & fwd+bwd calibration iter/s at 1/2/4/8 B200; % of HBM BW"
CONFIG = {"workload": "c1_ensemble_forward", "members_per_gpu": MEMBERS, "grid": [H, W],
          "steps": STEPS, "rng": "splitmix (reference-compatible keyed draws)",
          "params": "a=0.078 c1=0.045 c2=0.131 p_h=0.58*U[0.9,1.1] p_continue=0.3",
          "env": "synthetic config-0 generator at 2048^2 (seeded)",
          "l2": "flushed (256 MiB write) before every timed step",
          "activity_skipping": True, "steps_per_launch": WINDOW,
          "launch": "each timed run replays one CUDA graph of reset + the run (one persistent "
                    "dataflow launch: members advance window by window independently)"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-extras", action="store_true", help="skip calibration/dense probes")
    ap.add_argument("--cpu-sample-steps", type=int, default=500)
    ap.add_argument("--pyrocell-steps", type=int, default=300,
                    help="steps of the pyrocell (reference itself) CPU sample")
    return ap.parse_args()


def load_peaks():
    p = os.path.join(REPO, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    return 6650.0, "fallback (B200_PROFILING.md)"


# ------------------------------------------------------------------ clocks ---
class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region: NVML
    every 5 ms on the box (the timed region is tens of ms), else nvidia-smi
    -lms 100 (B200_PROFILING.md clocks line)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    # NVML clocks-event-reason bits
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown"}

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []
        self.sm, self.mx, self.reasons = [], None, set()
        self.nvml = None
        self._stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            self.mx = float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            return self
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(self.gpu)], stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _poll(self):
        p = self.nvml
        while not self._stop.is_set():
            try:
                self.sm.append(float(p.nvmlDeviceGetClockInfo(self.h, p.NVML_CLOCK_SM)))
                bits = p.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for b, n in self.REASONS.items():
                    if bits & b:
                        self.reasons.add(n)
            except Exception:
                pass
            time.sleep(0.005)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.nvml is not None:
            self._stop.set()
            self.t.join(timeout=1)
            return
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = list(self.sm), self.mx, set(self.reasons)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        src = "nvml 5 ms" if self.nvml is not None else "nvidia-smi 100 ms"
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": [], "samples": 0, "source": src}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "source": src}


# ----------------------------------------------------------- reference arm ---
def cpu_sample(env, members, steps, threads):
    """Oracle port (C, OpenMP) on `members` of the c1 workload."""
    from oracle import oracle as O
    from paper_2502_18738_b200 import synthetic as S
    arr = S.reference_landscape_arrays(env, O.slope_from_altitude)
    ph = S.ensemble_ph(MEMBERS)
    init = S.center_ignition(H)

    class _P:
        pass
    t0 = time.perf_counter()
    for m in members:
        p = _P()
        p.c1, p.c2, p.a, p.p_h, p.p_continue = 0.045, 0.131, 0.078, float(ph[m % MEMBERS]), 0.3
        O.run(**arr, params=p, init=init, steps=steps, seed=m, threads=threads, want_jac=False)
    dt = time.perf_counter() - t0
    return len(members) * H * W * steps / dt, dt


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def pyrocell_sample(env, steps, threads_list):
    """pyrocell 0.1.0 itself (the reference, pure NumPy, installed in
    baseline/_ref) on member 0 of the c1 workload: its own
    slope_from_altitude and run_simulation on the same fp32 rasters, bbox
    windowing on, for each thread count; cell-updates/s (full-grid)."""
    ref = os.path.join(REPO, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "pyrocell")):
        return {"unavailable": "baseline/_ref/pyrocell not installed"}
    sys.path.insert(0, ref)
    try:
        import pyrocell as P
        from pyrocell.data_io import slope_from_altitude
    finally:
        sys.path.remove(ref)
    if not os.path.dirname(P.__file__).startswith(ref):
        return {"unavailable": f"imported pyrocell from {P.__file__}, not baseline/_ref"}
    from paper_2502_18738_b200 import synthetic as S
    f64 = lambda a: np.asarray(a, dtype=np.float64)
    land = P.Landscape(wind_speed=f64(env.wind_speed), wind_direction=f64(env.wind_direction),
                       slope=slope_from_altitude(f64(env.elevation), env.cell_side),
                       canopy=f64(env.canopy), density=f64(env.density), cell_side=env.cell_side)
    ph = float(S.ensemble_ph(MEMBERS)[0])
    params = P.ModelParams(c1=0.045, c2=0.131, a=0.078, p_h=ph, p_continue=0.3)
    init = S.center_ignition(H)
    out = {"cpu_model": cpu_model(), "numpy": np.__version__,
           "sample": f"member 0 of c1: 1 x {H}^2 x {steps} steps, pyrocell.run_simulation "
                     f"(fp64, bbox window, row-band threads)"}
    for th in threads_list:
        t0 = time.perf_counter()
        P.run_simulation(land, params, init, steps, 0, threads=th)
        dt = time.perf_counter() - t0
        out[f"threads_{th}"] = {"value": H * W * steps / dt, "unit": "cell-updates/s",
                                "seconds": dt}
    return out


def run_reference(args):
    rank = int(os.environ.get("RANK", 0))
    if rank != 0:
        return
    from paper_2502_18738_b200 import synthetic as S
    env = S.make_environment(H, seed=1)
    cores = os.cpu_count() or 1
    for i in range(args.warmup):
        cpu_sample(env, [i % MEMBERS], args.cpu_sample_steps, cores)
    vals, times = [], []
    for i in range(args.steps):
        v, dt = cpu_sample(env, [i % MEMBERS], args.cpu_sample_steps, cores)
        vals.append(v)
        times.append(dt)
    value = float(len(vals) * H * W * args.cpu_sample_steps / sum(times))
    sample = (f"1 member (cycling 0..15) x {H}^2 x {args.cpu_sample_steps} steps per step, "
              f"oracle port (oracle/oracle.c, fp64, bbox window, OpenMP {cores} threads)")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "cell-updates/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * sum(times) / len(times), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": CONFIG,
        "cpu_baseline": {"value": value, "unit": "cell-updates/s", "cores": cores,
                         "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "cell-updates/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }))


# ------------------------------------------------------------------ ours ---
def timed_loop(fn, K, flush):
    import torch
    st = torch.cuda.current_stream()
    times = []
    for _ in range(K):
        flush()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        fn()
        e1.record(st)
        times.append((e0, e1))
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in times]


def launch_bytes(cnt, burning_pre, window, tiles_override=None, per_tile=512.0):
    """Algorithmic bytes of each window launch from the per-step counters:
    512 B per visited 32x32 tile (burning + burned words read and written
    once per launch), 16 B of env per ignition candidate and per burning
    source cell per step, 6 B (acc + t_ign) per ignition."""
    steps = cnt.shape[0]
    out = []
    for a in range(0, steps, window):
        b = min(a + window, steps)
        tiles = cnt[a, 2] if tiles_override is None else tiles_override
        out.append(per_tile * tiles + 16.0 * (cnt[a:b, 3].sum() + burning_pre[a:b].sum())
                   + 6.0 * cnt[a:b, 0].sum())
    return np.array(out)


def per_launch_profile(batch, land, steps, window, skip=True):
    """Average window-kernel duration with CUDA events around each launch
    on the launching stream (one launch per fc_run call of `window` steps)."""
    import torch
    st = torch.cuda.current_stream()
    batch.reset(batch._init_mask)
    evs = []
    for a in range(0, steps, window):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        batch.run(land, min(window, steps - a), window=window, skip_inactive=skip)
        e1.record(st)
        evs.append((e0, e1))
    torch.cuda.synchronize()
    ms = np.array([a.elapsed_time(b) for a, b in evs])
    cnt = batch.counters[:, :steps].to(torch.int64).sum(0).cpu().numpy()  # (steps, 4)
    ser = batch.series()  # (M, steps, 2)
    burning_pre = np.concatenate([[batch.init_burning.sum()], ser[:, :-1, 0].sum(0)])[:steps]
    tiles = None if skip else batch.m * batch.grid.tiles_y * batch.grid.tiles_x
    return ms, launch_bytes(cnt, burning_pre, window, tiles, 512.0 if skip else 256.0), cnt


def run_ours(args):
    import torch

    import paper_2502_18738_b200 as F
    from paper_2502_18738_b200 import synthetic as S
    from paper_2502_18738_b200.ensemble import EnsembleRunner
    from paper_2502_18738_b200.parallel import allreduce_max, barrier, init_distributed

    rank, world, local = init_distributed()
    dev = torch.device("cuda", local)
    peak, peak_src = load_peaks()
    env = S.make_environment(H, seed=1)
    dl = F.DeviceLandscape.from_environment(env, device=dev)
    members = [rank * MEMBERS + m for m in range(MEMBERS)]
    ph_all = S.ensemble_ph(MEMBERS * world)
    params = [(0.045, 0.131, 0.078, float(ph_all[m]), 0.3) for m in members]
    init = S.center_ignition(H)
    batch = F.FireBatch((H, W), MEMBERS, max_steps=STEPS, member0=members[0], device=dev)
    batch.set_params(np.array([F.pack_params(*p) for p in params]))
    batch.set_seeds(members)
    init_dev = torch.as_tensor(init.astype(np.uint8), device=dev)
    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def flush():
        flush_buf.fill_(1)

    def one_run():
        batch.reset(init_dev)
        batch.run(dl, STEPS, window=WINDOW)

    for _ in range(args.warmup):
        one_run()
    # one ensemble run (reset + every window launch) as a CUDA graph: the
    # same kernels on the same data, without per-launch host overhead
    graph = F.CapturedSequence(one_run)
    for _ in range(args.warmup):
        graph.replay()
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        ms = timed_loop(graph.replay, args.steps, flush)
    torch.cuda.synchronize()
    barrier()
    total_ms = allreduce_max(float(sum(ms)), dev)
    cu = world * MEMBERS * CELL_UPDATES_PER_MEMBER * args.steps
    value = cu / (total_ms / 1e3)
    nwin = (STEPS + WINDOW - 1) // WINDOW
    # reset (pack_init + tile_init; a reused batch resets lazily without
    # init_cells) + ensure_marking + the dataflow run: list split + scatter,
    # df_init, ONE persistent df_kernel for all 63 windows of the 16
    # members, list merge (FireBatch(dataflow=True), the default for M >= 2)
    launches_per_step = 2 + 1 + 5 if batch.sched is not None else 2 + 1 + nwin

    # final-state sanity (affected counts) for the log
    ser = batch.series()
    affected_final = int(ser[:, -1].sum())

    # -------------------------------------------------- roofline (live)
    # achieved = SURVEY.md 8(d) algorithmic bytes per cell-update x the
    # cell-updates the launches process / their CUDA-event time.  8(d):
    # B(M, k) = (16/M + 2)/k B per cell-update (16 B of fp32 env shared by M
    # members, 1 B state read + 1 B written, once per k fused steps).
    # the window kernel's time INSIDE the timed timeline: the same graph
    # replayed (reset + every PDL-chained window launch) minus a graph of the
    # reset alone, over the window launches -- CUDA events on the launching
    # stream, L2 flushed as in the timed loop
    reset_graph = F.CapturedSequence(lambda: batch.reset(init_dev))
    for _ in range(args.warmup):
        reset_graph.replay()
    ms_reset = timed_loop(reset_graph.replay, args.steps, flush)
    ms_full = timed_loop(graph.replay, args.steps, flush)
    win_ms = float(np.mean(ms_full) - np.mean(ms_reset))
    avg_us = 1e3 * win_ms / nwin
    lms, lbytes, cnt = per_launch_profile(batch, dl, STEPS, WINDOW)
    b_cu = (16.0 / MEMBERS + 2.0) / WINDOW
    run_cu = MEMBERS * H * W * STEPS
    alg_per_launch = b_cu * run_cu / nwin
    achieved = alg_per_launch / (avg_us / 1e6) / 1e9
    kern = float(lbytes.mean()) / (avg_us / 1e6) / 1e9
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": None, "peak_source": peak_src,
                "kernel": (f"df_kernel<SPLITMIX,elev,no-attach,K={WINDOW},G=8>: one persistent "
                           f"dataflow launch per run, every member advancing its {nwin} windows "
                           "on its own" if batch.sched is not None else
                           f"window_kernel<SPLITMIX,elev,no-attach,K={WINDOW},G=8>"),
                "avg_launch_us": avg_us, "launches": nwin,
                "avg_launch_timing": "per window of K steps, in the timed graph: (reset + the "
                                     "run) minus (reset alone), CUDA events, / windows; the "
                                     "run's share of the step is "
                                     f"{win_ms / float(np.mean(ms_full)):.3f}",
                "avg_launch_us_standalone": float(1e3 * lms.mean()),
                "algorithmic_bytes_per_cell_update": b_cu,
                "algorithmic_bytes_per_launch": alg_per_launch,
                "meaning": "dense-equivalent: SURVEY 8(d) B(M=16,k=8)=0.375 B per cell-update "
                           "over every cell of every member, whether or not the kernel visits "
                           "it (activity skipping visits ~1900 of 65536 tiles per launch)",
                "kernel_bytes_per_launch": float(lbytes.mean()),
                "kernel_bytes_GBps": kern, "kernel_bytes_frac": kern / peak,
                "tiles_visited_per_launch": float(cnt[::WINDOW, 2].mean())}
    prof = os.path.join(REPO, "profiles", "ncu_traffic.json")
    if os.path.exists(prof):
        with open(prof) as f:
            tr = json.load(f)
        dram = tr.get("c1_step_kernel_dram_bytes_per_launch")
        inst = tr.get("c1_step_kernel_warp_instructions_per_launch")
        roofline["traffic"] = dram
        roofline["traffic_source"] = tr.get("source")
        if dram:
            gbs = dram / (avg_us / 1e6) / 1e9
            # what the kernel really moves to and from HBM (ncu dram bytes)
            roofline["hbm_measured"] = {"GBps": gbs, "frac_of_measured_peak": gbs / peak,
                                        "frac_of_8TBps_spec": gbs / 8000.0}
        if inst:
            clk = 1.965e9
            floor_us = inst / (148 * 4 * clk) * 1e6  # 4 issue slots per SM per clock
            roofline["issue_roofline"] = {
                "warp_instructions_per_window": inst, "issue_floor_us": floor_us,
                "frac": floor_us / avg_us,
                "note": "148 SMs x 4 schedulers x 1 warp-instruction/clock at 1965 MHz; the "
                        "kernel is latency-bound (barrier and memory-latency stalls), "
                        "profiles/r2_ncu_summary.md"}
    # -------------------------------------------------------------- e2e
    # three slots, results read two calls behind: call i+1's upload then
    # overlaps call i-1's export instead of waiting for it on the host (two
    # slots: 0.45-0.6 ms between every other pair of runs, 3.20 against
    # 3.03-3.07 ms per call; profiles/r2_ncu_summary.md section 30)
    E2E_DEPTH = 3
    runner = EnsembleRunner((H, W), MEMBERS, STEPS, device=dev, depth=E2E_DEPTH)
    env_host = torch.stack([torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)) for a in
                            (env.elevation, env.wind_speed, env.wind_direction, env.canopy,
                             env.density)]).pin_memory()
    init_host = torch.from_numpy(init.astype(np.uint8)).pin_memory()
    for _ in range(max(len(runner.slots), args.warmup)):
        runner(env_host, init_host, params, members)
    barrier()
    # K calls pipelined three deep (EnsembleRunner.submit): call i-2's
    # results are read on the host while call i-1 exports, call i runs and
    # call i+1 uploads; every call's H2D and D2H lies inside the timed
    # region, L2 flushed between calls
    flush()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pending = []
    # at least 40 calls: the host side of a call varies by up to ~0.2 ms
    # between runs, which 20 calls (66 ms) do not average out
    n_e2e = max(args.steps, 40)
    for _ in range(n_e2e):
        # the L2 flush goes ahead of the call's kernels on the runner's compute
        # stream: on the caller's stream it would also hold back the call's
        # uploads, which wait for the caller's queued work (inputs it may
        # have produced)
        with torch.cuda.stream(runner.compute_stream):
            flush()
        pending.append(runner.submit(env_host, init_host, params, members))
        if len(pending) >= E2E_DEPTH:
            res = pending.pop(0).result()
            e2e_check = int(res.series[0, -1, 0])  # read the result on the host
    for prev in pending:
        res = prev.result()
        e2e_check = int(res.series[0, -1, 0])
    e2e_total = allreduce_max(1e3 * (time.perf_counter() - t0), dev)
    cu_e2e = world * MEMBERS * CELL_UPDATES_PER_MEMBER * n_e2e
    e2e = {"value": cu_e2e / (e2e_total / 1e3), "unit": "cell-updates/s", "calls": n_e2e,
           "h2d_bytes_per_step": int(runner.h2d_bytes), "d2h_bytes_per_step": int(runner.d2h_bytes(prev)),
           "d2h_note": "fc_state_export writes the (M,H,W) burning/burned/accumulator result "
                       "arrays in pinned host memory from the device, only for tiles affected "
                       "now or written by the slot's previous call (%d of %d tiles, in 128-column "
                       "spans); the "
                       "dense arrays would be %d B" % (prev.exported_tiles(),
                                                       runner.batch.grid.tiles_x * runner.batch.grid.tiles_y * MEMBERS,
                                                       runner.d2h_bytes_dense),
           "api": "paper_2502_18738_b200.ensemble.EnsembleRunner.submit (pinned host in/out, "
                  "3-deep pipeline: upload of call i+1, kernels of call i and export of "
                  "call i-1 on three streams, results of call i-2 read on the host)",
           "final_burning_member0": e2e_check}

    extras = {}

    def extra(name, fn, *a):
        # an extra that fails (on every rank alike: the same code and data)
        # is reported in the line instead of taking the headline with it
        try:
            return fn(*a)
        except Exception as exc:  # noqa: BLE001
            torch.cuda.synchronize()
            return {"error": f"{name}: {type(exc).__name__}: {exc}"[:300]}
    if not args.no_extras:
        c4 = extra("ensemble_calibration", bench_ensemble_calibration, dev, rank, world)
        c3 = extra("row_sharded", bench_row_sharded, dev, rank, world)
        if rank == 0:
            extras["ensemble_calibration"] = c4
            extras["row_sharded"] = c3
    if rank == 0 and world == 1 and not args.no_extras:
        extras["calibration"] = extra("calibration", bench_calibration, dev)
        extras["fig6_sweep"] = extra("fig6_sweep", bench_fig6_sweep, dev)
        extras["dense_probe"] = extra("dense_probe", bench_dense, dev, peak)
    cpu = None
    if rank == 0 and world == 1:
        cores = os.cpu_count() or 1
        v, dt = cpu_sample(env, [0], args.cpu_sample_steps, cores)
        cpu = {"value": v, "unit": "cell-updates/s", "cores": cores, "kind": "port",
               "sample": f"member 0 of c1: 1 x {H}^2 x {args.cpu_sample_steps} steps, oracle port "
                         f"(fp64, bbox window, OpenMP), {dt:.1f} s",
               "cpu_model": cpu_model(),
               # the reference itself beside the port: pyrocell
               # with one thread and with every core
               "reference_pyrocell": pyrocell_sample(env, args.pyrocell_steps, (1, cores))}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "cell-updates/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": float(np.mean(ms)),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "config": CONFIG, "parallelism": f"member-sharded x{world}",
            "gpu_launches": launches_per_step * args.steps, "clocks": clocks.summary(),
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "affected_cells_final": affected_final,
        }
        line.update(extras)
        print(json.dumps(line))


def bench_calibration(dev):
    """Config 2: 1024^2, targets from hidden params at 25/50/75/100 (seed 7),
    50 Adam iterations (lr 1e-2) of a 100-step all-attached forward + fused
    4-target loss/gradient + device AdamW; iter/s on the device."""
    import torch

    import paper_2502_18738_b200 as F
    from paper_2502_18738_b200 import synthetic as S
    n, T, iters = 1024, 100, 50
    env = S.make_environment(n, seed=2)
    dl = F.DeviceLandscape.from_environment(env, device=dev)
    init = torch.as_tensor(S.center_ignition(n).astype(np.uint8), device=dev)
    hid = S.HIDDEN_C2_PARAMS
    tb = F.FireBatch((n, n), 1, max_steps=T, device=dev)
    tb.set_params(F.pack_params(hid["c1"], hid["c2"], hid["a"], hid["p_h"], hid["p_continue"]))
    tb.set_seeds([7])
    tb.reset(init)
    targets = []
    for _ in range(4):
        tb.run(dl, 25)
        b, d = tb.unpack()
        targets.append((b[0] | d[0]))
    targets = torch.stack(targets)
    obs = [25, 50, 75, 100]
    b = F.FireBatch((n, n), 1, max_steps=T, with_jacobian=True, device=dev)
    p0 = S.DEFAULT_BENCH_PARAMS
    b.set_params(F.pack_params(p0["c1"], p0["c2"], p0["a"], p0["p_h"], p0["p_continue"]))
    b.set_seeds([F.derive_epoch_seed(7, 1)])
    attach = [True] * T

    out = {}

    def iteration():
        b.reset(init)
        b.run(dl, T, attach=attach)
        out["loss"], _, out["grad"], _ = b.loss_grad(targets, obs)
        b.adamw(out["grad"], None, 1e-2)  # device step counter: graph-replayable

    def restart():
        b.adam.zero_()
        b.adam_step.zero_()
        b.set_params(F.pack_params(p0["c1"], p0["c2"], p0["a"], p0["p_h"], p0["p_continue"]))

    def timed(fn):
        restart()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(iters):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)

    for _ in range(3):
        iteration()
    ms_plain = timed(iteration)
    graph = F.CapturedSequence(iteration)
    ms = timed(graph.replay)  # one CUDA graph per iteration (reset + windows + loss + AdamW)
    loss, grad = out["loss"], out["grad"]
    p = b.params[0, :5].cpu().numpy()
    return {"iter_per_s": iters / (ms / 1e3), "ms_per_iter": ms / iters, "iterations": iters,
            "iter_per_s_without_graph": iters / (ms_plain / 1e3),
            "grid": [n, n], "steps_per_iter": T, "attached": "all 100 steps",
            "loss": "sum over 4 targets of combined_loss (BCE crop + 4x4 pooled MSE)",
            "final_loss": float(loss[0, 0]), "final_params_c1_c2_a_ph_pc": p.tolist(),
            "note": "p_continue gradient is identically 0 under straight-through semantics",
            # a c2 iteration is 100 x 18 B + ~26 B per cell
            # (acc 4, ignition step 2, J 16, 4 target bits) = 1.83 kB/cell
            "effective_GBps_survey": 1826.0 * n * n * iters / (ms / 1e3) / 1e9,
            "effective_frac_survey": 1826.0 * n * n * iters / (ms / 1e3) / 1e9 / load_peaks()[0]}


def bench_ensemble_calibration(dev, rank, world, members_total=256, iters=3):
    """Config 4: 256 members x 1024^2 x 200 steps, all steps attached, wind
    rotating +90 deg and ramping 2 -> 12 m/s (device schedule), per-member
    4-target loss + gradient, gradients summed over members and all-reduced
    over ranks (NCCL), one AdamW step on the shared parameters.  Members are
    sharded by rank; iteration time is the max over ranks."""
    import torch

    import paper_2502_18738_b200 as F
    from paper_2502_18738_b200 import synthetic as S
    from paper_2502_18738_b200.device import wind_ramp_schedule
    from paper_2502_18738_b200.parallel import allreduce_max, allreduce_sum_, shard_members
    n, T = 1024, 200
    env = S.make_environment(n, seed=4)
    dl = F.DeviceLandscape.from_environment(env, device=dev)
    sched = wind_ramp_schedule(T, 2.0, 12.0, 90.0, device=dev)
    init = torch.as_tensor(S.center_ignition(n).astype(np.uint8), device=dev)
    hid = S.HIDDEN_C2_PARAMS
    tb = F.FireBatch((n, n), 1, max_steps=T, device=dev)
    tb.set_params(F.pack_params(hid["c1"], hid["c2"], hid["a"], hid["p_h"], hid["p_continue"]))
    tb.set_seeds([7])
    tb.reset(init)
    obs = [50, 100, 150, 200]
    targets = []
    for k in range(4):
        tb.run(dl, 50, wind_schedule=sched)
        b_, d_ = tb.unpack()
        targets.append(b_[0] | d_[0])
    targets = torch.stack(targets)
    del tb
    mine = shard_members(members_total, rank, world)
    from paper_2502_18738_b200.ensemble import EnsembleCalibrator
    p0 = S.DEFAULT_BENCH_PARAMS
    cal = EnsembleCalibrator(dl, init, targets, obs, mine,
                             (p0["c1"], p0["c2"], p0["a"], p0["p_h"], p0["p_continue"]),
                             steps=T, wind_schedule=sched, lr=1e-2, device=dev)
    cal.step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        loss = cal.step()
    e1.record()
    torch.cuda.synchronize()
    ms = allreduce_max(e0.elapsed_time(e1) / iters, dev)
    shared = cal.shared
    return {"iter_per_s": 1e3 / ms, "ms_per_iter": ms, "members": members_total,
            "timed": f"iterations 2-{iters + 1} (the first runs eagerly and captures the CUDA "
                     "graph); AdamW moves c1 down from its start value, so the fires, and the "
                     "work per iteration, shrink as calibration proceeds: the number depends on "
                     "this iteration count",
            "members_per_rank": len(mine), "grid": [n, n], "steps": T, "attached": "all",
            "fwd_bwd_cell_updates_per_s": members_total * n * n * T / (ms / 1e3),
            "wind": "direction +90 deg linear, speed 2->12 m/s linear (device schedule)",
            "targets": "hidden-parameter run (seed 7) affected masks at 50/100/150/200",
            "mean_member_loss": float(loss[:, 0].mean()),
            "params_after_c1_c2_a_ph": shared[0, :4].cpu().numpy().tolist()}


def bench_row_sharded(dev, rank, world, steps=1000, windows=(1, 4, 8)):
    """Config 3 row-sharded across the ranks, both scalings, with k = 1 (a
    halo exchange every step) and k = 4 fused steps:
      strong: the 16384^2 domain split into world row bands;
      weak:   2048*world x 16384, 2048 rows per rank.
    8 random 5x5 ignitions in the strong domain (2 per 2048-row band in the
    weak one), sigma x32 environment generated on the device.  Each window
    launch is split (fc_run_pass) so the NCCL exchange of its boundary rows
    overlaps the next launch's interior pass (sharded.run_overlapped).
    Device time (CUDA events, max over ranks) of the whole run; value =
    global cell-updates/s.  One rank runs the same domain unsharded
    (fc_run, activity lists)."""
    import torch

    import paper_2502_18738_b200 as F
    from paper_2502_18738_b200 import synthetic as S
    from paper_2502_18738_b200.parallel import allreduce_max, barrier
    from paper_2502_18738_b200.sharded import (RowPartition, RowShard, connect_peers,
                                               peer_handshake, run_peer, run_sharded)
    out = {"steps": steps, "ranks": world, "scaling": {"strong": "total work fixed",
                                                         "weak": "work per rank fixed"},
           "halo": "2 bit planes x 1 tile row (32 rows) each way per launch"}
    halo_peer = ("peer: the boundary pass stores its rows into the neighbours' ghost rows "
                 "(NVLink, CUDA IPC mappings) and counts the launch in their flag words; "
                 "streams wait on the flags (fc_peer_halo), no collective in the step loop")
    halo_nccl = ("nccl: NCCL P2P send/recv on a communication stream overlapped with the next "
                 "launch's interior pass")
    for kind in ("strong", "weak"):
        H, Wd = (16384, 16384) if kind == "strong" else (2048 * world, 16384)
        nfire = 8 if kind == "strong" else 2 * world
        e = S.make_environment_torch(H, Wd, seed=3, sigma_elev=640.0, sigma_wind=960.0,
                                     device=dev)
        init = torch.as_tensor(S.random_blocks(H, Wd, nfire, 5, seed=3).astype(np.uint8),
                               device=dev)
        res = {"grid": [H, Wd], "rows_per_rank": H // world, "ignitions": nfire}
        if world == 1:
            land = F.DeviceLandscape.from_elevation(e["elevation"], e["wind_speed"],
                                                    e["wind_direction"], e["canopy"],
                                                    e["density"], device=dev)
            b = F.FireBatch((H, Wd), 1, max_steps=steps, device=dev)
        else:
            sh = RowShard(RowPartition(H, world, rank), e["elevation"], e["wind_speed"],
                          e["wind_direction"], e["canopy"], e["density"], init, max_steps=steps,
                          device=dev)
            b = sh.batch
        del e
        b.set_params(F.pack_params(0.045, 0.131, 0.078, 0.58, 0.3))
        b.set_seeds([3])
        init_local = init if world == 1 else sh.batch._init_mask
        peer = False
        if world > 1:
            # the fused peer-memory halo unless FC_HALO=nccl or its handshake
            # fails (then NCCL P2P, recorded in the line)
            if os.environ.get("FC_HALO", "peer") == "peer":
                err = connect_peers(sh)  # collective; never raises on a mapping failure
                peer = peer_handshake(sh)
                if err or not peer:
                    res["peer_unavailable"] = (err or "handshake: flags did not arrive")[:200]
            if not peer:
                sh.shard.peer = None
            res["halo"] = halo_peer if peer else halo_nccl
        for k in windows:
            def one():
                if world > 1 and peer:
                    run_peer([sh], steps, k, reset=True)
                    return
                b.reset(init_local)
                if world == 1:
                    b.run(land, steps, window=k)
                else:
                    run_sharded(sh, steps, k)
            b.reset(init_local)  # warm-up: communicators, caches
            if world == 1:
                b.run(land, 2 * k, window=k)
            elif peer:
                run_peer([sh], 2 * k, k)
            else:
                run_sharded(sh, 2 * k, k)
            torch.cuda.synchronize()
            # the whole run (reset, every split launch, every halo exchange
            # on the communication stream) as one CUDA graph: the per-launch
            # host work (~0.1 ms per window in Python) would otherwise bound
            # the k = 1 schedule
            mode = "cuda-graph"
            if os.environ.get("FC_SHARD_GRAPH", "1") == "0":
                mode, run = "eager (FC_SHARD_GRAPH=0)", one
            else:
                try:
                    graph = F.CapturedSequence(one)
                    run = graph.replay
                except Exception as exc:  # fall back to eager launches, say so
                    torch.cuda.synchronize()
                    mode, run = f"eager (capture failed: {type(exc).__name__})", one
            barrier()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            run()
            e1.record()
            torch.cuda.synchronize()
            ms = allreduce_max(e0.elapsed_time(e1), dev)
            cus = H * Wd * steps / (ms / 1e3)
            # a dense sweep moves B(M=1, k) = (16 + 2) / k bytes per
            # cell-update, so it is capped at peak / B cell-updates/s; activity
            # skipping never touches quiet cells and legitimately exceeds that
            # cap ("Also report activity-skipping cu/s"): a ratio, not a bandwidth
            b_cu = 18.0 / k
            cap = load_peaks()[0] * 1e9 / b_cu
            res[f"k{k}"] = {"ms": ms, "cell_updates_per_s": cus, "launch": mode,
                            "dense_sweep_cap_cu_per_s": cap,
                            "x_dense_sweep_cap": cus / cap}
            del run
            if mode == "cuda-graph":
                del graph
        out[kind] = res
        del b, init
        if world > 1:
            del sh
        else:
            del land
        torch.cuda.empty_cache()
    return out


def bench_fig6_sweep(dev, sizes=(200, 1000, 2000, 4000, 8000, 14000), steps=300):
    """The paper's Fig.-6 style scaling sweep (the
    reference CLI bench, pyrocell/cli.py:241-287): flat landscape, V_w = 2,
    default ModelParams (p_continue 0.5), centre ignition, 300 steps.
    'device_s' = kernel time of the run; 'wall_s' = landscape build + state
    allocation + run + final state copied to host."""
    import torch

    import paper_2502_18738_b200 as F
    from paper_2502_18738_b200 import synthetic as S
    rows = []
    for n in sizes:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        z = torch.zeros((n, n), dtype=torch.float32, device=dev)
        dl = F.DeviceLandscape.from_elevation(z, torch.full_like(z, 2.0), z, z, z, device=dev)
        b = F.FireBatch((n, n), 1, max_steps=steps, device=dev)
        b.set_params(F.pack_params(0.045, 0.131, 0.078, 0.58, 0.5))
        b.set_seeds([0])
        b.reset(torch.as_tensor(S.center_ignition(n).astype(np.uint8), device=dev))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        b.run(dl, steps, window=WINDOW)
        e1.record()
        bu, bd = b.unpack()
        host = (bu.cpu(), bd.cpu(), b.acc.cpu())
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        rows.append({"size": n, "device_s": e0.elapsed_time(e1) / 1e3, "wall_s": wall,
                     "affected": int(host[0].sum() + host[1].sum())})
        del dl, b, z, host
        torch.cuda.empty_cache()
    return {"steps": steps, "rows": rows,
            "paper": "PyTorchFire: <1 s for maps <1200 (RTX 4090), <=1500 (A800); <60 s at 14000 "
                     "on 'a more advanced GPU'; CPU 300 steps at 1000^2 ~30 s (PAPER.md:456-467)"}


def bench_dense(dev, peak):
    """Config 3 on one GPU: 16384^2, 8 random 5x5 ignitions, sigma x32 env
    (FFT on the device).  Window kernel (K=8) timed per launch with CUDA
    events, once visiting every tile (the HBM-streaming regime) and once
    with activity lists."""
    import torch

    import paper_2502_18738_b200 as F
    from paper_2502_18738_b200 import synthetic as S
    n, steps = 16384, 200
    e = S.make_environment_torch(n, n, seed=3, device=dev)
    dl = F.DeviceLandscape.from_elevation(e["elevation"], e["wind_speed"], e["wind_direction"],
                                          e["canopy"], e["density"], device=dev)
    del e
    init = torch.as_tensor(S.random_blocks(n, n, 8, 5, seed=3).astype(np.uint8), device=dev)
    out = {"grid": [n, n], "steps": steps, "steps_per_launch": WINDOW}
    for skip in (False, True):
        b = F.FireBatch((n, n), 1, max_steps=steps, device=dev)
        b.set_params(F.pack_params(0.045, 0.131, 0.078, 0.58, 0.3))
        b.set_seeds([3])
        b.reset(init)
        b.run(dl, 2 * WINDOW, window=WINDOW, skip_inactive=skip)  # warm-up
        b.reset(init)
        b._init_mask = init
        torch.cuda.synchronize()
        ms, byts, cnt = per_launch_profile(b, dl, steps, WINDOW, skip)
        ach = float(byts.sum() / (ms.sum() / 1e3)) / 1e9
        key = "skip" if skip else "dense"
        cups = n * n * steps / (ms.sum() / 1e3)
        out[key] = {"avg_launch_us": float(1e3 * ms.mean()),
                    "cell_updates_per_s": cups,

                    "achieved_GBps": ach, "frac_of_peak": ach / peak,
                    "bytes_per_launch": float(byts.mean()),
                    "tiles_per_launch": float(n * n / 1024 if not skip else cnt[::WINDOW, 2].mean())}
        if not skip:
            # the HBM-streaming half of the dense sweep on its own: the
            # activity scan of the final state (reads the burning plane,
            # writes one flag per tile and the zero next state of quiet tiles)
            import ctypes as C
            from paper_2502_18738_b200 import _lib as L
            # 20 back-to-back scans in one CUDA graph (launch overhead
            # amortised), cycling over four states so that each scan's 67 MB
            # of plane traffic has left the 126 MB L2 before it comes round
            # again (inputs larger than L2)
            extra = []
            for k in range(3):
                bk = F.FireBatch((n, n), 1, max_steps=steps)
                bk.reset(torch.as_tensor(S.random_blocks(n, n, 8, 5, seed=4 + k).astype(np.uint8),
                                         device=dev))
                extra.append(bk)
            states = [(x, x.struct(), x.q) for x in [b] + extra]

            def scan(k):
                x, sx, qx = states[k % 4]
                L.check(L.lib().fc_activity_scan(C.byref(x.grid), C.byref(sx), qx, L.stream_ptr()),
                        "fc_activity_scan")
            g20 = F.CapturedSequence(lambda: [scan(k) for k in range(20)])
            g20.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                g20.replay()
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) * 1e3 / 100
            tiles = n * n // 1024
            live = int(b.list_count[b.q].item())
            sbytes = 128.0 * tiles + 128.0 * (tiles - live)  # plane read + quiet tiles' zero writes
            ach_s = sbytes / (us / 1e6) / 1e9
            del extra, states
            out["dense"]["activity_scan"] = {"avg_us": us, "timing": "20 scans per CUDA graph, "
                                                                      "four states in turn (L2 "
                                                                      "cold for each)",
                                             "bytes": sbytes, "achieved_GBps": ach_s,
                                             "frac_of_peak": ach_s / peak, "live_tiles": live}
        del b
    # every cell active: a random half of the domain burning at step 0, burning
    # on (p_continue 0.999: each burning cell still draws every step), ignition
    # of the rest within a few steps -- every tile is live in every launch and
    # every cell takes a continue draw per step.  Dense sweep (the mode that
    # takes dense tiles' draws in the sweep), K = 8, one warm-up launch
    gen = torch.Generator(device=dev)
    gen.manual_seed(11)
    half = (torch.rand((n, n), generator=gen, device=dev) < 0.5).to(torch.uint8)
    nl = 4
    b = F.FireBatch((n, n), 1, max_steps=WINDOW * (nl + 1), device=dev)
    b.set_params(F.pack_params(0.045, 0.131, 0.078, 0.2, 0.999))
    b.set_seeds([3])
    b.reset(half)
    b.run(dl, WINDOW, window=WINDOW, skip_inactive=False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    b.run(dl, WINDOW * nl, window=WINDOW, skip_inactive=False)
    e1.record()
    torch.cuda.synchronize()
    ms_l = e0.elapsed_time(e1) / nl
    burning = int(b.series()[0, -1, 0])
    cups = n * n * WINDOW / (ms_l / 1e3)
    cap = peak * 1e9 / 18.0
    out["regime_all_active"] = {
        "ms_per_launch": ms_l, "cell_updates_per_s": cups, "launches": nl,
        "burning_cells_at_end": burning, "cells": n * n,
        "survey_dense_cap_cu_per_s": cap, "frac_of_survey_dense_cap": cups / cap,
        "bound": "issue (SplitMix64 continue draws, 56 instructions per draw; ncu: 68 % of "
                 "issue slots busy, 0.1 % of DRAM; profiles/r2_ncu_summary.md section 14)",
        "setup": "16384^2, a random half burning at step 0, p_continue 0.999, p_h 0.2, dense "
                 "sweep, K = 8: every tile live, every cell drawn every step"}
    del b, half
    out["note"] = ("dense = every launch rescans the whole domain (fc_activity_scan, one fused "
                   "kernel: the burning plane read once, quiet tiles' next state written as zeros "
                   "= 256 B per 32x32 "
                   "tile per launch = 0.25/K B per cell-update) and advances the live tiles; "
                   "skip = incremental activity lists.  The SURVEY's 18 B/cell-update fp32-field "
                   "design would cap a dense sweep at peak/18 = 3.6e11 cu/s")
    return out


def spawn_ranks(args) -> bool:
    """--gpus N > 1 outside torchrun: re-launch this command as N ranks (one
    process per GPU) through torch.distributed.run; rank 0 prints the line."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return False
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    raise SystemExit(subprocess.call(cmd))


def main():
    args = parse()
    spawn_ranks(args)
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        # NCCL's INFO log (rings, channels, P2P over NVLink) on stderr, so the
        # run shows the N ranks it used; stdout keeps the one JSON line
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
