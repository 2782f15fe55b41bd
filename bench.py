#!/usr/bin/env python
"""bench.py — GSGP hot path on B200: precompute points/s (W^T W + W^T y) on the 3-D
radar-like config (BASELINE.json configs[2]: n = 1.2e8 fp32 rows, grid 80×80×20, cubic),
plus factorized-CG iterations/s of the posterior-mean solve on the resulting statistics.

One JSON line on rank 0 (contract in the task prompt):
  value   — whole-job precompute throughput, inputs resident in HBM (CUDA events, max over ranks)
  e2e     — same metric through the public API with HOST (pinned) rows: H2D of the rows and
            D2H of W^T y, y^T y, n inside the timed region
  roofline— K1 (per-cell moments kernel) vs its binding peak: the FP64 tensor pipe at d = 3
            (DMMA peak measured live), HBM otherwise; the HBM view is kept as a sub-object
  cpu_baseline — the reference's own sufficient_stats (oracle/_ref: the reference sources
            compiled against stand-in Eigen/FFTW headers, kind "reference"; the oracle
            restatement, kind "port", only if that library is absent) on one pinned host
            thread over a bounded prefix sample of the same workload
`--impl reference` times only that CPU path on the same config.

`--gpus N` (N > 1) starts N ranks itself under torch.distributed.run when no torchrun
environment is present.  Default scaling is strong: the config's n rows are split over the ranks
(rank r holds rows [r·n/N, (r+1)·n/N) of one synthetic stream); `--scaling weak` keeps n rows per
rank.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "precompute points/sec (W^T W+W^T y) & factorized-CG iters/sec; % of HBM roofline"
PUBLISHED_PTS_PER_S = 120e6 / 4861.60  # 1.2e8-point radar precompute, Xeon Gold 6240


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", type=int, default=3)
    p.add_argument("--n", type=int, default=0, help="rows per rank (default: the config's n)")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--no-cg", action="store_true")
    p.add_argument("--cpu-seconds", type=float, default=12.0,
                   help="all-core sharded CPU figure: target seconds of work")
    p.add_argument("--cpu-rows", type=int, default=200_000,
                   help="single-thread CPU baseline: prefix rows per trial (SURVEY §8(d): >= 2e5 at d = 3)")
    p.add_argument("--cpu-trials", type=int, default=3)
    p.add_argument("--ref-rows", type=int, default=0,
                   help="rows per step of the reference arm (0 = sized so that steps + warmup take ~4 minutes "
                        "at ~6e3 rows/s on one host thread, at most 1e5)")
    p.add_argument("--cpu-sharded", action="store_true",
                   help="also time the oracle sharded over all host threads (merge(); labelled separately)")
    p.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                   help="strong: the config's n rows split over the ranks (north star); weak: n rows per rank")
    p.add_argument("--traffic-file", default=os.path.join(ROOT, "profiles", "traffic.json"))
    return p.parse_args()


# ---------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:  # noqa: BLE001
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:  # noqa: BLE001
            self.proc.kill()
        rows = []
        for ln in open(self.path):
            parts = [s.strip() for s in ln.split(",")]
            if len(parts) >= 9:
                rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}

        def num(s):
            try:
                return float(s)
            except ValueError:
                return float("nan")

        sm = np.array([num(r[1]) for r in rows])
        mx = np.nanmax([num(r[2]) for r in rows])
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        load = sm[sm > 0.5 * np.nanmax(sm)] if np.isfinite(sm).any() else sm
        return {"sm_mhz": float(np.nanmedian(load)), "sm_max_mhz": float(mx), "reasons": reasons,
                "samples": len(rows)}


# ---------------------------------------------------------------- roofline arithmetic
def algorithmic_bytes(n, m, s_min, b_pt):
    """B_pre = n·b_pt + 8·m·(S_min + 1)."""
    return n * b_pt + 8.0 * m * (s_min + 1)


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        d = json.load(open(path))
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


# ---------------------------------------------------------------- CPU (reference / oracle) timing
def cpu_checker():
    """(front-end module, kind, what): the reference's own code when oracle/_ref is built
    (it travels to the GPU box prebuilt), else the oracle restatement."""
    import oracle as O

    try:
        import oracle.ref as R

        if R.available():
            return R._mod, "reference", ("the reference's own sufficient_stats (interp.cpp:244-263; its sources compiled "
                                         "against stand-in Eigen/FFTW headers, oracle/refshim)")
    except Exception:  # noqa: BLE001
        pass
    O.build()
    return O, "port", "oracle restatement of sufficient_stats (std::unordered_map accumulation, interp.cpp:179-221)"


def cpu_rate(x, y, grid_o, scheme, nthreads, target_s):
    """Points/s of the CPU checker (reference algorithm) on a prefix sample."""
    O = cpu_checker()[0]

    n_all = x.shape[0]
    s = min(n_all, 2000 * nthreads)
    while True:
        t0 = time.perf_counter()
        st = O.sufficient_stats(grid_o, x[:s], y[:s], scheme=scheme, nthreads=nthreads)
        el = time.perf_counter() - t0
        del st
        if el >= target_s / 3 or s >= n_all:
            return s / el, s, el
        s = min(n_all, int(s * max(2.0, (target_s / 2) / max(el, 1e-3))))


T975 = {1: 12.706, 2: 4.303, 3: 3.182, 4: 2.776, 5: 2.571, 6: 2.447, 7: 2.365, 8: 2.306, 9: 2.262}


def mean_ci(v):
    """Mean and 95 % CI half-width (Student t) of repeated trials (bench.cpp:105-121 style)."""
    v = np.asarray(v, dtype=np.float64)
    if v.size < 2:
        return float(v.mean()), float("nan")
    return float(v.mean()), float(T975.get(v.size - 1, 1.96) * v.std(ddof=1) / np.sqrt(v.size))


def cpu_single_thread(x, y, grid_o, rows, trials):
    """the oracle restatement (the reference algorithm: one std::unordered_map
    accumulator, interp.cpp:179-221) on ONE host thread pinned to one core (sched_setaffinity
    of the calling thread = taskset), 1 warm-up then `trials` timed runs over a `rows`-row prefix;
    sufficient_stats wall time → points/s, mean and 95 % CI."""
    O, kind, what = cpu_checker()

    rows = min(rows, x.shape[0])
    old = os.sched_getaffinity(0)
    core = max(old)
    os.sched_setaffinity(0, {core})
    try:
        w = min(rows, 20_000)
        O.sufficient_stats(grid_o, x[:w], y[:w], scheme=1, nthreads=1)
        times = []
        for _ in range(trials):
            t0 = time.perf_counter()
            st = O.sufficient_stats(grid_o, x[:rows], y[:rows], scheme=1, nthreads=1)
            times.append(time.perf_counter() - t0)
            del st
    finally:
        os.sched_setaffinity(0, old)
    rates = [rows / t for t in times]
    mean, ci = mean_ci(rates)
    return {"value": mean, "unit": "points/s", "cores": 1, "threads": 1, "kind": kind, "ci95": ci,
            "trials": [round(t, 3) for t in times],
            "sample": f"first {rows} rows of the bench workload, 1 warm-up + {trials} trials, one thread pinned "
                      f"to core {core} ({what})"}


def cpu_lscpu():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.lower().startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:  # noqa: BLE001
        pass
    return "unknown"


def oracle_grid(grid):
    O = cpu_checker()[0]

    d = grid.dim()
    return O.Grid([grid.min(k) for k in range(d)], [grid.max(k) for k in range(d)], [grid.size(k) for k in range(d)])


# ---------------------------------------------------------------- reference arm
def run_reference(args):
    """The reference's CPU path on this box: its own sufficient_stats (oracle/_ref; the oracle
    restatement if that library is absent) — one std::unordered_map accumulator in stream order,
    interp.cpp:179-221; the reference's precompute is single-threaded, so one thread pinned to
    one core is all the threads it can use — each step a bounded prefix sample of the bench
    workload."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2101_11751_b200 import synthetic as S

    O, kind, what = cpu_checker()
    cfg = S.CONFIGS[args.config]
    ref_rows = args.ref_rows or max(20_000, min(100_000, 1_400_000 // max(1, args.steps + args.warmup)))
    rows = min(cfg.n, ref_rows)
    x, y = S.generate(args.config, n=rows)
    grid = S.grid_for(cfg)
    og = oracle_grid(grid)
    old = os.sched_getaffinity(0)
    core = max(old)
    os.sched_setaffinity(0, {core})
    times = []
    try:
        for i in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            st = O.sufficient_stats(og, x, y, scheme=1, nthreads=1)
            el = time.perf_counter() - t0
            del st
            if i >= args.warmup:
                times.append(el)
    finally:
        os.sched_setaffinity(0, old)
    ms = 1e3 * float(np.mean(times))
    value = rows / (ms / 1e3)
    _, ci = mean_ci([rows / t for t in times])
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "points/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": value / PUBLISHED_PTS_PER_S, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"config{args.config} ({cfg.name}) prefix sample", "sample_rows": rows,
                   "grid": list(cfg.sizes), "scheme": "cubic"},
        "cpu_baseline": {"value": value, "unit": "points/s", "cores": 1, "threads": 1, "kind": kind, "ci95": ci,
                         "cpu": cpu_lscpu(), "trials": [round(t, 3) for t in times],
                         "sample": f"first {rows} rows of config {args.config} per step, one thread pinned to core "
                                   f"{core} ({what}; the reference precompute is single-threaded)"},
        "e2e": {"value": value, "unit": "points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- our arm
def run_ours(args):
    import torch

    import paper_2101_11751_b200 as G
    from paper_2101_11751_b200 import synthetic as S
    from paper_2101_11751_b200.build import build

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    build()
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist  # noqa: F811

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        from paper_2101_11751_b200.distributed import allreduce_stats

    cfg = S.CONFIGS[args.config]
    # strong scaling (default, the north star): the config's n rows split over the ranks, rank r
    # holding rows [r·n/N, (r+1)·n/N) of the one synthetic stream; weak: n rows per rank
    n_total = (args.n or cfg.n) * (world if args.scaling == "weak" else 1)
    lo, hi = S.shard_range(n_total, world, rank)
    n = hi - lo
    ctx = G.Context(local)
    ext = torch.cuda.ExternalStream(ctx.stream, device=torch.device("cuda", local))
    rows = S.generate_torch(args.config, n, device=f"cuda:{local}", start=lo)
    torch.cuda.synchronize()
    grid = S.grid_for(cfg)
    spec = S.kernel_for(cfg)
    acc = G.SufficientStatsAccumulator(grid, G.InterpScheme.Cubic, ctx=ctx)

    def step(src):
        acc.reset()
        acc.add(src)
        st = acc.finalize()
        if world > 1:
            allreduce_stats(st)
        return st

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()
        ctx.synchronize()

    def max_over_ranks(v):
        if dist is None:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(args.warmup):
        step(rows)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(local)
    clocks.start()
    l0 = ctx.launch_count
    barrier()
    e0.record(ext)
    for _ in range(args.steps):
        st = step(rows)
    e1.record(ext)
    e1.synchronize()
    barrier()
    launches = ctx.launch_count - l0
    clk = clocks.stop()
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps)
    value = n_total / (ms / 1e3)

    # per-phase device times (separate pass: phase events add host syncs)
    ctx.enable_phase_timing(True)
    ctx.reset_phase_times()
    for _ in range(args.steps):
        step(rows)
    phases = ctx.phase_times()
    ctx.enable_phase_timing(False)
    # per STEP (a batch above 2^27 rows runs in several device chunks: one K1 launch per chunk)
    ph_ms = {k: v[0] / args.steps for k, v in phases.items()}
    k1_ms = ph_ms.get("moments", float("nan"))
    k1_launches = phases.get("moments", (0.0, args.steps))[1] / args.steps

    m = grid.num_points()
    s_min = st.n_offsets()
    b_pt = (cfg.d + 1) * (4 if cfg.dtype == "f32" else 8)
    b_pre = algorithmic_bytes(n, m, s_min, b_pt)
    hbm_peak, peak_src = load_peaks()
    fp64_peak = ctx.fp64_peak_tflops()
    W = 4
    qx, qy = (2 * W - 1) ** cfg.d, W ** cfg.d
    flops_pt = 2.0 * (qx + qy)  # minimal FP64 work per point: one FMA per moment
    traffic = None
    if os.path.exists(args.traffic_file):
        try:
            tf = json.load(open(args.traffic_file))
            traffic = tf.get(f"config{args.config}", {}).get("k_moments_bytes_per_launch")
        except Exception:  # noqa: BLE001
            traffic = None
    achieved = b_pre / (k1_ms / 1e3) / 1e9
    flops_ach = flops_pt * n / (k1_ms / 1e3) / 1e12
    hbm = {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s", "frac": achieved / hbm_peak,
           "traffic": traffic, "peak_source": f"{peak_src} MEASURED_PEAKS.json hbm_gbs",
           "algorithmic_bytes_per_launch": b_pre / k1_launches, "k1_launches_per_step": k1_launches,
           "rows_per_launch": n / k1_launches, "k1_ms_per_launch": k1_ms / k1_launches}
    if cfg.d == 3:
        # K1 at d = 3 runs its 407 moment MACs per row on the FP64 tensor pipe (DMMA): that pipe,
        # not HBM, binds it (814 flop per 16-byte row).  MEASURED_PEAKS.json has no FP64 figure
        # and B200_PROFILING.md none either, so the peak is measured in this run by the
        # library's DMMA loop (gsgpc_diag_fp64_tensor).
        dmma_peak = ctx.fp64_tensor_tflops()[0]
        roofline = {
            "bound": "tensor", "kernel": "k_moments_d3c_mma (K1: per-cell polynomial moments, FP64 DMMA)",
            "achieved": flops_ach, "peak": dmma_peak, "unit": "TFLOP/s", "frac": flops_ach / dmma_peak,
            "traffic": traffic,
            "peak_source": "measured in this run: gsgpc_diag_fp64_tensor (mma.sync.m8n8k4.f64 loop); "
                           "MEASURED_PEAKS.json has no FP64 entry",
            "flops_per_point": flops_pt, "algorithmic_flops_per_launch": flops_pt * n / k1_launches,
            "k1_ms": k1_ms, "phase_ms": ph_ms,
            "hbm": hbm,
            "fp64_dfma_peak": fp64_peak,
            "note": "algorithmic flops = one FMA per needed moment (343 + 64 per row); the DMMA tiles execute "
                    "512 FMAs per row (8 m8n8k4 per 4 rows)",
        }
    else:
        k1_name = "k_moments_d2c_mma (K1: per-cell polynomial moments, FP64 DMMA)" if cfg.d == 2 else \
            "k_moments_lane (K1: per-cell polynomial moments)"
        roofline = dict(hbm, kernel=k1_name, k1_ms=k1_ms, phase_ms=ph_ms,
                        fp64={"achieved": flops_ach, "peak": fp64_peak, "unit": "TFLOP/s",
                              "frac": flops_ach / fp64_peak, "flops_per_point": flops_pt,
                              "peak_source": "measured (gsgpc_diag_fp64_peak DFMA loop, this run)"})
    roofline["step_achieved_gbs"] = b_pre / (ms / 1e3) / 1e9

    # factorized CG on the merged statistics (replicated on every rank, "replicas only"):
    # (1) iterations/s of the posterior-mean EFCG over a fixed window (loop_seconds, as the
    #     reference's bench does, bench.cpp:144-152);
    # (2) time to solution of posterior_mean_gsgp (gp.cpp:326-352) at the config's tolerance:
    #     prep (r̂0 = −K_G W^T y/σ², eps) + the converged loop + mean_coeffs = K_G(x̂ + W^T y/σ²)
    #     (bench.cpp:136-152 reports prep and loop times the same way).
    cg = None
    if not args.no_cg:
        kg = G.ToeplitzOperator(grid, spec, ctx=ctx)
        s2 = cfg.noise_std ** 2
        rhat0 = -kg.apply(st.wty()) / s2
        tol = G.GridRhsTolerance(eps_abs=cfg.tol * cfg.tol * st.yty())
        res = []
        for i in range(args.warmup + args.steps):
            r = G.factorized_cg_grid_rhs(kg, st, rhat0, cfg.noise_std, tol, 2000 if cfg.d == 3 else 500)
            if i >= args.warmup:
                res.append(r)
        iters = sum(r.iterations for r in res)
        secs = sum(r.loop_seconds for r in res)
        ips = iters / secs if secs > 0 else float("nan")
        b_it = 8.0 * m * s_min + 128.0 * m
        G.posterior_mean_gsgp(st, kg, spec, G.InterpScheme.Cubic, cfg.noise_std, cfg.tol, 50000)  # warm
        tts = []
        for _ in range(2):
            ctx.synchronize()
            t0 = time.perf_counter()
            model = G.posterior_mean_gsgp(st, kg, spec, G.InterpScheme.Cubic, cfg.noise_std, cfg.tol, 50000)
            tts.append((time.perf_counter() - t0, model))
        wall, model = min(tts, key=lambda t: t[0])
        cg = {"iters_per_sec": ips, "ms_per_iter": 1e3 / ips, "window_iterations": res[0].iterations,
              "tol": cfg.tol,
              "time_to_solution": {"seconds": wall, "loop_seconds": model.loop_seconds,
                                   "prep_seconds": wall - model.loop_seconds, "iterations": model.solve_iterations,
                                   "converged": True,
                                   "relative_residual": float(np.sqrt(model.solve_residual_sq / st.yty())),
                                   "what": "posterior_mean_gsgp(stats, K_G, tol) through the public API, converged "
                                           "(eps = tol²·yᵀy, gp.cpp:326-352), best of 2"},
              "roofline": {"bound": "hbm", "kernel": "k_efcg_persistent (K3 stencil SpMV + K4 K_G modes + updates)",
                           "algorithmic_bytes_per_iter": b_it, "achieved": b_it * ips / 1e9, "peak": hbm_peak,
                           "unit": "GB/s", "frac": b_it * ips / 1e9 / hbm_peak}}

    # end-to-end through the public API with host (pinned) rows
    e2e = None
    if not args.no_e2e:
        host_rows = rows.cpu().pin_memory()
        st = step(host_rows)
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            st = step(host_rows)
            wty = st.wty()
            yty = st.yty()
            nn = st.n()
        barrier()
        el = (time.perf_counter() - t0) / args.steps
        el = max_over_ranks(el)
        h2d = int(host_rows.numel() * host_rows.element_size())
        # the link roofline of the end-to-end number: pinned host→device copy bandwidth, measured
        # here with one 2 GiB copy, best of 5
        hb = torch.empty(1 << 29, dtype=torch.float32).pin_memory()
        db = torch.empty(1 << 29, dtype=torch.float32, device=f"cuda:{local}")
        best = float("inf")
        for _ in range(5):
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            db.copy_(hb, non_blocking=True)
            torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t1)
        link_gbs = hb.numel() * 4 / best / 1e9
        del hb, db
        e2e = {"value": n_total / el, "unit": "points/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": int(wty.nbytes + 16), "ms_per_step": el * 1e3,
               "timing": "host perf_counter around synchronous API calls (H2D staging + compute + D2H), max over "
                         "ranks",
               "roofline": {"bound": "h2d_link", "achieved": h2d / el / 1e9, "peak": link_gbs, "unit": "GB/s",
                            "frac": h2d / el / 1e9 / link_gbs,
                            "peak_source": "measured in this run: one 2 GiB pinned host→device copy, best of 5"}}
        assert nn == n_total and np.isfinite(yty)
        del host_rows

    # CPU baseline (rank 0, N = 1 only): the oracle restatement of the reference on one pinned
    # thread, plus the all-core sharded figure labelled separately
    cpu = None
    if not args.no_cpu and rank == 0 and world == 1:
        samp = rows[: min(n, max(args.cpu_rows, 4_000_000))].cpu().numpy()
        og = oracle_grid(grid)
        cpu = cpu_single_thread(samp[:, : cfg.d], samp[:, cfg.d], og, args.cpu_rows, args.cpu_trials)
        cpu["cpu"] = cpu_lscpu()
        if args.cpu_sharded:
            threads = os.cpu_count() or 1
            rate, s_all, el_all = cpu_rate(samp[:, : cfg.d], samp[:, cfg.d], og, 1, threads, args.cpu_seconds)
            cpu["sharded_all_cores"] = {
                "value": rate, "unit": "points/s", "cores": threads,
                "sample": f"sharded, {threads} cores: first {s_all} rows ({el_all:.1f} s; one accumulator per "
                          f"thread, merge(), interp.cpp:202-210)"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "points/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": value / PUBLISHED_PTS_PER_S, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"config{args.config}: {cfg.name}, n={n_total} rows "
                                   f"({'fp32' if cfg.dtype == 'f32' else 'fp64'} (x, y) rows), grid "
                                   f"{'x'.join(map(str, cfg.sizes))} (m={m}), cubic, fp64 accumulation",
                       "n_total": n_total, "n_per_rank": n, "grid": list(cfg.sizes), "scheme": "cubic",
                       "parallelism": f"dp{world} (rows sharded, NCCL all-reduce of statistics; solve replicated)",
                       "l2": f"inputs {n * b_pt / 1e9:.2f} GB per rank"
                             + (" > 126 MB L2" if n * b_pt > 126e6 else " (< L2: not flushed)")},
            "e2e": e2e, "roofline": roofline, "cpu_baseline": cpu, "cg": cg, "clocks": clk,
            "gpu_launches": int(launches), "gpu_launches_per_step": launches / args.steps,
            "version": G.version(),
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def relaunch_under_torchrun(args):
    """`--gpus N` without a torchrun environment: start the N ranks here (one process per GPU,
    torch.distributed.run on 127.0.0.1) with NCCL's INFO log in gpurun_out/ (not on stdout, where
    rank 0 prints the one JSON line)."""
    import socket

    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    if "NCCL_DEBUG_FILE" not in env:
        os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
        env["NCCL_DEBUG_FILE"] = os.path.join(ROOT, "gpurun_out", f"nccl_n{args.gpus}.%h.%p.log")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        sys.exit(relaunch_under_torchrun(args))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
