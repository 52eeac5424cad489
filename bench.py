#!/usr/bin/env python
"""AeroSketch update throughput on B200 (BASELINE.json metric: sketch update
throughput, rows/s, at given d, eps; roofline fraction; CPU baseline beside).

Workload (default): config C2 of BASELINE.json -- persistent (ATTP) stream,
d=4096, eps=1/512 (ell=1024), low-rank-plus-noise generator k=256,
sigma_j=0.99^j, noise 0.05, ||a||^2 log-uniform in [1,256]; fp64.
A "step" = one update_block over `rows_per_step` consecutive rows of the
stream. `value` = rows/s with inputs resident in HBM; `e2e` = the same through
the public C-ABI with pinned host rows (H2D + event-log D2H inside the timed
region). Multi-GPU: replicas only (one independent stream per GPU;
DESIGN.md section 6).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
"""
import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "c1": dict(kind="attp", d=1024, eps=1 / 16, k=32, rho=0.9, noise=0.1, r_max=64.0, n=131072,
               rows_per_step=16384, cpu_rows=4000,
               name="C1 persistent stream n=131072 d=1024 eps=1/16 (k=32, sigma=0.9^j, noise 0.1, R=64)"),
    "c2": dict(kind="attp", d=4096, eps=1 / 512, k=256, rho=0.99, noise=0.05, r_max=256.0, n=1048576,
               rows_per_step=8192, cpu_rows=400,
               name="C2 tight-eps persistent stream n=1048576 d=4096 eps=1/512 "
                    "(k=256, sigma=0.99^j, noise 0.05, R=256)"),
    "c3": dict(kind="sw", d=1024, eps=1 / 64, k=64, rho=0.9, noise=0.1, r_max=1024.0, n=1048576,
               window=65536, drift=131072, rows_per_step=8192, cpu_rows=600, steady_rows=131072,
               name="C3 sliding window N=65536 n=1048576 d=1024 eps=1/64 R=1024 (k=64, drift 131072)"),
    "c4": dict(kind="dist", d=2048, eps=1 / 128, k=128, rho=0.97, noise=0.1, r_max=64.0, n=1048576,
               k2=16, rho2=0.9, scale2=0.5, rows_per_step=4096, cpu_rows=300, sites=8,
               name="C4 distributed, m=8 sites spread over the GPUs (one per GPU at 8), d=2048 eps=1/128 "
                    "(global k=128 + site k=16, noise 0.1, R=64)"),
    "c5": dict(kind="amm", dx=1024, dy=768, d=1024, eps=1 / 64, latent=48, noise=0.1, r_max=64.0,
               n=1048576, window=65536, rows_per_step=4096, cpu_rows=200, steady_rows=65536,
               name="C5 sliding-window AMM dx=1024 dy=768 N=65536 eps=1/64 (latent 48, noise 0.1)"),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default=None, choices=sorted(CONFIGS),
                    help="default: c2 (the headline) on one GPU; c4 (the distributed config, "
                         "m=8 sites over the N GPUs) under torchrun with N > 1")
    ap.add_argument("--sites", type=int, default=0, help="C4 site count m (default 8, fixed as N grows)")
    ap.add_argument("--rows-per-step", type=int, default=0)
    ap.add_argument("--cpu-rows", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-steady", action="store_true",
                    help="C3/C5: skip the untimed steady-state prefix (2N / N rows)")
    ap.add_argument("--rng", default="device", choices=["device", "host"],
                    help="random projections drawn on the device, or on the host and uploaded "
                         "(AERO_FLAG_HOST_RNG: bit-identical to the reference's rng.hpp)")
    return ap.parse_args()


class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region, through
    NVML in-process (the library nvidia-smi reads; spawning nvidia-smi every
    few hundred ms takes driver locks and perturbs a host-driven loop), with
    the nvidia-smi CLI as the fallback."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.samples, self.stop_ev = index, [], threading.Event()
        self.th = threading.Thread(target=self.run, daemon=True)
        self.nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            phys = int(vis.split(",")[index]) if vis and vis.split(",")[index].strip().isdigit() else index
            self.h = pynvml.nvmlDeviceGetHandleByIndex(phys)
            self.nvml = pynvml
        except Exception:
            self.nvml = None

    def sample_nvml(self):
        n, h = self.nvml, self.h
        sm = n.nvmlDeviceGetClockInfo(h, n.NVML_CLOCK_SM)
        mx = n.nvmlDeviceGetMaxClockInfo(h, n.NVML_CLOCK_SM)
        pw = n.nvmlDeviceGetPowerUsage(h) / 1000.0
        r = n.nvmlDeviceGetCurrentClocksEventReasons(h)
        bits = [0x8, 0x40, 0x20, 0x4]  # hw_slowdown, hw_thermal, sw_thermal, sw_power_cap
        return [str(sm), str(mx), f"{pw:.1f}"] + ["Active" if r & b else "Not Active" for b in bits]

    def run(self):
        while not self.stop_ev.is_set():
            try:
                if self.nvml is not None:
                    self.samples.append(self.sample_nvml())
                else:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                         timeout=5).stdout.strip()
                    if out:
                        self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self.stop_ev.wait(0.25)

    def __enter__(self):
        self.th.start()
        return self

    def __exit__(self, *a):
        self.stop_ev.set()
        self.th.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 3 + i and s[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def fp64_peak_tflops(torch, dev):
    """Measured dense fp64 GEMM peak on this GPU (cuBLAS DGEMM 8192^3, best of
    5): the roofline denominator for the fp64 products (MEASURED_PEAKS.json
    carries only bf16 and HBM)."""
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device=dev)
    b = torch.randn(n, n, dtype=torch.float64, device=dev)
    torch.matmul(a, b)
    torch.cuda.synchronize(dev)
    best = 0.0
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b)
        e1.record()
        e1.synchronize()
        best = max(best, 2 * n ** 3 / (e0.elapsed_time(e1) * 1e-3) / 1e12)
    del a, b
    torch.cuda.empty_cache()
    return best


def reference_literal_flops(ev, d, ell):
    """SURVEY.md section 8(d) F_row: the reference's own flop count per row
    (power-iteration gate, simul_iter doubling calls, FD reduce by SVD, dumps),
    evaluated on this run's event log."""
    import math
    import numpy as np
    kp = math.ceil(math.log2(d)) + 1
    q = math.ceil(math.log2(d) / 0.4)
    r = ev["rows_after"].astype(np.float64)
    f = (4 * kp + 2) * d * r * (ev["gate_fired"] >= 0)
    steps = ev["doubling_steps"].astype(np.int64)
    for s_ in range(1, int(steps.max()) + 1 if len(steps) else 1):
        k = np.minimum(2.0 ** s_, r)
        on = steps >= s_
        f = f + on * ((4 * q + 4) * d * r * k + (8 * q + 10) * d * k * k)
    red = 2 * (2 * ell) ** 2 * d + 9 * (2 * ell) ** 3 + 2 * (ell - 1) * (2 * ell) * d
    f = f + ev["reduced"].astype(np.float64) * float(red) + 8.0 * r * d * ev["xi"].astype(np.float64)
    return float(f.mean())


def committed_product_flops(ev, d):
    """fp64-equivalent flops of the Gram-form products of the rows the run
    COMMITTED (2 r^2 per iterate column and phase: the gate's kp+1 phases on
    one column, every simul_iter call's q+1 phases on k columns), from the
    event log. Speculative rows that a dump discarded are not in the log, so
    they do not count here (they do in the kernel's own flop counter)."""
    import numpy as np
    kp = math.ceil(math.log2(d)) + 1
    q = math.ceil(math.log2(d) / 0.4)
    r = ev["rows_after"].astype(np.float64)
    f = 2.0 * r * r * (kp + 1)
    steps = ev["doubling_steps"].astype(np.int64)
    for s_ in range(1, int(steps.max()) + 1 if len(steps) else 1):
        k = np.minimum(2.0 ** s_, r)
        f = f + (steps >= s_) * 2.0 * r * r * k * (q + 1)
    return float(f.sum())


def attp_cycle(cfg, S, warm, steps):
    """The first full FD-reduce cycle inside the GPU arm's timed rows: the
    reduce fires at row 2*ell, then every ell+1 rows (sketch.cpp:92-95,
    data-independent), so the residual size r -- which sets the per-row cost --
    is periodic with period ell+1. Returns (first row after a reduce, ell)."""
    ell = int(math.ceil(2.0 / cfg["eps"]))
    start = warm * S + 1
    m = max(0, -(-(start - 1 - 2 * ell) // (ell + 1)))  # reduce rows 2ell + m(ell+1) >= start - 1
    t_red = 2 * ell + m * (ell + 1)
    if t_red + ell + 1 > (warm + steps) * S:
        raise ValueError("timed region shorter than one reduce cycle")
    return t_red + 1, ell


def attp_cpu_sample(cfg, S, warm, steps, threads, points, per_point, warm_points=0, device=0):
    """Like-for-like CPU timing of the GPU arm's steady-state rows (the oracle
    restatement, or the reference arm): the GPU engine (untimed setup) replays
    the same stream up to each sample point, its live state (residual rows,
    fork counter, clock, last dump time, mass) is imported into the oracle,
    and the oracle's update() is timed on the next `per_point` rows. The
    points are spread evenly over one FD-reduce cycle of the timed region
    (so their mean residual size is the cycle's), plus the cycle's reduce row
    timed on its own. Rate = (ell+1) / (ell * mean t_row + t_reduce_row)."""
    import numpy as np
    import torch
    import paper_2601_02019_b200 as prod
    from oracle import pyoracle as orc
    orc.set_threads(threads)
    c0, ell = attp_cycle(cfg, S, warm, steps)
    period = ell + 1
    xs = [c0 + (i * (period - per_point)) // max(1, points) for i in range(points)]
    warm_xs = [c0 + (i * (period - per_point)) // max(1, warm_points) for i in range(warm_points)]
    red_row = c0 + ell  # the cycle's reduce row
    d = cfg["d"]
    last = red_row
    dev = torch.device("cuda", device)
    rows = torch.empty((last, d), dtype=torch.float64, device=dev)
    prod.gen_rows_device(rows, 1, d, cfg["k"], cfg["rho"], cfg["noise"], cfg["r_max"], seed=1, stream=0,
                         device=device)
    torch.cuda.synchronize(dev)
    ts = np.arange(1, last + 1, dtype=np.int64)
    gpu = prod.AttpState(d, cfg["eps"], seed=1, stream=1000, device=device)
    pos = 0
    t_rows, t_warm, t_red = [], [], None
    targets = sorted(set([(x, "w") for x in warm_xs] + [(x, "t") for x in xs] + [(red_row, "r")]))
    for x, kind in targets:
        if x - 1 > pos:
            gpu.update_block(rows[pos:x - 1], ts[pos:x - 1])
            pos = x - 1
        inf = gpu.info()
        res = gpu.residual()
        o = orc.AttpState(d, cfg["eps"], 1, 1000)
        o.import_state(res, inf.forks, inf.clock, inf.last_dump_t, inf.theta, inf.fro_mass)
        n = 1 if kind == "r" else per_point
        host = rows[x - 1:x - 1 + n].cpu().numpy()
        t0 = time.perf_counter()
        ev = o.update_block(host, ts[x - 1:x - 1 + n])
        dt = time.perf_counter() - t0
        if kind == "r":
            assert ev["reduced"][0] == 1, "cycle reduce row did not reduce"
            t_red = dt
        elif kind == "t":
            assert not ev["reduced"].any()
            t_rows.append(dt / n)
        else:
            t_warm.append(dt / n)
    del gpu, rows
    torch.cuda.empty_cache()
    mean_row = float(np.mean(t_rows))
    rate = period / (ell * mean_row + t_red)
    sample = (f"{points} points x {per_point} rows spread over the FD-reduce cycle rows {c0}..{red_row} of the "
              f"GPU arm's timed region (rows {warm * S + 1}..{(warm + steps) * S}) plus that cycle's reduce row, "
              f"each from the GPU run's exported live state; rate = (ell+1)/(ell*mean_row + reduce_row) with "
              f"mean_row {mean_row * 1e3:.1f} ms, reduce_row {t_red * 1e3:.0f} ms")
    return rate, sample, t_rows, t_red


def gpu_arm_steps(args):
    """(warm-up, timed) steps of the GPU arm: the driver launches both arms
    with the same --steps/--warmup, so the reference arm samples the rows the
    GPU arm times."""
    return args.warmup, args.steps


def run_reference(args, cfg, rank):
    """--impl reference: the reference path's CPU implementation (the oracle
    port; the reference C++ needs Eigen, absent here) on all host threads."""
    if rank != 0:
        return
    from oracle import pyoracle as orc
    import numpy as np
    threads = os.cpu_count() or 1
    orc.set_threads(threads)
    if cfg["kind"] != "attp":
        sites = (args.sites or cfg.get("sites", 8)) if cfg["kind"] == "dist" else 1
        n = max(20, (args.cpu_rows or cfg["cpu_rows"]) // sites)
        v, _ = cpu_other_rate(cfg, n, threads, sites=sites)
        unit = "row-site updates/s" if cfg["kind"] == "dist" else "rows/s"
        print(json.dumps({
            "impl": "reference", "metric": "sketch update throughput", "value": v, "unit": unit,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": n * 1e3 / v, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg["name"], "rows_per_step": n},
            "cpu_baseline": {"value": v, "unit": unit, "cores": threads, "kind": "port",
                             "sample": f"rows 1..{n} of {args.config.upper()} ({sites} site(s)) from an empty state"},
            "e2e": {"value": v, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }), flush=True)
        return
    # the GPU arm's config and timed rows; each step = one sample point
    S = args.rows_per_step or cfg["rows_per_step"]
    gwarm, gsteps = gpu_arm_steps(args)
    v, sample, t_rows, t_red = attp_cpu_sample(cfg, S, gwarm, gsteps, threads, points=args.steps,
                                               per_point=cfg.get("ref_rows_per_point", 2),
                                               warm_points=args.warmup)
    print(json.dumps({
        "impl": "reference", "metric": "sketch update throughput", "value": v, "unit": "rows/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": float(np.mean(t_rows)) * cfg.get("ref_rows_per_point", 2) * 1e3,
        "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg["name"], "rows_per_step": S, "same_config": True,
                   "timed_rows": f"{gwarm * S + 1}..{(gwarm + gsteps) * S}"},
        "cpu_baseline": {"value": v, "unit": "rows/s", "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": v, "unit": "rows/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def oracle_stream(cfg, nrows, stream=0):
    """Host rows of the config generator (oracle restatement, CPU baseline only)."""
    from oracle import pyoracle as orc
    if cfg["kind"] == "amm":
        return orc.gen_amm_rows(1, cfg["dx"], cfg["dy"], cfg["latent"], cfg["noise"], cfg["r_max"], 1, nrows)
    return orc.gen_rows(cfg["d"], cfg["k"], cfg["rho"], cfg["noise"], cfg["r_max"], 1, stream, 1, nrows,
                        drift=cfg.get("drift", 0), k2=cfg.get("k2", 0), rho2=cfg.get("rho2", 0.9),
                        scale2=cfg.get("scale2", 0.5))


def cpu_other_rate(cfg, nrows, threads, sites=1):
    """Oracle restatement of the config's update loop over rows 1..nrows."""
    from oracle import pyoracle as orc
    import numpy as np
    orc.set_threads(threads)
    ts = np.arange(1, nrows + 1)
    if cfg["kind"] == "sw":
        rows = oracle_stream(cfg, nrows)
        s = orc.MlState(cfg["d"], cfg["window"], cfg["r_max"], cfg["eps"], 1, 1000)
        t0 = time.perf_counter()
        s.update_block(rows, ts)
        return nrows / (time.perf_counter() - t0), nrows
    if cfg["kind"] == "amm":
        x, y = oracle_stream(cfg, nrows)
        s = orc.CodState(cfg["dx"], cfg["dy"], cfg["eps"], cfg["eps"] * cfg["window"], cfg["window"], 1, 1000)
        t0 = time.perf_counter()
        s.update_block(x, y, ts)
        return nrows / (time.perf_counter() - t0), nrows
    streams = np.stack([oracle_stream(cfg, nrows, j) for j in range(sites)])
    t0 = time.perf_counter()
    orc.dist_run(streams, cfg["eps"], query_every=0, seed=1, probes=False)
    return sites * nrows / (time.perf_counter() - t0), nrows


def run_other(args, cfg, world, rank, local):
    """C3 (MlState), C4 (distributed, one site per GPU), C5 (CodState)."""
    import numpy as np
    import torch
    import paper_2601_02019_b200 as prod
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    group = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    S = args.rows_per_step or cfg["rows_per_step"]
    steps, warm = args.steps, args.warmup
    # untimed prefix that brings the window configs to steady state before the
    # W warm-up steps: C3 2N rows (window expiry, level caps, the first drift
    # epoch at 131072), C5 N rows (expiry of snapshots)
    pre = 0 if args.no_steady else cfg.get("steady_rows", 0)
    pre = (pre + S - 1) // S  # in steps
    nrows = S * (pre + steps + warm)
    kind = cfg["kind"]
    ts_all = np.arange(1, nrows + 1, dtype=np.int64)
    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize(dev)

    def timed(upd):
        """W warm-up steps, then K steps bracketed by barrier + CUDA events on the
        current stream (every update_block returns after its own streams finished)."""
        for w in range(pre + warm):
            upd(slice(w * S, (w + 1) * S))
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        l0 = prod.kernel_launches()
        with ClockSampler(local) as clk:
            e0.record()
            for k in range(pre + warm, pre + warm + steps):
                upd(slice(k * S, (k + 1) * S))
            e1.record()
            e1.synchronize()
        barrier()
        ms = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([ms], device=dev, dtype=torch.float64)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            ms = float(t.item())
        return ms, int(prod.kernel_launches() - l0), clk.summary()

    extra = {}
    if kind == "amm":
        g = torch.Generator(device=dev).manual_seed(1)
        W = torch.randn((cfg["latent"], cfg["dx"] + cfg["dy"]), generator=g, device=dev, dtype=torch.float64)
        z = torch.randn((nrows, cfg["latent"]), generator=g, device=dev, dtype=torch.float64)
        xy = z @ W + cfg["noise"] * torch.randn((nrows, cfg["dx"] + cfg["dy"]), generator=g, device=dev,
                                                dtype=torch.float64)
        x, y = xy[:, :cfg["dx"]].contiguous(), xy[:, cfg["dx"]:].contiguous()
        for t in (x, y):  # squared norms log-uniform on (1, R]
            u = torch.rand((nrows, 1), generator=g, device=dev, dtype=torch.float64)
            t.mul_(torch.sqrt(cfg["r_max"] ** u / (t * t).sum(1, keepdim=True)))
        x, y = x.cpu().pin_memory().numpy(), y.cpu().pin_memory().numpy()
        state = prod.CodState(cfg["dx"], cfg["dy"], cfg["eps"], cfg["eps"] * cfg["window"], cfg["window"],
                              seed=1, stream=1000, device=local)
        ms, launches, clocks = timed(lambda sl: state.update_block(x[sl], y[sl], ts_all[sl]))
        unit_rows = 1
        # the CodState API (amm.hpp:35-69) takes host rows: the only path is host -> device
        e2e = {"value": S * steps / (ms * 1e-3), "unit": "rows/s", "h2d_bytes_per_step": S * (cfg["dx"] + cfg["dy"]) * 8,
               "d2h_bytes_per_step": S * 64}
        extra["value_path"] = "host rows through the public API (CodState has no device-pointer entry point)"
    else:
        if kind == "sw":
            rows = torch.empty((nrows, cfg["d"]), dtype=torch.float64, device=dev)
            prod.gen_rows_device(rows, 1, cfg["d"], cfg["k"], cfg["rho"], cfg["noise"], cfg["r_max"], seed=1,
                                 stream=0, drift=cfg.get("drift", 0), device=local)
            torch.cuda.synchronize(dev)
            host = rows.cpu().pin_memory().numpy()
            def make():
                return prod.MlState(cfg["d"], cfg["window"], cfg["r_max"], cfg["eps"], seed=1, stream=1000,
                                    device=local)
            st1 = make()
            ms, launches, clocks = timed(lambda sl: st1.update_block(rows[sl], ts_all[sl]))
            del st1
            st2 = make()
            ms2, _, _ = timed(lambda sl: st2.update_block(host[sl], ts_all[sl]))
            del st2
            unit_rows = 1
        else:  # dist: m sites (fixed) spread over the ranks, j % world == rank
            from paper_2601_02019_b200.distributed import DistributedSketch, sites_of
            m = args.sites or cfg.get("sites", 8)
            mine = sites_of(rank, world, m)
            rows = {}
            for j in mine:  # site j = data stream j (bench.cpp:240-241)
                rows[j] = torch.empty((nrows, cfg["d"]), dtype=torch.float64, device=dev)
                prod.gen_rows_device(rows[j], 1, cfg["d"], cfg["k"], cfg["rho"], cfg["noise"], cfg["r_max"],
                                     seed=1, stream=j, k2=cfg.get("k2", 0), rho2=cfg.get("rho2", 0.9),
                                     scale2=cfg.get("scale2", 0.5), device=local)
            torch.cuda.synchronize(dev)
            host = {j: r.cpu().pin_memory().numpy() for j, r in rows.items()}

            def make():
                return DistributedSketch(cfg["d"], cfg["eps"], m, seed=1, rank=rank, world=world,
                                         group=group, device=local, use_nccl=world > 1)
            st1 = make()
            ms, launches, clocks = timed(lambda sl: st1.ingest({j: r[sl] for j, r in rows.items()}, sl.start + 1))
            # merged sketch over NCCL and its covariance error against the pooled
            # exact Gram of every row all sites ingested (outside the timed region,
            # like the reference's probes; acceptance.cpp:248-387)
            sk, _ = st1.probe()
            gram = torch.zeros((cfg["d"], cfg["d"]), dtype=torch.float64, device=dev)
            mass = torch.zeros((), dtype=torch.float64, device=dev)
            for r in rows.values():
                gram.addmm_(r.T, r)
                mass += (r * r).sum()
            if world > 1:
                torch.distributed.reduce(gram, 0)
                torch.distributed.reduce(mass, 0)
            if rank == 0:
                bt = torch.from_numpy(sk).to(dev)
                err = torch.linalg.eigvalsh(gram - bt.T @ bt).abs().max() / mass
                extra["merged_cov_err"] = float(err)
                extra["merged_cov_err_le_eps"] = bool(float(err) <= cfg["eps"])
                extra["merged_rows"] = m * nrows
            extra["comm_bytes_snapshots_rank0"] = st1.comm_bytes_local()
            extra["mass_protocol_bytes"] = st1.exchange.mass_bytes
            del st1
            st2 = make()
            ms2, _, _ = timed(lambda sl: st2.ingest({j: h[sl] for j, h in host.items()}, sl.start + 1))
            del st2
            unit_rows = m
        e2e = {"value": unit_rows * S * steps / (ms2 * 1e-3), "unit": "row-site updates/s" if kind == "dist" else "rows/s",
               "h2d_bytes_per_step": S * cfg["d"] * 8 * (len(rows) if kind == "dist" else 1), "d2h_bytes_per_step": 0}
    value = unit_rows * S * steps / (ms * 1e-3)
    if rank == 0:
        cpu = None
        if not args.no_cpu:
            rate, n_cpu = cpu_other_rate(cfg, args.cpu_rows or cfg["cpu_rows"], 1, sites=1)
            cpu = {"value": rate, "unit": "rows/s" if kind != "dist" else "row-site updates/s", "cores": 1,
                   "kind": "port", "sample": f"rows 1..{n_cpu} of {args.config.upper()} from an empty state"}
        print(json.dumps({
            "metric": "sketch update throughput", "value": value,
            "unit": "row-site updates/s" if kind == "dist" else "rows/s", "n_gpus": world, "steps": steps,
            "warmup": warm, "ms_per_step": ms / steps, "higher_is_better": True,
            "scaling": "strong" if kind == "dist" else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": cfg["name"], "rows_per_step": S, "timed_rows": f"{(pre + warm) * S + 1}..{nrows}",
                       "parallelism": (f"sites={unit_rows} over {world} GPU(s) ({unit_rows // world} per GPU), "
                                       f"ncclReduce merge") if kind == "dist" else "single"},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": clocks, **extra}), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.config is None:  # north_star: 1 GPU for the persistent configs, 1-8 for the distributed one
        args.config = "c4" if max(world, args.gpus) > 1 else "c2"
    cfg = CONFIGS[args.config]
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, cfg, rank)
        return
    if cfg["kind"] != "attp":
        run_other(args, cfg, world, rank, local)
        return
    import numpy as np
    import torch
    import paper_2601_02019_b200 as prod

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    S = args.rows_per_step or cfg["rows_per_step"]
    steps, warm = args.steps, args.warmup
    nrows = S * (steps + warm)
    d = cfg["d"]
    rows = torch.empty((nrows, d), dtype=torch.float64, device=dev)
    prod.gen_rows_device(rows, 1, d, cfg["k"], cfg["rho"], cfg["noise"], cfg["r_max"], seed=1 + rank,
                         stream=0, device=local)
    torch.cuda.synchronize(dev)
    ts_all = np.arange(1, nrows + 1, dtype=np.int64)

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize(dev)

    def run(sk, host_rows=None):
        for w in range(warm):
            sl = slice(w * S, (w + 1) * S)
            sk.update_block(rows[sl] if host_rows is None else host_rows[sl], ts_all[sl])
        sk.synchronize()
        sk.reset_profile()
        ext = torch.cuda.ExternalStream(sk.stream_handle(), device=dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        l0 = prod.kernel_launches()
        evs = []
        with ClockSampler(local) as clk:
            e0.record(ext)
            for k in range(warm, warm + steps):
                sl = slice(k * S, (k + 1) * S)
                evs.append(sk.update_block(rows[sl] if host_rows is None else host_rows[sl], ts_all[sl]))
            e1.record(ext)
            e1.synchronize()
        launches = prod.kernel_launches() - l0
        ms = e0.elapsed_time(e1)
        barrier()
        if world > 1:
            t = torch.tensor([ms], device=dev)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            ms = float(t.item())
        return ms, launches, clk.summary(), np.concatenate(evs)

    hr = args.rng == "host"
    sk = prod.AttpState(d, cfg["eps"], seed=1 + rank, stream=1000, device=local, host_rng=hr)
    ms, launches, clocks, ev = run(sk)
    info = sk.info()
    value = world * S * steps / (ms * 1e-3)
    del sk

    e2e = None
    if not args.no_e2e:
        host = rows.cpu().pin_memory().numpy()
        sk2 = prod.AttpState(d, cfg["eps"], seed=1 + rank, stream=1000, device=local, host_rng=hr)
        ms2, _, _, _ = run(sk2, host_rows=host)
        e2e = {"value": world * S * steps / (ms2 * 1e-3), "unit": "rows/s",
               "h2d_bytes_per_step": S * d * 8, "d2h_bytes_per_step": S * ev.dtype.itemsize}
        del sk2, host

    # roofline counters: a third, profiled pass over the same rows (per-launch
    # CUDA events around the product kernels slow the step, so `value` above
    # comes from the unprofiled pass)
    skp = prod.AttpState(d, cfg["eps"], seed=1 + rank, stream=1000, device=local, profile=True, host_rng=hr)
    ms_p, _, _, ev_p = run(skp)
    prof = skp.profile()
    del skp

    out = None
    if rank == 0:
        peak = fp64_peak_tflops(torch, dev)
        achieved = (prof["product_flops"] / max(prof["product_ms"], 1e-9)) / 1e9  # TFLOP/s
        # DRAM bytes per launch need an ncu capture of THIS launch; a bench run
        # cannot measure them, so the key is null here and the ncu --set full
        # numbers live under profiles/ 
        traffic = None
        i8 = info.ell * 2 >= 1024 and os.environ.get("AERO_PRODUCT_I8", "1") != "0"
        kern = ("k_iterate_i8 (persistent cooperative: every phase of a batch = G.X on the int8 tcgen05 tensor "
                "cores by 6-slice balanced-digit Ozaki splitting, TMEM accumulators, + per-job normalization; kernels.cu, "
                "ozaki.cuh); fp64-equivalent useful product flops (2 r^2 k per job per phase) over the whole kernel "
                "time, against the fp64 DGEMM peak the same products would have on the DMMA pipe") if i8 else (
                "k_iterate (persistent: split-K DMMA G.X products of every phase of a batch + per-job "
                "normalization, kernels.cu); useful product flops over the whole kernel time")
        # the same rate over committed rows only (what the verdict recomputes):
        # the kernel's counter also holds the speculative rows a dump discarded
        committed = committed_product_flops(ev_p, d) / max(prof["product_ms"], 1e-9) / 1e9
        roofline = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                    "frac": achieved / peak if peak > 0 else None, "traffic": traffic,
                    "achieved_committed_rows": committed,
                    "frac_committed_rows": committed / peak if peak > 0 else None,
                    "kernel": kern,
                    "peak_source": "measured in this run: cuBLAS DGEMM 8192^3 fp64 (not in MEASURED_PEAKS.json)",
                    "product_share_of_step": prof["product_ms"] / ms_p,
                    "flops_per_launch": prof["product_flops"] / max(1, prof["product_launches"]),
                    "ms_per_launch": prof["product_ms"] / max(1, prof["product_launches"])}
        if i8:  # the same kernel against the pipe it runs on: 21 int8 MMA slice pairs per fp64 product
            bf16 = None
            try:
                mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
                bf16 = mp.get("bf16_tflops")
            except Exception:
                pass
            i8_peak = 2.0 * bf16 if bf16 else 4500.0
            roofline["int8_pipe"] = {"achieved_tops": achieved * 21, "peak_tops": i8_peak,
                                     "frac": achieved * 21 / i8_peak,
                                     "peak_source": ("2 x measured dense bf16 (MEASURED_PEAKS.json)" if bf16
                                                     else "nominal B200 dense int8 4.5 POP/s")}
        f_row = reference_literal_flops(ev, d, info.ell)
        path = {"f_row_gflop": f_row / 1e9, "peak_tflops": peak, "bound_rows_per_s": peak * 1e12 / f_row,
                "frac": value / (peak * 1e12 / f_row),
                "basis": "SURVEY.md 8(d): reference-literal flops per row (gate (4kp+2)dr, simul_iter "
                         "(4q+4)drk+(8q+10)dk^2 per doubling call, SVD reduce, 8rd*xi dumps) from this run's "
                         "event log, at the measured fp64 DGEMM peak; the Gram-form engine executes fewer"}
        cpu = None
        if not args.no_cpu:
            threads = 1  # the reference is single-threaded (proj/CMakeLists.txt: no threads/OpenMP)
            t0 = time.perf_counter()
            rate, sample, _, _ = attp_cpu_sample(cfg, S, warm, steps, threads, points=cfg.get("cpu_points", 8),
                                                 per_point=1, device=local)
            cpu = {"value": rate, "unit": "rows/s", "cores": threads, "kind": "port", "same_config": True,
                   "sample": sample + f"; oracle restatement over OpenBLAS, 1 thread "
                                      f"({time.perf_counter() - t0:.0f} s incl. the GPU state replay)"}
        out = {
            "metric": "sketch update throughput", "value": value, "unit": "rows/s", "n_gpus": world,
            "steps": steps, "warmup": warm, "ms_per_step": ms / steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg["name"], "rows_per_step": S, "d": d, "eps": cfg["eps"],
                       "ell": info.ell, "timed_rows": f"{warm * S + 1}..{nrows}",
                       "l2": f"inputs larger than L2 ({S * d * 8 / 2**20:.0f} MiB per step)",
                       "parallelism": "replicas" if world > 1 else "single"},
            "roofline": roofline, "path_roofline": path, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clocks,
            "stats": {"gate_fire_rate": float(ev["gate_fired"].mean()), "dump_rate": float(ev["dumped"].mean()),
                      "reduces": int(ev["reduced"].sum()), "batches": int(info.device_batches),
                      "mispredicts": int(info.device_mispredicts), "snap_cols": int(info.snap_cols),
                      "batch_end": {"nofire": int(info.end_nofire), "fired": int(info.end_fired),
                                    "doubling": int(info.end_doubling), "dump": int(info.end_dump)},
                      "doubling_steps_hist": np.bincount(ev["doubling_steps"]).tolist(),
                      "xi_hist": np.bincount(ev["xi"]).tolist(),
                      "iterate_ms": prof["iterate_ms"], "reduce_ms": prof["reduce_ms"],
                      "product_ms": prof["product_ms"], "product_launches": int(prof["product_launches"])},
        }
        print(json.dumps(out), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
