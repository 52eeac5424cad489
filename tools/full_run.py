#!/usr/bin/env python
"""Covariance error at BASELINE size (north star: "covariance error <= eps on
all five configs"). Streams each config's FULL n through the product path on
one B200 and probes it against an exact fp64 Gram computed beside it on the
GPU (the checker, K9 of SURVEY.md 2.1: torch fp64 SYRK accumulation over the
same device-generated rows -- measurement, not the product). The error
criteria are the reference's own (acceptance.cpp:152-387):

  C1/C2 ATTP   ||A_t^T A_t - B_t^T B_t||_2 / ||A_t||_F^2, B_t = query(t)
  C3 SW        ||A_W^T A_W - B^T B||_2 / ||A_W||_F^2 every 4096 rows, W = last N
  C4 dist      merged probe vs the pooled Gram of all sites' rows
  C5 AMM       ||X_W^T Y_W - A* B*^T||_2 / (||X_W||_F ||Y_W||_F) per probe

  python tools/full_run.py --config c2 [--n N] [--probe P] [--out profiles/round2_full_c2.json]
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402  (CONFIGS)
import paper_2601_02019_b200 as prod  # noqa: E402

DEV = torch.device("cuda", 0)


def spec_sym(m):
    return float(torch.linalg.eigvalsh(m).abs().max())


def gen(cfg, t0, n, stream=0):
    rows = torch.empty((n, cfg["d"]), dtype=torch.float64, device=DEV)
    prod.gen_rows_device(rows, t0, cfg["d"], cfg["k"], cfg["rho"], cfg["noise"], cfg["r_max"], seed=1,
                         stream=stream, drift=cfg.get("drift", 0), k2=cfg.get("k2", 0),
                         rho2=cfg.get("rho2", 0.9), scale2=cfg.get("scale2", 0.5))
    torch.cuda.synchronize(DEV)
    return rows


def run_attp(cfg, n, probe, chunk):
    d = cfg["d"]
    s = prod.AttpState(d, cfg["eps"], seed=1, stream=1000)
    g = torch.zeros((d, d), dtype=torch.float64, device=DEV)
    mass, out, t_upd = 0.0, [], 0.0
    for t0 in range(0, n, chunk):
        m = min(chunk, n - t0)
        rows = gen(cfg, t0 + 1, m)
        ts = np.arange(t0 + 1, t0 + m + 1, dtype=np.int64)
        a = time.perf_counter()
        s.update_block(rows, ts)
        s.synchronize()
        t_upd += time.perf_counter() - a
        g.addmm_(rows.T, rows)
        mass += float((rows * rows).sum())
        t = t0 + m
        if t % probe == 0 or t == n:
            q0 = time.perf_counter()
            b = torch.from_numpy(s.query(t)).to(DEV)
            q_ms = (time.perf_counter() - q0) * 1e3
            err = spec_sym(g - b.T @ b) / mass
            out.append({"t": t, "err": err, "query_ms": q_ms, "snaps": int(s.info().snaps)})
            print(f"t={t} err={err:.5g} ({t / t_upd:.0f} rows/s) query {q_ms:.0f} ms", flush=True)
    inf = s.info()
    return out, {"rows_per_s_update": n / t_upd, "snap_cols": int(inf.snap_cols), "snaps": int(inf.snaps)}


def run_sw(cfg, n, probe, chunk):
    d, N = cfg["d"], cfg["window"]
    assert N % probe == 0 and chunk == probe
    s = prod.MlState(d, N, cfg["r_max"], cfg["eps"], seed=1, stream=1000)
    blocks, out, t_upd = [], [], 0.0
    for t0 in range(0, n, chunk):
        rows = gen(cfg, t0 + 1, chunk)
        ts = np.arange(t0 + 1, t0 + chunk + 1, dtype=np.int64)
        a = time.perf_counter()
        s.update_block(rows, ts)
        torch.cuda.synchronize(DEV)
        t_upd += time.perf_counter() - a
        blocks.append((rows.T @ rows, float((rows * rows).sum())))
        blocks = blocks[-(N // chunk):]
        t = t0 + chunk
        gw = sum(x[0] for x in blocks)
        mw = sum(x[1] for x in blocks)
        q = s.query()
        b = torch.from_numpy(q["sketch"]).to(DEV)
        err = spec_sym(gw - b.T @ b) / mw
        out.append({"t": t, "err": err, "level": q["level"], "fallback": bool(q["fallback"])})
        if (t // chunk) % 16 == 0:
            print(f"t={t} err={err:.5g} level={q['level']} ({t / t_upd:.0f} rows/s)", flush=True)
    return out, {"rows_per_s_update": n / t_upd}


def run_dist(cfg, n, probe, chunk, m):
    from paper_2601_02019_b200.distributed import DistributedSketch
    d = cfg["d"]
    ds = DistributedSketch(d, cfg["eps"], m, seed=1)
    g = torch.zeros((d, d), dtype=torch.float64, device=DEV)
    mass, out, t_upd = 0.0, [], 0.0
    for t0 in range(0, n, chunk):
        c = min(chunk, n - t0)
        blk = {j: gen(cfg, t0 + 1, c, stream=j) for j in range(m)}
        a = time.perf_counter()
        ds.ingest(blk, t0 + 1)
        torch.cuda.synchronize(DEV)
        t_upd += time.perf_counter() - a
        for rows in blk.values():
            g.addmm_(rows.T, rows)
            mass += float((rows * rows).sum())
        t = t0 + c
        if t % probe == 0 or t == n:
            sk, _ = ds.probe()
            b = torch.from_numpy(sk).to(DEV)
            err = spec_sym(g - b.T @ b) / mass
            out.append({"t": t, "err": err})
            print(f"t={t} err={err:.5g} ({m * t / t_upd:.0f} row-site/s)", flush=True)
    return out, {"row_site_per_s_update": m * n / t_upd, "comm_bytes": ds.exchange.mass_bytes + ds.snapshot_bytes}


def amm_rows(cfg, t0, n, gen_state):
    """C5 generator (DESIGN.md GENERATOR spec): x = z W_x + 0.1 g, y = z W_y + 0.1 h,
    squared norms of x and y independently log-uniform on (1, R]; seeded torch
    draws on the device (block t0 uses its own seed so blocks are independent of
    the chunking)."""
    wx, wy = gen_state
    gg = torch.Generator(device=DEV).manual_seed(1_000_003 * (t0 + 1))
    z = torch.randn((n, cfg["latent"]), generator=gg, device=DEV, dtype=torch.float64)
    x = z @ wx + cfg["noise"] * torch.randn((n, cfg["dx"]), generator=gg, device=DEV, dtype=torch.float64)
    y = z @ wy + cfg["noise"] * torch.randn((n, cfg["dy"]), generator=gg, device=DEV, dtype=torch.float64)
    for v in (x, y):
        u = torch.rand((n, 1), generator=gg, device=DEV, dtype=torch.float64)
        v.mul_(torch.sqrt(cfg["r_max"] ** u / (v * v).sum(1, keepdim=True)))
    return x, y


def run_amm(cfg, n, probe, chunk):
    N = cfg["window"]
    assert N % chunk == 0 and probe % chunk == 0
    g0 = torch.Generator(device=DEV).manual_seed(1)
    wx = torch.randn((cfg["latent"], cfg["dx"]), generator=g0, device=DEV, dtype=torch.float64)
    wy = torch.randn((cfg["latent"], cfg["dy"]), generator=g0, device=DEV, dtype=torch.float64)
    s = prod.CodState(cfg["dx"], cfg["dy"], cfg["eps"], cfg["eps"] * N, N, seed=1, stream=1000)
    blocks, out, t_upd = [], [], 0.0
    for t0 in range(0, n, chunk):
        x, y = amm_rows(cfg, t0, chunk, (wx, wy))
        xh, yh = x.cpu().numpy(), y.cpu().numpy()
        ts = np.arange(t0 + 1, t0 + chunk + 1, dtype=np.int64)
        a = time.perf_counter()
        s.update_block(xh, yh, ts)
        t_upd += time.perf_counter() - a
        blocks.append((x.T @ y, float((x * x).sum()), float((y * y).sum())))
        blocks = blocks[-(N // chunk):]
        t = t0 + chunk
        if t % probe == 0 or t == n:
            p = sum(b[0] for b in blocks)
            den = (sum(b[1] for b in blocks) * sum(b[2] for b in blocks)) ** 0.5
            a_, b_ = s.query()
            diff = p - torch.from_numpy(a_).to(DEV) @ torch.from_numpy(b_).to(DEV).T
            err = float(torch.linalg.matrix_norm(diff, ord=2)) / den
            out.append({"t": t, "err": err})
            print(f"t={t} err={err:.5g} ({t / t_upd:.0f} rows/s)", flush=True)
    return out, {"rows_per_s_update": n / t_upd}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", required=True, choices=sorted(bench.CONFIGS))
    ap.add_argument("--n", type=int, default=0)
    ap.add_argument("--probe", type=int, default=0)
    ap.add_argument("--sites", type=int, default=8)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    cfg = bench.CONFIGS[a.config]
    n = a.n or cfg["n"]
    t0 = time.time()
    kind = cfg["kind"]
    if kind == "attp":
        probes, extra = run_attp(cfg, n, a.probe or n // 8, 65536 if cfg["d"] <= 1024 else 16384)
    elif kind == "sw":
        probes, extra = run_sw(cfg, n, 4096, 4096)
    elif kind == "dist":
        probes, extra = run_dist(cfg, n, a.probe or n // 4, 8192, a.sites)
    else:
        probes, extra = run_amm(cfg, n, a.probe or 16384, 4096)
    errs = np.array([p["err"] for p in probes])
    res = {"config": a.config, "workload": cfg["name"], "n": n, "eps": cfg["eps"],
           "probes": len(probes), "max_err": float(errs.max()), "final_err": float(errs[-1]),
           "mean_err": float(errs.mean()), "all_le_eps": bool((errs <= cfg["eps"]).all()),
           "frac_probes_le_eps": float((errs <= cfg["eps"]).mean()),
           "wall_s": time.time() - t0, **extra,
           "checker": "exact fp64 Gram on the GPU (torch SYRK over the same device-generated rows)",
           "probe_list": probes}
    if kind == "dist":
        res["sites"] = a.sites
    out = a.out or os.path.join(ROOT, "gpurun_out", f"full_{a.config}.json")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps({k: v for k, v in res.items() if k != "probe_list"}))


if __name__ == "__main__":
    main()
