#!/usr/bin/env python
"""Golden fixture for BASELINE config C2 (d=4096, eps=1/512, ell=1024) from the
CPU ORACLE (test infrastructure; oracle/): rows 1..N of the C2 stream
(seed 1, data stream 0; sketch RngState(1, 1000) as bench.cpp:148), through
AttpState (attp.hpp:21-26 -> sketch.cpp:82-141). N=4096 crosses the FD
reduces at rows 2048 and 3073.

Stored in tests/golden/c2_prefix.npz (consumed by
tests/test_gpu_parity.py::test_c2_default_path_matches_oracle_fixture):
  * events      -- the oracle's per-row event log (decisions, forks, sigma^2)
  * probe_t     -- checkpoints t at which the restored Gram was probed
  * probe       -- query_gram(0, t) @ W for W = 4 seeded Gaussian columns
                   (RngState(99, 0) draws), one d x 4 block per checkpoint
  * gram_fro    -- ||query_gram(0, t)||_F per checkpoint
  * err         -- cov-err ||A^T A - B^T B||_2 / ||A||_F^2 of query(N) (the
                   reference's acceptance criterion, acceptance.cpp:190-221)
  * mass        -- ||A||_F^2 accumulated by the oracle (attp.hpp:22)
  * snaps       -- (s, t, xi) of every snapshot

  python tools/make_c2_fixture.py [--n 4096] [--threads 8]
"""
import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import pyoracle as orc  # noqa: E402

D, EPS, K, RHO, NOISE, RMAX = 4096, 1 / 512, 256, 0.99, 0.05, 256.0
CHECKPOINTS = (1024, 2047, 2048, 3072, 3073)


def probe_matrix(d, cols=4):
    return orc.rng_draw(99, 0, 0, d * cols).reshape(d, cols)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--out", default=os.path.join(ROOT, "tests", "golden", "c2_prefix.npz"))
    a = ap.parse_args()
    orc.set_threads(a.threads)
    n = a.n
    rows = orc.gen_rows(D, K, RHO, NOISE, RMAX, 1, 0, 1, n)
    ts = np.arange(1, n + 1, dtype=np.int64)
    w = probe_matrix(D)
    s = orc.AttpState(D, EPS, 1, 1000)
    cps = sorted({c for c in CHECKPOINTS if c < n} | {n})
    evs, probes, fros = [], [], []
    pos, t0 = 0, time.time()
    for cp in cps:
        evs.append(s.update_block(rows[pos:cp], ts[pos:cp]))
        pos = cp
        g = s.inner.query_gram(0, cp)
        probes.append(g @ w)
        fros.append(np.linalg.norm(g))
        print(f"t={cp}: {time.time() - t0:.0f} s, rows={evs[-1]['rows_after'][-1]}, "
              f"snaps={s.inner.snap_count()}", flush=True)
    ev = np.concatenate(evs)
    b = s.query(n)
    gram = orc.OracleGram(D)
    gram.add_block(rows, ts)
    err = gram.error(b)
    snaps = np.array([(x["s"], x["t"], x["z"].shape[1]) for x in s.inner.snaps()], np.int64).reshape(-1, 3)
    np.savez_compressed(a.out, events=ev, probe_t=np.array(cps, np.int64), probe=np.stack(probes),
                        gram_fro=np.array(fros), err=np.float64(err), mass=np.float64(s.fro_mass),
                        snaps=snaps, n=np.int64(n))
    print(f"wrote {a.out}: n={n} err={err:.6g} (eps={EPS:.6g}) reduces={int(ev['reduced'].sum())} "
          f"dumps={int(ev['dumped'].sum())} in {time.time() - t0:.0f} s")


if __name__ == "__main__":
    main()
