#!/usr/bin/env python
"""Golden fixture for the scaled C3 indexing-parity variant:
MlState (sliding_window.cpp:15-156) with d=1024, eps=1/64, R=1024 as BASELINE
C3, but window N=4096 over n=32768 rows (the C3 generator, k=64, basis
re-drawn every 2N = 8192 rows like C3's 131072 = 2N), run to completion by
the CPU ORACLE (test infrastructure; oracle/).

Stored in tests/golden/c3_scaled.npz, one probe every 1024 rows:
  * meta  -- int64 rows (probe, level, kind, s, t, xi): kind 0 = snapshot of
             the level's queue (s, t, xi), kind 1 = heavy row (s, t, 0)
  * query -- per probe (level, fallback, xi_sum, heavy_used)
  * err   -- per probe ||A_W^T A_W - B^T B||_2 / ||A_W||_F^2 of the oracle's
             query against the exact window Gram (OracleGram, oracle.hpp:22-76)
  * mass  -- per probe window mass (sliding_window.cpp ring)

  python tools/make_c3_fixture.py
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import pyoracle as orc  # noqa: E402

D, EPS, R, N, NROWS, DRIFT, PROBE = 1024, 1 / 64, 1024.0, 4096, 32768, 8192, 1024


def main():
    orc.set_threads(int(os.environ.get("THREADS", "1")))
    rows = orc.gen_rows(D, 64, 0.9, 0.1, R, 1, 0, 1, NROWS, drift=DRIFT)
    ts = np.arange(1, NROWS + 1, dtype=np.int64)
    s = orc.MlState(D, N, R, EPS, 1, 1000)
    g = orc.OracleGram(D, N)
    meta, query, err, mass = [], [], [], []
    t0 = time.time()
    for p, b in enumerate(range(0, NROWS, PROBE)):
        s.update_block(rows[b:b + PROBE], ts[b:b + PROBE])
        g.add_block(rows[b:b + PROBE], ts[b:b + PROBE])
        inf = s.info()
        for j in range(inf["levels"]):
            for x in s.level_state(j).snaps():
                meta.append((p, j, 0, x["s"], x["t"], x["z"].shape[1]))
            for h in s.heavy(j):
                meta.append((p, j, 1, h["s"], h["t"], 0))
        q = s.query()
        query.append((q["level"], int(q["fallback"]), q["xi_sum"], q["heavy_used"]))
        err.append(g.error(q["sketch"]))
        mass.append(inf["window_mass"])
        print(f"t={b + PROBE}: {time.time() - t0:.0f} s level={q['level']} err={err[-1]:.4g}", flush=True)
    out = os.path.join(ROOT, "tests", "golden", "c3_scaled.npz")
    np.savez_compressed(out, meta=np.array(meta, np.int64), query=np.array(query, np.int64),
                        err=np.array(err), mass=np.array(mass),
                        params=np.array([D, N, NROWS, DRIFT, PROBE], np.int64))
    print(f"wrote {out}: {len(meta)} meta rows, max err {max(err):.4g} (eps {EPS:.4g})")


if __name__ == "__main__":
    main()
