#!/usr/bin/env python
"""Run-to-run variance of the C2 step inside one process: R fresh AttpStates
over the same device rows (warm-up W steps, then K timed steps each), CUDA
events on the sketch stream; prints ms per pass. Dev tool."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import bench  # noqa: E402
import paper_2601_02019_b200 as prod  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
R = int(sys.argv[2]) if len(sys.argv) > 2 else 3
S, W, K = cfg["rows_per_step"], 3, 5
n = S * (W + K)
rows = torch.empty((n, cfg["d"]), dtype=torch.float64, device="cuda")
prod.gen_rows_device(rows, 1, cfg["d"], cfg["k"], cfg["rho"], cfg["noise"], cfg["r_max"], seed=1)
ts = np.arange(1, n + 1, dtype=np.int64)
for rep in range(R):
    sk = prod.AttpState(cfg["d"], cfg["eps"], seed=1, stream=1000,
                        max_batch=int(__import__("os").environ.get("MAXB", "0")))
    for w in range(W):
        sk.update_block(rows[w * S:(w + 1) * S], ts[w * S:(w + 1) * S])
    sk.synchronize()
    ext = torch.cuda.ExternalStream(sk.stream_handle())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    e0.record(ext)
    per = []
    for k in range(W, W + K):
        a = time.perf_counter()
        sk.update_block(rows[k * S:(k + 1) * S], ts[k * S:(k + 1) * S])
        per.append((time.perf_counter() - a) * 1e3)
    e1.record(ext)
    e1.synchronize()
    print(f"pass {rep}: {e0.elapsed_time(e1):.1f} ms device-clock, {1e3 * (time.perf_counter() - w0):.1f} ms wall, "
          f"per step {' '.join(f'{x:.0f}' for x in per)}", flush=True)
    del sk
