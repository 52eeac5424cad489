"""Time the device eigensolver on FD-reduce-shaped Grams: n x n Gram of n rows
that are rank-k signal plus noise (a long cluster of noise-floor eigenvalues,
as in the C3 / C5 buffers). Dev tool."""
import sys

import numpy as np

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import paper_2601_02019_b200 as prod  # noqa: E402

rng = np.random.default_rng(0)
for n, k, d in ((256, 64, 1024), (256, 48, 1024), (512, 128, 2048), (2048, 256, 4096)):
    u = np.linalg.qr(rng.standard_normal((d, k)))[0].T
    a = (rng.standard_normal((n, k)) * 0.9 ** np.arange(k)) @ u + 0.1 * rng.standard_normal((n, d))
    g = a @ a.T
    ms = []
    for _ in range(5):
        w, v, t = prod.eigh(g, return_ms=True)
        ms.append(t)
    err = np.linalg.norm(v @ np.diag(w) @ v.T - g) / np.linalg.norm(g)
    orth = np.linalg.norm(v.T @ v - np.eye(n))
    print(f"n={n} rank={k}+noise: eigh {min(ms):.3f} ms  recon {err:.1e} orth {orth:.1e}", flush=True)
