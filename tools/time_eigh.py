"""Time the device eigensolver (aero_eigh test hook) across n; realistic FD Gram at 2048."""
import sys, numpy as np
sys.path.insert(0, '/root/repo')
import torch
import paper_2601_02019_b200 as prod
rng = np.random.default_rng(0)
for n in [int(x) for x in (sys.argv[1:] or (64, 96, 128, 256, 512, 1024, 2048))]:
    a = rng.standard_normal((n + 5, n)); b = a.T @ a
    ms = []
    for _ in range(3 if n >= 1024 else 5):
        w, v, t = prod.eigh(b, return_ms=True); ms.append(t)
    err = np.linalg.norm(v @ np.diag(w) @ v.T - b) / np.linalg.norm(b)
    orth = np.linalg.norm(v.T @ v - np.eye(n))
    print(f"n={n:5d} eigh device ms min {min(ms):9.3f}  recon {err:.1e} orth {orth:.1e}", flush=True)
