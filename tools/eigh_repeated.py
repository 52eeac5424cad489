import sys, numpy as np
sys.path.insert(0, '/root/repo')
import paper_2601_02019_b200 as prod
rng = np.random.default_rng(0)
for n in (64, 200, 512):
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    lam = np.concatenate([np.full(n // 4, 5.0), np.full(n // 2, 3.0), np.linspace(1, 2, n - n // 4 - n // 2)])
    b = (q * lam) @ q.T
    w, v, t = prod.eigh(b, return_ms=True)
    print(n, 'recon', np.linalg.norm(v @ np.diag(w) @ v.T - b) / np.linalg.norm(b), 'orth', np.linalg.norm(v.T @ v - np.eye(n)), 'maxlamerr', np.abs(np.sort(w) - np.sort(lam)).max())
    # identity-like
    b = np.eye(n) * 2.0
    w, v, t = prod.eigh(b, return_ms=True)
    print(n, 'I: recon', np.linalg.norm(v @ np.diag(w) @ v.T - b) / np.linalg.norm(b), 'orth', np.linalg.norm(v.T @ v - np.eye(n)))
