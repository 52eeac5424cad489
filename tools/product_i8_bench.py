"""Time the iteration product Y = G X: int8 tensor cores (ozaki.cu) vs fp64
DMMA (product.cu) at the C2 iterate shapes (r = buffer rows, n = job columns)."""
import sys
import numpy as np
sys.path.insert(0, '/root/repo')
import paper_2601_02019_b200 as prod
rng = np.random.default_rng(0)
for r, n in [(1100, 96), (1500, 128), (1500, 192), (2000, 128), (2047, 192), (512, 128), (256, 64)]:
    a = rng.standard_normal((r, r // 2)); g = a @ a.T
    x = rng.standard_normal((r, n))
    y0, t0 = prod.dev_product(g, x, None, mode=0, return_ms=True)
    y1, t1 = prod.dev_product(g, x, None, mode=1, return_ms=True)
    fl = 2.0 * r * r * n
    rel = np.max(np.abs(y0 - y1)) / np.max(np.abs(y1))
    print(f"r={r:5d} n={n:4d}  int8-tc {t0*1e3:8.1f} us ({fl/t0/1e9:6.1f} TF/s fp64-equiv)   "
          f"dmma {t1*1e3:8.1f} us ({fl/t1/1e9:6.1f} TF/s)   max rel diff {rel:.1e}", flush=True)
