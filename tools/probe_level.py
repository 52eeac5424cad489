"""One C3 level (AeroState d=1024, eps=1/64, fixed theta) block by block."""
import sys, time
import numpy as np
sys.path.insert(0, '/root/repo')
import torch
import paper_2601_02019_b200 as prod

d, eps = 1024, 1 / 64
theta = float(sys.argv[1]) if len(sys.argv) > 1 else 1024.0
S, nblk = int(sys.argv[2]) if len(sys.argv) > 2 else 64, int(sys.argv[3]) if len(sys.argv) > 3 else 16
rows = torch.empty((S * nblk, d), dtype=torch.float64, device='cuda')
prod.gen_rows_device(rows, 1, d, 64, 0.9, 0.1, 1024.0, seed=1, drift=131072)
torch.cuda.synchronize()
s = prod.AeroState(d, eps, theta, seed=1, stream=1000)
keys = ('rows', 'snaps', 'snap_cols', 'forks', 'device_batches', 'end_nofire', 'end_fired', 'end_doubling',
        'end_dump')
for b in range(nblk):
    t0 = time.perf_counter()
    ev = s.update_block(rows[b * S:(b + 1) * S], np.arange(b * S + 1, (b + 1) * S + 1))
    dt = time.perf_counter() - t0
    i = s.info()
    print(f'block {b}: {S / dt:.0f} rows/s', {k: getattr(i, k) for k in keys}, flush=True)
