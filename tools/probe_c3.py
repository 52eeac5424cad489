"""Time MlState (C3 config) block by block on the GPU with per-level batch stats."""
import sys, time
import numpy as np
sys.path.insert(0, '/root/repo')
import torch
import paper_2601_02019_b200 as prod

d, N, R, eps = 1024, 65536, 1024.0, 1 / 64
S = int(sys.argv[1]) if len(sys.argv) > 1 else 512
nblk = int(sys.argv[2]) if len(sys.argv) > 2 else 8
rows = torch.empty((S * nblk, d), dtype=torch.float64, device='cuda')
prod.gen_rows_device(rows, 1, d, 64, 0.9, 0.1, R, seed=1, drift=131072)
torch.cuda.synchronize()
s = prod.MlState(d, N, R, eps, seed=1, stream=1000)
L = s.info().levels
for b in range(nblk):
    ts = np.arange(b * S + 1, (b + 1) * S + 1)
    t0 = time.perf_counter()
    s.update_block(rows[b * S:(b + 1) * S], ts)
    dt = time.perf_counter() - t0
    print(f'block {b}: {S / dt:.0f} rows/s ({dt * 1e3:.0f} ms)', flush=True)
for j in range(L):
    i = s.level_state(j).info()
    print(j, 'theta', s.theta(j), 'heavy', s.heavy_count(j), {k: getattr(i, k) for k in
          ('snaps', 'snap_cols', 'device_batches', 'device_rows_processed', 'end_nofire', 'end_fired',
           'end_doubling', 'end_dump', 'forks')}, flush=True)
