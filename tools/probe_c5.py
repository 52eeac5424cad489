"""Time CodState (C5 config) block by block on the GPU with event stats."""
import sys, time
import numpy as np
sys.path.insert(0, '/root/repo')
import torch
import paper_2601_02019_b200 as prod

dx, dy, N, eps = 1024, 768, 65536, 1 / 64
S = int(sys.argv[1]) if len(sys.argv) > 1 else 256
nblk = int(sys.argv[2]) if len(sys.argv) > 2 else 4
g = torch.Generator().manual_seed(1)
n = S * nblk
W = torch.randn((48, dx + dy), generator=g, dtype=torch.float64)
xy = torch.randn((n, 48), generator=g, dtype=torch.float64) @ W + 0.1 * torch.randn((n, dx + dy), generator=g, dtype=torch.float64)
x, y = xy[:, :dx].contiguous(), xy[:, dx:].contiguous()
for t in (x, y):
    u = torch.rand((n, 1), generator=g, dtype=torch.float64)
    t.mul_(torch.sqrt(64.0 ** u / (t * t).sum(1, keepdim=True)))
x, y = x.numpy(), y.numpy()
s = prod.CodState(dx, dy, eps, eps * N, N, seed=1, stream=1000)
for b in range(nblk):
    sl = slice(b * S, (b + 1) * S)
    t0 = time.perf_counter()
    ev = s.update_block(x[sl], y[sl], np.arange(b * S + 1, (b + 1) * S + 1))
    dt = time.perf_counter() - t0
    print(f'block {b}: {S / dt:.0f} rows/s; fired {ev["gate_fired"].sum()} dumped {ev["dumped"].sum()} '
          f'reduced {ev["reduced"].sum()} doubling {np.bincount(ev["doubling_steps"])} xi {np.bincount(ev["xi"])}', flush=True)
print(s.info())
