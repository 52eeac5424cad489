import sys, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import torch
import paper_2601_02019_b200 as prod
from oracle import pyoracle as orc
from refutil import uniform_rows
orc.set_threads(1)
d, n_win, eps, T = 32, 500, 0.2, 300
ref = orc.MlState(d, n_win, 32.0, eps, 0, 1000)
s = prod.MlState(d, n_win, 32.0, eps, seed=0, stream=1000)
rows = uniform_rows(orc, T, d, 0, 0)
for b in range(0, 200, 100):
    blk, ts = rows[b:b + 100], np.arange(b + 1, b + 101)
    ref.update_block(blk, ts); s.update_block(blk, ts)
    q, qr = s.query(), ref.query()
    print('block', b, 'level', q['level'], qr['level'])
    j = q['level']
    lv, lr = s.level_state(j), ref.level_state(j)
    print(' clock', lv.clock, lr.clock, 'rows', lv.residual().shape, lr.residual().shape)
    print(' resid diff', np.abs(lv.residual() - lr.residual()).max())
    g1, g2 = lv.query_gram(0, lv.clock), lr.query_gram(0, lr.clock)
    print(' level gram rel', np.linalg.norm(g1 - g2) / np.linalg.norm(g2))
    b1, b2 = lv.query(0, lv.clock), lr.query(0, lr.clock)
    print(' level query gram rel', np.linalg.norm(b1.T @ b1 - b2.T @ b2) / np.linalg.norm(b2.T @ b2))
    sk, skr = q['sketch'], qr['sketch']
    print(' final rel', np.linalg.norm(sk.T @ sk - skr.T @ skr) / np.linalg.norm(skr.T @ skr))
    # shrink check: state with huge theta, rows given -> query = shrink(C^T C)
    a = prod.AeroState(d, eps, 1e30); ao = orc.AeroState(d, eps, 1e30, 0, 0)
    a.update_block(rows[:15], np.arange(1, 16)); ao.update_block(rows[:15], np.arange(1, 16))
    x1, x2 = a.query(0, 15), ao.query(0, 15)
    print(' shrink check rel', np.linalg.norm(x1.T @ x1 - x2.T @ x2) / np.linalg.norm(x2.T @ x2))
    print(' eig gpu', np.round(np.linalg.norm(x1, axis=1), 4)[:6], 'ref', np.round(np.linalg.norm(x2, axis=1), 4)[:6])
