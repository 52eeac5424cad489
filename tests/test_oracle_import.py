"""The oracle's state import (bench.py like-for-like CPU timing): a sketch
rebuilt from an exported live state (residual rows, fork counter, clock, last
dump time, threshold, running mass) continues EXACTLY like the original --
update() reads nothing else (sketch.cpp:82-141, attp.hpp:21-26)."""
import numpy as np


def test_attp_import_continues_identically(orc):
    d, eps, n0, n1 = 64, 1 / 8, 300, 200
    rows = orc.gen_rows(d, 8, 0.9, 0.1, 64.0, 1, 0, 1, n0 + n1)
    ts = np.arange(1, n0 + n1 + 1)
    a = orc.AttpState(d, eps, 1, 1000)
    a.update_block(rows[:n0], ts[:n0])
    inner = a.inner
    b = orc.AttpState(d, eps, 1, 1000)
    b.import_state(inner.residual(), inner.forks, inner.clock, inner.last_dump_time, inner.theta, a.fro_mass)
    ea = a.update_block(rows[n0:], ts[n0:])
    eb = b.update_block(rows[n0:], ts[n0:])
    assert ea.tobytes() == eb.tobytes()
    assert np.array_equal(a.inner.residual(), b.inner.residual())
    assert ea["reduced"].sum() >= 1 and ea["dumped"].sum() >= 1
