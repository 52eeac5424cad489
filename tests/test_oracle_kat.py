"""Known-answer and property tests of the CPU oracle, ported from the
reference's own doctest suites (proj/tests/test_linalg.cpp, test_fd.cpp,
test_sketch.cpp, test_attp.cpp, test_sliding_window.cpp, test_distributed.cpp,
test_amm.cpp). Each test cites the reference test it restates."""
import math

import numpy as np
import pytest

from refutil import gaussian, gaussian_vec, orthonormal, rel_fro, uniform_rows


# ---------------------------------------------------------------- linalg
def test_svd_diagonal(orc):  # test_linalg.cpp:28-33
    u, s, vt = orc.svd(np.diag([4.0, 3, 2, 1]))
    assert np.allclose(s, [4, 3, 2, 1], rtol=1e-12)
    assert np.linalg.norm(u - np.eye(4)) < 1e-12 and np.linalg.norm(vt - np.eye(4)) < 1e-12


def test_svd_zero_and_reconstruction(orc):  # test_linalg.cpp:35-51
    _, s, _ = orc.svd(np.zeros((3, 2)))
    assert s.size == 2 and np.linalg.norm(s) == 0.0
    a = gaussian(orc, 8, 5, 7)
    u, s, vt = orc.svd(a)
    assert rel_fro(u @ np.diag(s) @ vt, a) < 1e-10
    assert np.all(np.diff(s) <= 0) and s[-1] >= 0


def test_svd_rejects_nonfinite(orc):  # test_linalg.cpp:53-57
    a = np.zeros((2, 2))
    a[0, 0] = np.nan
    with pytest.raises(orc.InvalidInput):
        orc.svd(a)


def test_eigh_kats(orc):  # test_linalg.cpp:59-82
    lam, v = orc.eigh(np.diag([2.0, -1.0]))
    assert np.allclose(lam, [2, -1]) and np.linalg.norm(v - np.eye(2)) < 1e-12
    lam, _ = orc.eigh(np.eye(4))
    assert np.allclose(lam, 1.0)
    with pytest.raises(orc.InvalidInput):
        orc.eigh(np.zeros((3, 2)))
    c = gaussian(orc, 6, 3, 11)
    lam, _ = orc.eigh(c.T @ c)
    s = orc.svd(c)[1]
    assert np.max(np.abs(lam[:3] - s ** 2)) < 1e-9


def test_qr_kats(orc):  # test_linalg.cpp:84-111
    q, r = orc.qr(np.eye(3))
    assert np.linalg.norm(q - np.eye(3)) < 1e-12 and np.linalg.norm(r - np.eye(3)) < 1e-12
    a = np.zeros((3, 2))
    a[0, 0], a[1, 0] = 3.0, 4.0
    q, r = orc.qr(a)
    assert abs(r[0, 0] - 5.0) < 1e-12 and np.all(np.diag(r) >= 0)
    a = gaussian(orc, 10, 4, 3)
    q, r = orc.qr(a)
    assert np.linalg.norm(q.T @ q - np.eye(4)) < 1e-10 and rel_fro(q @ r, a) < 1e-10
    assert np.all(np.tril(r, -1) == 0)
    with pytest.raises(orc.InvalidInput):
        orc.qr(np.zeros((2, 3)))


def test_factorizations_random_shapes(orc):  # test_linalg.cpp:113-132
    for seed in range(50):
        u = orc.rng_draw(seed, 99, 0, 2, "uniform")
        rows = 2 + int(u[0] * 62)
        cols = 1 + int(u[1] * rows)
        a = gaussian(orc, rows, cols, seed, 1)
        uu, s, vt = orc.svd(a)
        assert rel_fro(uu @ np.diag(s) @ vt, a) < 1e-10
        q, r = orc.qr(a)
        assert rel_fro(q @ r, a) < 1e-10
        g = a.T @ a
        lam, v = orc.eigh(g)
        assert rel_fro(v @ np.diag(lam) @ v.T, g) < 1e-10


def test_power_iteration_kats(orc):  # test_linalg.cpp:134-164
    a = np.zeros((2, 2))
    a[0, 0] = 2.0
    for seed in range(5):
        s2, v = orc.power_iteration(a, 1, seed, 0)
        assert abs(s2 - 4.0) < 1e-12 and abs(np.linalg.norm(v) - 1) < 1e-12
    s2, _ = orc.power_iteration(np.eye(6), 3, 1, 2)
    assert abs(s2 - 1.0) < 1e-12
    with pytest.raises(orc.InvalidInput):
        orc.power_iteration(np.eye(2), 0, 0, 0)
    s2, v = orc.power_iteration(np.zeros((3, 3)), 2, 0, 0)
    assert s2 == 0.0 and v[0] == 1.0 and np.linalg.norm(v[1:]) == 0.0
    a = gaussian(orc, 12, 8, 5)
    r1, r2 = orc.power_iteration(a, 4, 42, 7), orc.power_iteration(a, 4, 42, 7)
    assert r1[0] == r2[0] and np.array_equal(r1[1], r2[1])


def test_simul_iter_kats(orc):  # test_linalg.cpp:166-192
    z, sh = orc.simul_iter(np.diag([3.0, 2, 1]), 2, 0.4, 3, 0)
    assert abs(sh[0] ** 2 - 9) <= 0.4 and abs(sh[1] ** 2 - 4) <= 0.4
    assert np.linalg.norm(z.T @ z - np.eye(2)) < 1e-8 and sh[0] >= sh[1]
    z, sh = orc.simul_iter(np.zeros((5, 5)), 3, 0.4, 0, 0)
    assert np.array_equal(z, np.eye(5)[:, :3]) and np.linalg.norm(sh) == 0
    for k, e in ((0, 0.4), (4, 0.4), (2, 0.0)):
        with pytest.raises(orc.InvalidInput):
            orc.simul_iter(np.eye(3), k, e, 0, 0)


def test_spectral_norms(orc):  # test_linalg.cpp:194-199
    a = gaussian(orc, 10, 6, 13)
    s1 = orc.svd(a)[1][0]
    assert abs(orc.spectral_norm(a) - s1) < 1e-10 * s1
    assert abs(orc.spectral_norm_sym(a.T @ a) - s1 * s1) < 1e-10 * s1 * s1


def test_power_iteration_half_bound(orc):  # acceptance.cpp:115-124 (check 3)
    good = 0
    for seed in range(200):
        a = gaussian(orc, 64, 32, seed, 31)
        s1 = orc.svd(a)[1][0]
        s2, _ = orc.power_iteration(a, 7, seed, 32)
        good += s2 >= 0.5 * s1 * s1
    assert good >= 190


# ---------------------------------------------------------------- fd
def test_fd_reduce_kats(orc):  # test_fd.cpp:19-44
    out = orc.fd_reduce(np.diag([4.0, 3, 2, 1]), 2)
    s = orc.svd(out)[1]
    assert abs(s[0] - math.sqrt(7.0)) < 1e-12 and np.all(s[1:] < 1e-12) and out.shape[0] == 4
    assert np.linalg.norm(orc.fd_reduce(np.zeros((4, 6)), 2)) == 0.0
    with pytest.raises(orc.InvalidInput):
        orc.fd_reduce(np.zeros((5, 6)), 2)
    b = gaussian(orc, 8, 12, 17)
    out = orc.fd_reduce(b, 4)
    gap = orc.spectral_norm_sym(b.T @ b - out.T @ out)
    assert abs(gap - orc.svd(b)[1][3] ** 2) < 1e-9


def test_cod_reduce_kats(orc):  # test_fd.cpp:91-130
    a = np.diag([2.0, math.sqrt(3), math.sqrt(2), 1.0])
    ap, bp = orc.cod_reduce(a, a, 2)
    s = orc.svd(ap @ bp.T)[1]
    assert abs(s[0] - 1.0) < 1e-9 and np.all(s[1:] < 1e-9)
    ap, bp = orc.cod_reduce(np.zeros((3, 4)), gaussian(orc, 5, 4, 2), 2)
    assert np.linalg.norm(ap) == 0 and np.linalg.norm(bp) == 0
    with pytest.raises(orc.InvalidInput):
        orc.cod_reduce(np.zeros((3, 4)), np.zeros((3, 5)), 2)
    a, b = gaussian(orc, 7, 6, 21), gaussian(orc, 5, 6, 22)
    ap, bp = orc.cod_reduce(a, b, 3)
    p = a @ b.T
    assert abs(orc.spectral_norm(p - ap @ bp.T) - orc.svd(p)[1][2]) < 1e-9
    a, b = gaussian(orc, 6, 6, 31), gaussian(orc, 8, 6, 32)
    ap, bp = orc.cod_reduce(a, b, 3)
    sig = orc.svd(a @ b.T)[1]
    expect = np.maximum(sig - sig[2], 0).sum()
    assert abs(orc.svd(ap @ bp.T)[1].sum() - expect) < 1e-9 * max(1, expect)


# ---------------------------------------------------------------- sketch
def test_sketch_construction(orc):  # test_sketch.cpp:19-33
    assert orc.AeroState(4, 0.1, 0.0, 0, 0).ell == 20
    assert orc.AeroState(4, 1.0, 0.0, 0, 0).ell == 2
    assert orc.AeroState(300, 0.05, 0.0, 0, 0).ell == 40
    for args in ((4, 0.0, 0.0), (4, 1.5, 0.0), (4, 0.5, -1.0), (0, 0.5, 0.0)):
        with pytest.raises(orc.InvalidInput):
            orc.AeroState(*args, 0, 0)


def test_dominant_row_dumped(orc):  # test_sketch.cpp:35-51
    s = orc.AeroState(2, 1.0, 1.0, 7, 0)
    ev = s.update([10.0, 0.0], 1)
    sn = s.snaps()
    assert len(sn) == 1 and sn[0]["z"].shape[1] == 1
    assert abs(abs(sn[0]["z"][0, 0]) - 1) < 1e-9
    assert abs(abs(sn[0]["m"][0, 0]) - 100.0) < 1e-7 and abs(sn[0]["m"][0, 1]) < 1e-9
    assert sn[0]["s"] == 1 and sn[0]["t"] == 1 and sn[0]["theta"] == 1.0
    assert np.linalg.norm(s.residual()) < 1e-9 and ev["dumped"] == 1


def test_unreachable_threshold(orc):  # test_sketch.cpp:53-61
    s = orc.AeroState(2, 1.0, 1e6, 7, 0)
    ev = s.update([1.0, 0.0], 1)
    assert s.snap_count() == 0 and np.array_equal(s.residual()[0], [1.0, 0.0])
    assert ev["gate_fired"] == 0


def test_reduce_fires_once(orc):  # test_sketch.cpp:63-76
    s = orc.AeroState(8, 1.0, 1e9, 3, 0)
    reduces = 0
    for i in range(1, 6):
        a = gaussian_vec(orc, 8, 100 + i)
        ev = s.update(a / np.linalg.norm(a), i)
        if ev["reduced"]:
            reduces += 1
            assert s.residual().shape[0] <= s.ell - 1
        assert s.residual().shape[0] <= 2 * s.ell
    assert reduces == 1


def test_update_validation(orc):  # test_sketch.cpp:78-93
    s = orc.AeroState(4, 0.5, 0.0, 0, 0)
    s.update(np.ones(4), 1)
    with pytest.raises(orc.InvalidInput):
        s.update(np.ones(4), 1)
    s.update(np.ones(4), 5)
    assert s.clock == 5
    with pytest.raises(orc.InvalidInput):
        s.update(np.ones(3), 6)
    bad = np.ones(4)
    bad[2] = np.nan
    with pytest.raises(orc.InvalidInput):
        s.update(bad, 6)


def test_query_validation_and_zero(orc):  # test_sketch.cpp:114-130
    s = orc.AeroState(4, 0.5, 0.0, 0, 0)
    s.update(np.ones(4), 1)
    for lb, ub in ((1, 1), (2, 1), (0, 2)):
        with pytest.raises(orc.InvalidInput):
            s.query(lb, ub)
    s = orc.AeroState(4, 0.5, 1e9, 0, 0)
    s.update(np.zeros(4), 1)
    b = s.query(0, 1)
    assert b.shape == (s.ell, 4) and np.linalg.norm(b) == 0.0


def test_dump_reconstructed_by_query(orc):  # test_sketch.cpp:132-141
    s = orc.AeroState(2, 1.0, 1.0, 7, 0)
    a = np.array([10.0, 0.0])
    s.update(a, 1)
    b = s.query(0, 1)
    g = np.outer(a, a)
    assert np.linalg.norm(b.T @ b - g) / np.linalg.norm(g) < 1e-8


def test_restoration_identity(orc):  # test_sketch.cpp:143-176, acceptance check 1
    for seed in range(10):
        cp = gaussian(orc, 12, 16, seed, 4)
        z = orthonormal(orc, 16, 3, seed + 50)
        m = z.T @ cp.T @ cp
        c = cp - cp @ z @ z.T
        back = c.T @ c + orc.restore_contribution(z, m)
        want = cp.T @ cp
        assert np.linalg.norm(back - want) / np.linalg.norm(want) < 1e-9
    cp = gaussian(orc, 9, 6, 2)
    z = orthonormal(orc, 6, 6, 77)
    m = z.T @ cp.T @ cp
    want = cp.T @ cp
    assert np.linalg.norm(orc.restore_contribution(z, m) - want) / np.linalg.norm(want) < 1e-9
    x = orc.restore_contribution(orthonormal(orc, 16, 4, 5), orthonormal(orc, 16, 4, 5).T @ (gaussian(orc, 10, 16, 6).T @ gaussian(orc, 10, 16, 6)))
    assert np.linalg.norm(x - x.T) <= 1e-9 * max(1, np.linalg.norm(x))


def test_snapshot_queue_invariants(orc):  # test_sketch.cpp:178-204
    s = orc.AeroState(8, 0.5, 5.0, 21, 0)
    rows = np.stack([gaussian_vec(orc, 8, 300, i) for i in range(1, 201)])
    s.update_block(rows, np.arange(1, 201))
    sn = s.snaps()
    assert sn
    prev = 0
    for x in sn:
        xi = x["z"].shape[1]
        assert xi >= 1 and np.linalg.norm(x["z"].T @ x["z"] - np.eye(xi)) < 1e-8
        assert x["s"] == prev + 1 and x["s"] <= x["t"] and x["t"] > prev and x["theta"] == 5.0
        prev = x["t"]
    g = rows.T @ rows
    b = s.query(0, 200)
    assert orc.spectral_norm_sym(g - b.T @ b) < np.trace(g) / 2


def test_shrink_to_sketch_kat(orc):  # test_sketch.cpp:206-215
    out = orc.shrink_to_sketch(np.diag([9.0, 4, 1, -0.5]), 2)
    assert out.shape[0] == 2
    assert abs(np.linalg.norm(out[0]) - math.sqrt(5)) < 1e-9 and np.linalg.norm(out[1]) < 1e-12


def test_determinism(orc):  # test_sketch.cpp:217-226
    def run():
        s = orc.AeroState(8, 0.5, 3.0, 13, 4)
        rows = np.stack([gaussian_vec(orc, 8, 500, i) for i in range(1, 81)])
        s.update_block(rows, np.arange(1, 81))
        return s.query(0, 80)
    assert np.array_equal(run(), run())


# ---------------------------------------------------------------- attp
def test_attp_threshold_tracks_mass(orc):  # test_attp.cpp:19-27
    s = orc.AttpState(4, 0.1, 0, 0)
    s.update(np.eye(4)[0], 1)
    assert abs(s.inner.theta - 0.1) < 1e-12 and abs(s.fro_mass - 1.0) < 1e-12
    s.update(2 * np.eye(4)[1], 2)
    assert abs(s.fro_mass - 5.0) < 1e-12 and abs(s.inner.theta - 0.5) < 1e-12


def test_attp_persistence_and_bound(orc):  # test_attp.cpp:48-83
    s = orc.AttpState(8, 0.5, 3, 0)
    rows = np.stack([gaussian_vec(orc, 8, 41, i) for i in range(1, 401)])
    s.update_block(rows[:300], np.arange(1, 301))
    before = [s.query(t) for t in (50, 100, 200)]
    s.update_block(rows[300:], np.arange(301, 401))
    for t, b in zip((50, 100, 200), before):
        assert np.array_equal(s.query(t), b)
    d, eps = 8, 0.25
    s = orc.AttpState(d, eps, 5, 6)
    rows = uniform_rows(orc, 400, d, 5, 0)
    s.update_block(rows, np.arange(1, 401))
    for t in (100, 200, 300, 400):
        g = rows[:t].T @ rows[:t]
        b = s.query(t)
        assert orc.spectral_norm_sym(g - b.T @ b) <= eps * np.sum(rows[:t] ** 2)


def test_attp_width_bound(orc):  # test_attp.cpp:85-93
    eps = 0.25
    s = orc.AttpState(16, eps, 9, 2)
    rows = np.stack([gaussian_vec(orc, 16, 43, i) for i in range(1, 2001)])
    s.update_block(rows, np.arange(1, 2001))
    xi_sum = sum(x["z"].shape[1] for x in s.inner.snaps())
    assert xi_sum <= 2 * (2 / eps) * math.log2(2 * s.fro_mass / eps)


# ---------------------------------------------------------------- sliding window
def test_ml_ladder(orc):  # test_sliding_window.cpp:18-42
    s = orc.MlState(4, 1000, 8.0, 0.1, 0, 0)
    assert s.levels == 3 and [s.theta(j) for j in range(3)] == pytest.approx([100, 200, 400])
    assert orc.MlState(4, 100, 2.0, 0.5, 0, 0).levels == 1
    s = orc.MlState(4, 5000, 1024.0, 0.05, 0, 0)
    assert s.levels == 10 and s.theta(0) == pytest.approx(250.0)
    for args in ((4, 100, 0.5, 0.5), (4, 0, 8.0, 0.5), (4, 100, 8.0, 0.0)):
        with pytest.raises(orc.InvalidInput):
            orc.MlState(*args, 0, 0)


def test_ml_heavy_routing_expiry_cap(orc):  # test_sliding_window.cpp:44-83
    s = orc.MlState(4, 10, 16.0, 1.0, 1, 0)
    a = np.array([4.0, 0, 0, 0])
    s.update(a, 1)
    h = s.heavy(0)
    assert len(h) == 1 and np.array_equal(h[0]["row"], a) and h[0]["t"] == 1
    assert s.heavy_count(1) == 0 and s.level_state(0).clock == 0 and s.level_state(1).clock == 1
    s = orc.MlState(4, 10, 16.0, 1.0, 2, 0)
    s.update(a, 1)
    for i in range(2, 12):
        s.update(np.ones(4), i)
    clock = s.info()["clock"]
    for j in range(s.levels):
        assert all(x["t"] > clock - 10 for x in s.heavy(j))
        assert all(x["t"] > clock - 10 for x in s.level_state(j).snaps())
    s = orc.MlState(4, 1000, 1024.0, 1.0, 3, 0)
    hv = np.array([32.0, 0, 0, 0])
    for i in range(1, 31):
        s.update(hv, i)
        for j in range(s.levels):
            assert s.level_state(j).snap_count() + s.heavy_count(j) <= 8
    assert s.heavy_count(0) == 8


def test_ml_misc(orc):  # test_sliding_window.cpp:85-114, 149-161
    s = orc.MlState(4, 10, 8.0, 0.5, 4, 0)
    s.update(0.1 * np.ones(4), 1)
    assert s.info()["norm_warnings"] == 1
    s = orc.MlState(4, 10, 8.0, 0.5, 5, 0)
    with pytest.raises(orc.InvalidInput):
        s.query()
    s = orc.MlState(4, 3, 8.0, 0.5, 6, 0)
    for i in range(1, 6):
        s.update(np.ones(4), i)
    assert s.info()["window_mass"] == pytest.approx(12.0)
    s = orc.MlState(4, 100, 16.0, 0.5, 7, 0)
    s.update(np.ones(4), 1)
    q = s.query()
    guess = math.floor(math.log2(s.info()["window_mass"] / 100.0))
    assert q["fallback"] and q["level"] == int(min(max(guess, 0), s.levels - 1))
    s = orc.MlState(4, 10, 8.0, 0.5, 17, 0)
    for i in range(1, 13):
        s.update(np.ones(4), i)
    expect = 10
    for j in range(s.levels):
        lv = s.level_state(j)
        expect += lv.residual().size + sum(x["z"].size + x["m"].size for x in lv.snaps())
        expect += s.heavy_count(j) * 4
    assert s.stored_floats() == expect


def test_ml_error_budget(orc):  # test_sliding_window.cpp:116-147
    d, n, eps = 8, 100, 0.25
    s = orc.MlState(d, n, 8.0, eps, 11, 9)
    g = orc.OracleGram(d, n)
    rows = uniform_rows(orc, 300, d, 11, 0)
    for i in range(1, 301):
        s.update(rows[i - 1], i)
        g.add_block(rows[i - 1][None], [i])
        if i % 20 == 0:
            assert g.error(s.query()["sketch"]) <= eps
    s = orc.MlState(4, 50, 64.0, 1.0, 13, 0)
    g = orc.OracleGram(4, 50)
    for i in range(1, 21):
        a = 8.0 * np.eye(4)[0] if i == 10 else np.ones(4)
        s.update(a, i)
        g.add_block(a[None], [i])
    q = s.query()
    assert g.error(q["sketch"]) <= 1.0 and q["heavy_used"] >= 1


# ---------------------------------------------------------------- distributed
def test_dist_first_row_reports(orc):  # test_distributed.cpp:45-52
    site = orc.SiteState(0, 4, 0.5, 2, 1, 1000)
    msgs = site.update(np.ones(4), 1)
    assert msgs and msgs[0]["kind"] == "FroMass" and msgs[0]["f"] == pytest.approx(4.0)
    assert msgs[0]["bytes"] == 24


def test_dist_windowed_site_expires_once(orc):  # test_distributed.cpp:140-159
    site = orc.SiteState(0, 4, 1.0, 1, 11, 1000, window=10)
    site.on_broadcast(100.0)
    msgs = site.update(50.0 * np.eye(4)[0], 1)
    assert sum(m["kind"] == "SnapshotUpdate" for m in msgs) == 1
    exp = 0
    for i in range(2, 13):
        exp += sum(m["kind"] == "Expire" and m["t"] == 1 for m in site.update(0.01 * np.ones(4), i))
    assert exp == 1


def test_dist_single_site_equals_attp(orc):  # test_distributed.cpp:161-194
    d, eps, seed, T = 8, 0.25, 5, 300
    rows = uniform_rows(orc, T, d, seed, 0)
    res = orc.dist_run(rows[None], eps, query_every=50, seed=seed)
    attp = orc.AttpState(d, eps, seed, 1000)
    g = orc.OracleGram(d)
    k = 0
    for i in range(1, T + 1):
        attp.update(rows[i - 1], i)
        g.add_block(rows[i - 1][None], [i])
        if i % 50 == 0:
            assert res["probe_err"][k] == g.error(attp.query(i))  # bit-for-bit
            k += 1
    assert k == len(res["probe_err"])


def test_dist_determinism_and_budget(orc):  # test_distributed.cpp:196-222, acceptance check 9
    streams = np.stack([uniform_rows(orc, 200, 6, 3, j) for j in range(2)])
    r1 = orc.dist_run(streams, 0.5, query_every=25, seed=3)
    r2 = orc.dist_run(streams, 0.5, query_every=25, seed=3)
    assert np.array_equal(r1["probe_err"], r2["probe_err"]) and r1["comm_bytes"] == r2["comm_bytes"]
    assert np.all(np.diff(r1["probe_bytes"]) >= 0)
    streams = np.stack([uniform_rows(orc, 1500, 32, 3, j) for j in range(4)])
    res = orc.dist_run(streams, 0.2, query_every=20, seed=3)
    assert np.all(res["probe_err"] <= 0.2)
    mass = float(np.sum(streams ** 2))
    assert res["broadcasts"] <= math.ceil(math.log(mass) / math.log(1.2)) + 1


# ---------------------------------------------------------------- amm
def test_cod_kats(orc):  # test_amm.cpp:20-102
    s = orc.CodState(4, 4, 1.0, 1.0, 100, 2, 0)
    v = 10.0 * np.eye(4)[0]
    s.update(v, v, 1)
    assert s.info()["nsnaps"] == 1
    a, b = s.ab()
    assert np.linalg.norm(a @ b.T) < 1e-8
    s = orc.CodState(4, 4, 1.0, 1.0, 5, 3, 0)
    s.update(v, v, 1)
    for i in range(2, 7):
        s.update(0.01 * np.ones(4), 0.01 * np.ones(4), i)
    assert s.info()["nsnaps"] == 0
    a, b = s.query()
    assert (a @ b.T)[0, 0] < 1.0
    s = orc.CodState(5, 3, 0.5, 1.0, 10, 4, 0)
    a, b = s.query()
    assert a.shape == (5, s.ell) and np.linalg.norm(a) == 0 and np.linalg.norm(b) == 0
    s = orc.CodState(6, 5, 0.5, 1e9, 1000, 7, 0)
    for i in range(1, 41):
        s.update(gaussian_vec(orc, 6, 31, i), gaussian_vec(orc, 5, 32, i), i)
        assert s.info()["cols"] <= 2 * s.ell


def test_cod_error_budget(orc):  # test_amm.cpp:104-122, acceptance check 8
    dx, dy, n, eps = 8, 6, 100, 0.25
    s = orc.CodState(dx, dy, eps, eps * n, n, 8, 3)
    xs, ys = uniform_rows(orc, 300, dx, 8, 0), uniform_rows(orc, 300, dy, 8, 1)
    for i in range(1, 301):
        s.update(xs[i - 1], ys[i - 1], i)
        if i % 20 == 0:
            lo = max(0, i - n)
            p = xs[lo:i].T @ ys[lo:i]
            a, b = s.query()
            den = math.sqrt(np.sum(xs[lo:i] ** 2) * np.sum(ys[lo:i] ** 2))
            assert orc.spectral_norm(p - a @ b.T) / den <= eps


# ---------------------------------------------------------------- amplification (sketch.cpp:45-80)
def test_amplified_requires_delta(orc):  # test_sketch.cpp:94-97
    s = orc.AeroState(4, 0.5, 0.0, 0, 0)
    with pytest.raises(orc.InvalidInput):
        s.update_amplified(np.ones(4), 1)
    for bad in (-0.1, 1.0, 2.0):
        with pytest.raises(orc.InvalidInput):
            orc.AeroState(4, 0.5, 0.0, 0, 0, delta=bad)


def test_amplified_two_candidates_per_doubling_step(orc):  # test_sketch.cpp:99-112
    s = orc.AeroState(8, 0.5, 2.0, 9, 0, delta=0.01)
    saw_dump = False
    for i in range(1, 61):
        ev = s.update_amplified(gaussian_vec(orc, 8, 200 + i), i)
        if ev["doubling_steps"] > 0:
            assert ev["simul_calls"] == 2 * ev["doubling_steps"]  # r = 2 at delta = 0.01
            # r candidates x (1 simul_iter + s = 10 power iterations) forks per step
            assert ev["forks_after"] - ev["forks_before"] == 1 + 2 * 11 * ev["doubling_steps"]
            saw_dump = saw_dump or bool(ev["dumped"])
    assert saw_dump


def test_amplified_acceptance_check_11(orc):  # acceptance.cpp:390-408
    # amplified window sketch keeps the end-to-end error budget (check_window_end_to_end, :152-187)
    d, n, t_end, eps = 32, 500, 1500, 0.2
    for seed in range(3):
        s = orc.MlState(d, n, 32.0, eps, seed + 100, 1000, delta=0.01)
        g = orc.OracleGram(d, n, 100000)
        rows = uniform_rows(orc, t_end, d, seed + 100, 0)
        for b in range(0, t_end, 20):
            s.update_block(rows[b:b + 20], np.arange(b + 1, b + 21))
            g.add_block(rows[b:b + 20], np.arange(b + 1, b + 21))
            assert g.error(s.query()["sketch"]) <= eps
    # trace invariant: two factorization candidates per doubling step
    s = orc.AeroState(32, 0.2, 5.0, 1, 61, delta=0.01)
    rows = uniform_rows(orc, 300, 32, 1, 62)
    ev = s.update_block_amplified(rows, np.arange(1, 301))
    on = ev["doubling_steps"] > 0
    assert on.any() and np.all(ev["simul_calls"][on] == 2 * ev["doubling_steps"][on])


def test_attp_amplified_uses_update_amplified(orc):  # attp.hpp:17-26
    rows = uniform_rows(orc, 120, 16, 3, 0)
    a = orc.AttpState(16, 0.25, 3, 1000, delta=0.01)
    ev = a.update_block(rows, np.arange(1, 121))
    on = ev["doubling_steps"] > 0
    assert on.any() and np.all(ev["simul_calls"][on] == 2 * ev["doubling_steps"][on])
    b = orc.AttpState(16, 0.25, 3, 1000)
    ev_b = b.update_block(rows, np.arange(1, 121))
    assert np.all(ev_b["simul_calls"] == ev_b["doubling_steps"])
