"""ctypes wrapper of the CPU ORACLE (oracle/build/liboracle.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs as the checker and the CPU
baseline. The product package (paper_2601_02019_b200) never imports this.

Class and method names mirror the reference C++ API (AeroState, AttpState,
MlState, CodState, SiteState, OracleGram; /root/reference/proj/include/aero/*).
Matrices are numpy float64, row-major.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "liboracle.so")
_lib = None

i32, i64, u64, f64 = C.c_int, C.c_int64, C.c_uint64, C.c_double
vp = C.c_void_p
P = C.POINTER


class Event(C.Structure):
    """Per-row event record; same layout as the product's aero_event."""

    _fields_ = [
        ("t", i64), ("forks_before", i64), ("forks_after", i64),
        ("rows_after", C.c_int32), ("reduced", C.c_int32), ("gate_fired", C.c_int32),
        ("dumped", C.c_int32), ("doubling_steps", C.c_int32), ("simul_calls", C.c_int32),
        ("xi", C.c_int32), ("k_last", C.c_int32),
        ("theta", f64), ("sigma1_sq", f64), ("tail_sq", f64),
    ]


EVENT_DTYPE = np.dtype([
    ("t", "<i8"), ("forks_before", "<i8"), ("forks_after", "<i8"),
    ("rows_after", "<i4"), ("reduced", "<i4"), ("gate_fired", "<i4"), ("dumped", "<i4"),
    ("doubling_steps", "<i4"), ("simul_calls", "<i4"), ("xi", "<i4"), ("k_last", "<i4"),
    ("theta", "<f8"), ("sigma1_sq", "<f8"), ("tail_sq", "<f8"),
])
assert EVENT_DTYPE.itemsize == C.sizeof(Event)


class InvalidInput(ValueError):
    pass


class FormatError(RuntimeError):
    pass


class ProtocolError(RuntimeError):
    pass


class OracleCapExceeded(RuntimeError):
    pass


_ERRS = {1: InvalidInput, 2: FormatError, 3: ProtocolError, 4: OracleCapExceeded}


def build() -> None:
    subprocess.run(["make", "-s", "-C", _HERE, "build/liboracle.so"], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        _lib = C.CDLL(_LIB_PATH)
        _declare(_lib)
    return _lib


def _declare(L):
    def d(name, res, *args):
        f = getattr(L, name)
        f.restype = res
        f.argtypes = list(args)

    dp = P(f64)
    lp = P(i64)
    ip = P(i32)
    d("orc_last_error", C.c_char_p)
    d("orc_set_threads", None, i32)
    d("orc_event_size", i32)
    d("orc_rng_draw", i32, u64, u64, i64, i64, i32, dp)
    d("orc_svd", i32, dp, i32, i32, dp, dp, dp)
    d("orc_eigh", i32, dp, i32, dp, dp)
    d("orc_qr", i32, dp, i32, i32, dp, dp)
    d("orc_power_iteration", i32, dp, i32, i32, i32, u64, u64, dp, dp)
    d("orc_simul_iter", i32, dp, i32, i32, i32, f64, u64, u64, dp, dp)
    d("orc_fd_reduce", i32, dp, i32, i32, i32, dp)
    d("orc_cod_reduce", i32, dp, i32, dp, i32, i32, i32, dp, dp)
    d("orc_spectral_norm_sym", f64, dp, i32)
    d("orc_spectral_norm", f64, dp, i32, i32)
    d("orc_shrink_to_sketch", i32, dp, i32, i32, dp)
    d("orc_restore_contribution", i32, dp, dp, i32, i32, dp)
    d("orc_aero_create", vp, i32, f64, f64, u64, u64)
    d("orc_aero_create2", vp, i32, f64, f64, u64, u64, f64)
    d("orc_aero_update_block_amplified", i32, vp, dp, i64, lp, dp, P(Event))
    d("orc_attp_create2", vp, i32, f64, u64, u64, f64)
    d("orc_ml_create2", vp, i32, i64, f64, f64, u64, u64, f64)
    d("orc_aero_destroy", None, vp)
    d("orc_aero_set_theta", i32, vp, f64)
    d("orc_aero_update_block", i32, vp, dp, i64, lp, dp, P(Event))
    d("orc_aero_query", i32, vp, i64, i64, dp)
    d("orc_aero_query_gram", i32, vp, i64, i64, dp)
    d("orc_aero_rows", i64, vp)
    d("orc_aero_residual", i32, vp, dp)
    d("orc_aero_snap_count", i64, vp)
    d("orc_aero_snap_info", i32, vp, i64, ip, lp, lp, dp)
    d("orc_aero_snap_get", i32, vp, i64, dp, dp)
    d("orc_aero_snap_pop_front", i32, vp)
    d("orc_aero_info", i32, vp, ip, ip, lp, dp, lp, lp)
    d("orc_attp_create", vp, i32, f64, u64, u64)
    d("orc_attp_destroy", None, vp)
    d("orc_attp_update_block", i32, vp, dp, i64, lp, P(Event))
    d("orc_attp_query", i32, vp, i64, dp)
    d("orc_attp_mass", f64, vp)
    d("orc_attp_import", i32, vp, dp, i64, u64, i64, i64, f64, f64)
    d("orc_attp_inner", vp, vp)
    d("orc_ml_create", vp, i32, i64, f64, f64, u64, u64)
    d("orc_ml_destroy", None, vp)
    d("orc_ml_update_block", i32, vp, dp, i64, lp)
    d("orc_ml_query", i32, vp, dp, ip, ip, lp, ip)
    d("orc_ml_info", i32, vp, ip, ip, dp, lp, lp, lp)
    d("orc_ml_theta", f64, vp, i32)
    d("orc_ml_level", vp, vp, i32)
    d("orc_ml_heavy_count", i64, vp, i32)
    d("orc_ml_heavy_get", i32, vp, i32, i64, dp, lp, lp)
    d("orc_ml_stored_floats", i64, vp)
    d("orc_cod_create", vp, i32, i32, f64, f64, i64, u64, u64)
    d("orc_cod_destroy", None, vp)
    d("orc_cod_update_block", i32, vp, dp, dp, i32, i32, i64, lp, P(Event))
    d("orc_cod_query", i32, vp, dp, dp)
    d("orc_cod_query_product", i32, vp, dp)
    d("orc_cod_info", i32, vp, ip, lp, lp, lp)
    d("orc_cod_get_ab", i32, vp, dp, dp)
    d("orc_adaptive_create", vp, i32, i32, f64, f64, i64, u64, u64)
    d("orc_adaptive_destroy", None, vp)
    d("orc_adaptive_update_block", i32, vp, dp, dp, i32, i32, i64, lp, P(Event), ip, dp, lp)
    d("orc_adaptive_query", i32, vp, dp, dp)
    d("orc_adaptive_query_product", i32, vp, dp)
    d("orc_site_create", vp, i32, i32, f64, i32, u64, u64, i64)
    d("orc_site_destroy", None, vp)
    d("orc_site_update", i32, vp, dp, i64, ip)
    d("orc_site_msg", i32, vp, i32, ip, dp, lp, ip, lp, dp, dp)
    d("orc_site_on_broadcast", None, vp, f64)
    d("orc_site_theta", f64, vp)
    d("orc_site_inner", vp, vp)
    d("orc_dist_run", i32, i32, i32, f64, i64, i64, i64, u64, dp, i64, i64, dp, lp, lp, lp, dp, dp)
    d("orc_gram_create", vp, i32, i64, i64)
    d("orc_gram_destroy", None, vp)
    d("orc_gram_add_block", i32, vp, dp, i32, i64, lp)
    d("orc_gram_error", i32, vp, dp, i64, i32, dp)
    d("orc_gram_mass", f64, vp)
    d("orc_gram_get", i32, vp, dp)
    d("orc_gen_rows", i32, i32, i32, f64, f64, f64, u64, u64, i64, i32, f64, f64, u64, i64, i64, dp)
    d("orc_gen_basis", i32, u64, u64, i32, i32, dp)
    d("orc_gen_amm_rows", i32, u64, i32, i32, i32, f64, f64, i64, i64, dp, dp)


def _chk(rc):
    if rc != 0:
        msg = lib().orc_last_error().decode()
        raise _ERRS.get(rc, RuntimeError)(msg)


def _dp(a):
    return a.ctypes.data_as(P(f64))


def _lp(a):
    return a.ctypes.data_as(P(i64))


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def set_threads(n: int) -> None:
    lib().orc_set_threads(int(n))


# ------------------------------------------------------------------ rng
def rng_draw(seed: int, stream: int, fork: int, count: int, kind: str = "gaussian") -> np.ndarray:
    """Draws of fork #`fork` of RngState(seed, stream) (fork=0: the root)."""
    out = np.empty(count, np.float64)
    _chk(lib().orc_rng_draw(seed, stream, fork, count, 0 if kind == "gaussian" else 1, _dp(out)))
    return out


# ------------------------------------------------------------------ linalg
def svd(a):
    a = _f64(a)
    m, n = a.shape
    k = min(m, n)
    u, s, vt = np.empty((m, k)), np.empty(k), np.empty((k, n))
    _chk(lib().orc_svd(_dp(a), m, n, _dp(u), _dp(s), _dp(vt)))
    return u, s, vt


def eigh(b):
    b = _f64(b)
    n = b.shape[0]
    if b.ndim != 2 or b.shape[1] != n:
        raise InvalidInput("eigh: input not square")
    lam, v = np.empty(n), np.empty((n, n))
    _chk(lib().orc_eigh(_dp(b), n, _dp(lam), _dp(v)))
    return lam, v


def qr(a):
    a = _f64(a)
    m, n = a.shape
    q, r = np.empty((m, min(m, n))), np.empty((min(m, n), n))
    _chk(lib().orc_qr(_dp(a), m, n, _dp(q), _dp(r)))
    return q, r


def power_iteration(a, k, seed, stream):
    a = _f64(a)
    m, n = a.shape
    s2, x = np.empty(1), np.empty(n)
    _chk(lib().orc_power_iteration(_dp(a), m, n, k, seed, stream, _dp(s2), _dp(x)))
    return float(s2[0]), x


def simul_iter(a, k, eps_si, seed, stream):
    a = _f64(a)
    m, n = a.shape
    z, sh = np.empty((m, max(k, 0))), np.empty(max(k, 0))
    _chk(lib().orc_simul_iter(_dp(a), m, n, k, eps_si, seed, stream, _dp(z), _dp(sh)))
    return z, sh


def fd_reduce(b, ell):
    b = _f64(b)
    out = np.empty_like(b)
    _chk(lib().orc_fd_reduce(_dp(b), b.shape[0], b.shape[1], ell, _dp(out)))
    return out


def cod_reduce(a, b, ell):
    a, b = _f64(a), _f64(b)
    if a.shape[1] != b.shape[1]:
        raise InvalidInput("cod_reduce: column-count mismatch")
    ap, bp = np.empty_like(a), np.empty_like(b)
    _chk(lib().orc_cod_reduce(_dp(a), a.shape[0], _dp(b), b.shape[0], a.shape[1], ell, _dp(ap), _dp(bp)))
    return ap, bp


def spectral_norm_sym(s):
    s = _f64(s)
    return lib().orc_spectral_norm_sym(_dp(s), s.shape[0])


def spectral_norm(a):
    a = _f64(a)
    return lib().orc_spectral_norm(_dp(a), a.shape[0], a.shape[1])


def shrink_to_sketch(b, ell):
    b = _f64(b)
    out = np.empty((ell, b.shape[0]))
    _chk(lib().orc_shrink_to_sketch(_dp(b), b.shape[0], ell, _dp(out)))
    return out


def restore_contribution(z, m):
    z, m = _f64(z), _f64(m)
    d, xi = z.shape
    out = np.empty((d, d))
    _chk(lib().orc_restore_contribution(_dp(z), _dp(m), d, xi, _dp(out)))
    return out


# ------------------------------------------------------------------ states
class AeroState:
    """reference sketch.hpp:42-99 (non-amplified)."""

    def __init__(self, d, eps, theta, seed=0, stream=0, delta=None, _handle=None, _owner=None):
        if _handle is not None:
            self._h, self._own, self._owner = _handle, False, _owner
        else:
            h = lib().orc_aero_create2(d, eps, theta, seed, stream, float(delta or 0.0))
            if not h:
                raise InvalidInput(lib().orc_last_error().decode())
            self._h, self._own = h, True
        self._info()

    def __del__(self):
        if getattr(self, "_own", False) and self._h:
            lib().orc_aero_destroy(self._h)
            self._h = None

    def _info(self):
        d, ell, clock, theta, forks, ld = i32(), i32(), i64(), f64(), i64(), i64()
        lib().orc_aero_info(self._h, C.byref(d), C.byref(ell), C.byref(clock), C.byref(theta),
                            C.byref(forks), C.byref(ld))
        self.d, self.ell = d.value, ell.value
        return clock.value, theta.value, forks.value, ld.value

    @property
    def clock(self):
        return self._info()[0]

    @property
    def theta(self):
        return self._info()[1]

    @property
    def forks(self):
        return self._info()[2]

    @property
    def last_dump_time(self):
        return self._info()[3]

    def set_theta(self, theta):
        _chk(lib().orc_aero_set_theta(self._h, theta))

    def update(self, a, i):
        return self.update_block(np.asarray(a, np.float64)[None, :], [i])[0]

    def update_block(self, rows, ts, thetas=None):
        rows = _f64(rows)
        if rows.ndim != 2 or rows.shape[1] != self.d:
            raise InvalidInput("AeroState: row dimension mismatch")
        ts = np.ascontiguousarray(ts, np.int64)
        n = rows.shape[0]
        ev = (Event * max(n, 1))()
        th = _dp(_f64(thetas)) if thetas is not None else None
        if thetas is not None:
            thetas = _f64(thetas)
            th = _dp(thetas)
        _chk(lib().orc_aero_update_block(self._h, _dp(rows), n, _lp(ts), th, ev))
        return np.frombuffer(ev, dtype=EVENT_DTYPE, count=n).copy()

    def update_block_amplified(self, rows, ts, thetas=None):
        """n sequential update_amplified calls (sketch.cpp:45-48)."""
        rows = _f64(rows)
        ts = np.ascontiguousarray(ts, np.int64)
        n = rows.shape[0]
        ev = (Event * max(n, 1))()
        th = None
        if thetas is not None:
            thetas = _f64(thetas)
            th = _dp(thetas)
        _chk(lib().orc_aero_update_block_amplified(self._h, _dp(rows), n, _lp(ts), th, ev))
        return np.frombuffer(ev, dtype=EVENT_DTYPE, count=n).copy()

    def update_amplified(self, a, i):
        return self.update_block_amplified(np.asarray(a, np.float64)[None, :], [i])[0]

    def query(self, lb, ub):
        out = np.empty((self.ell, self.d))
        _chk(lib().orc_aero_query(self._h, lb, ub, _dp(out)))
        return out

    def query_gram(self, lb, ub):
        out = np.empty((self.d, self.d))
        _chk(lib().orc_aero_query_gram(self._h, lb, ub, _dp(out)))
        return out

    def residual(self):
        r = lib().orc_aero_rows(self._h)
        out = np.empty((r, self.d))
        _chk(lib().orc_aero_residual(self._h, _dp(out)))
        return out

    def snaps(self):
        out = []
        for idx in range(lib().orc_aero_snap_count(self._h)):
            xi, s, t, th = i32(), i64(), i64(), f64()
            _chk(lib().orc_aero_snap_info(self._h, idx, C.byref(xi), C.byref(s), C.byref(t), C.byref(th)))
            z, m = np.empty((self.d, xi.value)), np.empty((xi.value, self.d))
            _chk(lib().orc_aero_snap_get(self._h, idx, _dp(z), _dp(m)))
            out.append(dict(z=z, m=m, s=s.value, t=t.value, theta=th.value))
        return out

    def snap_count(self):
        return lib().orc_aero_snap_count(self._h)

    def snap_pop_front(self):
        _chk(lib().orc_aero_snap_pop_front(self._h))


class AttpState:
    """reference attp.hpp:15-43."""

    def __init__(self, d, eps, seed=0, stream=0, delta=None):
        h = lib().orc_attp_create2(d, eps, seed, stream, float(delta or 0.0))
        if not h:
            raise InvalidInput(lib().orc_last_error().decode())
        self._h = h
        self.inner = AeroState(0, 0, 0, _handle=lib().orc_attp_inner(h), _owner=self)
        self.d, self.ell = self.inner.d, self.inner.ell

    def __del__(self):
        if getattr(self, "_h", None):
            lib().orc_attp_destroy(self._h)
            self._h = None

    def update_block(self, rows, ts):
        rows = _f64(rows)
        if rows.ndim != 2 or rows.shape[1] != self.d:
            raise InvalidInput("AeroState: row dimension mismatch")
        ts = np.ascontiguousarray(ts, np.int64)
        n = rows.shape[0]
        ev = (Event * max(n, 1))()
        _chk(lib().orc_attp_update_block(self._h, _dp(rows), n, _lp(ts), ev))
        return np.frombuffer(ev, dtype=EVENT_DTYPE, count=n).copy()

    def update(self, a, i):
        return self.update_block(np.asarray(a, np.float64)[None, :], [i])[0]

    def query(self, t):
        out = np.empty((self.ell, self.d))
        _chk(lib().orc_attp_query(self._h, t, _dp(out)))
        return out

    @property
    def fro_mass(self):
        return lib().orc_attp_mass(self._h)

    def import_state(self, residual, forks, clock, last_dump_t, theta, fro_mass):
        """Adopt an exported live state (residual rows r x d, RngState fork
        counter, clock, last dump time, threshold, running mass)."""
        residual = _f64(residual).reshape(-1, self.d)
        _chk(lib().orc_attp_import(self._h, _dp(residual), residual.shape[0], int(forks), int(clock),
                                   int(last_dump_t), float(theta), float(fro_mass)))

    @property
    def clock(self):
        return self.inner.clock


class MlState:
    """reference sliding_window.hpp:39-81."""

    def __init__(self, d, n, r_max, eps, seed=0, stream=0, delta=None):
        h = lib().orc_ml_create2(d, n, r_max, eps, seed, stream, float(delta or 0.0))
        if not h:
            raise InvalidInput(lib().orc_last_error().decode())
        self._h, self.d, self.n = h, d, n
        self.levels, self.ell = self.info()["levels"], self.info()["ell"]

    def __del__(self):
        if getattr(self, "_h", None):
            lib().orc_ml_destroy(self._h)
            self._h = None

    def info(self):
        lv, ell, wm, nw, cap, clock = i32(), i32(), f64(), i64(), i64(), i64()
        lib().orc_ml_info(self._h, C.byref(lv), C.byref(ell), C.byref(wm), C.byref(nw), C.byref(cap),
                          C.byref(clock))
        return dict(levels=lv.value, ell=ell.value, window_mass=wm.value, norm_warnings=nw.value,
                    cap=cap.value, clock=clock.value)

    def theta(self, j):
        return lib().orc_ml_theta(self._h, j)

    def update_block(self, rows, ts):
        rows = _f64(rows)
        if rows.ndim != 2 or rows.shape[1] != self.d:
            raise InvalidInput("MlState: row dimension mismatch")
        ts = np.ascontiguousarray(ts, np.int64)
        _chk(lib().orc_ml_update_block(self._h, _dp(rows), rows.shape[0], _lp(ts)))

    def update(self, a, i):
        self.update_block(np.asarray(a, np.float64)[None, :], [i])

    def query(self):
        sk = np.empty((self.ell, self.d))
        lv, fb, xs, hu = i32(), i32(), i64(), i32()
        _chk(lib().orc_ml_query(self._h, _dp(sk), C.byref(lv), C.byref(fb), C.byref(xs), C.byref(hu)))
        return dict(sketch=sk, level=lv.value, fallback=bool(fb.value), xi_sum=xs.value,
                    heavy_used=hu.value)

    def level_state(self, j):
        return AeroState(0, 0, 0, _handle=lib().orc_ml_level(self._h, j), _owner=self)

    def heavy(self, j):
        out = []
        for idx in range(lib().orc_ml_heavy_count(self._h, j)):
            row, s, t = np.empty(self.d), i64(), i64()
            _chk(lib().orc_ml_heavy_get(self._h, j, idx, _dp(row), C.byref(s), C.byref(t)))
            out.append(dict(row=row, s=s.value, t=t.value))
        return out

    def heavy_count(self, j):
        return lib().orc_ml_heavy_count(self._h, j)

    def stored_floats(self):
        return lib().orc_ml_stored_floats(self._h)


class CodState:
    """reference amm.hpp:35-69."""

    def __init__(self, dx, dy, eps, theta, n, seed=0, stream=0):
        h = lib().orc_cod_create(dx, dy, eps, theta, n, seed, stream)
        if not h:
            raise InvalidInput(lib().orc_last_error().decode())
        self._h, self.dx, self.dy = h, dx, dy
        self.ell = self.info()["ell"]

    def __del__(self):
        if getattr(self, "_h", None):
            lib().orc_cod_destroy(self._h)
            self._h = None

    def info(self):
        ell, cols, ns, clock = i32(), i64(), i64(), i64()
        lib().orc_cod_info(self._h, C.byref(ell), C.byref(cols), C.byref(ns), C.byref(clock))
        return dict(ell=ell.value, cols=cols.value, nsnaps=ns.value, clock=clock.value)

    def update_block(self, xs, ys, ts):
        xs, ys = _f64(xs), _f64(ys)
        if xs.shape[1] != self.dx or ys.shape[1] != self.dy:
            raise InvalidInput("CodState: dimension mismatch")
        ts = np.ascontiguousarray(ts, np.int64)
        n = xs.shape[0]
        ev = (Event * max(n, 1))()
        _chk(lib().orc_cod_update_block(self._h, _dp(xs), _dp(ys), self.dx, self.dy, n, _lp(ts), ev))
        return np.frombuffer(ev, dtype=EVENT_DTYPE, count=n).copy()

    def update(self, x, y, i):
        return self.update_block(np.asarray(x, np.float64)[None], np.asarray(y, np.float64)[None], [i])[0]

    def query(self):
        a, b = np.empty((self.dx, self.ell)), np.empty((self.dy, self.ell))
        _chk(lib().orc_cod_query(self._h, _dp(a), _dp(b)))
        return a, b

    def query_product(self):
        p = np.empty((self.dx, self.dy))
        _chk(lib().orc_cod_query_product(self._h, _dp(p)))
        return p

    def ab(self):
        cols = self.info()["cols"]
        a, b = np.empty((self.dx, cols)), np.empty((self.dy, cols))
        _chk(lib().orc_cod_get_ab(self._h, _dp(a), _dp(b)))
        return a, b


class AdaptiveState:
    """reference amm.hpp:71-93 / amm.cpp:131-161 (main/aux CodState pair with
    queue-length-driven threshold doubling and halving)."""

    def __init__(self, dx, dy, eps, theta0, n, seed=0, stream=0):
        h = lib().orc_adaptive_create(dx, dy, eps, theta0, n, seed, stream)
        if not h:
            raise InvalidInput(lib().orc_last_error().decode())
        self._h, self.dx, self.dy, self.ell = h, dx, dy, int(np.ceil(2.0 / eps))

    def __del__(self):
        if getattr(self, "_h", None):
            lib().orc_adaptive_destroy(self._h)
            self._h = None

    def update_block(self, xs, ys, ts):
        """-> (main's events, level, main theta, main snapshot count) per row."""
        xs, ys = _f64(xs), _f64(ys)
        ts = np.ascontiguousarray(ts, np.int64)
        n = xs.shape[0]
        ev = (Event * max(n, 1))()
        lv = np.zeros(max(n, 1), np.int32)
        th = np.zeros(max(n, 1))
        ns = np.zeros(max(n, 1), np.int64)
        _chk(lib().orc_adaptive_update_block(self._h, _dp(xs), _dp(ys), self.dx, self.dy, n, _lp(ts), ev,
                                             lv.ctypes.data_as(P(i32)), _dp(th), _lp(ns)))
        return dict(events=np.frombuffer(ev, dtype=EVENT_DTYPE, count=n).copy(), level=lv[:n],
                    theta=th[:n], nsnaps=ns[:n])

    def query(self):
        a, b = np.empty((self.dx, self.ell)), np.empty((self.dy, self.ell))
        _chk(lib().orc_adaptive_query(self._h, _dp(a), _dp(b)))
        return a, b

    def query_product(self):
        p = np.empty((self.dx, self.dy))
        _chk(lib().orc_adaptive_query_product(self._h, _dp(p)))
        return p


MSG_KINDS = ("FroMass", "FroBroadcast", "SnapshotUpdate", "Expire")


class SiteState:
    """reference distributed.hpp:47-76."""

    def __init__(self, site_id, d, eps, m, seed, stream, window=0):
        h = lib().orc_site_create(site_id, d, eps, m, seed, stream, window)
        if not h:
            raise InvalidInput(lib().orc_last_error().decode())
        self._h, self.d = h, d

    def __del__(self):
        if getattr(self, "_h", None):
            lib().orc_site_destroy(self._h)
            self._h = None

    def update(self, a, i):
        a = _f64(a)
        n = i32()
        _chk(lib().orc_site_update(self._h, _dp(a), i, C.byref(n)))
        msgs = []
        for idx in range(n.value):
            kind, f, t, xi, nb = i32(), f64(), i64(), i32(), i64()
            _chk(lib().orc_site_msg(self._h, idx, C.byref(kind), C.byref(f), C.byref(t), C.byref(xi),
                                    C.byref(nb), None, None))
            z = m = None
            if MSG_KINDS[kind.value] == "SnapshotUpdate":
                z, m = np.empty((self.d, xi.value)), np.empty((xi.value, self.d))
                _chk(lib().orc_site_msg(self._h, idx, C.byref(kind), C.byref(f), C.byref(t),
                                        C.byref(xi), C.byref(nb), _dp(z), _dp(m)))
            msgs.append(dict(kind=MSG_KINDS[kind.value], f=f.value, t=t.value, xi=xi.value,
                             bytes=nb.value, z=z, m=m))
        return msgs

    def on_broadcast(self, f):
        lib().orc_site_on_broadcast(self._h, f)

    @property
    def theta(self):
        return lib().orc_site_theta(self._h)

    @property
    def inner(self):
        return AeroState(0, 0, 0, _handle=lib().orc_site_inner(self._h), _owner=self)


def dist_run(streams, eps, query_every=20, window=0, latency=0, seed=0, oracle_cap=50000,
             want_thetas=False, probes=True):
    """reference distributed.cpp:177-269 (run_simulation). streams: (m, T, d)."""
    streams = _f64(streams)
    m, T, d = streams.shape
    nprobe = T // query_every if (probes and query_every > 0) else 0
    perr = np.full(max(nprobe, 1), np.nan)
    pbytes = np.zeros(max(nprobe, 1), np.int64)
    cb, bc = i64(), i64()
    thetas = np.empty((m, T)) if want_thetas else None
    gram = np.empty((d, d)) if nprobe else None
    _chk(lib().orc_dist_run(m, d, eps, window, query_every, latency, seed, _dp(streams), T, oracle_cap,
                            _dp(perr) if nprobe else None, _lp(pbytes), C.byref(cb), C.byref(bc),
                            _dp(thetas) if want_thetas else None, _dp(gram) if nprobe else None))
    return dict(probe_err=perr[:nprobe], probe_bytes=pbytes[:nprobe], comm_bytes=cb.value,
                broadcasts=bc.value, thetas=thetas, last_probe_gram=gram)


class OracleGram:
    """reference oracle.hpp:22-76."""

    def __init__(self, d, window=0, cap=1 << 62):
        self._h, self.d = lib().orc_gram_create(d, window or 0, cap), d

    def __del__(self):
        if getattr(self, "_h", None):
            lib().orc_gram_destroy(self._h)
            self._h = None

    def add_block(self, rows, ts):
        rows = _f64(rows)
        ts = np.ascontiguousarray(ts, np.int64)
        _chk(lib().orc_gram_add_block(self._h, _dp(rows), self.d, rows.shape[0], _lp(ts)))

    def error(self, sketch):
        sketch = _f64(sketch)
        e = f64()
        _chk(lib().orc_gram_error(self._h, _dp(sketch), sketch.shape[0], self.d, C.byref(e)))
        return e.value

    @property
    def mass(self):
        return lib().orc_gram_mass(self._h)

    def gram(self):
        g = np.empty((self.d, self.d))
        _chk(lib().orc_gram_get(self._h, _dp(g)))
        return g


# ------------------------------------------------------------------ generators
def gen_rows(d, k, rho, noise, r_max, seed, stream, t0, n, drift=0, k2=0, rho2=0.9, scale2=0.5,
             basis_stream=0):
    out = np.empty((n, d))
    _chk(lib().orc_gen_rows(d, k, rho, noise, r_max, seed, stream, drift, k2, rho2, scale2,
                            basis_stream, t0, n, _dp(out)))
    return out


def gen_basis(seed, basis_id, d, k):
    out = np.empty((k, d))
    _chk(lib().orc_gen_basis(seed, basis_id, d, k, _dp(out)))
    return out


def gen_amm_rows(seed, dx, dy, latent, noise, r_max, t0, n):
    x, y = np.empty((n, dx)), np.empty((n, dy))
    _chk(lib().orc_gen_amm_rows(seed, dx, dy, latent, noise, r_max, t0, n, _dp(x), _dp(y)))
    return x, y


# ------------------------------------------------------------------ AERO files
def aero_bytes(rows):
    """save_stream(..., StreamFormat::Aero) restated (reference streams.cpp:150-168):
    'AERO', version 0x01, u32 d, u64 n, rows as little-endian fp64 row-major."""
    rows = np.ascontiguousarray(rows, "<f8")
    n, d = rows.shape
    return b"AERO" + bytes([1]) + np.uint32(d).tobytes() + np.uint64(n).tobytes() + rows.tobytes()


def load_aero_bytes(buf):
    """load_aero restated (reference streams.cpp:107-137); raises FormatError."""
    if len(buf) < 4 or buf[:4] != b"AERO":
        raise FormatError("bad magic")
    if len(buf) < 5 or buf[4] != 1:
        raise FormatError("unsupported version")
    if len(buf) < 17:
        raise FormatError("truncated header")
    d = int(np.frombuffer(buf[5:9], "<u4")[0])
    n = int(np.frombuffer(buf[9:17], "<u8")[0])
    if d == 0:
        raise FormatError("zero dimension")
    body = buf[17:]
    rb = 8 * d
    avail = len(body) // rb
    if n == 0:
        if len(body) % rb:
            raise FormatError(f"truncated row {avail + 1}")
        n = avail
    elif avail < n:
        raise FormatError(f"truncated row {avail + 1}")
    rows = np.frombuffer(body[:n * rb], "<f8").reshape(n, d).copy()
    if not np.all(np.isfinite(rows)):
        raise FormatError("non-finite value")
    return rows
