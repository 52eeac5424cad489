"""ctypes binding of libaero_b200.so (include/aero_b200.h).

Host-side mirror of the reference C++ sketch API (/root/reference/proj/include/
aero/*.hpp): AeroState, AttpState, MlState, the distributed site/coordinator
merge, and the stream generator. Every compute call goes through the C-ABI to
the sm_100a kernels; there is no CPU fallback -- on a machine without a CUDA
device the constructors raise CudaError.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libaero_b200.so")
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "aero_b200.h")

i32, i64, u64, f64 = C.c_int32, C.c_int64, C.c_uint64, C.c_double
vp = C.c_void_p
P = C.POINTER

AERO_THETA_FIXED, AERO_THETA_ATTP = 0, 1
AERO_FLAG_EXACT = 1
AERO_FLAG_PROFILE = 2
AERO_FLAG_HOST_RNG = 4


class InvalidInput(ValueError):
    pass


class FormatError(RuntimeError):
    pass


class ProtocolError(RuntimeError):
    pass


class OracleCapExceeded(RuntimeError):
    pass


class CudaError(RuntimeError):
    pass


_ERRS = {1: InvalidInput, 2: FormatError, 3: ProtocolError, 4: OracleCapExceeded, 10: CudaError}


class Cfg(C.Structure):
    _fields_ = [("d", i32), ("ell", i32), ("eps", f64), ("theta", f64), ("eps_si", f64),
                ("seed", u64), ("stream", u64), ("device", i32), ("theta_mode", i32),
                ("flags", i32), ("max_batch", i32), ("delta", f64)]


class Event(C.Structure):
    _fields_ = [("t", i64), ("forks_before", i64), ("forks_after", i64),
                ("rows_after", C.c_int32), ("reduced", C.c_int32), ("gate_fired", C.c_int32),
                ("dumped", C.c_int32), ("doubling_steps", C.c_int32), ("simul_calls", C.c_int32),
                ("xi", C.c_int32), ("k_last", C.c_int32),
                ("theta", f64), ("sigma1_sq", f64), ("tail_sq", f64)]


EVENT_DTYPE = np.dtype([
    ("t", "<i8"), ("forks_before", "<i8"), ("forks_after", "<i8"),
    ("rows_after", "<i4"), ("reduced", "<i4"), ("gate_fired", "<i4"), ("dumped", "<i4"),
    ("doubling_steps", "<i4"), ("simul_calls", "<i4"), ("xi", "<i4"), ("k_last", "<i4"),
    ("theta", "<f8"), ("sigma1_sq", "<f8"), ("tail_sq", "<f8"),
])
assert EVENT_DTYPE.itemsize == C.sizeof(Event)


class Info(C.Structure):
    _fields_ = [("d", i32), ("ell", i32), ("rows", i32), ("clock", i64), ("last_dump_t", i64),
                ("forks", i64), ("snaps", i64), ("snap_cols", i64), ("theta", f64),
                ("fro_mass", f64), ("device_rows_processed", i64), ("device_batches", i64),
                ("device_mispredicts", i64), ("end_nofire", i64), ("end_fired", i64),
                ("end_doubling", i64), ("end_dump", i64)]


class Profile(C.Structure):
    _fields_ = [("product_ms", f64), ("product_launches", i64), ("product_flops", f64),
                ("product_bytes", f64), ("iterate_ms", f64), ("reduce_ms", f64), ("reduces", i64)]


class MlQueryResult(C.Structure):
    _fields_ = [("level", i32), ("fallback", i32), ("heavy_used", i32), ("_pad", i32),
                ("xi_sum", i64)]


class MlInfo(C.Structure):
    _fields_ = [("d", i32), ("ell", i32), ("levels", i32), ("_pad", i32), ("n", i64), ("cap", i64),
                ("clock", i64), ("norm_warnings", i64), ("stored_floats", i64),
                ("window_mass", f64)]


class GenParams(C.Structure):
    _fields_ = [("d", i32), ("k", i32), ("k2", i32), ("_pad", i32), ("rho", f64), ("noise", f64),
                ("r_max", f64), ("rho2", f64), ("scale2", f64), ("seed", u64), ("stream", u64),
                ("basis_stream", u64), ("drift_period", i64)]


# every entry point declared in include/aero_b200.h: (name, restype, argtypes)
SIGNATURES = [
    ("aero_create", i32, [P(Cfg), P(vp)]),
    ("aero_destroy", i32, [vp]),
    ("aero_set_theta", i32, [vp, f64]),
    ("aero_set_rng_fill", i32, [vp, vp, vp]),
    ("aero_set_grid_share", i32, [vp, i32]),
    ("aero_update_block", i32, [vp, P(f64), i64, i64, P(i64), P(f64), P(Event)]),
    ("aero_file_open", i32, [C.c_char_p, P(vp), P(i32), P(u64)]),
    ("aero_file_read", i32, [vp, P(f64), i64, P(i64)]),
    ("aero_file_close", i32, [vp]),
    ("aero_file_write", i32, [C.c_char_p, P(f64), i64, i32]),
    ("aero_update_from_file", i32, [vp, C.c_char_p, i64, i64, P(Event), i64, P(i64)]),
    ("aero_update_block_device", i32, [vp, vp, i64, i64, P(i64), P(f64), P(Event)]),
    ("aero_update_block_amplified", i32, [vp, P(f64), i64, i64, P(i64), P(f64), P(Event)]),
    ("aero_query", i32, [vp, i64, i64, P(f64)]),
    ("aero_query_gram", i32, [vp, i64, i64, P(f64)]),
    ("aero_residual", i32, [vp, P(f64), i64]),
    ("aero_snap_count", i32, [vp, P(i64)]),
    ("aero_snap_info", i32, [vp, i64, P(i32), P(i64), P(i64), P(f64)]),
    ("aero_snap_get", i32, [vp, i64, P(f64), P(f64)]),
    ("aero_snap_pop_front", i32, [vp]),
    ("aero_last_stats", i32, [vp, P(Event)]),
    ("aero_get_info", i32, [vp, P(Info)]),
    ("aero_synchronize", i32, [vp]),
    ("aero_attp_query", i32, [vp, i64, P(f64)]),
    ("aero_stream", vp, [vp]),
    ("aero_get_profile", i32, [vp, P(Profile)]),
    ("aero_reset_profile", i32, [vp]),
    ("aero_ml_create", i32, [i32, i64, f64, f64, u64, u64, i32, P(vp)]),
    ("aero_ml_create_amplified", i32, [i32, i64, f64, f64, f64, u64, u64, i32, P(vp)]),
    ("aero_ml_destroy", i32, [vp]),
    ("aero_ml_update_block", i32, [vp, P(f64), i64, i64, P(i64)]),
    ("aero_ml_update_block_device", i32, [vp, vp, i64, i64, P(i64)]),
    ("aero_ml_query", i32, [vp, P(f64), P(MlQueryResult)]),
    ("aero_ml_get_info", i32, [vp, P(MlInfo)]),
    ("aero_ml_theta", f64, [vp, i32]),
    ("aero_ml_level", vp, [vp, i32]),
    ("aero_ml_heavy_count", i32, [vp, i32, P(i64)]),
    ("aero_ml_heavy_get", i32, [vp, i32, i64, P(f64), P(i64), P(i64)]),
    ("aero_dist_theta_schedule", i32, [i32, i64, f64, i64, P(f64), P(f64), P(i64), P(i64)]),
    ("aero_dist_protocol_create", i32, [i32, f64, i64, P(vp)]),
    ("aero_dist_protocol_destroy", i32, [vp]),
    ("aero_dist_protocol_advance", i32, [vp, i64, P(f64), P(f64)]),
    ("aero_dist_protocol_info", i32, [vp, P(i64), P(i64), P(i64), P(f64)]),
    ("aero_row_sq_norms_device", i32, [vp, i64, i64, i32, i32, P(f64)]),
    ("aero_coord_create", i32, [i32, i32, i32, vp, P(vp)]),
    ("aero_coord_destroy", i32, [vp]),
    ("aero_coord_absorb_snapshots", i32, [vp, vp, P(i64)]),
    ("aero_coord_probe", i32, [vp, P(vp), i32, i32, i32, P(f64), P(f64)]),
    ("aero_nccl_get_unique_id", i32, [C.c_char_p]),
    ("aero_nccl_comm_init", i32, [C.c_char_p, i32, i32, i32, P(vp)]),
    ("aero_nccl_comm_destroy", i32, [vp]),
    ("aero_cod_create", i32, [i32, i32, f64, f64, i64, u64, u64, i32, P(vp)]),
    ("aero_cod_destroy", i32, [vp]),
    ("aero_cod_update_block", i32, [vp, P(f64), P(f64), i64, P(i64), P(Event)]),
    ("aero_cod_query", i32, [vp, P(f64), P(f64)]),
    ("aero_cod_query_product", i32, [vp, P(f64)]),
    ("aero_cod_info", i32, [vp, P(i32), P(i64), P(i64), P(i64)]),
    ("aero_dist_protocol_create_window", i32, [i32, f64, i64, i64, P(vp)]),
    ("aero_coord_create_window", i32, [i32, i32, i32, vp, i64, i64, P(vp)]),
    ("aero_coord_shrink", i32, [vp, P(f64), i32, P(f64)]),
    ("aero_cod_theta", i32, [vp, P(f64)]),
    ("aero_cod_set_theta", i32, [vp, f64]),
    ("aero_adaptive_create", i32, [i32, i32, f64, f64, i64, u64, u64, i32, P(vp)]),
    ("aero_adaptive_destroy", i32, [vp]),
    ("aero_adaptive_update_block", i32, [vp, P(f64), P(f64), i64, P(i64), P(Event), P(i32)]),
    ("aero_adaptive_query", i32, [vp, P(f64), P(f64)]),
    ("aero_adaptive_query_product", i32, [vp, P(f64)]),
    ("aero_adaptive_info", i32, [vp, P(i32), P(f64), P(f64), P(i64), P(i64)]),
    ("aero_gen_rows_device", i32, [P(GenParams), i64, i64, vp, i32]),
    ("aero_last_error", C.c_char_p, []),
    ("aero_version", C.c_char_p, []),
    ("aero_kernel_launches", i64, []),
    ("aero_rng_gaussians_host", i32, [u64, u64, i64, i64, P(f64)]),
    ("aero_rng_gaussians", i32, [u64, u64, i64, i64, P(f64)]),
    ("aero_eigh", i32, [i32, P(f64), P(f64), P(f64), P(f64)]),
    ("aero_dev_product", i32, [i32, i32, P(f64), P(f64), P(i32), i32, P(f64), P(f64)]),
]

_lib = None


def lib():
    """Load the in-tree extension; raises if it was not built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run __graft_entry__.build() (no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _chk(rc):
    if rc != 0:
        raise _ERRS.get(rc, RuntimeError)(lib().aero_last_error().decode())


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _dp(a):
    return a.ctypes.data_as(P(f64)) if a is not None else None


def _lp(a):
    return a.ctypes.data_as(P(i64))


def kernel_launches() -> int:
    return int(lib().aero_kernel_launches())


def rng_gaussians(seed, stream, fork, count):
    out = np.empty(count)
    _chk(lib().aero_rng_gaussians(seed, stream, fork, count, _dp(out)))
    return out


def rng_gaussians_host(seed, stream, fork, count):
    """Host draws of AERO_FLAG_HOST_RNG (no GPU needed)."""
    out = np.empty(count)
    _chk(lib().aero_rng_gaussians_host(seed, stream, fork, count, _dp(out)))
    return out


def eigh(b, return_ms=False):
    """Device symmetric eigensolver (linalg.cpp:60-77 semantics)."""
    b = _f64(b)
    n = b.shape[0]
    w, v, ms = np.empty(n), np.empty((n, n)), f64()
    _chk(lib().aero_eigh(n, _dp(b), _dp(w), _dp(v), C.byref(ms)))
    return (w, v, ms.value) if return_ms else (w, v)


def dev_product(g, x, colmask=None, mode=0, return_ms=False):
    """Y = G X through the engine's product kernels (test hook): mode 0 = int8
    tensor cores by exact slicing (ozaki.cu), 1 = fp64 DMMA (product.cu).
    g: r x r symmetric; x: r x n; colmask: per-column prefix lengths."""
    g = _f64(g)
    r, n = g.shape[0], x.shape[1]
    xt = np.ascontiguousarray(np.asarray(x, dtype=np.float64).T)  # column-major r x n
    y = np.empty((n, r))
    ms = f64()
    cm = None
    if colmask is not None:
        cm = np.ascontiguousarray(colmask, dtype=np.int32)
    _chk(lib().aero_dev_product(r, n, _dp(g), _dp(xt), cm.ctypes.data_as(P(i32)) if cm is not None else None,
                                mode, _dp(y), C.byref(ms) if return_ms else None))
    return (y.T, ms.value) if return_ms else y.T


def _device_ptr(x, stream_handle=None):
    """(pointer, ld) of a CUDA torch tensor of shape (n, d), float64.

    The library reads device rows on its own stream; the rows may still be in
    flight on the caller's current torch stream, so the library stream is
    made to wait for it (an event, no host sync) when its handle is known,
    and the caller's stream is synchronized otherwise."""
    import torch
    if not (x.is_cuda and x.dtype == torch.float64 and x.dim() == 2 and x.stride(1) == 1):
        raise InvalidInput("device rows must be a CUDA float64 (n, d) tensor with unit column stride")
    cur = torch.cuda.current_stream(x.device)
    if stream_handle:
        torch.cuda.ExternalStream(stream_handle, device=x.device).wait_stream(cur)
    else:
        cur.synchronize()
    return C.c_void_p(x.data_ptr()), x.stride(0)


def _check_block(n_rows, n, thetas=None):
    """rows / thetas must cover exactly the n timestamps (the C side reads n of each)."""
    if n_rows != n:
        raise InvalidInput(f"row block has {n_rows} rows for {n} timestamps")
    if thetas is not None and len(thetas) != n:
        raise InvalidInput(f"{len(thetas)} thresholds for {n} timestamps")


# aero_rng_fill(ctx, fork_index, out, count) (include/aero_b200.h)
RNG_FILL = C.CFUNCTYPE(i32, vp, u64, P(f64), i64)


class AeroState:
    """reference AeroState (sketch.hpp:42-99): construct with d and eps (or an
    explicit ell), update by row or row block, query(lb, ub).

    host_rng=True draws every random projection on the host (the library's
    restatement of rng.hpp, AERO_FLAG_HOST_RNG); set_rng_fill(fn) hands them to
    a caller-owned source instead."""

    def __init__(self, d, eps, theta=0.0, seed=0, stream=0, device=0, ell=0, theta_mode=AERO_THETA_FIXED,
                 exact=False, max_batch=0, profile=False, host_rng=False, delta=None, _handle=None, _owner=None):
        self._owner = _owner
        self._rng_cb = None
        if _handle is not None:
            self._h, self._own = _handle, False
        else:
            cfg = Cfg(d=d, ell=ell, eps=eps, theta=theta, eps_si=0.0, seed=seed, stream=stream,
                      device=device, theta_mode=theta_mode,
                      flags=(AERO_FLAG_EXACT if exact else 0) | (AERO_FLAG_PROFILE if profile else 0)
                      | (AERO_FLAG_HOST_RNG if host_rng else 0),
                      max_batch=max_batch, delta=float(delta or 0.0))
            h = vp()
            _chk(lib().aero_create(C.byref(cfg), C.byref(h)))
            self._h, self._own = h, True
        inf = self.info()
        self.d, self.ell = inf.d, inf.ell

    def close(self):
        if getattr(self, "_own", False) and self._h:
            lib().aero_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def info(self):
        inf = Info()
        _chk(lib().aero_get_info(self._h, C.byref(inf)))
        return inf

    @property
    def clock(self):
        return self.info().clock

    @property
    def theta(self):
        return self.info().theta

    @property
    def forks(self):
        return self.info().forks

    @property
    def last_dump_time(self):
        return self.info().last_dump_t

    def set_theta(self, theta):
        _chk(lib().aero_set_theta(self._h, theta))

    def set_rng_fill(self, fn):
        """fn(fork_index, count) -> the first `count` Gaussians of fork
        #fork_index of the sketch's RngState (aero_set_rng_fill); None reverts."""
        if fn is None:
            self._rng_cb = None
            _chk(lib().aero_set_rng_fill(self._h, None, None))
            return

        def tramp(_ctx, fork, out, count):
            try:
                vals = np.asarray(fn(int(fork), int(count)), np.float64)
                if vals.shape != (count,):
                    return 1
                C.memmove(out, vals.ctypes.data, 8 * count)
                return 0
            except Exception:
                return 1

        self._rng_cb = RNG_FILL(tramp)  # kept alive as long as the sketch
        _chk(lib().aero_set_rng_fill(self._h, C.cast(self._rng_cb, vp), None))

    def update_block(self, rows, ts, thetas=None):
        """n sequential updates (sketch.cpp:82-141); returns the event log."""
        ts = np.ascontiguousarray(ts, np.int64)
        n = ts.shape[0]
        ev = (Event * max(n, 1))()
        th = _f64(thetas) if thetas is not None else None
        if hasattr(rows, "is_cuda") and rows.is_cuda:
            if rows.dim() != 2 or rows.shape[1] != self.d:
                raise InvalidInput("AeroState: row dimension mismatch")
            _check_block(rows.shape[0], n, th)
            ptr, ld = _device_ptr(rows, self.stream_handle())
            _chk(lib().aero_update_block_device(self._h, ptr, n, ld, _lp(ts), _dp(th), ev))
        else:
            rows = _f64(rows)
            if rows.ndim != 2 or rows.shape[1] != self.d:
                raise InvalidInput("AeroState: row dimension mismatch")
            _check_block(rows.shape[0], n, th)
            _chk(lib().aero_update_block(self._h, _dp(rows), n, self.d, _lp(ts), _dp(th), ev))
        return np.frombuffer(ev, dtype=EVENT_DTYPE, count=n).copy()

    def update(self, a, i):
        return self.update_block(np.asarray(a, np.float64)[None, :], [i])[0]

    def update_block_amplified(self, rows, ts, thetas=None):
        """n sequential update_amplified calls (sketch.cpp:45-48), host rows."""
        ts = np.ascontiguousarray(ts, np.int64)
        n = ts.shape[0]
        th = _f64(thetas) if thetas is not None else None
        rows = _f64(rows)
        if rows.ndim != 2 or rows.shape[1] != self.d:
            raise InvalidInput("AeroState: row dimension mismatch")
        _check_block(rows.shape[0], n, th)
        ev = (Event * max(n, 1))()
        _chk(lib().aero_update_block_amplified(self._h, _dp(rows), n, self.d, _lp(ts), _dp(th), ev))
        return np.frombuffer(ev, dtype=EVENT_DTYPE, count=n).copy()

    def update_amplified(self, a, i):
        return self.update_block_amplified(np.asarray(a, np.float64)[None, :], [i])[0]

    def query(self, lb, ub):
        out = np.empty((self.ell, self.d))
        _chk(lib().aero_query(self._h, lb, ub, _dp(out)))
        return out

    def set_grid_share(self, share):
        """Performance hint: `share` sketches run concurrently on this GPU."""
        _chk(lib().aero_set_grid_share(self._h, int(share)))

    def update_from_file(self, path, t0=None, chunk_rows=16384, want_log=False):
        """Stream an AERO file through the sketch (streams.cpp:105-137 format):
        row q gets timestamp t0 + q (default: clock + 1); the next chunk is
        read from disk while the current one is absorbed. Returns the events
        (want_log) or the row count."""
        t0 = self.clock + 1 if t0 is None else int(t0)
        cap = 0
        ev = None
        if want_log:
            with AeroFileReader(path) as f:
                cap = f.n_header or sum(1 for _ in f.chunks(65536)) * 65536
            ev = (Event * max(cap, 1))()
        got = i64()
        _chk(lib().aero_update_from_file(self._h, os.fsencode(path), t0, chunk_rows, ev, cap, C.byref(got)))
        if want_log:
            return np.frombuffer(ev, dtype=EVENT_DTYPE, count=got.value).copy()
        return got.value

    def query_gram(self, lb, ub):
        out = np.empty((self.d, self.d))
        _chk(lib().aero_query_gram(self._h, lb, ub, _dp(out)))
        return out

    def residual(self):
        r = self.info().rows
        out = np.empty((r, self.d))
        _chk(lib().aero_residual(self._h, _dp(out), r))
        return out

    def snap_count(self):
        n = i64()
        _chk(lib().aero_snap_count(self._h, C.byref(n)))
        return n.value

    def snaps(self):
        out = []
        for idx in range(self.snap_count()):
            xi, s, t, th = i32(), i64(), i64(), f64()
            _chk(lib().aero_snap_info(self._h, idx, C.byref(xi), C.byref(s), C.byref(t), C.byref(th)))
            z, m = np.empty((self.d, xi.value)), np.empty((xi.value, self.d))
            _chk(lib().aero_snap_get(self._h, idx, _dp(z), _dp(m)))
            out.append(dict(z=z, m=m, s=s.value, t=t.value, theta=th.value))
        return out

    def snap_meta(self):
        out = []
        for idx in range(self.snap_count()):
            xi, s, t, th = i32(), i64(), i64(), f64()
            _chk(lib().aero_snap_info(self._h, idx, C.byref(xi), C.byref(s), C.byref(t), C.byref(th)))
            out.append((xi.value, s.value, t.value, th.value))
        return out

    def snap_pop_front(self):
        _chk(lib().aero_snap_pop_front(self._h))

    def last_update_stats(self):
        ev = Event()
        _chk(lib().aero_last_stats(self._h, C.byref(ev)))
        return np.frombuffer(ev, dtype=EVENT_DTYPE, count=1)[0]

    def synchronize(self):
        _chk(lib().aero_synchronize(self._h))

    def stream_handle(self) -> int:
        return int(lib().aero_stream(self._h) or 0)

    def profile(self):
        p = Profile()
        _chk(lib().aero_get_profile(self._h, C.byref(p)))
        return {f: getattr(p, f) for f, _ in Profile._fields_}

    def reset_profile(self):
        _chk(lib().aero_reset_profile(self._h))


class AeroFileReader:
    """Chunked reader of an AERO stream file (reference load_stream with
    StreamFormat::Aero, streams.cpp:105-137): header validated on open,
    FormatError for truncated or non-finite rows."""

    def __init__(self, path):
        h, d, n = vp(), i32(), u64()
        _chk(lib().aero_file_open(os.fsencode(path), C.byref(h), C.byref(d), C.byref(n)))
        self._h, self.d, self.n_header = h, d.value, n.value

    def read(self, max_rows):
        out = np.empty((max(max_rows, 0), self.d))
        got = i64()
        _chk(lib().aero_file_read(self._h, _dp(out), max_rows, C.byref(got)))
        return out[:got.value]

    def chunks(self, rows=65536):
        while True:
            blk = self.read(rows)
            if blk.shape[0] == 0:
                return
            yield blk

    def close(self):
        if getattr(self, "_h", None):
            lib().aero_file_close(self._h)
        self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def read_aero(path):
    """All rows of an AERO file as an (n, d) array."""
    with AeroFileReader(path) as f:
        parts = list(f.chunks())
        return np.concatenate(parts) if parts else np.empty((0, f.d))


def write_aero(path, rows):
    """save_stream(..., StreamFormat::Aero) (streams.cpp:150-168)."""
    rows = _f64(rows)
    if rows.ndim != 2 or rows.shape[0] == 0:
        raise InvalidInput("save_stream: empty record set")
    _chk(lib().aero_file_write(os.fsencode(path), _dp(rows), rows.shape[0], rows.shape[1]))


class AttpState(AeroState):
    """reference AttpState (attp.hpp:15-43): theta = eps * running mass."""

    def __init__(self, d, eps, seed=0, stream=0, device=0, exact=False, max_batch=0, profile=False,
                 host_rng=False, delta=None):
        super().__init__(d, eps, 0.0, seed, stream, device, theta_mode=AERO_THETA_ATTP,
                         exact=exact, max_batch=max_batch, profile=profile, host_rng=host_rng, delta=delta)

    @property
    def inner(self):
        return self

    @property
    def fro_mass(self):
        return self.info().fro_mass

    def query(self, t, ub=None):  # AttpState::query(t); AeroState::query(lb, ub) if ub given
        if ub is not None:
            return AeroState.query(self, t, ub)
        out = np.empty((self.ell, self.d))
        _chk(lib().aero_attp_query(self._h, t, _dp(out)))
        return out


class MlState:
    """reference MlState (sliding_window.hpp:39-81)."""

    def __init__(self, d, n, r_max, eps, seed=0, stream=0, device=0, delta=None):
        h = vp()
        _chk(lib().aero_ml_create_amplified(d, n, r_max, eps, float(delta or 0.0), seed, stream, device,
                                            C.byref(h)))
        self._h, self.d, self.n = h, d, n
        inf = self.info()
        self.levels, self.ell = inf.levels, inf.ell

    def close(self):
        if getattr(self, "_h", None):
            lib().aero_ml_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def info(self):
        inf = MlInfo()
        _chk(lib().aero_ml_get_info(self._h, C.byref(inf)))
        return inf

    def theta(self, j):
        return lib().aero_ml_theta(self._h, j)

    def update_block(self, rows, ts):
        ts = np.ascontiguousarray(ts, np.int64)
        if hasattr(rows, "is_cuda") and rows.is_cuda:
            if rows.dim() != 2 or rows.shape[1] != self.d:
                raise InvalidInput("MlState: row dimension mismatch")
            _check_block(rows.shape[0], ts.shape[0])
            ptr, ld = _device_ptr(rows)
            _chk(lib().aero_ml_update_block_device(self._h, ptr, ts.shape[0], ld, _lp(ts)))
        else:
            rows = _f64(rows)
            if rows.ndim != 2 or rows.shape[1] != self.d:
                raise InvalidInput("MlState: row dimension mismatch")
            _check_block(rows.shape[0], ts.shape[0])
            _chk(lib().aero_ml_update_block(self._h, _dp(rows), rows.shape[0], self.d, _lp(ts)))

    def update(self, a, i):
        self.update_block(np.asarray(a, np.float64)[None, :], [i])

    def query(self):
        sk = np.empty((self.ell, self.d))
        r = MlQueryResult()
        _chk(lib().aero_ml_query(self._h, _dp(sk), C.byref(r)))
        return dict(sketch=sk, level=r.level, fallback=bool(r.fallback), xi_sum=r.xi_sum,
                    heavy_used=r.heavy_used)

    def level_state(self, j):
        h = lib().aero_ml_level(self._h, j)
        if not h:
            raise InvalidInput("MlState: level out of range")
        return AeroState(0, 0, _handle=vp(h), _owner=self)

    def heavy_count(self, j):
        n = i64()
        _chk(lib().aero_ml_heavy_count(self._h, j, C.byref(n)))
        return n.value

    def heavy(self, j):
        out = []
        for idx in range(self.heavy_count(j)):
            row, s, t = np.empty(self.d), i64(), i64()
            _chk(lib().aero_ml_heavy_get(self._h, j, idx, _dp(row), C.byref(s), C.byref(t)))
            out.append(dict(row=row, s=s.value, t=t.value))
        return out


class CodState:
    """reference CodState (amm.hpp:35-69): sliding-window AMM sketch."""

    def __init__(self, dx, dy, eps, theta, n, seed=0, stream=0, device=0):
        h = vp()
        _chk(lib().aero_cod_create(dx, dy, eps, theta, n, seed, stream, device, C.byref(h)))
        self._h, self.dx, self.dy = h, dx, dy
        self.ell = self.info()["ell"]

    def close(self):
        if getattr(self, "_h", None):
            lib().aero_cod_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def info(self):
        ell, cols, ns, clock = i32(), i64(), i64(), i64()
        _chk(lib().aero_cod_info(self._h, C.byref(ell), C.byref(cols), C.byref(ns), C.byref(clock)))
        return dict(ell=ell.value, cols=cols.value, nsnaps=ns.value, clock=clock.value)

    def update_block(self, xs, ys, ts):
        xs, ys = _f64(xs), _f64(ys)
        if xs.ndim != 2 or ys.ndim != 2 or xs.shape[1] != self.dx or ys.shape[1] != self.dy:
            raise InvalidInput("CodState: dimension mismatch")
        ts = np.ascontiguousarray(ts, np.int64)
        n = ts.shape[0]
        _check_block(xs.shape[0], n)
        _check_block(ys.shape[0], n)
        ev = (Event * max(n, 1))()
        _chk(lib().aero_cod_update_block(self._h, _dp(xs), _dp(ys), n, _lp(ts), ev))
        return np.frombuffer(ev, dtype=EVENT_DTYPE, count=n).copy()

    def update(self, x, y, i):
        return self.update_block(np.asarray(x, np.float64)[None], np.asarray(y, np.float64)[None], [i])[0]

    def query(self):
        a, b = np.empty((self.dx, self.ell)), np.empty((self.dy, self.ell))
        _chk(lib().aero_cod_query(self._h, _dp(a), _dp(b)))
        return a, b

    def query_product(self):
        p = np.empty((self.dx, self.dy))
        _chk(lib().aero_cod_query_product(self._h, _dp(p)))
        return p

    @property
    def theta(self):
        th = f64()
        _chk(lib().aero_cod_theta(self._h, C.byref(th)))
        return th.value

    def set_theta(self, theta):
        _chk(lib().aero_cod_set_theta(self._h, theta))


class AdaptiveState:
    """reference AdaptiveState (amm.hpp:71-93, amm.cpp:131-161): main/auxiliary
    CodState pair whose threshold doubles / halves with main's queue length;
    the auxiliary sketch, rebuilt from each window boundary, replaces the main
    one every n rows."""

    def __init__(self, dx, dy, eps, theta0, n, seed=0, stream=0, device=0):
        h = vp()
        _chk(lib().aero_adaptive_create(dx, dy, eps, theta0, n, seed, stream, device, C.byref(h)))
        self._h, self.dx, self.dy, self.ell = h, dx, dy, int(np.ceil(2.0 / eps))

    def close(self):
        if getattr(self, "_h", None):
            lib().aero_adaptive_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def info(self):
        lv, tm, ta, sm, sa = i32(), f64(), f64(), i64(), i64()
        _chk(lib().aero_adaptive_info(self._h, C.byref(lv), C.byref(tm), C.byref(ta), C.byref(sm), C.byref(sa)))
        return dict(level=lv.value, theta_main=tm.value, theta_aux=ta.value, snaps_main=sm.value,
                    snaps_aux=sa.value)

    @property
    def level(self):
        return self.info()["level"]

    def update_block(self, xs, ys, ts):
        """-> (main's per-row events, level() after each row)."""
        xs, ys = _f64(xs), _f64(ys)
        if xs.ndim != 2 or ys.ndim != 2 or xs.shape[1] != self.dx or ys.shape[1] != self.dy:
            raise InvalidInput("CodState: dimension mismatch")
        ts = np.ascontiguousarray(ts, np.int64)
        n = ts.shape[0]
        _check_block(xs.shape[0], n)
        _check_block(ys.shape[0], n)
        ev = (Event * max(n, 1))()
        lv = np.zeros(max(n, 1), np.int32)
        _chk(lib().aero_adaptive_update_block(self._h, _dp(xs), _dp(ys), n, _lp(ts), ev, lv.ctypes.data_as(P(i32))))
        return np.frombuffer(ev, dtype=EVENT_DTYPE, count=n).copy(), lv[:n].copy()

    def query(self):
        a, b = np.empty((self.dx, self.ell)), np.empty((self.dy, self.ell))
        _chk(lib().aero_adaptive_query(self._h, _dp(a), _dp(b)))
        return a, b

    def query_product(self):
        p = np.empty((self.dx, self.dy))
        _chk(lib().aero_adaptive_query_product(self._h, _dp(p)))
        return p


def dist_theta_schedule(sq_norms, eps, latency=0):
    """Per-site thresholds from the norm-only protocol replay
    (distributed.cpp:31-69,107-123,201-239). sq_norms: (m, T)."""
    sq = _f64(sq_norms)
    m, T = sq.shape
    th = np.empty_like(sq)
    mb, bc = i64(), i64()
    _chk(lib().aero_dist_theta_schedule(m, T, eps, latency, _dp(sq), _dp(th), C.byref(mb), C.byref(bc)))
    return th, mb.value, bc.value


class DistProtocol:
    """Streaming norm-only replay of the mass protocol (distributed.cpp:31-69,
    107-123, 201-239): per-site thresholds per tick; window > 0 = the
    sliding-window protocol (distributed.cpp:33-55)."""

    def __init__(self, m, eps, latency=0, window=0):
        h = vp()
        _chk(lib().aero_dist_protocol_create_window(m, eps, latency, window or 0, C.byref(h)))
        self._h, self.m = h, m

    def close(self):
        if getattr(self, "_h", None):
            lib().aero_dist_protocol_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def advance(self, sq_norms):
        sq = _f64(sq_norms)
        if sq.ndim != 2 or sq.shape[0] != self.m:
            raise InvalidInput("protocol: norms must be (m, T)")
        th = np.empty_like(sq)
        _chk(lib().aero_dist_protocol_advance(self._h, sq.shape[1], _dp(sq), _dp(th)))
        return th

    def info(self):
        t, b, bc, fh = i64(), i64(), i64(), f64()
        _chk(lib().aero_dist_protocol_info(self._h, C.byref(t), C.byref(b), C.byref(bc), C.byref(fh)))
        return dict(ticks=t.value, mass_bytes=b.value, broadcasts=bc.value, f_hat=fh.value)


def row_sq_norms_device(rows, device=0):
    """Squared row norms of a CUDA (n, d) float64 tensor (the K1 kernel)."""
    ptr, ld = _device_ptr(rows)
    out = np.empty(rows.shape[0])
    _chk(lib().aero_row_sq_norms_device(ptr, rows.shape[0], ld, rows.shape[1], device, _dp(out)))
    return out


class Coordinator:
    """reference CoordinatorState (distributed.hpp:78-105) as a device
    accumulator per rank, merged with ncclReduce at probe time."""

    def __init__(self, d, m, device=0, nccl_comm=None, window=0, latency=0):
        h = vp()
        _chk(lib().aero_coord_create_window(d, m, device, nccl_comm, window or 0, latency, C.byref(h)))
        self._h, self.d = h, d

    def close(self):
        if getattr(self, "_h", None):
            lib().aero_coord_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def absorb(self, site: AeroState) -> int:
        b = i64()
        _chk(lib().aero_coord_absorb_snapshots(self._h, site._h, C.byref(b)))
        return b.value

    def probe(self, sites, ell, root=0, want_gram=False):
        arr = (vp * max(len(sites), 1))(*[s._h for s in sites])
        out = np.empty((ell, self.d))
        gram = np.empty((self.d, self.d)) if want_gram else None
        _chk(lib().aero_coord_probe(self._h, arr, len(sites), root, ell, _dp(out), _dp(gram)))
        return out, gram

    def shrink(self, gram, ell):
        """shrink_to_sketch of a host-merged Gram on this coordinator's device."""
        g = _f64(gram)
        out = np.empty((ell, self.d))
        _chk(lib().aero_coord_shrink(self._h, _dp(g), ell, _dp(out)))
        return out


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _chk(lib().aero_nccl_get_unique_id(buf))
    return buf.raw


def nccl_comm_init(uid: bytes, nranks, rank, device):
    c = vp()
    _chk(lib().aero_nccl_comm_init(uid, nranks, rank, device, C.byref(c)))
    return c


def gen_rows_device(out, t0, d, k, rho, noise, r_max, seed, stream=0, drift=0, k2=0, rho2=0.9,
                    scale2=0.5, basis_stream=0, device=0):
    """Fill a CUDA float64 tensor (n, d) with rows t0..t0+n-1 of the config
    generator (DESIGN.md GENERATOR spec)."""
    p = GenParams(d=d, k=k, k2=k2, rho=rho, noise=noise, r_max=r_max, rho2=rho2, scale2=scale2,
                  seed=seed, stream=stream, basis_stream=basis_stream, drift_period=drift)
    _chk(lib().aero_gen_rows_device(C.byref(p), t0, out.shape[0], C.c_void_p(out.data_ptr()), device))
