"""Helpers mirroring the reference's tests/test_util.hpp:17-41 (seeded Gaussian
matrices from RngState(seed, stream), orthonormal bases, relative Frobenius)."""
import numpy as np


def gaussian(orc, rows, cols, seed, stream=0):
    return orc.rng_draw(seed, stream, 0, rows * cols).reshape(rows, cols)


def gaussian_vec(orc, n, seed, stream=0):
    return orc.rng_draw(seed, stream, 0, n)


def uniform_rows(orc, n, d, seed, stream=0):
    return orc.rng_draw(seed, stream, 0, n * d, "uniform").reshape(n, d)


def orthonormal(orc, d, k, seed):
    return orc.qr(gaussian(orc, d, k, seed))[0]


def rel_fro(got, want):
    den = np.linalg.norm(want)
    return np.linalg.norm(got - want) / den if den > 0 else np.linalg.norm(got - want)
