"""The library's host RngState restatement (AERO_FLAG_HOST_RNG panels,
rng_panels.cu host_gaussian_at) against the golden vectors compiled from the
REFERENCE's own rng.hpp (tests/golden/rng_golden.json) and against the
oracle's draws, bit for bit. Needs no GPU: the draws are host code of the
product library."""
import json
import os
import struct

import numpy as np

import paper_2601_02019_b200 as prod

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "rng_golden.json")


def _bits(x):
    return format(struct.unpack("<Q", struct.pack("<d", float(x)))[0], "016x")


def test_host_draws_match_reference_golden_vectors():
    cases = [c for c in json.load(open(GOLDEN))["cases"] if c["kind"] == 0]
    assert len(cases) >= 6
    for c in cases:
        got = prod.rng_gaussians_host(int(c["seed"]), int(c["stream"]), c["fork"], len(c["bits"]))
        assert [_bits(v) for v in got] == c["bits"], c


def test_host_draws_match_oracle_bitwise(orc):
    # forks and lengths of the C2 gate / simul_iter panels (r up to 2047, k=2)
    for seed, stream, fork, n in ((1, 1000, 1, 2047), (1, 1000, 4097, 4094), (2, 1000, 123456, 4095),
                                  (1, 2 ** 40 + 3, 77, 1001)):
        a = prod.rng_gaussians_host(seed, stream, fork, n)
        b = orc.rng_draw(seed, stream, fork, n)
        assert np.array_equal(a.view(np.uint64), b.view(np.uint64)), (seed, stream, fork)
