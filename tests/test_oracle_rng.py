"""Pins the oracle's RngState restatement bit-for-bit against golden vectors
generated from the REFERENCE's own rng.hpp (oracle/ref_rng_golden.cpp,
oracle/make_golden.sh -> tests/golden/rng_golden.json)."""
import json
import os
import struct

import numpy as np

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "rng_golden.json")


def _bits(x):
    return format(struct.unpack("<Q", struct.pack("<d", float(x)))[0], "016x")


def test_rng_golden_vectors(orc):
    cases = json.load(open(GOLDEN))["cases"]
    assert len(cases) >= 10
    for c in cases:
        if c["kind"] == 2:
            continue
        kind = "gaussian" if c["kind"] == 0 else "uniform"
        got = orc.rng_draw(int(c["seed"]), int(c["stream"]), c["fork"], len(c["bits"]), kind)
        assert [_bits(v) for v in got] == c["bits"], c


def test_rng_prefix_property(orc):
    # the first r draws of a fork do not depend on how many are requested
    a = orc.rng_draw(1, 1000, 3, 101)
    b = orc.rng_draw(1, 1000, 3, 40)
    assert np.array_equal(a[:40], b)
