"""CPU-side checks of the product boundary: the C-ABI library loads, exports
every symbol include/aero_b200.h declares, fails loudly without a GPU, and its
pure-host protocol logic (norm-only replay of the distributed mass protocol)
is bit-exact against the oracle."""
import re

import numpy as np
import pytest

import paper_2601_02019_b200 as prod
from paper_2601_02019_b200 import capi


def _declared_functions():
    text = open(capi.HEADER_PATH).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    names = re.findall(r"\b(aero_[a-z0-9_]+)\s*\(", text)
    return sorted(set(names))


def test_library_exports_every_declared_symbol():
    L = prod.lib()
    declared = _declared_functions()
    assert len(declared) >= 40
    missing = [n for n in declared if not hasattr(L, n)]
    assert not missing, missing
    bound = {name for name, _, _ in capi.SIGNATURES}
    assert set(declared) == bound, set(declared) ^ bound


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(prod.CudaError):
        prod.AeroState(8, 0.5)
    with pytest.raises(prod.CudaError):
        prod.MlState(8, 100, 8.0, 0.5)


def _seq_sq_norms(x):
    # sequential accumulation, same order as the oracle's sq_norm
    return np.cumsum(x * x, axis=-1)[..., -1]


@pytest.mark.parametrize("m,T,eps,latency", [(1, 300, 0.25, 0), (2, 200, 0.5, 0), (4, 1500, 0.2, 0),
                                             (3, 400, 0.3, 2)])
def test_dist_theta_schedule_bit_exact(orc, m, T, eps, latency):
    from refutil import uniform_rows
    d = 8
    streams = np.stack([uniform_rows(orc, T, d, 3, j) for j in range(m)])
    ref = orc.dist_run(streams, eps, query_every=0, latency=latency, seed=3, want_thetas=True,
                       probes=False)
    th, mass_bytes, bc = prod.dist_theta_schedule(_seq_sq_norms(streams), eps, latency)
    assert np.array_equal(th, ref["thetas"])
    assert bc == ref["broadcasts"]
    # protocol bytes: mass messages + broadcasts here, snapshot bytes at the coordinator
    snap_bytes = ref["comm_bytes"] - mass_bytes
    assert snap_bytes >= 0 and snap_bytes % 8 == 0


def test_dist_theta_rejects_bad_config():
    with pytest.raises(prod.InvalidInput):
        prod.dist_theta_schedule(np.ones((0, 3)), 0.5)
    with pytest.raises(prod.InvalidInput):
        prod.dist_theta_schedule(np.ones((2, 3)), 1.5)


def test_events_layout_matches_oracle(orc):
    assert capi.EVENT_DTYPE == orc.EVENT_DTYPE
