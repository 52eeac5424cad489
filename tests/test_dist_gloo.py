"""N>1 host path of the distributed sketch on CPU: world_size 2 over gloo.
Each rank holds only its own sites' rows; the ranks exchange squared norms and
replay the mass protocol. The per-site thresholds must equal the
single-process replay and the oracle simulator's trace bit for bit
(distributed.cpp:57-69, 107-123, 201-239)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

M, T, D, EPS, SEED = 4, 600, 8, 0.2, 3


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _streams():
    from oracle import pyoracle as orc
    return np.stack([orc.rng_draw(SEED, j, 0, T * D, "uniform").reshape(T, D) for j in range(M)])


def _worker(rank, world, port, outdir):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist
    from paper_2601_02019_b200.distributed import ThresholdExchange
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    streams = _streams()
    ex = ThresholdExchange(M, EPS, rank, world)
    thetas = []
    for b in range(0, T, 150):  # streamed in blocks
        local = {j: np.cumsum(streams[j, b:b + 150] ** 2, axis=1)[:, -1] for j in ex.local}
        thetas.append(ex.thresholds(local))
    np.save(os.path.join(outdir, f"theta_{rank}.npy"), np.concatenate(thetas, axis=1))
    np.save(os.path.join(outdir, f"meta_{rank}.npy"), np.array([ex.mass_bytes, ex.broadcasts]))
    dist.destroy_process_group()


def test_threshold_exchange_world2(tmp_path, orc):
    port = _free_port()
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    th0, th1 = np.load(tmp_path / "theta_0.npy"), np.load(tmp_path / "theta_1.npy")
    assert np.array_equal(th0, th1)  # every rank replays the same protocol
    streams = _streams()
    ref = orc.dist_run(streams, EPS, query_every=0, seed=SEED, want_thetas=True, probes=False)
    assert np.array_equal(th0, ref["thetas"])
    m0, m1 = np.load(tmp_path / "meta_0.npy"), np.load(tmp_path / "meta_1.npy")
    assert np.array_equal(m0, m1) and m0[1] == ref["broadcasts"]
    assert ref["comm_bytes"] - m0[0] >= 0  # remaining bytes are snapshot messages


def test_sites_partition():
    from paper_2601_02019_b200.distributed import sites_of
    for m in (1, 3, 8):
        for w in (1, 2, 4):
            got = sorted(j for r in range(w) for j in sites_of(r, w, m))
            assert got == list(range(m))


@pytest.mark.parametrize("window,latency", [(0, 2), (120, 0), (120, 3)])
def test_threshold_replay_window_and_latency(orc, window, latency):
    """The norm-only replay in sliding-window mode (distributed.cpp:33-55:
    exact window mass, signed deltas, the broadcast replaces the estimate) and
    with delivery latency (:226-239): thresholds bit-identical to the oracle
    simulator, broadcasts equal, mass bytes within its total."""
    from paper_2601_02019_b200.capi import DistProtocol
    streams = _streams()
    ref = orc.dist_run(streams, EPS, query_every=0, seed=SEED, want_thetas=True, probes=False,
                       window=window, latency=latency)
    p = DistProtocol(M, EPS, latency, window)
    sq = np.cumsum(streams ** 2, axis=-1)[..., -1]
    th = np.concatenate([p.advance(sq[:, b:b + 77]) for b in range(0, T, 77)], axis=1)
    assert np.array_equal(th, ref["thetas"])
    assert p.info()["broadcasts"] == ref["broadcasts"]
    assert 0 <= ref["comm_bytes"] - p.info()["mass_bytes"]
