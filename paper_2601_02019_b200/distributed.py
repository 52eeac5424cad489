"""Distributed sketch: sites -> coordinator merge, one process per GPU.

Reference: SiteState / CoordinatorState / run_simulation
(/root/reference/proj/include/aero/distributed.hpp:23-135,
 /root/reference/proj/src/distributed.cpp:16-269). The reference simulates all
m sites and the coordinator in one thread over FIFO deques. Here:

* every rank hosts the sites j with j % world == rank (one site per GPU when
  m == world), each a device AeroState on its own stream;
* the only protocol state that couples sites -- the FroMass / broadcast mass
  estimate that sets each site's threshold (distributed.cpp:57-69, 107-123)
  -- depends on squared row norms alone, so ranks all-gather the norms of a
  block (m x T doubles) and every rank replays the protocol identically
  (ThresholdExchange); no per-row communication;
* snapshots are absorbed into a per-rank device accumulator
  (CoordinatorState::receive, distributed.cpp:124-136) and merged with one
  ncclReduce of the d x d fp64 Gram per probe (probe_gram, :159-173).

Protocol bytes (Message::bytes, distributed.hpp:33-42) are accounted exactly:
mass messages and broadcasts from the replay, snapshot messages at absorb.
"""
from __future__ import annotations

import numpy as np

from .capi import AeroState, Coordinator, DistProtocol, nccl_comm_init, nccl_unique_id, row_sq_norms_device

SKETCH_STREAM_BASE = 1000  # kSketchStreamBase (distributed.hpp:135)


def sites_of(rank: int, world: int, m: int) -> list[int]:
    return [j for j in range(m) if j % world == rank]


class ThresholdExchange:
    """All-gather of per-site squared norms + deterministic protocol replay.
    Host-only (works with gloo or nccl process groups)."""

    def __init__(self, m: int, eps: float, rank: int = 0, world: int = 1, group=None, latency: int = 0,
                 window: int = 0):
        self.m, self.eps, self.rank, self.world, self.group = m, eps, rank, world, group
        self.local = sites_of(rank, world, m)
        self.proto = DistProtocol(m, eps, latency, window)

    def gather(self, local_norms: dict[int, np.ndarray]) -> np.ndarray:
        T = len(next(iter(local_norms.values()))) if local_norms else 0
        if self.world == 1:
            full = np.zeros((self.m, T))
            for j, v in local_norms.items():
                full[j] = v
            return full
        import torch
        import torch.distributed as dist
        mine = torch.zeros((self.m, T), dtype=torch.float64)
        for j, v in local_norms.items():
            mine[j] = torch.from_numpy(np.asarray(v, np.float64))
        backend = dist.get_backend(self.group)
        if backend == "nccl":
            mine = mine.cuda()
        # sites are disjoint across ranks: a sum all-reduce assembles the matrix
        dist.all_reduce(mine, op=dist.ReduceOp.SUM, group=self.group)
        return mine.cpu().numpy()

    def thresholds(self, local_norms: dict[int, np.ndarray]) -> np.ndarray:
        """theta (m x T) for the next T ticks, identical on every rank."""
        return self.proto.advance(self.gather(local_norms))

    @property
    def mass_bytes(self) -> int:
        return self.proto.info()["mass_bytes"]

    @property
    def broadcasts(self) -> int:
        return self.proto.info()["broadcasts"]


class DistributedSketch:
    """The sites hosted by this rank plus its share of the coordinator."""

    def __init__(self, d: int, eps: float, m: int, seed: int = 0, rank: int = 0, world: int = 1,
                 group=None, device: int = 0, use_nccl: bool | None = None, latency: int = 0,
                 window: int = 0):
        """window > 0: the sliding-window protocol (SiteState with a window,
        distributed.cpp:33-55, 87-97; CoordinatorState(window_mode=true),
        :137-144)."""
        self.d, self.eps, self.m, self.rank, self.world, self.device = d, eps, m, rank, world, device
        self.window = window or 0
        self.exchange = ThresholdExchange(m, eps, rank, world, group, latency, self.window)
        self.sites = {j: AeroState(d, eps, 0.0, seed=seed, stream=SKETCH_STREAM_BASE + j, device=device)
                      for j in self.exchange.local}
        if len(self.sites) > 1:  # co-hosted sites run concurrently: share the GPU's CTAs
            for s in self.sites.values():
                s.set_grid_share(len(self.sites))
        self.ell = next(iter(self.sites.values())).ell if self.sites else int(np.ceil(2.0 / eps))
        self._comm = None
        if use_nccl is None:
            use_nccl = world > 1
        if use_nccl:
            self._comm = self._nccl_comm(group)
        self.coord = Coordinator(d, m, device, self._comm, window=self.window, latency=latency)
        self.snapshot_bytes = 0
        self.clock = 0
        self._pool = None

    def _nccl_comm(self, group):
        import torch
        import torch.distributed as dist
        uid = nccl_unique_id() if self.rank == 0 else bytes(128)
        if self.world > 1:
            t = torch.tensor(list(uid), dtype=torch.uint8)
            if dist.get_backend(group) == "nccl":
                t = t.cuda()
            dist.broadcast(t, src=0, group=group)
            uid = bytes(t.cpu().tolist())
        return nccl_comm_init(uid, self.world, self.rank, self.device)

    def ingest(self, rows_by_site: dict, t0: int) -> None:
        """Feed ticks t0 .. t0+T-1 to the local sites (rows: (T, d) host arrays
        or CUDA float64 tensors)."""
        norms = {}
        rows_by_site = dict(rows_by_site)
        for j, rows in rows_by_site.items():
            if not (hasattr(rows, "is_cuda") and rows.is_cuda):
                # host rows: one H2D (asynchronous from pinned memory), then the
                # same device path -- norms by the ingestion kernel (K1)
                import torch
                t = torch.from_numpy(np.ascontiguousarray(rows, np.float64))
                rows_by_site[j] = t.to(torch.device("cuda", self.device), non_blocking=t.is_pinned())
            norms[j] = row_sq_norms_device(rows_by_site[j], self.device)
        theta = self.exchange.thresholds(norms)
        T = theta.shape[1]
        ts = np.arange(t0, t0 + T, dtype=np.int64)
        items = list(rows_by_site.items())
        if len(items) > 1:
            # several sites on this GPU: each is its own device state and
            # stream, so their update blocks run concurrently (the C-ABI call
            # releases the GIL); absorbs stay serial (one accumulator)
            if self._pool is None:
                from concurrent.futures import ThreadPoolExecutor
                self._pool = ThreadPoolExecutor(max_workers=len(self.sites))
            futs = [self._pool.submit(self.sites[j].update_block, rows, ts, thetas=theta[j]) for j, rows in items]
            for f in futs:
                f.result()
        else:
            for j, rows in items:
                self.sites[j].update_block(rows, ts, thetas=theta[j])
        for j, _ in items:
            self.snapshot_bytes += self.coord.absorb(self.sites[j])
        self.clock = t0 + T - 1

    def probe(self, want_gram: bool = False, root: int = 0, group=None):
        """Merged sketch (ell x d) and optionally the d x d Gram on `root`.

        With an NCCL communicator the per-rank Grams meet in one ncclReduce
        inside the library. Over a process group without NCCL (gloo, e.g.
        ranks sharing a GPU or a host-side test harness) each rank's Gram is
        summed with torch.distributed.reduce and the root shrinks it on its
        device; either way the merge is probe_gram (distributed.cpp:159-173)."""
        sites = list(self.sites.values())
        if self.world == 1 or self._comm is not None:
            return self.coord.probe(sites, self.ell, root=root, want_gram=want_gram)
        import torch
        import torch.distributed as dist
        _, g = self.coord.probe(sites, 0, root=0, want_gram=True)  # this rank only (no comm)
        t = torch.from_numpy(g)
        dist.reduce(t, dst=root, op=dist.ReduceOp.SUM, group=group)
        if self.rank != root:
            return None, None
        g = t.numpy()
        return self.coord.shrink(g, self.ell), (g if want_gram else None)

    def comm_bytes_local(self) -> int:
        """SnapshotUpdate (and, window mode, Expire) message bytes shipped by
        this rank's sites."""
        return self.snapshot_bytes
