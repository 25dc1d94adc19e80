"""Multi-GPU data parallelism: row shards, replicated centers, one allreduce per iteration.

The reference is single-process.  Here each rank (one
process per GPU, ``torch.distributed`` over NCCL) owns a contiguous row range
of the corpus balanced by nnz, its bounds and worklists; centers, sums and
counts are replicated.  Per iteration the only exchange is ONE allreduce(sum)
of an int64 buffer

    [ delta sums (k*d) | delta counts (k) | touched flags (k) | counters (8) ]

Sums are exact fixed point (int64), so the allreduce is exact and the
clustering is bit-identical for every GPU count.  Iteration 1 reduces the
from-scratch sums the same way.  Convergence is decided from the reduced
counters, so every rank leaves the loop in the same iteration.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def shard_rows(indptr: np.ndarray, world: int) -> list:
    """Contiguous row ranges [(r0, r1)] with near-equal nnz (and >= 0 rows each)."""
    indptr = np.asarray(indptr, dtype=np.int64)
    n = indptr.size - 1
    nnz = int(indptr[-1])
    cuts = [0]
    for q in range(1, world):
        target = nnz * q / world
        r = int(np.searchsorted(indptr, target, side="left"))
        r = min(max(r, cuts[-1]), n)
        cuts.append(r)
    cuts.append(n)
    return [(cuts[q], cuts[q + 1]) for q in range(world)]


class Exchange:
    """The per-iteration collective of one rank (plumbing over torch.distributed)."""

    def __init__(self, k: int, d: int, device, group=None):
        self.k, self.d = k, d
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        kd = k * d
        self.buf = torch.zeros(kd + 2 * k + 8, dtype=torch.int64, device=device)
        self.delta = self.buf[:kd]
        self.dcounts = self.buf[kd:kd + k]
        self.touched = self.buf[kd + k:kd + 2 * k]
        self.ctr = self.buf[kd + 2 * k:]
        self.bytes_per_iteration = self.buf.numel() * 8

    def _allreduce(self, t: torch.Tensor):
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)

    def scratch(self, sums: torch.Tensor, counts: torch.Tensor):
        """Iteration 1 / scratch rebuild: local sums+counts -> global (one allreduce)."""
        kd = self.k * self.d
        self.delta.copy_(sums)
        self.dcounts.copy_(counts)
        self._allreduce(self.buf[:kd + self.k])
        sums.copy_(self.delta)
        counts.copy_(self.dcounts)

    def begin(self):
        """Zero the delta section before the local move kernel writes into it."""
        self.buf[:self.k * self.d + self.k].zero_()

    def exchange(self, sums: torch.Tensor, counts: torch.Tensor, touched: torch.Tensor, ctr: torch.Tensor):
        """Allreduce [delta | dcounts | touched | ctr] and apply it (it >= 2)."""
        self.touched.copy_(touched)
        self.ctr.copy_(ctr)
        self._allreduce(self.buf)
        sums.add_(self.delta)
        counts.add_(self.dcounts)
        touched.copy_((self.touched > 0).to(touched.dtype))
        ctr.copy_(self.ctr)

    def gather_assignments(self, a_local: torch.Tensor, rows: tuple, n_total: int) -> np.ndarray:
        n_local = rows[1] - rows[0]
        sizes = torch.tensor([n_local], dtype=torch.int64, device=a_local.device)
        all_sizes = [torch.zeros_like(sizes) for _ in range(self.world)]
        dist.all_gather(all_sizes, sizes, group=self.group)
        m = int(max(int(s.item()) for s in all_sizes))
        pad = torch.full((max(m, 1),), -1, dtype=torch.int64, device=a_local.device)
        pad[:n_local] = a_local[:n_local].to(torch.int64)
        outs = [torch.zeros_like(pad) for _ in range(self.world)]
        dist.all_gather(outs, pad, group=self.group)
        parts = [o[:int(s.item())].cpu().numpy() for o, s in zip(outs, all_sizes)]
        a = np.concatenate(parts) if parts else np.zeros(0, np.int64)
        assert a.size == n_total
        return a


def run_sharded(data, k: int, variant: str, seeding=None, max_iter: int = 100, hamerly_update: str = "safe",
                device=None, group=None):
    """``engine.run`` on this rank's nnz-balanced shard (call on every rank)."""
    from .engine import DeviceCorpus, run
    from .seeding import SeedConfig, make_centroids

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    r0, r1 = shard_rows(data.indptr, world)[rank]
    device = torch.device(device or f"cuda:{torch.cuda.current_device()}")
    corpus = DeviceCorpus(data, device, rows=(r0, r1))
    cents0 = make_centroids(data, k, seeding if seeding is not None else SeedConfig())
    ex = Exchange(k, data.dim, device, group)
    return run(data, k, variant, max_iter=max_iter, hamerly_update=hamerly_update, device=device,
               corpus=corpus, init_centers=cents0.centers, comm=ex, n_total=data.n,
               seed_indices=cents0.seed_indices)
