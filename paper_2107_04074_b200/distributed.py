"""Multi-GPU data parallelism: replicated corpus, sharded scans, one allgather of moves per iteration.

The reference is single-process.  Here every rank (one
process per GPU, ``torch.distributed`` over NCCL) holds the WHOLE corpus in
its HBM (C4: 2.9 GB of CSR incl. the float64 copy, out of 180 GB) together
with replicated centers, sums and counts, and owns a contiguous range of
device rows (rows are stored longest first; ranges are balanced by nnz) for
everything that scales with n x k: the full passes, the bound updates and
the pruned scans, with their bounds and worklists.

Per iteration the exchange is ONE allgather of fixed-size int32 move
slots (``spkm_pack_moves``) -- plus, for the variants with center-center
bounds (elkan, hamerly), one allreduce of the rank-sharded Gram partials of
the center thresholds (``Engine.center_thresholds``):

    slot = [ move count | 8 int64 counters | (global row, old, new) x cap ]

after which every rank applies all ranks' moves to its replicated int64
fixed-point sums (``spkm_apply_move_slots``).  Integer atomics are
order-free, so the sums, the centers and every later decision are
bit-identical on every rank and for every GPU count, and the payload is
12 bytes per moved point instead of the k x d sums (8 GB at C4) a sum
allreduce would move.  Iteration 1 (and the 50-iteration scratch rebuild)
allgathers the shard's assignments instead and aggregates the whole corpus
locally.  Convergence comes from the summed counters, so all ranks leave the
loop in the same iteration.  Collectives are issued on the engine's stream
with no host synchronisation.
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
    """One rank's view of the sharded fit: its device-row range and the
    per-iteration move allgather (plumbing over torch.distributed)."""

    def __init__(self, k: int, d: int, device, shards: list, group=None, slot_ints=None):
        self.k, self.d = k, d
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.shards = [tuple(map(int, s)) for s in shards]
        if len(self.shards) != self.world:
            raise ValueError("one shard per rank")
        self.p0, self.p1 = self.shards[self.rank]
        self.cap = max(max(p1 - p0 for p0, p1 in self.shards), 1)
        if slot_ints is None:
            from . import _lib
            slot_ints = int(_lib.lib().spkm_move_slot_ints(self.cap))
        self.slot_len = int(slot_ints)
        self.slot = torch.zeros(self.slot_len, dtype=torch.int32, device=device)
        self.slots = torch.zeros(self.world * self.slot_len, dtype=torch.int32, device=device)
        self.a_slot = torch.zeros(self.cap, dtype=torch.int32, device=device)
        self.a_all = torch.zeros(self.world * self.cap, dtype=torch.int32, device=device)
        self.bytes_per_iteration = self.slots.numel() * 4

    @classmethod
    def for_corpus(cls, k: int, corpus, device, group=None):
        """Shards = device-row ranges of the (replicated) corpus balanced by nnz."""
        world = dist.get_world_size(group)
        cache = corpus.__dict__.setdefault("_shards", {})
        if world not in cache:
            cache[world] = shard_rows(corpus.indptr.cpu().numpy(), world)
        return cls(k, corpus.d, device, cache[world], group)

    def allgather_moves(self):
        """slot (packed by spkm_pack_moves) -> every rank's slot in ``slots``."""
        dist.all_gather_into_tensor(self.slots, self.slot, group=self.group)

    def allreduce_sum(self, t: torch.Tensor):
        """In-place sum over the ranks (the center-threshold Gram partials:
        each element is nonzero on one rank, so the float sum is exact)."""
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)

    def allgather_assignments(self, a_local: torch.Tensor, a_global: torch.Tensor):
        """Shard assignments (device order) -> the global device-order array."""
        n_loc = self.p1 - self.p0
        self.a_slot[:n_loc].copy_(a_local[:n_loc])
        dist.all_gather_into_tensor(self.a_all, self.a_slot, group=self.group)
        for q, (p0, p1) in enumerate(self.shards):
            a_global[p0:p1].copy_(self.a_all[q * self.cap:q * self.cap + (p1 - p0)])


def run_sharded(data, k: int, variant: str, seeding=None, max_iter: int = 100, hamerly_update: str = "safe",
                device=None, group=None):
    """``engine.run`` on every rank of a torch.distributed group (one process
    per GPU): same arguments and result as ``run``, identical on all ranks."""
    from .engine import device_corpus, run
    device = torch.device(device or f"cuda:{torch.cuda.current_device()}")
    corpus = device_corpus(data, device)
    ex = Exchange.for_corpus(k, corpus, device, group)
    return run(data, k, variant, seeding=seeding, max_iter=max_iter, hamerly_update=hamerly_update, device=device,
               corpus=corpus, comm=ex, n_total=data.n)
