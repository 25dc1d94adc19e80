"""Multi-rank fit on ONE GPU: W ranks as W host threads, each with its own
engine (own stream, own bound/worklist state, its nnz-balanced shard of the
replicated corpus), exchanging the packed move slots through device copies.

This runs the real multi-GPU kernels -- ``spkm_pack_moves`` and
``spkm_apply_move_slots`` with world > 1, the sharded row ranges, the shard
assignment allgather of iteration 1 -- which a one-rank NCCL group cannot
exercise (its collectives are trivial).  No kernel waits on another rank:
the exchange is host-synchronous (each rank syncs its stream, a host barrier,
then every rank copies all slots on its own stream), so there is no device
spin and nothing relies on two launches being co-resident
(B200_PROFILING.md, "kernels that wait on one another").

Contract checked: the W-rank fit equals the single-process fit bit for bit
(assignments, objective, per-iteration reassignments and sims, centers),
which is what the exact int64 fixed-point sums promise for any GPU count
(distributed.py).
"""

import threading

import numpy as np
import pytest
import torch

from conftest import golden_dataset, load_golden

pytestmark = pytest.mark.gpu


class _Group:
    def __init__(self, world):
        self.world = world
        self.barrier = threading.Barrier(world)
        self.bufs = [None] * world


class LoopbackExchange:
    """distributed.Exchange's interface, ranks = threads on one device."""

    def __init__(self, group, rank, k, d, device, shards):
        from paper_2107_04074_b200 import _lib
        self.g, self.rank, self.world = group, rank, group.world
        self.k, self.d = k, d
        self.shards = [tuple(map(int, s)) for s in shards]
        self.p0, self.p1 = self.shards[rank]
        self.cap = max(max(p1 - p0 for p0, p1 in self.shards), 1)
        self.slot_len = int(_lib.lib().spkm_move_slot_ints(self.cap))
        self.slot = torch.zeros(self.slot_len, dtype=torch.int32, device=device)
        self.slots = torch.zeros(self.world * self.slot_len, dtype=torch.int32, device=device)
        self.a_slot = torch.zeros(self.cap, dtype=torch.int32, device=device)
        self.a_all = torch.zeros(self.world * self.cap, dtype=torch.int32, device=device)
        self.bytes_per_iteration = self.slots.numel() * 4
        self.calls = 0

    def _allgather(self, mine, out, L):
        s = torch.cuda.current_stream()        # the engine's stream (callers enter it)
        s.synchronize()
        self.g.bufs[self.rank] = mine
        self.g.barrier.wait()
        for q in range(self.world):
            out[q * L:(q + 1) * L].copy_(self.g.bufs[q])
        s.synchronize()
        self.g.barrier.wait()                  # nobody rewrites its buffer before all have copied
        self.calls += 1

    def allreduce_sum(self, t):
        s = torch.cuda.current_stream()
        s.synchronize()
        self.g.bufs[self.rank] = t.clone()
        self.g.barrier.wait()
        acc = torch.zeros_like(t)
        for q in range(self.world):
            acc += self.g.bufs[q]
        t.copy_(acc)
        s.synchronize()
        self.g.barrier.wait()
        self.calls += 1

    def allgather_moves(self):
        self._allgather(self.slot, self.slots, self.slot_len)

    def allgather_assignments(self, a_local, a_global):
        n_loc = self.p1 - self.p0
        self.a_slot[:n_loc].copy_(a_local[:n_loc])
        self._allgather(self.a_slot, self.a_all, self.cap)
        for q, (p0, p1) in enumerate(self.shards):
            a_global[p0:p1].copy_(self.a_all[q * self.cap:q * self.cap + (p1 - p0)])


def _fit_ranks(data, k, variant, world, seed, max_iter):
    import paper_2107_04074_b200 as spk
    from paper_2107_04074_b200.distributed import shard_rows
    from paper_2107_04074_b200.engine import device_corpus
    dev = torch.device("cuda:0")
    corpus = device_corpus(data, dev)
    shards = shard_rows(corpus.indptr.cpu().numpy(), world)
    corpus.seed_struct(data)       # shared seeding buffers, built once before the ranks start
    g = _Group(world)
    out, err = [None] * world, [None] * world

    def rank(q):
        try:
            torch.cuda.set_device(dev)
            ex = LoopbackExchange(g, q, k, data.dim, dev, shards)
            out[q] = (spk.run(data, k, variant, spk.SeedConfig(seed=seed), max_iter=max_iter, device=dev,
                              corpus=corpus, comm=ex, n_total=data.n), ex)
        except BaseException as e:     # noqa: BLE001 -- surfaced below
            err[q] = e
            g.barrier.abort()

    th = [threading.Thread(target=rank, args=(q,)) for q in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    for e in err:
        if e is not None and not isinstance(e, threading.BrokenBarrierError):
            raise e
    assert all(o is not None for o in out), err
    return out, shards


def _corpus(name):
    if name == "C1":
        return golden_dataset(load_golden("C1")), 20
    from paper_2107_04074_b200 import synth
    return synth.config_dataset("C3", n_override=20_000), 50


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("variant", ["standard", "elkan", "simp_elkan", "hamerly", "simp_hamerly"])
@pytest.mark.parametrize("corpus", ["C1", "C3s"])
def test_loopback_ranks_equal_single_process(corpus, variant, world):
    import paper_2107_04074_b200 as spk
    data, k = _corpus(corpus)
    ref = spk.run(data, k, variant, spk.SeedConfig(seed=5), max_iter=40, use_graphs=False)
    out, shards = _fit_ranks(data, k, variant, world, 5, 40)
    assert len(shards) == world and all(p1 > p0 for p0, p1 in shards)
    for r, ex in out:
        assert np.array_equal(r.assignments, ref.assignments), variant
        assert r.objective == ref.objective
        assert [s.reassignments for s in r.iterations] == [s.reassignments for s in ref.iterations]
        assert [s.sim_count for s in r.iterations] == [s.sim_count for s in ref.iterations]
        assert np.array_equal(r.centers.centers, ref.centers.centers)
        assert np.array_equal(r.centers.counts, ref.centers.counts)
        assert ex.calls >= len(r.iterations)      # one move exchange per iteration >= 2, plus the assignments


@pytest.mark.parametrize("variant", ["elkan", "hamerly"])
def test_loopback_sharded_thresholds_multi_tile(variant):
    """k = 300: 3 x 3 Gram tiles, so the (tile, d-split) CTAs of the center
    thresholds are really dealt across the 3 ranks (spkm_gram_partial) and
    summed by the allreduce; the fit equals the single-process one."""
    import paper_2107_04074_b200 as spk
    from paper_2107_04074_b200 import synth
    data = synth.config_dataset("C3", n_override=20_000)
    ref = spk.run(data, 300, variant, spk.SeedConfig(seed=5), max_iter=25, use_graphs=False)
    out, _ = _fit_ranks(data, 300, variant, 3, 5, 25)
    for r, ex in out:
        assert np.array_equal(r.assignments, ref.assignments)
        assert r.objective == ref.objective
        assert [s.sim_count for s in r.iterations] == [s.sim_count for s in ref.iterations]
        assert ex.calls >= 2 * len(r.iterations) - 1      # moves + Gram partials every iteration >= 2
