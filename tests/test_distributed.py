"""Multi-rank host logic on CPU (gloo, world size 2): nnz-balanced device-row
shards and the one-allgather-per-iteration move exchange (distributed.py).

The CUDA kernels are not run here (no GPU).  Each rank emulates, with numpy,
exactly what its kernels do around the collectives -- spkm_pack_moves (slot =
[count, 0, 8 int64 counters, (global row, old, new) x cap]) and
spkm_apply_move_slots (every rank's moves into the replicated fixed-point
sums, counters summed) -- and the test checks that after the exchange every
rank holds the single-process sums, counts, touched set and counters
bit-for-bit, and that the assignment allgather rebuilds the global array.
"""

import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2107_04074_b200.distributed import Exchange, shard_rows

S_BITS = 40
HEAD = 2 + 16


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _corpus(n=400, d=50, seed=0):
    g = np.random.default_rng(seed)
    lens = g.integers(1, 12, n)
    ip = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    idx = np.concatenate([np.sort(g.choice(d, L, replace=False)) for L in lens]).astype(np.int32)
    val = g.uniform(0.05, 1.0, idx.size).astype(np.float32)
    return ip, idx, val


def _fixed(val):
    return np.rint(val.astype(np.float64) * 2.0 ** S_BITS).astype(np.int64)


def _fixed_sums(ip, idx, val, a, k, d):
    sums = np.zeros((k, d), np.int64)
    counts = np.zeros(k, np.int64)
    for i in range(ip.size - 1):
        np.add.at(sums[a[i]], idx[ip[i]:ip[i + 1]], _fixed(val[ip[i]:ip[i + 1]]))
        counts[a[i]] += 1
    return sums, counts


def _pack(slot, moves, ctr, p0):
    """spkm_pack_moves: moves = [(local row, old, new)]."""
    s = slot.numpy()
    s[0] = len(moves)
    s[1] = 0
    s[2:HEAD] = np.asarray(ctr, np.int64).view(np.int32)
    for m, (i, o, nw) in enumerate(moves):
        s[HEAD + 3 * m:HEAD + 3 * m + 3] = (p0 + i, o, nw)


def _apply(slots, world, slot_len, ip, idx, val, sums, counts, touched):
    """spkm_apply_move_slots."""
    s = slots.numpy()
    ctr = np.zeros(8, np.int64)
    for q in range(world):
        sl = s[q * slot_len:(q + 1) * slot_len]
        for m in range(int(sl[0])):
            i, o, nw = (int(x) for x in sl[HEAD + 3 * m:HEAD + 3 * m + 3])
            f = _fixed(val[ip[i]:ip[i + 1]])
            np.add.at(sums[o], idx[ip[i]:ip[i + 1]], -f)
            np.add.at(sums[nw], idx[ip[i]:ip[i + 1]], f)
            counts[o] -= 1
            counts[nw] += 1
            touched[o] = touched[nw] = 1
        ctr += sl[2:HEAD].copy().view(np.int64)
    return ctr


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        k, d = 5, 50
        ip, idx, val = _corpus()          # the replicated corpus (device row order)
        n = ip.size - 1
        g = np.random.default_rng(1)
        a0 = g.integers(0, k, n).astype(np.int32)
        shards = shard_rows(ip, world)
        ex = Exchange(k, d, torch.device("cpu"), shards, slot_ints=HEAD + 3 * max(p1 - p0 for p0, p1 in shards))
        p0, p1 = ex.p0, ex.p1
        # iteration 1: allgather the shard assignments, aggregate the whole corpus
        a_glob = torch.zeros(n, dtype=torch.int32)
        ex.allgather_assignments(torch.from_numpy(a0[p0:p1].copy()), a_glob)
        ok1 = np.array_equal(a_glob.numpy(), a0)
        sums, counts = _fixed_sums(ip, idx, val, a_glob.numpy(), k, d)
        # iteration 2: local scan moves -> slot -> allgather -> apply all
        a1 = a0.copy()
        flip = g.choice(n, 60, replace=False)
        a1[flip] = (a1[flip] + 1 + g.integers(0, k - 1, 60)) % k
        moves = [(i - p0, int(a0[i]), int(a1[i])) for i in range(p0, p1) if a1[i] != a0[i]]
        ctr = np.zeros(8, np.int64)
        ctr[2] = len(moves)
        ctr[3] = 1000 * (rank + 1)        # e.g. the sims counter
        _pack(ex.slot, moves, ctr, p0)
        ex.allgather_moves()
        touched = np.zeros(k, np.int32)
        ctr_all = _apply(ex.slots, ex.world, ex.slot_len, ip, idx, val, sums, counts, touched)
        s2, c2 = _fixed_sums(ip, idx, val, a1, k, d)
        moved = np.nonzero(a1 != a0)[0]
        t_ref = np.zeros(k, np.int32)
        t_ref[a0[moved]] = 1
        t_ref[a1[moved]] = 1
        ok2 = (np.array_equal(sums, s2) and np.array_equal(counts, c2) and np.array_equal(touched, t_ref)
               and int(ctr_all[2]) == moved.size and int(ctr_all[3]) == sum(1000 * (r + 1) for r in range(world)))
        out[rank] = (ok1, ok2, ex.bytes_per_iteration)
    finally:
        dist.destroy_process_group()


def test_shard_rows_balanced_by_nnz():
    ip, _, _ = _corpus(n=1000)
    for world in (1, 2, 4, 8):
        sh = shard_rows(ip, world)
        assert sh[0][0] == 0 and sh[-1][1] == ip.size - 1
        assert all(sh[q][1] == sh[q + 1][0] for q in range(world - 1))
        nnz = [ip[r1] - ip[r0] for r0, r1 in sh]
        assert max(nnz) - min(nnz) <= 2 * 12      # within two rows of perfect balance
    assert sum(r1 - r0 for r0, r1 in shard_rows(np.array([0, 3]), 4)) == 1


def test_move_exchange_world2_gloo():
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    res = dict(out)
    assert {r: v[:2] for r, v in res.items()} == {0: (True, True), 1: (True, True)}
    # payload: 12 bytes per shard row per rank (+ header), independent of k and d
    assert res[0][2] == 2 * 4 * (HEAD + 3 * 200) or res[0][2] < 2 * 4 * (HEAD + 3 * 400)
