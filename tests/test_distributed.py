"""Multi-rank host logic on CPU (gloo, world size 2): nnz-balanced shards and the
one-allreduce-per-iteration exchange of exact int64 center sums.

The CUDA kernels are not run here (no GPU); each rank computes its local
fixed-point partial sums with numpy from its shard, exactly what
spkm_aggregate_sums / spkm_apply_moves produce, and the test checks that the
exchange turns them into the global sums bit-for-bit.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2107_04074_b200.distributed import Exchange, shard_rows

S_BITS = 40


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


def _fixed_sums(ip, idx, val, a, rows, k, d):
    sums = np.zeros((k, d), np.int64)
    counts = np.zeros(k, np.int64)
    for i in range(*rows):
        q = np.rint(val[ip[i]:ip[i + 1]].astype(np.float64) * 2.0 ** S_BITS).astype(np.int64)
        np.add.at(sums[a[i]], idx[ip[i]:ip[i + 1]], q)
        counts[a[i]] += 1
    return sums, counts


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        k, d = 5, 50
        ip, idx, val = _corpus()
        n = ip.size - 1
        g = np.random.default_rng(1)
        a0 = g.integers(0, k, n)
        rows = shard_rows(ip, world)[rank]
        ex = Exchange(k, d, torch.device("cpu"))
        # iteration 1: scratch sums from the local shard -> global
        s_loc, c_loc = _fixed_sums(ip, idx, val, a0, rows, k, d)
        sums = torch.from_numpy(s_loc.ravel().copy())
        counts = torch.from_numpy(c_loc.copy())
        ex.scratch(sums, counts)
        s_ref, c_ref = _fixed_sums(ip, idx, val, a0, (0, n), k, d)
        ok1 = np.array_equal(sums.numpy().reshape(k, d), s_ref) and np.array_equal(counts.numpy(), c_ref)
        # iteration 2: local moves -> delta buffer -> one allreduce
        a1 = a0.copy()
        flip = g.choice(n, 60, replace=False)
        a1[flip] = (a1[flip] + 1 + g.integers(0, k - 1, 60)) % k
        ex.begin()
        delta = ex.delta.numpy().reshape(k, d)
        dcounts = ex.dcounts.numpy()
        touched = torch.zeros(k, dtype=torch.int32)
        for i in range(*rows):
            if a1[i] != a0[i]:
                q = np.rint(val[ip[i]:ip[i + 1]].astype(np.float64) * 2.0 ** S_BITS).astype(np.int64)
                np.add.at(delta[a0[i]], idx[ip[i]:ip[i + 1]], -q)
                np.add.at(delta[a1[i]], idx[ip[i]:ip[i + 1]], q)
                dcounts[a0[i]] -= 1
                dcounts[a1[i]] += 1
                touched[a0[i]] = 1
                touched[a1[i]] = 1
        ctr = torch.zeros(8, dtype=torch.int64)
        ctr[2] = int(np.sum(a1[rows[0]:rows[1]] != a0[rows[0]:rows[1]]))
        ex.exchange(sums, counts, touched, ctr)
        s2, c2 = _fixed_sums(ip, idx, val, a1, (0, n), k, d)
        moved = np.nonzero(a1 != a0)[0]
        t_ref = np.zeros(k, np.int32)
        t_ref[a0[moved]] = 1
        t_ref[a1[moved]] = 1
        ok2 = (np.array_equal(sums.numpy().reshape(k, d), s2) and np.array_equal(counts.numpy(), c2)
               and np.array_equal(touched.numpy(), t_ref) and int(ctr[2]) == moved.size)
        # gather the sharded assignment vector
        a_full = ex.gather_assignments(torch.from_numpy(a1[rows[0]:rows[1]].astype(np.int32)), rows, n)
        ok3 = np.array_equal(a_full, a1)
        out[rank] = (ok1, ok2, ok3)
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
    assert shard_rows(np.array([0, 3]), 4)[-1] == (1, 1) or sum(r1 - r0 for r0, r1 in shard_rows(np.array([0, 3]), 4)) == 1


def test_exchange_world2_gloo():
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    assert dict(out) == {0: (True, True, True), 1: (True, True, True)}
