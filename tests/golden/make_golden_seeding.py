#!/usr/bin/env python3
"""Golden picks of the reference's k-means++ / AFK-MC2 seedings.

Runs the REFERENCE package (/root/reference/pkg/src/spkmeans, read only,
imported in place with a writable NUMBA_CACHE_DIR) on corpora already pinned
in this directory (ds_*.npz hold the rows exactly as the reference
normalised them; they are rebuilt with ``normalize_rows=False``) plus two
tiny corner corpora of the reference's tests (antipodal pair,
tests/test_seeding.py:14-16; three parallel rows, 104-110), and stores

  seeding.npz  kmpp__<ds>__<k>__<alpha>__<seed>            picks (int64)
               afk__<ds>__<k>__<alpha>__<chain>__<seed>    picks (int64)
               trace__<ds>__<k>__<alpha>__<seed>           kmpp weight vectors
                                                           (seeding.py:80-81)

Usage:  python tests/golden/make_golden_seeding.py
"""

import os
import sys
from pathlib import Path

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
REF = Path("/root/reference/pkg/src")
HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(REF))

import numpy as np  # noqa: E402

from spkmeans import seeding  # noqa: E402
from spkmeans.sparse import Dataset, SparseVector  # noqa: E402


def load(name):
    z = np.load(HERE / f"ds_{name}.npz")
    ip, ix, dv = z["indptr"], z["indices"], z["data"]
    rows = [SparseVector(ix[ip[i]:ip[i + 1]].astype(np.int64), dv[ip[i]:ip[i + 1]]) for i in range(ip.size - 1)]
    return Dataset.from_rows(rows, dim=int(z["dim"]), normalize_rows=False)


def sv(pairs):
    idx, val = zip(*pairs)
    return SparseVector(np.array(idx, dtype=np.int64), np.array(val, dtype=float))


def corner_sets():
    return {
        "antipodal": Dataset.from_rows([sv([(0, 1.0)]), sv([(0, -1.0)])], dim=2),
        "dup3": Dataset.from_rows([sv([(0, 2.0)]), sv([(0, 3.0)]), sv([(0, 4.0)])], dim=1),
    }


def main():
    out = {}
    sets = {name: load(name) for name in ("five_points", "small", "signed", "pitfall", "clustered", "C1",
                                          "grid_200_5000_50_1007")}
    sets.update(corner_sets())
    kmpp_cases = [
        ("antipodal", 2, 1.0, range(6)), ("dup3", 3, 1.0, [5, 6]), ("five_points", 5, 2.0, range(6)),
        ("five_points", 3, 1.0, [0, 1]), ("small", 8, 1.0, [0, 1, 2]), ("small", 6, 1.5, [77]),
        ("small", 40, 1.0, [3]), ("signed", 12, 1.2, [4]), ("pitfall", 5, 1.0, [1]),
        ("clustered", 20, 1.0, [3, 8]), ("C1", 20, 1.0, [1]), ("C1", 100, 1.5, [2]),
        ("grid_200_5000_50_1007", 50, 1.0, [7]), ("grid_200_5000_50_1007", 200, 1.0, [9]),
    ]
    for ds, k, alpha, seeds in kmpp_cases:
        for s in seeds:
            tr = [] if ds in ("small", "five_points", "antipodal", "dup3") and k <= 8 else None
            cs = seeding.init_kmpp(sets[ds], k, alpha=alpha, seed=s, trace=tr)
            out[f"kmpp__{ds}__{k}__{alpha}__{s}"] = np.asarray(cs.seed_indices, np.int64)
            if tr is not None and tr:
                out[f"trace__{ds}__{k}__{alpha}__{s}"] = np.stack(tr)
    afk_cases = [
        ("antipodal", 2, 1.0, 10, range(4)), ("five_points", 3, 1.0, 1, [9]), ("five_points", 4, 1.0, 5, range(8)),
        ("small", 6, 1.0, 50, [31]), ("small", 10, 1.5, 200, [2]), ("signed", 8, 1.0, 20, [3]),
        ("dup3", 3, 1.0, 10, [1, 2]), ("clustered", 20, 1.0, 200, [3]), ("C1", 20, 1.0, 100, [4]),
        ("C1", 60, 2.0, 30, [5]), ("grid_200_5000_50_1007", 100, 1.0, 20, [6]),
    ]
    for ds, k, alpha, chain, seeds in afk_cases:
        for s in seeds:
            cs = seeding.init_afkmc2(sets[ds], k, alpha=alpha, chain_length=chain, seed=s)
            out[f"afk__{ds}__{k}__{alpha}__{chain}__{s}"] = np.asarray(cs.seed_indices, np.int64)
    # the corner corpora's rows (the others live in ds_*.npz)
    for name, ds in corner_sets().items():
        m = ds.matrix
        out[f"corpus__{name}__indptr"] = m.indptr.astype(np.int64)
        out[f"corpus__{name}__indices"] = m.indices.astype(np.int32)
        out[f"corpus__{name}__data"] = m.data.astype(np.float64)
        out[f"corpus__{name}__dim"] = np.int64(ds.dim)
    np.savez_compressed(HERE / "seeding.npz", **out)
    print(f"seeding.npz: {sum(1 for k in out if k.startswith(('kmpp', 'afk')))} pick vectors")


if __name__ == "__main__":
    main()
