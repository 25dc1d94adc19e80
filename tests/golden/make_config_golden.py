#!/usr/bin/env python3
"""Golden results of the float64 CPU oracle on the BASELINE configs C3, C4 (row
subsample) and C5 (row subsample) -- TEST INFRASTRUCTURE ONLY.

The oracle (oracle/spkm_oracle.c, a restatement of the reference loop
engine.py:201-346 + kernels.py:14-113, pinned bit-exactly to the reference's
own runs by tests/test_oracle.py) needs minutes and tens of GB of host RAM at
these sizes (C4: k x d float64 centers, sums, prev and the transposed copy are
8 GB each), so its results are computed once here and committed as small
fixtures; tests/test_gpu_config_parity.py compares the GPU fits with them.

Inputs are regenerated from the seeded generator (paper_2107_04074_b200/synth.py,
numpy PCG64: machine independent); each fixture stores a SHA-256 of the
normalised CSR so the test fails loudly if the generator's output differs.

Stored per case: oracle assignments (int16), packbits(best - second > 1e-5)
over the final centers, per-iteration objective / reassignments / sims,
iteration count, and the CSR digest.

usage: python tests/golden/make_config_golden.py [C3 C4s C5s ...]
"""

from __future__ import annotations

import hashlib
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))

# name -> (config, n_override, k, seed, max_iter)
CASES = {
    "C3": ("C3", None, 200, 2, 50),
    "C4s": ("C4", 250_000, 1000, 2, 50),
    "C5s": ("C5", 100_000, 1000, 5, 50),
}
MARGIN = 1e-5


def digest(ds) -> str:
    h = hashlib.sha256()
    for a in (np.ascontiguousarray(ds.indptr, np.int64), np.ascontiguousarray(ds.indices, np.int64),
              np.ascontiguousarray(ds.data, np.float64)):
        h.update(a.tobytes())
    h.update(str(int(ds.dim)).encode())
    return h.hexdigest()


def dataset(name):
    """The case's Dataset, normalised with the oracle's np.dot-order row norms."""
    from paper_2107_04074_b200 import synth
    from oracle import oracle as O
    cfg, n, _, _, _ = CASES[name]
    return synth.config_dataset(cfg, n_override=n, cache_dir="", row_norms=O.row_norms)


def make(name):
    from oracle import oracle as O
    _, _, k, seed, mi = CASES[name]
    t0 = time.time()
    ds = dataset(name)
    X = O.CSR(ds.indptr, ds.indices, ds.data, ds.dim)
    t1 = time.time()
    ref = O.run(X, k, "standard", seed=seed, max_iter=mi)
    t2 = time.time()
    margin = O.margins(X, ref["centers"])
    np.savez_compressed(
        HERE / f"cfg_{name}.npz",
        digest=np.array(digest(ds)), n=ds.n, dim=ds.dim, nnz=ds.indptr[-1], k=k, seed=seed, max_iter=mi,
        assignments=ref["assignments"].astype(np.int16), confident=np.packbits(margin > MARGIN),
        objective=ref["objective"], reassignments=ref["reassignments"], sim_count=ref["sim_count"],
        iterations=ref["iterations"], converged=ref["converged"], seed_indices=ref["seed_indices"])
    print(f"{name}: n={ds.n} nnz={ds.indptr[-1]} k={k} iterations={ref['iterations']} "
          f"objective={ref['objective'][-1]!r} confident={np.mean(margin > MARGIN):.4f} "
          f"(data {t1 - t0:.0f} s, oracle {t2 - t1:.0f} s)", flush=True)


if __name__ == "__main__":
    for nm in sys.argv[1:] or list(CASES):
        make(nm)
