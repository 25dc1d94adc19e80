#!/usr/bin/env python3
"""Time the UNMODIFIED reference package (``spkmeans``, shipped under
baseline/_ref by ``pip install --target``) on a row sample of a bench workload.

Test/measurement infrastructure for bench.py's ``cpu_baseline_reference``
entry; never imported by the product.  Runs in its own process so the thread
limits below apply before numpy/Numba load: the reference's hot loop is
serial (Numba without ``parallel``, single-threaded SciPy sparsetools), and
``OPENBLAS_NUM_THREADS=1`` pins its one BLAS call (``_center_thresholds``) to
one core as well: a strict 1-core figure.

Input: an .npz with the sample's normalised CSR (indptr, indices, data, dim)
-- the first ``n_sub`` rows of the bench corpus -- built by bench.py.  The
reference's own ``Dataset(rows=..., dim=...)`` is constructed from those rows
(they are already unit rows, bit-identical to what ``Dataset.from_rows``
produces from the raw generator rows), seeded with ``SeedConfig(seed)``
(``init_uniform``) and run with ``engine.run(..., max_iter=M)``.

Cost model for the full-size estimate: the reference's per-iteration time
splits into row-proportional work (similarities, bound updates, the scans,
the moves loop) and work on the k x d centers (``_move_centers``,
``_center_thresholds`` and the objective einsum), which does not grow with
n (with --d-full: the sample's term ids were folded to its d, and the center
phases, linear in d, are scaled by d_full / d).  The center phases are timed by wrapping the two functions and
``np.einsum`` in the reference module's namespace (timers only; the
reference code runs unchanged); the row part is scaled by n_full / n_sub.
"""

from __future__ import annotations

import os

for _v in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS", "NUMBA_NUM_THREADS"):
    os.environ[_v] = "1"
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/spkm_numba_cache")

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF = HERE / "_ref"


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--npz", required=True)
    p.add_argument("--k", type=int, required=True)
    p.add_argument("--variants", required=True)
    p.add_argument("--max-iter", type=int, default=3)
    p.add_argument("--seed", type=int, default=2)
    p.add_argument("--n-full", type=int, required=True)
    p.add_argument("--d-full", type=int, default=None, help="full d when the sample's term ids are folded")
    a = p.parse_args()
    if not (REF / "spkmeans").exists():
        print(json.dumps({"unavailable": f"{REF} missing (pip install --target baseline/_ref)"}))
        return
    sys.path.insert(0, str(REF))
    import spkmeans
    from spkmeans import engine as E
    from spkmeans.seeding import SeedConfig
    from spkmeans.sparse import Dataset, SparseVector

    z = np.load(a.npz)
    ip, ix, dv, dim = z["indptr"], z["indices"].astype(np.int64), z["data"], int(z["dim"])
    n_sub = ip.size - 1
    t = time.perf_counter()
    rows = tuple(SparseVector(ix[ip[i]:ip[i + 1]], dv[ip[i]:ip[i + 1]]) for i in range(n_sub))
    data = Dataset(rows=rows, dim=dim)
    build_s = time.perf_counter() - t

    # Numba JIT warm-up (kernels.py is compiled on first use) on a tiny corpus
    t = time.perf_counter()
    tiny = Dataset(rows=rows[:64], dim=dim)
    for v in a.variants.split(","):
        E.run(tiny, 4, v, SeedConfig(seed=1), max_iter=3)
    jit_s = time.perf_counter() - t

    other = [0.0]

    def timed(fn):
        def w(*args, **kw):
            t0 = time.perf_counter()
            try:
                return fn(*args, **kw)
            finally:
                other[0] += time.perf_counter() - t0
        return w

    class _NpProxy:
        """numpy with a timed einsum (the objective, engine.py:326)."""

        def __getattr__(self, name):
            return getattr(np, name)

    proxy = _NpProxy()
    proxy.einsum = timed(np.einsum)
    E._move_centers = timed(E._move_centers)
    E._center_thresholds = timed(E._center_thresholds)
    E.np = proxy

    out = {"n_sub": n_sub, "n_full": a.n_full, "d_sample": dim, "d_full": a.d_full or dim, "k": a.k, "max_iter": a.max_iter, "variants": {},
           "dataset_build_s": round(build_s, 2), "jit_warmup_s": round(jit_s, 2),
           "threads": "1 (OPENBLAS/OMP/MKL/NUMBA_NUM_THREADS=1)", "spkmeans": getattr(spkmeans, "__version__", "0.1.0")}
    its_tot, t_full_tot, t_sub_tot = 0, 0.0, 0.0
    for v in a.variants.split(","):
        other[0] = 0.0
        t0 = time.perf_counter()
        r = E.run(data, a.k, v, SeedConfig(seed=a.seed), max_iter=a.max_iter)
        wall = time.perf_counter() - t0
        its = len(r.iterations)
        el = sum(s.elapsed_ns for s in r.iterations) / 1e9     # seeding excluded (engine.py:240)
        oth = min(other[0], el)
        t_full = (el - oth) * a.n_full / n_sub + oth * (a.d_full or dim) / dim
        out["variants"][v] = {"iterations": its, "elapsed_s": round(el, 3), "wall_s": round(wall, 3),
                              "center_phase_s": round(oth, 3), "est_full_s": round(t_full, 3),
                              "sims": int(sum(s.sim_count for s in r.iterations))}
        its_tot += its
        t_full_tot += t_full
        t_sub_tot += el
    out["its_per_s_sample"] = its_tot / t_sub_tot
    out["its_per_s_full_est"] = its_tot / t_full_tot
    print(json.dumps(out))


if __name__ == "__main__":
    main()
