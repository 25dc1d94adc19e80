"""CPU oracle -- TEST INFRASTRUCTURE ONLY.

ctypes front-end over ``oracle/libspkm_oracle.so`` (a plain-C float64
restatement of the reference ``spkmeans`` iteration loop, see
``spkm_oracle.c``).  It is the checker for the CUDA path: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import it.  The product package never does.

Reference anchors:
  run            /root/reference/pkg/src/spkmeans/engine.py:201-346
  assign_full    engine.py:103-120
  init_uniform   seeding.py:56-61 + rng.py:31-73 (splitmix64)
  seed_kmpp      seeding.py:64-89;  seed_afkmc2  seeding.py:92-146
  geometry       geometry.py:20-68
Parity pin: tests/test_oracle.py against tests/golden/*.npz made by running
the reference itself (tests/golden/make_golden.py).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "libspkm_oracle.so"

VARIANTS = ("standard", "elkan", "simp_elkan", "hamerly", "simp_hamerly")

_i64p = ctypes.POINTER(ctypes.c_int64)
_i32p = ctypes.POINTER(ctypes.c_int32)
_f64p = ctypes.POINTER(ctypes.c_double)
_u64p = ctypes.POINTER(ctypes.c_uint64)

HOOK_T = ctypes.CFUNCTYPE(None, ctypes.c_int64, _i64p, _f64p, _f64p, _f64p, _f64p)

_lib = None


def build():
    """Compile the oracle with its Makefile (gcc, no cmake)."""
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        L = ctypes.CDLL(str(LIB_PATH))
        L.oracle_sm64_stream.argtypes = [ctypes.c_uint64, ctypes.c_int64, _u64p]
        L.oracle_sample_without_replacement.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64, _i64p]
        L.oracle_sample_without_replacement.restype = ctypes.c_int
        L.oracle_geometry.argtypes = [ctypes.c_int, ctypes.c_int64, _f64p, _f64p, _f64p]
        L.oracle_full_sims.argtypes = [ctypes.c_int64] * 3 + [_i64p, _i32p, _f64p, _f64p, _f64p]
        L.oracle_assign_full.argtypes = [ctypes.c_int64] * 3 + [_i64p, _i32p, _f64p, _f64p, _i64p, _f64p, _f64p]
        L.oracle_aggregate_sums.argtypes = [ctypes.c_int64] * 3 + [_i64p, _i32p, _f64p, _i64p, _f64p, _i64p]
        L.oracle_run.argtypes = (
            [ctypes.c_int64] * 3 + [_i64p, _i32p, _f64p, ctypes.c_int, ctypes.c_int64, ctypes.c_int]
            + [_f64p, _f64p, _i64p, _f64p, _i64p, _i64p, _i64p, _i64p, _f64p,
               ctypes.POINTER(ctypes.c_int), HOOK_T, _f64p, _f64p]
        )
        L.oracle_run.restype = ctypes.c_int64
        L.oracle_seed_kmpp.argtypes = ([ctypes.c_int64] * 2 + [_i64p, _i32p, _f64p, ctypes.c_int64, ctypes.c_double,
                                       ctypes.c_uint64, _i64p, _f64p])
        L.oracle_seed_kmpp.restype = ctypes.c_int
        L.oracle_seed_afkmc2.argtypes = ([ctypes.c_int64] * 2 + [_i64p, _i32p, _f64p, ctypes.c_int64,
                                         ctypes.c_double, ctypes.c_int64, ctypes.c_uint64, _i64p])
        L.oracle_seed_afkmc2.restype = ctypes.c_int
        L.oracle_np_ddot.argtypes = [ctypes.c_int64, _f64p, _f64p]
        L.oracle_np_ddot.restype = ctypes.c_double
        L.oracle_np_sum.argtypes = [_f64p, ctypes.c_int64]
        L.oracle_np_sum.restype = ctypes.c_double
        L.oracle_row_norms.argtypes = [ctypes.c_int64, _i64p, _f64p, _f64p]
        L.oracle_num_threads.restype = ctypes.c_int
        L.oracle_set_threads.argtypes = [ctypes.c_int]
        _lib = L
    return _lib


def _p(arr, t):
    return arr.ctypes.data_as(t)


def set_threads(t: int):
    lib().oracle_set_threads(int(t))


def num_threads() -> int:
    return int(lib().oracle_num_threads())


def sm64_stream(seed: int, count: int) -> np.ndarray:
    out = np.empty(count, dtype=np.uint64)
    lib().oracle_sm64_stream(seed & ((1 << 64) - 1), count, _p(out, _u64p))
    return out


def sample_without_replacement(seed: int, n: int, k: int) -> np.ndarray:
    out = np.empty(max(k, 1), dtype=np.int64)
    rc = lib().oracle_sample_without_replacement(seed & ((1 << 64) - 1), n, k, _p(out, _i64p))
    if rc != 0:
        raise ValueError(f"cannot draw {k} distinct values from {n}")
    return out[:k]


def geometry(op: str, a, b=None) -> np.ndarray:
    ops = {"lower": 0, "upper": 1, "hamerly": 2, "half_angle": 3, "clamp": 4}
    a = np.ascontiguousarray(np.broadcast_to(np.asarray(a, dtype=np.float64), np.shape(a)), dtype=np.float64)
    b = a if b is None else np.ascontiguousarray(np.broadcast_to(np.asarray(b, np.float64), a.shape), np.float64)
    out = np.empty_like(a)
    lib().oracle_geometry(ops[op], a.size, _p(a, _f64p), _p(b, _f64p), _p(out, _f64p))
    return out


def np_ddot(x, y) -> float:
    """np.dot of two float64 vectors in numpy's OpenBLAS order (spkm_oracle.c)."""
    x = np.ascontiguousarray(x, np.float64)
    y = np.ascontiguousarray(y, np.float64)
    return float(lib().oracle_np_ddot(x.size, _p(x, _f64p), _p(y, _f64p)))


def row_norms(indptr, data) -> np.ndarray:
    """sqrt(np.dot(v, v)) of every CSR row in numpy's order (SparseVector.norm, sparse.py:52)."""
    ip = np.ascontiguousarray(indptr, np.int64)
    dv = np.ascontiguousarray(data, np.float64)
    out = np.empty(max(ip.size - 1, 0))
    lib().oracle_row_norms(out.size, _p(ip, _i64p), _p(dv, _f64p), _p(out, _f64p))
    return out


def normalized_csr(indptr, indices, weights, n_cols) -> "CSR":
    """Rows normalised as Dataset.from_rows does (values / norm, sparse.py:54-58)."""
    ip = np.ascontiguousarray(indptr, np.int64)
    w = np.ascontiguousarray(weights, np.float64)
    nrm = row_norms(ip, w)
    if np.any(nrm == 0.0):
        raise ValueError("zero row")
    return CSR(ip, indices, w / np.repeat(nrm, np.diff(ip)), n_cols)


def np_sum(a) -> float:
    """np.sum of a float64 vector (numpy's pairwise summation)."""
    a = np.ascontiguousarray(a, np.float64)
    return float(lib().oracle_np_sum(_p(a, _f64p), a.size))


class CSR:
    """float64 CSR as the oracle consumes it (int64 indptr, int32 indices)."""

    def __init__(self, indptr, indices, data, n_cols):
        self.indptr = np.ascontiguousarray(indptr, dtype=np.int64)
        self.indices = np.ascontiguousarray(indices, dtype=np.int32)
        self.data = np.ascontiguousarray(data, dtype=np.float64)
        self.n = self.indptr.size - 1
        self.d = int(n_cols)

    def densify_rows(self, rows) -> np.ndarray:
        """CentroidSet.from_data_rows, engine.py:46-58."""
        rows = np.asarray(rows, dtype=np.int64)
        out = np.zeros((rows.size, self.d))
        for q, i in enumerate(rows):
            s, e = self.indptr[i], self.indptr[i + 1]
            out[q, self.indices[s:e]] = self.data[s:e]
        return out

    def args(self):
        return (_p(self.indptr, _i64p), _p(self.indices, _i32p), _p(self.data, _f64p))


def full_sims(X: CSR, centers) -> np.ndarray:
    C = np.ascontiguousarray(centers, dtype=np.float64)
    k = C.shape[0]
    S = np.empty((X.n, k))
    lib().oracle_full_sims(X.n, X.d, k, *X.args(), _p(C, _f64p), _p(S, _f64p))
    return S


def assign_full(X: CSR, centers):
    C = np.ascontiguousarray(centers, dtype=np.float64)
    k = C.shape[0]
    a = np.empty(X.n, np.int64)
    best = np.empty(X.n)
    second = np.empty(X.n)
    lib().oracle_assign_full(X.n, X.d, k, *X.args(), _p(C, _f64p), _p(a, _i64p), _p(best, _f64p), _p(second, _f64p))
    return a, best, second


def aggregate_sums(X: CSR, a, k):
    a = np.ascontiguousarray(a, dtype=np.int64)
    sums = np.empty((k, X.d))
    counts = np.empty(k, np.int64)
    lib().oracle_aggregate_sums(X.n, X.d, k, *X.args(), _p(a, _i64p), _p(sums, _f64p), _p(counts, _i64p))
    return sums, counts


def run(X: CSR, k: int, variant: str, seed: int = 0, max_iter: int = 100,
        hamerly_update: str = "safe", init_rows=None, hook=None) -> dict:
    """engine.run (engine.py:201-346) with uniform seeding (seeding.py:56-61).

    ``hook(it, a, l, u_matrix, u, centers)`` mirrors debug_hook
    (engine.py:304-309) with numpy views of the live state.
    """
    if variant not in VARIANTS:
        raise ValueError(f"unknown variant {variant!r}")
    if hamerly_update not in ("safe", "naive"):
        raise ValueError(f"unknown hamerly_update {hamerly_update!r}")
    if not 1 <= k <= X.n:
        raise ValueError(f"k={k} infeasible for n={X.n}")
    idx = sample_without_replacement(seed, X.n, k) if init_rows is None else np.asarray(init_rows, np.int64)
    centers = np.ascontiguousarray(X.densify_rows(idx))
    sums = np.zeros_like(centers)
    counts = np.zeros(k, np.int64)
    drift = np.ones(k)
    a = np.zeros(X.n, np.int64)
    sims = np.zeros(max_iter, np.int64)
    ccs = np.zeros(max_iter, np.int64)
    rea = np.zeros(max_iter, np.int64)
    obj = np.zeros(max_iter)
    t_rows = np.zeros(max_iter)
    t_other = np.zeros(max_iter)
    conv = ctypes.c_int(0)
    n, d = X.n, X.d

    if hook is not None:
        def _cb(it, ap, lp, ump, up, cp):
            av = np.ctypeslib.as_array(ap, shape=(n,))
            lv = np.ctypeslib.as_array(lp, shape=(n,))
            umv = np.ctypeslib.as_array(ump, shape=(n, k)) if ump else None
            uv = np.ctypeslib.as_array(up, shape=(n,)) if up else None
            cv = np.ctypeslib.as_array(cp, shape=(k, d))
            hook(int(it), av, lv, umv, uv, cv)
        cb = HOOK_T(_cb)
    else:
        cb = HOOK_T()
    iters = lib().oracle_run(
        n, d, k, *X.args(), VARIANTS.index(variant), max_iter, int(hamerly_update == "naive"),
        _p(centers, _f64p), _p(sums, _f64p), _p(counts, _i64p), _p(drift, _f64p), _p(a, _i64p),
        _p(sims, _i64p), _p(ccs, _i64p), _p(rea, _i64p), _p(obj, _f64p), ctypes.byref(conv), cb,
        _p(t_rows, _f64p), _p(t_other, _f64p),
    )
    return {
        "assignments": a,
        "centers": centers,
        "sums": sums,
        "counts": counts,
        "drift": drift,
        "seed_indices": idx,
        "sim_count": sims[:iters].copy(),
        "cc_sim_count": ccs[:iters].copy(),
        "reassignments": rea[:iters].copy(),
        "objective": obj[:iters].copy(),
        "iterations": int(iters),
        "converged": bool(conv.value),
        "t_rows": t_rows[:iters].copy(),      # seconds per iteration spent on row-proportional work
        "t_other": t_other[:iters].copy(),    # ... on the k x d centers
    }


def margins(X: CSR, centers) -> np.ndarray:
    """best - second similarity per point in float64 (for the 1e-5 margin rule)."""
    _, best, second = assign_full(X, centers)
    return best - second


if os.environ.get("SPKM_ORACLE_THREADS"):
    set_threads(int(os.environ["SPKM_ORACLE_THREADS"]))


def seed_kmpp(X: CSR, k: int, alpha: float, seed: int, trace: bool = False):
    """init_kmpp (seeding.py:64-89): picks, and the (k-1) x n weight trace."""
    picks = np.empty(k, np.int64)
    tr = np.empty((max(k - 1, 1), X.n)) if trace else None
    rc = lib().oracle_seed_kmpp(X.n, X.d, *X.args(), k, float(alpha), seed & ((1 << 64) - 1), _p(picks, _i64p),
                                _p(tr, _f64p) if trace else None)
    if rc != 0:
        raise ValueError(f"k={k} infeasible for n={X.n}")
    return (picks, tr[:k - 1]) if trace else picks


def seed_afkmc2(X: CSR, k: int, alpha: float, chain_length: int, seed: int):
    """init_afkmc2 (seeding.py:92-146): picks."""
    picks = np.empty(k, np.int64)
    rc = lib().oracle_seed_afkmc2(X.n, X.d, *X.args(), k, float(alpha), int(chain_length), seed & ((1 << 64) - 1),
                                  _p(picks, _i64p))
    if rc != 0:
        raise ValueError("infeasible seeding arguments")
    return picks
