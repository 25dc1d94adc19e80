"""Sparse unit rows and the CSR ``Dataset`` the iteration loop consumes.

API mirror of the reference (/root/reference/pkg/src/spkmeans/sparse.py):
``SparseVector`` (22-67), ``dot_sparse_sparse`` (70-77),
``dot_sparse_dense`` (80-87), ``normalize`` (90-98) and ``Dataset``
(101-156).  Unlike the reference, ``Dataset`` is CSR-first: it keeps one
set of flat arrays (int64 indptr, int32 indices, float64 values) and only
builds per-row ``SparseVector`` objects on demand, because per-row Python
objects are the reference's scalability wall at 10^5-10^7 rows
(SURVEY.md §2.1 row 4).  ``Dataset.from_csr`` is the scalable entry point.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import DimensionMismatchError, ZeroNormError


@dataclass(frozen=True)
class SparseVector:
    """One row: strictly increasing indices, explicit zeros removed."""

    indices: np.ndarray
    values: np.ndarray

    def __post_init__(self):
        idx = np.asarray(self.indices, dtype=np.int64)
        val = np.asarray(self.values, dtype=np.float64)
        if idx.ndim != 1 or idx.shape != val.shape:
            raise ValueError("indices and values must be 1-D and equal length")
        nz = val != 0.0
        if not nz.all():
            idx, val = idx[nz], val[nz]
        if idx.size:
            if idx[0] < 0:
                raise ValueError("negative index")
            if idx.size > 1 and np.any(idx[1:] <= idx[:-1]):
                raise ValueError("indices must be strictly increasing")
        idx.setflags(write=False)
        val.setflags(write=False)
        object.__setattr__(self, "indices", idx)
        object.__setattr__(self, "values", val)

    @property
    def nnz(self) -> int:
        return int(self.indices.size)

    def norm(self) -> float:
        return float(np.sqrt(np.dot(self.values, self.values)))

    def normalized(self) -> "SparseVector":
        nrm = self.norm()
        if nrm == 0.0:
            raise ZeroNormError()
        return SparseVector(self.indices, self.values / nrm)

    def densify(self, dim: int) -> np.ndarray:
        if self.indices.size and self.indices[-1] >= dim:
            raise DimensionMismatchError(f"index {int(self.indices[-1])} exceeds dimensionality {dim}")
        out = np.zeros(dim)
        out[self.indices] = self.values
        return out


def dot_sparse_sparse(x: SparseVector, y: SparseVector) -> float:
    _, xi, yi = np.intersect1d(x.indices, y.indices, assume_unique=True, return_indices=True)
    return float(np.dot(x.values[xi], y.values[yi])) if xi.size else 0.0


def dot_sparse_dense(x: SparseVector, c: np.ndarray) -> float:
    if x.indices.size and x.indices[-1] >= c.shape[0]:
        raise DimensionMismatchError(f"index {int(x.indices[-1])} exceeds dense length {c.shape[0]}")
    return float(np.dot(x.values, c[x.indices])) if x.indices.size else 0.0


def normalize(v):
    if isinstance(v, SparseVector):
        return v.normalized()
    v = np.asarray(v, dtype=np.float64)
    nrm = float(np.linalg.norm(v))
    if nrm == 0.0:
        raise ZeroNormError()
    return v / nrm


_HELPER_OK = None


def _helper_matches_numpy(L) -> bool:
    """The host helper replays the summation order of the ddot kernel numpy's
    bundled OpenBLAS uses on this machine (SkylakeX-style 32-accumulator
    blocks).  Another BLAS kernel would round differently in the last bit, so
    the helper is probed once against np.dot on rows of every length class
    and only used when it agrees bit for bit; otherwise the per-row np.dot
    loop (the reference's own arithmetic) is used."""
    global _HELPER_OK
    if _HELPER_OK is None:
        g = np.random.default_rng(12345)
        lens = [1, 2, 3, 7, 8, 15, 16, 17, 31, 32, 33, 47, 48, 63, 64, 65, 100, 127, 128, 129, 255, 400]
        ip = np.zeros(len(lens) + 1, np.int64)
        np.cumsum(lens, out=ip[1:])
        dv = g.random(int(ip[-1]))
        got = np.zeros(len(lens))
        L.spkm_host_row_norms(len(lens), ip.ctypes.data, dv.ctypes.data, got.ctypes.data)
        ref = np.array([np.sqrt(np.dot(dv[a:b], dv[a:b])) for a, b in zip(ip[:-1], ip[1:])])
        _HELPER_OK = bool(np.array_equal(got, ref))
    return _HELPER_OK


def _row_norms(indptr, data):
    """|row| of every CSR row exactly as SparseVector.norm computes it
    (np.sqrt(np.dot(v, v)), sparse.py:52): the library's host helper replays
    numpy's ddot order, so from_csr and from_rows give identical values."""
    n = indptr.size - 1
    out = np.zeros(n)
    if n == 0:
        return out
    from .errors import DeviceError
    try:
        from . import _lib
        L = _lib.lib()
    except DeviceError:
        L = None
    ip = np.ascontiguousarray(indptr, np.int64)
    dv = np.ascontiguousarray(data, np.float64)
    if L is not None and _helper_matches_numpy(L):
        L.spkm_host_row_norms(n, ip.ctypes.data, dv.ctypes.data, out.ctypes.data)
        return out
    for i in range(n):   # same values, one np.dot per row
        v = dv[ip[i]:ip[i + 1]]
        out[i] = np.sqrt(np.dot(v, v))
    return out


class Dataset:
    """Unit-normalised sparse rows held as one CSR.

    ``indptr`` int64[n+1], ``indices`` int32[nnz] (sorted within a row),
    ``data`` float64[nnz].  Zero rows are rejected with their row numbers
    (reference sparse.py:117-134).
    """

    def __init__(self, *args, rows=None, dim=None, indptr=None, indices=None, data=None):
        """Two forms:

        * ``Dataset(rows, dim)`` / ``Dataset(rows=..., dim=...)`` -- the
          reference's dataclass constructor (sparse.py:101-115): a sequence of
          ``SparseVector`` rows taken as they are (no normalisation; use
          ``from_rows`` for the checked, normalising constructor);
        * ``Dataset(indptr, indices, data, dim)`` -- flat CSR arrays (the
          scalable form; ``from_csr`` adds the checks and the normalisation).
        """
        if len(args) == 4:
            indptr, indices, data, dim = args
        elif len(args) == 2:
            rows, dim = args
        elif len(args) == 1 and rows is None and indptr is None:
            rows = args[0]
        elif args:
            raise TypeError("Dataset(rows, dim) or Dataset(indptr, indices, data, dim)")
        if dim is None:
            raise TypeError("Dataset needs dim")
        row_objs = None
        if rows is not None:
            if indptr is not None:
                raise TypeError("give rows or CSR arrays, not both")
            row_objs = tuple(rows)
            indptr = np.zeros(len(row_objs) + 1, np.int64)
            indptr[1:] = np.cumsum([r.nnz for r in row_objs])
            indices = (np.concatenate([np.asarray(r.indices) for r in row_objs]) if row_objs
                       else np.zeros(0, np.int32))
            data = (np.concatenate([np.asarray(r.values, np.float64) for r in row_objs]) if row_objs
                    else np.zeros(0))
        elif indptr is None or indices is None or data is None:
            raise TypeError("Dataset(rows, dim) or Dataset(indptr, indices, data, dim)")
        self.indptr = np.ascontiguousarray(indptr, dtype=np.int64)
        self.indices = np.ascontiguousarray(indices, dtype=np.int32)
        self.data = np.ascontiguousarray(data, dtype=np.float64)
        self.dim = int(dim)
        self.n = int(self.indptr.size - 1)
        self._rows = row_objs
        self._csr = None
        self._device_cache = {}

    # -- construction ------------------------------------------------------
    @classmethod
    def from_rows(cls, rows, dim=None, normalize_rows=True) -> "Dataset":
        rows = list(rows)
        if not rows:
            raise ValueError("dataset must contain at least one row")
        max_idx = max((int(r.indices[-1]) for r in rows if r.nnz), default=-1)
        if dim is None:
            dim = max_idx + 1
        elif max_idx >= dim:
            raise DimensionMismatchError(f"row index {max_idx} exceeds declared dimensionality {dim}")
        bad = [i for i, r in enumerate(rows) if r.nnz == 0 or r.norm() == 0.0]
        if bad:
            raise ZeroNormError(rows=bad)
        if normalize_rows:
            rows = [r.normalized() for r in rows]
        indptr = np.zeros(len(rows) + 1, np.int64)
        indptr[1:] = np.cumsum([r.nnz for r in rows])
        indices = np.concatenate([r.indices for r in rows]).astype(np.int32)
        data = np.concatenate([r.values for r in rows])
        ds = cls(indptr, indices, data, dim)
        ds._rows = tuple(rows)
        return ds

    @classmethod
    def from_csr(cls, indptr, indices, data, dim, normalize_rows=True,
                 check_sorted=True, row_norms=None) -> "Dataset":
        """Scalable constructor from flat CSR arrays (vectorised checks).

        ``row_norms(indptr, data)`` overrides the row-norm helper (default: the
        library's np.dot-order replay, falling back to np.dot per row)."""
        indptr = np.asarray(indptr, dtype=np.int64)
        indices = np.asarray(indices, dtype=np.int64)
        data = np.asarray(data, dtype=np.float64)
        if indptr.size < 2:
            raise ValueError("dataset must contain at least one row")
        if indices.size and (indices.min() < 0):
            raise ValueError("negative index")
        if indices.size and indices.max() >= dim:
            raise DimensionMismatchError(f"row index {int(indices.max())} exceeds declared dimensionality {dim}")
        if check_sorted and indices.size > 1:
            same_row = np.ones(indices.size - 1, bool)
            starts = indptr[1:-1]
            starts = starts[(starts > 0) & (starts < indices.size)]
            same_row[starts - 1] = False
            if np.any((indices[1:] <= indices[:-1]) & same_row):
                raise ValueError("indices must be strictly increasing within a row")
        if np.any(data == 0.0):
            keep = data != 0.0
            rowid = np.repeat(np.arange(indptr.size - 1), np.diff(indptr))
            counts = np.bincount(rowid[keep], minlength=indptr.size - 1)
            indptr = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
            indices, data = indices[keep], data[keep]
        norms = (row_norms or _row_norms)(indptr, data)
        bad = np.nonzero(norms == 0.0)[0]
        if bad.size:
            raise ZeroNormError(rows=bad.tolist())
        if normalize_rows:
            data = data / np.repeat(norms, np.diff(indptr))
        return cls(indptr, indices.astype(np.int32), data, dim)

    @classmethod
    def dense(cls, X, normalize_rows=True) -> "Dataset":
        """Dense vectors (config C5) as a CSR whose rows hold every column.

        Rows are L2-normalised in float64 (values / sqrt(<v, v>)); a zero row
        raises ZeroNormError like the sparse constructors.
        """
        X = np.asarray(X)
        n, d = X.shape
        data = np.ascontiguousarray(X, dtype=np.float64)
        if normalize_rows:
            nrm = np.sqrt(np.einsum("ij,ij->i", data, data))
            bad = np.nonzero(nrm == 0.0)[0]
            if bad.size:
                raise ZeroNormError(rows=bad.tolist())
            data /= nrm[:, None]
        indptr = np.arange(n + 1, dtype=np.int64) * d
        indices = np.tile(np.arange(d, dtype=np.int32), n)
        ds = cls(indptr, indices, data.reshape(-1), d)
        ds.dense_dim = d
        # float32 copy (round to nearest, what the device computes on): the
        # upload moves it instead of the float64 rows
        ds._values32 = ds.data.astype(np.float32)
        return ds

    # -- reference-compatible views ----------------------------------------
    @property
    def rows(self) -> tuple:
        if self._rows is None:
            ip, ix, dv = self.indptr, self.indices, self.data
            self._rows = tuple(
                SparseVector(ix[ip[i]:ip[i + 1]].astype(np.int64), dv[ip[i]:ip[i + 1]])
                for i in range(self.n))
        return self._rows

    @property
    def nnz(self) -> int:
        return int(self.indices.size)

    @property
    def matrix(self):
        if self._csr is None:
            from scipy import sparse as sp
            self._csr = sp.csr_matrix((self.data, self.indices, self.indptr), shape=(self.n, self.dim))
        return self._csr

    def csr_arrays(self):
        return self.indptr, self.indices.astype(np.int64), self.data

    def densify_rows(self, rows) -> np.ndarray:
        rows = np.asarray(rows, dtype=np.int64)
        out = np.zeros((rows.size, self.dim))
        for q, i in enumerate(rows):
            s, e = self.indptr[i], self.indptr[i + 1]
            out[q, self.indices[s:e]] = self.data[s:e]
        return out

    def row_lengths(self) -> np.ndarray:
        return np.diff(self.indptr)
