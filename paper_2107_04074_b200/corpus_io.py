"""Corpus ingestion, TF-IDF weighting and result files (reference corpus_io.py).

Same names, arguments, errors and file formats as
/root/reference/pkg/src/spkmeans/corpus_io.py:1-152.  The reference builds
one Python ``SparseVector`` per line; here the SVMlight text is parsed by a
multithreaded C++ parser in libspkm.so (``spkm_svml_parse``, csrc/ingest.cpp)
straight into flat CSR arrays, TF-IDF is vectorised over those arrays (idf
values from libm ``log`` like the reference's ``math.log``), and
``load_dataset`` hands the arrays to ``Dataset.from_csr`` (row norms in the
reference's np.dot order), so the resulting Dataset equals the reference's
bit for bit (tests/test_ingest.py against golden fixtures).  Host code: no
GPU is needed to ingest.
"""

from __future__ import annotations

import csv
import ctypes
from dataclasses import dataclass

import numpy as np

from .errors import DeviceError, ParseError, ZeroNormError
from .sparse import Dataset, SparseVector

STATS_HEADER = ["iteration", "sim_count", "cc_sim_count",
                "reassignments", "objective", "elapsed_ns"]


@dataclass
class CorpusMeta:
    n_rows: int
    n_cols: int
    density: float
    source: str


class RawRows:
    """Unnormalised parsed rows as one CSR (what parse_svmlight returns).

    Behaves like the reference's list of SparseVector (len, indexing,
    iteration) without building per-row objects unless asked.
    """

    def __init__(self, indptr, indices, values):
        self.indptr = np.asarray(indptr, dtype=np.int64)
        self.indices = np.asarray(indices, dtype=np.int64)
        self.values = np.asarray(values, dtype=np.float64)

    def __len__(self) -> int:
        return int(self.indptr.size - 1)

    def __getitem__(self, i) -> SparseVector:
        if isinstance(i, slice):
            return [self[j] for j in range(*i.indices(len(self)))]
        if i < 0:
            i += len(self)
        s, e = self.indptr[i], self.indptr[i + 1]
        return SparseVector(self.indices[s:e], self.values[s:e])

    def __iter__(self):
        for i in range(len(self)):
            yield self[i]

    @property
    def nnz(self) -> int:
        return int(self.indices.size)


def _lib():
    from . import _lib as L
    return L, L.lib()


def _as_raw(rows) -> RawRows:
    if isinstance(rows, RawRows):
        return rows
    rows = list(rows)
    lens = np.array([r.nnz for r in rows], dtype=np.int64)
    ip = np.zeros(len(rows) + 1, np.int64)
    np.cumsum(lens, out=ip[1:])
    idx = np.concatenate([r.indices for r in rows]) if rows else np.zeros(0, np.int64)
    val = np.concatenate([r.values for r in rows]) if rows else np.zeros(0)
    return RawRows(ip, idx, val)


def parse_svmlight(path, dim=None, threads: int = 0):
    """Parse a sparse matrix file into raw (unnormalised) rows (corpus_io.py:31-88).

    Returns (rows, meta).  Dimensionality is max index + 1 unless ``dim``
    is given.  Empty lines and ``#`` comments are skipped; explicit zeros
    are stripped; malformed pairs and non-increasing indices raise
    ParseError with the 1-based line number.
    """
    with open(path, "rb") as fh:
        buf = fh.read()
    L, lib = _lib()
    res = L.Svml()
    rc = lib.spkm_svml_parse(buf, len(buf), int(threads), ctypes.byref(res))
    if rc != 0:
        raise ParseError(int(res.err_line), res.err_msg.decode("utf-8", "replace"))
    n, nnz, max_idx = int(res.n_rows), int(res.nnz), int(res.max_idx)
    indptr = np.zeros(n + 1, np.int64)
    indices = np.empty(max(nnz, 1), np.int64)
    values = np.empty(max(nnz, 1), np.float64)
    lib.spkm_svml_fetch(ctypes.byref(res), indptr.ctypes.data, indices.ctypes.data, values.ctypes.data)
    rows = RawRows(indptr, indices[:nnz], values[:nnz])
    if dim is None:
        dim = max_idx + 1
    elif max_idx >= dim:
        raise ParseError(0, f"index {max_idx} exceeds declared dim {dim}")
    density = nnz / (n * dim) if n and dim else 0.0
    return rows, CorpusMeta(n_rows=n, n_cols=dim, density=density, source=str(path))


def write_svmlight(rows, path, labels=None):
    """corpus_io.py:91-98 (``label idx:value`` lines, values as %.17g)."""
    raw = _as_raw(rows)
    with open(path, "w", encoding="utf-8") as fh:
        for i in range(len(raw)):
            s, e = raw.indptr[i], raw.indptr[i + 1]
            label = labels[i] if labels is not None else 0
            pairs = " ".join(f"{int(j)}:{v:.17g}" for j, v in zip(raw.indices[s:e], raw.values[s:e]))
            fh.write(f"{label} {pairs}\n".rstrip() + "\n")


def apply_tfidf(rows, smooth=False) -> RawRows:
    """Weight raw term counts by inverse document frequency (corpus_io.py:101-126).

    Default tf * ln(n / df); with ``smooth`` tf * (ln((1+n)/(1+df)) + 1).
    Terms present in every document get idf 0 and are dropped; rows left
    empty raise ZeroNormError with their indices.
    """
    raw = _as_raw(rows)
    n = len(raw)
    d = int(raw.indices.max()) + 1 if raw.nnz else 0
    df = np.bincount(raw.indices, minlength=d).astype(np.int64)
    idf = np.zeros(d)
    if d:
        _, lib = _lib()
        lib.spkm_host_idf(d, df.ctypes.data, n, int(bool(smooth)), idf.ctypes.data)
    w = raw.values * idf[raw.indices]
    keep = w != 0.0
    rid = np.repeat(np.arange(n), np.diff(raw.indptr))
    counts = np.bincount(rid[keep], minlength=n)
    empty = np.nonzero(counts == 0)[0].tolist()
    if empty:
        raise ZeroNormError(rows=empty, message=f"TF-IDF zeroed rows {empty}")
    ip = np.zeros(n + 1, np.int64)
    np.cumsum(counts, out=ip[1:])
    return RawRows(ip, raw.indices[keep], w[keep])


def load_dataset(path, tfidf=False, smooth=False, dim=None) -> Dataset:
    """Parse, optionally TF-IDF weight, and normalise into a Dataset (corpus_io.py:129-134)."""
    rows, meta = parse_svmlight(path, dim=dim)
    if tfidf:
        rows = apply_tfidf(rows, smooth=smooth)
    return Dataset.from_csr(rows.indptr, rows.indices, rows.values, meta.n_cols, normalize_rows=True,
                            check_sorted=False)


def write_assignments(result, path):
    """corpus_io.py:137-140: ``row,cluster`` per line."""
    with open(path, "w", encoding="utf-8") as fh:
        fh.write("".join(f"{i},{int(c)}\n" for i, c in enumerate(result.assignments)))


def write_stats_csv(result, path):
    """corpus_io.py:143-150: per-iteration instrumentation columns."""
    with open(path, "w", encoding="utf-8", newline="") as fh:
        writer = csv.writer(fh)
        writer.writerow(STATS_HEADER)
        for s in result.iterations:
            writer.writerow([s.iteration, s.sim_count, s.cc_sim_count, s.reassignments, f"{s.objective:.17g}",
                             s.elapsed_ns])


def read_stats_csv(path):
    with open(path, "r", encoding="utf-8", newline="") as fh:
        return list(csv.DictReader(fh))


__all__ = ["CorpusMeta", "RawRows", "STATS_HEADER", "parse_svmlight", "write_svmlight", "apply_tfidf",
           "load_dataset", "write_assignments", "write_stats_csv", "read_stats_csv", "DeviceError"]
