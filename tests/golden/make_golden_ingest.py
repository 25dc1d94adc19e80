#!/usr/bin/env python3
"""Golden outputs of the reference's ingestion (corpus_io.py:31-134).

Runs the REFERENCE package (/root/reference/pkg/src/spkmeans, read only) on
the SVMlight files in tests/golden/svml/ (written by this repo: edge-case
grammar files and a 400-row raw-count corpus from the synthetic C1
generator) and stores in ingest.npz, per file:
  <f>__parse_indptr/indices/values, <f>__meta  (parse_svmlight)
  <f>__tfidf[_smooth]_indptr/indices/values   (apply_tfidf)
  <f>__ds_indptr/indices/data                  (load_dataset(tfidf=True))
  <f>__error = [line_no, message]              (files that raise ParseError)
Usage:  python tests/golden/make_golden_ingest.py
"""

import os
import sys
from pathlib import Path

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
REF = Path("/root/reference/pkg/src")
HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(REF))

import numpy as np  # noqa: E402

from spkmeans import corpus_io  # noqa: E402
from spkmeans.errors import ParseError, ZeroNormError  # noqa: E402

SVML = HERE / "svml"


def make_counts_file():
    """400 rows of the C1 generator's term ids with raw counts tf ~ Poisson(1)+1."""
    sys.path.insert(1, str(ROOT))
    from paper_2107_04074_b200 import synth
    ip, idx, _ = synth.sparse_corpus(synth.CONFIGS["C1"], synth.DATA_SEED_BASE + 1, return_raw=True)
    g = np.random.Generator(np.random.PCG64(7))
    n = 400
    with open(SVML / "counts_c1.svml", "w", encoding="utf-8") as fh:
        for i in range(n):
            s, e = ip[i], ip[i + 1]
            tf = g.poisson(1.0, e - s) + 1
            fh.write(f"{i % 5} " + " ".join(f"{int(j)}:{int(v)}" for j, v in zip(idx[s:e], tf)) + "\n")


def csr(rows):
    lens = np.array([r.nnz for r in rows], np.int64)
    ip = np.zeros(len(rows) + 1, np.int64)
    np.cumsum(lens, out=ip[1:])
    idx = np.concatenate([r.indices for r in rows]) if rows else np.zeros(0, np.int64)
    val = np.concatenate([r.values for r in rows]) if rows else np.zeros(0)
    return ip, idx.astype(np.int64), val.astype(np.float64)


def main():
    make_counts_file()
    out = {}
    for f in sorted(SVML.glob("*.svml")):
        key = f.stem
        try:
            rows, meta = corpus_io.parse_svmlight(f)
        except ParseError as e:
            out[key + "__error"] = np.array([str(e.line_no), str(e).split(": ", 1)[1]])
            continue
        ip, idx, val = csr(rows)
        out[key + "__parse_indptr"], out[key + "__parse_indices"], out[key + "__parse_values"] = ip, idx, val
        out[key + "__meta"] = np.array([meta.n_rows, meta.n_cols, meta.density])
        for smooth in (False, True):
            tag = "tfidf_smooth" if smooth else "tfidf"
            try:
                t = corpus_io.apply_tfidf(rows, smooth=smooth)
                a, b, c = csr(t)
                out[f"{key}__{tag}_indptr"], out[f"{key}__{tag}_indices"], out[f"{key}__{tag}_values"] = a, b, c
            except ZeroNormError as e:
                out[f"{key}__{tag}_zeroed"] = np.array(e.rows, np.int64)
        try:
            ds = corpus_io.load_dataset(f, tfidf=True)
            m = ds.matrix
            out[key + "__ds_indptr"] = m.indptr.astype(np.int64)
            out[key + "__ds_indices"] = m.indices.astype(np.int64)
            out[key + "__ds_data"] = m.data.astype(np.float64)
        except ZeroNormError as e:
            out[key + "__ds_zeronorm"] = np.array(e.rows if e.rows else [], np.int64)
        try:
            ds = corpus_io.load_dataset(f, tfidf=False)
            out[key + "__raw_ds_data"] = ds.matrix.data.astype(np.float64)
        except ZeroNormError as e:
            out[key + "__raw_ds_zeronorm"] = np.array(e.rows if e.rows else [], np.int64)
    np.savez_compressed(HERE / "ingest.npz", **out)
    print("ingest.npz:", sorted({k.split("__")[0] for k in out}))


if __name__ == "__main__":
    main()
