"""Ingestion (reference corpus_io.py:31-134) against the reference's own outputs.

Golden vectors: tests/golden/make_golden_ingest.py runs the reference on the
files in tests/golden/svml/.  CPU only (the parser is host code).
"""

import numpy as np
import pytest

from conftest import GOLDEN

import paper_2107_04074_b200 as spk
from paper_2107_04074_b200 import corpus_io

Z = np.load(GOLDEN / "ingest.npz")
FILES = sorted({k.split("__")[0] for k in Z.files})
GOOD = [f for f in FILES if f + "__error" not in Z.files]
BAD = [f for f in FILES if f + "__error" in Z.files]


@pytest.mark.parametrize("name", GOOD)
def test_parse_tfidf_dataset_match_reference(name):
    path = GOLDEN / "svml" / f"{name}.svml"
    for threads in (1, 4):
        rows, meta = corpus_io.parse_svmlight(path, threads=threads)
        assert np.array_equal(rows.indptr, Z[name + "__parse_indptr"])
        assert np.array_equal(rows.indices, Z[name + "__parse_indices"])
        assert np.array_equal(rows.values, Z[name + "__parse_values"])
        m = Z[name + "__meta"]
        assert (meta.n_rows, meta.n_cols) == (int(m[0]), int(m[1])) and meta.density == m[2]
    for smooth, tag in ((False, "tfidf"), (True, "tfidf_smooth")):
        if f"{name}__{tag}_zeroed" in Z.files:
            with pytest.raises(spk.ZeroNormError) as ei:
                corpus_io.apply_tfidf(rows, smooth=smooth)
            assert ei.value.rows == Z[f"{name}__{tag}_zeroed"].tolist()
            continue
        t = corpus_io.apply_tfidf(rows, smooth=smooth)
        assert np.array_equal(t.indptr, Z[f"{name}__{tag}_indptr"])
        assert np.array_equal(t.indices, Z[f"{name}__{tag}_indices"])
        assert np.array_equal(t.values, Z[f"{name}__{tag}_values"])        # bit-exact weights
    if name + "__ds_data" in Z.files:
        ds = corpus_io.load_dataset(path, tfidf=True)
        assert np.array_equal(ds.indptr, Z[name + "__ds_indptr"])
        assert np.array_equal(ds.indices, Z[name + "__ds_indices"])
        assert np.array_equal(ds.data, Z[name + "__ds_data"])             # bit-exact normalised rows
    if name + "__raw_ds_data" in Z.files:
        assert np.array_equal(corpus_io.load_dataset(path).data, Z[name + "__raw_ds_data"])


@pytest.mark.parametrize("name", BAD)
def test_parse_errors_match_reference(name):
    line, msg = Z[name + "__error"]
    with pytest.raises(spk.ParseError) as ei:
        corpus_io.parse_svmlight(GOLDEN / "svml" / f"{name}.svml")
    assert ei.value.line_no == int(line)
    assert str(ei.value) == f"line {line}: {msg}"


def test_declared_dim_and_missing_file(tmp_path):
    p = GOLDEN / "svml" / "edge.svml"
    rows, meta = corpus_io.parse_svmlight(p, dim=50)
    assert meta.n_cols == 50
    with pytest.raises(spk.ParseError) as ei:
        corpus_io.parse_svmlight(p, dim=10)
    assert ei.value.line_no == 0 and "exceeds declared dim 10" in str(ei.value)
    with pytest.raises(FileNotFoundError):
        corpus_io.parse_svmlight(tmp_path / "nope.svml")


def _big_file(path, n_rows, seed, bad_line=None):
    g = np.random.default_rng(seed)
    lines = []
    for i in range(n_rows):
        m = int(g.integers(1, 40))
        idx = np.sort(g.choice(100000, m, replace=False))
        val = np.round(g.random(m) * 10, 3)
        body = " ".join(f"{j}:{v}" for j, v in zip(idx, val))
        style = i % 7
        if style == 0:
            lines.append(f"{i % 3} {body}\r\n")
        elif style == 1:
            lines.append(f"{body}\r")
        elif style == 2:
            lines.append("# comment line\n")
            lines.append(f"1 {body}\n")
        elif style == 3:
            lines.append("\n")
            lines.append(f"2 {body} # tail\n")
        else:
            lines.append(f"0 {body}\n")
    if bad_line is not None:
        lines.insert(bad_line - 1, "1 5:1 4:1\n")
    with open(path, "w", newline="") as fh:
        fh.write("".join(lines))


def test_multithreaded_parse_equals_single_thread(tmp_path):
    """Chunked parallel parsing (line boundaries, universal newlines) is
    identical to the one-thread parse, and an error planted deep in the file
    is reported at its exact line."""
    p = tmp_path / "big.svml"
    _big_file(p, 60000, 3)
    assert p.stat().st_size > (1 << 20)
    a, ma = corpus_io.parse_svmlight(p, threads=1)
    b, mb = corpus_io.parse_svmlight(p, threads=7)
    assert ma == mb
    assert np.array_equal(a.indptr, b.indptr) and np.array_equal(a.indices, b.indices)
    assert np.array_equal(a.values, b.values)
    q = tmp_path / "big_bad.svml"
    _big_file(q, 60000, 4, bad_line=70001)
    for t in (1, 8):
        with pytest.raises(spk.ParseError) as ei:
            corpus_io.parse_svmlight(q, threads=t)
        assert ei.value.line_no == 70001


def test_write_svmlight_round_trip(tmp_path):
    rows, _ = corpus_io.parse_svmlight(GOLDEN / "svml" / "counts_c1.svml")
    out = tmp_path / "rt.svml"
    corpus_io.write_svmlight(rows, out)
    back, _ = corpus_io.parse_svmlight(out)
    assert np.array_equal(back.indptr, rows.indptr) and np.array_equal(back.values, rows.values)
    assert isinstance(rows[3], spk.SparseVector) and len(rows) == 400
