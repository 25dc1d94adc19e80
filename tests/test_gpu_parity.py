"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle and vs itself.

Contract (BASELINE.json north_star): final assignments identical wherever
the oracle's best-vs-second margin exceeds 1e-5; objective within 1e-6
relative; iteration count within +-1; every pruned variant EXACTLY equal to
the GPU's own Lloyd (assignments, objective, per-iteration reassignments).
"""

import numpy as np
import pytest

from conftest import golden_dataset, golden_names, golden_runs, load_golden

pytestmark = pytest.mark.gpu

VARIANTS = ("standard", "elkan", "simp_elkan", "hamerly", "simp_hamerly")
MARGIN = 1e-5
OBJ_RTOL = 1e-6


def check_vs_oracle(r, ref_assign, ref_obj, ref_iters, margin, check_iters=True):
    ok = margin > MARGIN
    bad = np.nonzero((r.assignments != ref_assign) & ok)[0]
    assert bad.size == 0, f"{bad.size} confident points differ, e.g. {bad[:5]}"
    assert abs(r.objective - ref_obj) <= OBJ_RTOL * max(1.0, abs(ref_obj)), (r.objective, ref_obj)
    if check_iters:
        assert abs(len(r.iterations) - ref_iters) <= 1, (len(r.iterations), ref_iters)


@pytest.mark.parametrize("name", golden_names())
def test_golden_parity_and_self_consistency(name, oracle_mod):
    import paper_2107_04074_b200 as spk
    z = load_golden(name)
    data = golden_dataset(z)
    base = {}
    for key, v, k, seed, upd, mi in golden_runs(z):
        r = spk.run(data, k, v, spk.SeedConfig(seed=seed), max_iter=mi, hamerly_update=upd)
        if upd == "safe" and mi >= 50:
            check_vs_oracle(r, z[key + "__assignments"], float(z[key + "__objective"][-1]),
                            len(z[key + "__objective"]), z[key + "__margin"])
        if upd != "safe":
            continue
        group = (k, seed, mi)
        if group not in base:
            base[group] = r
        else:
            b = base[group]
            assert np.array_equal(r.assignments, b.assignments), (v, group)
            assert r.objective == b.objective, (v, group)
            assert len(r.iterations) == len(b.iterations), (v, group)
            assert [s.reassignments for s in r.iterations] == [s.reassignments for s in b.iterations]
            assert all(s.sim_count <= data.n * k for s in r.iterations)


@pytest.mark.parametrize("k", [20, 100])
def test_c2_full_size_parity(k, oracle_mod):
    import paper_2107_04074_b200 as spk
    from paper_2107_04074_b200 import synth
    data = synth.config_dataset("C2")
    X = oracle_mod.CSR(data.indptr, data.indices, data.data, data.dim)
    ref = oracle_mod.run(X, k, "standard", seed=2, max_iter=50)
    margin = oracle_mod.margins(X, ref["centers"])
    base = None
    for v in VARIANTS:
        r = spk.run(data, k, v, spk.SeedConfig(seed=2), max_iter=50)
        if base is None:
            base = r
            check_vs_oracle(r, ref["assignments"], ref["objective"][-1], ref["iterations"], margin)
        else:
            assert np.array_equal(r.assignments, base.assignments), v
            assert r.objective == base.objective, v


def test_c1_parity_all_variants(oracle_mod):
    import paper_2107_04074_b200 as spk
    z = load_golden("C1")
    data = golden_dataset(z)
    for key, v, k, seed, upd, mi in golden_runs(z):
        r = spk.run(data, k, v, spk.SeedConfig(seed=seed), max_iter=mi)
        check_vs_oracle(r, z[key + "__assignments"], float(z[key + "__objective"][-1]),
                        len(z[key + "__objective"]), z[key + "__margin"])


def test_c5_dense_subsample_parity(oracle_mod, monkeypatch):
    """Config C5 (dense unit vectors, d=256, k=1000) on a 20k-row subsample of the generator."""
    import paper_2107_04074_b200 as spk
    from paper_2107_04074_b200 import synth
    data = synth.config_dataset("C5", n_override=20_000)
    X = oracle_mod.CSR(data.indptr, data.indices, data.data, data.dim)
    ref = oracle_mod.run(X, 1000, "standard", seed=5, max_iter=50)
    margin = oracle_mod.margins(X, ref["centers"])
    base = None
    for v in ("standard", "hamerly", "simp_hamerly"):       # tensor-core dense path
        r = spk.run(data, 1000, v, spk.SeedConfig(seed=5), max_iter=50)
        if base is None:
            base = r
            check_vs_oracle(r, ref["assignments"], ref["objective"][-1], ref["iterations"], margin)
        else:
            assert np.array_equal(r.assignments, base.assignments), v
            assert r.objective == base.objective, v
            assert [s.reassignments for s in r.iterations] == [s.reassignments for s in base.iterations]
    a, best, second = spk.assign_full(data, base.centers)
    _, rb, rs = oracle_mod.assign_full(X, base.centers.centers)
    assert np.max(np.abs(best - rb)) < 3e-5 and np.max(np.abs(second - rs)) < 3e-5
    # the Elkan family on dense rows runs the sparse kernels: equal to the Lloyd of that path
    from paper_2107_04074_b200 import engine
    monkeypatch.setenv("SPKM_DENSE_TC", "0")
    engine.clear_engine_cache()
    sbase = spk.run(data, 1000, "standard", spk.SeedConfig(seed=5), max_iter=50)
    check_vs_oracle(sbase, ref["assignments"], ref["objective"][-1], ref["iterations"], margin)
    monkeypatch.delenv("SPKM_DENSE_TC")
    engine.clear_engine_cache()
    for v in ("elkan", "simp_elkan"):
        r = spk.run(data, 1000, v, spk.SeedConfig(seed=5), max_iter=50)
        check_vs_oracle(r, ref["assignments"], ref["objective"][-1], ref["iterations"], margin)
        assert np.array_equal(r.assignments, sbase.assignments), v
        assert r.objective == sbase.objective, v
        assert [s.reassignments for s in r.iterations] == [s.reassignments for s in sbase.iterations]


def _edge_dataset(kind):
    from paper_2107_04074_b200.sparse import Dataset
    g = np.random.default_rng(11)
    if kind == "single_nnz":          # every row has one term: many exact ties between centers
        n, d = 300, 40
        ip = np.arange(n + 1, dtype=np.int64)
        idx = g.integers(0, d, n).astype(np.int64)
        val = np.ones(n)
    elif kind == "duplicates":        # blocks of identical rows
        n, d = 240, 60
        base = [np.sort(g.choice(d, 5, replace=False)) for _ in range(12)]
        rows = [base[i % 12] for i in range(n)]
        ip = np.zeros(n + 1, np.int64)
        ip[1:] = np.cumsum([r.size for r in rows])
        idx = np.concatenate(rows).astype(np.int64)
        val = np.tile(np.arange(1.0, 6.0), n)
    else:                             # long and short rows mixed (row-length extremes of the kernels)
        n, d = 200, 3000
        lens = np.where(np.arange(n) % 17 == 0, 1200, g.integers(1, 4, n))
        ip = np.zeros(n + 1, np.int64)
        ip[1:] = np.cumsum(lens)
        idx = np.concatenate([np.sort(g.choice(d, L, replace=False)) for L in lens]).astype(np.int64)
        val = g.uniform(0.1, 1.0, idx.size)
    return Dataset.from_csr(ip, idx, val, d, normalize_rows=True)


@pytest.mark.parametrize("kind", ["single_nnz", "duplicates", "long_rows"])
@pytest.mark.parametrize("k", [1, 7, 40])
def test_edge_corpora_parity(kind, k, oracle_mod):
    """Edge cases of the reference's tests (ties, k = 1, duplicate rows, extreme
    row lengths): every variant equals the GPU Lloyd and the oracle.  With
    exact ties between identical centers the iteration count is not compared:
    the GPU keeps the incumbent on ties from iteration 2 where
    the reference's Lloyd argmax moves tied points to the lowest index, so
    tie-only reassignments can take the reference extra iterations."""
    import paper_2107_04074_b200 as spk
    data = _edge_dataset(kind)
    X = oracle_mod.CSR(data.indptr, data.indices, data.data, data.dim)
    ref = oracle_mod.run(X, k, "standard", seed=4, max_iter=30)
    margin = oracle_mod.margins(X, ref["centers"])
    base = None
    for v in VARIANTS:
        r = spk.run(data, k, v, spk.SeedConfig(seed=4), max_iter=30)
        if base is None:
            base = r
            check_vs_oracle(r, ref["assignments"], ref["objective"][-1], ref["iterations"], margin,
                            check_iters=kind == "long_rows")
        else:
            assert np.array_equal(r.assignments, base.assignments), v
            assert r.objective == base.objective, v
            assert [s.reassignments for s in r.iterations] == [s.reassignments for s in base.iterations], v


def test_k_equals_n(oracle_mod):
    """k = n: every point its own seed; one iteration, objective n (unit rows)."""
    import paper_2107_04074_b200 as spk
    data = _edge_dataset("duplicates")
    sub = spk.Dataset.from_csr(data.indptr[:31], data.indices[:data.indptr[30]], data.data[:data.indptr[30]],
                               data.dim, normalize_rows=False)
    for v in VARIANTS:
        r = spk.run(sub, sub.n, v, spk.SeedConfig(seed=1), max_iter=10)
        assert r.objective == pytest.approx(float(sub.n), rel=1e-6), v
