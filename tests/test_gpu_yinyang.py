"""Yin-Yang group bounds (variant "yinyang").

The reference has no Yin-Yang, so the bar is the one every pruned variant
meets: the fit equals the GPU's own Lloyd bit for bit (assignments,
objective, per-iteration reassignments, iteration count) -- and through it
the float64 oracle within the BASELINE tolerances -- while the device
auditor (validation.audit_bounds, exact float64 similarities) finds every
group bound sound at every iteration.
"""

import numpy as np
import pytest

from conftest import golden_dataset, load_golden

pytestmark = pytest.mark.gpu


def _same(r, b):
    assert np.array_equal(r.assignments, b.assignments)
    assert r.objective == b.objective
    assert len(r.iterations) == len(b.iterations)
    assert [s.reassignments for s in r.iterations] == [s.reassignments for s in b.iterations]


@pytest.mark.parametrize("name,k,seed", [("C1", 20, 3), ("clustered", 20, 3), ("grid_2000_5000_20_2000", 50, 1),
                                         ("grid_200_5000_50_1007", 7, 2), ("pitfall", 5, 1)])
def test_yinyang_equals_lloyd_goldens(name, k, seed):
    import paper_2107_04074_b200 as spk
    data = golden_dataset(load_golden(name))
    base = spk.run(data, k, "standard", spk.SeedConfig(seed=seed), max_iter=50)
    for graphs in (False, True, True):         # eager, then the graph path (captured, replayed)
        r = spk.run(data, k, "yinyang", spk.SeedConfig(seed=seed), max_iter=50, use_graphs=graphs)
        _same(r, base)


@pytest.mark.parametrize("k", [20, 100, 1000])
def test_yinyang_equals_lloyd_c2_and_prunes(k):
    import paper_2107_04074_b200 as spk
    from paper_2107_04074_b200 import synth
    data = synth.config_dataset("C2")
    base = spk.run(data, k, "standard", spk.SeedConfig(seed=2), max_iter=50)
    r = spk.run(data, k, "yinyang", spk.SeedConfig(seed=2), max_iter=50)
    _same(r, base)
    sims = sum(s.sim_count for s in r.iterations[1:])
    full = (len(r.iterations) - 1) * data.n * k
    assert sims <= full + (len(r.iterations) - 1) * data.n      # + one tighten per survivor
    if k >= 100:     # at k = 20 (5 groups) C2's small cosines let one step of drift open every group
        assert sims < 0.8 * full, "group bounds prune nothing"


def test_yinyang_c3_subsample_vs_oracle(oracle_mod):
    import paper_2107_04074_b200 as spk
    from paper_2107_04074_b200 import synth
    data = synth.config_dataset("C3", n_override=30_000)
    X = oracle_mod.CSR(data.indptr, data.indices, data.data, data.dim)
    ref = oracle_mod.run(X, 200, "standard", seed=2, max_iter=50)
    margin = oracle_mod.margins(X, ref["centers"])
    r = spk.run(data, 200, "yinyang", spk.SeedConfig(seed=2), max_iter=50)
    ok = margin > 1e-5
    assert np.array_equal(r.assignments[ok], ref["assignments"][ok])
    assert abs(r.objective - ref["objective"][-1]) <= 1e-6 * abs(ref["objective"][-1])
    assert abs(len(r.iterations) - ref["iterations"]) <= 1


@pytest.mark.parametrize("name,k,seed", [("C1", 20, 3), ("clustered", 20, 5), ("grid_200_256_10_3000", 10, 1)])
def test_yinyang_bounds_sound_every_iteration(name, k, seed):
    from paper_2107_04074_b200 import validation
    data = golden_dataset(load_golden(name))
    rep = validation.audit_bounds(data, "yinyang", k, seed, max_iter=50)
    assert rep.passed, rep
    assert rep.decisions_audited > data.n


def test_yinyang_edge_cases():
    """k = 1, k = n, ties (single-nnz rows), k not a multiple of 4."""
    import paper_2107_04074_b200 as spk
    g = np.random.default_rng(11)
    n, d = 300, 40
    ties = spk.Dataset.from_csr(np.arange(n + 1), g.integers(0, d, n), np.ones(n), d)
    for data, ks in ((ties, (1, 3, 7, 13)), (golden_dataset(load_golden("five_points")), (1, 2, 5))):
        for k in ks:
            if k > data.n:
                continue
            base = spk.run(data, k, "standard", spk.SeedConfig(seed=4), max_iter=30)
            r = spk.run(data, k, "yinyang", spk.SeedConfig(seed=4), max_iter=30)
            _same(r, base)


def test_yinyang_dense_rows_equal_sparse_lloyd(monkeypatch):
    """Dense corpora: Yin-Yang runs the sparse kernels (as the Elkan family does)."""
    import paper_2107_04074_b200 as spk
    from paper_2107_04074_b200 import engine, synth
    data = synth.config_dataset("C5", n_override=8000)
    monkeypatch.setenv("SPKM_DENSE_TC", "0")
    engine.clear_engine_cache()
    base = spk.run(data, 100, "standard", spk.SeedConfig(seed=5), max_iter=30)
    monkeypatch.delenv("SPKM_DENSE_TC")
    engine.clear_engine_cache()
    r = spk.run(data, 100, "yinyang", spk.SeedConfig(seed=5), max_iter=30)
    _same(r, base)


def test_yinyang_debug_hook_sees_group_bounds():
    import paper_2107_04074_b200 as spk
    data = golden_dataset(load_golden("C1"))
    seen = []

    def hook(it, bounds, centroids):
        seen.append((it, bounds.u_matrix.shape))

    spk.run(data, 20, "yinyang", spk.SeedConfig(seed=3), max_iter=5, debug_hook=hook)
    assert seen and all(shape == (data.n, 5) for _, shape in seen)
