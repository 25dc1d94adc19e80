"""GPU k-means++ / AFK-MC2 seeding (csrc/seed.cuh) against the reference.

Reference: /root/reference/pkg/src/spkmeans/seeding.py:64-146 and the tests
it ships (tests/test_seeding.py, tests/test_acceptance.py:196-214).  The
picks must equal the reference's: golden picks from running the reference
(tests/golden/make_golden_seeding.py) and, at sizes the reference is slow
at, the oracle's restatement (pinned to the same goldens on CPU).
"""

import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT, seeding_cases, seeding_corpus, seeding_golden

pytestmark = pytest.mark.gpu

_SZ = seeding_golden()


def _dataset(name):
    from paper_2107_04074_b200.sparse import Dataset
    ip, ix, dv, dim = seeding_corpus(_SZ, name)
    return Dataset(ip, ix, dv, dim)


@pytest.mark.parametrize("case", seeding_cases(_SZ), ids=lambda c: c[0])
def test_gpu_seeding_matches_reference(case):
    import paper_2107_04074_b200 as spk
    key, method, name, k, alpha, chain, seed = case
    data = _dataset(name)
    tkey = f"trace__{name}__{k}__{alpha}__{seed}"
    if method == "kmpp":
        trace = [] if tkey in _SZ.files else None
        cs = spk.init_kmpp(data, k, alpha=alpha, seed=seed, trace=trace)
        if trace is not None:
            assert np.array_equal(np.stack(trace), _SZ[tkey])   # weights bit-exact (seeding.py:80-81)
    else:
        cs = spk.init_afkmc2(data, k, alpha=alpha, chain_length=chain, seed=seed)
    assert np.array_equal(cs.seed_indices, _SZ[key])
    assert np.array_equal(cs.centers, data.densify_rows(_SZ[key]))


def test_seeding_corner_semantics():
    """tests/test_seeding.py:84-110 of the reference, on the device."""
    import paper_2107_04074_b200 as spk
    from paper_2107_04074_b200.sparse import Dataset, SparseVector

    def sv(pairs):
        idx, val = zip(*pairs)
        return SparseVector(np.array(idx, dtype=np.int64), np.array(val, dtype=float))
    anti = Dataset.from_rows([sv([(0, 1.0)]), sv([(0, -1.0)])], dim=2)
    for s in range(20):
        assert set(spk.init_kmpp(anti, 2, alpha=1.0, seed=s).seed_indices.tolist()) == {0, 1}
        assert set(spk.init_afkmc2(anti, 2, alpha=1.0, chain_length=10, seed=s).seed_indices.tolist()) == {0, 1}
    five = _dataset("five_points")
    for s in range(20):
        assert len(set(spk.init_kmpp(five, 5, alpha=2.0, seed=s).seed_indices.tolist())) == 5
        assert len(set(spk.init_afkmc2(five, 4, alpha=1.0, chain_length=5, seed=s).seed_indices.tolist())) == 4
    dup = Dataset.from_rows([sv([(0, 2.0)]), sv([(0, 3.0)]), sv([(0, 4.0)])], dim=1)
    assert sorted(spk.init_kmpp(dup, 3, alpha=1.0, seed=5).seed_indices.tolist()) == [0, 1, 2]
    with pytest.raises(spk.InfeasibleError):
        spk.init_kmpp(five, 6, alpha=1.0, seed=0)


@pytest.mark.parametrize("method", ["kmpp", "afkmc2"])
def test_gpu_seeding_c2_matches_oracle(oracle_mod, method):
    """C2 (20k x 100k): the device picks equal the oracle's (which equals the
    reference on every golden case)."""
    import paper_2107_04074_b200 as spk
    from paper_2107_04074_b200 import synth
    data = synth.config_dataset("C2")
    X = oracle_mod.CSR(data.indptr, data.indices, data.data, data.dim)
    k = 100
    if method == "kmpp":
        got = spk.init_kmpp(data, k, alpha=1.0, seed=3).seed_indices
        want = oracle_mod.seed_kmpp(X, k, 1.0, 3)
    else:
        got = spk.init_afkmc2(data, k, alpha=1.5, chain_length=200, seed=4).seed_indices
        want = oracle_mod.seed_afkmc2(X, k, 1.5, 200, 4)
    assert np.array_equal(got, want)


def test_sequential_replay_path_gives_same_picks():
    """Force the exact sequential-cumsum replay for every draw (SPKM_SEED_EXACT=1)
    in a fresh process: the picks must not change."""
    code = (
        "import numpy as np, paper_2107_04074_b200 as spk\n"
        "from paper_2107_04074_b200 import synth\n"
        "d = synth.config_dataset('C1')\n"
        "a = spk.init_kmpp(d, 40, alpha=1.0, seed=9).seed_indices\n"
        "b = spk.init_afkmc2(d, 40, alpha=1.0, chain_length=1, seed=9).seed_indices\n"
        "print(','.join(map(str, np.concatenate([a, b]))))\n")
    outs = []
    for flag in ("0", "1"):
        env = dict(os.environ, SPKM_SEED_EXACT=flag)
        r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True, text=True,
                           timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(r.stdout.strip().splitlines()[-1])
    assert outs[0] == outs[1]


@pytest.mark.parametrize("variant", ["standard", "hamerly", "simp_elkan"])
def test_run_with_kmpp_seeding(oracle_mod, variant):
    """engine.run with SeedConfig(method='kmpp'|'afkmc2'): seeds equal the
    oracle's picks and the pruned variants still equal Lloyd exactly."""
    import paper_2107_04074_b200 as spk
    data = _dataset("clustered")
    X = oracle_mod.CSR(data.indptr, data.indices, data.data, data.dim)
    for cfg, want in ((spk.SeedConfig(method="kmpp", alpha=1.0, seed=3), oracle_mod.seed_kmpp(X, 20, 1.0, 3)),
                      (spk.SeedConfig(method="afkmc2", alpha=1.0, chain_length=50, seed=3),
                       oracle_mod.seed_afkmc2(X, 20, 1.0, 50, 3))):
        res = spk.run(data, 20, variant, seeding=cfg, max_iter=100)
        ref = spk.run(data, 20, "standard", seeding=cfg, max_iter=100)
        assert np.array_equal(res.centers.seed_indices, want)
        assert np.array_equal(res.assignments, ref.assignments)
        assert [s.reassignments for s in res.iterations] == [s.reassignments for s in ref.iterations]
        o = oracle_mod.run(X, 20, variant, init_rows=want, max_iter=100)
        assert abs(o["objective"][-1] - res.objective) <= 1e-6 * abs(o["objective"][-1])


def test_gpu_seeding_dense_corpus(oracle_mod):
    """k-means++ / AFK-MC2 on a dense (C5-shaped) corpus: float64 rows of the
    dense path, same picks as the oracle."""
    import paper_2107_04074_b200 as spk
    from paper_2107_04074_b200 import synth
    data = synth.config_dataset("C5", n_override=5000)
    X = oracle_mod.CSR(data.indptr, data.indices, data.data, data.dim)
    assert np.array_equal(spk.init_kmpp(data, 40, alpha=1.0, seed=11).seed_indices,
                          oracle_mod.seed_kmpp(X, 40, 1.0, 11))
    assert np.array_equal(spk.init_afkmc2(data, 40, alpha=1.5, chain_length=30, seed=12).seed_indices,
                          oracle_mod.seed_afkmc2(X, 40, 1.5, 30, 12))


def test_ingest_then_fit(oracle_mod, tmp_path):
    """corpus_io.load_dataset (C++ parser + TF-IDF) feeding the GPU fit: the
    fit matches the oracle run on the same rows."""
    import paper_2107_04074_b200 as spk
    from paper_2107_04074_b200 import corpus_io
    from conftest import GOLDEN
    data = corpus_io.load_dataset(GOLDEN / "svml" / "counts_c1.svml", tfidf=True)
    X = oracle_mod.CSR(data.indptr, data.indices, data.data, data.dim)
    ref = oracle_mod.run(X, 12, "standard", seed=4, max_iter=50)
    for v in ("standard", "elkan", "hamerly"):
        r = spk.run(data, 12, v, spk.SeedConfig(seed=4), max_iter=50)
        assert abs(r.objective - ref["objective"][-1]) <= 1e-6 * abs(ref["objective"][-1])
        assert abs(len(r.iterations) - ref["iterations"]) <= 1
