"""Pin the CPU oracle (the checker) against golden vectors produced by the reference itself.

tests/golden/make_golden.py ran /root/reference/pkg/src/spkmeans (engine.run,
rng, geometry, validation.audit_bounds) and stored its outputs; nothing
here needs /root/reference at run time.
"""

import numpy as np
import pytest

from conftest import GOLDEN, golden_names, golden_runs, load_golden


def test_splitmix64_streams(oracle_mod):
    z = np.load(GOLDEN / "rng.npz")
    for key in z.files:
        if key.startswith("stream_"):
            seed = int(key.split("_", 1)[1])
            assert np.array_equal(oracle_mod.sm64_stream(seed, 32), z[key]), key
    # reference KAT (tests/test_rng.py:8-13)
    assert oracle_mod.sm64_stream(0, 4).tolist() == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4,
                                                     0x06C45D188009454F, 0xF88BB8A8724C81EC]


def test_sample_without_replacement(oracle_mod):
    z = np.load(GOLDEN / "rng.npz")
    for key in z.files:
        if key.startswith("swr_"):
            _, n, k, seed = key.split("_")
            got = oracle_mod.sample_without_replacement(int(seed), int(n), int(k))
            assert np.array_equal(got, z[key]), key


@pytest.mark.parametrize("op", ["lower", "upper", "hamerly", "half_angle", "clamp"])
def test_geometry_bit_exact(oracle_mod, op):
    z = np.load(GOLDEN / "geometry.npz")
    got = oracle_mod.geometry(op, z["a"], z["b"])
    assert np.array_equal(got, z[op]), op


@pytest.mark.parametrize("name", golden_names())
def test_oracle_reproduces_reference_runs(oracle_mod, name):
    z = load_golden(name)
    X = oracle_mod.CSR(z["indptr"], z["indices"], z["data"], int(z["dim"]))
    for key, v, k, seed, upd, mi in golden_runs(z):
        r = oracle_mod.run(X, k, v, seed=seed, max_iter=mi, hamerly_update=upd)
        assert np.array_equal(r["seed_indices"], z[key + "__seed_indices"]), key
        assert np.array_equal(r["assignments"], z[key + "__assignments"]), key
        assert np.array_equal(r["sim_count"], z[key + "__sim_count"]), key
        assert np.array_equal(r["cc_sim_count"], z[key + "__cc_sim_count"]), key
        assert np.array_equal(r["reassignments"], z[key + "__reassignments"]), key
        assert np.allclose(r["objective"], z[key + "__objective"], rtol=1e-12, atol=0), key
        assert r["converged"] == bool(z[key + "__converged"]), key
        assert np.array_equal(r["counts"], z[key + "__counts"]), key


class _Auditor:
    """validation._BoundAuditor restated (validation.py:49-80) over oracle full sims."""

    def __init__(self, O, X):
        self.O, self.X = O, X
        self.max_lower = self.max_upper = 0.0
        self.count = 0

    def __call__(self, it, a, l, u_m, u, centers):
        S = self.O.full_sims(self.X, centers)
        n = S.shape[0]
        own = S[np.arange(n), a]
        self.max_lower = max(self.max_lower, float(np.max(l - own)))
        self.count += n
        if u_m is not None:
            self.max_upper = max(self.max_upper, float(np.max(S - u_m)))
            self.count += S.size
        elif u is not None and S.shape[1] > 1:
            m = S.copy()
            m[np.arange(n), a] = -np.inf
            self.max_upper = max(self.max_upper, float(np.max(m.max(axis=1) - u)))
            self.count += n


@pytest.mark.parametrize("name,variant,k,seed,upd", [
    ("pitfall", "hamerly", 5, 1, "naive"), ("pitfall", "hamerly", 5, 1, "safe"),
    ("signed", "elkan", 6, 2, "safe"), ("signed", "simp_elkan", 6, 2, "safe"),
    ("signed", "hamerly", 6, 2, "safe"), ("signed", "simp_hamerly", 6, 2, "safe"),
])
def test_oracle_audit_matches_reference(oracle_mod, name, variant, k, seed, upd):
    z = load_golden(name)
    X = oracle_mod.CSR(z["indptr"], z["indices"], z["data"], int(z["dim"]))
    aud = _Auditor(oracle_mod, X)
    oracle_mod.run(X, k, variant, seed=seed, max_iter=100, hamerly_update=upd, hook=aud)
    ref = z[f"audit_{variant}_{k}_{seed}_{upd}"]
    assert aud.count == int(ref[2])
    assert aud.max_lower == pytest.approx(ref[0], abs=1e-12)
    assert aud.max_upper == pytest.approx(ref[1], abs=1e-12)
    passed = aud.max_lower <= 1e-9 and aud.max_upper <= 1e-9
    assert passed == bool(ref[3])


def test_pitfall_naive_violates(oracle_mod):
    """Acceptance #4 (tests/test_acceptance.py:114-123): naive fails, safe passes."""
    z = load_golden("pitfall")
    assert z["audit_hamerly_5_1_naive"][1] > 1e-9
    assert z["audit_hamerly_5_1_safe"][1] <= 1e-9


def test_pruning_efficacy_clustered(oracle_mod):
    """Acceptance #5: elkan < 0.5x standard sims, hamerly < 1x on the clustered fixture."""
    z = load_golden("clustered")
    tot = {v: int(z[f"{v}_20_3_safe_100__sim_count"].sum()) for v in
           ("standard", "elkan", "hamerly")}
    assert tot["elkan"] / tot["standard"] < 0.5
    assert tot["hamerly"] / tot["standard"] < 1.0


# ------------------------------------------------------------------ seeding
from conftest import seeding_cases, seeding_corpus, seeding_golden  # noqa: E402

_SZ = seeding_golden()


@pytest.mark.parametrize("case", seeding_cases(_SZ), ids=lambda c: c[0])
def test_oracle_seeding_matches_reference(oracle_mod, case):
    """init_kmpp / init_afkmc2 picks (seeding.py:64-146) equal the reference's."""
    key, method, name, k, alpha, chain, seed = case
    X = oracle_mod.CSR(*seeding_corpus(_SZ, name))
    tkey = f"trace__{name}__{k}__{alpha}__{seed}"
    if method == "kmpp":
        if tkey in _SZ.files:
            picks, tr = oracle_mod.seed_kmpp(X, k, alpha, seed, trace=True)
            assert np.array_equal(tr, _SZ[tkey])        # every weight vector bit-exact
        else:
            picks = oracle_mod.seed_kmpp(X, k, alpha, seed)
    else:
        picks = oracle_mod.seed_afkmc2(X, k, alpha, chain, seed)
    assert np.array_equal(picks, _SZ[key])


def test_numpy_reduction_orders(oracle_mod):
    """The oracle's np.dot (OpenBLAS ddot, single-threaded sizes: rows have
    <= 400 nnz here) and np.sum (pairwise) orders are numpy's."""
    g = np.random.default_rng(5)
    for n in list(range(0, 300)) + [511, 1024, 4097, 100_003]:
        x, y = g.standard_normal(n), g.standard_normal(n)
        if n <= 4097:
            assert oracle_mod.np_ddot(x, y) == float(np.dot(x, y)), n
        a = g.random(n) * g.random(n) ** 6
        assert oracle_mod.np_sum(a) == float(a.sum()), n
