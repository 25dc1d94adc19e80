"""Device auditor / brute force / triangle fuzz (reference validation.py:18-116).

The audits are the reference's own acceptance check on the bounds
(tests/test_acceptance.py of the reference); golden audit reports of the
reference live in tests/golden/ds_*.npz (audit_<variant>_<k>_<seed>_<upd>).
"""

import numpy as np
import pytest

from conftest import golden_dataset, load_golden

pytestmark = pytest.mark.gpu

VARIANTS = ("elkan", "simp_elkan", "hamerly", "simp_hamerly")


def _v():
    from paper_2107_04074_b200 import validation
    return validation


@pytest.mark.parametrize("name", ["pitfall", "signed"])
def test_device_audit_matches_reference_reports(name):
    z = load_golden(name)
    data = golden_dataset(z)
    keys = [k for k in z.files if k.startswith("audit_")]
    assert keys
    for key in keys:
        variant, k, seed, upd = key[len("audit_"):].rsplit("_", 3)
        ref = z[key]
        rep = _v().audit_bounds(data, variant, int(k), seed=int(seed), hamerly_update=upd)
        assert rep.passed == bool(ref[3]), (key, rep)
        assert rep.decisions_audited == int(ref[2]), (key, rep)
        if not ref[3]:
            assert rep.max_upper_violation > 1e-3      # the naive update's violation is caught


@pytest.mark.parametrize("variant", VARIANTS)
def test_device_audit_at_scale(variant):
    """C3-shaped corpus (topics, d=250k) at n=40k, k=200: every bound sound at
    every iteration (the host auditor would need a 40k x 200 matrix per
    iteration; the device one keeps it in HBM)."""
    from paper_2107_04074_b200 import synth
    data = synth.config_dataset("C3", n_override=40_000)
    rep = _v().audit_bounds(data, variant, 200, seed=3, max_iter=15)
    assert rep.passed, rep
    assert rep.decisions_audited > 0


def test_brute_force_assign_matches_oracle(oracle_mod):
    import paper_2107_04074_b200 as spk
    for name in ("small", "clustered", "C1"):
        z = load_golden(name)
        data = golden_dataset(z)
        X = oracle_mod.CSR(z["indptr"], z["indices"], z["data"], int(z["dim"]))
        res = spk.run(data, 20 if name != "small" else 7, "standard", spk.SeedConfig(seed=1), max_iter=5)
        C = res.centers.centers
        got = _v().brute_force_assign(data, C)
        a, best, second = oracle_mod.assign_full(X, C)
        sure = (best - second) > 1e-12
        assert np.array_equal(got[sure], a[sure])


def test_fuzz_triangle():
    assert _v().fuzz_triangle(20000, 16, seed=1)
    assert _v().fuzz_triangle(5000, 3, seed=2)


def test_device_audit_dense_hamerly():
    """The dense tensor-core path's bounds are sound at every iteration (C5 shape, n=20k, k=200)."""
    from paper_2107_04074_b200 import synth
    data = synth.config_dataset("C5", n_override=20_000)
    for v in ("hamerly", "simp_hamerly"):
        rep = _v().audit_bounds(data, v, 200, seed=2, max_iter=20)
        assert rep.passed, (v, rep)
