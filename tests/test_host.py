"""Host-side logic that runs without a GPU: API validation, CSR dataset, rng, generator, geometry mirror."""

import numpy as np
import pytest

from conftest import GOLDEN

import paper_2107_04074_b200 as spk
from paper_2107_04074_b200 import geometry, synth
from paper_2107_04074_b200.engine import row_eps, scale_bits_for
from paper_2107_04074_b200.rng import PortableRng
from paper_2107_04074_b200.sparse import Dataset, SparseVector


def sv(pairs):
    idx, val = zip(*pairs)
    return SparseVector(np.array(idx), np.array(val, dtype=float))


# ------------------------------------------------------------------ errors / API
class TestValidation:
    def setup_method(self):
        self.data = Dataset.from_rows([sv([(0, 1.0)]), sv([(1, 2.0)]), sv([(0, 1.0), (2, 1.0)])], dim=3)

    def test_unknown_variant(self):
        with pytest.raises(spk.ConfigError):
            spk.run(self.data, 2, "bogus", spk.SeedConfig())

    def test_unknown_hamerly_update(self):
        with pytest.raises(spk.ConfigError):
            spk.run(self.data, 2, "hamerly", spk.SeedConfig(), hamerly_update="fast")

    @pytest.mark.parametrize("k", [0, 4, -1])
    def test_infeasible_k(self, k):
        with pytest.raises(spk.InfeasibleError):
            spk.run(self.data, k, "standard", spk.SeedConfig())

    def test_seed_config_validation(self):
        for bad in (spk.SeedConfig(method="x"), spk.SeedConfig(alpha=3.0), spk.SeedConfig(chain_length=0)):
            with pytest.raises(spk.ConfigError):
                bad.validate()

    def test_variants_tuple(self):
        assert spk.VARIANTS == ("standard", "elkan", "simp_elkan", "hamerly", "simp_hamerly")


# ------------------------------------------------------------------ dataset
class TestDataset:
    def test_from_rows_normalises_and_builds_csr(self):
        d = Dataset.from_rows([sv([(0, 3.0), (4, 4.0)]), sv([(2, 1.0)])], dim=6)
        assert d.n == 2 and d.dim == 6 and d.nnz == 3
        assert d.indptr.tolist() == [0, 2, 3]
        assert d.indices.dtype == np.int32 and d.indptr.dtype == np.int64
        assert np.allclose(d.data, [0.6, 0.8, 1.0])

    def test_zero_rows_rejected_with_indices(self):
        with pytest.raises(spk.ZeroNormError) as e:
            Dataset.from_rows([sv([(0, 1.0)]), SparseVector(np.array([], np.int64), np.array([])),
                               sv([(1, 0.0)])], dim=3)
        assert e.value.rows == [1, 2]

    def test_dimension_mismatch(self):
        with pytest.raises(spk.DimensionMismatchError):
            Dataset.from_rows([sv([(5, 1.0)])], dim=3)

    def test_from_csr_matches_from_rows(self):
        rows = [sv([(0, 1.0), (3, 2.0)]), sv([(1, 5.0)]), sv([(0, 1.0), (1, 1.0), (2, 1.0)])]
        a = Dataset.from_rows(rows, dim=4)
        ip = np.array([0, 2, 3, 6])
        ix = np.array([0, 3, 1, 0, 1, 2])
        dv = np.array([1.0, 2.0, 5.0, 1.0, 1.0, 1.0])
        b = Dataset.from_csr(ip, ix, dv, 4)
        assert np.array_equal(a.indptr, b.indptr) and np.array_equal(a.indices, b.indices)
        assert np.allclose(a.data, b.data, rtol=1e-15)

    def test_row_norm_helper_is_probed_and_has_an_exact_fallback(self, monkeypatch):
        """The ddot-order host helper is only used when it reproduces np.dot bit
        for bit on this machine; otherwise (another BLAS kernel) the per-row
        np.dot loop gives the reference's values.  Both paths agree here."""
        from paper_2107_04074_b200 import sparse
        g = np.random.default_rng(5)
        lens = g.integers(1, 300, 200)
        ip = np.zeros(lens.size + 1, np.int64)
        np.cumsum(lens, out=ip[1:])
        dv = g.random(int(ip[-1]))
        ref = np.array([np.sqrt(np.dot(dv[a:b], dv[a:b])) for a, b in zip(ip[:-1], ip[1:])])
        monkeypatch.setattr(sparse, "_HELPER_OK", None)
        fast = sparse._row_norms(ip, dv)
        monkeypatch.setattr(sparse, "_HELPER_OK", False)
        slow = sparse._row_norms(ip, dv)
        assert np.array_equal(slow, ref)
        assert np.array_equal(fast, ref)

    def test_from_csr_rejects_unsorted_and_zero_rows(self):
        with pytest.raises(ValueError):
            Dataset.from_csr([0, 2], [3, 1], [1.0, 1.0], 4)
        with pytest.raises(spk.ZeroNormError):
            Dataset.from_csr([0, 1, 1], [0], [1.0], 4)

    def test_rows_view_and_densify(self):
        d = Dataset.from_rows([sv([(0, 3.0), (4, 4.0)]), sv([(2, 1.0)])], dim=6)
        assert d.rows[0].nnz == 2
        c = d.densify_rows([1, 0])
        assert c.shape == (2, 6) and c[0, 2] == 1.0 and c[1, 4] == pytest.approx(0.8)


# ------------------------------------------------------------------ rng / seeding
def test_rng_matches_reference_golden():
    z = np.load(GOLDEN / "rng.npz")
    for key in z.files:
        if key.startswith("stream_"):
            r = PortableRng(int(key.split("_", 1)[1]))
            assert [r.next_uint64() for _ in range(32)] == z[key].tolist()
        if key.startswith("swr_"):
            _, n, k, seed = key.split("_")
            assert PortableRng(int(seed)).sample_without_replacement(int(n), int(k)) == z[key].tolist()


def test_random_resolution_and_mask():
    r = PortableRng(3)
    vals = [r.random() for _ in range(200)]
    assert all(0.0 <= v < 1.0 for v in vals)
    assert all(v * 2.0 ** 53 == int(v * 2.0 ** 53) for v in vals)
    assert PortableRng(1 << 64).next_uint64() == PortableRng(0).next_uint64()


def test_init_uniform_rows():
    d = Dataset.from_rows([sv([(i % 5, 1.0 + i)]) for i in range(30)], dim=5)
    cs = spk.init_uniform(d, 4, seed=9)
    assert cs.seed_indices.tolist() == PortableRng(9).sample_without_replacement(30, 4)
    assert np.array_equal(cs.centers, d.densify_rows(cs.seed_indices))
    assert np.all(cs.drift == 1.0) and cs.counts.sum() == 0


# ------------------------------------------------------------------ geometry mirror
def test_geometry_mirror_bit_exact_with_reference():
    z = np.load(GOLDEN / "geometry.npz")
    assert np.array_equal(geometry.cos_lower_bound(z["a"], z["b"]), z["lower"])
    assert np.array_equal(geometry.cos_upper_bound(z["a"], z["b"]), z["upper"])
    assert np.array_equal(geometry.hamerly_upper_update(z["a"], z["b"]), z["hamerly"])
    assert np.array_equal(geometry.half_angle_cc(z["a"]), z["half_angle"])


def test_triangle_fuzz_and_arccos_oracle():
    g = np.random.default_rng(0)
    for dims in (2, 3, 50):
        X, Z, Y = (g.normal(size=(20000, dims)) for _ in range(3))
        for M in (X, Z, Y):
            M /= np.linalg.norm(M, axis=1, keepdims=True)
        a, b = np.einsum("ij,ij->i", X, Z), np.einsum("ij,ij->i", Z, Y)
        ex = np.einsum("ij,ij->i", X, Y)
        assert np.all(geometry.cos_lower_bound(a, b) <= ex + 1e-9)
        assert np.all(geometry.cos_upper_bound(a, b) >= ex - 1e-9)
    a, b = g.uniform(-1, 1, 50000), g.uniform(-1, 1, 50000)
    near = (np.abs(a) > 1 - 1e-6) | (np.abs(b) > 1 - 1e-6)
    err = np.abs(geometry.cos_lower_bound(a, b) - geometry.arccos_triangle_oracle(a, b))
    assert np.all(err <= np.where(near, 1e-6, 1e-9))


def test_hamerly_dominance():
    """Safe single-bound update dominates every per-cluster update with p >= p_min (u, p >= 0)."""
    g = np.random.default_rng(1)
    u, pmin = g.uniform(0, 1, 100000), g.uniform(0, 1, 100000)
    p = pmin + (1 - pmin) * g.uniform(0, 1, 100000)
    assert np.all(geometry.hamerly_upper_update(u, pmin) >= geometry.cos_upper_bound(u, p) - 1e-12)
    # the reference's pitfall counter-example (tests/test_geometry.py:108-116)
    assert geometry.hamerly_upper_update(0.95, 0.5) >= geometry.update_upper_bound(0.95, 0.9)


# ------------------------------------------------------------------ numerics helpers
def test_row_eps_rounds_up_and_covers_fp32_error():
    m = np.array([1, 5, 50, 400])
    e = row_eps(m)
    assert e.dtype == np.float32
    assert np.all(e.astype(np.float64) >= (m + 6) * 6.1e-8)
    assert np.all(e.astype(np.float64) >= (m + 2) * 2.0 ** -24 * 1.001)


def test_fixed_point_scale_headroom():
    for n in (5, 2000, 20000, 500_000, 4_000_000, 10_000_000):
        s = scale_bits_for(n)
        assert n * 2.0 ** s <= 2.0 ** 62
    assert scale_bits_for(4_000_000) == 40


# ------------------------------------------------------------------ generator
def test_generator_deterministic_and_shaped():
    spec = synth.CorpusSpec("t", 3000, 5000, 50)
    a = synth.sparse_corpus(spec, seed=5)
    b = synth.sparse_corpus(spec, seed=5)
    assert np.array_equal(a.indptr, b.indptr) and np.array_equal(a.indices, b.indices)
    assert np.array_equal(a.data, b.data)
    L = a.row_lengths()
    assert L.min() >= 1 and L.max() <= 400
    assert 40 <= L.mean() <= 60
    # sorted unique indices per row, unit rows, positive tf-idf
    same = np.repeat(np.arange(a.n), L)
    d = np.diff(a.indices.astype(np.int64))
    assert np.all(d[same[1:] == same[:-1]] > 0)
    norms = np.sqrt(np.add.reduceat(a.data ** 2, a.indptr[:-1]))
    assert np.allclose(norms, 1.0, atol=1e-12)
    assert np.all(a.data > 0)


def test_generator_topics_concentrate_terms():
    spec = synth.CorpusSpec("t", 2000, 20000, 60, topics=10, topic_size=300)
    d = synth.sparse_corpus(spec, seed=1)
    df = np.bincount(d.indices, minlength=spec.d)
    top = np.sort(df)[::-1][:3000]
    assert top.sum() / df.sum() > 0.6       # ~70% of draws come from 10 x 300 topic ids


def test_dense_corpus_unit_rows():
    X, lab = synth.dense_corpus(2000, d=16, centers=5, seed=3)
    assert X.shape == (2000, 16) and X.dtype == np.float32
    assert np.allclose(np.linalg.norm(X, axis=1), 1.0, atol=1e-6)
    assert lab.min() >= 0 and lab.max() < 5


def test_device_corpus_permutations_roundtrip():
    """Rows longest-first and terms by document frequency: the device CSR holds the same rows."""
    import torch
    from paper_2107_04074_b200.engine import DeviceCorpus
    spec = synth.CorpusSpec("t", 500, 2000, 30)
    data = synth.sparse_corpus(spec, seed=3)
    for rows in [(0, data.n), (100, 357)]:
        dc = DeviceCorpus(data, torch.device("cpu"), rows=rows)
        ip, ix, dv = (t.numpy() for t in (dc.indptr, dc.indices, dc.values))
        lens = np.diff(ip)
        assert np.all(lens[:-1] >= lens[1:])                  # longest first
        for j in range(0, dc.n, 7):
            h = rows[0] + dc.row_perm[j]
            s, e = data.indptr[h], data.indptr[h + 1]
            assert np.array_equal(dc.order[ix[ip[j]:ip[j + 1]]], data.indices[s:e])   # same terms, CSR order kept
            assert np.array_equal(dv[ip[j]:ip[j + 1]], data.data[s:e].astype(np.float32))
        x = np.arange(dc.n)
        assert np.array_equal(dc.to_host_rows(dc.to_device_rows(x)), x)
    df = np.bincount(data.indices, minlength=data.dim)
    assert np.all(np.diff(df[dc.order]) <= 0)                  # hottest terms first


def test_from_csr_normalises_like_from_rows():
    """Dataset.from_csr row norms use the reference's np.dot order, so the
    normalised values are bit-identical to Dataset.from_rows (sparse.py:52-58)."""
    from paper_2107_04074_b200.sparse import Dataset, SparseVector
    g = np.random.default_rng(3)
    lens = g.integers(1, 420, 400)
    ip = np.zeros(lens.size + 1, np.int64)
    np.cumsum(lens, out=ip[1:])
    idx = np.concatenate([np.sort(g.choice(5000, m, replace=False)) for m in lens]).astype(np.int64)
    val = g.standard_normal(ip[-1]) * g.random(ip[-1]) ** 3 + 1e-3
    a = Dataset.from_csr(ip, idx, val, 5000)
    rows = [SparseVector(idx[ip[i]:ip[i + 1]], val[ip[i]:ip[i + 1]]) for i in range(lens.size)]
    b = Dataset.from_rows(rows, dim=5000)
    assert np.array_equal(a.data, np.concatenate([r.values for r in b.rows]))


def test_dataset_reference_constructor_forms():
    """Dataset(rows=..., dim=...) / Dataset(rows, dim): the reference dataclass
    form (sparse.py:101-115, rows taken as given) next to the CSR form."""
    from paper_2107_04074_b200.sparse import Dataset, SparseVector
    rows = [SparseVector(np.array([0, 3]), np.array([0.6, 0.8])), SparseVector(np.array([2]), np.array([1.0]))]
    a = Dataset(rows=rows, dim=5)
    b = Dataset(rows, 5)
    c = Dataset.from_rows(rows, dim=5, normalize_rows=False)
    for ds in (a, b):
        assert ds.n == 2 and ds.dim == 5 and ds.rows[0] is rows[0]
        assert np.array_equal(ds.indptr, c.indptr) and np.array_equal(ds.indices, c.indices)
        assert np.array_equal(ds.data, c.data)
        ip, ix, dv = ds.csr_arrays()
        assert ix.dtype == np.int64 and list(ip) == [0, 2, 3]
    d = Dataset(c.indptr, c.indices, c.data, 5)
    assert np.array_equal(d.data, c.data) and d.rows[1].indices.tolist() == [2]
    with pytest.raises(TypeError):
        Dataset(rows)
    with pytest.raises(TypeError):
        Dataset(c.indptr, c.indices, 5)


def test_yinyang_is_an_extra_variant():
    """VARIANTS stays the reference's five; "yinyang" is accepted on top."""
    from paper_2107_04074_b200 import engine
    assert spk.VARIANTS == ("standard", "elkan", "simp_elkan", "hamerly", "simp_hamerly")
    assert "yinyang" in engine.EXTRA_VARIANTS
    data = Dataset.from_csr(np.array([0, 1, 2]), np.array([0, 1]), np.array([1.0, 1.0]), 2)
    engine._validate(data, 2, "yinyang", "safe")
    with pytest.raises(spk.ConfigError):
        engine._validate(data, 2, "yin_yang", "safe")
