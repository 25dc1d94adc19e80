"""GPU kernel-level parity and the reference test suite's engine properties (through the C ABI).

Mirrors /root/reference/pkg/tests/test_engine.py, test_validation.py and
test_acceptance.py (#2 soundness, #4 pitfall, #5 efficacy, #6 monotone,
#7 cc accounting) against the CUDA path.
"""

import numpy as np
import pytest
import torch

from conftest import GOLDEN, golden_dataset, load_golden

pytestmark = pytest.mark.gpu

VARIANTS = ("standard", "elkan", "simp_elkan", "hamerly", "simp_hamerly")


def spk():
    import paper_2107_04074_b200 as m
    return m


def sv(pairs):
    from paper_2107_04074_b200.sparse import SparseVector
    idx, val = zip(*pairs)
    return SparseVector(np.array(idx), np.array(val, dtype=float))


# ------------------------------------------------------------------ device geometry
@pytest.mark.parametrize("op,key", [(0, "lower"), (1, "upper"), (2, "hamerly"), (3, "half_angle")])
def test_device_geometry_bit_exact(op, key):
    from paper_2107_04074_b200 import _lib
    z = np.load(GOLDEN / "geometry.npz")
    a = torch.from_numpy(z["a"]).cuda()
    b = torch.from_numpy(z["b"]).cuda()
    out = torch.empty_like(a)
    import ctypes
    _lib.call("spkm_geometry", op, a.numel(), a.data_ptr(), b.data_ptr(), out.data_ptr(), ctypes.c_void_p(0))
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), z[key]), key


def test_device_lower_update_guard():
    """l < -p -> -1 (theta_l + theta_p > pi), SURVEY.md §2.4 item 6."""
    from paper_2107_04074_b200 import _lib
    import ctypes
    l = torch.tensor([np.cos(0.6 * np.pi), 0.5], dtype=torch.float64, device="cuda")
    p = torch.tensor([np.cos(0.6 * np.pi) * -1 + 0.0 - 0.5, 0.9], dtype=torch.float64, device="cuda")
    out = torch.empty_like(l)
    _lib.call("spkm_geometry", 4, 2, l.data_ptr(), p.data_ptr(), out.data_ptr(), ctypes.c_void_p(0))
    torch.cuda.synchronize()
    o = out.cpu().numpy()
    assert o[0] == -1.0
    assert o[1] == pytest.approx(0.5 * 0.9 - np.sqrt(0.75 * 0.19), abs=1e-15)


# ------------------------------------------------------------------ predict / objective
def test_assign_full_matches_oracle(oracle_mod):
    z = load_golden("C1")
    data = golden_dataset(z)
    X = oracle_mod.CSR(z["indptr"], z["indices"], z["data"], int(z["dim"]))
    r = oracle_mod.run(X, 20, "standard", seed=1, max_iter=3)
    a_ref, best_ref, second_ref = oracle_mod.assign_full(X, r["centers"])
    a, best, second = spk().assign_full(data, r["centers"])
    ok = (best_ref - second_ref) > 1e-5
    assert np.array_equal(a[ok], a_ref[ok])
    assert np.max(np.abs(best - best_ref)) < 3e-5
    assert np.max(np.abs(second - second_ref)) < 3e-5
    assert np.all(best >= second)


def test_tie_breaks_to_lowest_index():
    m = spk()
    data = m.Dataset.from_rows([sv([(0, 1.0)]), sv([(1, 1.0)])], dim=2)
    a, _, _ = m.assign_full(data, np.array([[1.0, 0.0], [1.0, 0.0]]))
    assert list(a) == [0, 0]


def test_compute_objective_matches_oracle(oracle_mod):
    z = load_golden("small")
    data = golden_dataset(z)
    X = oracle_mod.CSR(z["indptr"], z["indices"], z["data"], int(z["dim"]))
    r = oracle_mod.run(X, 7, "standard", seed=11, max_iter=100)
    got = spk().compute_objective(data, r["assignments"], r["centers"])
    S = oracle_mod.full_sims(X, r["centers"])
    ref = float(S[np.arange(data.n), r["assignments"]].sum())
    assert got == pytest.approx(ref, rel=1e-6)


# ------------------------------------------------------------------ center updates
def test_incremental_update_equals_scratch_bitwise():
    m = spk()
    z = load_golden("small")
    data = golden_dataset(z)
    g = np.random.default_rng(0)
    k = 6
    a0 = g.integers(0, k, data.n)
    cs = m.CentroidSet.from_data_rows(data, range(k))
    m.update_centers(data, a0, cs)
    a1 = a0.copy()
    flip = g.choice(data.n, 40, replace=False)
    a1[flip] = g.integers(0, k, 40)
    m.update_centers(data, a1, cs, prev_assignments=a0)
    sc = m.CentroidSet.from_data_rows(data, range(k))
    m.update_centers(data, a0, sc)
    m.update_centers(data, a1, sc)
    assert np.array_equal(cs.counts, sc.counts)
    assert np.array_equal(cs.sums, sc.sums)          # exact fixed point: bit-identical
    assert np.allclose(cs.centers, sc.centers, atol=1e-12)


def test_untouched_cluster_bit_identical_and_empty_cluster_kept():
    m = spk()
    z = load_golden("small")
    data = golden_dataset(z)
    k = 4
    a0 = np.zeros(data.n, dtype=np.int64)
    a0[: data.n // 2] = 1
    a0[:10] = 2
    a0[10:20] = 3
    cs = m.CentroidSet.from_data_rows(data, range(k))
    m.update_centers(data, a0, cs)
    frozen = cs.centers[3].copy()
    a1 = a0.copy()
    a1[0] = 1
    m.update_centers(data, a1, cs, prev_assignments=a0)
    assert np.array_equal(cs.centers[3], frozen)
    assert cs.drift[3] == 1.0
    cs2 = m.CentroidSet.from_data_rows(data, range(3))
    before = cs2.centers[2].copy()
    a = np.zeros(data.n, dtype=np.int64)
    a[:5] = 1
    m.update_centers(data, a, cs2)
    assert np.array_equal(cs2.centers[2], before)
    assert cs2.drift[2] == 1.0


# ------------------------------------------------------------------ engine properties
def test_k1_and_k_equals_n():
    m = spk()
    z = load_golden("small")
    data = golden_dataset(z)
    for v in VARIANTS:
        r = m.run(data, 1, v, m.SeedConfig(seed=3))
        assert r.converged and len(r.iterations) == 1 and np.all(r.assignments == 0)
    five = golden_dataset(load_golden("five_points"))
    r = m.run(five, 5, "standard", m.SeedConfig(seed=0))
    assert r.converged and len(r.iterations) <= 2          # reference: 1 (iteration count +-1)
    assert sorted(r.assignments.tolist()) == [0, 1, 2, 3, 4]


def test_instrumentation_and_max_iter():
    m = spk()
    data = golden_dataset(load_golden("small"))
    r = m.run(data, 4, "standard", m.SeedConfig(seed=1))
    assert r.iterations[0].reassignments == data.n
    assert all(s.sim_count == data.n * 4 and s.cc_sim_count == 0 for s in r.iterations)
    assert r.iterations[-1].reassignments == 0
    assert len(m.run(data, 10, "standard", m.SeedConfig(seed=1), max_iter=2).iterations) <= 2
    k = 8
    for v in ("elkan", "hamerly"):
        r = m.run(data, k, v, m.SeedConfig(seed=5))
        assert all(s.cc_sim_count == k * (k - 1) // 2 for s in r.iterations)
    for v in ("standard", "simp_elkan", "simp_hamerly"):
        assert m.run(data, k, v, m.SeedConfig(seed=5)).total_cc_sims == 0


def test_objective_monotone_and_deterministic():
    m = spk()
    data = golden_dataset(load_golden("grid_2000_5000_20_2000"))
    for v in VARIANTS:
        r = m.run(data, 20, v, m.SeedConfig(seed=13))
        objs = [s.objective for s in r.iterations]
        assert all(b >= a - 1e-9 * data.n for a, b in zip(objs, objs[1:])), v
        r2 = m.run(data, 20, v, m.SeedConfig(seed=13))
        assert np.array_equal(r.assignments, r2.assignments) and r.objective == r2.objective
        assert [s.sim_count for s in r.iterations] == [s.sim_count for s in r2.iterations]


def test_pruning_efficacy_clustered():
    """Acceptance #5 on the regenerated clustered_2000x5000 fixture, k=20, seed=3."""
    m = spk()
    data = golden_dataset(load_golden("clustered"))
    tot = {v: m.run(data, 20, v, m.SeedConfig(seed=3)).total_sims for v in ("standard", "elkan", "hamerly")}
    assert tot["elkan"] / tot["standard"] < 0.5
    assert tot["hamerly"] / tot["standard"] < 1.0


# ------------------------------------------------------------------ bound soundness audits
class Auditor:
    """validation._BoundAuditor (validation.py:49-80) with the oracle's exact fp64 similarities."""

    def __init__(self, O, X):
        self.O, self.X = O, X
        self.max_lower = self.max_upper = 0.0
        self.count = 0

    def __call__(self, it, bounds, cents):
        S = self.O.full_sims(self.X, cents.centers)
        n = S.shape[0]
        own = S[np.arange(n), bounds.a]
        self.max_lower = max(self.max_lower, float(np.max(bounds.l - own)))
        self.count += n
        if bounds.u_matrix is not None:
            self.max_upper = max(self.max_upper, float(np.max(S - bounds.u_matrix)))
            self.count += S.size
        elif bounds.u is not None and S.shape[1] > 1:
            mm = S.copy()
            mm[np.arange(n), bounds.a] = -np.inf
            self.max_upper = max(self.max_upper, float(np.max(mm.max(axis=1) - bounds.u)))
            self.count += n


@pytest.mark.parametrize("name,k,seed", [("small", 7, 11), ("signed", 6, 2), ("grid_200_256_10_3000", 10, 3007),
                                         ("C1", 20, 1), ("clustered", 20, 3)])
@pytest.mark.parametrize("variant", VARIANTS[1:])
def test_bounds_sound_every_iteration(oracle_mod, name, k, seed, variant):
    m = spk()
    z = load_golden(name)
    data = golden_dataset(z)
    X = oracle_mod.CSR(z["indptr"], z["indices"], z["data"], int(z["dim"]))
    aud = Auditor(oracle_mod, X)
    m.run(data, k, variant, m.SeedConfig(seed=seed), debug_hook=aud)
    assert aud.max_lower <= 1e-9 and aud.max_upper <= 1e-9, (aud.max_lower, aud.max_upper)


def test_pitfall_naive_violates_safe_passes(oracle_mod):
    """Acceptance #4 (tests/test_acceptance.py:114-123) on the GPU bounds."""
    m = spk()
    z = load_golden("pitfall")
    data = golden_dataset(z)
    X = oracle_mod.CSR(z["indptr"], z["indices"], z["data"], int(z["dim"]))
    naive, safe = Auditor(oracle_mod, X), Auditor(oracle_mod, X)
    m.run(data, 5, "hamerly", m.SeedConfig(seed=1), debug_hook=naive, hamerly_update="naive")
    m.run(data, 5, "hamerly", m.SeedConfig(seed=1), debug_hook=safe)
    assert naive.max_upper > 1e-9
    assert safe.max_upper <= 1e-9 and safe.max_lower <= 1e-9


# ------------------------------------------------------------------ edge cases
def test_single_nnz_rows_and_duplicates():
    m = spk()
    rows = [sv([(i % 7, 1.0)]) for i in range(60)] + [sv([(0, 1.0), (1, 1.0)])] * 5
    data = m.Dataset.from_rows(rows, dim=7)
    base = None
    for v in VARIANTS:
        r = m.run(data, 5, v, m.SeedConfig(seed=4))
        if base is None:
            base = r
        assert np.array_equal(r.assignments, base.assignments), v
        assert r.objective == base.objective


def test_max_length_rows(oracle_mod):
    """Rows at the generator's 400-nnz clip mixed with 1-nnz rows."""
    m = spk()
    g = np.random.default_rng(11)
    n, d = 300, 5000
    lens = np.where(np.arange(n) % 3 == 0, 400, np.where(np.arange(n) % 3 == 1, 1, 37))
    ip = np.concatenate([[0], np.cumsum(lens)])
    idx = np.concatenate([np.sort(g.choice(d, L, replace=False)) for L in lens])
    val = g.uniform(0.1, 1.0, idx.size)
    data = m.Dataset.from_csr(ip, idx, val, d)
    assert data.row_lengths().max() == 400
    X = oracle_mod.CSR(data.indptr, data.indices, data.data, data.dim)
    ref = oracle_mod.run(X, 8, "standard", seed=5, max_iter=50)
    margin = oracle_mod.margins(X, ref["centers"])
    base = None
    for v in VARIANTS:
        r = m.run(data, 8, v, m.SeedConfig(seed=5), max_iter=50)
        ok = margin > 1e-5
        assert np.array_equal(r.assignments[ok], ref["assignments"][ok]), v
        assert r.objective == pytest.approx(ref["objective"][-1], rel=1e-6)
        base = base or r
        assert np.array_equal(r.assignments, base.assignments), v


@pytest.mark.parametrize("name,k", [("C1", 20), ("grid_200_5000_50_1007", 50), ("signed", 6), ("C1", 200),
                                    ("C1", 300)])
def test_center_thresholds_upper_bound(name, k):
    """cc from the 3xTF32 tensor-core Gram is an upper bound within 1e-4 of the float64 half-angle cosine."""
    from paper_2107_04074_b200 import engine as E
    z = load_golden(name)
    data = golden_dataset(z)
    eng = E.Engine(data, k, "elkan")
    eng.seed_rows(data, np.arange(k))
    eng.reset()
    eng.iteration(1)
    eng.center_thresholds()
    torch.cuda.synchronize()
    C = eng.C.host_centers()
    G = np.clip(C @ C.T, -1, 1)
    cc_ref = np.sqrt(np.maximum(0.0, (G + 1) / 2))
    np.fill_diagonal(cc_ref, -1.0)
    cc = eng.C.cc.view(k, k).cpu().numpy().astype(np.float64)
    off = ~np.eye(k, dtype=bool)
    assert np.all(cc[off] >= cc_ref[off]), float(np.min(cc[off] - cc_ref[off]))
    assert np.max(cc[off] - cc_ref[off]) < 1e-4
    s = eng.C.s.cpu().numpy()
    assert np.array_equal(s, np.where(off, cc, -np.inf).max(axis=1).astype(np.float32))


def test_seed_rows_match_host_densify():
    from paper_2107_04074_b200 import engine as E
    z = load_golden("C1")
    data = golden_dataset(z)
    rows = [5, 17, 1999, 0]
    eng = E.Engine(data, 4, "standard")
    eng.seed_rows(data, rows)
    torch.cuda.synchronize()
    assert np.array_equal(eng.C.host_centers(), data.densify_rows(rows))
    ct = eng.C.ct32[:data.dim * eng.C.kp].view(data.dim, eng.C.kp)[:, :4].cpu().numpy()[eng.corpus.new_id]   # device rows are renumbered
    assert np.array_equal(ct, data.densify_rows(rows).T.astype(np.float32))


@pytest.mark.parametrize("variant", VARIANTS)
def test_cuda_graph_replay_matches_eager(variant):
    """Steady-state iterations replayed as one CUDA graph give bit-identical results."""
    m = spk()
    data = golden_dataset(load_golden("C1"))
    m.run(data, 20, variant, m.SeedConfig(seed=1), max_iter=50, use_graphs=True)       # eager, warms the engine
    g = m.run(data, 20, variant, m.SeedConfig(seed=1), max_iter=50, use_graphs=True)   # captured + replayed
    e = m.run(data, 20, variant, m.SeedConfig(seed=1), max_iter=50, use_graphs=False)
    assert np.array_equal(g.assignments, e.assignments)
    assert g.objective == e.objective
    assert [s.sim_count for s in g.iterations] == [s.sim_count for s in e.iterations]
    assert [s.reassignments for s in g.iterations] == [s.reassignments for s in e.iterations]
    assert len(g.iterations) >= 3


@pytest.mark.parametrize("variant", ["standard", "elkan", "hamerly"])
def test_device_loop_max_iter_and_reuse(variant):
    """The device-driven loop (conditional WHILE graph) stops exactly at
    max_iter or at convergence, across repeated fits with different limits,
    and equals the eager host loop."""
    m = spk()
    data = golden_dataset(load_golden("C1"))
    m.run(data, 20, variant, m.SeedConfig(seed=4), max_iter=50, use_graphs=True)   # warm (eager)
    for mi in (1, 2, 3, 4, 7, 50, 5):
        g = m.run(data, 20, variant, m.SeedConfig(seed=4), max_iter=mi, use_graphs=True)
        e = m.run(data, 20, variant, m.SeedConfig(seed=4), max_iter=mi, use_graphs=False)
        assert len(g.iterations) == len(e.iterations) <= mi
        assert g.converged == e.converged
        assert np.array_equal(g.assignments, e.assignments)
        assert g.objective == e.objective
        assert [s.reassignments for s in g.iterations] == [s.reassignments for s in e.iterations]
        assert all(s.elapsed_ns > 0 for s in g.iterations)


@pytest.mark.parametrize("variant", VARIANTS)
def test_whole_fit_graph_matches_eager_across_seeds(variant):
    """From the second fit on, an engine runs the whole fit as one CUDA graph
    (seed upload, iterations 1-2, WHILE loop, result downloads) with the seed
    rows and max_iter read from pinned memory at launch: every fit equals
    the eager host loop (stats, assignments, centers, counts, sums)."""
    m = spk()
    data = golden_dataset(load_golden("C1"))
    m.run(data, 12, variant, m.SeedConfig(seed=1), max_iter=30, use_graphs=True)   # first fit: eager
    for seed, mi in ((5, 30), (6, 30), (5, 4), (7, 30)):
        g = m.run(data, 12, variant, m.SeedConfig(seed=seed), max_iter=mi, use_graphs=True)
        e = m.run(data, 12, variant, m.SeedConfig(seed=seed), max_iter=mi, use_graphs=False)
        assert len(g.iterations) == len(e.iterations) <= mi
        assert g.converged == e.converged
        assert np.array_equal(g.assignments, e.assignments)
        assert g.assignments.dtype == e.assignments.dtype
        assert g.objective == e.objective
        for a, b in zip(g.iterations, e.iterations):
            assert (a.iteration, a.sim_count, a.cc_sim_count, a.reassignments, a.objective) == \
                (b.iteration, b.sim_count, b.cc_sim_count, b.reassignments, b.objective)
        assert np.array_equal(g.centers.centers, e.centers.centers)
        assert np.array_equal(g.centers.counts, e.centers.counts)
        assert np.array_equal(g.centers.sums, e.centers.sums)
        assert list(g.centers.seed_indices) == list(e.centers.seed_indices)


@pytest.mark.parametrize("variant", ["standard", "elkan", "hamerly"])
def test_sharded_path_single_rank_matches_run(variant):
    """distributed.run_sharded (replicated corpus, move slots, assignment
    allgather) on a one-rank NCCL group gives the single-process result
    bit-for-bit (the kernels of the multi-GPU exchange run; the collectives
    are trivial at world size 1)."""
    import os
    import socket
    import torch.distributed as dist
    from paper_2107_04074_b200.distributed import run_sharded
    m = spk()
    data = golden_dataset(load_golden("C1"))
    if not dist.is_initialized():
        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
        s.close()
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        r = run_sharded(data, 20, variant, m.SeedConfig(seed=5), max_iter=30)
        e = m.run(data, 20, variant, m.SeedConfig(seed=5), max_iter=30, use_graphs=False)
        assert np.array_equal(r.assignments, e.assignments)
        assert r.objective == e.objective
        assert [s.reassignments for s in r.iterations] == [s.reassignments for s in e.iterations]
        assert [s.sim_count for s in r.iterations] == [s.sim_count for s in e.iterations]
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("variant", ["standard", "elkan", "hamerly"])
def test_result_sums_rebuilt_on_host_equal_device_aggregate(variant):
    """run() results rebuild the fixed-point sums on the host from the final
    assignments instead of copying k x d int64 on the device; they must equal
    a from-scratch device aggregation bit for bit."""
    m = spk()
    z = load_golden("small")
    data = golden_dataset(z)
    k = 5
    r = m.run(data, k, variant, m.SeedConfig(seed=3), max_iter=20)
    cs = m.CentroidSet.from_data_rows(data, range(k))
    m.update_centers(data, r.assignments, cs)
    assert np.array_equal(r.centers.sums, cs.sums)
    assert np.array_equal(r.centers.counts, cs.counts)


@pytest.mark.parametrize("variant", ["hamerly", "simp_hamerly"])
def test_hamerly_fused_rescan_matches_separate_tighten(variant, monkeypatch):
    """The rescan that applies the tighten test itself (SPKM_HAMERLY_FUSE=1)
    and the separate tighten kernel (=0) give identical fits, iteration
    statistics included (eager loop: the policy is read at every launch)."""
    m = spk()
    data = golden_dataset(load_golden("C1"))
    out = {}
    for pol in ("0", "1", "2"):
        monkeypatch.setenv("SPKM_HAMERLY_FUSE", pol)
        r = m.run(data, 12, variant, m.SeedConfig(seed=3), max_iter=30, use_graphs=False)
        out[pol] = r
    ref = out["0"]
    for pol in ("1", "2"):
        r = out[pol]
        assert np.array_equal(r.assignments, ref.assignments)
        assert r.objective == ref.objective
        key = lambda s: (s.sim_count, s.reassignments, s.survivors, s.survivors2, s.nnz_tighten, s.nnz_rescan,
                         s.objective)
        assert [key(s) for s in r.iterations] == [key(s) for s in ref.iterations]


@pytest.mark.parametrize("variant", ["elkan", "simp_elkan"])
@pytest.mark.parametrize("graphs", [False, True])
def test_elkan_fused_bounds_scan_matches_two_passes(variant, graphs, monkeypatch):
    """spkm_elkan_bounds_scan (drift update + prune test + scan in one pass)
    and spkm_elkan_bounds + spkm_elkan_scan give identical fits and iteration
    statistics."""
    from paper_2107_04074_b200 import engine as E
    m = spk()
    data = golden_dataset(load_golden("C1"))
    out = {}
    for fuse in ("0", "1"):
        monkeypatch.setenv("SPKM_ELKAN_FUSE", fuse)
        E.clear_engine_cache()
        for _ in range(2 if graphs else 1):    # the second fit runs the captured whole-fit graph
            r = m.run(data, 12, variant, m.SeedConfig(seed=3), max_iter=30, use_graphs=graphs)
        out[fuse] = r
    E.clear_engine_cache()
    a, b = out["0"], out["1"]
    assert np.array_equal(a.assignments, b.assignments)
    assert a.objective == b.objective
    key = lambda s: (s.sim_count, s.reassignments, s.survivors, s.nnz_elkan, s.objective)
    assert [key(s) for s in a.iterations] == [key(s) for s in b.iterations]


def test_order_by_cluster_is_a_grouping_permutation():
    """spkm_order_by_cluster: in-place on a list with a device count, and the
    identity form; the output holds the same rows, grouped by a(i) ascending."""
    import ctypes
    from paper_2107_04074_b200 import _lib
    g = np.random.default_rng(5)
    n, k = 100_003, 777
    a = torch.from_numpy(g.integers(0, k, n).astype(np.int32)).cuda()
    lst_h = g.permutation(n)[:60_001].astype(np.int32)
    lst = torch.from_numpy(np.concatenate([lst_h, np.full(n - lst_h.size, -7, np.int32)])).cuda()
    cnt = torch.tensor([lst_h.size], dtype=torch.int64, device="cuda")
    ctl = torch.zeros(2, dtype=torch.int64, device="cuda")
    tmp = torch.empty(n, dtype=torch.int32, device="cuda")
    bins = torch.empty(2 * k, dtype=torch.int32, device="cuda")
    out = torch.empty(n, dtype=torch.int32, device="cuda")
    s = ctypes.c_void_p(0)
    _lib.call("spkm_order_by_cluster", k, a.data_ptr(), lst.data_ptr(), cnt.data_ptr(), n, tmp.data_ptr(), None,
              bins.data_ptr(), ctl.data_ptr(), s)
    _lib.call("spkm_order_by_cluster", k, a.data_ptr(), None, None, n, tmp.data_ptr(), out.data_ptr(),
              bins.data_ptr(), ctl.data_ptr(), s)
    torch.cuda.synchronize()
    ah = a.cpu().numpy()
    got = lst.cpu().numpy()
    assert np.array_equal(got[lst_h.size:], np.full(n - lst_h.size, -7))      # past the count: untouched
    got = got[:lst_h.size]
    assert np.array_equal(np.sort(got), np.sort(lst_h))
    assert np.all(np.diff(ah[got]) >= 0)
    full = out.cpu().numpy()
    assert np.array_equal(np.sort(full), np.arange(n))
    assert np.all(np.diff(ah[full]) >= 0)
    # converged (ctl[1] != 0): a no-op
    ctl[1] = 1
    before = lst.clone()
    _lib.call("spkm_order_by_cluster", k, a.data_ptr(), lst.data_ptr(), cnt.data_ptr(), n, tmp.data_ptr(), None,
              bins.data_ptr(), ctl.data_ptr(), s)
    torch.cuda.synchronize()
    assert torch.equal(before, lst)


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("graphs", [False, True])
def test_cluster_ordered_worklists_give_identical_fits(variant, graphs, monkeypatch):
    """Survivor lists ordered by cluster (SPKM_ORDER=1, the default when the
    center table exceeds L2) give the same fit and iteration statistics as
    storage order (=0): the scans' results do not depend on visiting order."""
    from paper_2107_04074_b200 import engine as E
    m = spk()
    data = golden_dataset(load_golden("C1"))
    monkeypatch.setenv("SPKM_ELKAN_FUSE", "0")      # the Elkan survivor list exists only unfused
    out = {}
    for order in ("0", "1"):
        monkeypatch.setenv("SPKM_ORDER", order)
        E.clear_engine_cache()
        for _ in range(2 if graphs else 1):
            r = m.run(data, 12, variant, m.SeedConfig(seed=3), max_iter=30, use_graphs=graphs)
        out[order] = r
    E.clear_engine_cache()
    a, b = out["0"], out["1"]
    assert np.array_equal(a.assignments, b.assignments)
    assert a.objective == b.objective
    key = lambda s: (s.sim_count, s.reassignments, s.survivors, s.survivors2, s.nnz_elkan, s.nnz_rescan,
                     s.objective)
    assert [key(s) for s in a.iterations] == [key(s) for s in b.iterations]




@pytest.mark.parametrize("k", [300, 1000])
@pytest.mark.parametrize("variant", ["standard", "hamerly", "simp_hamerly", "elkan", "yinyang"])
def test_sparse_center_index_full_pass_equals_dense(k, variant, monkeypatch):
    """SPKM_CSPARSE=1: the full passes gather the centers through the sparse
    term-major index (spkm_cindex) -- the same canonical chains, so the fit is
    the dense-gather fit bit for bit, counters included."""
    from paper_2107_04074_b200 import engine, synth
    m = spk()
    data = synth.config_dataset("C3", n_override=20_000)
    engine.clear_engine_cache()
    monkeypatch.setenv("SPKM_CSPARSE", "0")
    monkeypatch.setenv("SPKM_EK_HEAVY_PCT", "0")     # the heavy-row pass changes the counters (tested below)
    ref = m.run(data, k, variant, m.SeedConfig(seed=3), max_iter=30)
    monkeypatch.setenv("SPKM_CSPARSE", "1")
    engine.clear_engine_cache()
    for graphs in (False, True, True):
        r = m.run(data, k, variant, m.SeedConfig(seed=3), max_iter=30, use_graphs=graphs)
        assert np.array_equal(r.assignments, ref.assignments)
        assert r.objective == ref.objective
        key = lambda s: (s.sim_count, s.reassignments, s.survivors, s.survivors2, s.nnz_rescan)  # noqa: E731
        assert [key(s) for s in r.iterations] == [key(s) for s in ref.iterations]
    engine.clear_engine_cache()


@pytest.mark.parametrize("k", [300, 1000])
@pytest.mark.parametrize("variant", ["elkan", "simp_elkan"])
def test_elkan_heavy_rows_full_pass_equals_scan(k, variant, monkeypatch):
    """spkm_elkan_heavy: rows with many unpruned centers take one full pass over
    the sparse center index instead of the block scan.  Both are the Lloyd
    argmax on the canonical s~ (incumbent wins ties, else the lowest index), so
    assignments, objective and per-iteration reassignments equal the scan-only
    fit and the GPU Lloyd for every threshold; the full pass computes k
    similarities per row, so sim_count can only differ."""
    from paper_2107_04074_b200 import engine, synth
    m = spk()
    data = synth.config_dataset("C3", n_override=20_000)
    engine.clear_engine_cache()
    monkeypatch.setenv("SPKM_EK_HEAVY_PCT", "0")
    ref = m.run(data, k, variant, m.SeedConfig(seed=3), max_iter=30)
    lloyd = m.run(data, k, "standard", m.SeedConfig(seed=3), max_iter=30)
    assert np.array_equal(ref.assignments, lloyd.assignments) and ref.objective == lloyd.objective
    assert all(s.survivors2 == 0 for s in ref.iterations)
    # SPKM_EK_ALLHEAVY: while an iteration moves >= n / 256 rows the next one skips the bound pass and every
    # row takes the full pass (a performance switch; "0" keeps the bound pass in every iteration)
    for pct, allheavy in (("1", "0"), ("25", "0"), ("60", "0"), ("1", "1"), ("25", "1")):
        monkeypatch.setenv("SPKM_EK_HEAVY_PCT", pct)
        monkeypatch.setenv("SPKM_EK_ALLHEAVY", allheavy)
        engine.clear_engine_cache()
        for graphs in (False, True, True):
            r = m.run(data, k, variant, m.SeedConfig(seed=3), max_iter=30, use_graphs=graphs)
            assert np.array_equal(r.assignments, ref.assignments)
            assert r.objective == ref.objective
            assert [s.reassignments for s in r.iterations] == [s.reassignments for s in ref.iterations]
            assert any(s.survivors2 > 0 for s in r.iterations[1:])       # the heavy pass did run
            if allheavy == "0":
                assert (sum(s.survivors + s.survivors2 for s in r.iterations[1:])
                        <= sum(s.survivors for s in ref.iterations[1:]))     # exact u(i, j): never more survivors
            else:
                assert r.iterations[1].survivors2 == data.n and r.iterations[1].survivors == 0   # iteration 2: all rows
    engine.clear_engine_cache()


def test_elkan_heavy_rows_bounds_audited(monkeypatch):
    """Bounds written by the heavy pass (l and every u(i, j) exact + eps) pass
    the device auditor at every iteration, mixed with the block scan's."""
    from paper_2107_04074_b200 import engine, synth, validation
    data = synth.config_dataset("C3", n_override=20_000)
    for pct in ("1", "10"):
        monkeypatch.setenv("SPKM_EK_HEAVY_PCT", pct)
        engine.clear_engine_cache()
        for variant in ("elkan", "simp_elkan"):
            rep = validation.audit_bounds(data, variant, 300, seed=3, max_iter=12)
            assert rep.passed, rep
            assert rep.decisions_audited > 0
    engine.clear_engine_cache()


@pytest.mark.parametrize("k", [300, 1000])
def test_elkan_light_rows_listed_centers_equal_block_scan(k, monkeypatch):
    """simp_elkan, default heavy threshold (ceil(k / 200) <= 5): the bound pass lists each light row's
    failing centers and k_elkan_light computes exactly those.  Same scan semantics as k_elkan_scan, so
    the fit AND every counter (sim_count, survivors, nnz) equal the block-scan fit (SPKM_EK_LIGHT=0)."""
    from paper_2107_04074_b200 import engine, synth
    m = spk()
    data = synth.config_dataset("C3", n_override=20_000)
    key = lambda s: (s.sim_count, s.reassignments, s.survivors, s.survivors2, s.nnz_elkan, s.nnz_rescan)  # noqa: E731
    for pct in (None, "1.5"):          # k = 300: thresholds 2 and 5; k = 1000: 5 and 15 (15: no lists, same path twice)
        if pct is None:
            monkeypatch.delenv("SPKM_EK_HEAVY_PCT", raising=False)
        else:
            monkeypatch.setenv("SPKM_EK_HEAVY_PCT", pct)
        monkeypatch.setenv("SPKM_EK_LIGHT", "0")
        engine.clear_engine_cache()
        ref = m.run(data, k, "simp_elkan", m.SeedConfig(seed=3), max_iter=30)
        if k == 300:
            assert any(s.survivors > 0 for s in ref.iterations[1:])      # light rows exist
        monkeypatch.setenv("SPKM_EK_LIGHT", "1")
        engine.clear_engine_cache()
        for graphs in (False, True, True):
            r = m.run(data, k, "simp_elkan", m.SeedConfig(seed=3), max_iter=30, use_graphs=graphs)
            assert np.array_equal(r.assignments, ref.assignments)
            assert r.objective == ref.objective
            assert [key(s) for s in r.iterations] == [key(s) for s in ref.iterations]
    engine.clear_engine_cache()


@pytest.mark.parametrize("k", [257, 511, 513, 1023, 1024])
def test_elkan_heavy_and_light_rows_at_boundary_k(k):
    """Boundary k of the k > 256 paths (16- and 32-column lanes, u rows whose last float4 is partial, ku padding):
    the Elkan family with heavy rows, light-row lists and the all-heavy switch equals the GPU Lloyd fit bit for bit,
    and its bounds pass the device auditor."""
    from paper_2107_04074_b200 import engine, synth, validation
    m = spk()
    data = synth.config_dataset("C3", n_override=6_000)
    engine.clear_engine_cache()
    lloyd = m.run(data, k, "standard", m.SeedConfig(seed=5), max_iter=12)
    for variant in ("simp_elkan", "elkan"):
        r = m.run(data, k, variant, m.SeedConfig(seed=5), max_iter=12)
        assert np.array_equal(r.assignments, lloyd.assignments), variant
        assert r.objective == lloyd.objective
        assert [s.reassignments for s in r.iterations] == [s.reassignments for s in lloyd.iterations]
        assert any(s.survivors2 > 0 for s in r.iterations[1:])
    rep = validation.audit_bounds(data, "simp_elkan", k, seed=5, max_iter=8)
    assert rep.passed, rep
    engine.clear_engine_cache()

