#!/usr/bin/env python3
"""Generate the golden vectors that pin the oracle (run in the build container).

Runs the REFERENCE package itself (/root/reference/pkg/src/spkmeans; read
only, imported in place with a writable NUMBA_CACHE_DIR) and stores its
outputs as small .npz fixtures next to this script:

  rng.npz        splitmix64 streams + sample_without_replacement draws
                 (reference rng.py:31-73; KAT of tests/test_rng.py:8-18)
  geometry.npz   cos_lower/upper_bound, hamerly_upper_update, half_angle_cc
                 on random and edge inputs (reference geometry.py:20-68)
  ds_<name>.npz  a corpus as the reference normalised it (Dataset.from_rows)
                 plus engine.run results for several (variant, k, seed)
                 (reference engine.py:201-346): assignments, per-iteration
                 sim_count / cc_sim_count / reassignments / objective,
                 convergence, seed rows; and audit_bounds reports for the
                 pitfall corpus (validation.py:83-99).

/root/reference does not exist on the GPU box; only these fixtures travel.
Usage:  python tests/golden/make_golden.py
"""

import os
import sys
from pathlib import Path

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
REF = Path("/root/reference/pkg/src")
HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(REF))
sys.path.insert(1, str(ROOT))

import numpy as np  # noqa: E402

from spkmeans import corpus_io, datagen, engine, geometry, validation  # noqa: E402
from spkmeans.rng import PortableRng  # noqa: E402
from spkmeans.seeding import SeedConfig  # noqa: E402
from spkmeans.sparse import Dataset, SparseVector  # noqa: E402

FIX = Path("/root/reference/pkg/tests/fixtures")


def rng_golden():
    out = {}
    for seed in (0, 1, 42, 1234567, (1 << 64) - 1):
        r = PortableRng(seed)
        out[f"stream_{seed}"] = np.array([r.next_uint64() for _ in range(32)], dtype=np.uint64)
    for (n, k, seed) in [(100, 5, 1), (10, 7, 2), (2000, 20, 1), (5, 5, 0), (20000, 100, 2),
                         (50, 5, 1), (500, 7, 11), (7, 3, 9)]:
        out[f"swr_{n}_{k}_{seed}"] = np.array(PortableRng(seed).sample_without_replacement(n, k), np.int64)
    np.savez_compressed(HERE / "rng.npz", **out)


def geometry_golden():
    g = np.random.default_rng(7)
    a = g.uniform(-1, 1, 4000)
    b = g.uniform(-1, 1, 4000)
    edge = np.array([-1.0, -0.5, 0.0, 0.5, 1.0, 1 - 1e-12, -1 + 1e-12, 1.5, -1.5])
    ea, eb = np.meshgrid(edge, edge)
    a = np.concatenate([a, ea.ravel()])
    b = np.concatenate([b, eb.ravel()])
    np.savez_compressed(
        HERE / "geometry.npz", a=a, b=b,
        lower=geometry.cos_lower_bound(a, b), upper=geometry.cos_upper_bound(a, b),
        hamerly=geometry.hamerly_upper_update(a, b), half_angle=geometry.half_angle_cc(a),
        clamp=geometry.clamp_cos(a))


def save_dataset(name, data: Dataset, runs, audits=None):
    m = data.matrix
    out = {"indptr": m.indptr.astype(np.int64), "indices": m.indices.astype(np.int32),
           "data": m.data.astype(np.float64), "dim": np.int64(data.dim)}
    keys = []
    for (variant, k, seed, upd, max_iter) in runs:
        r = engine.run(data, k, variant, SeedConfig(seed=seed), max_iter=max_iter, hamerly_update=upd)
        key = f"{variant}_{k}_{seed}_{upd}_{max_iter}"
        keys.append(key)
        out[key + "__assignments"] = r.assignments.astype(np.int64)
        out[key + "__sim_count"] = np.array([s.sim_count for s in r.iterations], np.int64)
        out[key + "__cc_sim_count"] = np.array([s.cc_sim_count for s in r.iterations], np.int64)
        out[key + "__reassignments"] = np.array([s.reassignments for s in r.iterations], np.int64)
        out[key + "__objective"] = np.array([s.objective for s in r.iterations])
        out[key + "__converged"] = np.bool_(r.converged)
        out[key + "__seed_indices"] = np.asarray(r.centers.seed_indices, np.int64)
        out[key + "__counts"] = r.centers.counts.astype(np.int64)
        # final-center margins: best - second (fp64) for the 1e-5 rule
        _, best, second = engine.assign_full(data, r.centers)
        out[key + "__margin"] = best - second
    for (variant, k, seed, upd) in (audits or []):
        rep = validation.audit_bounds(data, variant, k, seed=seed, hamerly_update=upd)
        key = f"audit_{variant}_{k}_{seed}_{upd}"
        out[key] = np.array([rep.max_lower_violation, rep.max_upper_violation,
                             rep.decisions_audited, float(rep.passed)])
    out["runs"] = np.array(keys)
    np.savez_compressed(HERE / f"ds_{name}.npz", **out)
    print(f"ds_{name}: n={data.n} d={data.dim} runs={len(keys)}")


ALL5 = engine.VARIANTS


def main():
    rng_golden()
    geometry_golden()

    pit = corpus_io.load_dataset(FIX / "pitfall.svml")
    save_dataset("pitfall", pit,
                 [(v, 5, 1, "safe", 100) for v in ALL5] + [("hamerly", 5, 1, "naive", 100)],
                 audits=[("hamerly", 5, 1, "naive"), ("hamerly", 5, 1, "safe")])

    five = corpus_io.load_dataset(FIX / "five_points.svml")
    save_dataset("five_points", five, [(v, 5, 0, "safe", 100) for v in ALL5]
                 + [("standard", 2, 4, "safe", 100)])

    small = datagen.random_dataset(500, 64, 5, seed=7)
    save_dataset("small", small,
                 [(v, 7, 11, "safe", 100) for v in ALL5] + [(v, 1, 3, "safe", 100) for v in ALL5]
                 + [(v, 8, 13, "safe", 100) for v in ALL5] + [("standard", 10, 1, "safe", 2)])

    signed = datagen.random_dataset(300, 40, 6, seed=5, signed=True)
    save_dataset("signed", signed, [(v, 6, 2, "safe", 100) for v in ALL5],
                 audits=[(v, 6, 2, "safe") for v in ALL5[1:]])

    for (n, d, k, seed) in [(200, 256, 10, 3000), (2000, 5000, 20, 2000), (200, 5000, 50, 1007)]:
        nnz = max(2, round(0.01 * d))
        ds = datagen.random_dataset(n, d, nnz, seed=seed)
        save_dataset(f"grid_{n}_{d}_{k}_{seed}", ds, [(v, k, seed + 7, "safe", 100) for v in ALL5])

    clustered = Dataset.from_rows(
        datagen.clustered_sparse_rows(2000, 5000, 20, 50, seed=99, group_dims=150, noise_frac=0.5),
        dim=5000)
    save_dataset("clustered", clustered, [(v, 20, 3, "safe", 100) for v in ALL5])

    # BASELINE config 1 (C1) from this repo's generator, normalised by the reference
    from paper_2107_04074_b200 import synth
    indptr, idx, w = synth.sparse_corpus(synth.CONFIGS["C1"], synth.DATA_SEED_BASE + 1, return_raw=True)
    rows = [SparseVector(idx[indptr[i]:indptr[i + 1]].astype(np.int64), w[indptr[i]:indptr[i + 1]])
            for i in range(indptr.size - 1)]
    c1 = Dataset.from_rows(rows, dim=synth.CONFIGS["C1"].d)
    save_dataset("C1", c1, [(v, 20, 1, "safe", 50) for v in ALL5])


if __name__ == "__main__":
    main()
