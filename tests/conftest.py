"""Shared test setup: the `gpu` marker, golden fixtures and the CPU oracle (the checker)."""

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = Path(__file__).resolve().parent / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def golden_names():
    return sorted(p.stem[3:] for p in GOLDEN.glob("ds_*.npz"))


def load_golden(name):
    return np.load(GOLDEN / f"ds_{name}.npz")


def golden_runs(z):
    """[(key, variant, k, seed, update, max_iter)] stored in a ds_*.npz."""
    out = []
    for key in z["runs"]:
        v, k, seed, upd, mi = str(key).rsplit("_", 4)
        out.append((str(key), v, int(k), int(seed), upd, int(mi)))
    return out


def golden_dataset(z):
    from paper_2107_04074_b200.sparse import Dataset
    return Dataset(z["indptr"], z["indices"], z["data"], int(z["dim"]))


@pytest.fixture(scope="session")
def oracle_mod():
    from oracle import oracle as O
    O.lib()
    return O


def seeding_golden():
    """tests/golden/seeding.npz (reference init_kmpp / init_afkmc2 picks)."""
    return np.load(GOLDEN / "seeding.npz")


def seeding_cases(z):
    """[(key, method, corpus, k, alpha, chain_length, seed)]."""
    out = []
    for key in z.files:
        p = key.split("__")
        if p[0] == "kmpp":
            out.append((key, "kmpp", p[1], int(p[2]), float(p[3]), 0, int(p[4])))
        elif p[0] == "afk":
            out.append((key, "afkmc2", p[1], int(p[2]), float(p[3]), int(p[4]), int(p[5])))
    return out


def seeding_corpus(z, name):
    """(indptr, indices, data, dim) of a seeding golden corpus."""
    if f"corpus__{name}__indptr" in z.files:
        return (z[f"corpus__{name}__indptr"], z[f"corpus__{name}__indices"], z[f"corpus__{name}__data"],
                int(z[f"corpus__{name}__dim"]))
    g = load_golden(name)
    return g["indptr"], g["indices"], g["data"], int(g["dim"])
