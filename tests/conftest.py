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
