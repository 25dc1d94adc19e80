"""Seeded starts of the loop (reference seeding.py).

``SeedConfig``, ``init_uniform``, ``init_kmpp``, ``init_afkmc2`` and
``make_centroids`` mirror /root/reference/pkg/src/spkmeans/seeding.py:24-155
(names, arguments, errors, result type).  Uniform seeding is k splitmix64
draws on the host (no data involved); k-means++ and AFK-MC2 run on the GPU
(``spkm_seed_kmpp`` / ``spkm_seed_afkmc2``, csrc/seed.cuh): one float64
similarity pass over the corpus per pick, in the reference's np.dot order,
with the device running the same splitmix64 stream, so the picked rows equal
the reference's (tests/test_gpu_seeding.py against golden picks of the
reference).  Centers are the picked rows densified (CentroidSet.from_data_rows).
"""

import functools
from dataclasses import dataclass

import numpy as np

from .errors import ConfigError, InfeasibleError
from .rng import PortableRng

METHODS = ("uniform", "kmpp", "afkmc2")


@dataclass
class SeedConfig:
    method: str = "uniform"
    alpha: float = 1.0
    chain_length: int = 200
    seed: int = 0

    def validate(self):
        if self.method not in METHODS:
            raise ConfigError(f"unknown init method {self.method!r}")
        if not 1.0 <= self.alpha <= 2.0:
            raise ConfigError(f"alpha must be in [1, 2], got {self.alpha}")
        if self.chain_length < 1:
            raise ConfigError(f"chain_length must be >= 1, got {self.chain_length}")


def _check_k(data, k):
    if not 1 <= k <= data.n:
        raise InfeasibleError(f"k={k} infeasible for n={data.n}")


@functools.lru_cache(maxsize=64)
def _uniform_rows(n: int, k: int, seed: int) -> tuple:
    return tuple(PortableRng(seed).sample_without_replacement(n, k))


def uniform_rows(n: int, k: int, seed: int):
    """The k seed row ids of init_uniform (rng.py:54-73); a pure function of
    (n, k, seed), memoised so repeated fits skip the Python splitmix64 loop."""
    return list(_uniform_rows(int(n), int(k), int(seed)))


def init_uniform(data, k: int, seed: int):
    from .engine import CentroidSet
    _check_k(data, k)
    return CentroidSet.from_data_rows(data, uniform_rows(data.n, k, seed))


def _device_seed(data, k: int, method: str, alpha: float, chain_length: int, seed: int, trace=None,
                 device=None, corpus=None) -> np.ndarray:
    import torch

    from . import _lib
    from .engine import _ptr, _require_cuda, ctypes_void, device_corpus
    dev = _require_cuda(device)
    dc = corpus if corpus is not None and corpus.rows == (0, data.n) else device_corpus(data, dev)
    st = dc.seed_struct(data)
    picks = torch.empty(k, dtype=torch.int64, device=dev)
    tr = torch.empty(max(k - 1, 1) * data.n, dtype=torch.float64, device=dev) if trace is not None else None
    sp = ctypes_void(torch.cuda.current_stream(dev).cuda_stream)
    s64 = int(seed) & ((1 << 64) - 1)
    if method == "kmpp":
        _lib.call("spkm_seed_kmpp", st, k, float(alpha), s64, _ptr(picks), _ptr(tr), sp)
        _lib.note_launches(1 + 4 * (k - 1))
    else:
        _lib.call("spkm_seed_afkmc2", st, k, float(alpha), int(chain_length), s64, _ptr(picks), sp)
        _lib.note_launches(8 + 4 * (k - 1))
    out = picks.cpu().numpy().astype(np.int64)
    if trace is not None and k > 1:
        trace.extend(list(tr.view(k - 1, data.n).cpu().numpy()))
    return out


def init_kmpp(data, k: int, alpha: float, seed: int, trace: list | None = None, device=None):
    """Spherical k-means++ (seeding.py:64-89) on the GPU: each next center is
    drawn with probability proportional to alpha - (best similarity so far)."""
    from .engine import CentroidSet
    _check_k(data, k)
    return CentroidSet.from_data_rows(data, _device_seed(data, k, "kmpp", alpha, 0, seed, trace, device))


def init_afkmc2(data, k: int, alpha: float, chain_length: int, seed: int, device=None):
    """AFK-MC2 (seeding.py:92-146) on the GPU: Metropolis-Hastings chains
    over the proposal q built from the first center."""
    from .engine import CentroidSet
    _check_k(data, k)
    return CentroidSet.from_data_rows(data, _device_seed(data, k, "afkmc2", alpha, chain_length, seed,
                                                         None, device))


def seed_rows_for(data, k: int, cfg: SeedConfig, device=None, corpus=None) -> np.ndarray:
    """The seed row ids of ``cfg`` (what make_centroids densifies)."""
    cfg.validate()
    _check_k(data, k)
    if cfg.method == "uniform":
        return np.asarray(uniform_rows(data.n, k, cfg.seed), dtype=np.int64)
    return _device_seed(data, k, cfg.method, cfg.alpha, cfg.chain_length, cfg.seed, None, device, corpus)


def make_centroids(data, k: int, cfg: SeedConfig):
    from .engine import CentroidSet
    return CentroidSet.from_data_rows(data, seed_rows_for(data, k, cfg))
