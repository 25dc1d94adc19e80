"""Seeded starts (host-side input of the loop).

``SeedConfig`` and ``init_uniform`` mirror the reference
(/root/reference/pkg/src/spkmeans/seeding.py:24-61, 149-155): k distinct
rows drawn with the splitmix64 stream, densified as float64 centers, so the
GPU loop and the reference start from bit-identical centers.  The
k-means++ / AFK-MC2 seedings (seeding.py:64-146) are the next widening of
this build and are not implemented yet.
"""

from dataclasses import dataclass

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


def uniform_rows(n: int, k: int, seed: int):
    """The k seed row ids of init_uniform (rng.py:54-73)."""
    return PortableRng(seed).sample_without_replacement(n, k)


def init_uniform(data, k: int, seed: int):
    from .engine import CentroidSet
    _check_k(data, k)
    return CentroidSet.from_data_rows(data, uniform_rows(data.n, k, seed))


def make_centroids(data, k: int, cfg: SeedConfig):
    cfg.validate()
    if cfg.method == "uniform":
        return init_uniform(data, k, cfg.seed)
    raise NotImplementedError(f"seeding {cfg.method!r} is not part of this build yet (uniform only)")
