"""Independent checks on the device: brute-force assignment, bound audits, triangle fuzz.

Mirror of /root/reference/pkg/src/spkmeans/validation.py:1-116 (same names,
arguments, AuditReport fields and BOUND_TOL).  The reference materialises the
exact n x k similarity matrix on the host for every audited iteration, which
is infeasible at the C3/C4 sizes; here the exact
float64 similarities are recomputed on the GPU (``spkm_audit``: float64 rows,
term-major float64 centers, FMA chains; error ~1e-16 << BOUND_TOL) and folded
into the worst violations on the device, so nothing of size n x k leaves HBM.
The audit shares no pruning code with the engine.
"""

from __future__ import annotations

import ctypes
import struct
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .sparse import Dataset

BOUND_TOL = 1e-9


def _key_to_double(key: int) -> float:
    b = key & ((1 << 63) - 1) if key >> 63 else (~key) & ((1 << 64) - 1)
    return struct.unpack("<d", struct.pack("<Q", b))[0]


def _double_key(v: float) -> int:
    b = struct.unpack("<Q", struct.pack("<d", v))[0]
    return (~b) & ((1 << 64) - 1) if b >> 63 else b | (1 << 63)


def _ptr(t):
    return None if t is None else t.data_ptr()


def _stream(dev):
    return ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def brute_force_assign(data: Dataset, centroids, device=None) -> np.ndarray:
    """Argmax assignment from exact float64 similarities; ties to the lowest
    index (validation.py:18-29)."""
    from .engine import _require_cuda, device_corpus
    dev = _require_cuda(device)
    C = np.asarray(centroids.centers if hasattr(centroids, "centers") else centroids, dtype=np.float64)
    k = C.shape[0]
    dc = device_corpus(data, dev)
    st = dc.seed_struct(data)
    kp = (k + 31) // 32 * 32
    h = np.zeros((data.dim, kp))
    h[:, :k] = C[:, dc.order].T                      # device term order, term-major
    ct64 = torch.from_numpy(h).to(dev)
    a = torch.empty(max(data.n, 1), dtype=torch.int32, device=dev)
    _lib.call("spkm_audit", st, k, kp, _ptr(ct64), None, None, None, 1, 3, None, _ptr(a), _stream(dev))
    return dc.to_host_rows(a[:data.n].cpu().numpy().astype(np.int64))


@dataclass
class AuditReport:
    max_lower_violation: float
    max_upper_violation: float
    decisions_audited: int
    passed: bool

    @classmethod
    def from_violations(cls, lower, upper, count):
        return cls(max_lower_violation=lower, max_upper_violation=upper, decisions_audited=count,
                   passed=lower <= BOUND_TOL and upper <= BOUND_TOL)


class DeviceBoundAuditor:
    """Debug hook checking every maintained bound against exact similarities
    (validation.py:49-80), called by the engine pre-scan each iteration with
    the device state itself (no host copies of bounds or centers)."""

    def __init__(self, data: Dataset):
        self.data = data
        self.count = 0
        self.keys = None
        self.ct64 = None

    def device_audit(self, iteration, eng):
        C, P = eng.C, eng.P
        dev = C.cent64.device
        st = eng.corpus.seed_struct(self.data)
        k, d = C.k, C.d
        kp = (k + 31) // 32 * 32
        if self.keys is None:
            zero = _double_key(0.0)
            self.keys = torch.tensor([zero - (1 << 64) if zero >= 1 << 63 else zero] * 2, dtype=torch.int64,
                                     device=dev)
        if self.ct64 is None or self.ct64.numel() != d * kp:
            self.ct64 = torch.empty(d * kp, dtype=torch.float64, device=dev)
        sp = eng.sp
        with torch.cuda.stream(eng.stream):
            _lib.call("spkm_audit_transpose", k, d, kp, _ptr(C.cent64), _ptr(self.ct64), sp)
            mode = 0 if eng.elkan else 2 if eng.yy else 1
            _lib.call("spkm_audit", st, k, kp, _ptr(self.ct64), _ptr(P.a), _ptr(P.l), _ptr(P.u), P.ku, mode,
                      _ptr(self.keys), None, sp)
        n = eng.corpus.n
        self.count += n
        if eng.elkan:
            self.count += n * k
        elif eng.yy:
            self.count += n * ((k + 3) // 4)
        elif k > 1:
            self.count += n

    def violations(self):
        ks = self.keys.cpu().numpy().astype(np.uint64) if self.keys is not None else None
        if ks is None:
            return 0.0, 0.0
        return _key_to_double(int(ks[0])), _key_to_double(int(ks[1]))


def audit_bounds(data: Dataset, variant: str, k: int, seed: int, init: str = "uniform", alpha: float = 1.0,
                 max_iter: int = 100, hamerly_update: str = "safe", device=None) -> AuditReport:
    """Run a variant to convergence with exact recomputation at every pruning
    decision point; report the worst bound violations (validation.py:83-99)."""
    from .engine import run
    from .seeding import SeedConfig
    auditor = DeviceBoundAuditor(data)
    run(data, k, variant, SeedConfig(method=init, alpha=alpha, seed=seed), max_iter=max_iter,
        debug_hook=auditor, hamerly_update=hamerly_update, device=device)
    lo, up = auditor.violations()
    return AuditReport.from_violations(lo, up, auditor.count)


def fuzz_triangle(n_triples: int, dims: int, seed: int, device=None) -> bool:
    """Random unit triples: lower bound <= exact <= upper bound with BOUND_TOL
    slack (validation.py:100-116); the bounds are evaluated by the device
    geometry (the kernels' own cos_lower / cos_upper)."""
    from .engine import _require_cuda
    dev = _require_cuda(device)
    gen = np.random.default_rng(seed)
    X = gen.normal(size=(n_triples, dims))
    Z = gen.normal(size=(n_triples, dims))
    Y = gen.normal(size=(n_triples, dims))
    for M in (X, Z, Y):
        M /= np.linalg.norm(M, axis=1, keepdims=True)
    a = np.einsum("ij,ij->i", X, Z)
    b = np.einsum("ij,ij->i", Z, Y)
    exact = np.einsum("ij,ij->i", X, Y)
    ta, tb = torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev)
    lo, up = torch.empty_like(ta), torch.empty_like(ta)
    sp = _stream(dev)
    _lib.call("spkm_geometry", 0, n_triples, _ptr(ta), _ptr(tb), _ptr(lo), sp)
    _lib.call("spkm_geometry", 1, n_triples, _ptr(ta), _ptr(tb), _ptr(up), sp)
    lower, upper = lo.cpu().numpy(), up.cpu().numpy()
    return bool(np.all(lower <= exact + BOUND_TOL) and np.all(upper >= exact - BOUND_TOL))


__all__ = ["BOUND_TOL", "AuditReport", "DeviceBoundAuditor", "audit_bounds", "brute_force_assign",
           "fuzz_triangle"]
