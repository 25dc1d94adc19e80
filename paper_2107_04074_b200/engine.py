"""The accelerated spherical k-means loop on B200 (fit = ``run``, predict = ``assign_full``).

Host mirror of the reference's engine (/root/reference/pkg/src/spkmeans/
engine.py:1-346): same names, arguments, variants, dataclasses, errors and
phase order, but every numeric phase is a CUDA kernel of libspkm.so called
through the C ABI (include/spkm.h).  PyTorch only allocates device buffers
and provides the stream.  There is no CPU fallback.

Phase order per iteration (engine.py:239-337):
  it == 1   full pass + top-2 (bounds init)  -> scratch sums -> move all
  it >= 2   [cc/s]  -> bound drift update + prune test + compaction
            -> debug_hook -> scan survivors -> incremental sums (moves)
            -> renormalise touched -> objective / drift / convergence stats
One 64-byte stats read (D2H) per iteration drives IterationStats and the
convergence test, exactly like the reference's per-iteration bookkeeping.

Documented deviations: similarities are float32 in
a fixed FMA order; bounds carry a per-row error margin so pruned variants
are exactly equal to this module's Lloyd; exact ties keep the incumbent
from iteration 2 on; center sums are exact int64 fixed point (so the
reference's 50-iteration scratch rebuild is a no-op, kept for its schedule).
"""

from __future__ import annotations

import ctypes
import math
import os
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._lib import Bounds, Centers, CSR, Work
from .errors import ConfigError, DeviceError, InfeasibleError
from .sparse import Dataset

VARIANTS = ("standard", "elkan", "simp_elkan", "hamerly", "simp_hamerly")
# beyond the reference's five: Yin-Yang group bounds (SURVEY.md 8(f) rank 4,
# PAPER.md:409-414; the reference does not implement it)
EXTRA_VARIANTS = ("yinyang",)
_ELKAN_FAMILY = frozenset({"elkan", "simp_elkan"})
_HAMERLY_FAMILY = frozenset({"hamerly", "simp_hamerly"})
_CC_VARIANTS = frozenset({"elkan", "hamerly"})
_SCRATCH_INTERVAL = 50
EPS_UNIT = 6.1e-8


# --------------------------------------------------------------- dataclasses
@dataclass
class CentroidSet:
    """Unit centers plus the state needed to move them (engine.py:31-58)."""

    centers: np.ndarray
    sums: np.ndarray
    counts: np.ndarray
    prev_centers: np.ndarray | None
    drift: np.ndarray
    seed_indices: np.ndarray | None = None

    @property
    def k(self) -> int:
        return self.centers.shape[0]

    @classmethod
    def from_data_rows(cls, data: Dataset, row_indices) -> "CentroidSet":
        idx = np.asarray(row_indices, dtype=np.int64)
        centers = data.densify_rows(idx)
        k = centers.shape[0]
        return cls(centers=centers, sums=np.zeros_like(centers), counts=np.zeros(k, np.int64),
                   prev_centers=centers.copy(), drift=np.ones(k), seed_indices=idx)


class DeviceCentroidSet:
    """Result centers that stay in HBM until read (same attributes as CentroidSet).

    ``centers``/``sums``/``counts``/``drift`` are copied to the host on first
    access; ``device_centers`` exposes the float64 device tensor directly.
    """

    def __init__(self, C: "CenterState", seed_indices=None):
        self._C = C
        self.seed_indices = seed_indices
        self.prev_centers = None
        self._cache = {}

    @property
    def k(self) -> int:
        return self._C.k

    @property
    def device_centers(self):
        return self._C.cent64.view(self._C.k, self._C.d)

    def _get(self, name, fn):
        if name not in self._cache:
            self._cache[name] = fn()
        return self._cache[name]

    @property
    def centers(self) -> np.ndarray:
        return self._get("centers", self._C.host_centers)

    @property
    def sums(self) -> np.ndarray:
        return self._get("sums", self._C.host_sums)

    @property
    def counts(self) -> np.ndarray:
        return self._get("counts", lambda: self._C.counts.cpu().numpy())

    @property
    def drift(self) -> np.ndarray:
        return self._get("drift", lambda: self._C.drift.cpu().numpy())

    def to_host(self) -> CentroidSet:
        return CentroidSet(self.centers, self.sums, self.counts, None, self.drift, self.seed_indices)


@dataclass
class BoundsState:
    """Bounds handed to debug hooks (engine.py:61-69); host copies of device state."""

    variant: str
    a: np.ndarray
    l: np.ndarray
    u_matrix: np.ndarray | None = None
    u: np.ndarray | None = None


@dataclass
class IterationStats:
    iteration: int
    sim_count: int
    cc_sim_count: int
    reassignments: int
    objective: float
    elapsed_ns: int
    # instrumentation beyond the reference's fields (defaults keep its constructor)
    survivors: int = 0          # points failing the drift-updated bound test
    survivors2: int = 0         # Hamerly: points still failing after tightening
    nnz_tighten: int = 0        # CSR nnz re-read by the Hamerly tighten pass
    nnz_rescan: int = 0         # CSR nnz re-read by the Hamerly full-k rescan
    nnz_elkan: int = 0          # CSR nnz re-read by the Elkan survivor scan
    touched: int = 0            # clusters renormalised (moved in or out)
    nnz_moved: int = 0          # CSR nnz of the points that changed cluster


@dataclass
class ClusteringResult:
    assignments: np.ndarray
    centers: CentroidSet
    objective: float
    iterations: list = field(default_factory=list)
    converged: bool = False

    @property
    def total_sims(self) -> int:
        return sum(s.sim_count for s in self.iterations)

    @property
    def total_cc_sims(self) -> int:
        return sum(s.cc_sim_count for s in self.iterations)


# --------------------------------------------------------------- device state
def _stream_ptr(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes_void(s.cuda_stream)


def ctypes_void(v):
    import ctypes
    return ctypes.c_void_p(int(v))


def _ptr(t: torch.Tensor | None):
    return None if t is None else t.data_ptr()


def row_eps(lengths: np.ndarray) -> np.ndarray:
    """eps_i = (nnz_i + 6) * 6.1e-8, rounded up to float32 (spkm.cu header)."""
    e = (lengths.astype(np.float64) + 6.0) * EPS_UNIT
    f = e.astype(np.float32)
    low = f.astype(np.float64) < e
    f[low] = np.nextafter(f[low], np.float32(np.inf))
    return f


def row_eps_dense(D: int, n: int) -> np.ndarray:
    e = (3.0 * D / 8.0 + 8.0) * 2.0 ** -22 + 4e-6
    f = np.float32(e)
    if float(f) < e:
        f = np.nextafter(f, np.float32(np.inf))
    return np.full(n, f, dtype=np.float32)


def scale_bits_for(n_total: int) -> int:
    """Fixed-point scale with n * 2^S <= 2^62 (SURVEY.md §7 hard part 1d)."""
    return int(62 - math.ceil(math.log2(n_total + 1)))


def term_order(data: Dataset):
    """Vocabulary renumbering by descending document frequency (stable).

    Returns (order, new_id): order[new] = old term id, new_id[old] = new id.
    The device keeps term ids in this numbering so the Zipf head is the
    contiguous block of term rows [0, hot) that the row-pass kernels stage in
    shared memory.  The CSR positions are untouched, so every similarity keeps
    the canonical order (CSR order) and is bit-identical to the unrenumbered
    computation.  Computed once per Dataset over ALL rows, so every shard of a
    multi-GPU run uses the same numbering.
    """
    cached = getattr(data, "_term_order", None)
    if cached is not None:
        return cached
    df = np.bincount(data.indices, minlength=data.dim)
    order = np.argsort(-df, kind="stable").astype(np.int64)
    new_id = np.empty(data.dim, np.int64)
    new_id[order] = np.arange(data.dim, dtype=np.int64)
    data._term_order = (order, new_id)
    return data._term_order


def _host_registered(arr: np.ndarray) -> np.ndarray:
    """Page-lock a host array in place (cudaHostRegister) so H2D copies from it
    are DMA transfers; unregistered when the array is garbage collected."""
    import weakref
    if not arr.flags.c_contiguous or arr.nbytes == 0:
        return arr
    key = arr.ctypes.data
    if key in _REGISTERED:
        return arr
    cudart = torch.cuda.cudart()
    if int(cudart.cudaHostRegister(key, arr.nbytes, 0)) != 0:
        return arr                     # not registrable: the caller stages it
    _REGISTERED.add(key)

    def _release(ptr=key):
        try:
            torch.cuda.cudart().cudaHostUnregister(ptr)
        except Exception:
            pass
        _REGISTERED.discard(ptr)
    weakref.finalize(arr, _release)
    return arr


_REGISTERED: set = set()


class DeviceCorpus:
    """A CSR (or row range of one) resident in HBM: int64 indptr, int32 indices, fp32 values.

    Term ids are stored renumbered by document frequency (see term_order) and
    rows longest-first; both permutations are invisible to callers (every
    per-row result is independent of them, and host-facing arrays are mapped
    back with to_host_rows / to_device_rows).
    """

    @property
    def row_perm(self) -> np.ndarray:
        """device row r holds host row row_perm[r]."""
        if self._row_perm is None:
            self._row_perm = self.perm_dev.cpu().numpy()
        return self._row_perm

    @property
    def row_pos(self) -> np.ndarray:
        """host row i sits at device row row_pos[i]."""
        if self._row_pos is None:
            rp = self.row_perm
            self._row_pos = np.empty_like(rp)
            self._row_pos[rp] = np.arange(rp.size, dtype=np.int64)
        return self._row_pos

    def to_host_rows(self, x: np.ndarray) -> np.ndarray:
        out = np.empty_like(x)
        out[self.row_perm] = x
        return out

    def to_device_rows(self, x: np.ndarray) -> np.ndarray:
        return np.asarray(x)[self.row_perm]

    def __init__(self, data: Dataset, device: torch.device, rows: tuple | None = None,
                 pinned_host: bool = False):
        r0, r1 = rows if rows is not None else (0, data.n)
        s, e = int(data.indptr[r0]), int(data.indptr[r1])
        self.n, self.d, self.nnz = r1 - r0, data.dim, e - s
        self.rows = (r0, r1)
        self.device = torch.device(device)
        self.pinned_host = pinned_host
        self._stage = None
        self._seed = None
        self._upload = None
        self._prep = None                # spkm_prepare_rows scratch
        self._row_perm = self._row_pos = None
        self.dense_dim = getattr(data, "dense_dim", None) if self.device.type == "cuda" else None
        if self.dense_dim is not None and self.dense_dim % 32 != 0:
            self.dense_dim = None
        if self.device.type != "cuda":
            self._host_prepare(data)
        else:
            i32, f32 = dict(dtype=torch.int32, device=self.device), dict(dtype=torch.float32, device=self.device)
            self.indptr = torch.empty(self.n + 1, dtype=torch.int64, device=self.device)
            self.indices = torch.empty(max(self.nnz, 1), **i32)
            self.values = torch.empty(max(self.nnz, 1), **f32)
            self.reps = torch.empty(max(self.n, 1), **f32)
            # float64 rows in device order (seeding); dense corpora skip it
            self.values64 = (torch.empty(max(self.nnz, 1), dtype=torch.float64, device=self.device)
                             if self.dense_dim is None else None)
            self._device_prepare(data)
        self.struct = CSR(self.n, self.d, self.nnz, _ptr(self.indptr), _ptr(self.indices), _ptr(self.values),
                          _ptr(self.reps))

    def _host_prepare(self, data: Dataset):
        """numpy path (CPU devices: host-logic tests)."""
        r0, r1 = self.rows
        self.order, self.new_id = term_order(data)
        lens = np.diff(data.indptr[r0:r1 + 1])
        self._row_perm = np.argsort(-lens, kind="stable").astype(np.int64)
        self._row_pos = None
        plen = lens[self.row_perm]
        ip = np.zeros(self.n + 1, np.int64)
        np.cumsum(plen, out=ip[1:])
        sel = self._device_order(data, ip, plen)
        host = [torch.from_numpy(ip),
                torch.from_numpy(self.new_id[data.indices[sel]].astype(np.int32)),
                torch.from_numpy(np.ascontiguousarray(data.data[sel], np.float32)),
                torch.from_numpy(row_eps(plen))]
        self.indptr, self.indices, self.values, self.reps = [h.to(self.device) for h in host]
        self.h2d_bytes = sum(h.numel() * h.element_size() for h in host)

    def _device_prepare(self, data: Dataset):
        """Upload the raw CSR rows once and build the device layout on the GPU:
        rows longest first (stable), term ids renumbered by document frequency
        (stable), float32 values, row_eps (spkm_permute_rows)."""
        r0, r1 = self.rows
        s, e = int(data.indptr[r0]), int(data.indptr[r1])
        dev = self.device
        stream = torch.cuda.current_stream(dev)
        sp = ctypes_void(stream.cuda_stream)
        # a dense corpus (Dataset.from_dense) has the term ids 0..D-1 in every
        # row: they are generated on the device instead of uploaded
        dense_ids = self.dense_dim is not None and getattr(data, "dense_dim", None) == self.dense_dim
        if dense_ids and getattr(data, "_values32", None) is not None:
            return self._device_prepare_dense(data, data._values32, sp)
        if self.pinned_host and (r0, r1) == (0, data.n):
            # the whole corpus: page-lock the Dataset's own arrays once and copy
            # straight from them (no staging copy on the host)
            ip_h, val_h = (torch.from_numpy(_host_registered(a)) for a in (data.indptr, data.data))
            idx_h = None if dense_ids else torch.from_numpy(_host_registered(data.indices))
        else:
            ip_h = torch.from_numpy(np.asarray(data.indptr[r0:r1 + 1], dtype=np.int64) - s)
            idx_h = None if dense_ids else torch.from_numpy(np.ascontiguousarray(data.indices[s:e], dtype=np.int32))
            val_h = torch.from_numpy(np.ascontiguousarray(data.data[s:e], dtype=np.float64))
        if self.pinned_host:
            # anything not page-locked in place goes through persistent pinned staging
            hs = [ip_h, idx_h, val_h]
            if self._stage is None:
                self._stage = [None, None, None]
            for q, t in enumerate(hs):
                if t is not None and not t.is_pinned():
                    if self._stage[q] is None or self._stage[q].shape != t.shape:
                        self._stage[q] = torch.empty(t.shape, dtype=t.dtype).pin_memory()
                    self._stage[q].copy_(t)
                    hs[q] = self._stage[q]
            ip_h, idx_h, val_h = hs
        # the row offsets first; the term ids and values stream in on a side
        # stream while the row order is sorted out on this one
        ip_raw = ip_h.to(dev, non_blocking=True)
        if self._upload is None:
            self._upload = torch.cuda.Stream(device=dev)
        up = self._upload
        up.wait_stream(stream)
        with torch.cuda.stream(up):
            if idx_h is None:
                idx_raw = torch.empty((r1 - r0) * self.dense_dim, dtype=torch.int32, device=dev)
                _lib.call("spkm_dense_ids", r1 - r0, self.dense_dim, _ptr(idx_raw), None, None,
                          ctypes_void(up.cuda_stream))
            else:
                idx_raw = idx_h.to(dev, non_blocking=True)
            val_raw = val_h.to(dev, non_blocking=True)
        self.h2d_bytes = sum(t.numel() * t.element_size() for t in (ip_h, idx_h, val_h) if t is not None)
        # device layout by spkm_prepare_rows (csrc/prepare.cuh): rows longest
        # first (stable radix sort) and their offsets, then -- once per
        # Dataset -- the term order by document frequency
        nb = int(_lib.lib().spkm_prepare_scratch_bytes(self.n, self.d))
        if nb < 0:
            raise ConfigError("corpus too large for one device (n and d must be < 2^31)")
        if self._prep is None or self._prep.numel() < nb:
            self._prep = torch.empty(max(nb, 1), dtype=torch.uint8, device=dev)
        perm = torch.empty(max(self.n, 1), dtype=torch.int64, device=dev)
        key = getattr(data, "_row_key", None)
        pos = self._seed[3] if self._seed is not None else None    # refresh: the seeding maps follow
        if key is None:
            _lib.call("spkm_prepare_rows", self.n, self.d, 0, _ptr(ip_raw), None, _ptr(perm),
                      None if pos is None else _ptr(pos), _ptr(self.indptr), None, None, _ptr(self._prep), nb, sp)
        else:   # locality experiments (tools/c4_locality.py): rows grouped by key, longest first within a group
            kk = np.asarray(key, np.int64)[r0:r1]
            lens = np.diff(data.indptr[r0:r1 + 1])
            ph = np.lexsort((-lens, kk)).astype(np.int64)
            perm.copy_(torch.from_numpy(ph))
            ip = np.zeros(self.n + 1, np.int64)
            np.cumsum(lens[ph], out=ip[1:])
            self.indptr.copy_(torch.from_numpy(ip))
            if pos is not None:
                inv = np.empty_like(ph)
                inv[ph] = np.arange(ph.size)
                pos.copy_(torch.from_numpy(inv))
        stream.wait_stream(up)
        idx_raw.record_stream(stream)
        val_raw.record_stream(stream)
        cached = getattr(data, "_term_order", None)
        if cached is None and self.rows == (0, data.n):
            order_d = torch.empty(max(self.d, 1), dtype=torch.int64, device=dev)
            new_id_d = torch.empty_like(order_d)
            _lib.call("spkm_prepare_rows", self.n, self.d, self.nnz, None, _ptr(idx_raw), None, None, None,
                      _ptr(order_d), _ptr(new_id_d), _ptr(self._prep), nb, sp)
            order_h, new_id_h = order_d[:self.d].cpu().numpy(), new_id_d[:self.d].cpu().numpy()
            data._term_order = (order_h, new_id_h)
            self._new_id_dev, self._new_id_src = new_id_d, new_id_h
        else:
            order_h, new_id_h = term_order(data)
            if getattr(self, "_new_id_src", None) is not new_id_h:   # the device copy follows the host map
                self._new_id_dev = torch.from_numpy(new_id_h).to(dev)
                self._new_id_src = new_id_h
            new_id_d = self._new_id_dev
        self.order, self.new_id = order_h, new_id_h
        dense = self.dense_dim is not None
        _lib.call("spkm_permute_rows", self.n, _ptr(ip_raw), _ptr(idx_raw), _ptr(val_raw), _ptr(perm),
                  _ptr(self.indptr), _ptr(new_id_d), _ptr(self.indices), _ptr(self.values), _ptr(self.values64),
                  None if dense else _ptr(self.reps), sp)
        if dense:
            # tensor-core path: every similarity is the 3xTF32 tcgen05 value
            # with error <= (3D/8 + 8) 2^-22 + 4e-6 (spkm.cu, dense rows)
            self.reps.fill_(float(row_eps_dense(self.dense_dim, 1)[0]))
        self.perm_dev = perm
        self._row_perm = self._row_pos = None   # host copies on first use (no sync here)
        if self._seed is not None:          # refresh: the seeding maps follow the new rows (pos written above)
            self._seed[2].copy_(perm)
        del ip_raw, idx_raw, val_raw        # stream-ordered frees (caching allocator)

    def _device_prepare_dense(self, data: Dataset, v32: np.ndarray, sp):
        """Dense rows (Dataset.dense keeps a float32 copy of its normalised
        rows): every row holds the D terms in order, so the stable length
        order and the document-frequency term order are the identity -- the
        float32 values go H2D straight into the device buffer (half the bytes
        of the float64 rows), term ids, offsets and row order are generated
        (spkm_dense_ids); nothing is permuted."""
        r0, r1 = self.rows
        D, dev, n = self.dense_dim, self.device, r1 - r0
        src = v32[r0 * D:r1 * D]
        h = torch.from_numpy(_host_registered(v32) if (r0, r1) == (0, data.n) else np.ascontiguousarray(src))
        if (r0, r1) == (0, data.n):
            h = h[r0 * D:r1 * D]
        if self.pinned_host and not h.is_pinned():
            if self._stage is None or self._stage[0] is None or self._stage[0].shape != h.shape:
                self._stage = [torch.empty(h.shape, dtype=h.dtype).pin_memory(), None, None]
            self._stage[0].copy_(h)
            h = self._stage[0]
        self.values[:n * D].copy_(h, non_blocking=True)
        perm = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
        _lib.call("spkm_dense_ids", n, D, _ptr(self.indices), _ptr(self.indptr), _ptr(perm), sp)
        self.reps.fill_(float(row_eps_dense(D, 1)[0]))
        ident = np.arange(self.d, dtype=np.int64)
        if getattr(data, "_term_order", None) is None and (r0, r1) == (0, data.n):
            data._term_order = (ident, ident.copy())
        self.order, self.new_id = term_order(data) if (r0, r1) != (0, data.n) else data._term_order
        self.h2d_bytes = int(src.nbytes)
        self.perm_dev = perm
        self._row_perm = self._row_pos = None
        if self._seed is not None:
            self._seed[2].copy_(perm)
            self._seed[3].copy_(perm)          # identity: position == row

    def refresh(self, data: Dataset):
        """Upload new rows of the same shape (n, nnz, d) into the same device
        buffers: every pointer an engine or a captured loop holds stays valid."""
        r0, r1 = self.rows
        if (r1 - r0, int(data.indptr[r1] - data.indptr[r0]), data.dim) != (self.n, self.nnz, self.d):
            raise ValueError("refresh needs a corpus of the same shape (n, nnz, d)")
        self._device_prepare(data)

    def _device_order(self, data: Dataset, ip=None, plen=None) -> np.ndarray:
        """nnz positions of the host CSR in device order (rows longest first)."""
        r0, r1 = self.rows
        if plen is None:
            plen = np.diff(data.indptr[r0:r1 + 1])[self.row_perm]
            ip = np.zeros(self.n + 1, np.int64)
            np.cumsum(plen, out=ip[1:])
        src = data.indptr[r0:r1][self.row_perm]
        return (np.repeat(src - ip[:-1], plen) + np.arange(int(ip[-1]), dtype=np.int64)) if self.n else \
            np.zeros(0, np.int64)

    def seed_struct(self, data: Dataset):
        """spkm_seed inputs (built once): float64 rows in device order, the row
        maps and the seeding scratch.  Needs the whole corpus (not a shard)."""
        if self.rows != (0, data.n):
            raise ConfigError("device seeding needs the whole corpus on one device")
        if self._seed is None:
            dev = self.indptr.device
            v64 = self.values64
            if v64 is None:     # dense corpora: float64 rows on demand
                v64 = torch.from_numpy(np.ascontiguousarray(data.data[self._device_order(data)])).to(dev)
            row_host = self.perm_dev.clone()
            row_dev = torch.from_numpy(self.row_pos).to(dev)
            scratch = torch.empty(int(_lib.lib().spkm_seed_scratch_doubles(self.n, self.d)), dtype=torch.float64,
                                  device=dev)
            st = _lib.Seed(self.n, self.d, _ptr(self.indptr), _ptr(self.indices), _ptr(v64), _ptr(row_host),
                           _ptr(row_dev), _ptr(scratch))
            self._seed = (st, v64, row_host, row_dev, scratch)
        return self._seed[0]


def device_corpus(data: Dataset, device=None, cache: bool = True) -> DeviceCorpus:
    device = torch.device(device or "cuda")
    key = str(device)
    if cache and key in data._device_cache:
        return data._device_cache[key]
    dc = DeviceCorpus(data, device)
    if cache:
        data._device_cache[key] = dc
    return dc


class CenterState:
    """Replicated center buffers (spkm_centers)."""

    def __init__(self, k: int, d: int, n_total: int, device, with_cc: bool, order=None):
        L = _lib.lib()
        self.k, self.d = k, d
        self.order = order                      # device column c holds host term order[c]
        self.kp = int(L.spkm_padded_k(k))
        self.nchunk = int(L.spkm_center_chunks(d))
        self.scale_bits = scale_bits_for(n_total)
        dev = device
        f64 = dict(dtype=torch.float64, device=dev)
        self.cent64 = torch.empty(k * d, **f64)
        # + 1024 floats: the row pass's last lanes read whole float4 groups past kp on the last term row
        self.ct32_buf = torch.zeros(d * self.kp + 1024, dtype=torch.float32, device=dev)
        self.ct32 = self.ct32_buf[:d * self.kp]
        # fp16 copy for the screening full pass: off unless SPKM_CT16=1 -- measured
        # slower at C4 and C3 (the gathers are not limited by their bytes;
        # profiles/r02_ab_notes.txt), kept tested as an option
        use16 = k > 128 and os.environ.get("SPKM_CT16") == "1"
        self.ct16_buf = torch.zeros(d * self.kp + 1024, dtype=torch.float16, device=dev) if use16 else None
        self.sums = torch.empty(k * d, dtype=torch.int64, device=dev)
        self.counts = torch.zeros(k, dtype=torch.int64, device=dev)
        self.drift = torch.ones(k, **f64)
        self.sinp = torch.zeros(k, **f64)
        self.tlist = torch.zeros(k, dtype=torch.int32, device=dev)
        self.tcount = torch.zeros(1, dtype=torch.int32, device=dev)
        self.ctl = torch.zeros(2, dtype=torch.int64, device=dev)
        self.touched = torch.zeros(k, dtype=torch.int32, device=dev)
        self.objc = torch.zeros(k, **f64)
        self.part = torch.empty(int(L.spkm_center_scratch_doubles(k, d)), **f64)
        self.norm = torch.empty(k, **f64)
        self.cc = torch.zeros(k * k if with_cc else 1, dtype=torch.float32, device=dev)
        self.s = torch.zeros(k if with_cc else 1, dtype=torch.float32, device=dev)
        self.hstat = torch.zeros(8, **f64)
        if with_cc:
            ntiles = int(L.spkm_gram_tiles(k, None))
            pairs = np.zeros(2 * ntiles, np.int32)
            L.spkm_gram_tiles(k, pairs.ctypes.data)
            self.tiles = torch.from_numpy(pairs).to(dev)
            self.gram = torch.empty(int(L.spkm_gram_scratch_doubles(k, d)), **f64)
        self.dense = None
        self.cindex = None
        self.struct = Centers(k, d, self.kp, self.scale_bits, 0, _ptr(self.cent64), _ptr(self.ct32),
                              _ptr(self.sums), _ptr(self.counts), _ptr(self.drift), _ptr(self.sinp),
                              _ptr(self.touched), _ptr(self.objc), _ptr(self.part), _ptr(self.norm), _ptr(self.cc),
                              _ptr(self.s), _ptr(self.hstat), _ptr(self.tlist), _ptr(self.tcount),
                              _ptr(self.ctl), _ptr(self.ct16_buf))
        self.cc_valid = False

    def load(self, centers, stream):
        """Seed centers (numpy, or a float64 torch tensor already on the device)."""
        if isinstance(centers, torch.Tensor) and centers.device == self.cent64.device:
            src = centers.reshape(self.k, self.d).to(torch.float64)
            if self.order is not None:
                src = src.index_select(1, torch.from_numpy(self.order).to(src.device))
            src = src.reshape(-1).contiguous()
        else:
            h = np.asarray(centers, np.float64).reshape(self.k, self.d)
            if self.order is not None:
                h = h[:, self.order]
            src = torch.from_numpy(np.ascontiguousarray(h).ravel()).to(self.cent64.device)
        if src.numel() != self.k * self.d:
            raise ValueError(f"centers must be {self.k} x {self.d}")
        _lib.call("spkm_load_centers", self.struct, _ptr(src), stream)
        return src  # keep alive until the stream passes

    def attach_cindex(self, capacity: int):
        """Sparse term-major index of the centers for the full pass (k > 256):
        pairs for term rows with at most kp/4 nonzero centers (spkm_cindex)."""
        L = _lib.lib()
        dev = self.cent64.device
        cap = max(int(min(capacity, self.k * self.d)), 1)
        nb = int(L.spkm_cindex_scratch_bytes(self.d))
        self._ci = (torch.empty(max(self.d, 1), dtype=torch.int64, device=dev),
                    torch.empty(2 * cap + 8, dtype=torch.int32, device=dev),   # + slack for 16-byte bulk prefetches
                    torch.empty(max(self.d, 1), dtype=torch.int64, device=dev),
                    torch.empty(max(nb, 1), dtype=torch.uint8, device=dev))
        # term rows with more nonzero centers than kp / SPKM_CI_DIV stay dense float4 rows (A/B: profiles/r02_ab_notes.txt)
        div = max(int(os.environ.get("SPKM_CI_DIV", "4")), 1)
        self.cindex = _lib.CIndex(_ptr(self._ci[0]), _ptr(self._ci[1]), _ptr(self._ci[2]), _ptr(self._ci[3]), nb, cap,
                                  self.kp // div, 0)
        self.struct.cindex = ctypes.addressof(self.cindex)

    def build_cindex(self, sp):
        if self.cindex is not None:
            _lib.call("spkm_cindex_build", self.struct, sp)

    def attach_dense(self, corpus: "DeviceCorpus", row0: int = 0, n_rows: int = 0, rescan: bool = False):
        """float32 center rows (padded to 256) for the dense tensor-core pass
        (rows from device row ``row0`` on: a multi-GPU shard), and the
        survivor scratch of the Hamerly rescan."""
        D = corpus.dense_dim
        kpad = (self.k + 255) // 256 * 256
        dev = self.cent64.device
        self.b32 = torch.zeros(kpad * D, dtype=torch.float32, device=dev)
        self.xs = torch.empty(max(n_rows, 1) * D, dtype=torch.float32, device=dev) if rescan else None
        self.dense = _lib.Dense(D, kpad, _ptr(corpus.values) + 4 * D * row0, _ptr(self.b32), _ptr(self.xs))

    def refresh_dense(self, stream):
        if self.dense is not None:
            _lib.call("spkm_dense_centers", self.struct, self.dense, stream)

    def snapshot(self, sums_from=None, stream=None, lazy_sums: bool = False) -> "CenterState":
        """A shallow CenterState whose result tensors are private copies (for ClusteringResult).

        ``sums_from=(data, assignments)`` (or ``lazy_sums`` with ``_sums_from``
        set later) skips the device copy of the k x d fixed-point sums: they
        are an exact integer function of the final assignments, rebuilt on
        the host only if the caller reads them.  With ``stream`` the copies
        are enqueued on it (allocated on the current stream, then marked as
        used by ``stream``)."""
        snap = object.__new__(CenterState)
        snap.k, snap.d, snap.kp, snap.scale_bits, snap.order = self.k, self.d, self.kp, self.scale_bits, self.order
        skip_sums = lazy_sums or sums_from is not None
        snap._sums_from = sums_from
        if stream is None:
            snap.cent64 = self.cent64.clone()
            snap.sums = None if skip_sums else self.sums.clone()
            snap.counts = self.counts.clone()
            snap.drift = self.drift.clone()
            return snap
        names = ("cent64", "counts", "drift") + (() if skip_sums else ("sums",))
        snap.sums = None
        outs = {nm: torch.empty_like(getattr(self, nm)) for nm in names}
        with torch.cuda.stream(stream):
            for nm, t in outs.items():
                t.copy_(getattr(self, nm), non_blocking=True)
                t.record_stream(stream)
                setattr(snap, nm, t)
        return snap

    def _to_host_order(self, dev: np.ndarray) -> np.ndarray:
        if self.order is None:
            return dev
        out = np.empty_like(dev)
        out[:, self.order] = dev
        return out

    def host_centers(self) -> np.ndarray:
        return self._to_host_order(self.cent64.view(self.k, self.d).cpu().numpy())

    def host_sums(self) -> np.ndarray:
        if self.sums is None:
            data, a = self._sums_from
            return fixed_sums_host(data, a, self.k, self.scale_bits).astype(np.float64) * 2.0 ** -self.scale_bits
        s = self.sums.view(self.k, self.d).cpu().numpy().astype(np.float64) * 2.0 ** -self.scale_bits
        return self._to_host_order(s)


def fixed_sums_host(data: Dataset, a: np.ndarray, k: int, scale_bits: int) -> np.ndarray:
    """The device's exact cluster sums, host term order: sum over members of
    rint(float32(x) * 2^S) as int64 (k_aggregate / k_apply_moves; integer
    addition is order-free, so this equals the incrementally maintained sums)."""
    rows = np.repeat(np.asarray(a, dtype=np.int64), np.diff(data.indptr))
    fixed = np.rint(np.asarray(data.data, np.float32).astype(np.float64) * 2.0 ** scale_bits).astype(np.int64)
    out = np.zeros(k * data.dim, np.int64)
    np.add.at(out, rows * data.dim + np.asarray(data.indices, np.int64), fixed)
    return out.reshape(k, data.dim)


class PointState:
    """Per-point bounds and worklists (spkm_bounds + spkm_work)."""

    def __init__(self, n: int, k: int, variant: str, device, elkan_heavy: int = 0, n_total: int | None = None):
        i32 = dict(dtype=torch.int32, device=device)
        self.elkan_heavy = int(elkan_heavy)     # spkm_work.elkan_heavy (0: every bound survivor is scanned)
        # spkm_work.allheavy_rows: skip the bound pass while an iteration still moves >= n / 256 rows
        # (SPKM_EK_ALLHEAVY=0 turns it off; run() clears it while a debug hook reads the bounds)
        # (n_total: the move counter k_finalize compares it with is summed over the ranks of a multi-GPU fit,
        # so every rank and the single-GPU fit take the same decision)
        self.allheavy_rows = ((n_total if n_total is not None else n)
                              if (self.elkan_heavy > 0 and os.environ.get("SPKM_EK_ALLHEAVY", "1") != "0") else 0)
        # simp_elkan with a small heavy threshold: the bound pass lists each light row's (<= 4) failing
        # centers and the scan computes exactly those (spkm_work.lightj; SPKM_EK_LIGHT=0 turns it off)
        self.lightj = (torch.full((max(n, 1) * 4,), -1, **i32)
                       if variant == "simp_elkan" and 0 < self.elkan_heavy <= 5
                       and os.environ.get("SPKM_EK_LIGHT", "1") != "0" else None)
        self.a = torch.zeros(max(n, 1), **i32)
        self.l = torch.zeros(max(n, 1), dtype=torch.float32, device=device)
        if variant in _ELKAN_FAMILY:
            self.ku = (k + 3) // 4 * 4
            self.u = torch.zeros(max(n, 1) * self.ku, dtype=torch.float32, device=device)
        elif variant == "yinyang":      # group bounds ug[n][ceil(k/4) rounded up to 4]
            self.ku = ((k + 3) // 4 + 3) // 4 * 4
            self.u = torch.zeros(max(n, 1) * self.ku, dtype=torch.float32, device=device)
        else:
            self.ku = 1
            self.u = torch.zeros(max(n, 1), dtype=torch.float32, device=device)
        self.surv1 = torch.zeros(max(n, 1), **i32)
        self.surv2 = torch.zeros(max(n, 1), **i32)
        self.mv_i = torch.zeros(max(n, 1), **i32)
        self.mv_old = torch.zeros(max(n, 1), **i32)
        self.ctr = torch.zeros(8, dtype=torch.int64, device=device)
        self.stats = torch.zeros(_lib.ST_COUNT, dtype=torch.float64, device=device)
        self.stats_host = torch.zeros(_lib.ST_COUNT, dtype=torch.float64).pin_memory()
        self.device = device
        self.set_history(128)

    def set_history(self, cap: int):
        """(Re)allocate the per-iteration stats history (device + pinned host mirror)."""
        self.hist_cap = cap
        self.hist = torch.zeros(cap * _lib.ST_COUNT, dtype=torch.float64, device=self.device)
        self.hist_host = torch.zeros(cap * _lib.ST_COUNT + 2, dtype=torch.float64).pin_memory()
        self.bounds = Bounds(_ptr(self.a), _ptr(self.l), _ptr(self.u), self.ku)
        self.work = Work(_ptr(self.surv1), _ptr(self.surv2), _ptr(self.mv_i), _ptr(self.mv_old), _ptr(self.ctr),
                         _ptr(self.stats), _ptr(self.hist), cap, self.elkan_heavy, self.allheavy_rows,
                         _ptr(self.lightj) if self.lightj is not None else None)


# --------------------------------------------------------------- validation
def _validate(data: Dataset, k: int, variant: str, hamerly_update: str):
    if variant not in VARIANTS and variant not in EXTRA_VARIANTS:
        raise ConfigError(f"unknown variant {variant!r}")
    if hamerly_update not in ("safe", "naive"):
        raise ConfigError(f"unknown hamerly_update {hamerly_update!r}")
    if not 1 <= k <= data.n:
        raise InfeasibleError(f"k={k} infeasible for n={data.n}")


def _require_cuda(device):
    if not torch.cuda.is_available():
        raise DeviceError("a CUDA device is required (this build has no CPU path)")
    return torch.device(device or "cuda")


# --------------------------------------------------------------- the loop
class Engine:
    """One clustering run's device state and the per-phase kernel calls.

    ``comm`` (optional) is a ``distributed.Exchange`` for multi-GPU runs:
    the corpus is replicated, this rank's scans run on its device-row range
    [p0, p1) (``self.xs``, a view of the corpus CSR), and the moves of all
    ranks are exchanged with one allgather per iteration.
    """

    def __init__(self, data: Dataset, k: int, variant: str, device=None, hamerly_update: str = "safe",
                 corpus: DeviceCorpus | None = None, comm=None, n_total: int | None = None,
                 use_graphs: bool = True):
        self.device = _require_cuda(device)
        self.k, self.variant = k, variant
        self.naive = int(hamerly_update == "naive")
        self.corpus = corpus if corpus is not None else device_corpus(data, self.device)
        self.comm = comm
        self.n_total = n_total if n_total is not None else self.corpus.n
        self.elkan = variant in _ELKAN_FAMILY
        self.hamerly = variant in _HAMERLY_FAMILY
        self.yy = variant == "yinyang"
        self.needs_cc = variant in _CC_VARIANTS
        self.C = CenterState(k, data.dim, self.n_total, self.device, self.needs_cc, order=self.corpus.order)
        # dense corpora: the tcgen05 similarity pass for standard and the Hamerly
        # family; the Elkan family (per-(point, center) bounds and pair scans)
        # runs the sparse kernels over the dense rows (every row holds all D
        # terms), as does everything when SPKM_DENSE_TC=0 (A/B, tests)
        self.dense = (self.corpus.dense_dim is not None and not self.elkan and not self.yy
                      and os.environ.get("SPKM_DENSE_TC", "1") != "0")
        # rows this rank scans: all of them, or its shard [p0, p1) of the replicated corpus
        self.p0, self.p1 = (comm.p0, comm.p1) if comm is not None else (0, self.corpus.n)
        self.n_loc = self.p1 - self.p0
        cs = self.corpus
        self.xs = cs.struct if comm is None else CSR(
            self.n_loc, cs.d, cs.nnz, _ptr(cs.indptr) + 8 * self.p0, _ptr(cs.indices), _ptr(cs.values),
            _ptr(cs.reps) + 4 * self.p0)
        if self.dense:
            self.C.attach_dense(self.corpus, row0=self.p0, n_rows=self.n_loc, rescan=self.hamerly)
        # sparse center index for the full passes (k > 256; SPKM_CSPARSE=0 turns
        # it off): C4 full pass 222 -> 134 ms, Hamerly rescan -34% (profiles/r02_ab_notes.txt)
        if not self.dense and k > 256 and os.environ.get("SPKM_CSPARSE", "1") != "0":
            self.C.attach_cindex(self.corpus.nnz)
        # Elkan family with a center index: the bound pass routes rows with many unpruned centers to
        # spkm_elkan_heavy (threshold from the library: SPKM_EK_HEAVY_PCT percent of k, 0 = off)
        self.elkan_heavy = (int(_lib.lib().spkm_elkan_heavy_threshold(k))
                            if self.elkan and self.corpus.dense_dim is None else 0)
        self.P = PointState(self.n_loc, k, variant, self.device, elkan_heavy=self.elkan_heavy, n_total=self.n_total)
        self.a_global = torch.zeros(max(cs.n, 1), dtype=torch.int32, device=self.device) if comm is not None else None
        # a dedicated stream: steady-state iterations are replayed as one CUDA graph
        self.stream = torch.cuda.Stream(device=self.device)
        self.stream.wait_stream(torch.cuda.current_stream(self.device))
        self.sp = ctypes_void(self.stream.cuda_stream)
        # the next iteration's center thresholds run on a second stream beside
        # the drift/objective reduction and finalize (fork/join by events); one
        # side stream per main stream, so a graph body captured while the
        # whole-fit capture is open forks to a stream of its own
        self._side = {}
        self.use_graphs = use_graphs and comm is None
        # Elkan family: bound update + scan as one pass (spkm_elkan_bounds_scan)
        # for k <= 128; above, the separate bound pass routes rows to the heavy
        # full pass / the light scan (C3: 221 -> 311 it/s, C4: 13.2 -> 20.7).
        # SPKM_ELKAN_FUSE=0/1 forces it (A/B measurements).
        env = os.environ.get("SPKM_ELKAN_FUSE")
        self.fuse_elkan = (k <= 256 and not self.elkan_heavy) if env is None else env != "0"
        # cluster-ordered survivor lists (spkm_order_by_cluster), SPKM_ORDER=1:
        # the gather passes visit the survivors grouped by a(i).  Off by
        # default: at C4 the clusters are too impure to share term rows, and
        # storage order (longest rows first) was 3% faster (8.94 vs 8.71 it/s,
        # profiles/r02_ab_notes.txt).
        env = os.environ.get("SPKM_ORDER")
        self.order_rows = (not self.dense and 1 < k <= 12288 and env is not None and env != "0")
        if self.order_rows:
            self.P.ord_tmp = torch.empty(max(self.n_loc, 1), dtype=torch.int32, device=self.device)
            self.P.ord_bins = torch.empty(2 * k, dtype=torch.int32, device=self.device)
        self.loop = None                 # device-driven fit loop (CUDA graph with a WHILE node)
        self.fit = None                  # the whole fit as one CUDA graph (fit_launch)
        self.loop_kernels = 0            # kernels per loop-body iteration
        self.limit = torch.zeros(1, dtype=torch.int64, device=self.device)
        self.a_host = torch.empty(max(self.corpus.n, 1), dtype=torch.int32).pin_memory()
        self.rows_host = None
        self._keep = None                # host->device staging kept alive until the stream passes
        self.runs = 0

    def drop_loop(self):
        for name in ("loop", "fit"):
            h = getattr(self, name, None)
            if h is not None:
                self.stream.synchronize()
                _lib.lib().spkm_loop_destroy(h)
                setattr(self, name, None)

    def __del__(self):
        try:
            self.drop_loop()
        except Exception:
            pass

    # -- phases --------------------------------------------------------------
    def load_centers(self, centers: np.ndarray):
        with torch.cuda.stream(self.stream):       # H2D ordered before the kernel on this stream
            keep = self.C.load(centers, self.sp)
        self.C.refresh_dense(self.sp)
        self.stream.synchronize()
        del keep

    def seed_rows(self, data: Dataset, rows):
        """Seed centers = the given data rows (CentroidSet.from_data_rows) built on the device.

        Sparse corpora: only the k row ids travel (pinned, async); the rows
        are gathered from the corpus's float64 device copy.  No host sync."""
        rows = np.asarray(rows, dtype=np.int64)
        dev = self.device
        if self.corpus.dense_dim is None and self.corpus.rows == (0, data.n):
            st = self.corpus.seed_struct(data)
            if self.rows_host is None or self.rows_host.numel() < rows.size:
                self.rows_host = torch.empty(max(rows.size, 1), dtype=torch.int64).pin_memory()
            self.stream.synchronize()          # the pinned staging may still feed the previous fit
            self.rows_host[:rows.size].copy_(torch.from_numpy(rows))
            with torch.cuda.stream(self.stream):
                t_rows = self.rows_host[:rows.size].to(dev, non_blocking=True)
                _lib.call("spkm_seed_rows_csr", self.C.struct, st, _ptr(t_rows), self.sp)
            self._keep = (t_rows,)
            self.seed_h2d_bytes = int(rows.nbytes)
            return
        starts, ends = data.indptr[rows], data.indptr[rows + 1]
        lens = ends - starts
        sptr = np.zeros(rows.size + 1, np.int64)
        np.cumsum(lens, out=sptr[1:])
        sel = np.repeat(starts - sptr[:-1], lens) + np.arange(int(sptr[-1]), dtype=np.int64)
        with torch.cuda.stream(self.stream):       # H2D ordered before the kernel on this stream
            t_ptr = torch.from_numpy(sptr).to(dev)
            t_idx = torch.from_numpy(self.corpus.new_id[data.indices[sel]].astype(np.int32)).to(dev)
            t_val = torch.from_numpy(np.ascontiguousarray(data.data[sel], np.float64)).to(dev)
            _lib.call("spkm_seed_rows", self.C.struct, _ptr(t_ptr), _ptr(t_idx), _ptr(t_val), self.sp)
        self.C.refresh_dense(self.sp)
        self._keep = (t_ptr, t_idx, t_val)
        self.seed_h2d_bytes = int(sptr.nbytes + t_idx.numel() * 4 + t_val.numel() * 8)

    def reset(self):
        _lib.call("spkm_reset_counters", self.P.work, self.sp)
        with torch.cuda.stream(self.stream):
            self.C.ctl.zero_()

    def center_thresholds(self, stream=None, sp=None):
        """cc / s of the current centers (engine.py:192-198).  Multi-GPU: each
        rank computes its round-robin share of the Gram partials, one
        allreduce sums them (exact: each float is nonzero on one rank), every
        rank maps them to cc and s -- the same values as one GPU."""
        stream = self.stream if stream is None else stream
        sp = self.sp if sp is None else sp
        full = int(not self.C.cc_valid)
        ex = self.comm
        if ex is None or ex.world == 1 or not hasattr(ex, "allreduce_sum"):
            _lib.call("spkm_center_thresholds", self.C.struct, _ptr(self.C.gram), _ptr(self.C.tiles), full, sp)
        else:
            _lib.call("spkm_gram_partial", self.C.struct, _ptr(self.C.gram), _ptr(self.C.tiles), full, ex.rank,
                      ex.world, sp)
            nfl = int(_lib.lib().spkm_gram_partial_floats(self.k, self.C.d))
            with torch.cuda.stream(stream):
                ex.allreduce_sum(self.C.gram.view(torch.float32)[:nfl])
            _lib.call("spkm_gram_finish", self.C.struct, _ptr(self.C.gram), full, sp)
        self.C.cc_valid = True

    def _dense(self, mode: int, use_s: int = 0):
        _lib.call("spkm_dense_assign", self.xs, self.C.struct, self.C.dense, self.P.bounds, self.P.work,
                  mode, use_s, None, None, self.sp)

    def init_pass(self):
        mode = (_lib.MODE_INIT_ELKAN if self.elkan else _lib.MODE_INIT_HAMERLY if self.hamerly
                else _lib.MODE_INIT_YINYANG if self.yy else _lib.MODE_INIT_PLAIN)
        if self.dense:
            return self._dense(mode)
        self.C.build_cindex(self.sp)
        _lib.call("spkm_full_assign", self.xs, self.C.struct, self.P.bounds, self.P.work, mode, self.sp)

    def scratch_sums(self):
        if self.comm is None:
            _lib.call("spkm_aggregate_sums", self.corpus.struct, self.C.struct, self.P.bounds,
                      _ptr(self.C.sums), _ptr(self.C.counts), self.sp)
            return
        # multi-GPU: gather every shard's assignments, aggregate the whole
        # (replicated) corpus locally: identical exact sums on every rank
        with torch.cuda.stream(self.stream):
            self.comm.allgather_assignments(self.P.a, self.a_global)
            _lib.call("spkm_aggregate_sums", self.corpus.struct, self.C.struct, Bounds(_ptr(self.a_global), None, None, 1),
                      _ptr(self.C.sums), _ptr(self.C.counts), self.sp)

    def lloyd_pass(self):
        if self.dense:
            return self._dense(_lib.MODE_LLOYD)
        self.C.build_cindex(self.sp)
        _lib.call("spkm_full_assign", self.xs, self.C.struct, self.P.bounds, self.P.work,
                  _lib.MODE_LLOYD, self.sp)

    def bounds_pass(self, use_flag: int):
        if self.yy:
            _lib.call("spkm_yy_bounds", self.xs, self.C.struct, self.P.bounds, self.P.work, self.sp)
        elif self.elkan:
            _lib.call("spkm_elkan_bounds", self.xs, self.C.struct, self.P.bounds, self.P.work, use_flag, self.sp)
        else:
            _lib.call("spkm_hamerly_bounds", self.xs, self.C.struct, self.P.bounds, self.P.work, use_flag,
                      self.naive, self.sp)

    def order_survivors(self):
        """Group the bound survivors (surv1) by cluster before the gather passes."""
        if not self.order_rows:
            return
        P = self.P
        _lib.call("spkm_order_by_cluster", self.k, _ptr(P.a), _ptr(P.surv1), _ptr(P.ctr) + 8 * _lib.CTR_SURV1,
                  self.n_loc, _ptr(P.ord_tmp), None, _ptr(P.ord_bins), _ptr(self.C.ctl), self.sp)

    def scan_pass(self, use_flag: int):
        self.order_survivors()
        if self.yy:
            _lib.call("spkm_yy_scan", self.xs, self.C.struct, self.P.bounds, self.P.work, self.sp)
        elif self.elkan:
            if self.elkan_heavy:
                # rows the stored bounds barely prune: one full pass (over the sparse center index for k > 256)
                self.C.build_cindex(self.sp)
                _lib.call("spkm_elkan_heavy", self.xs, self.C.struct, self.P.bounds, self.P.work, self.sp)
            _lib.call("spkm_elkan_scan", self.xs, self.C.struct, self.P.bounds, self.P.work, use_flag, self.sp)
        elif self.dense:
            self._dense(_lib.DMODE_RESCAN_H, use_flag)   # tighten + full scan on the canonical TC values
        else:
            self.C.build_cindex(self.sp)
            _lib.call("spkm_hamerly_tighten", self.xs, self.C.struct, self.P.bounds, self.P.work, use_flag, self.sp)
            _lib.call("spkm_hamerly_rescan", self.xs, self.C.struct, self.P.bounds, self.P.work, use_flag, self.sp)

    def apply_moves(self):
        if self.comm is None:
            _lib.call("spkm_apply_moves", self.corpus.struct, self.C.struct, self.P.bounds, self.P.work,
                      _ptr(self.C.sums), _ptr(self.C.counts), _ptr(self.C.touched), self.sp)
            return
        # multi-GPU: pack this rank's moves + counters, allgather the slots,
        # apply every rank's moves to the replicated sums (distributed.py)
        ex = self.comm
        with torch.cuda.stream(self.stream):
            _lib.call("spkm_pack_moves", self.P.work, self.P.bounds, self.C.struct, self.p0, ex.cap, _ptr(ex.slot),
                      self.sp)
            ex.allgather_moves()
            _lib.call("spkm_apply_move_slots", self.corpus.struct, self.C.struct, _ptr(ex.slots), ex.world,
                      ex.slot_len, _ptr(self.C.touched), _ptr(self.P.ctr), self.sp)

    def move_centers(self, all_clusters: bool, defer_reduce: bool = False):
        _lib.call("spkm_move_centers", self.C.struct, int(all_clusters) | (4 if defer_reduce else 0), self.sp)
        self.C.refresh_dense(self.sp)

    def update_and_finalize(self, all_clusters: bool, sims_extra: int, scratch: bool = False):
        """Center update (engine.py:321-324), then -- for the variants that
        use center-center bounds -- the NEXT iteration's thresholds
        (engine.py:243) on the side stream: they need only the new centers and
        the touched list, so they run beside the drift/objective reduction
        and the finalize; the main stream joins before the next iteration."""
        if not self.needs_cc:
            self.move_centers(all_clusters)
            if scratch:
                self.scratch_sums()
            self.finalize_launch(all_clusters, sims_extra)
            return
        self.move_centers(all_clusters, defer_reduce=True)
        key = self.stream.cuda_stream
        if key not in self._side:
            side = torch.cuda.Stream(device=self.device)
            self._side[key] = (side, ctypes_void(side.cuda_stream), torch.cuda.Event(), torch.cuda.Event())
        side, side_sp, fork, join = self._side[key]
        fork.record(self.stream)
        side.wait_event(fork)
        self.center_thresholds(side, side_sp)
        join.record(side)
        _lib.call("spkm_center_reduce", self.C.struct, self.sp)
        if scratch:
            self.scratch_sums()
        self.finalize_launch(all_clusters, sims_extra)
        self.stream.wait_event(join)

    def finalize_launch(self, all_clusters: bool, sims_extra: int):
        _lib.call("spkm_finalize", self.C.struct, self.P.work, int(all_clusters), int(sims_extra), self.sp)

    def read_stats(self) -> np.ndarray:
        """The one per-iteration D2H read (64 B stats) and the host sync."""
        with torch.cuda.stream(self.stream):
            self.P.stats_host.copy_(self.P.stats, non_blocking=True)
        self.stream.synchronize()
        return self.P.stats_host.numpy().copy()

    def finalize(self, all_clusters: bool, sims_extra: int) -> np.ndarray:
        self.finalize_launch(all_clusters, sims_extra)
        return self.read_stats()

    def host_bounds(self) -> BoundsState:
        n, h = self.corpus.n, self.corpus.to_host_rows
        a = h(self.P.a[:n].cpu().numpy().astype(np.int64))
        l = h(self.P.l[:n].cpu().numpy().astype(np.float64))
        if self.elkan:
            um = h(self.P.u.view(-1, self.P.ku)[:n, :self.k].cpu().numpy().astype(np.float64))
            return BoundsState(self.variant, a, l, u_matrix=um)
        if self.yy:         # group bounds: u_matrix[i, g] over the centers 4g .. 4g+3
            ug = h(self.P.u.view(-1, self.P.ku)[:n, :(self.k + 3) // 4].cpu().numpy().astype(np.float64))
            return BoundsState(self.variant, a, l, u_matrix=ug)
        u = h(self.P.u[:n].cpu().numpy().astype(np.float64))
        return BoundsState(self.variant, a, l, u=u)

    def centroid_set(self, seed_indices=None) -> CentroidSet:
        C = self.C
        return CentroidSet(centers=C.host_centers(), sums=C.host_sums(), counts=C.counts.cpu().numpy(),
                           prev_centers=None, drift=C.drift.cpu().numpy(), seed_indices=seed_indices)

    # -- one iteration ---------------------------------------------------------
    def _steady(self, debug_hook=None, it=0, seed_indices=None):
        """Kernel sequence of an iteration >= 2 (engine.py:240-337), no host sync."""
        if self.variant == "standard":
            self.lloyd_pass()
            sims_extra = self.n_total * self.k
        elif self.elkan and debug_hook is None and self.fuse_elkan:
            use = int(self.needs_cc)       # cc / s were computed at the end of the previous iteration
            _lib.call("spkm_elkan_bounds_scan", self.xs, self.C.struct, self.P.bounds, self.P.work, use, self.sp)
            sims_extra = 0
        else:
            use = int(self.needs_cc)
            self.bounds_pass(use)
            if debug_hook is not None:
                if hasattr(debug_hook, "device_audit"):    # validation.DeviceBoundAuditor: stays on the device
                    debug_hook.device_audit(it, self)
                else:
                    self.stream.synchronize()
                    debug_hook(it, self.host_bounds(), self.centroid_set(seed_indices))
            self.scan_pass(use)
            sims_extra = 0
        self.apply_moves()
        # exact fixed-point sums: the it % 50 rebuild reproduces the incremental
        # sums bit-for-bit; kept so the reference's schedule is visible
        self.update_and_finalize(False, sims_extra, scratch=(it % _SCRATCH_INTERVAL == 0))

    def enqueue(self, it: int):
        """Launch iteration ``it`` (>= 2) eagerly without a host sync (a no-op
        on the device once the run has converged)."""
        self._steady(None, it)

    def _body(self):
        """One iteration >= 3 as captured into the device loop.  The reference's
        50-iteration scratch rebuild (engine.py:317-320) is left out here: the
        sums are exact int64 fixed point, so the rebuild is the identity
        (tests/test_gpu_kernels.py::test_incremental_update_equals_scratch_bitwise);
        the eager host loop still runs it on schedule."""
        if self.variant == "standard":
            self.lloyd_pass()
            sims_extra = self.n_total * self.k
        elif self.elkan and self.fuse_elkan:
            _lib.call("spkm_elkan_bounds_scan", self.xs, self.C.struct, self.P.bounds, self.P.work,
                      int(self.needs_cc), self.sp)
            sims_extra = 0
        else:
            use = int(self.needs_cc)
            self.bounds_pass(use)
            self.scan_pass(use)
            sims_extra = 0
        self.apply_moves()
        self.update_and_finalize(False, sims_extra)

    def loop_launch(self, max_iter: int):
        """Iterations 3..max_iter as ONE graph launch: a conditional WHILE node
        repeats the captured iteration until the device-side convergence flag
        is set (captured once per engine)."""
        import ctypes
        with torch.cuda.stream(self.stream):
            self.limit.fill_(max_iter)
        if self.loop is None:
            self.stream.synchronize()
            h = ctypes.c_void_p()
            _lib.call("spkm_loop_begin", _ptr(self.C.ctl), _ptr(self.limit), self.sp, ctypes.byref(h))
            _lib._capture = []
            saved, _lib._profiler = _lib._profiler, None
            try:
                self._body()
            finally:
                n = sum(_lib._capture)
                _lib._capture = None
                _lib._profiler = saved
                _lib.call("spkm_loop_end", h)
            self.loop, self.loop_kernels = h, n + 1
        _lib.call("spkm_loop_launch", self.loop, self.sp)

    def fit_graph_ok(self, data: Dataset, max_iter: int) -> bool:
        """The whole-fit graph covers sparse single-device fits seeded by row ids."""
        return (self.use_graphs and self.runs > 0 and self.comm is None and max_iter >= 3
                and self.corpus.dense_dim is None and self.corpus.rows == (0, data.n)
                and self.P.hist_cap >= max_iter + 1)

    def fit_launch(self, data: Dataset, rows, max_iter: int):
        """The whole fit as ONE graph launch: seed-row upload and gather, reset,
        iterations 1-2, the WHILE loop over iterations 3..max_iter, and the
        result downloads (stats history, control words, assignments in host
        row order).  Host inputs (seed row ids, max_iter) are read from a
        pinned buffer by the graph's H2D node, so one capture serves every
        fit of this engine."""
        rows = np.asarray(rows, dtype=np.int64)
        if self.fit is None:
            self._fit_capture(data)
        self.fit_in_np[:self.k] = rows
        self.fit_in_np[self.k] = max_iter
        _lib.call("spkm_loop_launch", self.fit, self.sp)

    def fit_results(self):
        """After the fit graph has finished: (history rows, iterations done, assignments)."""
        F, cap = _lib.ST_COUNT, self.P.hist_cap
        done = int(self.fit_ctl_np[0])
        _lib.note_launches(self.fit_kernels[0] + self.fit_kernels[1] * max(0, done - 2))
        rows = self.P.hist_host.numpy()[:cap * F].reshape(cap, F)
        return rows, done, self.fit_a_np[:self.corpus.n].copy()

    def _fit_capture(self, data: Dataset):
        import ctypes
        k, n, dev = self.k, self.corpus.n, self.device
        F, cap = _lib.ST_COUNT, self.P.hist_cap
        st = self.corpus.seed_struct(data)
        row_perm = self.corpus._seed[2]                 # device row -> host row (kept current by refresh)
        self.fit_in = torch.zeros(k + 1, dtype=torch.int64).pin_memory()
        self.fit_in_np = self.fit_in.numpy()
        self.fit_ctl = torch.zeros(2, dtype=torch.int64).pin_memory()
        self.fit_ctl_np = self.fit_ctl.numpy()
        self.fit_a = torch.zeros(max(n, 1), dtype=torch.int64).pin_memory()
        self.fit_a_np = self.fit_a.numpy()
        self.fit_rows = torch.zeros(k, dtype=torch.int64, device=dev)
        self.fit_out = torch.zeros(max(n, 1), dtype=torch.int64, device=dev)
        body = torch.cuda.Stream(device=dev)
        self.stream.synchronize()
        h = ctypes.c_void_p()
        _lib.call("spkm_fit_graph_begin", self.sp, ctypes.byref(h))
        saved, _lib._profiler = _lib._profiler, None
        _lib._capture = []
        outer = (self.stream, self.sp)
        ok = False
        try:
            _lib.call("spkm_memcpy_async", _ptr(self.fit_rows), self.fit_in.data_ptr(), 8 * k, self.sp)
            _lib.call("spkm_seed_rows_csr", self.C.struct, st, _ptr(self.fit_rows), self.sp)
            _lib.call("spkm_reset_counters", self.P.work, self.sp)
            _lib.call("spkm_memset_async", _ptr(self.C.ctl), 0, 16, self.sp)
            self.C.cc_valid = False
            self.iteration1_launch()
            self.enqueue(2)
            _lib.call("spkm_memcpy_async", _ptr(self.limit), self.fit_in.data_ptr() + 8 * k, 8, self.sp)
            n_pre = sum(_lib._capture) + 1               # + the loop's first condition kernel
            _lib._capture = []
            _lib.call("spkm_fit_graph_loop", h, _ptr(self.C.ctl), _ptr(self.limit), ctypes_void(body.cuda_stream))
            self.stream, self.sp = body, ctypes_void(body.cuda_stream)
            try:
                self._body()
            finally:
                self.stream, self.sp = outer
            n_body = sum(_lib._capture) + 1              # + the condition kernel
            _lib._capture = None
            _lib.call("spkm_loop_end", h)
            _lib.call("spkm_memcpy_async", self.P.hist_host.data_ptr(), _ptr(self.P.hist), 8 * F * cap, self.sp)
            _lib.call("spkm_memcpy_async", self.fit_ctl.data_ptr(), _ptr(self.C.ctl), 16, self.sp)
            _lib.call("spkm_rows_to_host", n, _ptr(row_perm), _ptr(self.P.a), _ptr(self.fit_out), self.sp)
            _lib.call("spkm_memcpy_async", self.fit_a.data_ptr(), _ptr(self.fit_out), 8 * n, self.sp)
            _lib.call("spkm_fit_graph_end", h)
            ok = True
        finally:
            _lib._capture = None
            _lib._profiler = saved
            self.stream, self.sp = outer
            if not ok:
                _lib.lib().spkm_fit_graph_abort(h)
        self.fit = h
        self.fit_kernels = (n_pre + 1, n_body)          # + rows_to_host
        self._fit_keep = (body, row_perm)

    def read_history(self, first: int, count: int, with_a: bool = False):
        """One D2H of stats rows [first, first+count) and the control words
        (and the assignments into a pinned buffer), then one host sync."""
        F = _lib.ST_COUNT
        n = self.n_loc
        with torch.cuda.stream(self.stream):
            self.P.hist_host[:count * F].copy_(self.P.hist[first * F:(first + count) * F], non_blocking=True)
            self.P.hist_host[-2:].copy_(self.C.ctl.to(torch.float64), non_blocking=True)
            if with_a and n:
                self.a_host[:n].copy_(self.P.a[:n], non_blocking=True)
        self.stream.synchronize()
        h = self.P.hist_host.numpy()
        return h[:count * F].reshape(count, F).copy(), int(h[-2]), bool(h[-1])

    def iteration1_launch(self):
        """Iteration 1 (engine.py:249-271): full pass, scratch sums, move all, stats."""
        self.init_pass()
        self.scratch_sums()
        self.update_and_finalize(True, self.n_total * self.k)

    def iteration(self, it: int, debug_hook=None, seed_indices=None) -> tuple:
        if it == 1:
            self.iteration1_launch()
            return self.read_stats(), None
        if debug_hook is not None:
            self._steady(debug_hook, it, seed_indices)
        else:
            self.enqueue(it)
        return self.read_stats(), None


def run(data: Dataset, k: int, variant: str, seeding=None, max_iter: int = 100, debug_hook=None,
        hamerly_update: str = "safe", *, device=None, corpus: DeviceCorpus | None = None,
        init_centers: np.ndarray | None = None, comm=None, n_total: int | None = None,
        seed_indices=None, use_graphs: bool = True) -> ClusteringResult:
    """Cluster ``data`` into ``k`` groups (reference engine.run, engine.py:201-346)."""
    from .seeding import SeedConfig, seed_rows_for

    _validate(data, k, variant, hamerly_update)
    if comm is not None and debug_hook is not None:
        raise ConfigError("debug_hook is single-process only (the reference's hook sees every row)")
    cfg = seeding if seeding is not None else SeedConfig()
    if init_centers is None:
        cfg.validate()
        seed_indices = seed_rows_for(data, k, cfg, device=device, corpus=corpus)
    eng = _engine_for(data, k, variant, device, hamerly_update, corpus, comm, n_total, use_graphs)
    if eng.P.hist_cap < max_iter + 1:
        eng.drop_loop()                     # the captured loop holds the old history pointer
        eng.P.set_history(max_iter + 1)
    # a debug hook reads the bounds between the bound pass and the scans: never skip the bound pass then
    # (hook runs are eager, so the struct is read at every call; captured graphs hold the no-hook value)
    eng.P.work.allheavy_rows = 0 if debug_hook is not None else eng.P.allheavy_rows
    prof = _lib.active_profiler()
    untimed = not (prof is not None and prof.timed)
    device_loop = (eng.use_graphs and eng.runs > 0 and debug_hook is None and comm is None and untimed)
    whole_fit = device_loop and init_centers is None and eng.fit_graph_ok(data, max_iter)
    if whole_fit:
        pass                                # seeding and reset are nodes of the fit graph
    elif init_centers is None:
        eng.seed_rows(data, seed_indices)
        eng.reset()
    else:
        eng.load_centers(init_centers)
        eng.reset()
    cc_per_it = k * (k - 1) // 2 if variant in _CC_VARIANTS else 0
    stats: list = []
    converged = False
    prev_t = [None]

    def record(it, st, dt_ns=None):
        reassign = data.n if it == 1 else int(st[_lib.ST_REASSIGN])
        if dt_ns is None:   # device timestamps (%globaltimer) bracket every iteration
            t_end = st[_lib.ST_TSTAMP]
            t_beg = st[_lib.ST_T0] if it == 1 or prev_t[0] is None else prev_t[0]
            dt_ns = int(max(0.0, t_end - t_beg))
            prev_t[0] = t_end
        stats.append(IterationStats(iteration=it, sim_count=int(st[_lib.ST_SIMS]), cc_sim_count=cc_per_it,
                                    reassignments=reassign, objective=float(st[_lib.ST_OBJECTIVE]),
                                    elapsed_ns=dt_ns, survivors=int(st[_lib.ST_SURV1]),
                                    survivors2=int(st[_lib.ST_SURV2]), nnz_tighten=int(st[_lib.ST_NNZ_TIGHTEN]),
                                    nnz_rescan=int(st[_lib.ST_NNZ_RESCAN]), nnz_elkan=int(st[_lib.ST_NNZ_ELKAN]),
                                    touched=int(st[_lib.ST_TOUCHED]), nnz_moved=int(st[_lib.ST_NNZ_MOVED])))
        return k == 1 or st[_lib.ST_ALLONE] == 1.0 or (it >= 2 and reassign == 0)

    a_read = False
    a_host = None
    if whole_fit:
        # one graph launch per fit; the result snapshot is enqueued behind it
        # so the host builds nothing while the device runs
        eng.fit_launch(data, seed_indices, max_iter)
        snap = eng.C.snapshot(sums_from=None, stream=eng.stream, lazy_sums=True)
        eng.stream.synchronize()
        eng.C.cc_valid = True
        rows, done_its, a_host = eng.fit_results()
        for q in range(min(done_its, max_iter)):
            converged = record(q + 1, rows[q])
            if converged:
                break
    elif device_loop:
        # the whole fit without a host round trip: iteration 1 and 2 eagerly
        # enqueued (iteration 2 rebuilds the full cc table), then iterations
        # 3..max_iter as one graph launch; one D2H of the stats history and
        # the assignments at the end
        eng.iteration1_launch()
        if max_iter >= 2:
            eng.enqueue(2)
        if max_iter >= 3:
            eng.loop_launch(max_iter)
            _lib.note_launches(0)
        rows, done_its, _ = eng.read_history(0, max(1, min(max_iter, eng.P.hist_cap)), with_a=True)
        a_read = True
        if max_iter >= 3:
            _lib.note_launches(eng.loop_kernels * max(0, done_its - 2) + 1)
        for q in range(min(done_its, max_iter)):
            converged = record(q + 1, rows[q])
            if converged:
                break
    else:
        st, _ = eng.iteration(1, debug_hook, seed_indices)
        converged = record(1, st)
        it, chunk = 2, 1
        while not converged and it <= max_iter:
            if debug_hook is not None:
                st, _ = eng.iteration(it, debug_hook, seed_indices)
                converged = record(it, st)
                it += 1
                continue
            # enqueue a chunk of iterations without syncing: the convergence test
            # runs on the device and turns later iterations into no-ops; chunks
            # never cross a scratch-rebuild iteration (it % 50 == 0)
            nxt50 = (it // _SCRATCH_INTERVAL + 1) * _SCRATCH_INTERVAL
            c = min(chunk, max_iter - it + 1, (nxt50 - it) if it % _SCRATCH_INTERVAL else 1)
            for j in range(it, it + c):
                eng.enqueue(j)
            rows, done_its, dev_conv = eng.read_history(it - 1, c)
            for q in range(c):
                if it + q > done_its:
                    break
                converged = record(it + q, rows[q])
                if converged:
                    break
            it += c
            chunk = min(chunk * 2, 8)
    eng.stream.synchronize()
    eng.runs += 1
    torch.cuda.current_stream(eng.device).wait_stream(eng.stream)
    if a_host is not None:
        snap._sums_from = (data, a_host)
        return ClusteringResult(assignments=a_host, centers=DeviceCentroidSet(snap, seed_indices),
                                objective=stats[-1].objective, iterations=stats, converged=converged)
    if comm is not None:
        with torch.cuda.stream(eng.stream):
            comm.allgather_assignments(eng.P.a, eng.a_global)
        eng.stream.synchronize()
        a_dev = eng.a_global[:eng.corpus.n].cpu().numpy()
    else:
        a_dev = eng.a_host[:eng.n_loc].numpy() if a_read else eng.P.a[:eng.n_loc].cpu().numpy()
    a = eng.corpus.to_host_rows(a_dev.astype(np.int64))
    snap = eng.C.snapshot(sums_from=(data, a))
    return ClusteringResult(assignments=a, centers=DeviceCentroidSet(snap, seed_indices),
                            objective=stats[-1].objective, iterations=stats, converged=converged)


# Engines (device buffers + captured CUDA graph) are cached per
# (corpus, k, variant, ...) so repeated fits reuse the same buffers and the
# same graph; results get their own snapshot of the center state.
_ENGINES: "dict" = {}
_ENGINE_CACHE_MAX = 6
_ENGINE_CACHE_HBM_SHARE = 0.45


def _engine_for(data, k, variant, device, hamerly_update, corpus, comm, n_total, use_graphs):
    dev = _require_cuda(device)
    corpus = corpus if corpus is not None else device_corpus(data, dev)
    key = (str(dev), id(corpus), k, variant, hamerly_update, n_total, use_graphs, data.dim, id(comm))
    eng = _ENGINES.pop(key, None)
    if eng is None or eng.corpus is not corpus or eng.comm is not comm:
        eng = None
        # keep the cache within a share of HBM (a C4 engine holds ~20 GB of
        # sums / centers / bounds): drop the least recently used engines first
        total = torch.cuda.get_device_properties(dev).total_memory
        while _ENGINES and torch.cuda.memory_allocated(dev) > _ENGINE_CACHE_HBM_SHARE * total:
            _ENGINES.pop(next(iter(_ENGINES)))
        try:
            eng = Engine(data, k, variant, device=dev, hamerly_update=hamerly_update, corpus=corpus, comm=comm,
                         n_total=n_total, use_graphs=use_graphs)
        except torch.OutOfMemoryError:
            # cached engines of other fits hold HBM (C4: ~25 GB each): drop them and retry once
            if not _ENGINES:
                raise
        if eng is None:
            _ENGINES.clear()
            torch.cuda.synchronize(dev)
            torch.cuda.empty_cache()
            eng = Engine(data, k, variant, device=dev, hamerly_update=hamerly_update, corpus=corpus, comm=comm,
                         n_total=n_total, use_graphs=use_graphs)
    else:
        eng.C.cc_valid = False
        eng.stream.wait_stream(torch.cuda.current_stream(dev))
    _ENGINES[key] = eng
    while len(_ENGINES) > _ENGINE_CACHE_MAX:
        _ENGINES.pop(next(iter(_ENGINES)))
    return eng


def clear_engine_cache():
    _ENGINES.clear()


# --------------------------------------------------------------- predict etc.
def _centers_array(centroids) -> np.ndarray:
    return np.asarray(centroids.centers if hasattr(centroids, "centers") else centroids, dtype=np.float64)


def assign_full(data: Dataset, centroids, device=None):
    """Full argmax pass (engine.py:103-120): (assignments, best, second).

    Ties resolve to the lowest index; best/second are the float32
    canonical similarities widened to float64.
    """
    dev = _require_cuda(device)
    C = _centers_array(centroids)
    k = C.shape[0]
    dc = device_corpus(data, dev)
    cs = CenterState(k, data.dim, data.n, dev, False, order=dc.order)
    keep = cs.load(C, ctypes_void(torch.cuda.current_stream(dev).cuda_stream))
    a = torch.empty(max(data.n, 1), dtype=torch.int32, device=dev)
    best = torch.empty(max(data.n, 1), dtype=torch.float64, device=dev)
    second = torch.empty_like(best)
    sp = ctypes_void(torch.cuda.current_stream(dev).cuda_stream)
    if dc.dense_dim is not None:
        # dense corpora: the same tensor-core similarity the fit uses
        cs.attach_dense(dc)
        cs.refresh_dense(sp)
        b = Bounds(_ptr(a), None, None, 1)
        work = PointState(1, k, "standard", dev)
        _lib.call("spkm_dense_assign", dc.struct, cs.struct, cs.dense, b, work.work, 5, 0, _ptr(best),
                  _ptr(second), sp)
    else:
        _lib.call("spkm_predict", dc.struct, cs.struct, _ptr(a), _ptr(best), _ptr(second), sp)
    torch.cuda.current_stream(dev).synchronize()
    del keep
    h = dc.to_host_rows
    return (h(a[:data.n].cpu().numpy().astype(np.int64)), h(best[:data.n].cpu().numpy()),
            h(second[:data.n].cpu().numpy()))


def _sums_for(data: Dataset, a: np.ndarray, cs: CenterState, dev):
    dc = device_corpus(data, dev)
    at = torch.from_numpy(np.ascontiguousarray(dc.to_device_rows(a), np.int32)).to(dev)
    b = Bounds(_ptr(at), None, None, 1)
    sp = ctypes_void(torch.cuda.current_stream(dev).cuda_stream)
    _lib.call("spkm_aggregate_sums", dc.struct, cs.struct, b, _ptr(cs.sums), _ptr(cs.counts), sp)
    return at


def compute_objective(data: Dataset, assignments, centroids, device=None) -> float:
    """Sum_i <x_i, c_a(i)> (engine.py:123-127), as Sum_j <sums_j, c_j> in float64."""
    dev = _require_cuda(device)
    C = _centers_array(centroids)
    cs = CenterState(C.shape[0], data.dim, data.n, dev, False, order=device_corpus(data, dev).order)
    sp = ctypes_void(torch.cuda.current_stream(dev).cuda_stream)
    keep = cs.load(C, sp)
    at = _sums_for(data, np.asarray(assignments), cs, dev)
    out = torch.zeros(1, dtype=torch.float64, device=dev)
    _lib.call("spkm_objective", cs.struct, _ptr(cs.sums), _ptr(out), sp)
    val = float(out.item())
    del keep, at
    return val


def update_centers(data: Dataset, assignments, centroids: CentroidSet, prev_assignments=None,
                   device=None) -> CentroidSet:
    """Move centers for the given assignments (engine.py:163-189); mutates and returns.

    Sums are rebuilt exactly on the device (fixed point) in both branches;
    with ``prev_assignments`` only the clusters touched by moved points are
    renormalised, as in the reference.
    """
    dev = _require_cuda(device)
    a = np.asarray(assignments, dtype=np.int64)
    k = centroids.k
    cs = CenterState(k, data.dim, data.n, dev, False, order=device_corpus(data, dev).order)
    sp = ctypes_void(torch.cuda.current_stream(dev).cuda_stream)
    keep = cs.load(centroids.centers, sp)
    at = _sums_for(data, a, cs, dev)
    if prev_assignments is None:
        cs.touched.fill_(1)
        all_c = True
    else:
        prev = np.asarray(prev_assignments, dtype=np.int64)
        moved = np.nonzero(a != prev)[0]
        t = np.zeros(k, np.int32)
        t[prev[moved]] = 1
        t[a[moved]] = 1
        cs.touched.copy_(torch.from_numpy(t))
        cs.touched_host = t
        all_c = False
    _lib.call("spkm_move_centers", cs.struct, int(all_c), sp)
    work = PointState(1, k, "standard", dev)
    _lib.call("spkm_finalize", cs.struct, work.work, int(all_c), 0, sp)
    torch.cuda.current_stream(dev).synchronize()
    prev_c = centroids.centers.copy()
    centroids.centers = cs.host_centers()
    centroids.sums = cs.host_sums()
    centroids.counts = cs.counts.cpu().numpy()
    centroids.drift = cs.drift.cpu().numpy()
    changed = np.nonzero(cs.touched_host)[0] if prev_assignments is not None else np.arange(k)
    if centroids.prev_centers is None:
        centroids.prev_centers = prev_c
    else:
        centroids.prev_centers[changed] = prev_c[changed]
    del keep, at
    return centroids
