"""ctypes binding of libspkm.so (the C ABI declared in include/spkm.h).

The library is built in-tree (``build()``, or ``__graft_entry__.build()``)
and loaded from this package directory.  There is no fallback: if the
library is missing or a call fails, a ``DeviceError`` is raised.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

from .errors import DeviceError

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
# SPKM_LIB: an alternative build of the same library (A/B measurements only)
LIB_PATH = Path(os.environ["SPKM_LIB"]) if os.environ.get("SPKM_LIB") else PKG / "libspkm.so"
SRC = PKG / "csrc" / "spkm.cu"
SRC_HOST = PKG / "csrc" / "ingest.cpp"
HEADER = ROOT / "include" / "spkm.h"
ABI_VERSION = 3

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-shared", "-Xcompiler", "-fPIC", "-Xptxas", "-v"]

c_i64 = ctypes.c_int64
c_i32 = ctypes.c_int32
c_vp = ctypes.c_void_p


class CSR(ctypes.Structure):
    _fields_ = [("n", c_i64), ("d", c_i64), ("nnz", c_i64), ("indptr", c_vp), ("indices", c_vp),
                ("values", c_vp), ("row_eps", c_vp)]


class CIndex(ctypes.Structure):
    _fields_ = [("desc", c_vp), ("pairs", c_vp), ("off", c_vp), ("scratch", c_vp), ("scratch_bytes", c_i64),
                ("capacity", c_i64), ("dense_thr", c_i32), ("_pad", c_i32)]


class Centers(ctypes.Structure):
    _fields_ = [("k", c_i64), ("d", c_i64), ("kp", c_i64), ("scale_bits", c_i32), ("_pad", c_i32),
                ("cent64", c_vp), ("ct32", c_vp), ("sums", c_vp), ("counts", c_vp), ("drift", c_vp),
                ("sinp", c_vp), ("touched", c_vp), ("objc", c_vp), ("part", c_vp), ("norm", c_vp), ("cc", c_vp),
                ("s", c_vp), ("hstat", c_vp), ("tlist", c_vp), ("tcount", c_vp), ("ctl", c_vp), ("ct16", c_vp),
                ("cindex", c_vp)]


class Bounds(ctypes.Structure):
    _fields_ = [("a", c_vp), ("l", c_vp), ("u", c_vp), ("ku", c_i64)]


class Dense(ctypes.Structure):
    _fields_ = [("D", c_i64), ("kpad", c_i64), ("x", c_vp), ("b", c_vp), ("xs", c_vp)]


class Seed(ctypes.Structure):
    _fields_ = [("n", c_i64), ("d", c_i64), ("indptr", c_vp), ("indices", c_vp), ("values", c_vp),
                ("row_host", c_vp), ("row_dev", c_vp), ("scratch", c_vp)]


class Svml(ctypes.Structure):
    _fields_ = [("n_rows", c_i64), ("nnz", c_i64), ("max_idx", c_i64), ("err_line", c_i64),
                ("err_msg", ctypes.c_char * 256), ("handle", c_vp)]


class Work(ctypes.Structure):
    _fields_ = [("surv1", c_vp), ("surv2", c_vp), ("mv_i", c_vp), ("mv_old", c_vp), ("ctr", c_vp),
                ("stats", c_vp), ("stats_hist", c_vp), ("hist_cap", c_i64), ("elkan_heavy", c_i64), ("allheavy_rows", c_i64), ("lightj", c_vp)]


# modes / enums (include/spkm.h)
MODE_INIT_PLAIN, MODE_INIT_ELKAN, MODE_INIT_HAMERLY, MODE_LLOYD = 0, 1, 2, 3
MODE_PREDICT, DMODE_RESCAN_H = 5, 6
MODE_INIT_YINYANG = 6          # spkm_full_assign (the dense modes are a separate enum)
CTR_SURV1, CTR_SURV2, CTR_MOVES, CTR_SIMS, CTR_NNZ_TIGHTEN, CTR_NNZ_RESCAN, CTR_NNZ_ELKAN, CTR_NNZ_MOVED = range(8)
(ST_SIMS, ST_REASSIGN, ST_OBJECTIVE, ST_ALLONE, ST_SURV1, ST_SURV2, ST_TOUCHED, ST_NNZ_TIGHTEN, ST_NNZ_RESCAN,
 ST_NNZ_ELKAN, ST_ITER, ST_TSTAMP, ST_T0, ST_NNZ_MOVED) = range(14)
ST_COUNT = 16

# name -> argtypes (restype int unless listed in _RESTYPES)
_P = ctypes.POINTER
_SIGS = {
    "spkm_abi_version": [],
    "spkm_last_error": [],
    "spkm_center_chunks": [c_i64],
    "spkm_padded_k": [c_i64],
    "spkm_reset_counters": [_P(Work), c_vp],
    "spkm_full_assign": [_P(CSR), _P(Centers), _P(Bounds), _P(Work), ctypes.c_int, c_vp],
    "spkm_hamerly_bounds": [_P(CSR), _P(Centers), _P(Bounds), _P(Work), ctypes.c_int, ctypes.c_int, c_vp],
    "spkm_hamerly_tighten": [_P(CSR), _P(Centers), _P(Bounds), _P(Work), ctypes.c_int, c_vp],
    "spkm_hamerly_rescan": [_P(CSR), _P(Centers), _P(Bounds), _P(Work), ctypes.c_int, c_vp],
    "spkm_elkan_bounds": [_P(CSR), _P(Centers), _P(Bounds), _P(Work), ctypes.c_int, c_vp],
    "spkm_yy_bounds": [_P(CSR), _P(Centers), _P(Bounds), _P(Work), c_vp],
    "spkm_yy_scan": [_P(CSR), _P(Centers), _P(Bounds), _P(Work), c_vp],
    "spkm_elkan_scan": [_P(CSR), _P(Centers), _P(Bounds), _P(Work), ctypes.c_int, c_vp],
    "spkm_elkan_bounds_scan": [_P(CSR), _P(Centers), _P(Bounds), _P(Work), ctypes.c_int, c_vp],
    "spkm_elkan_heavy": [_P(CSR), _P(Centers), _P(Bounds), _P(Work), c_vp],
    "spkm_elkan_heavy_threshold": [c_i64],
    "spkm_aggregate_sums": [_P(CSR), _P(Centers), _P(Bounds), c_vp, c_vp, c_vp],
    "spkm_order_by_cluster": [c_i64, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp],
    "spkm_apply_moves": [_P(CSR), _P(Centers), _P(Bounds), _P(Work), c_vp, c_vp, c_vp, c_vp],
    "spkm_move_centers": [_P(Centers), ctypes.c_int, c_vp],
    "spkm_center_reduce": [_P(Centers), c_vp],
    "spkm_gram_tiles": [c_i64, c_vp],
    "spkm_gram_scratch_doubles": [c_i64, c_i64],
    "spkm_center_thresholds": [_P(Centers), c_vp, c_vp, ctypes.c_int, c_vp],
    "spkm_center_scratch_doubles": [c_i64, c_i64],
    "spkm_finalize": [_P(Centers), _P(Work), ctypes.c_int, ctypes.c_longlong, c_vp],
    "spkm_predict": [_P(CSR), _P(Centers), c_vp, c_vp, c_vp, c_vp],
    "spkm_objective": [_P(Centers), c_vp, c_vp, c_vp],
    "spkm_load_centers": [_P(Centers), c_vp, c_vp],
    "spkm_geometry": [ctypes.c_int, c_i64, c_vp, c_vp, c_vp, c_vp],
    "spkm_seed_scratch_doubles": [c_i64, c_i64],
    "spkm_seed_rows_csr": [_P(Centers), _P(Seed), c_vp, c_vp],
    "spkm_loop_begin": [c_vp, c_vp, c_vp, _P(c_vp)],
    "spkm_move_slot_ints": [c_i64],
    "spkm_pack_moves": [_P(Work), _P(Bounds), _P(Centers), c_i64, c_i64, c_vp, c_vp],
    "spkm_apply_move_slots": [_P(CSR), _P(Centers), c_vp, ctypes.c_int, c_i64, c_vp, c_vp, c_vp],
    "spkm_audit_transpose": [c_i64, c_i64, c_i64, c_vp, c_vp, c_vp],
    "spkm_audit": [_P(Seed), c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, c_i64, ctypes.c_int, c_vp, c_vp, c_vp],
    "spkm_permute_rows": [c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp],
    "spkm_prepare_scratch_bytes": [c_i64, c_i64],
    "spkm_dense_ids": [c_i64, c_i64, c_vp, c_vp, c_vp, c_vp],
    "spkm_gram_partial_floats": [c_i64, c_i64],
    "spkm_cindex_scratch_bytes": [c_i64],
    "spkm_cindex_build": [_P(Centers), c_vp],
    "spkm_gram_partial": [_P(Centers), c_vp, c_vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, c_vp],
    "spkm_gram_finish": [_P(Centers), c_vp, ctypes.c_int, c_vp],
    "spkm_prepare_rows": [c_i64, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_vp],
    "spkm_loop_end": [c_vp],
    "spkm_fit_graph_begin": [c_vp, _P(c_vp)],
    "spkm_fit_graph_loop": [c_vp, c_vp, c_vp, c_vp],
    "spkm_fit_graph_end": [c_vp],
    "spkm_fit_graph_abort": [c_vp],
    "spkm_rows_to_host": [c_i64, c_vp, c_vp, c_vp, c_vp],
    "spkm_memcpy_async": [c_vp, c_vp, c_i64, c_vp],
    "spkm_memset_async": [c_vp, ctypes.c_int, c_i64, c_vp],
    "spkm_loop_launch": [c_vp, c_vp],
    "spkm_loop_destroy": [c_vp],
    "spkm_seed_kmpp": [_P(Seed), c_i64, ctypes.c_double, ctypes.c_uint64, c_vp, c_vp, c_vp],
    "spkm_seed_afkmc2": [_P(Seed), c_i64, ctypes.c_double, c_i64, ctypes.c_uint64, c_vp, c_vp],
    "spkm_host_row_norms": [c_i64, c_vp, c_vp, c_vp],
    "spkm_svml_parse": [c_vp, c_i64, ctypes.c_int, _P(Svml)],
    "spkm_svml_fetch": [_P(Svml), c_vp, c_vp, c_vp],
    "spkm_svml_free": [_P(Svml)],
    "spkm_host_idf": [c_i64, c_vp, c_i64, ctypes.c_int, c_vp],
    "spkm_seed_rows": [_P(Centers), c_vp, c_vp, c_vp, c_vp],
    "spkm_dense_centers": [_P(Centers), _P(Dense), c_vp],
    "spkm_dense_assign": [_P(CSR), _P(Centers), _P(Dense), _P(Bounds), _P(Work), ctypes.c_int, ctypes.c_int,
                          c_vp, c_vp, c_vp],
}
_RESTYPES = {
    "spkm_last_error": ctypes.c_char_p,
    "spkm_center_chunks": c_i64,
    "spkm_padded_k": c_i64,
    "spkm_gram_tiles": c_i64,
    "spkm_gram_scratch_doubles": c_i64,
    "spkm_center_scratch_doubles": c_i64,
    "spkm_seed_scratch_doubles": c_i64,
    "spkm_move_slot_ints": c_i64,
    "spkm_prepare_scratch_bytes": c_i64,
    "spkm_gram_partial_floats": c_i64,
    "spkm_cindex_scratch_bytes": c_i64,
    "spkm_elkan_heavy_threshold": c_i64,
}

# kernels each entry point launches (for the bench's gpu_launches count)
KERNELS_PER_CALL = {
    "spkm_full_assign": 1, "spkm_hamerly_bounds": 1, "spkm_hamerly_tighten": 1, "spkm_hamerly_rescan": 1,
    "spkm_elkan_bounds": 1, "spkm_elkan_scan": 1, "spkm_elkan_heavy": 1, "spkm_yy_bounds": 1, "spkm_yy_scan": 1, "spkm_elkan_bounds_scan": 1, "spkm_aggregate_sums": 1, "spkm_apply_moves": 1,
    "spkm_move_centers": 5, "spkm_center_reduce": 1, "spkm_center_thresholds": 3, "spkm_finalize": 1, "spkm_predict": 1,
    "spkm_objective": 2, "spkm_load_centers": 1, "spkm_geometry": 1, "spkm_seed_rows": 1,
    "spkm_dense_centers": 1, "spkm_dense_assign": 1, "spkm_reset_counters": 1,
    "spkm_seed_rows_csr": 1, "spkm_permute_rows": 1, "spkm_prepare_rows": 7, "spkm_dense_ids": 1, "spkm_gram_partial": 1, "spkm_gram_finish": 2, "spkm_cindex_build": 1, "spkm_audit": 1, "spkm_audit_transpose": 1,
    "spkm_pack_moves": 1, "spkm_apply_move_slots": 1, "spkm_rows_to_host": 1,
    "spkm_order_by_cluster": 4,
}

_lib = None


class CallProfiler:
    """Counts launches per entry point; optionally brackets each call with CUDA events.

    Events are recorded on the stream argument of the call (the stream the
    kernels run on), so they time exactly that entry point's kernels.
    """

    def __init__(self, timed: bool = False):
        self.timed = timed
        self.launches = 0
        self.calls = {}
        self.records = []   # (name, start_event, end_event, tag)
        self.tag = None

    def __enter__(self):
        global _profiler
        self._prev = _profiler
        _profiler = self
        return self

    def __exit__(self, *exc):
        global _profiler
        _profiler = self._prev
        return False

    def times_ms(self) -> dict:
        out = {}
        for name, e0, e1, tag in self.records:
            key = (name, tag)
            out[key] = out.get(key, 0.0) + e0.elapsed_time(e1)
        return out


_profiler = None
_capture = None     # list collecting kernel counts while a CUDA graph is captured


def build(verbose: bool = False) -> Path:
    """Compile csrc/spkm.cu for sm_100a into the package directory."""
    nvcc = os.environ.get("NVCC", "nvcc")
    cmd = [nvcc, *NVCC_FLAGS, "-I", str(ROOT / "include"), "-o", str(LIB_PATH), str(SRC), str(SRC_HOST)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise DeviceError(f"nvcc failed:\n{r.stderr[-4000:]}")
    if verbose:
        print(r.stderr)
    return LIB_PATH


CHECK_LIB_PATH = PKG / "libspkm_check.so"


def build_check(verbose: bool = False) -> Path:
    """The debug build with device-side bounds checks (-DSPKM_CHECKS=1): same
    ABI, loaded with SPKM_LIB=libspkm_check.so by tests/test_gpu_checks.py."""
    nvcc = os.environ.get("NVCC", "nvcc")
    cmd = [nvcc, *NVCC_FLAGS, "-DSPKM_CHECKS=1", "-I", str(ROOT / "include"), "-o", str(CHECK_LIB_PATH), str(SRC),
           str(SRC_HOST)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise DeviceError(f"nvcc failed:\n{r.stderr[-4000:]}")
    return CHECK_LIB_PATH


def exported_symbols() -> list:
    return sorted(_SIGS)


def lib():
    """Load libspkm.so (raises DeviceError if it is missing)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise DeviceError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback exists)")
    L = ctypes.CDLL(str(LIB_PATH))
    for name, args in _SIGS.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = _RESTYPES.get(name, ctypes.c_int)
    if L.spkm_abi_version() != ABI_VERSION:
        raise DeviceError("libspkm.so ABI mismatch; rebuild")
    _lib = L
    return L


def active_profiler():
    return _profiler


def note_launches(n: int):
    """Credit kernels launched outside call() (CUDA-graph replays) to the active profiler."""
    if _profiler is not None:
        _profiler.launches += n


def kernels_for(name: str, args) -> int:
    n = KERNELS_PER_CALL.get(name, 0)
    if name == "spkm_order_by_cluster" and len(args) > 2 and args[2] is None:
        n -= 1                                   # identity input: no copy back
    if name == "spkm_move_centers" and len(args) > 1:
        if int(args[1]) & 4:
            n -= 1                               # the reduction is issued by spkm_center_reduce
        k, d = getattr(args[0], "k", 1 << 30), getattr(args[0], "d", 1 << 30)
        if k <= 2048 and (d + 4095) // 4096 * k <= 65536:
            n -= 1                               # the touched list is built inside the norm pass
    if name == "spkm_prepare_rows" and len(args) > 8:
        # rows: keys, 1 + 4 radix-sort passes, lengths, 2 scan kernels; terms: df, iota, 1 + 4, inverse
        n = (9 if args[5] is not None else 0) + (8 if args[8] is not None else 0)
    return n


def call(name: str, *args):
    """Call an int-returning entry point and raise on a non-zero status."""
    L = lib()
    prof = _profiler
    if _capture is not None:
        _capture.append(kernels_for(name, args))
    if prof is not None:
        prof.launches += kernels_for(name, args)
        prof.calls[name] = prof.calls.get(name, 0) + 1
        if prof.timed:
            import torch
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            stream = torch.cuda.ExternalStream(args[-1].value) if args and isinstance(args[-1], ctypes.c_void_p) \
                and args[-1].value else torch.cuda.current_stream()
            e0.record(stream)
            rc = getattr(L, name)(*args)
            e1.record(stream)
            prof.records.append((name, e0, e1, prof.tag))
        else:
            rc = getattr(L, name)(*args)
    else:
        rc = getattr(L, name)(*args)
    if rc != 0:
        msg = L.spkm_last_error().decode(errors="replace")
        raise DeviceError(f"{name} failed ({rc}): {msg}")
    return rc
