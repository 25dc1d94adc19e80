"""The C ABI boundary: libspkm.so loads, exports every symbol include/spkm.h declares,
and the ctypes mirrors of the header structs have the C layout.  No compute calls
(there may be no GPU here)."""

import re
import subprocess
import tempfile
from pathlib import Path

import pytest

from conftest import ROOT

from paper_2107_04074_b200 import _lib

HEADER = ROOT / "include" / "spkm.h"


def declared():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char \*)\s*(spkm_\w+)\(", text, re.M)))


def test_header_declares_the_bound_entry_points():
    assert set(declared()) == set(_lib.exported_symbols())


def test_library_exports_every_declared_symbol():
    if not _lib.LIB_PATH.exists():
        _lib.build()
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True, text=True,
                         check=True).stdout
    syms = set(re.findall(r"\bT (spkm_\w+)", out))
    missing = [s for s in declared() if s not in syms]
    assert not missing, missing
    L = _lib.lib()                       # loads + binds every signature
    assert L.spkm_abi_version() == _lib.ABI_VERSION
    assert L.spkm_padded_k(20) == 24 and L.spkm_padded_k(100) == 104 and L.spkm_padded_k(1000) == 1024


def test_struct_layouts_match_header():
    import ctypes
    src = r'''
#include <stdio.h>
#include <stddef.h>
#include "spkm.h"
#define P(s, f) printf(#s "." #f " %zu\n", offsetof(s, f));
int main(void) {
  printf("spkm_csr %zu\nspkm_centers %zu\nspkm_bounds %zu\nspkm_work %zu\n", sizeof(spkm_csr),
         sizeof(spkm_centers), sizeof(spkm_bounds), sizeof(spkm_work));
  P(spkm_csr, row_eps) P(spkm_centers, scale_bits) P(spkm_centers, hstat) P(spkm_centers, cc)
  P(spkm_bounds, ku) P(spkm_work, stats) P(spkm_centers, ct16)
  return 0;
}
'''
    with tempfile.TemporaryDirectory() as td:
        c = Path(td) / "l.c"
        c.write_text(src)
        exe = Path(td) / "l"
        subprocess.run(["gcc", "-I", str(ROOT / "include"), str(c), "-o", str(exe)], check=True)
        lines = dict(l.split() for l in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split("\n")
                     if l)
    assert int(lines["spkm_csr"]) == ctypes.sizeof(_lib.CSR)
    assert int(lines["spkm_centers"]) == ctypes.sizeof(_lib.Centers)
    assert int(lines["spkm_bounds"]) == ctypes.sizeof(_lib.Bounds)
    assert int(lines["spkm_work"]) == ctypes.sizeof(_lib.Work)
    assert int(lines["spkm_csr.row_eps"]) == _lib.CSR.row_eps.offset
    assert int(lines["spkm_centers.scale_bits"]) == _lib.Centers.scale_bits.offset
    assert int(lines["spkm_centers.hstat"]) == _lib.Centers.hstat.offset
    assert int(lines["spkm_centers.cc"]) == _lib.Centers.cc.offset
    assert int(lines["spkm_bounds.ku"]) == _lib.Bounds.ku.offset
    assert int(lines["spkm_centers.ct16"]) == _lib.Centers.ct16.offset
    assert int(lines["spkm_work.stats"]) == _lib.Work.stats.offset


def test_no_gpu_means_loud_failure(monkeypatch):
    """The product path refuses to run without CUDA (there is no CPU fallback)."""
    import torch
    import paper_2107_04074_b200 as spk
    from paper_2107_04074_b200.sparse import Dataset, SparseVector
    import numpy as np
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    d = Dataset.from_rows([SparseVector(np.array([0]), np.array([1.0])),
                           SparseVector(np.array([1]), np.array([1.0]))], dim=2)
    with pytest.raises(spk.DeviceError):
        spk.run(d, 2, "standard", spk.SeedConfig())
