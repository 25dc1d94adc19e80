"""The bounds-checked debug build (-DSPKM_CHECKS=1, libspkm_check.so) runs the
small-case workload of tools/sanitize_fits.py -- every variant eager and via
the CUDA graphs, predict, k-means++ / AFK-MC2 seeding, the bound auditor, a
dense (tcgen05) fit -- with device-side checks on the indices the kernels
trust (term ids < d, rows < n, assignments < k, moves <= slot capacity, active
groups <= groups).  A failed check traps the kernel with a message.  This and
the bit-exact comparisons stand in for compute-sanitizer, which this GPU pool
does not allow."""

import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent


def test_checked_build_runs_the_workload_clean():
    from paper_2107_04074_b200 import _lib
    lib = _lib.CHECK_LIB_PATH
    if not lib.exists():
        _lib.build_check()
    env = dict(os.environ, SPKM_LIB=str(lib))
    r = subprocess.run([sys.executable, str(ROOT / "tools" / "sanitize_fits.py")], env=env, capture_output=True,
                       text=True, timeout=900)
    out = r.stdout + r.stderr
    assert "SPKM_CHECK failed" not in out, out[-3000:]
    assert r.returncode == 0, out[-3000:]
    assert "sanitize workload done" in r.stdout
    # the checked library is the one that ran
    assert "libspkm_check.so" in subprocess.run(
        [sys.executable, "-c", "from paper_2107_04074_b200 import _lib; print(_lib.LIB_PATH)"], env=env,
        capture_output=True, text=True, cwd=ROOT).stdout
