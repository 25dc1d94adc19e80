"""Host logic of bench.py (CPU): the multi-GPU re-exec under torch.distributed.run
and the CPU legs' folded sample."""

import importlib.util
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent


def _bench():
    spec = importlib.util.spec_from_file_location("bench_mod", ROOT / "bench.py")
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def test_gpus_flag_reexecs_under_torchrun(monkeypatch):
    b = _bench()
    seen = {}

    def fake_call(cmd):
        seen["cmd"] = cmd
        return 0

    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(b.subprocess, "call", fake_call)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "2"])
    args = b.parse()
    try:
        b.maybe_launch_ranks(args)
    except SystemExit as e:
        assert e.code == 0
    cmd = seen["cmd"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "127.0.0.1" in cmd
    assert cmd[-4:] == ["--gpus", "4", "--steps", "2"]
    # already under torchrun, or one GPU: no re-exec
    monkeypatch.setenv("WORLD_SIZE", "4")
    assert b.maybe_launch_ranks(args) is False


def test_cpu_sample_folds_terms_and_renormalises():
    from paper_2107_04074_b200.sparse import Dataset
    b = _bench()
    g = np.random.default_rng(3)
    n, d = 50, 100_000
    lens = g.integers(2, 30, n)
    ip = np.concatenate([[0], np.cumsum(lens)])
    idx = np.concatenate([np.sort(g.choice(d, L, replace=False)) for L in lens])
    data = Dataset.from_csr(ip, idx, g.uniform(0.1, 1.0, idx.size), d)
    fip, fidx, fval, ds = b.cpu_sample(data, 40, d_fold=1000)
    assert ds == 1000 and fip.size == 41 and fidx.max() < 1000
    for i in range(40):
        s, e = fip[i], fip[i + 1]
        assert np.all(np.diff(fidx[s:e]) > 0)                     # merged duplicates, sorted
        assert abs(np.sum(fval[s:e] ** 2) - 1.0) < 1e-12          # unit rows again
        # the folded row is the original row's weights summed per id mod d'
        ref = np.zeros(1000)
        np.add.at(ref, data.indices[data.indptr[i]:data.indptr[i + 1]] % 1000,
                  data.data[data.indptr[i]:data.indptr[i + 1]])
        ref /= np.linalg.norm(ref)
        assert np.allclose(ref[fidx[s:e]], fval[s:e], rtol=0, atol=1e-15)
    # d <= d': the sample is the first rows unchanged
    sip, sidx, sval, sd = b.cpu_sample(data, 10, d_fold=10 ** 6)
    assert sd == d and np.array_equal(sval, data.data[:sip[-1]])
