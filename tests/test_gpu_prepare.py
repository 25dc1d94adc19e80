"""spkm_prepare_rows (csrc/prepare.cuh): the device layout of an uploaded corpus
equals the host definition -- rows longest first (stable), their offsets, the
term order by document frequency (stable) and its inverse -- bit for bit."""

import ctypes

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _prepare(ip, idx, d, with_pos=True, with_terms=True):
    from paper_2107_04074_b200 import _lib
    dev = torch.device("cuda:0")
    n, nnz = ip.size - 1, int(ip[-1])
    nb = int(_lib.lib().spkm_prepare_scratch_bytes(n, d))
    scratch = torch.empty(max(nb, 1), dtype=torch.uint8, device=dev)
    ip_d = torch.from_numpy(ip).to(dev)
    idx_d = torch.from_numpy(idx.astype(np.int32)).to(dev)
    perm = torch.full((max(n, 1),), -7, dtype=torch.int64, device=dev)
    pos = torch.full((max(n, 1),), -7, dtype=torch.int64, device=dev)
    indptr = torch.full((n + 1,), -7, dtype=torch.int64, device=dev)
    order = torch.full((max(d, 1),), -7, dtype=torch.int64, device=dev)
    new_id = torch.full((max(d, 1),), -7, dtype=torch.int64, device=dev)
    p = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    sp = ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
    _lib.call("spkm_prepare_rows", n, d, nnz, p(ip_d), p(idx_d), p(perm), p(pos) if with_pos else None, p(indptr),
              p(order) if with_terms else None, p(new_id) if with_terms else None, p(scratch), nb, sp)
    torch.cuda.synchronize()
    return (perm[:n].cpu().numpy(), pos[:n].cpu().numpy(), indptr.cpu().numpy(), order[:d].cpu().numpy(),
            new_id[:d].cpu().numpy())


@pytest.mark.parametrize("n,d,maxlen", [(1, 1, 1), (7, 5, 3), (5000, 300, 40), (200_000, 50_000, 400),
                                        (3000, 70_000, 70_000)])
def test_prepare_rows_matches_host(n, d, maxlen):
    g = np.random.default_rng(n + d)
    lens = g.integers(1, maxlen + 1, n)
    lens[g.random(n) < 0.3] = 1 + maxlen // 2          # many ties: stability matters
    ip = np.zeros(n + 1, np.int64)
    np.cumsum(lens, out=ip[1:])
    idx = (g.zipf(1.3, int(ip[-1])) - 1) % d
    perm, pos, indptr, order, new_id = _prepare(ip, idx, d)
    ref_perm = np.argsort(-lens, kind="stable")
    assert np.array_equal(perm, ref_perm)
    inv = np.empty(n, np.int64)
    inv[ref_perm] = np.arange(n)
    assert np.array_equal(pos, inv)
    ref_ip = np.zeros(n + 1, np.int64)
    np.cumsum(lens[ref_perm], out=ref_ip[1:])
    assert np.array_equal(indptr, ref_ip)
    df = np.bincount(idx, minlength=d)
    ref_order = np.argsort(-df, kind="stable")
    assert np.array_equal(order, ref_order)
    ref_new = np.empty(d, np.int64)
    ref_new[ref_order] = np.arange(d)
    assert np.array_equal(new_id, ref_new)


def test_prepare_rows_parts_and_errors():
    from paper_2107_04074_b200 import _lib
    ip = np.array([0, 2, 5, 6], np.int64)
    idx = np.array([0, 1, 1, 2, 3, 3])
    perm, pos, indptr, order, new_id = _prepare(ip, idx, 4, with_pos=False, with_terms=False)
    assert list(perm) == [1, 0, 2] and list(indptr) == [0, 3, 5, 6]
    assert list(order) == [-7] * 4                       # term part skipped
    assert _lib.lib().spkm_prepare_scratch_bytes(1 << 31, 4) == -1
    with pytest.raises(_lib.DeviceError):
        _lib.call("spkm_prepare_rows", 3, 4, 6, None, None, None, None, None, None, None, None, 0, None)


def test_device_corpus_layout_equals_host_layout():
    """DeviceCorpus built on the GPU == the numpy layout (_host_prepare) of the same Dataset."""
    from paper_2107_04074_b200 import synth
    from paper_2107_04074_b200.engine import DeviceCorpus
    data = synth.config_dataset("C3", n_override=30_000)
    gpu = DeviceCorpus(data, "cuda:0")
    data2 = type(data)(data.indptr, data.indices, data.data, data.dim)
    cpu = DeviceCorpus(data2, "cpu")
    for name in ("indptr", "indices", "values", "reps"):
        a = getattr(gpu, name)[: getattr(cpu, name).numel()].cpu()
        assert torch.equal(a, getattr(cpu, name)), name
    assert np.array_equal(gpu.new_id, cpu.new_id) and np.array_equal(gpu.order, cpu.order)
    assert np.array_equal(gpu.row_perm, cpu.row_perm)


def test_dense_corpus_float32_upload_equals_host_layout():
    """Dense corpora upload their float32 rows (Dataset.dense keeps them) straight into the device
    buffer; the layout equals the float64-upload path's and the host layout's."""
    from paper_2107_04074_b200 import synth
    from paper_2107_04074_b200.engine import DeviceCorpus
    data = synth.config_dataset("C5", n_override=3000, cache_dir="")
    assert data._values32.dtype == np.float32
    fast = DeviceCorpus(data, "cuda:0")
    slow_data = type(data)(data.indptr, data.indices, data.data, data.dim)
    slow_data.dense_dim = data.dense_dim                 # no _values32: the float64 path
    slow = DeviceCorpus(slow_data, "cuda:0")
    cpu = DeviceCorpus(type(data)(data.indptr, data.indices, data.data, data.dim), "cpu")
    for name in ("indptr", "indices", "values", "reps"):
        a = getattr(fast, name)[: getattr(slow, name).numel()].cpu()
        assert torch.equal(a, getattr(slow, name).cpu()), name
    for name in ("indptr", "indices", "values"):
        assert torch.equal(getattr(fast, name)[: getattr(cpu, name).numel()].cpu(), getattr(cpu, name)), name
    assert fast.h2d_bytes * 2 <= slow.h2d_bytes
    assert np.array_equal(fast.row_perm, np.arange(data.n))
