"""Experiment: does processing rows grouped by cluster speed up the full row pass (L1/L2 reuse)?"""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2107_04074_b200 import synth, engine as E, _lib
cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
k = int(sys.argv[2]) if len(sys.argv) > 2 else 100
data = synth.config_dataset(cfg)
eng = E.Engine(data, k, "standard", use_graphs=False)
eng.seed_rows(data, np.arange(k) * 7)
eng.reset()
eng.iteration(1)
eng.iteration(2)
torch.cuda.synchronize()
A = E.ctypes_void(eng.stream.cuda_stream)
def timeit(fn, reps=20):
    st = eng.stream
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn(); st.synchronize()
    e0.record(st)
    for _ in range(reps): fn()
    e1.record(st); st.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3
def lloyd_plain():
    _lib.call("spkm_full_assign", eng.corpus.struct, eng.C.struct, eng.P.bounds, eng.P.work, _lib.MODE_INIT_PLAIN, A)
print("plain rows (init mode) us:", timeit(lloyd_plain))
if len(sys.argv) > 3: sys.exit(0)
a = eng.P.a[:data.n].clone()
with torch.cuda.stream(eng.stream):
    order = torch.argsort(a.long(), stable=True).to(torch.int32)
    cnt = torch.tensor([data.n], dtype=torch.int64, device="cuda")
# rescan machinery: rowlist = order via surv2 + ctr
eng.P.surv2.copy_(order)
def sorted_pass():
    eng.P.ctr[1] = data.n  # SURV2 count
    _lib.call("spkm_hamerly_rescan", eng.corpus.struct, eng.C.struct, eng.P.bounds, eng.P.work, A) if False else None
# use predict with a permuted corpus instead: emulate by building a permuted DeviceCorpus
perm = order.cpu().numpy().astype(np.int64)
ip = data.indptr
rows = [np.arange(ip[i], ip[i+1]) for i in perm]
sel = np.concatenate(rows)
lens = np.diff(ip)[perm]
ip2 = np.concatenate([[0], np.cumsum(lens)])
d2 = E.Dataset(ip2, data.indices[sel], data.data[sel], data.dim)
c2 = E.DeviceCorpus(d2, torch.device("cuda"))
torch.cuda.synchronize()
def lloyd_sorted():
    _lib.call("spkm_full_assign", c2.struct, eng.C.struct, eng.P.bounds, eng.P.work, _lib.MODE_INIT_PLAIN, A)
print("cluster-sorted rows us:", timeit(lloyd_sorted))
rp = np.random.default_rng(0).permutation(data.n)
rows = [np.arange(ip[i], ip[i+1]) for i in rp]
sel = np.concatenate(rows); lens = np.diff(ip)[rp]
d3 = E.Dataset(np.concatenate([[0], np.cumsum(lens)]), data.indices[sel], data.data[sel], data.dim)
c3 = E.DeviceCorpus(d3, torch.device("cuda")); torch.cuda.synchronize()
def lloyd_rand():
    _lib.call("spkm_full_assign", c3.struct, eng.C.struct, eng.P.bounds, eng.P.work, _lib.MODE_INIT_PLAIN, A)
print("random-order rows us:", timeit(lloyd_rand))

lp = np.argsort(-np.diff(ip), kind="stable")
rows = [np.arange(ip[i], ip[i+1]) for i in lp]
sel = np.concatenate(rows); lens = np.diff(ip)[lp]
d4 = E.Dataset(np.concatenate([[0], np.cumsum(lens)]), data.indices[sel], data.data[sel], data.dim)
c4 = E.DeviceCorpus(d4, torch.device("cuda")); torch.cuda.synchronize()
def lloyd_len():
    _lib.call("spkm_full_assign", c4.struct, eng.C.struct, eng.P.bounds, eng.P.work, _lib.MODE_INIT_PLAIN, A)
print("length-desc rows us:", timeit(lloyd_len))
