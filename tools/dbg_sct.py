"""Debug: sparse cold term rows, eager vs whole-fit graph (C2, k=100, standard)."""
import os, sys
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2107_04074_b200 import synth, engine as E
import paper_2107_04074_b200 as m
data = synth.config_dataset("C2")
k = int(sys.argv[1]) if len(sys.argv) > 1 else 100
v = sys.argv[2] if len(sys.argv) > 2 else "standard"
res = {}
for sct in ("0", "1"):
    os.environ["SPKM_SCT"] = sct
    E.clear_engine_cache()
    r1 = m.run(data, k, v, m.SeedConfig(seed=2), max_iter=50)
    r2 = m.run(data, k, v, m.SeedConfig(seed=2), max_iter=50)
    eng = next(iter(E._ENGINES.values()))
    res[sct] = (r1, r2, eng)
    print("SCT", sct, "eng.sct", eng.sct, "eager its", len(r1.iterations), r1.objective, "graph its", len(r2.iterations), r2.objective)
a = res["0"][0]
for name, r in (("sct eager", res["1"][0]), ("sct graph", res["1"][1]), ("dense graph", res["0"][1])):
    oa = [s.objective for s in a.iterations]
    ob = [s.objective for s in r.iterations]
    first = next((i for i in range(min(len(oa), len(ob))) if oa[i] != ob[i]), None)
    print(name, "first differing iteration", first, "assign equal", np.array_equal(a.assignments, r.assignments))
eng = res["1"][2]
C = eng.C
torch.cuda.synchronize()
print("hstat", C.hstat.cpu().numpy())
ct = C.ct32.view(data.dim, C.kp)[C.hot:, :k].cpu().numpy()
ptr = C.sct_ptr.cpu().numpy()
pairs = C.sct_pairs.view(-1, 2).cpu().numpy()
nzc = (ct != 0).sum(1)
print("counts match", np.array_equal(np.diff(ptr), nzc), "total", ptr[-1], "cap", C.sct_cap)
bad = 0
for t in range(0, ct.shape[0], 997):
    seg = pairs[ptr[t]:ptr[t + 1]]
    js = np.nonzero(ct[t])[0]
    vals = ct[t][js]
    if not (np.array_equal(seg[:, 0], js) and np.array_equal(seg[:, 1].view(np.float32), vals)):
        bad += 1
print("sampled rows mismatching", bad)
