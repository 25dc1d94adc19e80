"""Host time per fit outside the device wait (C2 k=100, 5 variants): where the GPU idles between fits."""
import sys, time
sys.path.insert(0, ".")
import torch
import numpy as np
from paper_2107_04074_b200 import synth, run, SeedConfig
from paper_2107_04074_b200 import engine as E
data = synth.config_dataset(sys.argv[1] if len(sys.argv) > 1 else "C2")
dev = torch.device("cuda")
corpus = E.device_corpus(data, dev)
V = ("standard", "elkan", "simp_elkan", "hamerly", "simp_hamerly")
T = {}
orig_rh = E.Engine.read_history
def rh(self, *a, **kw):
    t0 = time.perf_counter()
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    r = orig_rh(self, *a, **kw)
    t2 = time.perf_counter()
    T.setdefault("pre_wait", []).append(t0)
    T.setdefault("wait_end", []).append(t1)
    T.setdefault("rh_end", []).append(t2)
    return r
E.Engine.read_history = rh
import functools, collections
PH = collections.defaultdict(list)
def wrap(obj, name):
    f = getattr(obj, name)
    @functools.wraps(f)
    def g(*a, **kw):
        t0 = time.perf_counter()
        r = f(*a, **kw)
        PH[name].append(time.perf_counter() - t0)
        return r
    setattr(obj, name, g)
import paper_2107_04074_b200.seeding as S
wrap(S, "seed_rows_for")
wrap(E, "_engine_for")
for m in ("seed_rows", "reset", "iteration1_launch", "enqueue", "loop_launch"):
    wrap(E.Engine, m)
wrap(E.CenterState, "snapshot")
wrap(E.DeviceCorpus, "to_host_rows")
def step(log):
    for v in V:
        t0 = time.perf_counter()
        run(data, 100, v, SeedConfig(seed=2), max_iter=50, device=dev, corpus=corpus)
        t1 = time.perf_counter()
        if log:
            T.setdefault("run", []).append((t0, t1))
for _ in range(3): step(False)
T.clear()
PH.clear()
for _ in range(5): step(True)
for k2, v in PH.items():
    print(f"  {k2:20s} median {np.median(v) * 1e6:7.1f} us  x{len(v)}")
runs = T["run"]
T.setdefault("pre_wait", [t for t, _ in runs]); T.setdefault("wait_end", [t for t, _ in runs]); T.setdefault("rh_end", [t for t, _ in runs])
pre = np.array([T["pre_wait"][i] - runs[i][0] for i in range(len(runs))]) * 1e6
rdh = np.array([T["rh_end"][i] - T["wait_end"][i] for i in range(len(runs))]) * 1e6
post = np.array([runs[i][1] - T["rh_end"][i] for i in range(len(runs))]) * 1e6
between = np.array([runs[i + 1][0] - runs[i][1] for i in range(len(runs) - 1)]) * 1e6
print(f"per fit (us, median): enqueue {np.median(pre):.0f}  read_history after wait {np.median(rdh):.0f}  "
      f"post {np.median(post):.0f}  between runs {np.median(between):.0f}")
