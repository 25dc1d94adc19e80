"""Wall-clock breakdown of bench.py's e2e step on C2: refresh + 5 fits through the public API."""
import sys, time
sys.path.insert(0, ".")
import torch
from paper_2107_04074_b200 import synth, run, SeedConfig
from paper_2107_04074_b200.engine import DeviceCorpus
data = synth.config_dataset("C2")
dev = torch.device("cuda")
c = DeviceCorpus(data, dev, pinned_host=True)
V = ("standard", "elkan", "simp_elkan", "hamerly", "simp_hamerly")
def step(log=None):
    t0 = time.perf_counter(); c.refresh(data); torch.cuda.synchronize(); t1 = time.perf_counter()
    ts = []
    for v in V:
        a = time.perf_counter()
        run(data, 100, v, SeedConfig(seed=2), max_iter=50, device=dev, corpus=c, n_total=data.n)
        ts.append((time.perf_counter() - a) * 1e3)
    if log is not None:
        log.append(((t1 - t0) * 1e3, ts))
for _ in range(3): step()
L = []
for _ in range(5): step(L)
for r, ts in L:
    print(f"refresh {r:.3f} ms  fits " + " ".join(f"{t:.3f}" for t in ts))
