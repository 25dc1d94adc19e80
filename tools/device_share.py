"""Device time inside fits (globaltimer stamps of the stats) vs wall time per bench step (C2 k=100)."""
import sys, time
sys.path.insert(0, ".")
import torch
from paper_2107_04074_b200 import synth, run, SeedConfig
from paper_2107_04074_b200.engine import device_corpus
cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
k = int(sys.argv[2]) if len(sys.argv) > 2 else 100
data = synth.config_dataset(cfg)
dev = torch.device("cuda")
corpus = device_corpus(data, dev)
V = ("standard", "elkan", "simp_elkan", "hamerly", "simp_hamerly")
def step():
    out = []
    for v in V:
        r = run(data, k, v, SeedConfig(seed=2), max_iter=50, device=dev, corpus=corpus)
        out.append((v, len(r.iterations), sum(s.elapsed_ns for s in r.iterations) / 1e3))
    return out
for _ in range(4): step()
torch.cuda.synchronize()
walls, devs = [], []
for _ in range(10):
    t = time.perf_counter(); o = step(); torch.cuda.synchronize(); walls.append((time.perf_counter() - t) * 1e6)
    devs.append(sum(x[2] for x in o))
print("per fit device us:", [(v, n, round(us)) for v, n, us in o])
import statistics as st
print(f"step wall {st.median(walls):.0f} us, device (iterations) {st.median(devs):.0f} us, share {st.median(devs) / st.median(walls):.3f}")
