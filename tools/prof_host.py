"""Host-side profile of one bench step (5 fits on C2 k=100) with cProfile."""
import cProfile, pstats, sys, time
sys.path.insert(0, ".")
import torch
from paper_2107_04074_b200 import synth, run, SeedConfig
from paper_2107_04074_b200.engine import device_corpus
data = synth.config_dataset("C2")
dev = torch.device("cuda")
corpus = device_corpus(data, dev)
V = ("standard", "elkan", "simp_elkan", "hamerly", "simp_hamerly")
def step():
    for v in V:
        run(data, 100, v, SeedConfig(seed=2), max_iter=50, device=dev, corpus=corpus)
for _ in range(3): step()
torch.cuda.synchronize()
t = time.perf_counter(); step(); torch.cuda.synchronize(); print("step ms", (time.perf_counter() - t) * 1e3)
pr = cProfile.Profile(); pr.enable(); step(); torch.cuda.synchronize(); pr.disable()
pstats.Stats(pr).sort_stats(sys.argv[1] if len(sys.argv) > 1 else "cumulative").print_stats(45)
