"""GPU timeline of one bench step (5 fits, C2 k=100): busy vs idle and the largest gaps.

Uses torch.profiler (CUPTI) to list kernels and memcpys with device
timestamps, then reports where the GPU sits idle between them and which
host call was running.  Diagnostic only.
"""
import sys, time
sys.path.insert(0, ".")
import torch
from torch.profiler import profile, ProfilerActivity
from paper_2107_04074_b200 import synth, run, SeedConfig
from paper_2107_04074_b200.engine import device_corpus

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
k = int(sys.argv[2]) if len(sys.argv) > 2 else 100
data = synth.config_dataset(cfg)
dev = torch.device("cuda")
corpus = device_corpus(data, dev)
V = ("standard", "elkan", "simp_elkan", "hamerly", "simp_hamerly")


def step():
    for v in V:
        run(data, k, v, SeedConfig(seed=2), max_iter=50, device=dev, corpus=corpus)


for _ in range(3):
    step()
torch.cuda.synchronize()
t = time.perf_counter(); step(); torch.cuda.synchronize(); print("step ms (no profiler)", (time.perf_counter() - t) * 1e3)
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    step()
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
busy = sum(e.time_range.end - e.time_range.start for e in ev)
span = ev[-1].time_range.end - ev[0].time_range.start
print(f"device span {span/1e3:.2f} ms, busy {busy/1e3:.2f} ms ({busy/span:.1%}), kernels {len(ev)}")
gaps = []
for a, b in zip(ev, ev[1:]):
    g = b.time_range.start - a.time_range.end
    if g > 0:
        gaps.append((g, a.name[:40], b.name[:40]))
gaps.sort(reverse=True)
tot = sum(g for g, *_ in gaps)
print(f"idle total {tot/1e3:.2f} ms in {len(gaps)} gaps")
from collections import Counter
c = Counter()
cn = Counter()
for g, a, b in gaps:
    c[(a, b)] += g
    cn[(a, b)] += 1
for (a, b), g in c.most_common(25):
    print(f"{g/1e3:8.3f} ms  x{cn[(a, b)]:<4d} {a:40s} -> {b}")
