"""Cost of DeviceCorpus.refresh (the e2e leg's per-step upload + device-side layout) on C2."""
import sys, time
sys.path.insert(0, ".")
import torch
from paper_2107_04074_b200 import synth
from paper_2107_04074_b200.engine import DeviceCorpus
data = synth.config_dataset(sys.argv[1] if len(sys.argv) > 1 else "C2")
dev = torch.device("cuda")
c = DeviceCorpus(data, dev, pinned_host=True)
c.seed_struct(data)
for _ in range(3):
    c.refresh(data)
torch.cuda.synchronize()
ts = []
for _ in range(10):
    t = time.perf_counter(); c.refresh(data); torch.cuda.synchronize(); ts.append((time.perf_counter() - t) * 1e3)
ts.sort()
print(f"refresh median {ts[5]:.3f} ms, h2d bytes {c.h2d_bytes}")
import cProfile, pstats
pr = cProfile.Profile(); pr.enable(); c.refresh(data); torch.cuda.synchronize(); pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(15)
# the raw uploads alone (same registered host arrays)
from paper_2107_04074_b200.engine import _host_registered
hs = [torch.from_numpy(_host_registered(a)) for a in (data.indptr, data.indices, data.data)]
print("pinned:", [h.is_pinned() for h in hs])
outs = [torch.empty_like(h, device=dev) for h in hs]
for _ in range(3):
    for o, h in zip(outs, hs): o.copy_(h, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    for o, h in zip(outs, hs): o.copy_(h, non_blocking=True)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
nb = sum(h.numel() * h.element_size() for h in hs)
print(f"raw H2D {ms:.3f} ms for {nb} B = {nb / ms / 1e6:.1f} GB/s")
