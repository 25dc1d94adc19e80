"""Time one dense tcgen05 Lloyd pass (C5 shape) under experiment switches (SPKM_DN_DBG)."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2107_04074_b200 import synth, _lib
from paper_2107_04074_b200 import engine as E
from paper_2107_04074_b200.seeding import uniform_rows

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
data = synth.config_dataset("C5", n_override=n)
eng = E.Engine(data, 1000, "standard", use_graphs=False)
eng.seed_rows(data, uniform_rows(data.n, 1000, 2))
eng.reset()
eng.iteration(1)
torch.cuda.synchronize()
ev = lambda: torch.cuda.Event(enable_timing=True)
with torch.cuda.stream(eng.stream):
    eng.C.ctl.zero_()
    for _ in range(2):
        eng._dense(_lib.MODE_LLOYD)
    e0, e1 = ev(), ev()
    e0.record(eng.stream)
    for _ in range(5):
        eng.C.ctl.zero_()
        eng._dense(_lib.MODE_LLOYD)
    e1.record(eng.stream)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
fl = 6 * n * 1024 * 256
print(f"n={n} pass {ms:.3f} ms  {fl / ms / 1e9:.1f} TFLOP/s (3xTF32 MMA work)")
