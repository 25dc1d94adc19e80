#!/usr/bin/env python3
"""Workload for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
every variant on the C1 golden corpus (eager and graph paths), predict, k-means++
and AFK-MC2 seeding, the bound auditor, and a dense (tcgen05) fit on a small C5
subsample.  Small sizes: racecheck runs every shared-memory access through the
tool.  Run with PYTORCH_NO_CUDA_MEMORY_CACHING=1 so every tensor is its own
allocation and memcheck sees out-of-bounds accesses at tensor granularity.

usage: compute-sanitizer --tool memcheck python tools/sanitize_fits.py [quick]
"""

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def main():
    import torch
    import paper_2107_04074_b200 as spk
    from paper_2107_04074_b200 import synth, validation
    from conftest import golden_dataset, load_golden
    quick = len(sys.argv) > 1 and sys.argv[1] == "quick"
    data = golden_dataset(load_golden("C1"))
    k = 20
    for v in spk.VARIANTS:
        for g in ((False,) if quick else (False, True)):
            r = spk.run(data, k, v, spk.SeedConfig(seed=3), max_iter=12, use_graphs=g)
            r = spk.run(data, k, v, spk.SeedConfig(seed=3), max_iter=12, use_graphs=g)   # 2nd run: graph replay
            print(v, "graphs" if g else "eager", len(r.iterations), r.objective, flush=True)
    a, best, second = spk.assign_full(data, r.centers)
    spk.init_kmpp(data, k, alpha=1.0, seed=3, device="cuda:0")
    spk.init_afkmc2(data, k, alpha=1.0, chain_length=20, seed=3, device="cuda:0")
    rep = validation.audit_bounds(data, "elkan", k, 3, max_iter=6)
    print("audit", rep)
    dense = synth.config_dataset("C5", n_override=2048, cache_dir="")
    for v in ("standard", "hamerly"):
        r = spk.run(dense, 64, v, spk.SeedConfig(seed=5), max_iter=6)
        print("dense", v, len(r.iterations), r.objective, flush=True)
    torch.cuda.synchronize()
    print("sanitize workload done")


if __name__ == "__main__":
    main()
