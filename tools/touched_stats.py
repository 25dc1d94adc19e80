import sys; sys.path.insert(0, ".")
import torch
from paper_2107_04074_b200 import synth, run, SeedConfig
data = synth.config_dataset("C2")
for v in ("standard", "elkan", "hamerly"):
    r = run(data, 100, v, SeedConfig(seed=2), max_iter=50)
    print(v, [(s.touched, s.reassignments, s.nnz_moved) for s in r.iterations])
