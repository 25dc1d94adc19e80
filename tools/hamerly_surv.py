"""Hamerly survivor counts per iteration (bounds survivors -> tighten survivors) on a bench config."""
import sys
sys.path.insert(0, ".")
from paper_2107_04074_b200 import synth, run, SeedConfig
cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
k = int(sys.argv[2]) if len(sys.argv) > 2 else 100
data = synth.config_dataset(cfg)
r = run(data, k, "hamerly", SeedConfig(seed=2), max_iter=50)
print(cfg, "n", data.n, [(s.iteration, s.survivors, s.survivors2) for s in r.iterations])
