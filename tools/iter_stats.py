#!/usr/bin/env python3
"""Per-iteration counters of one fit (survivors, heavy rows, similarities, moves, touched clusters)."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", default="C4")
    p.add_argument("--k", type=int, default=None)
    p.add_argument("--variant", default="simp_elkan")
    p.add_argument("--seed", type=int, default=2)
    p.add_argument("--max-iter", type=int, default=50)
    a = p.parse_args()
    import paper_2107_04074_b200 as spk
    from paper_2107_04074_b200 import synth
    data = synth.config_dataset(a.config)
    k = a.k or {"C1": 20, "C2": 100, "C3": 200, "C4": 1000}[a.config]
    r = spk.run(data, k, a.variant, spk.SeedConfig(seed=a.seed), max_iter=a.max_iter)
    print(f"# {a.config} k={k} {a.variant}: n={data.n} iterations={len(r.iterations)} objective={r.objective:.6f}")
    print("it  light_rows  heavy_rows  sims/n  moves  touched  ms")
    for i, s in enumerate(r.iterations, 1):
        print(f"{i:2d} {s.survivors:10d} {s.survivors2:10d} {s.sim_count / data.n:8.1f} {s.reassignments:8d} "
              f"{getattr(s, 'touched', 0):6d} {s.elapsed_ns / 1e6:8.2f}")


if __name__ == "__main__":
    main()
