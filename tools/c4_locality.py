#!/usr/bin/env python3
"""C4 locality experiment (GPU): does grouping rows by cluster / planted topic
cut the center-row gather time of the full passes?

1. fit hamerly on C4 in the default row order (longest first) -> assignments;
2. replay the generator's RNG to recover each row's planted topic (synth.py:
   lognormal lengths, term permutation, topic sets, row topics -- in that order);
3. purity of the fitted clusters w.r.t. the planted topics;
4. for each device row order (length / cluster+length / topic+length) time
   `standard` for 4 iterations (iterations >= 2 are one full Lloyd pass each)
   and full hamerly + simp_elkan fits.
Prints one JSON line per measurement.  Tooling only (not product, not a test).
"""

import gc
import json
import math
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def planted_topics(spec, seed):
    g = np.random.Generator(np.random.PCG64(seed))
    mu = math.log(spec.mean_nnz) - spec.sigma ** 2 / 2.0
    g.lognormal(mu, spec.sigma, spec.n)
    g.permutation(spec.d)
    tsz = min(spec.topic_size, spec.d)
    for _ in range(spec.topics):
        g.choice(spec.d, tsz, replace=False)
    return g.integers(0, spec.topics, spec.n)


def main():
    import torch
    import paper_2107_04074_b200 as spk
    from paper_2107_04074_b200 import synth, engine
    cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
    k = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
    base = synth.config_dataset(cfg)
    spec = synth.CONFIGS[cfg]
    topic = planted_topics(spec, synth.DATA_SEED_BASE + int(cfg[1:]))

    def fresh(key):
        engine.clear_engine_cache()
        gc.collect()
        torch.cuda.empty_cache()
        ds = spk.Dataset(base.indptr, base.indices, base.data, base.dim)
        if key is not None:
            ds._row_key = key
        return ds

    def fit(ds, v, mi=50):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = spk.run(ds, k, v, spk.SeedConfig(seed=2), max_iter=mi)
        torch.cuda.synchronize()
        return r, time.perf_counter() - t0

    ds = fresh(None)
    fit(ds, "hamerly", 3)                       # warm (graphs, allocator)
    r, t = fit(ds, "hamerly")
    a = r.assignments
    # purity: share of each cluster's rows in its majority planted topic
    M = np.zeros((k, spec.topics), np.int64)
    np.add.at(M, (a, topic), 1)
    purity = M.max(1).sum() / a.size
    inv = M.max(0).sum() / a.size                # share of each topic's rows in its majority cluster
    print(json.dumps({"what": "purity", "cluster_purity": purity, "topic_concentration": inv,
                      "nonempty_clusters": int((M.sum(1) > 0).sum())}), flush=True)
    for name, key in (("length", None), ("cluster", a.astype(np.int64)), ("topic", topic.astype(np.int64))):
        ds = fresh(key)
        fit(ds, "standard", 2)
        r, t = fit(ds, "standard", 4)
        its = [s.elapsed_ns / 1e6 for s in r.iterations]
        out = {"what": "order", "order": name, "standard_iter_ms": its}
        for v in ("hamerly", "simp_elkan"):
            fit(ds, v, 2)
            rv, tv = fit(ds, v)
            out[v] = {"s": round(tv, 3), "iterations": len(rv.iterations), "objective": rv.objective,
                      "iter_ms": [round(s.elapsed_ns / 1e6, 2) for s in rv.iterations]}
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
