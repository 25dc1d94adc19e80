"""Seeded synthetic corpora with the BASELINE.json shapes.

The paper's corpora (DBLP, Simpsons, 20news, RCV-1) are
not available, and the reference's own ``datagen.py`` does not implement
the BASELINE generator, so this module writes it.  All draws come from
``numpy.random.Generator(PCG64(seed))``; a (config, seed) pair pins the
bytes on any machine.

Sparse rows (configs C1-C4):
  * row length m_i = clip(round(LogNormal(mu, 0.8)), 5, 400),
    mu = ln(mean) - 0.8^2/2 (so E[m] ~ mean before clipping);
  * term ids: bounded Zipf(s=1.1) over ranks 1..d (alias-table draws),
    mapped through a seeded permutation of [0, d); draws with replacement
    until m_i distinct ids (first m_i distinct in draw order);
  * topic configs: each draw comes with probability 0.7 uniformly from the
    row's topic set (topic uniform per row; each set = 2,000 ids drawn
    without replacement from [0, d)), otherwise from the global Zipf;
  * tf ~ Poisson(1) + 1, idf = ln(n / df) (the reference's default TF-IDF,
    corpus_io.py:110-111); zero weights (df = n) are dropped and rows left
    empty are removed (only possible at toy sizes);
  * rows L2-normalised in float64 by ``Dataset.from_csr``.
Dense rows (config C5): unit centers + N(0, sigma^2 I) noise, renormalised.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .sparse import Dataset

DATA_SEED_BASE = 2107_04074


@dataclass(frozen=True)
class CorpusSpec:
    name: str
    n: int
    d: int
    mean_nnz: float
    topics: int = 0
    topic_size: int = 2000
    topic_frac: float = 0.7
    zipf_s: float = 1.1
    sigma: float = 0.8
    min_nnz: int = 5
    max_nnz: int = 400


# BASELINE.json configs (C5 is dense, see dense_corpus)
CONFIGS = {
    "C1": CorpusSpec("C1", 2_000, 5_000, 50),
    "C2": CorpusSpec("C2", 20_000, 100_000, 120),
    "C3": CorpusSpec("C3", 500_000, 250_000, 80, topics=200),
    "C4": CorpusSpec("C4", 4_000_000, 1_000_000, 60, topics=1000),
}


def _alias_table(p: np.ndarray):
    """Walker alias table for O(1) draws from a discrete distribution."""
    n = p.size
    q = p * n
    alias = np.zeros(n, np.int64)
    prob = np.zeros(n)
    small = list(np.nonzero(q < 1.0)[0])
    large = list(np.nonzero(q >= 1.0)[0])
    q = q.copy()
    while small and large:
        s = small.pop()
        g = large.pop()
        prob[s] = q[s]
        alias[s] = g
        q[g] = (q[g] + q[s]) - 1.0
        (small if q[g] < 1.0 else large).append(g)
    for g in large:
        prob[g] = 1.0
    for s in small:
        prob[s] = 1.0
    return prob, alias


def _zipf_sampler(d: int, s: float):
    w = np.arange(1, d + 1, dtype=np.float64) ** (-s)
    return _alias_table(w / w.sum())


def _first_distinct(rows_local, terms, m, nrows):
    """Keep, per row, the first m[row] distinct terms in draw order.

    rows_local/terms are in draw order.  Returns (rows, terms) kept and the
    per-row count kept.
    """
    d_key = np.int64(terms.max() + 1 if terms.size else 1)
    keys = rows_local.astype(np.int64) * d_key + terms
    _, first = np.unique(keys, return_index=True)       # earliest draw per key
    first.sort()                                          # back to draw order
    r = rows_local[first]
    t = terms[first]
    # rank within row in draw order
    order = np.argsort(r, kind="stable")
    r_sorted = r[order]
    starts = np.searchsorted(r_sorted, np.arange(nrows))
    rank = np.empty(r.size, np.int64)
    rank[order] = np.arange(r.size) - starts[r_sorted]
    keep = rank < m[r]
    r, t = r[keep], t[keep]
    cnt = np.bincount(r, minlength=nrows)
    return r, t, cnt


def sparse_corpus(spec: CorpusSpec, seed: int | None = None, chunk_rows: int = 1 << 18,
                  return_raw: bool = False, row_norms=None):
    """Generate the corpus of ``spec``; returns a normalised ``Dataset``.

    With ``return_raw`` returns (indptr, indices, weights) before
    normalisation instead (used to feed the reference's own
    ``Dataset.from_rows`` when pinning golden vectors).
    """
    seed = DATA_SEED_BASE if seed is None else seed
    g = np.random.Generator(np.random.PCG64(seed))
    n, d = spec.n, spec.d
    mu = math.log(spec.mean_nnz) - spec.sigma ** 2 / 2.0
    m = np.clip(np.rint(g.lognormal(mu, spec.sigma, n)), spec.min_nnz, spec.max_nnz).astype(np.int64)
    if spec.topics:
        m = np.minimum(m, d)
    else:
        m = np.minimum(m, d)
    perm = g.permutation(d).astype(np.int64)
    prob, alias = _zipf_sampler(d, spec.zipf_s)
    if spec.topics:
        tsz = min(spec.topic_size, d)
        topic_sets = np.stack([g.choice(d, tsz, replace=False) for _ in range(spec.topics)]).astype(np.int64)
        row_topic = g.integers(0, spec.topics, n)
    row_parts, term_parts = [], []
    for c0 in range(0, n, chunk_rows):
        c1 = min(n, c0 + chunk_rows)
        nr = c1 - c0
        mc = m[c0:c1]
        have_r = np.empty(0, np.int64)
        have_t = np.empty(0, np.int64)
        cnt = np.zeros(nr, np.int64)
        for _attempt in range(64):
            need = mc - cnt
            if not need.any():
                break
            want = np.where(need > 0, np.ceil(need * 1.3).astype(np.int64) + 4, 0)
            rr = np.repeat(np.arange(nr), want)
            u = g.random(rr.size)
            col = np.minimum((u * d).astype(np.int64), d - 1)
            acc = g.random(rr.size) < prob[col]
            rank = np.where(acc, col, alias[col])
            tt = perm[rank]
            if spec.topics:
                from_topic = g.random(rr.size) < spec.topic_frac
                pick = g.integers(0, topic_sets.shape[1], rr.size)
                tt = np.where(from_topic, topic_sets[row_topic[c0 + rr], pick], tt)
            have_r, have_t, cnt = _first_distinct(
                np.concatenate([have_r, rr]), np.concatenate([have_t, tt]), mc, nr)
        # sort terms within each row
        key = have_r * np.int64(d) + have_t
        key.sort()
        row_parts.append(key // d + c0)
        term_parts.append(key % d)
    rows = np.concatenate(row_parts)
    terms = np.concatenate(term_parts)
    tf = g.poisson(1.0, terms.size).astype(np.float64) + 1.0
    df = np.bincount(terms, minlength=d)
    idf = np.log(n / np.maximum(df, 1))
    w = tf * idf[terms]
    keep = w != 0.0
    rows, terms, w = rows[keep], terms[keep], w[keep]
    counts = np.bincount(rows, minlength=n)
    nonempty = counts > 0
    if not nonempty.all():       # only possible at toy sizes (a term in every row)
        remap = np.cumsum(nonempty) - 1
        rows = remap[rows]
        counts = counts[nonempty]
    indptr = np.zeros(counts.size + 1, np.int64)
    np.cumsum(counts, out=indptr[1:])
    if return_raw:
        return indptr, terms.astype(np.int32), w
    return Dataset.from_csr(indptr, terms, w, d, normalize_rows=True, check_sorted=False, row_norms=row_norms)


def dense_corpus(n: int, d: int = 256, centers: int = 1000, sigma_total: float = 0.3,
                 seed: int | None = None):
    """C5: unit vectors around ``centers`` random unit directions.

    Noise is N(0, (sigma_total^2/d) I), i.e. the *total* noise norm is
    ~sigma_total (SURVEY.md §7 hard part 8 discusses the per-coordinate
    reading, which buries the clusters).  Returns (X float32 [n, d], labels).
    """
    seed = DATA_SEED_BASE + 5 if seed is None else seed
    g = np.random.Generator(np.random.PCG64(seed))
    C = g.standard_normal((centers, d))
    C /= np.linalg.norm(C, axis=1, keepdims=True)
    lab = g.integers(0, centers, n)
    X = np.empty((n, d), np.float32)
    step = 1 << 20
    for s in range(0, n, step):
        e = min(n, s + step)
        x = C[lab[s:e]] + g.standard_normal((e - s, d)) * (sigma_total / math.sqrt(d))
        x /= np.linalg.norm(x, axis=1, keepdims=True)
        X[s:e] = x
    return X, lab


# C5: n=10M dense unit vectors, d=256, 1,000 generating centers, noise of
# total norm 0.3 (sigma = 0.3 / sqrt(256) per coordinate; see dense_corpus)
C5 = dict(n=10_000_000, d=256, centers=1000, sigma_total=0.3)


def config_dataset(name: str, seed: int | None = None, n_override: int | None = None,
                   cache_dir: str | None = None, row_norms=None) -> Dataset:
    """The Dataset of BASELINE config ``name`` (optionally its first-``n_override``-rows variant:
    the same generator with n = n_override).  ``row_norms`` overrides the
    row-norm helper of ``Dataset.from_csr`` (bench.py's reference arm passes
    the oracle's, so that process never loads the product library).

    ``cache_dir`` (default: $SPKM_DATA_CACHE, unset = no cache) keeps the
    normalised CSR as .npy files keyed by (config, seed, n) so repeated runs
    in one session skip the generator (C4 takes minutes on the host).  The
    cache only stores this function's own output; nothing is read from it
    that the generator did not write.
    """
    import os
    cache_dir = cache_dir if cache_dir is not None else os.environ.get("SPKM_DATA_CACHE")
    if cache_dir:
        from pathlib import Path
        key = f"{name}_s{seed}_n{n_override}"
        base = Path(cache_dir) / key
        files = [base.with_name(key + f".{part}.npy") for part in ("indptr", "indices", "data", "meta")]
        if all(f.exists() for f in files):
            ip, ix, dv, meta = (np.load(f, mmap_mode=None) for f in files)
            ds = Dataset(ip, ix, dv, int(meta[0]))
            if int(meta[1]) > 0:
                ds.dense_dim = int(meta[1])
                ds._values32 = ds.data.astype(np.float32)     # as Dataset.dense keeps it
            return ds
        ds = config_dataset(name, seed, n_override, cache_dir="", row_norms=row_norms)
        base.parent.mkdir(parents=True, exist_ok=True)
        for f, arr in zip(files, (ds.indptr, ds.indices, ds.data,
                                  np.array([ds.dim, getattr(ds, "dense_dim", 0) or 0], np.int64))):
            tmp = f.with_name(f.name + ".tmp.npy")
            np.save(tmp, arr)
            os.replace(tmp, f)
        return ds
    if name == "C5":
        n = n_override if n_override is not None else C5["n"]
        X, _ = dense_corpus(n, C5["d"], C5["centers"], C5["sigma_total"],
                            seed=DATA_SEED_BASE + 5 if seed is None else seed)
        return Dataset.dense(X)
    spec = CONFIGS[name]
    if n_override is not None:
        spec = CorpusSpec(spec.name + f"[n={n_override}]", n_override, spec.d, spec.mean_nnz,
                          spec.topics, spec.topic_size, spec.topic_frac)
    base = DATA_SEED_BASE + int(name[1:])
    return sparse_corpus(spec, base if seed is None else seed, row_norms=row_norms)
