"""Center sparsity of the term-major copy after a few iterations (for the sparse-center design)."""
import sys
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2107_04074_b200 import synth, engine as E
cfg, k, its = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
data = synth.config_dataset(cfg)
eng = E.Engine(data, k, "hamerly", use_graphs=False)
from paper_2107_04074_b200.seeding import uniform_rows
eng.seed_rows(data, uniform_rows(data.n, k, 2))
eng.reset()
for it in range(1, its + 1):
    eng.iteration(it)
torch.cuda.synchronize()
ct = eng.C.ct32.view(data.dim, eng.C.kp)[:, :k]
nz = (ct != 0).sum(dim=1).double().cpu().numpy()
df = np.bincount(data.indices, minlength=data.dim).astype(np.float64)[eng.corpus.order]
w = df / df.sum()
print(cfg, "k", k, "after", its, "its: center density", float((nz.sum()) / (k * data.dim)),
      "nnz-weighted nz/k", float((w * nz).sum() / k))
for thr in (0.05, 0.1, 0.25, 0.5):
    dense_rows = nz > thr * k
    cost = (w * np.where(dense_rows, 4 * k, 8 * nz)).sum()
    print(f"  hybrid (dense if nz > {thr}k): bytes/nnz {cost:.0f} vs dense {4*k}; dense-row frac of nnz {w[dense_rows].sum():.3f}")
# 32-center lines (128 B of a term row): share of (nnz, line) gathers that hit an all-zero line
ctl = eng.C.ct32.view(data.dim, eng.C.kp)
for width in (32, 8):
    kq = (ctl.shape[1] + width - 1) // width * width
    padded = torch.nn.functional.pad(ctl, (0, kq - ctl.shape[1]))
    lines = (padded.view(data.dim, -1, width) != 0).any(dim=2).double().cpu().numpy()   # [d, kq/width]
    live = (w[:, None] * lines).sum() / lines.shape[1]
    print(f"  {width}-center blocks: nnz-weighted live fraction {live:.3f}")
# per-cluster blocks of consecutive terms (device term order): share of (cluster, block) holding a nonzero
c64 = eng.C.cent64.view(k, data.dim)
for tb in (32, 64, 256):
    dq = (data.dim + tb - 1) // tb * tb
    pc = torch.nn.functional.pad(c64, (0, dq - data.dim))
    live = (pc.view(k, -1, tb) != 0).any(dim=2).double().mean().item()
    print(f"  cluster x {tb}-term blocks live: {live:.3f}")
# split by the gathers' L2 head (term rows [0, hot) kept in L2 by the eviction hints)
hot = min(data.dim, (64 << 20) // (eng.C.kp * 4))
wc = w.copy(); wc[:hot] = 0
print(f"  head rows [0,{hot}) carry {w[:hot].sum():.3f} of the nnz")
for width in (32, 16, 8, 4):
    kq = (ctl.shape[1] + width - 1) // width * width
    padded = torch.nn.functional.pad(ctl, (0, kq - ctl.shape[1]))
    lines = (padded.view(data.dim, -1, width) != 0).any(dim=2).double().cpu().numpy()
    live = (wc[:, None] * lines).sum() / lines.shape[1] / max(wc.sum(), 1e-30)
    print(f"  cold rows, {width}-center blocks: nnz-weighted live fraction {live:.3f}")
nzc = (wc * nz).sum() / max(wc.sum(), 1e-30) / k
print(f"  cold rows: nnz-weighted nonzero fraction {nzc:.3f} (bitmap+packed bytes/nnz {k/8 + 4*nzc*k:.0f} vs dense {4*k})")
