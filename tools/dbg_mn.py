import sys
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_2107_04074_b200 import engine as E, _lib
np.set_printoptions(linewidth=200, precision=3, suppress=True)
def go(k, d, C):
    cs = E.CenterState(k, d, 100, torch.device("cuda"), True)
    cs.load(C, E.ctypes_void(0))
    cs.sinp.fill_(1.0)
    torch.cuda.synchronize()
    _lib.call("spkm_center_thresholds", cs.struct, cs.gram.data_ptr(), cs.tiles.data_ptr(), 1, E.ctypes_void(0))
    torch.cuda.synchronize()
    ds = cs.gram.numel() // (k * k)
    G = cs.gram.view(ds, k, k).cpu().numpy().sum(0)
    return G
k, d = 8, 32
C = np.zeros((k, d)); 
for i in range(k): C[i, i] = 1.0
G = go(k, d, C); print("onehot k8 d32\n", G)
C = np.zeros((k, d))
for i in range(k): C[i, 3 * i + 1] = 1.0; C[i, 0] = 0.5
G = go(k, d, C); print("shared term0 k8\n", G)
k = 40
C = np.zeros((k, d))
for i in range(k): C[i, i % d] = 1.0
G = go(k, d, C); print("onehot k40 nonzero pattern rows 0..40:")
for i in range(k): print(i, np.nonzero(np.abs(G[i]) > 1e-3)[0].tolist())
g = np.random.default_rng(0); C = g.uniform(0.1, 1, (20, 100)); C /= np.linalg.norm(C, axis=1, keepdims=True)
G = go(20, 100, C); print("random err", np.abs(np.triu(G - C @ C.T)).max())
