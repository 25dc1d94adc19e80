"""Debug harness for the tcgen05 Gram: known centers -> raw split partials."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_2107_04074_b200 import engine as E, _lib

k, d = int(sys.argv[1]) if len(sys.argv) > 1 else 8, int(sys.argv[2]) if len(sys.argv) > 2 else 64
g = np.random.default_rng(0)
C = g.uniform(0.1, 1.0, (k, d))
C /= np.linalg.norm(C, axis=1, keepdims=True)
cs = E.CenterState(k, d, 100, torch.device("cuda"), True)
cs.load(C, E.ctypes_void(0))
cs.sinp.fill_(1.0)
torch.cuda.synchronize()
_lib.call("spkm_center_thresholds", cs.struct, cs.gram.data_ptr(), cs.tiles.data_ptr(), 1, E.ctypes_void(0))
torch.cuda.synchronize()
ds = cs.gram.numel() // (k * k)
G = cs.gram.view(ds, k, k).cpu().numpy()
ref = C @ C.T
iu = np.triu_indices(k)
print("dsplit", ds, "upper-triangle max abs err:", np.abs(G.sum(0)[iu] - ref[iu]).max())
print("split0 row0:", G[0, 0, :min(k, 8)])
print("ref row0  :", ref[0, :min(k, 8)])
ct = cs.ct32.view(d, cs.kp).cpu().numpy()[:, :k]
print("ct32 ok:", np.abs(ct - C.T).max())
