"""Per-layer error of mlpv_eval potentials against the oracle (debug aid for the large kernels)."""
import sys, os
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import mlpv_inputs as M
import paper_1907_12933_b200 as P
from oracle import oracle as O
from tests.parity import to_device_bases

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
cfg = M.make_config(name)
chk = P.Checker(cfg.net)
bases = to_device_bases(cfg)
idx = [0, 1, 2, 3, 127, 128, 129, 255, 256, 1000, 2 ** 20 + 7]
for b in (0, 5):
    g = chk.eval(bases, b, cfg.pert, torch.tensor(np.asarray(idx, np.int64), device="cuda")).cpu().numpy().astype(np.float64)
    o = np.stack([np.concatenate(O.forward(cfg.net, O.decode(cfg.net.numeric, cfg.pert, cfg.bases[b], b, int(i)))) for i in idx])
    s = np.cumsum([0] + list(cfg.net.sizes[1:]))
    for l in range(len(s) - 1):
        e = np.abs(g[:, s[l]:s[l + 1]] - o[:, s[l]:s[l + 1]])
        print(f"base {b} layer {l + 1}: max abs err {e.max():.3e}  per-row max {np.round(e.max(1), 6).tolist()}")
    print("g logits row0", np.round(g[0, s[-2]:], 5).tolist())
    print("o logits row0", np.round(o[0, s[-2]:], 5).tolist())
