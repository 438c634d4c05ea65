"""Session 4: run-to-run determinism of mlpv_eval (every layer's potentials of a list of candidates,
bitwise) on the tensor-core paths, and of a check with a restriction.
usage: python tools/s4_determinism_eval.py CFG RUNS"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import mlpv_inputs as M
import paper_1907_12933_b200 as P
from tests.parity import to_device_bases

name, runs = sys.argv[1], int(sys.argv[2])
cfg = M.make_config(name).subset(n_base=4, begin=0, end=1 << 12)
chk = P.Checker(cfg.net)
bases = to_device_bases(cfg)
rng = np.random.default_rng(7)
idx = torch.from_numpy(np.sort(rng.choice(1 << 12, size=700, replace=False)).astype(np.int64)).cuda()
bad = 0
ref = None
for i in range(runs):
    out = chk.eval(bases, i % 4 if ref is None else 1, cfg.pert, idx)
    chk.sync()
    o = out.cpu().numpy().view(np.uint32).copy()
    if i == 0:
        out = chk.eval(bases, 1, cfg.pert, idx); chk.sync()
        ref = out.cpu().numpy().view(np.uint32).copy()
        continue
    if not np.array_equal(o, ref):
        bad += 1
        d = np.nonzero(o != ref)
        print(f"run {i}: {len(d[0])} words differ, rows {sorted(set(d[0].tolist()))[:8]} cols {sorted(set(d[1].tolist()))[:8]}", flush=True)
print(f"{name} eval 700 candidates: {bad} of {runs - 1} runs differ")
