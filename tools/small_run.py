"""A few checks of one config on a subset, for profilers (ncu) that replay every kernel:
    python tools/small_run.py cfg3 N_BASE RANGE_END REPS"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import mlpv_inputs as M  # noqa: E402
import paper_1907_12933_b200 as P  # noqa: E402
from tests.parity import to_device_bases  # noqa: E402

name, nb, end, reps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
cfg = M.make_config(name).subset(n_base=nb, begin=0, end=end)
chk = P.Checker(cfg.net)
bases = to_device_bases(cfg)
for _ in range(reps):
    r = chk.check(bases, cfg.pert, cfg.prop, cfg.cov)
chk.sync()
torch.cuda.synchronize()
print(name, "violated", r["violated"][:nb].sum().item())
