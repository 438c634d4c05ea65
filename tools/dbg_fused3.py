import sys, numpy as np, torch
sys.path.insert(0, '.')
import mlpv_inputs as M, paper_1907_12933_b200 as P
from tests.parity import run_gpu
cfg = M.make_config("cfg4").subset(n_base=1, begin=0, end=256)
chk = P.Checker(cfg.net)
print("layout", chk.coverage_layout(cfg.cov)[0], flush=True)
g = run_gpu(chk, cfg)
print("ok", g["checked"], g["violated"], flush=True)
