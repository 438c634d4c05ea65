"""Debug helper: one k_large check on a cfg5 subset (pair with MLPV_WAIT_TIMEOUT builds to locate a
lost mbarrier arrive).  usage: python tools/dbg_large.py cfg5_bf16 N_BASE N_SAMPLES"""
import sys, os
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import mlpv_inputs as M
import paper_1907_12933_b200 as P
from tests.parity import run_gpu
cfg = M.make_config(sys.argv[1]).subset(n_base=int(sys.argv[2]), begin=0, end=int(sys.argv[3]))
chk = P.Checker(cfg.net)
r = run_gpu(chk, cfg)
torch.cuda.synchronize()
print("ok", int(r["checked"].sum()))
