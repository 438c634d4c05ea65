"""Session 4: violated[8] / violated[11] of runs 0..4 of fresh cfg5-bf16 handles (canonical 0x8e5 / 0x59)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import mlpv_inputs as M
import paper_1907_12933_b200 as P
from tests.parity import run_gpu
mode = sys.argv[1]
cfg = M.make_config("cfg5_bf16").subset(n_base=16, begin=0, end=4096)
buf = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
keep = []
for i in range(14):
    chk = P.Checker(cfg.net)
    if mode in ("sync", "flush"):
        torch.cuda.synchronize()
    if mode == "flush":
        buf.fill_(i); torch.cuda.synchronize()
    if mode == "keep":
        keep.append(chk)
    vals = []
    for r in range(5):
        g = run_gpu(chk, cfg)
        vals.append((hex(int(g["violated"][8])), hex(int(g["violated"][11])), int(g["flagged"].sum())))
    print(mode, i, vals, flush=True)
