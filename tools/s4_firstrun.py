"""Session 4: does the FIRST check of a fresh handle (fresh scratch / workspace, cold L2) differ from
the steady-state result?  usage: python tools/s4_firstrun.py CFG N_BASE END HANDLES [flush]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import mlpv_inputs as M
import paper_1907_12933_b200 as P
from tests.parity import run_gpu

name, nb, end, n = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
flush = len(sys.argv) > 5
cfg = M.make_config(name).subset(n_base=nb, begin=0, end=end)
keys = ("checked", "violated", "flagged", "first_cex", "first_cex_unflagged", "cov_all", "cov_certain")
chk0 = P.Checker(cfg.net)
run_gpu(chk0, cfg)
ref = run_gpu(chk0, cfg)                      # steady state of a warmed handle
buf = torch.empty(512 << 20, dtype=torch.uint8, device="cuda") if flush else None
bad1 = bad2 = 0
for i in range(n):
    chk = P.Checker(cfg.net)
    if flush:
        buf.fill_(i & 0xFF)
        torch.cuda.synchronize()
    g1 = run_gpu(chk, cfg)
    g2 = run_gpu(chk, cfg)
    d1 = [k for k in keys if not np.array_equal(g1[k], ref[k])]
    d2 = [k for k in keys if not np.array_equal(g2[k], ref[k])]
    if d1:
        bad1 += 1
        k = d1[0]; ix = np.nonzero(g1[k] != ref[k])[0][:3]
        print(f"handle {i}: first run differs in {d1}: {k} {[(int(j), hex(int(ref[k][j])), hex(int(g1[k][j]))) for j in ix]}", flush=True)
    if d2:
        bad2 += 1
    del chk
print(f"{name} {nb} x {end} flush={flush}: first runs differing {bad1} / {n}, second runs differing {bad2} / {n}")
