"""Session 4: fraction of irregularly timed cfg5-bf16 checks (fresh handles, 5 runs each, host work
between the runs) whose result differs from the canonical one (the mode of all runs)."""
import sys, os, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import mlpv_inputs as M
import paper_1907_12933_b200 as P
from tests.parity import run_gpu
name = sys.argv[1] if len(sys.argv) > 1 else "cfg5_bf16"
cfg = M.make_config(name).subset(n_base=16, begin=0, end=int(sys.argv[2]) if len(sys.argv) > 2 else 4096)
sig = []
for i in range(40):
    chk = P.Checker(cfg.net)
    for r in range(5):
        g = run_gpu(chk, cfg)
        sig.append(hash((g["violated"].tobytes(), g["flagged"].tobytes(), g["cov_all"].tobytes())))
        print("", end="", flush=True)
c = collections.Counter(sig)
print(f"{name} lib={os.path.basename(os.environ.get('MLPV_LIB', 'libmlpv.so'))}: {len(sig) - c.most_common(1)[0][1]} of {len(sig)} runs differ from the most common result ({len(c)} distinct results)")
