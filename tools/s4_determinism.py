"""Session 4: run-to-run determinism of a config's GPU result (every count, index and coverage word must
be bitwise identical from run to run) and parity with the oracle on the first run.
usage: MLPV_LIB=... python tools/s4_determinism.py CFG N_BASE END RUNS [oracle]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import mlpv_inputs as M
import paper_1907_12933_b200 as P
from tests.parity import run_gpu, assert_float_parity, assert_fixed_parity

name, nb, end, runs = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
cfg = M.make_config(name).subset(n_base=nb, begin=0, end=end)
chk = P.Checker(cfg.net)
ref = run_gpu(chk, cfg)
keys = ("checked", "violated", "flagged", "first_cex", "first_cex_unflagged", "cov_all", "cov_certain")
bad = 0
for i in range(1, runs):
    g = run_gpu(chk, cfg)
    d = [k for k in keys if not np.array_equal(g[k], ref[k])]
    if d:
        bad += 1
        det = {k: int(np.count_nonzero(g[k] != ref[k])) for k in d}
        print(f"run {i}: differs from run 0 in {det}", flush=True)
        for k in d:
            ix = np.nonzero(g[k] != ref[k])[0][:4]
            print("   ", k, [(int(j), hex(int(ref[k][j])), hex(int(g[k][j]))) for j in ix], flush=True)
print(f"{name} {nb} x {end} lib={os.environ.get('MLPV_LIB', 'default')}: {bad} of {runs - 1} runs differ from run 0")
if len(sys.argv) > 5:
    from oracle import oracle as O
    O.build_oracle()
    o = O.check(cfg)
    (assert_float_parity if cfg.net.numeric == M.NUM_BF16 else assert_fixed_parity)(ref, o)
    print("run 0 parity with the oracle: ok")
