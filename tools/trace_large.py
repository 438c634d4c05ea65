"""Timeline of k_large (debug build with -DMLPV_TRACE): per-tile clock64 stamps of block 0 on cfg5.

    python tools/trace_large.py [cfg5_bf16|cfg5_int8] [samples_per_base]
"""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1907_12933_b200 import build as B  # noqa: E402

os.environ["MLPV_LIB"] = B.build(trace=True)
import torch  # noqa: E402

import mlpv_inputs as M  # noqa: E402
import paper_1907_12933_b200 as P  # noqa: E402

P.LIB_PATH = os.environ["MLPV_LIB"]
from tests.parity import to_device_bases  # noqa: E402

EV = ["top", "p0.start", "p0.issued", "p1.start", "p1.issued", "L2.accE", "L2.pfull", "L2.issued", "L3.accE",
      "L3.pfull", "L3.issued", "E1c0", "E1c1", "E1c2", "E1c3", "E2c0", "E2c1", "E3", "h1rdy", "h2rdy"]
name = sys.argv[1] if len(sys.argv) > 1 else "cfg5_bf16"
S = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
cfg = M.make_config(name).subset(begin=0, end=S)
chk = P.Checker(cfg.net)
bases = to_device_bases(cfg)
for _ in range(2):
    chk.check(bases, cfg.pert, cfg.prop, cfg.cov)
torch.cuda.synchronize()
buf = np.zeros((32, 24), np.uint64)
assert P.lib().mlpv_kl_trace_read(buf.ctypes.data_as(C.c_void_p)) == 0
t0 = int(buf[1, 0])
for tl in range(1, 6):
    row = [(EV[e], (int(buf[tl, e]) - t0) if buf[tl, e] else None) for e in range(len(EV))]
    row = [r for r in row]
    print(f"tile {tl}: " + "  ".join(f"{n}={v}" for n, v in sorted([r for r in row if r[1] is not None], key=lambda r: r[1])))
for tl in range(1, 4):
    print(f"tile {tl}: issuer waits (cycles) pair0 gfull {int(buf[tl, 20])} pfull {int(buf[tl, 21])}; pair1 gfull {int(buf[tl, 22])} pfull {int(buf[tl, 23])}")
per = [int(buf[tl + 1, 0]) - int(buf[tl, 0]) for tl in range(1, 10) if buf[tl + 1, 0]]
print("tile period (cycles):", per)

st = np.zeros((2, 2, 16, 4), np.uint64)
if hasattr(P.lib(), "mlpv_kl_step_read") and P.lib().mlpv_kl_step_read(st.ctypes.data_as(C.c_void_p)) == 0:
    for hh in range(2):
        for ch in range(2):
            t0s = int(st[hh, ch, 0, 0])
            if not t0s:
                continue
            steps = [(int(st[hh, ch, k, 0]) - t0s, int(st[hh, ch, k, 1]) - int(st[hh, ch, k, 0]),
                      int(st[hh, ch, k, 2]) - int(st[hh, ch, k, 1])) for k in range(16) if st[hh, ch, k, 0]]
            print(f"E1 tile 2 quad 0 half {hh} chunk {ch}: (start, ld, compute) per step {steps}; end {int(st[hh, ch, 15, 3]) - t0s}")

gn = np.zeros((2, 48, 4), np.uint64)
if hasattr(P.lib(), "mlpv_kl_gen_read") and P.lib().mlpv_kl_gen_read(gn.ctypes.data_as(C.c_void_p)) == 0:
    for g in range(2):
        ks = [k for k in range(48) if gn[g, k, 0]]
        if not ks:
            continue
        w = [int(gn[g, k, 1]) - int(gn[g, k, 0]) for k in ks]
        c = [int(gn[g, k, 2]) - int(gn[g, k, 1]) for k in ks]
        f = [int(gn[g, k, 3]) - int(gn[g, k, 2]) for k in ks]
        per = [int(gn[g, ks[i + 1], 0]) - int(gn[g, ks[i], 0]) for i in range(len(ks) - 1)]
        med = lambda x: sorted(x)[len(x) // 2]
        print(f"gen group {g} tile 2 pass 1: {len(ks)} stages; median wait {med(w)} compute {med(c)} fence+arrive {med(f)} stage-to-stage {med(per)}")
        print(f"   waits {w[:24]}")

wr = np.zeros((192, 4), np.uint64)
if hasattr(P.lib(), "mlpv_kl_w_read") and P.lib().mlpv_kl_w_read(wr.ctypes.data_as(C.c_void_p)) == 0:
    med = lambda x: sorted(x)[len(x) // 2] if x else None
    ok = [i for i in range(192) if all(wr[i, e] for e in range(4))]
    emp = [int(wr[i, 1]) - int(wr[i, 0]) for i in ok]
    lat = [int(wr[i, 3]) - int(wr[i, 1]) for i in ok]
    iw = [int(wr[i, 3]) - int(wr[i, 2]) for i in ok]
    ahead = [int(wr[i, 2]) - int(wr[i, 1]) for i in ok]
    print(f"W ring tile 2 (leader): {len(ok)} sub-stages; median producer empty-wait {med(emp)}, copy issue -> issuer sees full {med(lat)}, issuer wait {med(iw)}, copy issued before the issuer wanted it {med(ahead)}")
    print("   issue->full", lat[:40])
    print("   issuer wait", iw[:40])
