"""Timeline of k_fused3 (debug build with -DMLPV_TRACE): per-tile clock64 stamps of cluster 0.

    python tools/trace_fused3.py [n_samples_per_base]      (MLPV_TRACE_CFG=cfg4_box: the unclamped box)
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

EV = {0: "iss.top", 1: "iss.kb0", 2: "iss.kblast", 3: "iss.h1rdy", 4: "iss.acc2free", 5: "iss.L2done",
      6: "gen.start", 7: "gen.end", 8: "epi.acc1", 9: "epi.E1done", 10: "epi.acc2", 11: "epi.E2done",
      12: "epi.acc3", 13: "epi.E3done", 14: "l3.first", 15: "l3.last", 29: "epi1.E1done", 30: "epi1.E2pieces",
      31: "prod.w0"}

S = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
cfg = M.make_config(os.environ.get("MLPV_TRACE_CFG", "cfg4"))
cfg = cfg.subset(n_base=cfg.n_base, begin=0, end=S)
chk = P.Checker(cfg.net)
bases = to_device_bases(cfg)
for _ in range(2):
    chk.check(bases, cfg.pert, cfg.prop, cfg.cov)
torch.cuda.synchronize()
buf = np.zeros((2, 64, 32), np.uint64)
assert P.lib().mlpv_f3_trace_read(buf.ctypes.data_as(C.c_void_p)) == 0
t0 = int(buf[0, 8, 0])
for rank in (0, 1):
    print(f"== rank {rank}")
    for tl in range(8, 14):
        row = buf[rank, tl].astype(np.int64)
        items = sorted(((int(row[e]) - t0, EV.get(e, f"g{e-16}")) for e in range(32) if row[e]), key=lambda x: x[0])
        print(f"tile {tl}: " + "  ".join(f"{n}={v}" for v, n in items))
r0 = buf[0].astype(np.int64)
per = np.diff(r0[8:60, 0])
print("issuer tile period (cycles): median", np.median(per), "min", per.min(), "max", per.max())
for name, a, b in (("L1 gen-wait span kb0->kblast", 1, 2), ("h1 wait after kblast", 2, 3), ("acc2free after h1", 3, 4),
                   ("E1 (acc1->E1done)", 8, 9), ("E2 (acc2->E2done)", 10, 11), ("E3 (acc3->E3done)", 12, 13),
                   ("gen tile", 6, 7)):
    d = r0[8:60, b] - r0[8:60, a]
    print(f"{name:32s} median {np.median(d):8.0f}  min {d.min():8d}  max {d.max():8d}")

g = np.zeros((2, 2, 4, 13, 5), np.uint64)
assert P.lib().mlpv_f3_trace_gen_read(g.ctypes.data_as(C.c_void_p)) == 0
g = g.astype(np.int64)
for rank in (0, 1):
    for grp in (0, 1):
        d = g[rank, grp]
        m = d[:, :, 0] != 0
        comp = (d[:, :, 1] - d[:, :, 0])[m]
        wait = (d[:, :, 2] - d[:, :, 1])[m]
        store = (d[:, :, 3] - d[:, :, 2])[m]
        arr = (d[:, :, 4] - d[:, :, 3])[m]
        print(f"gen rank {rank} grp {grp}: per-stage median compute {np.median(comp):.0f} wait {np.median(wait):.0f} "
              f"store+fence {np.median(store):.0f} arrive {np.median(arr):.0f}")
        row = d[1]
        print("   tile 9 stage starts", [int(x - row[0, 0]) if x else None for x in row[:, 0]])
        print("   tile 9 waits       ", [int(a - b) if a else None for a, b in zip(row[:, 2], row[:, 1])])

q = np.zeros((4, 13, 8), np.uint64)
assert P.lib().mlpv_f3_trace_iss_read(q.ctypes.data_as(C.c_void_p)) == 0
q = q.astype(np.int64)
thr = q[:, :, 1] - q[:, :, 0]     # stage top -> before the next-stage waits (2 MMAs issued)
gf = q[:, :, 2] - q[:, :, 1]
wf = q[:, :, 3] - q[:, :, 2]
print(f"issuer per-stage median: throttle wait {np.median(thr):.0f}  g_full wait {np.median(gf):.0f}  w_full wait {np.median(wf):.0f}")
print("  tile 9 throttle", thr[1].tolist())
print("  tile 9 g_full  ", gf[1].tolist())
print("  tile 9 w_full  ", wf[1].tolist())
print("  tile 9 stage-to-stage", np.diff(q[1, :, 0]).tolist())
for tt in range(4):
    row = []
    for kb in range(12):
        e = q[tt, kb]
        top = e[0]; nxt = q[tt, kb + 1, 0]
        w = (e[3] - e[1]) if (e[1] > top and e[3] > e[1] and e[1] < nxt) else 0
        row.append(f"{nxt - top}/{w}")
    print(f"  tile {8 + tt} stage-to-stage/blocking-wait: " + " ".join(row))
print("  tile 9 mma issue     ", (q[1, :, 4] - q[1, :, 3]).tolist())
print("  tile 9 serialized stage latency", (q[1, :, 7] - q[1, :, 6]).tolist())
print("  tile 9 commits       ", (q[1, :, 5] - q[1, :, 4]).tolist())
print("  tile 9 to next top   ", (q[1, 1:, 0] - q[1, :-1, 5]).tolist())

dn = np.zeros((4, 13), np.uint64)
assert P.lib().mlpv_f3_trace_done_read(dn.ctypes.data_as(C.c_void_p)) == 0
dn = dn.astype(np.int64)
print("stage completion - issue (tile 9):", (dn[1] - q[1, :, 3]).tolist())
print("completion intervals (tile 9):   ", np.diff(dn[1]).tolist())

ep = np.zeros((2, 4, 8), np.uint64)
assert P.lib().mlpv_f3_trace_epi_read(ep.ctypes.data_as(C.c_void_p)) == 0
ep = ep.astype(np.int64)
for team, nm in ((0, "E1"), (1, "E2")):
    for k in range(4):
        r = ep[team, k]
        print(f"{nm} tile {8 + k}: passA {r[1] - r[0]}  kb signals " + " ".join(str(r[2 + j] - r[0]) for j in range(4)))

e2 = np.zeros((2, 12, 2, 8), np.uint64)
assert P.lib().mlpv_f3_trace_e2_read(e2.ctypes.data_as(C.c_void_p)) == 0
e2 = e2.astype(np.int64)
t0 = {team: e2[0, 0, team, 0] for team in (0, 1)}
for team, nm in ((0, "E1"), (1, "E2")):
    print(f"{nm} tile 9 per warp (relative to rank 0 warp 0 start): start, signs, kb0..kb3 signals, end")
    for rk in range(2):
        for w in range(12):
            r = e2[rk, w, team]
            rel = lambda x: str(int(x - t0[team])) if x else "-"
            print(f"  rank {rk} warp {w}: start {rel(r[0])} signs {rel(r[1])} kb " + " ".join(rel(r[2 + j]) for j in range(4)) + f" end {rel(r[6])}")

gp = np.zeros((12, 8, 5), np.uint64)
assert P.lib().mlpv_f3_trace_grp_read(gp.ctypes.data_as(C.c_void_p)) == 0
gp = gp.astype(np.int64)
print("E2 pass B per group (rank 0, tile 9): stats / split / stores+signal / ld wait / to next top")
for w in range(8):
    row = []
    for i in range(8):
        e = gp[w, i]
        nxt = gp[w, i + 1, 0] if i < 7 else e[4]
        row.append(f"{e[1]-e[0]}/{e[2]-e[1]}/{e[3]-e[2]}/{e[4]-e[3]}/{nxt-e[4]}")
    print(f"  warp {w} (q{w & 3} h{w >> 2}): " + "  ".join(row))

e1 = np.zeros((2, 12, 5, 4), np.uint64)
assert P.lib().mlpv_f3_trace_e1p_read(e1.ctypes.data_as(C.c_void_p)) == 0
e1 = e1.astype(np.int64)
print("E1 per piece (tile 9): ld latency / compute / sign-off (st wait + fence + arrive) / gap to next piece")
for rk in range(2):
    for w in range(12):
        row = []
        for i in range(5):
            e = e1[rk, w, i]
            if not e[0]:
                continue
            nxt = e1[rk, w, i + 1, 0] if i < 4 and e1[rk, w, i + 1, 0] else e[3]
            row.append(f"{e[1]-e[0]}/{e[2]-e[1]}/{e[3]-e[2]}/{nxt-e[3]}")
        print(f"  rank {rk} warp {w}: " + "  ".join(row))
