"""Session 4: which layer's potentials differ between irregularly timed runs of cfg5 bf16?
mlpv_eval of base 8's first 4096 candidates on fresh handles; per layer, the number of potentials that
differ (bitwise) from the first handle's first run, and their largest absolute difference."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import mlpv_inputs as M
import paper_1907_12933_b200 as P
from tests.parity import to_device_bases
cfg = M.make_config("cfg5_bf16").subset(n_base=16, begin=0, end=4096)
bases = to_device_bases(cfg)
idx = torch.arange(4096, dtype=torch.int64, device="cuda")
sizes = cfg.net.sizes[1:]
offs = np.concatenate([[0], np.cumsum(sizes)])
ref = None
for i in range(30):
    chk = P.Checker(cfg.net)
    for r in range(3):
        out = chk.eval(bases, 8, cfg.pert, idx); chk.sync()
        o = out.cpu().numpy()
        if ref is None:
            ref = o.copy(); continue
        if not np.array_equal(o.view(np.uint32), ref.view(np.uint32)):
            msg = []
            for l in range(len(sizes)):
                a, b = o[:, offs[l]:offs[l + 1]], ref[:, offs[l]:offs[l + 1]]
                d = a.view(np.uint32) != b.view(np.uint32)
                rows = np.nonzero(d.any(axis=1))[0]
                msg.append(f"L{l + 1}: {int(d.sum())} elems in {len(rows)} rows (first rows {rows[:6].tolist()}, cols {np.nonzero(d.any(axis=0))[0][:6].tolist()}), max |diff| {float(np.abs(a - b).max()):.3g}")
            print(f"handle {i} run {r}: " + "; ".join(msg), flush=True)
print("done")
