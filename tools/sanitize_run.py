"""One small check per config for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
    compute-sanitizer --tool memcheck python tools/sanitize_run.py cfg4
Parity against the oracle is the tests' job; this only drives the kernels on small slices."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import mlpv_inputs as M  # noqa: E402
import paper_1907_12933_b200 as P  # noqa: E402
from tests.parity import to_device_bases  # noqa: E402

SLICES = {"cfg1": (1, 0, 76_800), "cfg2": (2, 0, 20_000), "cfg3": (1, 0, 4096), "cfg4": (2, 0, 600),
          "cfg5_bf16": (1, 0, 300), "cfg5_int8": (1, 0, 300)}
for name in sys.argv[1:]:
    nb, b, e = SLICES[name]
    cfg = M.make_config(name).subset(n_base=nb, begin=b, end=e)
    chk = P.Checker(cfg.net)
    r = chk.check(to_device_bases(cfg), cfg.pert, cfg.prop, cfg.cov)
    chk.sync()
    torch.cuda.synchronize()
    print(name, "violated", r["violated"][:nb].tolist(), flush=True)
    chk.close()
