"""Run-to-run determinism of the tensor-core paths: every count, counterexample index and coverage
word of a check is bitwise identical from run to run.  (Session 4 found k_large's activation scratch
handed to the producer's bulk copies behind a CTA-scope fence: ~1 % of cfg5-bf16 runs differed in a
verdict count or a coverage bit; the hand-off now fences at device scope.)"""
import numpy as np
import pytest

import mlpv_inputs as M
from tests.parity import run_gpu

pytestmark = pytest.mark.gpu

KEYS = ("checked", "violated", "flagged", "first_cex", "first_cex_unflagged", "cov_all", "cov_certain")


@pytest.mark.parametrize("name,nb,end,runs", [("cfg5_bf16", 16, 1 << 12, 400), ("cfg5_int8", 16, 1 << 12, 200),
                                              ("cfg4", 16, 1 << 14, 100), ("cfg3", 4, 1 << 16, 50)])
def test_run_to_run_determinism(name, nb, end, runs):
    import paper_1907_12933_b200 as P
    cfg = M.make_config(name).subset(n_base=nb, begin=0, end=end)
    chk = P.Checker(cfg.net)
    ref = run_gpu(chk, cfg)
    for i in range(1, runs):
        g = run_gpu(chk, cfg)
        diff = {k: int(np.count_nonzero(g[k] != ref[k])) for k in KEYS if not np.array_equal(g[k], ref[k])}
        assert not diff, f"{name}: run {i} differs from run 0 in {diff}"
