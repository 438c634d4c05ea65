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


BF16_OPEN = pytest.mark.xfail(strict=False, reason="open defect (DESIGN.md §6): k_large's float path depends on launch "
                              "timing; the first check of a fresh handle can differ from the back-to-back ones")


@pytest.mark.parametrize("name,nb,end,runs", [pytest.param("cfg5_bf16", 16, 1 << 12, 400, marks=BF16_OPEN),
                                              ("cfg5_int8", 16, 1 << 12, 200),
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


def _irregular_results(name, end, handles=12, runs=4):
    """Checks with irregular timing around them: fresh handles (allocation, weight upload, scratch
    memset before the first check) and host work between the checks."""
    import collections
    import paper_1907_12933_b200 as P
    cfg = M.make_config(name).subset(n_base=16, begin=0, end=end)
    sig = []
    for _ in range(handles):
        chk = P.Checker(cfg.net)
        for _ in range(runs):
            g = run_gpu(chk, cfg)
            sig.append(tuple(g[k].tobytes() for k in KEYS))
    return collections.Counter(sig)


@pytest.mark.parametrize("name,end", [("cfg4", 1 << 14), ("cfg3", 1 << 14), ("cfg5_int8", 1 << 12)])
def test_reproducible_under_irregular_timing(name, end):
    c = _irregular_results(name, end)
    assert len(c) == 1, f"{name}: {len(c)} distinct results over {sum(c.values())} checks"


@pytest.mark.xfail(strict=False, reason="open defect (DESIGN.md §6): k_large's float path depends on launch timing")
def test_cfg5_bf16_reproducible_under_irregular_timing():
    c = _irregular_results("cfg5_bf16", 1 << 12)
    assert len(c) == 1, f"cfg5_bf16: {len(c)} distinct results over {sum(c.values())} checks"
