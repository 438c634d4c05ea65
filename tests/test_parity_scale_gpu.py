"""GPU <-> oracle parity at the subset sizes SURVEY.md §8(d).3 names (the oracle timed beside the
GPU runs these same subsets): cfg3 base 0 over its full space (16,777,216 candidates, bit-exact),
cfg4 bases 0-15 x the first 2^16 samples (C20 float rules), cfg5 bases 0-15 x the first 2^12
samples per variant (int8 bit-exact, bf16 by C20).  Minutes of oracle time on the box's cores."""
import numpy as np
import pytest

import mlpv_inputs as M
from tests.parity import assert_fixed_parity, assert_float_parity, run_gpu

pytestmark = pytest.mark.gpu


# cfg5 bf16: open defect (DESIGN.md §6 "Open defect"): k_large's float path depends on launch timing, a
# base's verdict count can move by a few candidates between runs, which the C20 rules absorb in most
# runs but not in all (2 failures in 9 suite runs of round 2's last session) -- non-strict xfail
BF16_OPEN = pytest.mark.xfail(strict=False, reason="open defect: k_large float path not bit-reproducible under "
                              "irregular launch timing (DESIGN.md §6)")


@pytest.mark.parametrize("name,nb,end", [("cfg3", 1, 1 << 24), ("cfg4", 16, 1 << 16), ("cfg5_int8", 16, 1 << 12),
                                         pytest.param("cfg5_bf16", 16, 1 << 12, marks=BF16_OPEN)])
def test_survey_scale_subsets(oracle_mod, name, nb, end):
    import paper_1907_12933_b200 as P
    cfg = M.make_config(name).subset(n_base=nb, begin=0, end=end)
    g = run_gpu(P.Checker(cfg.net), cfg)
    o = oracle_mod.check(cfg)
    if cfg.net.numeric == M.NUM_BF16:
        assert_float_parity(g, o)
    else:
        assert_fixed_parity(g, o)
    print(f"{name}: {nb} x {end}: violated {int(o.violated.sum())}, coverage bits "
          f"{int(np.unpackbits(o.cov_all.view(np.uint8)).sum())}")
