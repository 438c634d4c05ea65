"""GPU <-> oracle parity of the tcgen05 large-net path (Philox lattice spaces, configs 4 and 5)."""
import numpy as np
import pytest

import mlpv_inputs as M
from tests.parity import (UMAX, assert_fixed_parity, assert_float_parity, assert_logits_close, run_gpu,
                          to_device_bases)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch
    assert torch.cuda.is_available()
    from paper_1907_12933_b200 import build
    build.build()
    import paper_1907_12933_b200 as P
    return P


_CHK = {}


def _checker(P, name):
    if name not in _CHK:
        _CHK[name] = P.Checker(M.make_config(name).net)
    return _CHK[name]


def _eval(P, chk, cfg, b, idx, oracle_mod):
    import torch
    bases = to_device_bases(cfg)
    g = chk.eval(bases, b, cfg.pert, torch.tensor(np.asarray(idx, np.int64), device="cuda")).cpu().numpy()
    o = np.stack([np.concatenate(oracle_mod.forward(cfg.net, oracle_mod.decode(cfg.net.numeric, cfg.pert, cfg.bases[b], b, int(i))))
                  for i in idx])
    return g, o


def test_cfg4_ranges(P, oracle_mod):
    cfg = M.make_config("cfg4")
    chk = _checker(P, "cfg4")
    for s in (cfg.subset(n_base=16, begin=0, end=1000),                       # 8 tiles, ragged tail of 104
              cfg.subset(n_base=3, base_start=997, begin=2 ** 32 - 300, end=2 ** 32),   # top of the index space
              cfg.subset(n_base=5, base_start=400, begin=12345, end=12346)):   # single candidate
        o = oracle_mod.check(s)
        g = run_gpu(chk, s)
        assert_float_parity(g, o)


def test_cfg4_logits(P, oracle_mod):
    cfg = M.make_config("cfg4")
    chk = _checker(P, "cfg4")
    rng = np.random.default_rng(4)
    idx = [0, 1, 127, 128, 2 ** 32 - 1] + list(rng.integers(0, 2 ** 32, 250))
    for b in (0, 999):
        g, o = _eval(P, chk, cfg, b, idx, oracle_mod)
        T = g.shape[1]
        err = assert_logits_close(g[:, T - 10:], o[:, T - 10:])
        print(f"cfg4 base {b}: max logit err {err:.3e}")
        assert np.allclose(g, o, rtol=1e-5, atol=2e-5)          # hidden potentials too


def test_cfg5_bf16(P, oracle_mod):
    cfg = M.make_config("cfg5_bf16")
    chk = _checker(P, "cfg5_bf16")
    s = cfg.subset(n_base=4, begin=0, end=300)
    assert_float_parity(run_gpu(chk, s), oracle_mod.check(s))
    g, o = _eval(P, chk, cfg, 2, [0, 5, 2 ** 30 - 1, 777777], oracle_mod)
    T = g.shape[1]
    assert_logits_close(g[:, T - 10:], o[:, T - 10:])


def test_cfg5_int8_bitexact(P, oracle_mod):
    cfg = M.make_config("cfg5_int8")
    chk = _checker(P, "cfg5_int8")
    s = cfg.subset(n_base=4, begin=0, end=300)
    assert_fixed_parity(run_gpu(chk, s), oracle_mod.check(s))
    s = cfg.subset(n_base=2, base_start=254, begin=2 ** 30 - 129, end=2 ** 30)
    assert_fixed_parity(run_gpu(chk, s), oracle_mod.check(s))
    g, o = _eval(P, chk, cfg, 1, [0, 1, 2 ** 30 - 1, 123456, 999], oracle_mod)
    assert np.array_equal(g.astype(np.int64), o.astype(np.int64))
