"""Incremental bounds (reading C28) through the C ABI vs
the oracle's literal iteration-by-iteration loop (`-m gpu`).

The GPU enumerates the gamma ball once and keys each violation by (step of the smallest ball
holding it, index); the oracle re-runs the restricted check for b_1, b_2, .. and stops at the
first hit.  Fixed point: step / first_cex bit-exact.  Float: the (step, index) keys obey the flag
rule of reading C20 (key_gpu <= key_unflagged_oracle and key_oracle <= key_unflagged_gpu)."""
import numpy as np
import pytest

import mlpv_inputs as M
from tests.parity import UMAX, to_device_bases
from tests.test_parity_gpu import _stress_cfg2

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch
    assert torch.cuda.is_available(), "gpu tests need a GPU"
    from paper_1907_12933_b200 import build
    build.build()
    import paper_1907_12933_b200 as P
    return P


def _gpu(P, cfg, gamma, mb, g, early_exit=False):
    chk = P.Checker(cfg.net)
    try:
        r = chk.check_incremental(to_device_bases(cfg), cfg.pert, cfg.prop, cfg.cov, gamma, mb, g,
                                  early_exit=early_exit)
        out = {k: r[k][:cfg.n_base].cpu().numpy() for k in ("step", "step_unflagged")}
        for k in ("first_cex", "first_cex_unflagged", "checked", "violated", "flagged"):
            out[k] = r[k][:cfg.n_base].cpu().numpy().view(np.uint64)
        nw = r["n_words"]
        out["cov_all"] = r["cov_all"][:nw].cpu().numpy().view(np.uint32) if nw else np.zeros(0, np.uint32)
        return out
    finally:
        chk.close()


def _key(step, idx):
    return [(int(s), int(i)) if s > 0 else (1 << 30, 0) for s, i in zip(step, idx)]


def _exact(g, o):
    assert np.array_equal(g["step"], o["step"]), (g["step"], o["step"])
    assert np.array_equal(g["first_cex"], o["first_cex"])
    assert np.array_equal(g["step_unflagged"], o["step_unflagged"])
    assert np.array_equal(g["first_cex_unflagged"], o["first_cex_unflagged"])


def _float_rule(g, o):
    kg, kgu = _key(g["step"], g["first_cex"]), _key(g["step_unflagged"], g["first_cex_unflagged"])
    ko, kou = _key(o["step"], o["first_cex"]), _key(o["step_unflagged"], o["first_cex_unflagged"])
    for b in range(len(kg)):
        assert kg[b] <= kou[b] and ko[b] <= kgu[b], b


def test_threshold_net(P, oracle_mod):
    """SPEC.md's 2-pixel threshold net: the pinned (step, index) pairs, g = 1 / 2 / 3, none at 0.17."""
    from tests.test_oracle_pins import _flip_cfg
    cfg = _flip_cfg()
    for gamma, g, want in ((0.5, 1, (4, 18)), (0.5, 2, (2, 18)), (0.5, 3, (2, 14)), (0.17, 1, (0, None))):
        r = _gpu(P, cfg, gamma, 10, g)
        assert int(r["step"][0]) == want[0]
        if want[1] is not None:
            assert int(r["first_cex"][0]) == want[1]
        else:
            assert r["first_cex"][0] == UMAX
        _exact(r, oracle_mod.incremental_verify(cfg, gamma, 10, g))


@pytest.mark.parametrize("g", [1, 2, 5])
def test_gamma_workload_q412(P, oracle_mod, g):
    """Table III-style: 50 binary 5x5 bases, 8 pixels x {0, .5, 1}, gamma = 3 in 12 unit steps."""
    cfg = M.gamma_config(50)
    r = _gpu(P, cfg, 3.0, 12, g)
    o = oracle_mod.incremental_verify(cfg, 3.0, 12, g)
    _exact(r, o)
    assert len(set(r["step"].tolist()) - {0}) >= 2           # bases decided at several steps
    # the whole-ball counts are those of the restricted check at gamma
    cfg.pert.restrict_l2 = 3.0
    full = oracle_mod.check(cfg)
    assert np.array_equal(r["checked"], full.checked) and np.array_equal(r["violated"], full.violated)


def test_stress_cfg2_offsets(P, oracle_mod):
    cfg = _stress_cfg2().subset(begin=0, end=120_000)
    _exact(_gpu(P, cfg, 0.6, 6, 1), oracle_mod.incremental_verify(cfg, 0.6, 6, 1))


def test_int8_cfg3_subset(P, oracle_mod):
    cfg = M.make_config("cfg3").subset(n_base=3, begin=0, end=60_000)
    _exact(_gpu(P, cfg, 1.0, 5, 1), oracle_mod.incremental_verify(cfg, 1.0, 5, 1))


def test_fp32_cfg1_pairs(P, oracle_mod):
    cfg = M.make_config("cfg1")
    for gamma, mb in ((1.0, 5), (1.4, 7)):
        _float_rule(_gpu(P, cfg, gamma, mb, 1), oracle_mod.incremental_verify(cfg, gamma, mb, 1))


def test_rejections(P):
    import torch
    from tests.test_oracle_pins import _flip_cfg
    cfg = _flip_cfg()
    for gamma, mb, g in ((0.0, 10, 1), (float("nan"), 10, 1), (0.5, 0, 1), (0.5, 10, 0), (0.5, 5000, 1)):
        with pytest.raises(P.MlpvError) as e:
            _gpu(P, cfg, gamma, mb, g)
        assert e.value.status == 1
    c4 = M.make_config("cfg4").subset(n_base=1, begin=0, end=10)
    with pytest.raises(P.MlpvError) as e:
        _gpu(P, c4, 0.5, 4, 1)
    assert e.value.status == 3
    torch.cuda.synchronize()


def _final_cov(oracle_mod, cfg, o):
    """OR over the base inputs of the coverage of the ball each one stopped at (oracle only)."""
    import copy
    acc = None
    for j in range(cfg.n_base):
        s = int(o["step_unflagged"][j]) or len(o["bounds"])
        c = cfg.subset(n_base=1, base_start=j, begin=cfg.pert.index_begin, end=cfg.pert.index_end)
        c.pert = copy.copy(c.pert)
        c.pert.restrict_l2 = o["bounds"][s - 1]
        w = np.asarray(oracle_mod.check(c).cov_all, np.uint32)
        acc = w if acc is None else acc | w
    return acc


@pytest.mark.parametrize("g", [1, 3])
def test_early_exit_gamma_workload_q412(P, oracle_mod, g):
    """NEXT-2 early exit (the loop's own order, one shell per pass): the (step, index) results equal
    the one-enumeration keys and the oracle's loop bit for bit; checked / violated per base input and
    the coverage words are those of the ball each base's loop stopped at (oracle: restricted checks
    at b_(s_b))."""
    cfg = M.gamma_config(50)
    r = _gpu(P, cfg, 3.0, 12, g, early_exit=True)
    o = oracle_mod.incremental_verify(cfg, 3.0, 12, g)
    _exact(r, o)
    one = _gpu(P, cfg, 3.0, 12, g)
    _exact(r, one)
    assert np.array_equal(r["checked"], o["final"]["checked"]), (r["checked"], o["final"]["checked"])
    assert np.array_equal(r["violated"], o["final"]["violated"])
    decided = r["step"] > 0
    assert decided.any() and (r["checked"][decided] < one["checked"][decided]).any()   # work saved
    assert np.array_equal(r["cov_all"], _final_cov(oracle_mod, cfg, o))


def test_early_exit_threshold_and_int8(P, oracle_mod):
    from tests.test_oracle_pins import _flip_cfg
    cfg = _flip_cfg()
    r = _gpu(P, cfg, 0.5, 10, 1, early_exit=True)
    assert (int(r["step"][0]), int(r["first_cex"][0]), int(r["checked"][0]), int(r["violated"][0])) == (4, 18, 9, 1)
    cfg = M.make_config("cfg3").subset(n_base=3, begin=0, end=60_000)
    r = _gpu(P, cfg, 1.0, 5, 1, early_exit=True)
    o = oracle_mod.incremental_verify(cfg, 1.0, 5, 1)
    _exact(r, o)
    assert np.array_equal(r["checked"], o["final"]["checked"]) and np.array_equal(r["violated"], o["final"]["violated"])


def test_early_exit_fp32_cfg1(P, oracle_mod):
    cfg = M.make_config("cfg1")
    r = _gpu(P, cfg, 1.4, 7, 1, early_exit=True)
    o = oracle_mod.incremental_verify(cfg, 1.4, 7, 1)
    _float_rule(r, o)
    same = r["step_unflagged"] == o["step_unflagged"]
    assert np.array_equal(r["checked"][same], o["final"]["checked"][same])
