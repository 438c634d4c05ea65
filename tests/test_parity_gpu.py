"""GPU <-> oracle parity through the C ABI (`-m gpu`), subset / tuple spaces (configs 1-3).

Fixed point (Q4.12, int8): bit-exact counts, counterexample indices and coverage words.
Float (fp32): logits within 1e-6 + 1e-5 * max|o| per candidate; verdicts / coverage by the
flag rules of reading C20 (tests/parity.py)."""
import numpy as np
import pytest

import mlpv_inputs as M
from mlpv_inputs.configs import Config, CovSpec, Net, Pert, Prop
from tests.parity import (UMAX, assert_fixed_parity, assert_float_parity, assert_logits_close, run_gpu,
                          to_device_bases)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch
    assert torch.cuda.is_available(), "gpu tests need a GPU"
    from paper_1907_12933_b200 import build
    build.build()
    import paper_1907_12933_b200 as P
    return P


def _stress_cfg2():
    cfg = M.make_config("cfg2").subset(n_base=3)
    net = cfg.net
    cfg.net = Net(net.sizes, net.act, net.numeric,
                  [np.clip(net.W[0].astype(int) * 4, -32768, 32767).astype(np.int16),
                   np.clip(net.W[1].astype(int) * 16, -32768, 32767).astype(np.int16)],
                  net.b, sigmoid_knots=net.sigmoid_knots, acc_scale=net.acc_scale)
    cfg.pert = Pert(M.PERT_SUBSET_OFFSET, pixels=cfg.pert.pixels,
                    levels=np.array([-2048, -1024, 0, 1024, 2048], np.int16), index_begin=0, index_end=390_625)
    return cfg


def _eval_check(P, chk, cfg, idx, oracle_mod, fixed):
    import torch
    bases = to_device_bases(cfg)
    for b in sorted({0, cfg.n_base - 1}):
        it = torch.tensor(np.asarray(idx, np.int64), device="cuda")
        g = chk.eval(bases, b, cfg.pert, it).cpu().numpy()
        o = np.stack([np.concatenate(oracle_mod.forward(cfg.net, oracle_mod.decode(cfg.net.numeric, cfg.pert, cfg.bases[b], b, int(i))))
                      for i in idx])
        if fixed:
            assert np.array_equal(g.astype(np.int64), o.astype(np.int64))
        else:
            L = cfg.net.L
            T = g.shape[1]
            nL = cfg.net.sizes[L]
            assert_logits_close(g[:, T - nL:], o[:, T - nL:])
            assert np.allclose(g, o, rtol=1e-5, atol=1e-5)


def test_cfg1_full(P, oracle_mod):
    cfg = M.make_config("cfg1")
    chk = P.Checker(cfg.net)
    o = oracle_mod.check(cfg)
    g = run_gpu(chk, cfg)
    assert_float_parity(g, o)
    rng = np.random.default_rng(0)
    _eval_check(P, chk, cfg, [0, 1, 255, 256, 76_799] + list(rng.integers(0, 76_800, 500)), oracle_mod, False)


def test_cfg2_full(P, oracle_mod):
    cfg = M.make_config("cfg2")
    chk = P.Checker(cfg.net)
    assert_fixed_parity(run_gpu(chk, cfg), oracle_mod.check(cfg))
    rng = np.random.default_rng(0)
    _eval_check(P, chk, cfg, [0, 195_312, 390_624] + list(rng.integers(0, 390_625, 300)), oracle_mod, True)


def test_cfg2_stress(P, oracle_mod):
    """Non-trivial verdicts and coverage (sharper net, eps = 0.5)."""
    cfg = _stress_cfg2()
    chk = P.Checker(cfg.net)
    o = oracle_mod.check(cfg)
    assert o.violated.sum() > 0 and o.cov_all.any()
    assert_fixed_parity(run_gpu(chk, cfg), o)
    # ragged sub-ranges
    for a, b in [(1, 2), (7, 70_001), (390_000, 390_625), (123, 123)]:
        s = cfg.subset(begin=a, end=b)
        assert_fixed_parity(run_gpu(chk, s), oracle_mod.check(s))


def test_cfg3_prefixes(P, oracle_mod):
    cfg = M.make_config("cfg3")
    chk = P.Checker(cfg.net)
    s = cfg.subset(n_base=4, begin=0, end=1 << 18)
    assert_fixed_parity(run_gpu(chk, s), oracle_mod.check(s))
    s = cfg.subset(begin=(1 << 20) + 13, end=(1 << 20) + 13 + 2_003)      # all 100 bases, ragged
    assert_fixed_parity(run_gpu(chk, s), oracle_mod.check(s))
    s = cfg.subset(n_base=2, base_start=50, begin=16_777_216 - 70_001, end=16_777_216)
    assert_fixed_parity(run_gpu(chk, s), oracle_mod.check(s))
    rng = np.random.default_rng(3)
    _eval_check(P, chk, cfg, [0, 16_777_215] + list(rng.integers(0, 16_777_216, 200)), oracle_mod, True)


def test_cfg3_full_size_properties(P, oracle_mod):
    """Full BASELINE size (100 bases x 16.7M) in the bench launch configuration: checked counts, and
    each reported counterexample re-evaluates to a misclassification in the oracle and nothing in
    the first 2^14 indices below it is a violation."""
    cfg = M.make_config("cfg3")
    chk = P.Checker(cfg.net)
    g = run_gpu(chk, cfg)
    assert np.all(g["checked"] == 16_777_216)
    assert np.all(g["violated"] <= g["checked"])
    for b in range(0, 100, 7):
        c = int(g["first_cex"][b])
        if c == UMAX:
            assert g["violated"][b] == 0
            continue
        x = cfg.bases[b]
        y = oracle_mod.decode(cfg.net.numeric, cfg.pert, x, b, c)
        assert int(np.argmax(oracle_mod.forward(cfg.net, y)[-1])) != int(np.argmax(oracle_mod.forward(cfg.net, x)[-1]))
        lo = cfg.subset(n_base=1, base_start=b, begin=max(0, c - (1 << 14)), end=c)
        assert int(oracle_mod.check(lo).violated[0]) == 0


def _thr(numeric, levels):
    if numeric == M.NUM_Q4_12:
        net = Net([2, 2, 2], M.ACT_RELU, M.NUM_Q4_12, [np.array([[4096, 4096], [0, 0]], np.int16),
                  np.array([[0, 4096], [4096, 0]], np.int16)], [np.array([0, 1 << 24], np.int32), np.zeros(2, np.int32)],
                  acc_scale=[2.0 ** -24] * 2)
        base = np.array([[1638, 1638]], np.int16)
    else:
        net = Net([2, 2, 2], M.ACT_RELU, M.NUM_FP32, [np.array([[1, 1], [0, 0]], np.float32),
                  np.array([[0, 1], [1, 0]], np.float32)], [np.array([0, 1], np.float32), np.zeros(2, np.float32)],
                  acc_scale=[1.0, 1.0])
        base = np.array([[0.4, 0.4]], np.float32)
    pert = Pert(M.PERT_TUPLE_REPLACE, tuple=2, levels=levels)
    pert.index_end = pert.space_size(2)
    return Config("thr", "threshold net", net, base, pert, Prop(), CovSpec([1]))


def test_threshold_nets(P, oracle_mod):
    """The closed-form threshold net on the GPU: 10 violations of 25, first 9."""
    cfg = _thr(M.NUM_Q4_12, np.array([1024 * l for l in range(5)], np.int16))
    g = run_gpu(P.Checker(cfg.net), cfg)
    assert int(g["violated"][0]) == 10 and int(g["first_cex"][0]) == 9
    assert_fixed_parity(g, oracle_mod.check(cfg))
    cfg = _thr(M.NUM_FP32, np.array([l / 15 for l in range(16)], np.float32))
    g = run_gpu(P.Checker(cfg.net), cfg)
    assert int(g["flagged"][0]) == 16 and int(g["first_cex_unflagged"][0]) == 31
    assert_float_parity(g, oracle_mod.check(cfg))


def test_other_properties(P, oracle_mod):
    """TARGET_NEVER and THRESHOLD_LITERAL on the stress net."""
    cfg = _stress_cfg2()
    chk = P.Checker(cfg.net)
    for prop in (Prop(M.PROP_TARGET_NEVER, 1, 0.0), Prop(M.PROP_THRESHOLD_LITERAL, -1, 0.25),
                 Prop(M.PROP_THRESHOLD_LITERAL, 2, -0.5), Prop(M.PROP_THRESHOLD_LITERAL_ALL, -1, 0.25),
                 Prop(M.PROP_THRESHOLD_LITERAL_ALL, 1, -0.5)):
        s = cfg.subset(begin=0, end=50_000)
        s.prop = prop
        assert_fixed_parity(run_gpu(chk, s), oracle_mod.check(s))


def test_merge_and_neuron_coverage(P, oracle_mod):
    import torch
    cfg = _stress_cfg2()
    chk = P.Checker(cfg.net)
    bases = to_device_bases(cfg)
    a = chk.check(bases, cfg.subset(begin=0, end=100_000).pert, cfg.prop, cfg.cov)
    b = chk.check(bases, cfg.subset(begin=100_000, end=390_625).pert, cfg.prop, cfg.cov)
    nw = a["n_words"]
    m = P.merge([a, b], cfg.n_base, nw)
    torch.cuda.synchronize()
    g = P.result_to_numpy(m, cfg.n_base, nw)
    o = oracle_mod.check(cfg)
    assert_fixed_parity(g, o)
    covered, counts = chk.neuron_coverage(cfg.cov, m["cov_all"])
    sets = oracle_mod.covered_neurons(cfg.net.sizes, cfg.cov.pairs, o.cov_all)
    cnt = counts.cpu().numpy()
    cv = covered.cpu().numpy()
    offs = np.cumsum([0] + cfg.net.sizes[1:])
    for mi, meth in enumerate(oracle_mod.METHODS):
        assert cnt[mi] == len(sets[meth])
        got = {(l, i) for l in range(1, cfg.net.L + 1) for i in range(cfg.net.sizes[l]) if cv[mi, offs[l - 1] + i]}
        assert got == sets[meth]


def test_empty_and_single(P, oracle_mod):
    cfg = M.make_config("cfg2")
    chk = P.Checker(cfg.net)
    g = run_gpu(chk, cfg.subset(begin=5, end=5))
    assert np.all(g["checked"] == 0) and np.all(g["first_cex"] == UMAX) and not g["cov_all"].any()
    s = cfg.subset(begin=195_312, end=195_313)
    assert_fixed_parity(run_gpu(chk, s), oracle_mod.check(s))


def test_invalid_range_rejected(P):
    cfg = M.make_config("cfg2")
    chk = P.Checker(cfg.net)
    bad = cfg.subset()
    bad.pert = bad.pert.with_range(0, 390_626)
    with pytest.raises(P.MlpvError) as e:
        run_gpu(chk, bad)
    assert e.value.status == 1 and "index range" in str(e.value)


def test_literal_readings_gpu(P, oracle_mod):
    """The closed-form literal net (tests/test_oracle_pins.py): 16 / 4 violations, first 3 / 18."""
    from tests.test_oracle_pins import _literal_cfg
    for numeric in (M.NUM_FP32, M.NUM_Q4_12):
        for kind, nv, first in ((M.PROP_THRESHOLD_LITERAL, 16, 3), (M.PROP_THRESHOLD_LITERAL_ALL, 4, 18)):
            cfg = _literal_cfg(numeric, kind)
            g = run_gpu(P.Checker(cfg.net), cfg)
            assert int(g["violated"][0]) == nv and int(g["first_cex"][0]) == first
            o = oracle_mod.check(cfg)
            (assert_float_parity if numeric == M.NUM_FP32 else assert_fixed_parity)(g, o)


def test_lut_revalidation(P, oracle_mod):
    """NEXT-4: the first counterexamples of the stress Q4.12 net re-checked by the library under the
    real-valued network it approximates (exact sigmoid, FP32 path, a one-candidate space that
    reproduces the counterexample): the candidate is the decoded image, its potentials agree with
    the oracle's double forward of that network, and the library's verdict is the oracle's own
    check of the same one-candidate space (C20 rules)."""
    from paper_1907_12933_b200.revalidate import exact_net, one_candidate_space, revalidate
    from mlpv_inputs.configs import CovSpec
    cfg = _stress_cfg2()
    g = run_gpu(P.Checker(cfg.net), cfg)
    recs = revalidate(cfg.net, cfg.bases, cfg.pert, cfg.prop, g["first_cex"])
    assert len(recs) == int(np.count_nonzero(g["first_cex"] != UMAX)) and len(recs) > 0
    en = exact_net(cfg.net)
    for r in recs:
        assert r["checked"] == 1
        img = (oracle_mod.decode(cfg.net.numeric, cfg.pert, cfg.bases[r["base"]], r["base"], r["index"]).astype(np.float64) / 4096).astype(np.float32)
        base = (cfg.bases[r["base"]].astype(np.float64) / 4096).astype(np.float32)
        sp, idx = one_candidate_space(base, img)
        assert np.array_equal(oracle_mod.decode(M.NUM_FP32, sp, base, 0, idx), img)
        yo = np.concatenate(oracle_mod.forward(en, img))
        assert_logits_close(r["potentials"], yo)
        c = M.Config("reval", "one candidate", en, base[None, :], sp, cfg.prop, CovSpec([]))
        o = oracle_mod.check(c)
        vo, fo = int(o.violated[0]), int(o.flagged[0])
        assert int(r["violated_exact"]) == vo or (fo or r["flagged_exact"])
    print("LUT artefacts:", sum(not r["violated_exact"] for r in recs), "of", len(recs))


def test_restriction_gpu(P, oracle_mod):
    """Restriction R (reading C27) on every subset / tuple path against the oracle:
    the binary-image pin (57 / 63 / 64 of 64), Q4.12 subset offsets, fp32 pairs, int8 subset."""
    from tests.test_oracle_pins import _restrict_cfg
    for b, n in ((2.0, 57), (2.449, 63), (2.4495, 64)):
        cfg = _restrict_cfg(b)
        g = run_gpu(P.Checker(cfg.net), cfg)
        assert int(g["checked"][0]) == n
        assert_fixed_parity(g, oracle_mod.check(cfg))
    cfg = _stress_cfg2()
    chk = P.Checker(cfg.net)
    for b in (0.1, 0.3):
        s = cfg.subset(begin=0, end=120_000)
        s.pert.restrict_l2 = b
        g = run_gpu(chk, s)
        assert np.all(g["checked"] < 120_000)
        assert_fixed_parity(g, oracle_mod.check(s))
    cfg = M.make_config("cfg1")
    cfg.pert.restrict_l2 = 0.9
    g = run_gpu(P.Checker(cfg.net), cfg)
    assert 0 < int(g["checked"][0]) < 76_800
    assert_float_parity(g, oracle_mod.check(cfg))
    cfg = M.make_config("cfg3").subset(n_base=2, begin=0, end=200_000)
    cfg.pert.restrict_l2 = 0.8
    g = run_gpu(P.Checker(cfg.net), cfg)
    assert np.all(g["checked"] < 200_000)
    assert_fixed_parity(g, oracle_mod.check(cfg))


def test_incremental_rejected_on_philox(P):
    """Incremental bounds (NEXT-2) are built for the enumerated spaces; the Philox spaces say so."""
    import torch
    cfg = M.make_config("cfg4").subset(n_base=1, begin=0, end=10)
    with pytest.raises(P.MlpvError) as e:
        P.Checker(cfg.net).check_incremental(to_device_bases(cfg), cfg.pert, cfg.prop, cfg.cov, gamma=0.5, max_bound=4)
    assert e.value.status == 3


def test_device_found_input_errors(P):
    """Input rules that hold for device-resident data are checked on the device and reported by
    mlpv_sync (MLPV_E_INVALID): a Q4.12 base pixel outside [0, 4096] (reading C16), a PHILOX_CLAMP
    base pixel that breaks the exact-contraction rule of mlpv.h.  Replace levels outside the input
    domain are rejected synchronously."""
    import torch
    cfg = M.make_config("cfg2").subset(n_base=2, begin=0, end=1000)
    chk = P.Checker(cfg.net)
    bad = cfg.bases.copy()
    bad[1, 3] = 5000
    chk.check(torch.from_numpy(bad).cuda(), cfg.pert, cfg.prop, cfg.cov)
    with pytest.raises(P.MlpvError) as ei:
        chk.sync()
    assert ei.value.status == 1 and "4096" in str(ei.value)
    chk.check(torch.from_numpy(cfg.bases).cuda(), cfg.pert, cfg.prop, cfg.cov)
    chk.sync()                                              # the status was cleared
    rep = M.Pert(M.PERT_SUBSET_REPLACE, pixels=cfg.pert.pixels, levels=np.array([0, 4097], np.int16), index_end=2)
    with pytest.raises(P.MlpvError) as ei:
        chk.check(torch.from_numpy(cfg.bases).cuda(), rep, cfg.prop, cfg.cov)
    assert ei.value.status == 1
    c4 = M.make_config("cfg4").subset(n_base=1, begin=0, end=300)
    chk4 = P.Checker(c4.net)
    b4 = c4.bases.copy()
    b4[0, 5] = M.f32_to_bf16_bits(np.array([1e-7], np.float32))[0]   # 0 < x < 2^-16: -x / 2 is not an fp16 value
    chk4.check(to_device_bases(M.Config("x", "", c4.net, b4, c4.pert, c4.prop, c4.cov)), c4.pert, c4.prop, c4.cov)
    with pytest.raises(P.MlpvError) as ei:
        chk4.sync()
    assert ei.value.status == 1 and "PHILOX_CLAMP" in str(ei.value)
