"""Dataset-pair coverage through the C ABI vs
the oracle's `pair_coverage` (`-m gpu`).

Fixed point (Q4.12, int8): cov_all and cov_certain bit-exact, and the covered-neuron literal
l_covered_neuron (P = 80 %) identical.  Float (fp32, bf16): the flag rules of reading C20 -- every
bit the GPU calls certain is covered in the oracle, every bit the oracle calls certain is covered
on the GPU."""
import numpy as np
import pytest

import mlpv_inputs as M
from mlpv_inputs.configs import CovSpec

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch
    assert torch.cuda.is_available(), "gpu tests need a GPU"
    from paper_1907_12933_b200 import build
    build.build()
    import paper_1907_12933_b200 as P
    return P


def _dev(imgs):
    import torch
    x = imgs.view(np.int16) if imgs.dtype == np.uint16 else imgs
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def _run(P, net, imgs, cov, tau=None):
    chk = P.Checker(net)
    try:
        a, c = chk.pair_coverage(_dev(imgs), cov, tau=tau)
        a_np = a.cpu().numpy().view(np.uint32)
        c_np = c.cpu().numpy().view(np.uint32)
        _, counts = chk.neuron_coverage(cov, a) if a.numel() else (None, None)
        return a_np, c_np, (counts.cpu().numpy() if counts is not None else None)
    finally:
        chk.close()


def _near_duplicates(net, n, seed):
    """One image and n - 1 copies with 1-3 pixels redrawn: few sign changes per layer, so the
    one-change (SS / SV) and no-change (DS / DV) premises of the covers occur."""
    rng = np.random.default_rng([12933, 404, seed])
    x = M.pair_images(net, 1, seed=seed)[0]
    pool = M.pair_images(net, n, seed=seed + 100)
    out = [x.copy()]
    for i in range(1, n):
        y = x.copy()
        pix = rng.choice(len(x), int(rng.integers(1, 4)), replace=False)
        y[pix] = pool[i][pix]
        out.append(y)
    return np.stack(out)


def _layers_ratio(net, cov, counts):
    """GPU neuron counts -> ratio over the layers spanned by the pairs (reading C9)."""
    layers = sorted({k for k in cov.pairs} | {k + 1 for k in cov.pairs})
    N = sum(net.sizes[l] for l in layers)
    return {m: counts[i] / N for i, m in enumerate(("SS", "SV", "VS", "VV"))}


@pytest.mark.parametrize("d", [0.0, 0.05, 0.1, 0.5])
def test_vowel_q412_200_images(P, oracle_mod, d):
    """EG1's workload shape: 200 images -> 19,900 pairs on the 25-5-4-5 Q4.12 net, bit-exact."""
    net = M.vowel_net(M.NUM_Q4_12)
    imgs = M.pair_images(net, 200, seed=0)
    cov = CovSpec([1, 2], d_value=d, d_distance=d)
    a, c, counts = _run(P, net, imgs, cov)
    oa, oc = oracle_mod.pair_coverage(net, imgs, cov.pairs, d, d)
    assert np.array_equal(a, oa), np.nonzero(a != oa)
    assert np.array_equal(c, oc)
    ratio, N = oracle_mod.coverage_ratio(net.sizes, cov.pairs, oa)
    g = _layers_ratio(net, cov, counts)
    for m in ratio:
        assert g[m] == pytest.approx(ratio[m], abs=0)
        assert oracle_mod.coverage_literal(g[m], 0.8) == oracle_mod.coverage_literal(ratio[m], 0.8)


def test_vowel_fp32_flag_rules(P, oracle_mod):
    net = M.vowel_net(M.NUM_FP32)
    imgs = M.pair_images(net, 120, seed=2)
    cov = CovSpec([1, 2], d_value=0.08, d_distance=0.08)
    a, c, _ = _run(P, net, imgs, cov)
    oa, oc = oracle_mod.pair_coverage(net, imgs, cov.pairs, 0.08, 0.08)
    assert not np.any(c & ~oa)
    assert not np.any(oc & ~a)
    assert not np.any(c & ~a)
    assert a.any()


def test_explicit_tau(P, oracle_mod):
    """cov.tau given: tau = 0 -> certain = all on both sides and then all must agree exactly unless
    a predicate sits exactly on its boundary in one precision; a huge tau -> nothing certain."""
    net = M.vowel_net(M.NUM_FP32)
    imgs = M.pair_images(net, 40, seed=3)
    cov = CovSpec([1, 2], d_value=0.08, d_distance=0.08)
    a, c, _ = _run(P, net, imgs, cov, tau=[1e9] * 3)
    assert a.any() and not c.any()
    a0, c0, _ = _run(P, net, imgs, cov, tau=[0.0] * 3)
    assert np.array_equal(a0, c0) and np.array_equal(a0, a)


def test_int8_cfg3_net_exact(P, oracle_mod):
    """784-64-32-10 int8 (config 3's net), 60 blob images -> 1,770 pairs, both pairs of layers."""
    net = M.make_config("cfg3").net
    for imgs in (M.pair_images(net, 60, seed=4), _near_duplicates(net, 60, seed=4)):
        cov = CovSpec([1, 2], d_value=0.2, d_distance=0.5)
        a, c, _ = _run(P, net, imgs, cov)
        oa, oc = oracle_mod.pair_coverage(net, imgs, cov.pairs, 0.2, 0.5)
        assert np.array_equal(a, oa)
        assert np.array_equal(c, oc)
    assert a.any()


def test_bf16_cfg5_net_global_words(P, oracle_mod):
    """3072-1024-512-10 bf16 (config 5's net): 66 KB of words per pair of layers -> the kernel's
    global-atomic path; flag rules of reading C20."""
    net = M.make_config("cfg5_bf16").net
    imgs = _near_duplicates(net, 12, seed=5)
    cov = CovSpec([1, 2], d_value=0.05, d_distance=0.05)
    a, c, _ = _run(P, net, imgs, cov)
    oa, oc = oracle_mod.pair_coverage(net, imgs, cov.pairs, 0.05, 0.05)
    assert not np.any(c & ~oa)
    assert not np.any(oc & ~a)
    assert a.any()


def test_edge_cases(P):
    import torch
    net = M.vowel_net(M.NUM_Q4_12)
    imgs = M.pair_images(net, 5, seed=6)
    a, c, _ = _run(P, net, imgs[:1], CovSpec([1, 2]))       # one image: no pair
    assert not a.any() and not c.any()
    chk = P.Checker(net)
    try:
        a, c = chk.pair_coverage(_dev(imgs), CovSpec([]))       # no pairs of layers: no words
        assert a.numel() == 0
        with pytest.raises(Exception):
            chk.pair_coverage(_dev(imgs)[:0], CovSpec([1]))    # n_images = 0
        with pytest.raises(Exception):
            chk.pair_coverage(_dev(imgs), CovSpec([3]))        # lower layer out of range
    finally:
        chk.close()
    torch.cuda.synchronize()
