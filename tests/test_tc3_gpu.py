"""k_tc3 (tcgen05 kind::i8 per layer, thread = candidate; SURVEY.md's K2) through the C ABI vs the
oracle, bit-exact (reading C18: every verdict, counterexample index and coverage word), on shapes and
spaces beyond config 3: padded MMA widths (n_1 = 48 -> N 48, n_2 = 24 -> N 32, n_3 = 7 -> N 16),
non-power-of-two level counts (64-bit / 32-bit digit division), clamped SUBSET_OFFSET pixels, a
one-pixel subset, ragged ranges whose tiles cross base inputs, every property kind; and the same
results with k_tc3 disabled (k_warp3 / k_small take the call)."""
import os

import numpy as np
import pytest

import mlpv_inputs as M
from mlpv_inputs.configs import Config, CovSpec, Net, Pert, Prop, _quant_int8
from tests.parity import assert_fixed_parity, run_gpu

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch
    assert torch.cuda.is_available(), "gpu tests need a GPU"
    from paper_1907_12933_b200 import build
    build.build()
    import paper_1907_12933_b200 as P
    return P


def _net(sizes, seed, shifts):
    rng = np.random.default_rng([12933, 77, seed])
    W = [rng.normal(0.0, np.sqrt(2.0 / sizes[l - 1]), (sizes[l], sizes[l - 1])).astype(np.float32)
         for l in range(1, len(sizes))]
    b = [rng.normal(0.0, np.sqrt(1.0 / sizes[l - 1]), sizes[l]).astype(np.float32) for l in range(1, len(sizes))]
    Wq, bq, acc = _quant_int8(W, b, shifts)
    return Net(list(sizes), M.ACT_RELU, M.NUM_INT8, Wq, bq, requant_shift=list(shifts), acc_scale=acc)


def _cfg(sizes, seed, shifts, kind, pixels, levels, n_base, pairs=(1, 2)):
    rng = np.random.default_rng([12933, 78, seed])
    net = _net(sizes, seed, shifts)
    bases = rng.integers(0, 256, (n_base, sizes[0]), dtype=np.uint8)
    bases[:, pixels[0]] = 3                          # pixels at the clamp edges
    if len(pixels) > 1:
        bases[:, pixels[1]] = 250
    pert = Pert(kind, pixels=np.asarray(pixels, np.int32), levels=np.asarray(levels, np.int16))
    pert.index_end = pert.space_size(sizes[0])
    return Config("tc3", "k_tc3 test", net, bases, pert, Prop(), CovSpec(list(pairs)))


def _both(P, cfg, oracle_mod):
    """GPU with k_tc3, then with it disabled; both against the oracle, bit-exact."""
    o = oracle_mod.check(cfg)
    g = run_gpu(P.Checker(cfg.net), cfg)
    assert_fixed_parity(g, o)
    os.environ["MLPV_NO_TC3"] = "1"
    try:
        assert_fixed_parity(run_gpu(P.Checker(cfg.net), cfg), o)
    finally:
        del os.environ["MLPV_NO_TC3"]
    return o


def test_padded_widths_offset_q5(P, oracle_mod):
    """n = 100-48-24-7, SUBSET_OFFSET over 7 pixels x 5 offsets (q = 5: divisions), clamped at 0 / 255."""
    cfg = _cfg([100, 48, 24, 7], 1, [9, 8], M.PERT_SUBSET_OFFSET, [2, 11, 30, 31, 57, 80, 99],
               [-240, -120, 0, 120, 240], 6)
    o = _both(P, cfg, oracle_mod)
    assert o.cov_all.any()
    for a, b in [(0, 1), (5, 130), (127, 129), (1000, 78_125 - 3)]:
        _both(P, cfg.subset(begin=a, end=b), oracle_mod)


def test_replace_one_pixel_and_small_widths(P, oracle_mod):
    """n = 64-16-16-3, one pixel x 256 replacement values; a 3-pixel subset x 16 values."""
    cfg = _cfg([64, 16, 16, 3], 2, [8, 7], M.PERT_SUBSET_REPLACE, [17], list(range(256)), 5)
    _both(P, cfg, oracle_mod)
    cfg = _cfg([64, 32, 16, 5], 3, [8, 7], M.PERT_SUBSET_REPLACE, [5, 40, 41], [17 * l for l in range(16)], 4)
    _both(P, cfg, oracle_mod)


def test_properties(P, oracle_mod):
    """TARGET_NEVER and both threshold literals (reading C12, NEXT-4) on a cfg3-shaped slice."""
    cfg = M.make_config("cfg3").subset(n_base=3, begin=0, end=40_000)
    for prop in (Prop(kind=M.PROP_TARGET_NEVER, target=1), Prop(kind=M.PROP_THRESHOLD_LITERAL, target=-1, V=0),
                 Prop(kind=M.PROP_THRESHOLD_LITERAL_ALL, target=2, V=-0.5)):
        c = cfg.subset(n_base=3, begin=0, end=40_000)
        c.prop = prop
        _both(P, c, oracle_mod)


def test_cfg3_tiles_across_bases(P, oracle_mod):
    """A range whose length is not a multiple of 128, over 7 base inputs: warpgroup ranges that
    straddle base inputs (counts flushed per base)."""
    cfg = M.make_config("cfg3").subset(n_base=7, base_start=20, begin=333, end=333 + 5_000)
    _both(P, cfg, oracle_mod)


def test_tiny_spaces_many_bases(P, oracle_mod):
    """300 base inputs with a 5-candidate space each: every tile is one base's only, mostly empty
    tile (123 invalid rows), and each warpgroup's range crosses many bases (per-base count flushes)."""
    cfg = _cfg([64, 32, 16, 10], 4, [8, 7], M.PERT_SUBSET_REPLACE, [9], [0, 60, 120, 180, 255], 300)
    _both(P, cfg, oracle_mod)
    _both(P, cfg.subset(begin=1, end=4), oracle_mod)
