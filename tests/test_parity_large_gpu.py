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
        err, ratio = assert_logits_close(g[:, T - 10:], o[:, T - 10:])
        herr, hratio = assert_logits_close(g, o)                 # hidden potentials too, same rule
        print(f"cfg4 base {b}: max logit err {err:.3e} (worst err/tol {ratio:.3f}); "
              f"all potentials {herr:.3e} ({hratio:.3f})")


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


# ----------------------------------------------------------------------------- k_fused3 variants
def _box_cfg(n0=784, n3=10, eps=0.05, n_base=6, w_var=2.0, seed=7, prop=None, kind=None):
    """A 3-layer n0-256-256-n3 ReLU bf16 net on the PHILOX_CLAMP space (reading C14; or PHILOX_BOX,
    C14b), i.e. the k_fused3 path with another input width / class count / radius / property.
    8-bit base images; the lattice of cfg4's rule (step = bf16(2 eps / 15), origin = -7.5 step)."""
    kind = M.PERT_PHILOX_CLAMP if kind is None else kind
    rng = np.random.default_rng([12933, 900, seed])
    sizes = [n0, 256, 256, n3]
    W = [M.f32_to_bf16_bits(rng.normal(0.0, np.sqrt(w_var / sizes[l - 1]), (sizes[l], sizes[l - 1])).astype(np.float32))
         for l in range(1, 4)]
    b = [rng.normal(0.0, np.sqrt(1.0 / sizes[l - 1]), sizes[l]).astype(np.float32) for l in range(1, 4)]
    net = M.Net(sizes, M.ACT_RELU, M.NUM_BF16, W, b, acc_scale=[1.0, 1.0, 1.0])
    bases = M.eight_bit_bf16(rng.random((n_base, n0)))
    step, origin = M.cfg4_lattice(eps)
    pert = M.Pert(kind, seed=int(rng.integers(2 ** 63)), n_samples=2 ** 32, lattice_step=step, lattice_origin=origin)
    pert.index_end = pert.n_samples
    return M.Config("box", "k_fused3 variant", net, bases, pert, prop or M.Prop(), M.CovSpec([1, 2]))


def test_fused3_small_radius_coverage_paths(P, oracle_mod):
    """eps = 0.002: most candidates keep (almost) every sign, so the rare-row statistics paths of
    E1/E2 (cond1 rows, <= 1 layer-2 change, one and several such rows per warp) carry the load."""
    cfg = _box_cfg(eps=0.002, n_base=4)
    chk = P.Checker(cfg.net)
    s = cfg.subset(begin=0, end=1500)
    o = oracle_mod.check(s)
    assert o.cov_all.any()
    assert_float_parity(run_gpu(chk, s), o)


def test_fused3_large_radius_verdicts(P, oracle_mod):
    """eps = 0.4: many violations (first counterexample, flagged counts) on the fused path."""
    cfg = _box_cfg(eps=0.4, n_base=5, seed=8)
    chk = P.Checker(cfg.net)
    s = cfg.subset(begin=1000, end=2300)
    o = oracle_mod.check(s)
    assert o.violated.sum() > 0
    assert_float_parity(run_gpu(chk, s), o)


@pytest.mark.parametrize("kind", [M.PERT_PHILOX_CLAMP, M.PERT_PHILOX_BOX])
@pytest.mark.parametrize("n0,n3", [(200, 7), (1024, 16), (2, 2), (786, 10)])
def test_fused3_shapes(P, oracle_mod, n0, n3, kind):
    """Other input widths (K tail inside a stage, the largest K, a single K step, n_0 not a multiple
    of 8) and class counts, on both box spaces."""
    cfg = _box_cfg(n0=n0, n3=n3, eps=0.05, n_base=3, seed=n0, kind=kind)
    chk = P.Checker(cfg.net)
    s = cfg.subset(begin=17, end=17 + 700)
    assert_float_parity(run_gpu(chk, s), oracle_mod.check(s))
    g, o = _eval(P, chk, cfg, 1, [0, 3, 2 ** 32 - 1, 99999], oracle_mod)
    assert_logits_close(g[:, -n3:], o[:, -n3:])


def test_fused3_properties(P, oracle_mod):
    for prop in (M.Prop(M.PROP_TARGET_NEVER, 3, 0.0), M.Prop(M.PROP_THRESHOLD_LITERAL, -1, 0.2),
                 M.Prop(M.PROP_THRESHOLD_LITERAL, 1, -0.1), M.Prop(M.PROP_THRESHOLD_LITERAL_ALL, -1, -0.3),
                 M.Prop(M.PROP_THRESHOLD_LITERAL_ALL, 2, 0.1)):
        cfg = _box_cfg(eps=0.2, n_base=3, seed=11, prop=prop)
        chk = P.Checker(cfg.net)
        s = cfg.subset(begin=0, end=900)
        assert_float_parity(run_gpu(chk, s), oracle_mod.check(s))


def test_cfg4_bench_launch(P, oracle_mod):
    """The launch bench.py times (all 1000 bases x a 65,536-sample slice, the fused kernel over
    256,000 tiles, base changes inside every cluster's tile range).  Base 0 (whose Philox base
    index is the same in a one-base oracle run) against the oracle on the same slice; for the
    other bases, properties that hold at any size: every candidate counted, and each reported
    first counterexample re-evaluates (oracle decode + forward in double) to a changed class or
    a flagged near-tie."""
    cfg = M.make_config("cfg4")
    chk = _checker(P, "cfg4")
    lo, hi = 3 * 65536, 4 * 65536
    g = run_gpu(chk, cfg.subset(begin=lo, end=hi))
    assert np.all(g["checked"] == hi - lo)
    tau = oracle_mod.default_tau(cfg)                       # tau_l from all 1000 bases, as on the GPU
    o = oracle_mod.check(cfg.subset(n_base=1, base_start=0, begin=lo, end=hi), tau=tau)
    vg, vo = int(g["violated"][0]), int(o.violated[0])
    assert abs(vg - vo) <= min(int(g["flagged"][0]), int(o.flagged[0]))
    assert int(g["first_cex"][0]) <= int(o.first_cex_unflagged[0])
    assert int(o.first_cex[0]) <= int(g["first_cex_unflagged"][0])
    assert not np.any(o.cov_certain & ~g["cov_all"][:len(o.cov_certain)])
    bad = np.nonzero(g["first_cex"] != UMAX)[0]
    for b in bad[:20]:
        c = int(g["first_cex"][b])
        assert lo <= c < hi
        y = oracle_mod.forward(cfg.net, oracle_mod.decode(cfg.net.numeric, cfg.pert, cfg.bases[b], int(b), c))[-1]
        yb = oracle_mod.forward(cfg.net, cfg.bases[b])[-1]
        top = np.sort(y)[::-1]
        assert int(np.argmax(y)) != int(np.argmax(yb)) or top[0] - top[1] < 1e-5, (b, c)


def test_cfg5_literal_all(P, oracle_mod):
    """The universal literal on the generic tcgen05 path (both numerics)."""
    for name, chk_par in (("cfg5_bf16", assert_float_parity), ("cfg5_int8", assert_fixed_parity)):
        cfg = M.make_config(name)
        s = cfg.subset(n_base=2, begin=0, end=260)
        s.prop = M.Prop(M.PROP_THRESHOLD_LITERAL_ALL, -1, 0.0)
        chk_par(run_gpu(_checker(P, name), s), oracle_mod.check(s))


@pytest.mark.parametrize("n0,step,origin", [(3072, -3.0, 20.0), (1000, 2.0, -15.0), (997, 1.0, -8.0),
                                            (256, 17.0, -255.0)])
def test_int8_lattice_generator_paths(P, oracle_mod, n0, step, origin):
    """k_large's int8 lattice generator: the 16-bit-lane fast path (whole 32-pixel blocks, step >= 0)
    and the per-pixel path (negative step, a ragged last block, n_0 not a multiple of 8), extreme
    offsets that clamp at 0 and 255; bit-exact against the oracle."""
    from mlpv_inputs.configs import _quant_int8
    rng = np.random.default_rng([12933, 950, n0])
    sizes = [n0, 256, 64, 10]
    W = [rng.normal(0.0, np.sqrt(2.0 / sizes[l - 1]), (sizes[l], sizes[l - 1])).astype(np.float32) for l in range(1, 4)]
    b = [rng.normal(0.0, np.sqrt(1.0 / sizes[l - 1]), sizes[l]).astype(np.float32) for l in range(1, 4)]
    sh = [7, 6]
    Wq, bq, acc = _quant_int8(W, b, sh)
    net = M.Net(sizes, M.ACT_RELU, M.NUM_INT8, Wq, bq, requant_shift=sh, acc_scale=acc)
    bases = np.rint(rng.random((3, n0)) * 255.0).astype(np.uint8)
    bases[0, : n0 // 3] = 0
    bases[1, : n0 // 3] = 255
    pert = M.Pert(M.PERT_PHILOX_LATTICE, seed=int(rng.integers(2 ** 63)), n_samples=2 ** 20,
                  lattice_step=step, lattice_origin=origin)
    pert.index_end = 300
    cfg = M.Config("i8gen", "int8 generator paths", net, bases, pert, M.Prop(), M.CovSpec([1, 2]))
    chk = P.Checker(net)
    assert_fixed_parity(run_gpu(chk, cfg), oracle_mod.check(cfg))
    g, o = _eval(P, chk, cfg, 1, [0, 1, 299, 12345], oracle_mod)
    assert np.array_equal(g.astype(np.int64), o.astype(np.int64))


@pytest.mark.parametrize("name", ["cfg5_bf16", "cfg5_int8"])
def test_cfg5_bench_launch(P, oracle_mod, name):
    """The launch bench.py times for cfg5 (all 256 bases x a 1,024 (bf16) / 2,048 (int8) sample slice
    of step 3).  Base 0 against the oracle on the same slice (int8 bit-exact, bf16 by the flag
    rules of reading C20); every other base: every candidate counted and each first counterexample
    re-evaluated by the oracle (decode + forward) to a changed class, or a near-tie for bf16."""
    cfg = M.make_config(name)
    chk = _checker(P, name)
    S = 1024 if name == "cfg5_bf16" else 2048
    lo, hi = 3 * S, 4 * S
    g = run_gpu(chk, cfg.subset(begin=lo, end=hi))
    assert np.all(g["checked"] == hi - lo)
    fixed = name == "cfg5_int8"
    tau = None if fixed else oracle_mod.default_tau(cfg)
    o = oracle_mod.check(cfg.subset(n_base=1, base_start=0, begin=lo, end=hi), tau=tau)
    if fixed:
        assert int(g["violated"][0]) == int(o.violated[0]) and int(g["first_cex"][0]) == int(o.first_cex[0])
        assert np.array_equal(g["cov_all"][:len(o.cov_all)] & o.cov_all, o.cov_all)
    else:
        vg, vo = int(g["violated"][0]), int(o.violated[0])
        assert abs(vg - vo) <= min(int(g["flagged"][0]), int(o.flagged[0]))
        assert int(g["first_cex"][0]) <= int(o.first_cex_unflagged[0])
        assert int(o.first_cex[0]) <= int(g["first_cex_unflagged"][0])
    for b in np.nonzero(g["first_cex"] != UMAX)[0][:12]:
        c = int(g["first_cex"][b])
        assert lo <= c < hi
        y = oracle_mod.forward(cfg.net, oracle_mod.decode(cfg.net.numeric, cfg.pert, cfg.bases[b], int(b), c))[-1]
        yb = oracle_mod.forward(cfg.net, cfg.bases[b])[-1]
        top = np.sort(y)[::-1]
        assert int(np.argmax(y)) != int(np.argmax(yb)) or (not fixed and top[0] - top[1] < 1e-5), (b, c)


@pytest.mark.parametrize("name,b,nb,n", [("cfg4", 0.753, 3, 700), ("cfg4_box", 0.857, 2, 500), ("cfg5_bf16", 1.004, 2, 300),
                                          ("cfg5_int8", 1.0, 2, 300)])
def test_restriction_on_philox_spaces(P, oracle_mod, name, b, nb, n):
    """Restriction R on the Philox spaces: the mask pass keeps the
    candidates with delta <= b; checked (= inside R) is bit-exact against the oracle, verdicts and
    coverage by the numeric's rules.  b is chosen to cut each slice roughly in half."""
    cfg = M.make_config(name).subset(n_base=nb, begin=1000, end=1000 + n)
    cfg.pert.restrict_l2 = b
    o = oracle_mod.check(cfg)
    assert 0 < int(o.checked.sum()) < nb * n
    g = run_gpu(_checker(P, name) if name != "cfg4_box" else P.Checker(cfg.net), cfg)
    if cfg.net.numeric == M.NUM_INT8:
        assert_fixed_parity(g, o)
    else:
        assert_float_parity(g, o)
