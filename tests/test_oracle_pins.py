"""Pins of the CPU oracle against things other than itself (CPU only, `-m "not gpu"`).

Each test names the passage of PAPER.md / SPEC.md or the closed form / library routine it uses.
A plausible mistake in the oracle (dropped term, wrong sign or index, transposed operand, wrong
rounding) should fail at least one of these.
"""
import itertools
import math
import os

import numpy as np
import pytest

import mlpv_inputs as M
from mlpv_inputs.configs import Config, CovSpec, Net, Pert, Prop

GOLD = os.path.join(os.path.dirname(__file__), "golden")


# ----------------------------------------------------------------------------- helpers
def _table(name):
    rows = []
    for line in open(os.path.join(GOLD, name)):
        line = line.strip()
        if line and not line.startswith("#"):
            rows.append(line.split())
    return rows


def _t1():
    out = {}
    for r in _table("table1.txt"):
        v = [float(x) for x in r[3:]]
        out[r[0]] = [np.array(v[0:3]), np.array(v[3:5]), np.array(v[5:6])]
    return out


def _t2():
    rows = _table("table2.txt")
    u = [[], [], []]
    n = [[], [], []]
    for r in rows:
        layer = int(r[1])
        u[layer - 1].append(float(r[3]))
        n[layer - 1].append(float(r[4]))
    return [np.array(x) for x in u], [np.array(x) for x in n]


def _pairs_of(O, sizes, pairs, words):
    """set of (method, lower_layer, i, j); i is None for the VS/VV column masks"""
    _, offs = O.coverage_layout(sizes, pairs)
    out = set()
    for p, k in enumerate(pairs):
        nk, nu = sizes[k], sizes[k + 1]
        wpr = (nu + 31) // 32
        for mi, m in enumerate(O.METHODS):
            rows = nk if m in ("SS", "SV") else 1
            for i in range(rows):
                for j in range(nu):
                    if (int(words[offs[p, mi] + i * wpr + j // 32]) >> (j % 32)) & 1:
                        out.add((m, k, i if m in ("SS", "SV") else None, j))
    return out


def _cover(O, sizes, t1, t2, pairs, d=0.1):
    L = len(sizes) - 1
    return _pairs_of(O, sizes, pairs, O.cover_traces(sizes, t1, t2, pairs, [d] * L, [d] * L))


T1_SIZES = [2, 3, 2, 1]
T2_SIZES = [25, 5, 4, 5]


# ----------------------------------------------------------------------------- Table I (§III.B)
def test_table1_ss_ex1_ex2(oracle_mod):
    """only n_{3,1} changes sign in layer 1 between Ex1 and Ex2, so every layer-2
    neuron with a sign change forms an SS pair with it; the paper names (n31, n12).  Under C3 both
    layer-2 neurons change sign, so exactly (n31,n12) and (n31,n22) are SS-covered."""
    t = _t1()
    got = _cover(oracle_mod, T1_SIZES, t["Ex1"], t["Ex2"], [1, 2])
    assert ("SS", 1, 2, 0) in got                     # the pair the paper prints
    assert got == {("SS", 1, 2, 0), ("SS", 1, 2, 1)}


def test_table1_ds_sv_ex2_ex3(oracle_mod):
    """Ex2/Ex3 have no layer-1 sign change and a distance change (dc), and n_{2,2}
    changes sign -> DS(=VS) column n22 (reading C8); only n22 changes sign in layer 2 and n13
    changes value -> SV pair (n22, n13).  Under C5 (|du| >= 0.1) n12 changes value -> VV column n12."""
    t = _t1()
    got = _cover(oracle_mod, T1_SIZES, t["Ex2"], t["Ex3"], [1, 2])
    assert ("SV", 2, 1, 0) in got                     # the SV pair the paper prints
    assert ("VS", 1, None, 1) in got                  # DS column n22
    assert got == {("VS", 1, None, 1), ("VV", 1, None, 0), ("SV", 2, 1, 0)}


def test_table1_dv_ex1_ex4(oracle_mod):
    """Ex1/Ex4 have no sign change anywhere; distance change in layers 1 and 2 and
    value changes in layers 2 and 3 give DV(=VV) pairs."""
    t = _t1()
    got = _cover(oracle_mod, T1_SIZES, t["Ex1"], t["Ex4"], [1, 2])
    assert got == {("VV", 1, None, 0), ("VV", 1, None, 1), ("VV", 2, None, 0)}


def test_table1_symmetry_and_identity(oracle_mod):
    """sc and the L-inf / |du| metrics are symmetric in (x1, x2); identical traces cover nothing
    (SPEC.md:269, 287, 300, 323)."""
    t = _t1()
    for a, b in itertools.combinations(sorted(t), 2):
        assert _cover(oracle_mod, T1_SIZES, t[a], t[b], [1, 2]) == _cover(oracle_mod, T1_SIZES, t[b], t[a], [1, 2])
    for a in t:
        assert _cover(oracle_mod, T1_SIZES, t[a], t[a], [1, 2]) == set()


# ----------------------------------------------------------------------------- Table II (§IV.C)
def test_table2_ss_pairs_and_ratio(oracle_mod):
    """SS pairs {n11,n42} and {n42,n53}; 3 of 14 neurons = 21 %; P = 80 % fails."""
    O = oracle_mod
    u, nz = _t2()
    w = O.cover_traces(T2_SIZES, u, nz, [1, 2], [0.1] * 3, [0.1] * 3)
    got = {x for x in _pairs_of(O, T2_SIZES, [1, 2], w) if x[0] == "SS"}
    assert got == {("SS", 1, 0, 3), ("SS", 2, 3, 4)}
    sets = O.covered_neurons(T2_SIZES, [1, 2], w)
    assert sets["SS"] == {(1, 0), (2, 3), (3, 4)}
    ratios, N = O.coverage_ratio(T2_SIZES, [1, 2], w)
    assert N == 14
    assert abs(ratios["SS"] - 3 / 14) < 1e-12 and round(100 * ratios["SS"]) == 21
    assert O.coverage_literal(ratios["SS"], 0.80) is False
    assert O.coverage_literal(0.80, 0.80) is True                 # "equal or greater"


def test_table2_derived_sv_vs_vv(oracle_mod):
    """Derived from the printed potentials under C5/C7 (d = 0.1): SV neurons
    {n11,n12,n32,n42,n13,n23,n33,n43} = 8/14; every layer has a sign change, so VS = VV = {}."""
    O = oracle_mod
    u, nz = _t2()
    w = O.cover_traces(T2_SIZES, u, nz, [1, 2], [0.1] * 3, [0.1] * 3)
    sets = O.covered_neurons(T2_SIZES, [1, 2], w)
    assert sets["SV"] == {(1, 0), (2, 0), (2, 2), (2, 3), (3, 0), (3, 1), (3, 2), (3, 3)}
    assert sets["VS"] == set() and sets["VV"] == set()


def test_sign_at_zero(oracle_mod):
    """sign(i) = 1 iff i >= 0: +0 vs -0 is no change, 0 vs -1e-9 is a change."""
    O = oracle_mod
    s = [1, 1, 1]
    assert _cover(O, s, [np.array([0.0]), np.array([1.0])], [np.array([-0.0]), np.array([1.0])], [1]) == set()
    got = _cover(O, s, [np.array([0.0]), np.array([1.0])], [np.array([-1e-9]), np.array([-1.0])], [1])
    assert got == {("SS", 1, 0, 0)}


def test_cover_invariants_random(oracle_mod):
    """vc and sc exclusive; dc implies no sc in layer k; symmetry."""
    O = oracle_mod
    rng = np.random.default_rng(7)
    sizes, pairs = [4, 6, 5, 3], [1, 2]
    for _ in range(300):
        t1 = [rng.normal(0, 1, n) for n in sizes[1:]]
        t2 = [a + rng.normal(0, rng.choice([0.05, 0.3, 2.0]), a.shape) for a in t1]
        got = _cover(O, sizes, t1, t2, pairs)
        assert got == _cover(O, sizes, t2, t1, pairs)
        for k in pairs:
            ss = {(i, j) for m, kk, i, j in got if m == "SS" and kk == k}
            sv = {(i, j) for m, kk, i, j in got if m == "SV" and kk == k}
            vs = {j for m, kk, i, j in got if m == "VS" and kk == k}
            vv = {j for m, kk, i, j in got if m == "VV" and kk == k}
            assert not (ss & sv) and not (vs & vv)
            assert len({i for i, _ in ss | sv}) <= 1            # a single sign-changing row
            if vs or vv:
                assert not ss and not sv
            nsc = int(np.sum((t1[k - 1] >= 0) != (t2[k - 1] >= 0)))
            if nsc != 1:
                assert not ss and not sv


# ----------------------------------------------------------------------------- argmax / property
def test_argmax_tie_and_table2():
    """lowest index on ties; Table II output potentials -> index 4 (n_{5,3})."""
    from oracle import oracle as O
    sizes = [1, 2]
    net = Net(sizes, M.ACT_RELU, M.NUM_FP32, [np.array([[0.0], [0.0]], np.float32)],
              [np.array([0.5, 0.5], np.float32)], acc_scale=[1.0])
    assert int(np.argmax(O.forward(net, np.array([0.3], np.float32))[-1])) == 0
    u, nz = _t2()
    assert int(np.argmax(u[2])) == 4 and int(np.argmax(nz[2])) == 4


# ----------------------------------------------------------------------------- PL sigmoid (C17)
def test_pl_sigmoid_table_and_error(oracle_mod):
    O = oracle_mod
    T = M.configs.pl_sigmoid_knots()
    assert T[64] == 2048 and T[0] == 1 and T[128] == 4095
    assert np.all(np.diff(T.astype(int)) >= 0)
    for m in range(128):
        assert O.plsig(T, -32768 + 512 * m) == T[m]
    ys = np.array([O.plsig(T, u) for u in range(-32768, 32768)])
    assert np.all(np.diff(ys) >= 0)
    assert ys[32768] == 2048                                   # sigma(0) = 1/2 (Eq. 2)
    exact = 4096.0 / (1.0 + np.exp(-np.arange(-32768, 32768) / 4096.0))
    assert np.max(np.abs(ys - exact)) <= 1.6


# ----------------------------------------------------------------------------- fixed-point forward
def _net_q(sizes, Ws, bs, act=M.ACT_RELU):
    return Net(sizes, act, M.NUM_Q4_12, [np.array(w, np.int16) for w in Ws],
               [np.array(b, np.int32) for b in bs], sigmoid_knots=M.configs.pl_sigmoid_knots(),
               acc_scale=[2.0 ** -24] * (len(sizes) - 1))


def _net_i8(sizes, Ws, bs, shifts):
    return Net(sizes, M.ACT_RELU, M.NUM_INT8, [np.array(w, np.int8) for w in Ws],
               [np.array(b, np.int32) for b in bs], requant_shift=list(shifts),
               acc_scale=[1.0] * (len(sizes) - 1))


def test_gemm_2x2_example(oracle_mod):
    """SPEC.md:202 / Alg. 1 (read as C = A*B, C24): [[1,2],[3,4]]*[[5,6],[7,8]]
    = [[19,22],[43,50]], as one-layer nets applied to the columns of B."""
    O = oracle_mod
    for net in (_net_q([2, 2], [[[1, 2], [3, 4]]], [[0, 0]]), _net_i8([2, 2], [[[1, 2], [3, 4]]], [[0, 0]], [])):
        dt = np.int16 if net.numeric == M.NUM_Q4_12 else np.uint8
        assert list(O.forward(net, np.array([5, 7], dt))[0]) == [19, 43]
        assert list(O.forward(net, np.array([6, 8], dt))[0]) == [22, 50]


def test_zero_weights_give_bias(oracle_mod):
    """all-zero weights -> u = b in every layer."""
    O = oracle_mod
    net = _net_q([3, 2, 2], [np.zeros((2, 3)), np.zeros((2, 2))], [[5 << 12, -7 << 12], [11, -13]], M.ACT_PL_SIGMOID)
    t = O.forward(net, np.array([100, 200, 300], np.int16))
    assert list(t[0]) == [5 << 12, -7 << 12] and list(t[1]) == [11, -13]


def test_identity_onehot_int8(oracle_mod):
    """Identity layer 1 with shift 0 passes clamp(x) through; a permutation layer 2 permutes it."""
    O = oracle_mod
    net = _net_i8([3, 3, 3], [np.eye(3), [[0, 0, 1], [1, 0, 0], [0, 1, 0]]], [[0, 0, 0], [0, 0, 0]], [0])
    t = O.forward(net, np.array([7, 0, 255], np.uint8))
    assert list(t[0]) == [7, 0, 255] and list(t[1]) == [255, 7, 0]


def test_q412_requant_rounding(oracle_mod):
    """C16: u16 = sat16((acc + 2^11) >> 12), arithmetic shift = floor; hand-computed cases."""
    O = oracle_mod
    T = M.configs.pl_sigmoid_knots()
    for acc, u16 in [(2047, 0), (2048, 1), (6143, 1), (6144, 2), (4096 * 32767, 32767), (4096 * 40000, 32767)]:
        # zero weights, bias = acc: the hidden potential is exactly acc
        relu = _net_q([1, 1, 1], [[[0]], [[4096]]], [[acc], [0]], M.ACT_RELU)
        t = O.forward(relu, np.array([0], np.int16))
        assert t[0][0] == acc and t[1][0] == 4096 * u16, (acc, u16)
    pls = _net_q([1, 1, 1], [[[1]], [[1]]], [[0], [0]], M.ACT_PL_SIGMOID)
    # acc = -2048 -> floor(0 / 4096) = 0 -> plsig(0) = 2048;  acc = -2049 -> -1 -> plsig(-1)
    assert O.forward(pls, np.array([-2048], np.int16))[1][0] == 2048
    y_m1 = T[63] + (((int(T[64]) - int(T[63])) * 511 + 256) >> 9)
    assert O.forward(pls, np.array([-2049], np.int16))[1][0] == y_m1


def test_int8_requant_rounding(oracle_mod):
    """C18: y = min(255, max(0, (acc + 2^(sh-1)) >> sh)); hand-computed cases with sh = 3."""
    O = oracle_mod
    net = _net_i8([1, 1, 1], [[[1]], [[1]]], [[0], [0]], [3])
    for x, y in [(3, 0), (4, 1), (11, 1), (12, 2), (255, 32)]:
        assert O.forward(net, np.array([x], np.uint8))[1][0] == y
    net2 = _net_i8([1, 1, 1], [[[127]], [[1]]], [[0], [-5000]], [3])
    assert O.forward(net2, np.array([255], np.uint8))[1][0] == 255 - 5000      # 127*255>>3 clamps
    net3 = _net_i8([1, 1, 1], [[[-1]], [[1]]], [[0], [0]], [3])
    assert O.forward(net3, np.array([200], np.uint8))[1][0] == 0                # ReLU


def test_fixed_forward_vs_numpy(oracle_mod):
    """Library routine: numpy int64 matmul of every layer's contraction on random nets."""
    O = oracle_mod
    rng = np.random.default_rng(3)
    for trial in range(60):
        sizes = [int(rng.integers(1, 40)), int(rng.integers(1, 20)), int(rng.integers(1, 20)), int(rng.integers(1, 12))]
        if trial % 2 == 0:
            Ws = [rng.integers(-127, 128, (sizes[l + 1], sizes[l])) for l in range(3)]
            bs = [rng.integers(-20000, 20000, sizes[l + 1]) for l in range(3)]
            sh = [int(rng.integers(0, 8)), int(rng.integers(0, 8))]
            net = _net_i8(sizes, Ws, bs, sh)
            x = rng.integers(0, 256, sizes[0]).astype(np.uint8)
        else:
            Ws = [rng.integers(-6000, 6000, (sizes[l + 1], sizes[l])) for l in range(3)]
            bs = [rng.integers(-3000, 3000, sizes[l + 1]) << 12 for l in range(3)]
            net = _net_q(sizes, Ws, bs, M.ACT_PL_SIGMOID if trial % 4 == 1 else M.ACT_RELU)
            x = rng.integers(0, 4097, sizes[0]).astype(np.int16)
        t = O.forward(net, x)
        h = x.astype(np.int64)
        for l in range(3):
            acc = np.asarray(net.W[l], np.int64) @ h + np.asarray(net.b[l], np.int64)
            assert np.array_equal(t[l], acc.astype(np.float64))
            # feed the oracle's own next-layer input back through the rule pinned above
            if l < 2:
                if net.numeric == M.NUM_INT8:
                    s = net.requant_shift[l]
                    r = (1 << (s - 1)) if s > 0 else 0
                    h = np.clip((acc + r) >> s, 0, 255)
                else:
                    u16 = np.clip((acc + 2048) >> 12, -32768, 32767)
                    h = (np.array([O.plsig(net.sigmoid_knots, int(v)) for v in u16], np.int64)
                         if net.act == M.ACT_PL_SIGMOID else np.maximum(u16, 0))


# ----------------------------------------------------------------------------- float forward / bf16
def test_float_forward_vs_numpy(oracle_mod):
    """Library routine: numpy float64 matmul on the exact fp32 / bf16 operands (C19)."""
    O = oracle_mod
    cfg = M.make_config("cfg1")
    x = cfg.bases[0]
    t = O.forward(cfg.net, x)
    h = x.astype(np.float64)
    for l in range(2):
        u = cfg.net.W[l].astype(np.float64) @ h + cfg.net.b[l].astype(np.float64)
        assert np.allclose(t[l], u, rtol=1e-13, atol=1e-14)
        h = 1.0 / (1.0 + np.exp(-u))
    rng = np.random.default_rng(5)
    sizes = [33, 17, 9, 4]
    Wf = [rng.normal(0, 0.3, (sizes[l + 1], sizes[l])).astype(np.float32) for l in range(3)]
    net = Net(sizes, M.ACT_RELU, M.NUM_BF16, [M.f32_to_bf16_bits(w) for w in Wf],
              [rng.normal(0, 0.1, sizes[l + 1]).astype(np.float32) for l in range(3)], acc_scale=[1.0] * 3)
    xb = M.f32_to_bf16_bits(rng.random(33, dtype=np.float32))
    t = O.forward(net, xb)
    h = M.bf16_bits_to_f32(xb).astype(np.float64)
    for l in range(3):
        u = M.bf16_bits_to_f32(net.W[l]).astype(np.float64) @ h + net.b[l].astype(np.float64)
        assert np.allclose(t[l], u, rtol=1e-13, atol=1e-14)
        h = np.maximum(u, 0.0)


def test_bf16_rounding_vs_torch(oracle_mod):
    """Library routine: torch fp32 -> bf16 conversion (round to nearest even)."""
    torch = pytest.importorskip("torch")
    O = oracle_mod
    rng = np.random.default_rng(11)
    v = np.concatenate([rng.normal(0, 1, 4000), rng.uniform(-1e-3, 1e-3, 2000), rng.uniform(0, 1, 2000)]).astype(np.float32)
    # exact ties: bf16 value + half an ulp
    base = M.bf16_bits_to_f32(rng.integers(0x3C00, 0x3F80, 500).astype(np.uint16))
    ties = (base.view(np.uint32) + np.uint32(0x8000)).view(np.float32)
    v = np.concatenate([v, ties])
    ref = torch.from_numpy(v).to(torch.bfloat16).to(torch.float32).numpy()
    got = np.array([O.rne_bf16(float(a)) for a in v], dtype=np.float32)
    assert np.array_equal(got, ref)


# ----------------------------------------------------------------------------- decoders (C14)
def test_space_sizes(oracle_mod):
    O = oracle_mod
    assert O.space_size(M.make_config("cfg1").pert, 25) == math.comb(25, 2) * 256 == 76_800
    assert O.space_size(M.make_config("cfg2").pert, 25) == 5 ** 8 == 390_625
    assert O.space_size(M.make_config("cfg3").pert, 784) == 16 ** 6 == 16_777_216


def test_decode_special_indices(oracle_mod):
    O = oracle_mod
    c1 = M.make_config("cfg1")
    x = c1.bases[0]
    d0 = O.decode(M.NUM_FP32, c1.pert, x, 0, 0)
    assert d0[0] == 0.0 and d0[1] == 0.0 and np.array_equal(d0[2:], x[2:])
    dl = O.decode(M.NUM_FP32, c1.pert, x, 0, 76_799)
    assert dl[23] == 1.0 and dl[24] == 1.0 and np.array_equal(dl[:23], x[:23])
    c2 = M.make_config("cfg2")
    for b in range(c2.n_base):
        x = c2.bases[b]
        assert np.array_equal(O.decode(M.NUM_Q4_12, c2.pert, x, b, 195_312), x)   # all digits 2 -> offset 0
        d0 = O.decode(M.NUM_Q4_12, c2.pert, x, b, 0)
        dl = O.decode(M.NUM_Q4_12, c2.pert, x, b, 390_624)
        P = c2.pert.pixels
        assert np.array_equal(d0[P], np.clip(x[P].astype(int) - 410, 0, 4096))
        assert np.array_equal(dl[P], np.clip(x[P].astype(int) + 410, 0, 4096))
        mask = np.ones(25, bool); mask[P] = False
        assert np.array_equal(d0[mask], x[mask])
    c3 = M.make_config("cfg3")
    x = c3.bases[0]
    P = c3.pert.pixels
    assert np.all(O.decode(M.NUM_INT8, c3.pert, x, 0, 0)[P] == 0)
    assert np.all(O.decode(M.NUM_INT8, c3.pert, x, 0, 16 ** 6 - 1)[P] == 255)


def _enum_tuple(x, q_levels, n0):
    """itertools enumerator in the C14 order: pairs i<j (i outer), then (l_i, l_j)."""
    for i, j in itertools.combinations(range(n0), 2):
        for a, b in itertools.product(range(len(q_levels)), repeat=2):
            y = x.copy(); y[i] = q_levels[a]; y[j] = q_levels[b]
            yield y


def _enum_subset(x, pixels, levels, offset, lo, hi):
    for digs in itertools.product(range(len(levels)), repeat=len(pixels)):   # P[0] most significant
        y = x.copy()
        for p, d in zip(pixels, digs):
            y[p] = np.clip(int(x[p]) + int(levels[d]), lo, hi) if offset else levels[d]
        yield y


def test_decode_vs_itertools(oracle_mod):
    O = oracle_mod
    x = np.array([0.1, 0.2, 0.3, 0.4, 0.5, 0.6], np.float32)
    lv = np.array([0.0, 0.5, 1.0], np.float32)
    p = Pert(M.PERT_TUPLE_REPLACE, tuple=2, levels=lv)
    for idx, y in enumerate(_enum_tuple(x, lv, 6)):
        assert np.array_equal(O.decode(M.NUM_FP32, p, x, 0, idx), y)
    assert idx + 1 == O.space_size(p, 6)
    xi = np.array([0, 100, 4000, 4096, 2000, 7, 3000], np.int16)
    pix = np.array([1, 2, 5], np.int32)
    lv = np.array([-300, 0, 150, 500], np.int16)
    p = Pert(M.PERT_SUBSET_OFFSET, pixels=pix, levels=lv)
    for idx, y in enumerate(_enum_subset(xi, pix, lv, True, 0, 4096)):
        assert np.array_equal(O.decode(M.NUM_Q4_12, p, xi, 0, idx), y)
    xu = np.array([0, 100, 200, 255, 20, 7, 30], np.uint8)
    lv = np.array([0, 17, 255], np.int16)
    p = Pert(M.PERT_SUBSET_REPLACE, pixels=pix, levels=lv)
    for idx, y in enumerate(_enum_subset(xu, pix, lv, False, 0, 255)):
        assert np.array_equal(O.decode(M.NUM_INT8, p, xu, 0, idx), y)


def test_philox_lattice_values_and_uniformity(oracle_mod):
    """Every PHILOX_LATTICE pixel equals clamp(x + off_l) for one of the 16 offsets, with
    off_l = RNE_bf16(l*s + c) computed by torch (library rounding); levels are uniform (chi^2)."""
    torch = pytest.importorskip("torch")
    O = oracle_mod
    cfg = M.make_config("cfg4")
    s = float(M.bf16_bits_to_f32(M.f32_to_bf16_bits(np.float32(0.1 / 15.0)))[()])
    c = float(M.bf16_bits_to_f32(M.f32_to_bf16_bits(np.float32(-0.05)))[()])
    cfg.pert = Pert(M.PERT_PHILOX_LATTICE, seed=cfg.pert.seed, n_samples=2 ** 32, lattice_step=s, lattice_origin=c)
    offs = torch.tensor([l * s + c for l in range(16)], dtype=torch.float32).to(torch.bfloat16).to(torch.float32).numpy()
    # base pixels that are multiples of 2^-8 keep x + off exact in fp32
    x = (np.arange(784) % 257 / 256.0).astype(np.float32)
    xb = M.f32_to_bf16_bits(x)
    xv = M.bf16_bits_to_f32(xb)
    cand = torch.from_numpy(np.clip(xv[:, None] + offs[None, :], 0, 1).astype(np.float32)).to(torch.bfloat16).to(torch.float32).numpy()
    counts = np.zeros(16)
    for idx in range(40):
        y = M.bf16_bits_to_f32(O.decode(M.NUM_BF16, cfg.pert, xb, 3, idx))
        hit = (cand == y[:, None])
        assert np.all(hit.any(axis=1))
        # pixels away from the clamp bounds identify their level uniquely
        mid = (xv > 0.06) & (xv < 0.94)
        lv = np.argmax(hit[mid], axis=1)
        counts += np.bincount(lv, minlength=16)
    e = counts.sum() / 16
    chi2 = float(np.sum((counts - e) ** 2 / e))
    assert chi2 < 50.0                                   # 15 dof; p < 1e-4 at 44
    # u8 lattice: x + l*s + c clamped, here l - 8
    c5 = M.make_config("cfg5_int8")
    xb = c5.bases[0]
    y = O.decode(M.NUM_INT8, c5.pert, xb, 0, 5).astype(int)
    d = y - xb.astype(int)
    inner = (xb >= 8) & (xb <= 248)
    assert np.all((d[inner] >= -8) & (d[inner] <= 7))
    assert np.all((y >= 0) & (y <= 255))


def test_philox_box_values_and_linearity(oracle_mod):
    """PHILOX_BOX (reading C14b): every pixel moves by exactly origin + l*step for a level l in
    0..15 (the same levels as PHILOX_LATTICE: pixels away from the clamp bounds pick the same l
    in both spaces), |x' - x| <= eps, levels uniform (chi^2), and the layer-1 potentials of a
    candidate equal W1 x' + b1 by numpy's float64 matmul (library routine)."""
    O = oracle_mod
    cfg = M.make_config("cfg4_box")
    p = cfg.pert
    assert p.kind == M.PERT_PHILOX_BOX
    step, org = p.lattice_step, p.lattice_origin
    xb = cfg.bases[3]
    xv = M.bf16_bits_to_f32(xb).astype(np.float64)
    lat = Pert(M.PERT_PHILOX_LATTICE, seed=p.seed, n_samples=p.n_samples,
               lattice_step=float(M.bf16_bits_to_f32(M.f32_to_bf16_bits(np.float32(step)))[()]),
               lattice_origin=float(M.bf16_bits_to_f32(M.f32_to_bf16_bits(np.float32(org)))[()]))
    counts = np.zeros(16)
    W1 = M.bf16_bits_to_f32(cfg.net.W[0]).astype(np.float64)
    b1 = np.asarray(cfg.net.b[0], np.float64)
    for idx in (0, 1, 77, 2 ** 31 + 5, 2 ** 32 - 1):
        y = O.decode(cfg.net.numeric, p, xb, 3, idx)
        assert y.dtype == np.float64
        lv = (y - xv - org) / step
        li = np.rint(lv)
        assert np.all(np.abs(lv - li) < 1e-9) and li.min() >= 0 and li.max() <= 15
        assert np.max(np.abs(y - xv)) <= 0.05 + 1e-12
        counts += np.bincount(li.astype(int), minlength=16)
        # same levels as the clamped lattice where no clamping can happen
        yl = M.bf16_bits_to_f32(O.decode(cfg.net.numeric, lat, xb, 3, idx)).astype(np.float64)
        mid = (xv > 0.06) & (xv < 0.94)
        ol = np.array([float(M.bf16_bits_to_f32(M.f32_to_bf16_bits(np.float32(l * lat.lattice_step + lat.lattice_origin)))[()]) for l in range(16)])
        cand = M.bf16_bits_to_f32(M.f32_to_bf16_bits((xv[:, None] + ol[None, :]).astype(np.float32))).astype(np.float64)
        assert np.all(cand[mid, li[mid].astype(int)] == yl[mid])
        u1 = O.forward(cfg.net, y)[0]
        assert np.allclose(u1, W1 @ y + b1, rtol=1e-12, atol=1e-12)
    e = counts.sum() / 16
    assert float(np.sum((counts - e) ** 2 / e)) < 50.0


def test_philox_clamp_is_the_clipped_box(oracle_mod):
    """PHILOX_CLAMP (reading C14; "normalized", I in M^{mn} PAPER.md:438/454): each
    candidate is the PHILOX_BOX point (pinned above) clipped to [0, 1] by numpy (library routine):
    x'_p = x_p + origin + l_p step where that lies in [0, 1], else 0 / 1; so |x' - x| <= 7.5 step,
    every pixel in [0, 1], the zero lattice (step = origin = 0) reproduces the base, and the
    layer-1 potentials equal W1 x' + b1 by numpy's float64 matmul."""
    O = oracle_mod
    cfg = M.make_config("cfg4")
    p = cfg.pert
    assert p.kind == M.PERT_PHILOX_CLAMP and p.lattice_step == 109 * 2.0 ** -14 and p.lattice_origin == -7.5 * p.lattice_step
    box = M.make_config("cfg4_box").pert
    W1 = M.bf16_bits_to_f32(cfg.net.W[0]).astype(np.float64)
    b1 = np.asarray(cfg.net.b[0], np.float64)
    n_lo = n_hi = 0
    for bi in (3, 500):
        xb = cfg.bases[bi]
        xv = M.bf16_bits_to_f32(xb).astype(np.float64)
        for idx in (0, 1, 77, 2 ** 31 + 5, 2 ** 32 - 1):
            y = O.decode(cfg.net.numeric, p, xb, bi, idx)
            yb = O.decode(cfg.net.numeric, box, xb, bi, idx)
            assert y.dtype == np.float64 and np.array_equal(y, np.clip(yb, 0.0, 1.0))
            assert y.min() >= 0.0 and y.max() <= 1.0 and np.max(np.abs(y - xv)) <= 7.5 * p.lattice_step
            n_lo += int(np.sum(yb < 0)); n_hi += int(np.sum(yb > 1))
            u1 = O.forward(cfg.net, y)[0]
            assert np.allclose(u1, W1 @ y + b1, rtol=1e-12, atol=1e-12)
        z = Pert(M.PERT_PHILOX_CLAMP, seed=p.seed, n_samples=p.n_samples, lattice_step=0.0, lattice_origin=0.0)
        assert np.array_equal(O.decode(cfg.net.numeric, z, xb, bi, 12345), xv)
    assert n_lo > 1000 and n_hi > 0                       # both bounds are exercised on cfg4's bases


def _clamp_net_cfg():
    """n_0 = 2 (pixel 0 takes nibble 0 of Philox word 0), hidden u = (x0', -x0', x0' - 1) ReLU, logits
    y0 = 0.995, y1 = 1000 (h1 + h2), y2 = 1.97 - h0.  With the clamp h1 = h2 = 0, so y1 = 0.
    Base A, x0 = 253/256: class 0; violated iff x0' < 0.975, i.e. origin + l step < -0.0133, l <= 5.
    Base B, x0 = bf16(0.01): class 2; never violated.  A candidate outside [0, 1] would light y1:
    without the upper clamp A gains the l >= 10 candidates, without the lower one B gains l <= 5."""
    f = np.float32
    W = [M.f32_to_bf16_bits(np.array([[1, 0], [-1, 0], [1, 0]], f)),
         M.f32_to_bf16_bits(np.array([[0, 0, 0], [0, 1000, 1000], [-1, 0, 0]], f))]
    b = [np.array([0, 0, -1], f), np.array([0.995, 0, 1.97], f)]
    net = Net([2, 3, 3], M.ACT_RELU, M.NUM_BF16, W, b, acc_scale=[1.0, 1.0])
    bases = M.f32_to_bf16_bits(np.array([[253 / 256, 0.5], [0.01, 0.5]], f))
    step, origin = M.cfg4_lattice(0.05)
    pert = Pert(M.PERT_PHILOX_CLAMP, seed=0x1234_5678_9ABC_DEF0, n_samples=2 ** 32, lattice_step=step,
                lattice_origin=origin, index_begin=1000, index_end=3000)
    return Config("clampnet", "clamp closed form", net, bases, pert, Prop(), CovSpec([1]))


def test_clamp_net_closed_form(oracle_mod):
    """The check on PHILOX_CLAMP against levels read straight off the Philox stream: violations of
    base A = #{c : l_0(c) <= 5}, first counterexample the first such c, base B none (C14/C15)."""
    O = oracle_mod
    cfg = _clamp_net_cfg()
    r = O.check(cfg)
    key = [cfg.pert.seed & 0xFFFFFFFF, cfg.pert.seed >> 32]
    lv = np.array([int(O.philox([c, 0, 0, 0], key)[0]) & 15 for c in range(1000, 3000)])
    hits = np.nonzero(lv <= 5)[0]
    assert int(r.checked[0]) == 2000 and int(r.violated[0]) == len(hits) and int(r.first_cex[0]) == 1000 + hits[0]
    assert int(r.violated[1]) == 0 and int(r.flagged.sum()) == 0
    assert 2000 * 6 / 16 - 150 < len(hits) < 2000 * 6 / 16 + 150


def test_restriction_on_philox_clamp_closed_form(oracle_mod):
    """Restriction R on a Philox space (reading C27): base (0.5, 0.5), no clamping, so
    delta^2 = step^2 ((l_0 - 7.5)^2 + (l_1 - 7.5)^2) with the two levels read straight off the Philox
    stream; checked = #{c : that <= b^2}.  Also b -> large keeps all, and counts grow with b."""
    O = oracle_mod
    cfg = _clamp_net_cfg()
    cfg.bases = M.f32_to_bf16_bits(np.array([[0.5, 0.5]], np.float32))
    step = cfg.pert.lattice_step
    key = [cfg.pert.seed & 0xFFFFFFFF, cfg.pert.seed >> 32]
    lv = np.array([[int(O.philox([c, 0, 0, 0], key)[0]) >> (4 * n) & 15 for n in (0, 1)] for c in range(1000, 3000)])
    r2 = ((lv - 7.5) ** 2).sum(axis=1) * step * step
    prev = -1
    for b in (0.01, 0.03, 0.05, 0.07, 1.0):
        cfg.pert.restrict_l2 = b
        n = int(O.check(cfg).checked[0])
        assert n == int(np.sum(r2 <= b * b)), b
        assert n >= prev
        prev = n
    assert prev == 2000


def test_philox_is_counter_sensitive(oracle_mod):
    """Distinct counters / keys give distinct outputs; the same inputs give the same outputs."""
    O = oracle_mod
    a = O.philox([0, 0, 0, 0], [0, 0])
    assert np.array_equal(a, O.philox([0, 0, 0, 0], [0, 0]))
    outs = {tuple(O.philox([i, 0, 0, 0], [1, 2])) for i in range(256)}
    outs |= {tuple(O.philox([0, 0, i, 0], [1, 2])) for i in range(1, 256)}
    outs |= {tuple(O.philox([0, 0, 0, 0], [i, 2])) for i in range(256)}
    assert len(outs) == 256 + 255 + 256 - 1 or len(outs) >= 765
    bits = np.unpackbits(np.array([O.philox([i, 7, 9, 1], [3, 4]) for i in range(512)], np.uint32).view(np.uint8))
    assert abs(bits.mean() - 0.5) < 0.02


# ----------------------------------------------------------------------------- whole-check pins
def _threshold_cfg(numeric, q, levels):
    """After SPEC.md:392 / SURVEY §8(c): 2-2-2 ReLU net with logits (1, p0 + p1); base (0.4, 0.4)."""
    if numeric == M.NUM_Q4_12:
        net = _net_q([2, 2, 2], [[[4096, 4096], [0, 0]], [[0, 4096], [4096, 0]]], [[0, 1 << 24], [0, 0]])
        base = np.array([[1638, 1638]], np.int16)
    else:
        net = Net([2, 2, 2], M.ACT_RELU, M.NUM_FP32, [np.array([[1, 1], [0, 0]], np.float32),
                  np.array([[0, 1], [1, 0]], np.float32)], [np.array([0, 1], np.float32),
                  np.array([0, 0], np.float32)], acc_scale=[1.0, 1.0])
        base = np.array([[0.4, 0.4]], np.float32)
    pert = Pert(M.PERT_TUPLE_REPLACE, tuple=2, levels=levels)
    pert.index_end = pert.space_size(2)
    return Config("thr", "threshold net", net, base, pert, Prop(), CovSpec([1]))


def test_threshold_net_fixed(oracle_mod):
    """Violations = #{a+b > q-1} = q(q-1)/2 = 10 of 25 for q = 5; exact ties a+b = q-1 go to class 0;
    first counterexample c = a*q + b with (a, b) = (1, 4) -> 9.  Only VV column 1 (logit p0+p1)."""
    O = oracle_mod
    cfg = _threshold_cfg(M.NUM_Q4_12, 5, np.array([1024 * l for l in range(5)], np.int16))
    r = O.check(cfg)
    assert int(r.checked[0]) == 25 and int(r.violated[0]) == 10 and int(r.first_cex[0]) == 9
    assert _pairs_of(O, [2, 2, 2], [1], r.cov_all) == {("VV", 1, None, 1)}


def test_threshold_net_float(oracle_mod):
    """Same net on fp32: dyadic levels l/4 give exact ties (margin 0) -> 5 flagged non-violations;
    levels l/15 (q = 16): the 16 candidates with a+b = 15 are near-ties and flagged (C20); 120
    candidates with a+b > 15 are unflagged violations; the first is (1, 15) -> 31."""
    O = oracle_mod
    r = O.check(_threshold_cfg(M.NUM_FP32, 5, np.array([l / 4 for l in range(5)], np.float32)))
    assert int(r.violated[0]) == 10 and int(r.flagged[0]) == 5 and int(r.first_cex[0]) == 9
    r = O.check(_threshold_cfg(M.NUM_FP32, 16, np.array([l / 15 for l in range(16)], np.float32)))
    assert int(r.flagged[0]) == 16
    assert 120 <= int(r.violated[0]) <= 136
    assert int(r.first_cex_unflagged[0]) == 31


def _stress_cfg2():
    """cfg2 with a sharper output layer and eps = 0.5 so verdicts and coverage are non-trivial."""
    cfg = M.make_config("cfg2").subset(n_base=3)
    net = cfg.net
    cfg.net = Net(net.sizes, net.act, net.numeric, [np.clip(net.W[0].astype(int) * 4, -32768, 32767).astype(np.int16),
                                                    np.clip(net.W[1].astype(int) * 16, -32768, 32767).astype(np.int16)],
                  net.b, sigmoid_knots=net.sigmoid_knots, acc_scale=net.acc_scale)
    cfg.pert = Pert(M.PERT_SUBSET_OFFSET, pixels=cfg.pert.pixels,
                    levels=np.array([-2048, -1024, 0, 1024, 2048], np.int16), index_begin=0, index_end=390_625)
    return cfg


def test_check_invariants(oracle_mod):
    """checked = range length; sub-range merge = one run (sum / min / OR); coverage monotone in the
    index set; the zero perturbation reproduces the base trace; counterexamples re-evaluate to
    misclassifications (SURVEY §8(c) invariants)."""
    O = oracle_mod
    cfg = _stress_cfg2()
    full = O.check(cfg)
    assert np.all(full.checked == 390_625)
    assert full.violated.sum() > 0 and np.unpackbits(full.cov_all.view(np.uint8)).sum() > 0
    a = O.check(cfg.subset(begin=0, end=123_457))
    b = O.check(cfg.subset(begin=123_457, end=390_625))
    assert np.array_equal(a.checked + b.checked, full.checked)
    assert np.array_equal(a.violated + b.violated, full.violated)
    assert np.array_equal(np.minimum(a.first_cex, b.first_cex), full.first_cex)
    assert np.array_equal(a.cov_all | b.cov_all, full.cov_all)
    assert np.array_equal(a.cov_all & ~full.cov_all, np.zeros_like(a.cov_all))
    e = O.check(cfg.subset(begin=77, end=77))
    assert np.all(e.checked == 0) and np.all(e.first_cex == np.iinfo(np.uint64).max) and not e.cov_all.any()
    for bi in range(cfg.n_base):
        x = cfg.bases[bi]
        tb = O.forward(cfg.net, x)
        z = O.decode(cfg.net.numeric, cfg.pert, x, bi, 195_312)
        assert all(np.array_equal(u, v) for u, v in zip(tb, O.forward(cfg.net, z)))
        if full.first_cex[bi] != np.iinfo(np.uint64).max:
            y = O.decode(cfg.net.numeric, cfg.pert, x, bi, int(full.first_cex[bi]))
            assert int(np.argmax(O.forward(cfg.net, y)[-1])) != int(np.argmax(tb[-1]))
            # and nothing below it is a violation
            lo = O.check(cfg.subset(n_base=1, base_start=bi, begin=0, end=int(full.first_cex[bi])))
            assert int(lo.violated[0]) == 0


def test_target_never_closed_form(oracle_mod):
    """TARGET_NEVER (C12, PAPER.md:466-479 with a target class): on the q = 5 threshold net class 1
    iff a + b > 4 (ties to class 0), so t = 0 is violated by the 15 pairs with a + b <= 4, first at
    c = 0, and t = 1 by the other 10, first at (1, 4) -> 9 -- unlike ARGMAX_UNCHANGED, t = 0 is
    violated by the base class itself.  Float (levels l/4, exact): the 5 ties a + b = 4 are flagged."""
    O = oracle_mod
    for numeric, levels in ((M.NUM_Q4_12, np.array([1024 * l for l in range(5)], np.int16)),
                            (M.NUM_FP32, np.array([l / 4 for l in range(5)], np.float32))):
        for t, nv, first in ((0, 15, 0), (1, 10, 9)):
            cfg = _threshold_cfg(numeric, 5, levels)
            cfg.prop = Prop(M.PROP_TARGET_NEVER, t, 0.0)
            r = O.check(cfg)
            assert int(r.violated[0]) == nv and int(r.first_cex[0]) == first, (numeric, t)
            assert int(r.flagged[0]) == (5 if numeric == M.NUM_FP32 else 0)


def test_ambiguity_rules_inside_outside(oracle_mod):
    """Reading C20, one rule at a time on a hand-built trace pair for pair (1, 2), tau = 0.01,
    d = 0.1: a sign predicate with |u| < tau, a value predicate with ||du| - d| < tau and a
    distance predicate (no layer-1 sign change) with |Linf - d| < tau make the pair uncertain;
    the same traces with the quantity at 2 tau from the boundary are certain.  The covered words
    do not depend on tau."""
    O = oracle_mod
    sizes, tau, d = [2, 2, 2], [0.01, 0.01], 0.1

    def run(t1, t2):
        w, cert = O.cover_traces_tau(sizes, [np.array(x, float) for x in t1], [np.array(x, float) for x in t2],
                                     [1], [d, d], [d, d], tau)
        w0 = O.cover_traces(sizes, [np.array(x, float) for x in t1], [np.array(x, float) for x in t2], [1], [d, d], [d, d])
        assert np.array_equal(w, w0)
        return bool(cert[0])

    base = ([1.0, 2.0], [1.0, -1.0])
    # everything far from every boundary: layer-1 Linf 0.5, layer-2 |du| = 0.5, no sign changes
    assert run(base, ([1.5, 2.0], [1.5, -1.5]))
    # sign: a layer-2 potential of the candidate at 0.005 (inside) / 0.02 (outside)
    assert not run(base, ([1.5, 2.0], [0.005, -1.5]))
    assert run(base, ([1.5, 2.0], [0.02, -1.5]))
    # sign on layer 1 (the lower layer of the pair), and on the base trace
    assert not run(base, ([-0.005, 2.0], [1.5, -1.5]))
    assert not run(([0.005, 2.0], [1.0, -1.0]), ([1.5, 2.0], [1.5, -1.5]))
    # value: layer-2 |du| = 0.105 (inside) / 0.12 (outside) of d = 0.1
    assert not run(base, ([1.5, 2.0], [1.105, -1.5]))
    assert run(base, ([1.5, 2.0], [1.12, -1.5]))
    # distance: layer-1 Linf = 0.095 (inside) / 0.08 (outside), no sign change in layer 1
    assert not run(base, ([1.095, 2.0], [1.5, -1.5]))
    assert run(base, ([1.08, 2.0], [1.5, -1.5]))
    # the distance rule applies only without a layer-1 sign change
    assert run(([1.0, 2.0], [1.0, -1.0]), ([-1.0, 2.095], [1.5, -1.5]))


def test_default_tau_closed_form(oracle_mod):
    """C20: tau_l = 1e-6 + 1e-5 max over the bases of max |u_l^base|; on W1 = I, W2 = 2 I (fp32,
    zero biases, ReLU) the base potentials are u1 = x, u2 = 2 ReLU(x)."""
    O = oracle_mod
    net = Net([2, 2, 2], M.ACT_RELU, M.NUM_FP32, [np.eye(2, dtype=np.float32), 2 * np.eye(2, dtype=np.float32)],
              [np.zeros(2, np.float32), np.zeros(2, np.float32)], acc_scale=[1.0, 1.0])
    bases = np.array([[0.5, -0.75], [0.25, 0.375]], np.float32)
    cfg = Config("tau", "tau", net, bases, Pert(M.PERT_TUPLE_REPLACE, tuple=1, levels=np.zeros(1, np.float32)),
                 Prop(), CovSpec([1]))
    t = O.default_tau(cfg)
    assert np.allclose(t, [1e-6 + 1e-5 * 0.75, 1e-6 + 1e-5 * 1.0], rtol=0, atol=1e-15)


def _literal_cfg(numeric, prop_kind):
    """2-2-3 ReLU net: identity hidden layer, logits y0 = 0.45 (bias), y1 = h0, y2 = h1; base (0, 0)
    -> class 0; both pixels replaced by l/4, l = 0..4 (25 candidates, c = 5 l0 + l1)."""
    if numeric == M.NUM_Q4_12:
        W = [np.array([[4096, 0], [0, 4096]], np.int16), np.array([[0, 0], [4096, 0], [0, 4096]], np.int16)]
        b = [np.zeros(2, np.int32), np.array([int(0.45 * 4096) << 12, 0, 0], np.int32)]
        net = Net([2, 2, 3], M.ACT_RELU, M.NUM_Q4_12, W, b, acc_scale=[2.0 ** -24] * 2)
        base, levels, V = np.zeros((1, 2), np.int16), np.array([1024 * l for l in range(5)], np.int16), 0.5
    else:
        W = [np.eye(2, dtype=np.float32), np.array([[0, 0], [1, 0], [0, 1]], np.float32)]
        b = [np.zeros(2, np.float32), np.array([0.45, 0, 0], np.float32)]
        net = Net([2, 2, 3], M.ACT_RELU, M.NUM_FP32, W, b, acc_scale=[1.0, 1.0])
        base, levels, V = np.zeros((1, 2), np.float32), np.array([l / 4 for l in range(5)], np.float32), 0.5
    pert = Pert(M.PERT_TUPLE_REPLACE, tuple=2, levels=levels)
    pert.index_end = pert.space_size(2)
    return Config("lit", "literal net", net, base, pert, Prop(prop_kind, 0, V), CovSpec([1]))


def test_literal_readings(oracle_mod):
    """l_image_misclassified with D = 0, V = 0.5 and y_D = 0.45 < V always:
    existential reading (C12) violated iff l0 > 2 or l1 > 2 -> 25 - 9 = 16, first c = 3;
    universal reading (NEXT-4) iff l0 > 2 and l1 > 2 -> 4, first c = 18.  Float: the 9
    candidates with a logit exactly at V (l = 2) are flagged; Q4.12: exact, nothing flagged."""
    O = oracle_mod
    for numeric in (M.NUM_FP32, M.NUM_Q4_12):
        r_any = O.check(_literal_cfg(numeric, M.PROP_THRESHOLD_LITERAL))
        r_all = O.check(_literal_cfg(numeric, M.PROP_THRESHOLD_LITERAL_ALL))
        assert int(r_any.violated[0]) == 16 and int(r_any.first_cex[0]) == 3
        assert int(r_all.violated[0]) == 4 and int(r_all.first_cex[0]) == 18
        nflag = 9 if numeric == M.NUM_FP32 else 0
        assert int(r_any.flagged[0]) == nflag and int(r_all.flagged[0]) == nflag


def _restrict_cfg(b):
    """Binary 5x5 images: base all 0, six pixels each replaced by 0 or 1 (Q4.12 raw 0 / 4096), so the
    candidate with k ones lies at L2 distance sqrt(k) from the base (delta(A, O) =
    sqrt(6) = 2.449 for images differing in 6 pixels)."""
    cfg = M.make_config("cfg2").subset(n_base=1)
    cfg.bases = np.zeros((1, 25), np.int16)
    cfg.pert = Pert(M.PERT_SUBSET_REPLACE, pixels=np.array([0, 3, 7, 12, 18, 24], np.int32),
                    levels=np.array([0, 4096], np.int16), index_begin=0, index_end=64, restrict_l2=b)
    return cfg


def test_restriction_distances(oracle_mod):
    """Restriction R (reading C27): checked = #{k <= b^2} candidates; b = 2 -> C(6,0..4) = 57,
    b = 2.449 (< sqrt 6) -> 63, b = 2.4495 (> sqrt 6) -> 64, b = 0.99 -> only the base; b = 0 means
    no restriction.  The double sqrt(6) squares to 5.999999999999999 < 6, so floor(b^2 4096^2) is
    one below 6 * 4096^2 and the k = 6 candidate stays outside."""
    O = oracle_mod
    for b, n in ((2.0, 57), (2.449, 63), (math.sqrt(6.0), 63), (2.4495, 64), (3.0, 64), (0.99, 1), (0.0, 64)):
        assert int(O.check(_restrict_cfg(b)).checked[0]) == n, b


def test_restriction_monotone(oracle_mod):
    """Violations, checked counts and coverage grow with the bound."""
    O = oracle_mod
    cfg = _stress_cfg2()
    cfg = cfg.subset(n_base=2, begin=0, end=60_000)
    prev = None
    for b in (0.05, 0.1, 0.2, 0.3, 0.45, 0.7):
        c = cfg.subset(n_base=2, begin=0, end=60_000)
        c.pert = c.pert.with_range(0, 60_000)
        c.pert.restrict_l2 = b
        r = O.check(c)
        if prev is not None:
            assert np.all(r.checked >= prev.checked) and np.all(r.violated >= prev.violated)
            assert not np.any(prev.cov_all & ~r.cov_all)
        prev = r
    assert int(prev.violated.sum()) > 0


# ------------------------------------------------ dataset-pair coverage (NEXT-3)
def _pc_pairs(numeric):
    net = M.vowel_net(numeric)
    return net, M.pair_images(net, 7, seed=1)


@pytest.mark.parametrize("numeric", [M.NUM_Q4_12, M.NUM_FP32])
def test_pair_coverage_is_or_over_unordered_pairs(oracle_mod, numeric):
    """The set-level covers of Eqs. sscover..dvcover are the OR of the two-image covers over all
    unordered pairs (the covers are symmetric in x1, x2): an explicit double loop over
    cover_traces, with thresholds converted to trace units here (d / 2^-24 for Q4.12)."""
    O = oracle_mod
    net, imgs = _pc_pairs(numeric)
    pairs, d = [1, 2], 0.08
    scale = 1.0 if numeric == M.NUM_FP32 else 2.0 ** 24
    tr = [O.forward(net, x) for x in imgs]
    want = None
    for a in range(len(imgs)):
        for b in range(len(imgs)):
            if a == b:
                continue                            # ordered pairs: symmetry must make b<a redundant
            w = O.cover_traces(net.sizes, tr[a], tr[b], pairs, [d * scale] * 3, [d * scale] * 3)
            want = w if want is None else want | w
    got, cert = O.pair_coverage(net, imgs, pairs, d, d)
    assert np.array_equal(got, want)
    assert got.any()
    assert not np.any(cert & ~got)
    if numeric == M.NUM_Q4_12:
        assert np.array_equal(cert, got)           # fixed point: exact, nothing ambiguous


def test_pair_coverage_set_invariants(oracle_mod):
    """Order of the images is irrelevant; adding an image only adds covered pairs; one image
    covers nothing."""
    O = oracle_mod
    net, imgs = _pc_pairs(M.NUM_Q4_12)
    full, _ = O.pair_coverage(net, imgs, [1, 2], 0.1, 0.1)
    perm, _ = O.pair_coverage(net, imgs[::-1].copy(), [1, 2], 0.1, 0.1)
    assert np.array_equal(full, perm)
    part, _ = O.pair_coverage(net, imgs[:4], [1, 2], 0.1, 0.1)
    assert not np.any(part & ~full) and part.sum() <= full.sum()
    one, _ = O.pair_coverage(net, imgs[:1], [1, 2], 0.1, 0.1)
    assert not one.any()


def test_pair_coverage_duplicates_closed_form(oracle_mod):
    """Two copies of one image: no sign change anywhere, all distances 0.  With d_h = d_g = 0 the
    DS premise holds and every upper neuron is value-changed by 0 >= 0, so
    exactly the DV columns are full and SS / SV / DS are empty; with d > 0 nothing is covered."""
    O = oracle_mod
    net, imgs = _pc_pairs(M.NUM_Q4_12)
    two = np.stack([imgs[2], imgs[2]])
    w0, _ = O.pair_coverage(net, two, [1, 2], 0.0, 0.0)
    sets = _pairs_of(O, net.sizes, [1, 2], w0)
    assert sets == {("VV", k, None, j) for k in (1, 2) for j in range(net.sizes[k + 1])}
    w1, _ = O.pair_coverage(net, two, [1, 2], 0.01, 0.01)
    assert not w1.any()


def test_pair_coverage_certainty_widths(oracle_mod):
    """Float certainty (reading C20): tau = 0 makes every pair certain; a tau above every |u|
    makes none certain."""
    O = oracle_mod
    net, imgs = _pc_pairs(M.NUM_FP32)
    a0, c0 = O.pair_coverage(net, imgs, [1, 2], 0.08, 0.08, tau=[0.0] * 3)
    assert np.array_equal(a0, c0)
    a1, c1 = O.pair_coverage(net, imgs, [1, 2], 0.08, 0.08, tau=[1e9] * 3)
    assert np.array_equal(a0, a1) and not c1.any()


# ------------------------------------------ incremental bounds (NEXT-2, C28)
def _flip_cfg(levels=(0.15, 0.275, 0.4, 0.525, 0.65)):
    """SPEC.md's hand-built 2-pixel threshold net: class flips when pixel0 + pixel1 > 1.  2-2-2
    ReLU, identity hidden layer, y0 = 1 - h0 - h1, y1 = 0; I^d = (0.4, 0.4) (class 0); both pixels
    take the q = 5 levels of [I^d - r, I^d + r], r = 0.25 (c = 5 d0 + d1)."""
    W = [np.eye(2, dtype=np.float32), np.array([[-1, -1], [0, 0]], np.float32)]
    b = [np.zeros(2, np.float32), np.array([1, 0], np.float32)]
    net = Net([2, 2, 2], M.ACT_RELU, M.NUM_FP32, W, b, acc_scale=[1.0, 1.0])
    pert = Pert(M.PERT_SUBSET_REPLACE, pixels=np.array([0, 1], np.int32), levels=np.array(levels, np.float32))
    pert.index_end = pert.space_size(2)
    return Config("thr", "threshold net", net, np.array([[0.4, 0.4]], np.float32), pert, Prop(), CovSpec([]))


def test_incremental_schedule_closed_form(oracle_mod):
    """b_i = i g gamma / max_bound, the last one exactly gamma; ceil(max_bound / g) steps
    (SPEC.md completeness_phase: first complete at the smallest i with b_i >= gamma)."""
    O = oracle_mod
    assert O.incremental_schedule(0.5, 10, 1)[-1] == 0.5 and len(O.incremental_schedule(0.5, 10, 1)) == 10
    b = O.incremental_schedule(0.5, 10, 3)
    assert len(b) == 4 and b[-1] == 0.5 and b[:3] == pytest.approx([0.15, 0.3, 0.45], abs=1e-15)
    assert O.incremental_schedule(1.0, 1, 7) == [1.0]


def test_incremental_threshold_net(oracle_mod):
    """Nearest grid counterexamples (brute force over the 25 points): (0.525, 0.525) at
    sqrt(2)/8 = 0.177 (c = 18), then (0.4, 0.65) / (0.65, 0.4) at 0.25 (c = 14 / 22).
    gamma = 0.5, Delta = 0.05: g = 1 finds c = 18 at step 4 (b = 0.2, the smallest ball holding
    0.177); g = 2 at step 2 (b = 0.2), the same; g = 3 at step 2 (b = 0.3), where c = 14 at
    distance 0.25 is the lowest index -- not the nearest one.  gamma = 0.17:
    none after all 10 steps.  q = 2, r = 0 (both levels = I^d): only I^d, none."""
    O = oracle_mod
    cfg = _flip_cfg()
    # brute force of the nearest flipping grid point
    lv = np.array(cfg.pert.levels, np.float64)
    d = min(math.hypot(lv[i] - np.float32(0.4), lv[j] - np.float32(0.4)) for i in range(5) for j in range(5)
            if np.float32(lv[i]) + np.float32(lv[j]) > 1)
    assert d == pytest.approx(math.sqrt(2) / 8, abs=1e-6)
    r = O.incremental_verify(cfg, 0.5, 10, 1)
    assert (int(r["step"][0]), int(r["first_cex"][0]), r["iterations"]) == (4, 18, 4)
    r = O.incremental_verify(cfg, 0.5, 10, 2)
    assert (int(r["step"][0]), int(r["first_cex"][0])) == (2, 18)
    r = O.incremental_verify(cfg, 0.5, 10, 3)
    assert (int(r["step"][0]), int(r["first_cex"][0])) == (2, 14)
    r = O.incremental_verify(cfg, 0.17, 10, 1)
    assert int(r["step"][0]) == 0 and r["iterations"] == 10
    r = O.incremental_verify(_flip_cfg((0.4, 0.4)), 0.5, 10, 1)
    assert int(r["step"][0]) == 0


def test_incremental_final_ball_counts(oracle_mod):
    """The counts of the ball the loop stopped at (what the early-exit mode reports): brute force
    over the 25 grid points of the threshold net.  g = 1 stops at b_4 = 0.2: the points with
    offsets a^2 + b^2 <= 0.04 are (0,0), the four (+-0.125, 0) / (0, +-0.125) and the four
    (+-0.125, +-0.125) = 9, of which only (0.525, 0.525) (c = 18) flips; gamma = 0.17 never
    decides and stops at b_10 = 0.17: the same 9 points minus the diagonal ones (0.177 > 0.17) = 5,
    none violated."""
    O = oracle_mod
    cfg = _flip_cfg()
    lv = np.array(cfg.pert.levels, np.float32).astype(np.float64)
    x = float(np.float32(0.4))

    def brute(bound):
        pts = [(i, j) for i in range(5) for j in range(5) if (lv[i] - x) ** 2 + (lv[j] - x) ** 2 <= bound * bound]
        return len(pts), sum(1 for i, j in pts if np.float32(lv[i]) + np.float32(lv[j]) > 1)

    r = O.incremental_verify(cfg, 0.5, 10, 1)
    assert brute(0.2) == (9, 1)
    assert (int(r["final"]["checked"][0]), int(r["final"]["violated"][0])) == (9, 1)
    r = O.incremental_verify(cfg, 0.17, 10, 1)
    assert brute(0.17) == (5, 0)
    assert (int(r["final"]["checked"][0]), int(r["final"]["violated"][0])) == (5, 0)
