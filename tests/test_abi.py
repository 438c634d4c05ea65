"""C-ABI library checks that need no GPU: it loads, exports every symbol include/mlpv.h
declares, validates arguments synchronously, and its host decoder agrees with the oracle."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import mlpv_inputs as M

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def P():
    from paper_1907_12933_b200 import build
    build.build()
    import paper_1907_12933_b200 as P
    return P


def _declared():
    src = open(os.path.join(ROOT, "include", "mlpv.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mlpv_[a-z_]+)\s*\(", src)))


def test_exports_every_declared_symbol(P):
    names = _declared()
    assert set(names) >= {"mlpv_create", "mlpv_check", "mlpv_eval", "mlpv_decode", "mlpv_merge"}
    lib = C.CDLL(P.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), n
    assert set(P.EXPORTS) == set(names)
    assert "sm_100a" in P.version()


def test_library_is_sm100a(P):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", P.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def _create(P, net):
    try:
        P.Checker(net)
    except P.MlpvError as e:
        return e.status, str(e)
    return 0, ""


def test_create_validation_is_synchronous(P):
    c = M.make_config("cfg2").net
    bad_layers = M.configs.Net([25], c.act, c.numeric, [], [], sigmoid_knots=c.sigmoid_knots)
    assert _create(P, bad_layers)[0] == 1                                      # E_INVALID
    big = M.configs.Net([4, 17], M.ACT_RELU, M.NUM_FP32, [np.zeros((17, 4), np.float32)], [np.zeros(17, np.float32)])
    assert _create(P, big)[0] == 2                                             # E_SHAPE
    sig = M.configs.Net([4, 3, 2], M.ACT_SIGMOID, M.NUM_BF16, [np.zeros((3, 4), np.uint16), np.zeros((2, 3), np.uint16)],
                        [np.zeros(3, np.float32), np.zeros(2, np.float32)])
    assert _create(P, sig)[0] == 3                                             # E_UNSUPPORTED
    ov = M.configs.Net([16, 2], M.ACT_RELU, M.NUM_Q4_12, [np.full((2, 16), 32767, np.int16)], [np.zeros(2, np.int32)],
                       acc_scale=[2.0 ** -24])
    s, msg = _create(P, ov)
    assert s == 4 and "2^30" in msg                                             # E_OVERFLOW
    nan = M.configs.Net([2, 2], M.ACT_RELU, M.NUM_FP32, [np.array([[1, np.nan], [0, 0]], np.float32)], [np.zeros(2, np.float32)])
    s, msg = _create(P, nan)
    assert s == 1 and "finite" in msg
    # BF16: hidden activations travel as fp16 hi / lo; a net whose worst case leaves that range
    big = M.configs.Net([64, 8, 2], M.ACT_RELU, M.NUM_BF16,
                        [M.f32_to_bf16_bits(np.full((8, 64), 600.0, np.float32)), np.zeros((2, 8), np.uint16)],
                        [np.zeros(8, np.float32), np.zeros(2, np.float32)])
    s, msg = _create(P, big)
    assert s == 3 and "fp16" in msg


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3", "cfg4", "cfg4_box", "cfg5_int8"])
def test_host_decoder_matches_oracle(P, name, oracle_mod):
    cfg = M.make_config(name)
    rng = np.random.default_rng(1)
    idx = list(rng.integers(0, cfg.space, 40)) + [0, cfg.space - 1]
    for b in (0, cfg.n_base - 1):
        for i in idx:
            g = P.decode(cfg.net.numeric, cfg.pert, cfg.bases[b], b, int(i))
            o = oracle_mod.decode(cfg.net.numeric, cfg.pert, cfg.bases[b], b, int(i))
            assert np.array_equal(g, o), (name, b, i)
