"""Python face of the CPU oracle (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / ``--impl reference`` leg may
import this module.  It loads ``oracle/liboracle.so`` (plain C, built by ``build_oracle()`` with
gcc) and never touches the CUDA path.  Neuron-coverage post-processing (the
l_covered_neuron literals) is written here in plain Python over the oracle's pair bitmaps.

Parity status per function: every entry point is pinned by
tests/test_oracle_pins.py, except the synthetic configs' actual verdicts/coverage (no closed form:
pinned only through the pinned pieces; SURVEY.md §8(c) "Unpinned").
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass
from typing import List, Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.environ.get("MLPV_ORACLE_SRC", os.path.join(HERE, "mlpv_oracle.c"))
LIB = os.environ.get("MLPV_ORACLE_LIB", os.path.join(HERE, "liboracle.so"))


def build_oracle(force: bool = False) -> str:
    """gcc -O2 -fopenmp: plain loops, no intrinsics, no BLAS."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        tmp = LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                               "-o", tmp, SRC, "-lm"])
        os.replace(tmp, LIB)
    return LIB


class _Net(C.Structure):
    _fields_ = [("L", C.c_int32), ("sizes", C.POINTER(C.c_int32)), ("numeric", C.c_int32),
                ("act", C.c_int32), ("W", C.POINTER(C.c_void_p)), ("b", C.POINTER(C.c_void_p)),
                ("shift", C.POINTER(C.c_int32)), ("knots", C.POINTER(C.c_int16)),
                ("acc_scale", C.POINTER(C.c_double))]


class _Pert(C.Structure):
    _fields_ = [("kind", C.c_int32), ("tuple", C.c_int32), ("n_pixels", C.c_int32),
                ("pixels", C.POINTER(C.c_int32)), ("n_levels", C.c_int32), ("levels", C.c_void_p),
                ("seed", C.c_uint64), ("n_samples", C.c_uint64), ("step", C.c_double),
                ("origin", C.c_double), ("begin", C.c_uint64), ("end", C.c_uint64),
                ("restrict_l2", C.c_double)]


class _Prop(C.Structure):
    _fields_ = [("kind", C.c_int32), ("target", C.c_int32), ("V", C.c_double)]


class _Cov(C.Structure):
    _fields_ = [("n_pairs", C.c_int32), ("lower", C.POINTER(C.c_int32)), ("d_value", C.c_double),
                ("d_distance", C.c_double), ("near_tie", C.c_double), ("tau", C.POINTER(C.c_double))]


class _Res(C.Structure):
    _fields_ = [("checked", C.POINTER(C.c_uint64)), ("violated", C.POINTER(C.c_uint64)),
                ("flagged", C.POINTER(C.c_uint64)), ("first_cex", C.POINTER(C.c_uint64)),
                ("first_cex_unflagged", C.POINTER(C.c_uint64)),
                ("cov_all", C.POINTER(C.c_uint32)), ("cov_certain", C.POINTER(C.c_uint32))]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build_oracle())
        _lib.orc_rne_bf16.restype = C.c_double
        _lib.orc_rne_bf16.argtypes = [C.c_double]
        _lib.orc_plsig.restype = C.c_int32
        _lib.orc_plsig.argtypes = [C.POINTER(C.c_int16), C.c_int32]
        _lib.orc_philox.argtypes = [C.POINTER(C.c_uint32)] * 3
        _lib.orc_forward.restype = C.c_int
        _lib.orc_forward.argtypes = [C.POINTER(_Net), C.c_void_p, C.POINTER(C.c_double)]
        _lib.orc_space_size.restype = C.c_uint64
        _lib.orc_space_size.argtypes = [C.POINTER(_Pert), C.c_int]
        _lib.orc_decode.argtypes = [C.c_int, C.POINTER(_Pert), C.c_void_p, C.c_int, C.c_int,
                                    C.c_uint64, C.c_void_p]
        _lib.orc_decode_box.argtypes = [C.c_int, C.POINTER(_Pert), C.c_void_p, C.c_int, C.c_int,
                                        C.c_uint64, C.POINTER(C.c_double)]
        _lib.orc_forward_dbl.restype = C.c_int
        _lib.orc_forward_dbl.argtypes = [C.POINTER(_Net), C.POINTER(C.c_double), C.POINTER(C.c_double)]
        _lib.orc_coverage_layout.restype = C.c_size_t
        _lib.orc_coverage_layout.argtypes = [C.POINTER(C.c_int32), C.c_int, C.POINTER(C.c_int32),
                                             C.POINTER(C.c_size_t)]
        _lib.orc_cover.argtypes = [C.POINTER(C.c_int32), C.c_int, C.POINTER(C.c_double),
                                   C.POINTER(C.c_double), C.c_int, C.POINTER(C.c_int32),
                                   C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_uint32)]
        _lib.orc_cover_tau.argtypes = [C.POINTER(C.c_int32), C.c_int, C.POINTER(C.c_double),
                                       C.POINTER(C.c_double), C.c_int, C.POINTER(C.c_int32),
                                       C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_double),
                                       C.POINTER(C.c_uint32), C.POINTER(C.c_int)]
        _lib.orc_check.restype = C.c_int
        _lib.orc_check.argtypes = [C.POINTER(_Net), C.c_void_p, C.c_int, C.POINTER(_Pert),
                                   C.POINTER(_Prop), C.POINTER(_Cov), C.POINTER(_Res), C.c_int]
    return _lib


def _p(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


class _Keep:
    """holds numpy buffers referenced by ctypes structs"""
    def __init__(self):
        self.refs = []

    def arr(self, a, dtype):
        a = np.ascontiguousarray(a, dtype=dtype)
        self.refs.append(a)
        return a


def _mk_net(net, keep: _Keep) -> _Net:
    sizes = keep.arr(net.sizes, np.int32)
    Ws = [keep.arr(w, w.dtype) for w in net.W]
    bdt = np.float32 if net.numeric in (0, 1) else np.int32
    bs = [keep.arr(v, bdt) for v in net.b]
    Wp = (C.c_void_p * len(Ws))(*[w.ctypes.data for w in Ws])
    bp = (C.c_void_p * len(bs))(*[v.ctypes.data for v in bs])
    keep.refs += [Wp, bp]
    shift = keep.arr(net.requant_shift if net.requant_shift is not None else [0], np.int32)
    knots = keep.arr(net.sigmoid_knots if net.sigmoid_knots is not None else [0], np.int16)
    sc = keep.arr(net.acc_scale if net.acc_scale is not None else [1.0] * net.L, np.float64)
    return _Net(net.L, _p(sizes, C.c_int32), net.numeric, net.act, Wp, bp,
                _p(shift, C.c_int32), _p(knots, C.c_int16), _p(sc, C.c_double))


def _mk_pert(pert, keep: _Keep) -> _Pert:
    pix = keep.arr(pert.pixels if pert.pixels is not None else [0], np.int32)
    lv = pert.levels if pert.levels is not None else np.zeros(1, np.int16)
    lv = keep.arr(lv, lv.dtype)
    return _Pert(pert.kind, pert.tuple, 0 if pert.pixels is None else len(pert.pixels),
                 _p(pix, C.c_int32), 0 if pert.levels is None else len(pert.levels),
                 lv.ctypes.data, C.c_uint64(pert.seed), C.c_uint64(pert.n_samples),
                 pert.lattice_step, pert.lattice_origin, C.c_uint64(pert.index_begin),
                 C.c_uint64(pert.index_end), float(getattr(pert, "restrict_l2", 0.0)))


# ----------------------------------------------------------------------------- primitives
def rne_bf16(v: float) -> float:
    return lib().orc_rne_bf16(float(v))


def plsig(knots: np.ndarray, u16: int) -> int:
    k = np.ascontiguousarray(knots, dtype=np.int16)
    return lib().orc_plsig(_p(k, C.c_int16), int(u16))


def philox(ctr, key) -> np.ndarray:
    c = np.ascontiguousarray(ctr, dtype=np.uint32)
    k = np.ascontiguousarray(key, dtype=np.uint32)
    out = np.zeros(4, np.uint32)
    lib().orc_philox(_p(c, C.c_uint32), _p(k, C.c_uint32), _p(out, C.c_uint32))
    return out


def forward(net, img) -> List[np.ndarray]:
    """Potentials u_1..u_L (Eq. 1) of one image given in the net's input type, or as exact
    real values (float64, the PHILOX_BOX candidates)."""
    keep = _Keep()
    n = _mk_net(net, keep)
    x = keep.arr(img, img.dtype)
    T = int(sum(net.sizes[1:]))
    out = np.zeros(T, np.float64)
    if img.dtype == np.float64:
        rc = lib().orc_forward_dbl(C.byref(n), _p(x, C.c_double), _p(out, C.c_double))
    else:
        rc = lib().orc_forward(C.byref(n), x.ctypes.data, _p(out, C.c_double))
    if rc != 0:
        raise OverflowError("fixed-point accumulator left int32")
    res, o = [], 0
    for l in range(1, net.L + 1):
        res.append(out[o:o + net.sizes[l]].copy())
        o += net.sizes[l]
    return res


def space_size(pert, n0: int) -> int:
    keep = _Keep()
    return int(lib().orc_space_size(C.byref(_mk_pert(pert, keep)), n0))


def decode(numeric: int, pert, base: np.ndarray, base_id: int, index: int) -> np.ndarray:
    """Candidate `index` of base `base_id` in the net's input type; PHILOX_BOX / PHILOX_CLAMP
    candidates are exact real values and come back as float64."""
    keep = _Keep()
    p = _mk_pert(pert, keep)
    b = keep.arr(base, base.dtype)
    if pert.kind in (4, 5):                             # PHILOX_BOX, PHILOX_CLAMP
        out = np.empty(b.shape[0], np.float64)
        lib().orc_decode_box(numeric, C.byref(p), b.ctypes.data, b.shape[0], base_id, C.c_uint64(index),
                             _p(out, C.c_double))
        return out
    out = np.empty_like(b)
    lib().orc_decode(numeric, C.byref(p), b.ctypes.data, b.shape[0], base_id, C.c_uint64(index),
                     out.ctypes.data)
    return out


def coverage_layout(sizes, pairs):
    s = np.ascontiguousarray(sizes, dtype=np.int32)
    lo = np.ascontiguousarray(pairs, dtype=np.int32)
    offs = np.zeros(4 * len(pairs), dtype=np.uintp)
    n = lib().orc_coverage_layout(_p(s, C.c_int32), len(pairs), _p(lo, C.c_int32),
                                  offs.ctypes.data_as(C.POINTER(C.c_size_t)))
    return int(n), offs.astype(np.int64).reshape(-1, 4)


def cover_traces(sizes, t1: List[np.ndarray], t2: List[np.ndarray], pairs, dg, dh) -> np.ndarray:
    """Pair bitmaps of the four covering methods for two given traces (fixture entry point).
    dg/dh: per-layer thresholds (list of L values, trace units)."""
    s = np.ascontiguousarray(sizes, dtype=np.int32)
    a = np.ascontiguousarray(np.concatenate(t1), dtype=np.float64)
    b = np.ascontiguousarray(np.concatenate(t2), dtype=np.float64)
    lo = np.ascontiguousarray(pairs, dtype=np.int32)
    g = np.ascontiguousarray(dg, dtype=np.float64)
    h = np.ascontiguousarray(dh, dtype=np.float64)
    n, _ = coverage_layout(sizes, pairs)
    w = np.zeros(max(n, 1), np.uint32)
    lib().orc_cover(_p(s, C.c_int32), len(sizes) - 1, _p(a, C.c_double), _p(b, C.c_double),
                    len(pairs), _p(lo, C.c_int32), _p(g, C.c_double), _p(h, C.c_double),
                    _p(w, C.c_uint32))
    return w[:n]


def cover_traces_tau(sizes, t1: List[np.ndarray], t2: List[np.ndarray], pairs, dg, dh, tau):
    """As cover_traces, plus certain[p] = no predicate of pair p within tau of its decision
    boundary (reading C20; tau per layer, trace units)."""
    s = np.ascontiguousarray(sizes, dtype=np.int32)
    a = np.ascontiguousarray(np.concatenate(t1), dtype=np.float64)
    b = np.ascontiguousarray(np.concatenate(t2), dtype=np.float64)
    lo = np.ascontiguousarray(pairs, dtype=np.int32)
    g = np.ascontiguousarray(dg, dtype=np.float64)
    h = np.ascontiguousarray(dh, dtype=np.float64)
    tu = np.ascontiguousarray(tau, dtype=np.float64)
    n, _ = coverage_layout(sizes, pairs)
    w = np.zeros(max(n, 1), np.uint32)
    cert = np.zeros(max(len(pairs), 1), np.int32)
    lib().orc_cover_tau(_p(s, C.c_int32), len(sizes) - 1, _p(a, C.c_double), _p(b, C.c_double),
                        len(pairs), _p(lo, C.c_int32), _p(g, C.c_double), _p(h, C.c_double),
                        _p(tu, C.c_double), _p(w, C.c_uint32), _p(cert, C.c_int))
    return w[:n], cert[:len(pairs)].astype(bool)


def incremental_schedule(gamma: float, max_bound: int, granularity: int = 1) -> List[float]:
    """Reading C28 (SPEC.md incremental_verify): Delta = gamma / max_bound,
    b_i = gamma once i*g >= max_bound, else (i*g) * Delta; i = 1 .. ceil(max_bound / g)."""
    n = -(-max_bound // granularity)
    delta = gamma / max_bound
    return [gamma if i * granularity >= max_bound else float(i * granularity) * delta for i in range(1, n + 1)]


def incremental_verify(cfg, gamma: float, max_bound: int, granularity: int = 1, nthreads: int = 0):
    """The two-step incremental loop of PAPER.md:152-168, per base input, literally: iteration i
    checks the ball delta <= b_i (restriction R, reading C27) -- step one, a violation ends the
    base's loop with that iteration and the ball's first counterexample -- and b_i = gamma ends
    it as complete (step two).  Returns step (1-based, 0 = none), first_cex, and the same over
    unflagged violations, plus the bounds and the iterations run."""
    import copy
    bounds = incremental_schedule(gamma, max_bound, granularity)
    n = cfg.n_base
    none = np.uint64(0xFFFFFFFFFFFFFFFF)
    step = np.zeros(n, np.int32)
    step_u = np.zeros(n, np.int32)
    first = np.full(n, none, np.uint64)
    first_u = np.full(n, none, np.uint64)
    it = 0
    # counts of the last ball checked for each base input: the ball of its deciding iteration, or
    # of the last iteration run (the early-exit mode of the library reports these)
    fin = {k: np.zeros(n, np.uint64) for k in ("checked", "violated", "flagged")}
    for i, b in enumerate(bounds, 1):
        it = i
        c = copy.copy(cfg)
        c.pert = copy.copy(cfg.pert)
        c.pert.restrict_l2 = b
        r = check(c, nthreads)
        for j in range(n):
            if step[j] == 0 and r.first_cex[j] != none:
                step[j], first[j] = i, r.first_cex[j]
            if step_u[j] == 0 and r.first_cex_unflagged[j] != none:
                step_u[j], first_u[j] = i, r.first_cex_unflagged[j]
            if step_u[j] in (0, i):
                for k in fin:
                    fin[k][j] = getattr(r, k)[j]
        if np.all(step_u > 0):
            break                                   # every base input decided
    return {"step": step, "first_cex": first, "step_unflagged": step_u, "first_cex_unflagged": first_u,
            "bounds": bounds, "iterations": it, "final": fin}


def pair_coverage(net, images, pairs, d_value: float, d_distance: float,
                  tau: Optional[np.ndarray] = None):
    """Dataset-pair coverage: the four covers
    of every unordered pair {x_a, x_b}, a < b, of `images`, OR-ed over all pairs, in the layout of
    `coverage_layout`.  Thresholds in potential units as in the check (fixed point: d / scale,
    RNE).  Float numerics also return the words of pairs none of whose predicates lies within
    tau of its boundary (reading C20; tau defaults to C20's widths over the image set); fixed
    point returns the same words twice.  Returns (cov_all, cov_certain)."""
    sizes = list(net.sizes)
    L = net.L
    fl = net.numeric in (0, 1)                         # FP32, BF16
    traces = [forward(net, np.asarray(x)) for x in images]
    if fl:
        dg = [float(d_value)] * L
        dh = [float(d_distance)] * L
        if tau is None:
            tau = [1e-6 + 1e-5 * max(float(np.max(np.abs(t[l]))) for t in traces) for l in range(L)]
    else:
        dg = [float(np.rint(d_value / net.acc_scale[l])) for l in range(L)]
        dh = [float(np.rint(d_distance / net.acc_scale[l])) for l in range(L)]
    n, offs = coverage_layout(sizes, pairs)
    ends = [int(offs[p, 0]) + 2 * sizes[k] * ((sizes[k + 1] + 31) // 32) + 2 * ((sizes[k + 1] + 31) // 32)
            for p, k in enumerate(pairs)]
    s = np.ascontiguousarray(sizes, dtype=np.int32)
    lo = np.ascontiguousarray(pairs, dtype=np.int32)
    g = np.ascontiguousarray(dg, dtype=np.float64)
    h = np.ascontiguousarray(dh, dtype=np.float64)
    tu = np.ascontiguousarray(tau if fl else [0.0] * L, dtype=np.float64)
    flat = [np.ascontiguousarray(np.concatenate(t), dtype=np.float64) for t in traces]
    cov_all = np.zeros(max(n, 1), np.uint32)
    cov_cert = np.zeros(max(n, 1), np.uint32)
    w = np.zeros(max(n, 1), np.uint32)
    cert = np.zeros(max(len(pairs), 1), np.int32)
    for a in range(len(images)):
        for b in range(a + 1, len(images)):
            w[:] = 0
            lib().orc_cover_tau(_p(s, C.c_int32), L, _p(flat[a], C.c_double), _p(flat[b], C.c_double),
                                len(pairs), _p(lo, C.c_int32), _p(g, C.c_double), _p(h, C.c_double),
                                _p(tu, C.c_double) if fl else None, _p(w, C.c_uint32), _p(cert, C.c_int))
            cov_all |= w
            for p in range(len(pairs)):
                if not fl or cert[p]:
                    o = int(offs[p, 0])
                    cov_cert[o:ends[p]] |= w[o:ends[p]]
    return cov_all[:n], cov_cert[:n]


@dataclass
class CheckResult:
    checked: np.ndarray
    violated: np.ndarray
    flagged: np.ndarray
    first_cex: np.ndarray
    first_cex_unflagged: np.ndarray
    cov_all: np.ndarray
    cov_certain: np.ndarray


def default_tau(cfg, base_traces: Optional[List[List[np.ndarray]]] = None) -> np.ndarray:
    """C20: tau_l = 1e-6 + 1e-5 * max over bases of max |u_l^base| (float numerics)."""
    net = cfg.net
    if base_traces is None:
        base_traces = [forward(net, cfg.bases[i]) for i in range(cfg.n_base)]
    tau = []
    for l in range(net.L):
        m = max(float(np.max(np.abs(t[l]))) for t in base_traces)
        tau.append(1e-6 + 1e-5 * m)
    return np.array(tau, np.float64)


def check(cfg, nthreads: int = 0, tau: Optional[np.ndarray] = None) -> CheckResult:
    """Brute-force check of cfg.bases over cfg.pert's index range."""
    keep = _Keep()
    net = cfg.net
    n = _mk_net(net, keep)
    p = _mk_pert(cfg.pert, keep)
    pr = _Prop(cfg.prop.kind, cfg.prop.target, cfg.prop.V)
    lo = keep.arr(cfg.cov.pairs if cfg.cov.pairs else [0], np.int32)
    if net.numeric in (0, 1):
        tau = default_tau(cfg) if tau is None else tau
    tau_a = keep.arr(tau if tau is not None else np.zeros(net.L), np.float64)
    cv = _Cov(len(cfg.cov.pairs), _p(lo, C.c_int32), cfg.cov.d_value, cfg.cov.d_distance,
              cfg.cov.near_tie, _p(tau_a, C.c_double))
    nb = cfg.n_base
    nw, _ = coverage_layout(net.sizes, cfg.cov.pairs)
    out = CheckResult(*[np.zeros(nb, np.uint64) for _ in range(5)],
                      np.zeros(max(nw, 1), np.uint32), np.zeros(max(nw, 1), np.uint32))
    r = _Res(_p(out.checked, C.c_uint64), _p(out.violated, C.c_uint64), _p(out.flagged, C.c_uint64),
             _p(out.first_cex, C.c_uint64), _p(out.first_cex_unflagged, C.c_uint64),
             _p(out.cov_all, C.c_uint32), _p(out.cov_certain, C.c_uint32))
    bases = keep.arr(cfg.bases, cfg.bases.dtype)
    rc = lib().orc_check(C.byref(n), bases.ctypes.data, nb, C.byref(p), C.byref(pr), C.byref(cv),
                         C.byref(r), int(nthreads))
    if rc != 0:
        raise OverflowError("fixed-point accumulator left int32")
    out.cov_all = out.cov_all[:nw]
    out.cov_certain = out.cov_certain[:nw]
    return out


# ----------------------------------------------------------------------------- a11: neuron coverage
METHODS = ("SS", "SV", "VS", "VV")   # VS = the paper's DS-Cover, VV = DV-Cover


def covered_neurons(sizes, pairs, words: np.ndarray):
    """Neuron sets per method (reading C9): a neuron is covered iff it is an endpoint of at least
    one covered pair; a VS/VV column j covers every neuron of layer k and n_{k+1,j}.
    Returns {method: set of (layer, index)} with 1-based layers, 0-based indices."""
    _, offs = coverage_layout(sizes, pairs)
    out = {m: set() for m in METHODS}
    for p, k in enumerate(pairs):
        nk, nu = sizes[k], sizes[k + 1]
        wpr = (nu + 31) // 32
        for mi, m in enumerate(METHODS):
            base = int(offs[p, mi])
            rows = nk if m in ("SS", "SV") else 1
            for i in range(rows):
                for j in range(nu):
                    if (int(words[base + i * wpr + j // 32]) >> (j % 32)) & 1:
                        out[m].add((k + 1, j))
                        if m in ("SS", "SV"):
                            out[m].add((k, i))
                        else:
                            out[m].update((k, ii) for ii in range(nk))
    return out


def coverage_ratio(sizes, pairs, words: np.ndarray):
    """Eqs. sscover..dvcover: ratio = |covered| / N, N = neurons of the layers
    spanned by the configured pairs (reading C9; Table II: 5 + 4 + 5 = 14)."""
    layers = sorted({k for k in pairs} | {k + 1 for k in pairs})
    N = sum(sizes[l] for l in layers)
    sets = covered_neurons(sizes, pairs, words)
    return {m: (len(s) / N if N else 0.0) for m, s in sets.items()}, N


def coverage_literal(ratio: float, P: float) -> bool:
    """l_covered_neuron <=> ratio >= P."""
    return ratio >= P
