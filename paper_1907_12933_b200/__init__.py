"""Thin Python binding of the C ABI in include/mlpv.h (argument marshalling only).

Every step of the check runs in libmlpv.so (sm_100a kernels).  PyTorch is used for device
memory and streams only.  There is no CPU fallback: if the extension is missing, importing the
library raises.

    from paper_1907_12933_b200 import Checker
    chk = Checker(net)                        # net: sizes, act, numeric, W, b, requant_shift, ...
    res = chk.check(bases, pert, prop, cov)   # dict of CUDA tensors
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Dict, Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MLPV_LIB") or os.path.join(HERE, "libmlpv.so")   # MLPV_LIB: debug builds only

NUM_FP32, NUM_BF16, NUM_Q4_12, NUM_INT8 = 0, 1, 2, 3
STATUS = {0: "OK", 1: "E_INVALID", 2: "E_SHAPE", 3: "E_UNSUPPORTED", 4: "E_OVERFLOW", 5: "E_OOM", 6: "E_CUDA"}
EXPORTS = ["mlpv_create", "mlpv_destroy", "mlpv_last_error", "mlpv_coverage_layout", "mlpv_space_size",
           "mlpv_check", "mlpv_eval", "mlpv_decode", "mlpv_merge", "mlpv_neuron_coverage", "mlpv_pair_coverage",
           "mlpv_check_incremental", "mlpv_incremental_steps", "mlpv_incremental_bound",
           "mlpv_profile", "mlpv_sync", "mlpv_version"]


class MlpvError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class _Net(C.Structure):
    _fields_ = [("n_layers", C.c_int32), ("sizes", C.POINTER(C.c_int32)), ("W", C.POINTER(C.c_void_p)),
                ("b", C.POINTER(C.c_void_p)), ("hidden_act", C.c_int)]


class _Quant(C.Structure):
    _fields_ = [("numeric", C.c_int), ("requant_shift", C.POINTER(C.c_int32)),
                ("sigmoid_knots", C.POINTER(C.c_int16)), ("acc_scale", C.POINTER(C.c_double))]


class _Pert(C.Structure):
    _fields_ = [("kind", C.c_int), ("tuple", C.c_int32), ("n_pixels", C.c_int32),
                ("pixels", C.POINTER(C.c_int32)), ("n_levels", C.c_int32), ("levels", C.c_void_p),
                ("seed", C.c_uint64), ("n_samples", C.c_uint64), ("lattice_step", C.c_double),
                ("lattice_origin", C.c_double), ("index_begin", C.c_uint64), ("index_end", C.c_uint64),
                ("restrict_l2", C.c_double)]


class _Prop(C.Structure):
    _fields_ = [("kind", C.c_int), ("target", C.c_int32), ("V", C.c_double)]


class _Cov(C.Structure):
    _fields_ = [("n_pairs", C.c_int32), ("lower_layer", C.POINTER(C.c_int32)), ("d_value", C.c_double),
                ("d_distance", C.c_double), ("near_tie", C.c_double), ("tau", C.POINTER(C.c_double))]


class _Inc(C.Structure):
    _fields_ = [("gamma", C.c_double), ("max_bound", C.c_int32), ("granularity", C.c_int32),
                ("early_exit", C.c_int32), ("reserved", C.c_int32)]


class _Res(C.Structure):
    _fields_ = [("checked", C.c_void_p), ("violated", C.c_void_p), ("flagged", C.c_void_p),
                ("first_cex", C.c_void_p), ("first_cex_unflagged", C.c_void_p),
                ("cov_all", C.c_void_p), ("cov_certain", C.c_void_p)]


_lib = None


def lib() -> C.CDLL:
    """Load libmlpv.so; raises if the extension has not been built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built; run `python -m paper_1907_12933_b200.build` "
                              "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        L.mlpv_create.argtypes = [C.POINTER(_Net), C.POINTER(_Quant), C.c_int, C.POINTER(C.c_void_p)]
        L.mlpv_destroy.argtypes = [C.c_void_p]
        L.mlpv_last_error.restype = C.c_char_p
        L.mlpv_last_error.argtypes = [C.c_void_p]
        L.mlpv_coverage_layout.argtypes = [C.c_void_p, C.POINTER(_Cov), C.POINTER(C.c_size_t), C.POINTER(C.c_size_t)]
        L.mlpv_space_size.argtypes = [C.c_void_p, C.POINTER(_Pert), C.POINTER(C.c_uint64)]
        L.mlpv_check.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.POINTER(_Pert), C.POINTER(_Prop),
                                 C.POINTER(_Cov), C.POINTER(_Res), C.c_void_p]
        L.mlpv_eval.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.POINTER(_Pert), C.c_void_p,
                                C.c_int64, C.c_void_p, C.c_void_p]
        L.mlpv_decode.argtypes = [C.c_int, C.POINTER(_Pert), C.c_void_p, C.c_int32, C.c_int32, C.c_uint64, C.c_void_p]
        L.mlpv_merge.argtypes = [C.POINTER(_Res), C.c_int32, C.c_int32, C.c_size_t, C.POINTER(_Res), C.c_void_p]
        L.mlpv_neuron_coverage.argtypes = [C.c_void_p, C.POINTER(_Cov), C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.mlpv_pair_coverage.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.POINTER(_Cov), C.c_void_p,
                                         C.c_void_p, C.c_void_p]
        L.mlpv_check_incremental.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.POINTER(_Pert), C.POINTER(_Prop),
                                             C.POINTER(_Cov), C.POINTER(_Inc), C.POINTER(_Res), C.c_void_p,
                                             C.c_void_p, C.c_void_p]
        L.mlpv_incremental_steps.restype = C.c_int32
        L.mlpv_incremental_steps.argtypes = [C.POINTER(_Inc)]
        L.mlpv_incremental_bound.restype = C.c_double
        L.mlpv_incremental_bound.argtypes = [C.POINTER(_Inc), C.c_int32]
        L.mlpv_profile.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_uint64)]
        L.mlpv_sync.argtypes = [C.c_void_p, C.c_void_p]
        L.mlpv_version.restype = C.c_char_p
        for f in ("mlpv_create", "mlpv_coverage_layout", "mlpv_space_size", "mlpv_check", "mlpv_eval",
                  "mlpv_decode", "mlpv_merge", "mlpv_neuron_coverage", "mlpv_profile", "mlpv_sync"):
            getattr(L, f).restype = C.c_int
        _lib = L
    return _lib


def _ck(status: int, handle=None):
    if status != 0:
        msg = lib().mlpv_last_error(handle).decode()
        raise MlpvError(status, msg)


class _Keep(list):
    def arr(self, a, dtype):
        a = np.ascontiguousarray(a, dtype=dtype)
        self.append(a)
        return a


def _ptr(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


def _mk_pert(pert, keep: _Keep) -> _Pert:
    pix = keep.arr(pert.pixels if pert.pixels is not None else [0], np.int32)
    if pert.levels is not None:
        lv = keep.arr(pert.levels, pert.levels.dtype)
        lvp, nl = lv.ctypes.data, len(pert.levels)
    else:
        lvp, nl = None, 0
    return _Pert(pert.kind, pert.tuple, 0 if pert.pixels is None else len(pert.pixels), _ptr(pix, C.c_int32),
                 nl, lvp, C.c_uint64(int(pert.seed)), C.c_uint64(int(pert.n_samples)),
                 float(pert.lattice_step), float(pert.lattice_origin), C.c_uint64(int(pert.index_begin)),
                 C.c_uint64(int(pert.index_end)), float(getattr(pert, "restrict_l2", 0.0)))


def _mk_cov(cov, keep: _Keep, tau=None) -> _Cov:
    lo = keep.arr(cov.pairs if cov.pairs else [0], np.int32)
    tp = None
    if tau is not None:
        tp = _ptr(keep.arr(tau, np.float64), C.c_double)
    return _Cov(len(cov.pairs), _ptr(lo, C.c_int32), float(cov.d_value), float(cov.d_distance),
                float(cov.near_tie), tp)


def _stream_ptr(stream):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def decode(numeric: int, pert, base: np.ndarray, base_id: int, index: int) -> np.ndarray:
    """Host-side candidate reconstruction (counterexample images); PHILOX_BOX / PHILOX_CLAMP
    candidates are exact reals and come back as float64."""
    keep = _Keep()
    p = _mk_pert(pert, keep)
    b = keep.arr(base, base.dtype)
    out = np.empty(b.shape[0], np.float64) if pert.kind in (4, 5) else np.empty_like(b)
    _ck(lib().mlpv_decode(numeric, C.byref(p), b.ctypes.data, b.shape[0], base_id, C.c_uint64(int(index)),
                          out.ctypes.data))
    return out


def _res_struct(d: Dict) -> _Res:
    g = lambda k: C.c_void_p(d[k].data_ptr()) if d.get(k) is not None else None  # noqa: E731
    return _Res(g("checked"), g("violated"), g("flagged"), g("first_cex"), g("first_cex_unflagged"),
                g("cov_all"), g("cov_certain"))


def merge(parts: Sequence[Dict], n_base: int, n_words: int, stream=None) -> Dict:
    """Merge partial results of disjoint index ranges by sum / min / OR (on the GPU)."""
    import torch
    dev = parts[0]["checked"].device
    out = alloc_result(n_base, n_words, dev)
    arr = (_Res * len(parts))(*[_res_struct(p) for p in parts])
    o = _res_struct(out)
    _ck(lib().mlpv_merge(arr, len(parts), n_base, n_words, C.byref(o), _stream_ptr(stream)))
    return out


def alloc_result(n_base: int, n_words: int, device) -> Dict:
    import torch
    z = lambda n, dt: torch.empty(max(n, 1), dtype=dt, device=device)  # noqa: E731
    return {"checked": z(n_base, torch.int64), "violated": z(n_base, torch.int64),
            "flagged": z(n_base, torch.int64), "first_cex": z(n_base, torch.int64),
            "first_cex_unflagged": z(n_base, torch.int64),
            "cov_all": z(n_words, torch.int32), "cov_certain": z(n_words, torch.int32)}


def result_to_numpy(r: Dict, n_base: int, n_words: int) -> Dict[str, np.ndarray]:
    out = {}
    for k in ("checked", "violated", "flagged", "first_cex", "first_cex_unflagged"):
        out[k] = r[k][:n_base].cpu().numpy().view(np.uint64)
    for k in ("cov_all", "cov_certain"):
        out[k] = r[k][:n_words].cpu().numpy().view(np.uint32)
    return out


class Checker:
    """One mlpv handle (net resident on one device)."""

    def __init__(self, net, device: int = 0):
        self.net = net
        self.device = device
        keep = _Keep()
        sizes = keep.arr(net.sizes, np.int32)
        Ws = [keep.arr(w, w.dtype) for w in net.W]
        bdt = np.float32 if net.numeric in (NUM_FP32, NUM_BF16) else np.int32
        bs = [keep.arr(v, bdt) for v in net.b]
        Wp = (C.c_void_p * len(Ws))(*[w.ctypes.data for w in Ws])
        bp = (C.c_void_p * len(bs))(*[v.ctypes.data for v in bs])
        n = _Net(len(net.sizes) - 1, _ptr(sizes, C.c_int32), Wp, bp, net.act)
        sh = _ptr(keep.arr(net.requant_shift, np.int32), C.c_int32) if net.requant_shift is not None else None
        kn = _ptr(keep.arr(net.sigmoid_knots, np.int16), C.c_int16) if net.sigmoid_knots is not None else None
        sc = _ptr(keep.arr(net.acc_scale, np.float64), C.c_double) if net.acc_scale is not None else None
        q = _Quant(net.numeric, sh, kn, sc)
        h = C.c_void_p()
        _ck(lib().mlpv_create(C.byref(n), C.byref(q), device, C.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            lib().mlpv_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def coverage_layout(self, cov):
        keep = _Keep()
        c = _mk_cov(cov, keep)
        nw = C.c_size_t()
        offs = (C.c_size_t * max(4 * len(cov.pairs), 1))()
        _ck(lib().mlpv_coverage_layout(self._h, C.byref(c), C.byref(nw), offs), self._h)
        return int(nw.value), np.array(offs[:4 * len(cov.pairs)], dtype=np.int64).reshape(-1, 4)

    def space_size(self, pert) -> int:
        keep = _Keep()
        p = _mk_pert(pert, keep)
        s = C.c_uint64()
        _ck(lib().mlpv_space_size(self._h, C.byref(p), C.byref(s)), self._h)
        return int(s.value)

    def check(self, bases, pert, prop, cov, tau=None, out: Optional[Dict] = None, stream=None) -> Dict:
        """bases: CUDA tensor [n_base, n_0] in the input element type (enqueued on `stream`)."""
        import torch
        n_base = int(bases.shape[0])
        nw, _ = self.coverage_layout(cov)
        r = out if out is not None else alloc_result(n_base, nw, bases.device)
        keep = _Keep()
        p = _mk_pert(pert, keep)
        pr = _Prop(prop.kind, prop.target, float(prop.V))
        c = _mk_cov(cov, keep, tau)
        rs = _res_struct(r)
        if nw == 0:
            rs.cov_all = None
            rs.cov_certain = None
        _ck(lib().mlpv_check(self._h, C.c_void_p(bases.data_ptr()), n_base, C.byref(p), C.byref(pr), C.byref(c),
                             C.byref(rs), _stream_ptr(stream)), self._h)
        r["n_words"] = nw
        return r

    def check_incremental(self, bases, pert, prop, cov, gamma: float, max_bound: int, granularity: int = 1,
                          tau=None, stream=None, early_exit: bool = False) -> Dict:
        """mlpv_check_incremental: the check's result dict plus "step" / "step_unflagged" (CUDA
        int32 [n_base]; 1-based iteration of the incremental loop, 0 = none in the gamma ball).
        early_exit: the loop's own order, one shell per pass, a base input's work ending at its
        counterexample's iteration (the counts / coverage are then those of that ball)."""
        import torch
        n_base = int(bases.shape[0])
        nw, _ = self.coverage_layout(cov)
        r = alloc_result(n_base, nw, bases.device)
        r["step"] = torch.empty(n_base, dtype=torch.int32, device=bases.device)
        r["step_unflagged"] = torch.empty(n_base, dtype=torch.int32, device=bases.device)
        keep = _Keep()
        p = _mk_pert(pert, keep)
        pr = _Prop(prop.kind, prop.target, float(prop.V))
        c = _mk_cov(cov, keep, tau)
        inc = _Inc(float(gamma), int(max_bound), int(granularity), 1 if early_exit else 0, 0)
        rs = _res_struct(r)
        if nw == 0:
            rs.cov_all = None
            rs.cov_certain = None
        _ck(lib().mlpv_check_incremental(self._h, C.c_void_p(bases.data_ptr()), n_base, C.byref(p), C.byref(pr),
                                         C.byref(c), C.byref(inc), C.byref(rs), C.c_void_p(r["step"].data_ptr()),
                                         C.c_void_p(r["step_unflagged"].data_ptr()), _stream_ptr(stream)), self._h)
        r["n_words"] = nw
        return r

    def eval(self, bases, base_id: int, pert, indices, stream=None):
        """Potentials of every layer for candidates `indices` (CUDA int64 tensor) of base base_id."""
        import torch
        T = int(sum(self.net.sizes[1:]))
        n = int(indices.numel())
        dt = torch.float32 if self.net.numeric in (NUM_FP32, NUM_BF16) else torch.int32
        out = torch.empty((max(n, 1), T), dtype=dt, device=bases.device)
        keep = _Keep()
        p = _mk_pert(pert, keep)
        _ck(lib().mlpv_eval(self._h, C.c_void_p(bases.data_ptr()), int(bases.shape[0]), int(base_id), C.byref(p),
                            C.c_void_p(indices.data_ptr()), n, C.c_void_p(out.data_ptr()), _stream_ptr(stream)),
            self._h)
        return out[:n]

    def sync(self, stream=None):
        """mlpv_sync: wait for `stream` and raise MlpvError for an asynchronous kernel fault or an
        input error the device found (call before reading results)."""
        _ck(lib().mlpv_sync(self._h, _stream_ptr(stream)), self._h)

    def profile(self, ev_begin=None, ev_end=None) -> int:
        """Record torch.cuda.Event pair around the enumeration kernel of later checks (None
        disables); returns the number of kernels this handle has launched."""
        n = C.c_uint64()
        b = C.c_void_p(ev_begin.cuda_event) if ev_begin is not None else None
        e = C.c_void_p(ev_end.cuda_event) if ev_end is not None else None
        _ck(lib().mlpv_profile(self._h, b, e, C.byref(n)), self._h)
        return int(n.value)

    def pair_coverage(self, images, cov, tau=None, stream=None):
        """Dataset-pair coverage (mlpv_pair_coverage): images = CUDA tensor [n, n_0] in the input
        element type.  Returns (cov_all, cov_certain), CUDA int32 tensors of n_words words."""
        import torch
        nw, _ = self.coverage_layout(cov)
        cov_all = torch.empty(max(nw, 1), dtype=torch.int32, device=images.device)
        cov_cert = torch.empty(max(nw, 1), dtype=torch.int32, device=images.device)
        keep = _Keep()
        c = _mk_cov(cov, keep, tau)
        _ck(lib().mlpv_pair_coverage(self._h, C.c_void_p(images.data_ptr()), int(images.shape[0]), C.byref(c),
                                     C.c_void_p(cov_all.data_ptr()), C.c_void_p(cov_cert.data_ptr()),
                                     _stream_ptr(stream)), self._h)
        return cov_all[:nw], cov_cert[:nw]

    def neuron_coverage(self, cov, words, stream=None):
        import torch
        T = int(sum(self.net.sizes[1:]))
        covered = torch.empty(4 * T, dtype=torch.uint8, device=words.device)
        counts = torch.empty(4, dtype=torch.int32, device=words.device)
        keep = _Keep()
        c = _mk_cov(cov, keep)
        _ck(lib().mlpv_neuron_coverage(self._h, C.byref(c), C.c_void_p(words.data_ptr()),
                                       C.c_void_p(covered.data_ptr()), C.c_void_p(counts.data_ptr()),
                                       _stream_ptr(stream)), self._h)
        return covered.view(4, T), counts


def incremental_schedule(gamma: float, max_bound: int, granularity: int = 1):
    """The bounds b_1 .. b_n of the incremental loop as the library computes them (reading C28)."""
    inc = _Inc(float(gamma), int(max_bound), int(granularity))
    n = lib().mlpv_incremental_steps(C.byref(inc))
    return [lib().mlpv_incremental_bound(C.byref(inc), i) for i in range(1, n + 1)]


def version() -> str:
    return lib().mlpv_version().decode()
