"""LUT revalidation of fixed-point counterexamples.

A Q4.12 net evaluates its sigmoid through the 129-knot piecewise-linear table of reading C17, so a
reported counterexample may be an artefact of the table rather than of the network it stands for.
`revalidate` re-evaluates each base input's first counterexample, and the base input itself, under
that real-valued network -- weights raw / 4096 (exact in fp32), biases in accumulator units times
the layer's scale (2^-24 for Q4.12), the exact logistic sigmoid -- on the library's FP32 path, and
reports whether the property is still violated there.

Everything runs through the public API (`Checker.eval`, `decode`): an arbitrary image x is the
candidate of a two-pixel TUPLE_REPLACE space over the base x whose two levels are x_0 and x_1
(index 1 replaces pixel 0 by x_0 and pixel 1 by x_1, i.e. reproduces x).
"""
from __future__ import annotations

from typing import Dict, List

import numpy as np

from mlpv_inputs import ACT_PL_SIGMOID, ACT_SIGMOID

from . import NUM_FP32, NUM_Q4_12, Checker, decode

UMAX = np.uint64(0xFFFFFFFFFFFFFFFF)


def exact_net(qnet):
    """The FP32 network a Q4.12 net approximates (reading C16/C17): W = raw / 4096, b = raw * scale,
    PL-sigmoid -> exact sigmoid."""
    from mlpv_inputs.configs import Net
    if qnet.numeric != NUM_Q4_12:
        raise ValueError("revalidation applies to Q4.12 nets")
    W = [np.asarray(w, np.float64) / 4096.0 for w in qnet.W]
    b = [np.asarray(v, np.float64) * s for v, s in zip(qnet.b, qnet.acc_scale)]
    act = ACT_SIGMOID if qnet.act == ACT_PL_SIGMOID else qnet.act
    return Net(list(qnet.sizes), act, NUM_FP32, [w.astype(np.float32) for w in W], [v.astype(np.float32) for v in b],
               acc_scale=[1.0] * (len(qnet.sizes) - 1))


def _logits(chk: Checker, x: np.ndarray, n_out: int) -> np.ndarray:
    """Logits of the FP32 net for image x (see the module docstring)."""
    import torch
    from mlpv_inputs.configs import Pert
    from mlpv_inputs import PERT_TUPLE_REPLACE
    x = np.ascontiguousarray(x, np.float32)
    pert = Pert(PERT_TUPLE_REPLACE, tuple=2, levels=np.array([x[0], x[1]], np.float32))
    pert.index_end = pert.space_size(len(x))
    base = torch.from_numpy(x[None, :]).cuda()
    u = chk.eval(base, 0, pert, torch.tensor([1], dtype=torch.int64, device="cuda"))
    return u[0, -n_out:].double().cpu().numpy()


def _violated(prop, y: np.ndarray, base_cls: int) -> bool:
    from mlpv_inputs import (PROP_ARGMAX_UNCHANGED, PROP_TARGET_NEVER, PROP_THRESHOLD_LITERAL,
                             PROP_THRESHOLD_LITERAL_ALL)
    cls = int(np.argmax(y))                        # lowest index on ties (reading C12)
    if prop.kind == PROP_ARGMAX_UNCHANGED:
        return cls != base_cls
    if prop.kind == PROP_TARGET_NEVER:
        return cls == prop.target
    D = prop.target if prop.target >= 0 else base_cls
    others = [y[i] > prop.V for i in range(len(y)) if i != D]
    lit = all(others) if prop.kind == PROP_THRESHOLD_LITERAL_ALL else any(others)
    assert prop.kind in (PROP_THRESHOLD_LITERAL, PROP_THRESHOLD_LITERAL_ALL)
    return bool(y[D] < prop.V and lit)


def revalidate(qnet, bases_q: np.ndarray, pert, prop, first_cex: np.ndarray, device: int = 0) -> List[Dict]:
    """One record per base input with a counterexample: its index, the exact network's logits for
    the counterexample and the base, whether the property is violated under the exact network,
    and the top-2 margin there (a small margin means the verdict rests on rounding, not on the
    table)."""
    net = exact_net(qnet)
    chk = Checker(net, device)
    n_out = net.sizes[-1]
    out = []
    try:
        for b, c in enumerate(np.asarray(first_cex, np.uint64)):
            if c == UMAX:
                continue
            img = decode(NUM_Q4_12, pert, bases_q[b], b, int(c)).astype(np.float64) / 4096.0
            base = np.asarray(bases_q[b], np.float64) / 4096.0
            yb = _logits(chk, base, n_out)
            y = _logits(chk, img, n_out)
            top = np.sort(y)[::-1]
            out.append({"base": b, "index": int(c), "logits": y, "base_logits": yb,
                        "base_class": int(np.argmax(yb)), "class": int(np.argmax(y)),
                        "violated_exact": _violated(prop, y, int(np.argmax(yb))),
                        "margin": float(top[0] - top[1]) if len(top) > 1 else float("inf")})
    finally:
        chk.close()
    return out
