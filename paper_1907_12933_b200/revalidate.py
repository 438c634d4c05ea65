"""LUT revalidation of fixed-point counterexamples.

A Q4.12 net evaluates its sigmoid through the 129-knot piecewise-linear table of reading C17, so a
reported counterexample may be an artefact of the table rather than of the network it stands for.
`revalidate` re-checks each base input's first counterexample under that real-valued network --
weights raw / 4096 (exact in fp32), biases in accumulator units times the layer's scale (2^-24 for
Q4.12), the exact logistic sigmoid -- with the library's own check on the FP32 path: the base
input is the real-valued base image and the perturbation space is a one-candidate SUBSET_REPLACE
space that reproduces the counterexample (its changed pixels, each replaced by its own value).
The verdict (violated / near-tie flagged) is mlpv_check's; this module only builds the arguments
(no forward pass, argmax or property test here).
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


def one_candidate_space(base: np.ndarray, img: np.ndarray):
    """A SUBSET_REPLACE space over `base` whose candidate `index` is `img` (float32 images): the
    K <= 16 pixels where they differ, level k = img's value of the k-th of them, index digits 0..K-1
    (pixel 0 most significant, reading C14).  K = 0 replaces pixel 0 by its own value."""
    from mlpv_inputs import PERT_SUBSET_REPLACE
    from mlpv_inputs.configs import Pert
    px = np.nonzero(img != base)[0].astype(np.int32)
    if len(px) == 0:
        px = np.array([0], np.int32)
    if len(px) > 16:
        raise ValueError("counterexample differs from its base in more than 16 pixels")
    K = len(px)
    idx = 0
    for k in range(K):
        idx = idx * K + k
    pert = Pert(PERT_SUBSET_REPLACE, pixels=px, levels=np.ascontiguousarray(img[px], np.float32),
                index_begin=idx, index_end=idx + 1)
    return pert, idx


def revalidate(qnet, bases_q: np.ndarray, pert, prop, first_cex: np.ndarray, device: int = 0) -> List[Dict]:
    """One record per base input with a counterexample: its index, the exact network's potentials
    for the counterexample (mlpv_eval) and the library's verdict under the exact network
    (violated_exact, flagged_exact: the near-tie flag of reading C20).  violated_exact = False marks
    a LUT artefact."""
    import torch
    from mlpv_inputs.configs import CovSpec
    net = exact_net(qnet)
    chk = Checker(net, device)
    out = []
    try:
        for b, c in enumerate(np.asarray(first_cex, np.uint64)):
            if c == UMAX:
                continue
            img = (decode(NUM_Q4_12, pert, bases_q[b], b, int(c)).astype(np.float64) / 4096.0).astype(np.float32)
            base = (np.asarray(bases_q[b], np.float64) / 4096.0).astype(np.float32)
            sp, idx = one_candidate_space(base, img)
            bt = torch.from_numpy(base[None, :]).cuda(device)
            r = chk.check(bt, sp, prop, CovSpec([]))
            u = chk.eval(bt, 0, sp, torch.tensor([idx], dtype=torch.int64, device=bt.device))
            chk.sync()
            out.append({"base": b, "index": int(c), "potentials": u[0].double().cpu().numpy(),
                        "violated_exact": bool(int(r["violated"][0]) == 1),
                        "flagged_exact": bool(int(r["flagged"][0]) == 1),
                        "checked": int(r["checked"][0])})
    finally:
        chk.close()
    return out
