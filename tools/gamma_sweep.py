"""γ sweep in the style of the paper's Table III on the GPU.

A synthetic 25-5-4-5 sigmoid network -- the paper's architecture, inferred from Table II -- in
Q4.12 with the piecewise-linear sigmoid (readings C16/C17), a set of 5x5 binary-ish base images,
and the restriction R of checkNN (reading C27): every candidate of a SUBSET_REPLACE space over 8
pixels (values 0 / 0.5 / 1) whose L2 distance to its base image is at most γ is checked for
"classification unchanged".  Prints, per γ, the candidates inside R, the violations, the bases
with a counterexample and the first one, and the time of the check.  Weights, inputs and pixels
are seeded synthetic stand-ins: the vocalic dataset and the trained net of the
paper are not available, so the numbers are the method's behaviour on this net, not Table III's.

usage: python tools/gamma_sweep.py [--bases 50] [--gammas 0.5,1,1.5,2,2.5,3]
"""
import argparse
import math
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import mlpv_inputs as M                                             # noqa: E402
from mlpv_inputs.configs import Config, CovSpec, Net, Pert, Prop, pl_sigmoid_knots    # noqa: E402


def make(n_base: int) -> Config:
    rng = np.random.default_rng([12933, 77, 0])
    sizes = [25, 5, 4, 5]
    W, b = [], []
    for l in range(1, 4):
        w = rng.normal(0.0, math.sqrt(4.0 / sizes[l - 1]), (sizes[l], sizes[l - 1]))
        W.append(np.clip(np.rint(w * 4096), -32768, 32767).astype(np.int16))
        b.append((np.rint(rng.normal(0.0, 0.5, sizes[l]) * 4096).astype(np.int64) << 12).astype(np.int32))
    net = Net(sizes, M.ACT_PL_SIGMOID, M.NUM_Q4_12, W, b, sigmoid_knots=pl_sigmoid_knots(),
              acc_scale=[2.0 ** -24] * 3)
    bases = (rng.random((n_base, 25)) < 0.4).astype(np.int16) * 4096
    pixels = np.sort(rng.choice(25, 8, replace=False)).astype(np.int32)
    pert = Pert(M.PERT_SUBSET_REPLACE, pixels=pixels, levels=np.array([0, 2048, 4096], np.int16),
                index_begin=0, index_end=3 ** 8)
    return Config("gamma", "25-5-4-5 PL-sigmoid Q4.12", net, bases, pert, Prop(), CovSpec([1, 2]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--bases", type=int, default=50)
    ap.add_argument("--gammas", default="0.5,1,1.5,2,2.5,3")
    args = ap.parse_args()
    import torch
    import paper_1907_12933_b200 as P
    from tests.parity import run_gpu
    cfg = make(args.bases)
    chk = P.Checker(cfg.net)
    run_gpu(chk, cfg)                                                # warm-up
    print(f"{'gamma':>6} {'inside R':>10} {'violations':>11} {'bases hit':>10} {'first cex':>10} {'ms':>8}")
    for g in (float(x) for x in args.gammas.split(",")):
        cfg.pert.restrict_l2 = g
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = run_gpu(chk, cfg)
        dt = (time.perf_counter() - t0) * 1e3
        hit = r["first_cex"] != np.uint64(0xFFFFFFFFFFFFFFFF)
        first = int(r["first_cex"][hit].min()) if hit.any() else -1
        print(f"{g:6.2f} {int(r['checked'].sum()):10d} {int(r['violated'].sum()):11d} {int(hit.sum()):10d} "
              f"{first:10d} {dt:8.2f}")


if __name__ == "__main__":
    main()
