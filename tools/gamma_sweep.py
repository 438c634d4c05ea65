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
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import mlpv_inputs as M                                             # noqa: E402
from mlpv_inputs.configs import Config                              # noqa: E402


def make(n_base: int) -> Config:
    return M.gamma_config(n_base)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--bases", type=int, default=50)
    ap.add_argument("--gammas", default="0.5,1,1.5,2,2.5,3")
    ap.add_argument("--max-bound", type=int, default=12)
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
    # the incremental loop (NEXT-2) over the same gammas as one schedule: gamma_max, max_bound
    gs = [float(x) for x in args.gammas.split(",")]
    mb = args.max_bound
    cfg.pert.restrict_l2 = 0.0
    bases = torch.from_numpy(cfg.bases).cuda()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = chk.check_incremental(bases, cfg.pert, cfg.prop, cfg.cov, max(gs), mb, 1)
    st = r["step"].cpu().numpy()
    dt = (time.perf_counter() - t0) * 1e3
    sched = P.incremental_schedule(max(gs), mb, 1)
    print(f"incremental: gamma = {max(gs)}, {mb} steps, {dt:.2f} ms; bases violated at step i (b_i):")
    for i, b in enumerate(sched, 1):
        print(f"  step {i:3d}  b = {b:6.3f}  bases {int((st == i).sum()):4d}")
    print(f"  safe over the grid: {int((st == 0).sum())}")
    # the same loop in its own order with early exit (one shell per pass, decided bases stop)
    for ee in (False, True):
        chk.check_incremental(bases, cfg.pert, cfg.prop, cfg.cov, max(gs), mb, 1, early_exit=ee)   # warm-up
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r2 = chk.check_incremental(bases, cfg.pert, cfg.prop, cfg.cov, max(gs), mb, 1, early_exit=ee)
        st2 = r2["step"].cpu().numpy()
        dt = (time.perf_counter() - t0) * 1e3
        assert np.array_equal(st2, st)
        print(f"incremental early_exit={int(ee)}: {dt:.2f} ms, candidates checked "
              f"{int(r2['checked'][:cfg.n_base].cpu().numpy().view(np.uint64).sum())}")


if __name__ == "__main__":
    main()
