"""Timing of the dataset-pair coverage workload (the paper's EG1 timing,
PAPER.md:584-589: ~20 min for the four covers over a set of 200 images on ESBMC-GPU).

Times mlpv_pair_coverage (image traces + tau + the pair kernel) with CUDA events for a few set
sizes on the 25-5-4-5 net and on config 3's 784-64-32-10 int8 net.  Synthetic images
(mlpv_inputs.pair_images); pairs/s = n (n - 1) / 2 / time.
usage: python tools/pair_cov_bench.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np                                                  # noqa: E402

import mlpv_inputs as M                                             # noqa: E402
from mlpv_inputs.configs import CovSpec                             # noqa: E402


def main():
    import torch
    import paper_1907_12933_b200 as P
    cases = [("25-5-4-5 Q4.12", M.vowel_net(M.NUM_Q4_12), [200, 2000, 20000]),
             ("25-5-4-5 fp32", M.vowel_net(M.NUM_FP32), [200, 20000]),
             ("784-64-32-10 int8", M.make_config("cfg3").net, [200, 5000])]
    print(f"{'net':>20} {'images':>7} {'pairs':>12} {'ms':>9} {'pairs/s':>10}")
    for name, net, ns in cases:
        chk = P.Checker(net)
        cov = CovSpec([1, 2], d_value=0.1, d_distance=0.1)
        for n in ns:
            x = M.pair_images(net, n, seed=0)
            x = torch.from_numpy(x.view(np.int16) if x.dtype == np.uint16 else x).cuda()
            for _ in range(2):
                chk.pair_coverage(x, cov)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 5
            e0.record()
            for _ in range(reps):
                chk.pair_coverage(x, cov)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            pairs = n * (n - 1) // 2
            print(f"{name:>20} {n:7d} {pairs:12d} {ms:9.3f} {pairs / ms * 1e3:10.3e}")
        chk.close()


if __name__ == "__main__":
    main()
