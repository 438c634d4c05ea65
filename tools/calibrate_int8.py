"""Calibrate the int8 requantisation shifts (reading C18) using ONLY oracle/.

sh_l = smallest shift >= 0 with  max over base inputs, neurons of ReLU(acc_l) >> sh_l  <= 255,
chosen layer by layer (layer l's accumulators do not depend on sh_l, only on earlier shifts).
Prints the INT8_SHIFTS entries stored in mlpv_inputs/configs.py.

    python tools/calibrate_int8.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import mlpv_inputs.configs as Cfg  # noqa: E402
from oracle import oracle as O  # noqa: E402


def calibrate(name: str, n_bases: int = 64):
    L = {"cfg3": 3, "cfg5_int8": 3}[name]
    shifts = [20] * (L - 1)          # placeholders for layers not yet calibrated
    for l in range(L - 1):
        Cfg.INT8_SHIFTS[name] = list(shifts)
        Cfg._CACHE.clear()
        cfg = Cfg.make_config(name)
        m = 0
        for i in range(min(n_bases, cfg.n_base)):
            u = O.forward(cfg.net, cfg.bases[i])[l]
            m = max(m, int(np.max(np.maximum(u, 0))))
        sh = 0
        while (m >> sh) > 255:
            sh += 1
        shifts[l] = sh
    return shifts


if __name__ == "__main__":
    for name in ("cfg3", "cfg5_int8"):
        print(f'    "{name}": {calibrate(name)},')
