"""Command-line front end over the C ABI (SPEC-style exit codes, SPEC.md run_cli):
0 = property holds / task done, 10 = property violated, 2 = usage error, 3 = resource / not built.

    python -m paper_1907_12933_b200.cli check  --config cfg2 [--bases N] [--begin B --end E] [--restrict-l2 b]
    python -m paper_1907_12933_b200.cli verify --config gamma --gamma 3 --max-bound 12 [--granularity 1]
    python -m paper_1907_12933_b200.cli cover  --config cfg3 --images 200 [--threshold 0.8] [--d 0.1]

Inputs are the seeded synthetic workloads of `mlpv_inputs` (BASELINE configs cfg1..cfg5_*, and
"gamma", the Table III-style 25-5-4-5 workload).  Prints one JSON report on stdout.
"""
from __future__ import annotations

import argparse
import json
import sys

import numpy as np

EXIT_OK, EXIT_VIOLATED, EXIT_USAGE, EXIT_RESOURCE = 0, 10, 2, 3


def _config(name: str):
    import mlpv_inputs as M
    if name == "gamma":
        return M.gamma_config()
    return M.make_config(name)


def _to_device(x):
    import torch
    x = np.ascontiguousarray(x)
    return torch.from_numpy(x.view(np.int16) if x.dtype == np.uint16 else x).cuda()


def _subset(cfg, a):
    if a.bases or a.begin is not None or a.end is not None:
        cfg = cfg.subset(n_base=a.bases or cfg.n_base,
                         begin=cfg.pert.index_begin if a.begin is None else a.begin,
                         end=cfg.pert.index_end if a.end is None else a.end)
    return cfg


def _ratios(chk, net, cov, words):
    """Neuron-coverage ratios per method over the layers the pairs span (reading C9)."""
    _, counts = chk.neuron_coverage(cov, words)
    layers = sorted({k for k in cov.pairs} | {k + 1 for k in cov.pairs})
    N = sum(net.sizes[l] for l in layers)
    c = counts.cpu().numpy()
    return {m: (int(c[i]) / N if N else 0.0) for i, m in enumerate(("SS", "SV", "DS", "DV"))}


def _check(P, a):
    import torch
    cfg = _subset(_config(a.config), a)
    if a.restrict_l2:
        cfg.pert.restrict_l2 = a.restrict_l2
    chk = P.Checker(cfg.net)
    try:
        r = chk.check(_to_device(cfg.bases), cfg.pert, cfg.prop, cfg.cov)
        torch.cuda.synchronize()
        n = cfg.n_base
        first = r["first_cex"][:n].cpu().numpy().view(np.uint64)
        viol = r["violated"][:n].cpu().numpy()
        rep = {"command": "check", "config": cfg.name, "bases": n,
               "checked": int(r["checked"][:n].sum()), "violated": int(viol.sum()),
               "bases_violated": int((viol > 0).sum()),
               "first_counterexample": {str(b): int(first[b]) for b in range(n) if viol[b] > 0}}
        if r["n_words"]:
            rep["neuron_coverage"] = _ratios(chk, cfg.net, cfg.cov, r["cov_all"][:r["n_words"]])
    finally:
        chk.close()
    return rep, EXIT_VIOLATED if rep["violated"] else EXIT_OK


def _verify(P, a):
    import torch
    cfg = _subset(_config(a.config), a)
    chk = P.Checker(cfg.net)
    try:
        r = chk.check_incremental(_to_device(cfg.bases), cfg.pert, cfg.prop, cfg.cov, a.gamma, a.max_bound,
                                  a.granularity, early_exit=a.early_exit)
        torch.cuda.synchronize()
        n = cfg.n_base
        step = r["step"][:n].cpu().numpy()
        first = r["first_cex"][:n].cpu().numpy().view(np.uint64)
        bounds = P.incremental_schedule(a.gamma, a.max_bound, a.granularity)
        rep = {"command": "verify", "config": cfg.name, "bases": n, "steps": len(bounds),
               "violated": {str(b): {"step": int(step[b]), "bound": bounds[step[b] - 1], "index": int(first[b])}
                            for b in range(n) if step[b] > 0},
               "safe_over_grid": int((step == 0).sum()),
               "early_exit": bool(a.early_exit),
               "candidates_checked": int(r["checked"][:n].cpu().numpy().view(np.uint64).sum())}
    finally:
        chk.close()
    return rep, EXIT_VIOLATED if rep["violated"] else EXIT_OK


def _cover(P, a):
    import torch
    import mlpv_inputs as M
    from mlpv_inputs.configs import CovSpec
    cfg = _config(a.config)
    pairs = list(cfg.cov.pairs) or list(range(1, cfg.net.L))
    cov = CovSpec(pairs, d_value=a.d, d_distance=a.d)
    imgs = M.pair_images(cfg.net, a.images, seed=a.seed)
    chk = P.Checker(cfg.net)
    try:
        words, _ = chk.pair_coverage(_to_device(imgs), cov)
        torch.cuda.synchronize()
        ratios = _ratios(chk, cfg.net, cov, words)
    finally:
        chk.close()
    fails = {m: v for m, v in ratios.items() if v < a.threshold}
    rep = {"command": "cover", "config": cfg.name, "images": a.images, "pairs_of_images": a.images * (a.images - 1) // 2,
           "threshold": a.threshold, "ratios": ratios,
           "literal": {m: v >= a.threshold for m, v in ratios.items()}}
    return rep, EXIT_VIOLATED if fails else EXIT_OK


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="mlpv", description=__doc__.split("\n")[0])
    sub = ap.add_subparsers(dest="cmd", required=True)
    for name in ("check", "verify"):
        p = sub.add_parser(name)
        p.add_argument("--config", required=True)
        p.add_argument("--bases", type=int, default=0)
        p.add_argument("--begin", type=int, default=None)
        p.add_argument("--end", type=int, default=None)
        if name == "check":
            p.add_argument("--restrict-l2", type=float, default=0.0)
        else:
            p.add_argument("--gamma", type=float, required=True)
            p.add_argument("--max-bound", type=int, required=True)
            p.add_argument("--granularity", type=int, default=1)
            p.add_argument("--early-exit", action="store_true",
                           help="the loop's own order: one shell per pass, a base input stops at its counterexample")
    p = sub.add_parser("cover")
    p.add_argument("--config", required=True)
    p.add_argument("--images", type=int, default=200)
    p.add_argument("--threshold", type=float, default=0.8)
    p.add_argument("--d", type=float, default=0.1)
    p.add_argument("--seed", type=int, default=0)
    a = ap.parse_args(argv)
    import paper_1907_12933_b200 as P
    try:
        rep, code = {"check": _check, "verify": _verify, "cover": _cover}[a.cmd](P, a)
    except KeyError as e:
        print(f"mlpv: unknown config {e}", file=sys.stderr)
        return EXIT_USAGE
    except P.MlpvError as e:
        print(f"mlpv: {e}", file=sys.stderr)
        return EXIT_USAGE if e.status in (1, 2) else EXIT_RESOURCE
    print(json.dumps(rep))
    return code


if __name__ == "__main__":
    sys.exit(main())
