"""Shared helpers of the GPU <-> oracle parity tests (the comparison rules of DESIGN.md)."""
import numpy as np

UMAX = np.iinfo(np.uint64).max

# Float tolerance (north_star; reading C20, SURVEY.md:541): element-wise, the allclose form
#   |g_i - o_i| <= ATOL + RTOL * |o_i|
RTOL, ATOL = 1e-5, 1e-6


def to_device_bases(cfg, device="cuda"):
    import torch
    b = cfg.bases
    if b.dtype == np.uint16:
        t = torch.from_numpy(b.view(np.int16).copy())
    else:
        t = torch.from_numpy(np.ascontiguousarray(b))
    return t.to(device)


def run_gpu(chk, cfg, tau=None):
    import torch
    import paper_1907_12933_b200 as P
    bases = to_device_bases(cfg)
    r = chk.check(bases, cfg.pert, cfg.prop, cfg.cov, tau=tau)
    chk.sync()                                  # raises on a kernel fault / device-found input error
    torch.cuda.synchronize()
    return P.result_to_numpy(r, cfg.n_base, r["n_words"])


def assert_fixed_parity(g, o):
    """bit-exact: every count, every counterexample index, every coverage bit"""
    for k in ("checked", "violated", "first_cex"):
        assert np.array_equal(g[k], getattr(o, k)), (k, g[k], getattr(o, k))
    assert np.all(g["flagged"] == 0)
    assert np.array_equal(g["first_cex_unflagged"], g["first_cex"])
    assert np.array_equal(g["cov_all"], o.cov_all), ("cov_all", np.nonzero(g["cov_all"] != o.cov_all))
    assert np.array_equal(g["cov_certain"], o.cov_all)


def assert_float_parity(g, o):
    """C20: (ii) |violated_g - violated_o| <= min(flagged_g, flagged_o); (iii) first counterexamples
    bracket each other's unflagged ones; (iv) certain coverage of each side is contained in the
    other side's full coverage."""
    assert np.array_equal(g["checked"], o.checked)
    vg, vo = g["violated"].astype(np.int64), o.violated.astype(np.int64)
    fmin = np.minimum(g["flagged"], o.flagged).astype(np.int64)
    assert np.all(np.abs(vg - vo) <= fmin), (vg, vo, g["flagged"], o.flagged)
    assert np.all(g["first_cex"] <= o.first_cex_unflagged), (g["first_cex"], o.first_cex_unflagged)
    assert np.all(o.first_cex <= g["first_cex_unflagged"]), (o.first_cex, g["first_cex_unflagged"])
    assert np.array_equal(o.cov_certain & ~g["cov_all"], np.zeros_like(o.cov_certain))
    assert np.array_equal(g["cov_certain"] & ~o.cov_all, np.zeros_like(o.cov_all))


def assert_logits_close(g, o):
    """C20 logits: every element within ATOL + RTOL * |o| (no vector scaling).  Returns the max
    absolute error and the worst err / tol ratio (reported by the tests)."""
    g = np.asarray(g, np.float64)
    o = np.asarray(o, np.float64)
    tol = ATOL + RTOL * np.abs(o)
    err = np.abs(g - o)
    ratio = err / tol
    bad = np.argwhere(ratio > 1.0)
    assert bad.size == 0, (f"{len(bad)} logits outside |g-o| <= 1e-6 + 1e-5|o|: max err {err.max():.3e}, "
                           f"worst ratio {ratio.max():.3f} at o = {o[tuple(bad[0])]:.6g}")
    return float(err.max()), float(ratio.max())
