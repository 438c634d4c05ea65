"""Host-side multi-GPU logic on CPU with gloo at world size 2: each rank checks its
shard of every base input's index space (here with the oracle standing in for the per-rank GPU
work), the packed results go through the same all-gather as the NCCL path, and the merged result
equals a single full run."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1907_12933_b200 import dist as PD


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _np_merge(parts, n_base, n_words):
    """sum / min / OR over partial results (test-side reference of mlpv_merge)"""
    out = {}
    for k in ("checked", "violated", "flagged"):
        out[k] = sum(p[k][:n_base].numpy().view(np.uint64) for p in parts)
    for k in ("first_cex", "first_cex_unflagged"):
        out[k] = np.minimum.reduce([p[k][:n_base].numpy().view(np.uint64) for p in parts])
    for k in ("cov_all", "cov_certain"):
        out[k] = np.bitwise_or.reduce([p[k][:n_words].numpy().view(np.uint32) for p in parts])
    return out


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import mlpv_inputs as M
    from oracle import oracle as O
    from tests.test_oracle_pins import _stress_cfg2
    cfg = _stress_cfg2()
    b, e = PD.shard(0, cfg.space, rank, world)
    r = O.check(cfg.subset(begin=b, end=e))
    nw = len(r.cov_all)
    res = {k: torch.from_numpy(getattr(r, k).view(np.int64).copy()) for k in PD.COUNT_KEYS}
    res.update({k: torch.from_numpy(getattr(r, k).view(np.int32).copy()) for k in PD.WORD_KEYS})
    parts = PD.allgather_results(res, cfg.n_base, nw)
    merged = _np_merge(parts, cfg.n_base, nw)
    if rank == 0:
        full = O.check(cfg)
        ok = all(np.array_equal(merged[k], getattr(full, k)) for k in merged)
        q.put((ok, [int(x) for x in merged["violated"]]))
    dist.barrier()
    dist.destroy_process_group()


def test_shard_bounds():
    for n, G in [(10, 3), (390_625, 8), (7, 8), (2 ** 32, 8)]:
        sl = [PD.shard(5, 5 + n, g, G) for g in range(G)]
        assert sl[0][0] == 5 and sl[-1][1] == 5 + n
        assert all(sl[i][1] == sl[i + 1][0] for i in range(G - 1))
        assert max(e - b for b, e in sl) - min(e - b for b, e in sl) <= 1


def test_gloo_world2_allgather_merge_equals_full_run():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    ok, viol = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
    assert ok, viol
    assert sum(viol) > 0


def _worker_inc(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import mlpv_inputs as M
    from oracle import oracle as O
    cfg = M.gamma_config(20)
    b, e = PD.shard(0, cfg.pert.index_end, rank, world)
    r = O.incremental_verify(cfg.subset(begin=b, end=e), 3.0, 12, 1)   # this rank's slice
    res = {"step": torch.from_numpy(r["step"]), "first_cex": torch.from_numpy(r["first_cex"].view(np.int64)),
           "step_unflagged": torch.from_numpy(r["step_unflagged"]),
           "first_cex_unflagged": torch.from_numpy(r["first_cex_unflagged"].view(np.int64))}
    merged = PD.allgather_incremental(res, cfg.n_base)
    if rank == 0:
        full = O.incremental_verify(cfg, 3.0, 12, 1)
        ok = np.array_equal(merged["step"].numpy(), full["step"]) and \
            np.array_equal(merged["first_cex"].numpy().view(np.uint64), full["first_cex"])
        q.put((ok, int((full["step"] > 0).sum())))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_incremental_merge_equals_full_loop():
    """NEXT-2 sharded: each rank runs the incremental loop on half of every base's index range; the
    lexicographic (step, index) minimum over ranks equals the loop over the whole range."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_inc, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    ok, n_hit = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
    assert ok and n_hit > 0
