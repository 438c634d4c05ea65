"""The multi-GPU path as bench.py runs it, on the one GPU this environment has:
two processes on cuda:0 each check their shard of every base input's index space through the C ABI
and call the unchanged `dist.reduce_results` (all-gather of the packed results -- gloo, staged
through host memory -- then the mlpv_merge kernel); the merged result equals the oracle's single run.
And the shard invariance §8(e) asks for: G in {1, 2, 4, 8} sub-range calls merged by mlpv_merge
equal one call, bit for bit, on fixed-point and float configs."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import mlpv_inputs as M
from tests.parity import assert_fixed_parity, assert_float_parity, to_device_bases

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _cfg(name):
    if name == "cfg2":
        return M.make_config("cfg2").subset(n_base=4)                      # 4 x 390,625, bit-exact
    if name == "cfg4":
        return M.make_config("cfg4").subset(n_base=3, begin=5000, end=5000 + 1537)
    return M.make_config("cfg5_int8").subset(n_base=2, begin=0, end=777)


def _worker(rank, world, port, name, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        import paper_1907_12933_b200 as P
        from paper_1907_12933_b200 import dist as PD
        cfg = _cfg(name)
        chk = P.Checker(cfg.net)
        b, e = PD.shard(cfg.pert.index_begin, cfg.pert.index_end, rank, world)
        s = cfg.subset(begin=b, end=e)
        r = chk.check(to_device_bases(s), s.pert, s.prop, s.cov)
        chk.sync()
        nw = r["n_words"]
        merged = PD.reduce_results(r, cfg.n_base, nw)
        torch.cuda.synchronize()
        out = P.result_to_numpy(merged, cfg.n_base, nw)
        q.put((rank, {k: v.copy() for k, v in out.items()}))
    finally:
        dist.barrier()
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["cfg2", "cfg4", "cfg5_int8"])
def test_two_process_reduce_matches_oracle(oracle_mod, name):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=600) for _ in range(2))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    cfg = _cfg(name)
    o = oracle_mod.check(cfg)
    for rank in (0, 1):                       # every rank holds the merged result
        g = got[rank]
        if cfg.net.numeric == M.NUM_BF16:
            assert_float_parity(g, o)
        else:
            assert_fixed_parity(g, o)
    assert all(np.array_equal(got[0][k], got[1][k]) for k in got[0])


@pytest.mark.parametrize("name,n_base,begin,end", [("cfg2", 3, 0, 390_625), ("cfg3", 2, 1_000_000, 1_262_144),
                                                   ("cfg5_int8", 2, 100, 2148), ("cfg4", 4, 0, 4099)])
def test_shard_invariance(name, n_base, begin, end):
    """G = 1, 2, 4, 8 contiguous shards of every base's range, merged by mlpv_merge, are identical to
    one call: counts, first counterexamples and every coverage word (float configs included: a
    candidate's arithmetic does not depend on the tile it lands in)."""
    import torch
    import paper_1907_12933_b200 as P
    from paper_1907_12933_b200 import dist as PD
    cfg = M.make_config(name).subset(n_base=n_base, begin=begin, end=end)
    chk = P.Checker(cfg.net)
    bases = to_device_bases(cfg)
    one = chk.check(bases, cfg.pert, cfg.prop, cfg.cov)
    chk.sync()
    nw = one["n_words"]
    ref = P.result_to_numpy(one, cfg.n_base, nw)
    for G in (2, 4, 8):
        parts = []
        for g in range(G):
            b, e = PD.shard(begin, end, g, G)
            s = cfg.subset(begin=b, end=e)
            parts.append(chk.check(bases, s.pert, s.prop, s.cov))
        chk.sync()
        m = P.result_to_numpy(P.merge(parts, cfg.n_base, nw), cfg.n_base, nw)
        torch.cuda.synchronize()
        for k in ref:
            assert np.array_equal(m[k], ref[k]), (name, G, k)


def test_bench_two_ranks_one_gpu():
    """bench.py's N > 1 path as the driver launches it (torch.distributed.run, two ranks), with gloo
    and both ranks on the one GPU of this box (MLPV_BENCH_GLOO, tests only): index-space shards, the
    all-gather + merge exchange every step, the max-over-ranks timing and rank 0's single JSON line."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, MLPV_BENCH_GLOO="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29517", "bench.py", "--gpus", "2",
           "--config", "cfg2", "--steps", "2", "--warmup", "1", "--no-cpu-baseline"]
    out = subprocess.run(cmd, cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]          # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["parallelism"].startswith("dp2") and d["value"] > 0
    assert d["config"]["candidates_per_step"] == 10 * 390_625       # both shards of every base
