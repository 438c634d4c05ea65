"""Multi-GPU plumbing: every rank checks a contiguous slice of every base input's
index space; the only exchange is one all-gather of the packed partial results followed by the
sum / min / OR merge kernel (mlpv_merge) on every rank.  Works with any torch.distributed backend
(NCCL on GPUs; gloo on CPU tensors for the host-side tests)."""
from __future__ import annotations

from typing import Dict, List, Tuple

COUNT_KEYS = ("checked", "violated", "flagged", "first_cex", "first_cex_unflagged")
WORD_KEYS = ("cov_all", "cov_certain")


def shard(begin: int, end: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous slice [floor(n*g/G), floor(n*(g+1)/G)) of [begin, end) for rank g of G."""
    n = end - begin
    return begin + n * rank // world, begin + n * (rank + 1) // world


def pack(res: Dict, n_base: int, n_words: int):
    """One flat int32 tensor: 5 x n_base int64 counts (as int32 pairs) + 2 x n_words words."""
    import torch
    parts = [res[k][:n_base].view(torch.int32) for k in COUNT_KEYS]
    parts += [res[k][:n_words] for k in WORD_KEYS]
    return torch.cat(parts)


def unpack(flat, n_base: int, n_words: int) -> Dict:
    import torch
    out, o = {}, 0
    for k in COUNT_KEYS:
        out[k] = flat[o:o + 2 * n_base].view(torch.int64)
        o += 2 * n_base
    for k in WORD_KEYS:
        out[k] = flat[o:o + n_words]
        o += n_words
    return out


def allgather_results(res: Dict, n_base: int, n_words: int, group=None) -> List[Dict]:
    """The single collective of a multi-GPU check: all-gather of every rank's packed result."""
    import torch
    import torch.distributed as dist
    flat = pack(res, n_base, n_words).contiguous()
    dev = flat.device
    if dist.get_backend(group) == "gloo" and flat.is_cuda:
        flat = flat.cpu()                      # gloo: stage through host memory (tests, CPU-only boxes)
    world = dist.get_world_size(group)
    bufs = [torch.empty_like(flat) for _ in range(world)]
    dist.all_gather(bufs, flat, group=group)
    return [unpack(b.to(dev), n_base, n_words) for b in bufs]


def reduce_results(res: Dict, n_base: int, n_words: int, group=None, stream=None) -> Dict:
    """All-gather + GPU merge (sum counts, min counterexample indices, OR coverage words)."""
    import paper_1907_12933_b200 as P
    parts = allgather_results(res, n_base, n_words, group)
    return P.merge(parts, n_base, n_words, stream=stream)


STEP_SHIFT = 48   # candidate indices < 2^48 in incremental mode (include/mlpv.h)


def merge_incremental(parts: List[Dict], n_base: int) -> Dict:
    """Incremental bounds across shards (SURVEY.md §8(f) NEXT-2 on several GPUs): the loop's answer for
    a base input is the lexicographic minimum of the shards' (step, index) pairs, step 0 = none.
    parts: per shard {"step", "first_cex", "step_unflagged", "first_cex_unflagged"} tensors."""
    import torch
    out = {}
    for sk, ik in (("step", "first_cex"), ("step_unflagged", "first_cex_unflagged")):
        keys = []
        for p in parts:
            st = p[sk][:n_base].to(torch.int64)
            idx = p[ik][:n_base].to(torch.int64) & ((1 << STEP_SHIFT) - 1)
            keys.append(torch.where(st > 0, (st << STEP_SHIFT) | idx, torch.full_like(st, 2 ** 63 - 1)))
        k = torch.stack(keys).min(dim=0).values
        hit = k != 2 ** 63 - 1
        out[sk] = torch.where(hit, k >> STEP_SHIFT, torch.zeros_like(k)).to(torch.int32)
        out[ik] = torch.where(hit, k & ((1 << STEP_SHIFT) - 1), torch.full_like(k, -1))   # -1 = UINT64_MAX
    return out


def allgather_incremental(res: Dict, n_base: int, group=None) -> Dict:
    """All-gather of every rank's (step, index) pairs and their merge (merge_incremental)."""
    import torch
    import torch.distributed as dist
    flat = torch.cat([res["step"][:n_base].to(torch.int64), res["first_cex"][:n_base].to(torch.int64),
                      res["step_unflagged"][:n_base].to(torch.int64),
                      res["first_cex_unflagged"][:n_base].to(torch.int64)]).contiguous()
    bufs = [torch.empty_like(flat) for _ in range(dist.get_world_size(group))]
    dist.all_gather(bufs, flat, group=group)
    parts = [{"step": b[:n_base], "first_cex": b[n_base:2 * n_base], "step_unflagged": b[2 * n_base:3 * n_base],
              "first_cex_unflagged": b[3 * n_base:]} for b in bufs]
    return merge_incremental(parts, n_base)
