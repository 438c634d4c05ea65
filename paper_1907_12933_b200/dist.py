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
    world = dist.get_world_size(group)
    bufs = [torch.empty_like(flat) for _ in range(world)]
    dist.all_gather(bufs, flat, group=group)
    return [unpack(b, n_base, n_words) for b in bufs]


def reduce_results(res: Dict, n_base: int, n_words: int, group=None, stream=None) -> Dict:
    """All-gather + GPU merge (sum counts, min counterexample indices, OR coverage words)."""
    import paper_1907_12933_b200 as P
    parts = allgather_results(res, n_base, n_words, group)
    return P.merge(parts, n_base, n_words, stream=stream)
