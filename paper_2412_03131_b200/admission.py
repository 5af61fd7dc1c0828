"""Multi-GPU plumbing of the path: head sharding and the per-step count all-reduce.

P:555-556: "each worker includes a dedicated memory manager that oversees the KV cache for its assigned
attention heads" — GPU g owns KV heads [g*H/G, (g+1)*H/G) of every request and layer, in an independent
pool; no KV byte crosses GPUs.  The only exchange is one all-reduce (MIN) of the pools' int64[4]
admission counters {free_pages, -last_demand, -used_pages, status} per step, which the scheduler
(it "batches as many requests as possible within the available GPU memory") uses to admit a
request only if EVERY GPU has room for its shard.  torch.distributed (NCCL on GPUs, gloo in CPU tests)
carries it on a side stream; the counters are written by dkv_compact_alloc inside the arena.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch


def shard_heads(num_kv_heads: int, world: int, rank: int):
    """(first global KV head, heads on this rank).  Every BASELINE config has 8 KV heads, so 1/2/4/8-way
    sharding is even; otherwise extra GPUs could only hold replicas (not supported here)."""
    if num_kv_heads % world:
        raise ValueError(f"{num_kv_heads} KV heads do not shard evenly over {world} GPUs")
    hl = num_kv_heads // world
    return rank * hl, hl


def count_allreduce(stats: torch.Tensor, out: torch.Tensor | None = None, group=None, stream=None, async_op=False):
    """MIN all-reduce of the int64[4] admission counters.  `stats` may be the pool's device view; it is
    copied so the pool's own counters stay untouched.  Returns (result tensor, work handle or None)."""
    import torch.distributed as dist
    out = stats.clone() if out is None else out.copy_(stats)
    if stream is not None:
        with torch.cuda.stream(stream):
            w = dist.all_reduce(out, op=dist.ReduceOp.MIN, group=group, async_op=async_op)
    else:
        w = dist.all_reduce(out, op=dist.ReduceOp.MIN, group=group, async_op=async_op)
    return out, w


@dataclass
class Admission:
    """Admission rule on the reduced counters (one-step lag): a request whose shard needs at most
    `prefill_pages` pages on every GPU is admitted if min_g free_g >= prefill_pages + decode_reserve,
    where decode_reserve covers one page per active unit for the next decode step."""
    decode_reserve: int

    def free_min(self, reduced) -> int:
        return int(reduced[0])

    def healthy(self, reduced) -> bool:
        return int(reduced[3]) == 0                     # status <= 0: MIN == 0 <=> no GPU has a pending error

    def admit(self, reduced, prefill_pages: int) -> bool:
        return self.healthy(reduced) and self.free_min(reduced) >= prefill_pages + self.decode_reserve


def prefill_page_bound(prompt_len: int, window: int, c_high: int, units: int) -> int:
    """Upper bound on the pages one request's shard needs at admission: every stored token High
    (ceil((n - W)/C_h) pages per unit, the paper's conservative bound) plus one page per unit for
    the ceil of the low section."""
    stored = max(prompt_len - window, 0)
    return units * (-(-stored // c_high) + 1)
