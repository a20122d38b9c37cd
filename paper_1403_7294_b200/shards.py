"""Multi-GPU text sharding for the scan (BASELINE north_star:
"text sharded across 1/2/4/8 GPUs, automaton replicated, overlap-aware shard
boundaries, an NCCL allreduce of per-pattern counts and a host gather of
match lists").

This replaces the reference's dictionary partition (proj/include/acmatch/
partition.hpp:108-170, one automaton per pattern chunk, every worker reading
the whole text) with the data-parallel split the GPU wants: every rank holds
the whole automaton and scans a disjoint range of the text. A match belongs
to the rank whose range holds its END offset; a rank reads `halo` bytes
(>= the longest pattern) before its range so its automaton state is exact at
its first owned byte (window states equal whole-text states past maxlen
bytes). The per-rank match lists are therefore disjoint and, concatenated in
rank order, already in canonical (end, pattern_id) order — no merge.

One process per GPU (torch.distributed; NCCL on the GPU box, gloo in the CPU
tests). The only data-path exchange is the per-pattern count all-reduce and
the final gather of match lists; the scan itself needs no communication.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

ALIGN = 256  # shard boundaries on 256-byte multiples (32-byte vector loads stay aligned)


@dataclass(frozen=True)
class Shard:
    rank: int
    start: int      # first byte the rank reads (lo - halo, clamped at 0)
    lo: int         # first owned end offset
    hi: int         # one past the last owned end offset

    @property
    def emit_from(self) -> int:
        """Offset of `lo` inside the rank's window (acg_scanner_run's emit_from)."""
        return self.lo - self.start

    @property
    def window(self) -> int:
        return self.hi - self.start


def shard_span(n: int, world: int, rank: int, halo: int, align: int = ALIGN) -> Shard:
    """Rank `rank`'s share of an n-byte text: owned ends [lo, hi) and its read
    window [start, hi). Owned ranges tile [0, n) in rank order; boundaries sit
    on `align` multiples (trailing ranks may own nothing when n is small)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    if n < 0 or halo < 0:
        raise ValueError("n and halo must be non-negative")
    units = -(-n // align)
    per, extra = divmod(units, world)

    def edge(r: int) -> int:
        return min(n, (r * per + min(r, extra)) * align)

    lo, hi = edge(rank), edge(rank + 1)
    return Shard(rank, max(0, lo - halo), lo, hi)


def weak_shard(n_per_rank: int, world: int, rank: int, halo: int) -> Shard:
    """Weak scaling: rank r owns [r*n, (r+1)*n) of a world*n byte text."""
    lo = rank * n_per_rank
    return Shard(rank, max(0, lo - halo), lo, lo + n_per_rank)


def reduce_counts(counts, group=None):
    """All-reduce (sum) a per-pattern count tensor in place across ranks
    (NCCL on device tensors, gloo on CPU tensors). Returns the tensor."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(counts, op=dist.ReduceOp.SUM, group=group)
    return counts


def gather_matches(ids, ends, group=None, dst: int = 0):
    """Host gather of the per-rank match lists to rank `dst`, concatenated in
    rank order (= canonical order, since owned end ranges ascend with rank).
    ids/ends: 1-D torch tensors (uint32-compatible int64 / int64) on the
    collective's device. Only `dst` receives list data: the list sizes are
    all-gathered (one int64 per rank), then every other rank sends its exact
    (2, k) slice point-to-point. Returns (ids, ends) numpy arrays on `dst`,
    None on the other ranks."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return ids.cpu().numpy().astype(np.uint32), ends.cpu().numpy().astype(np.uint64)
    world = dist.get_world_size(group)
    me = dist.get_rank(group)
    if dist.get_backend(group) == "gloo":  # gloo's point-to-point path takes host tensors
        ids, ends = ids.cpu(), ends.cpu()
    dev = ids.device
    n_local = torch.tensor([ids.numel()], dtype=torch.int64, device=dev)
    sizes = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(sizes, n_local, group=group)
    sizes = [int(s.item()) for s in sizes]
    ranks = list(range(world)) if group is None else dist.get_process_group_ranks(group)
    if me != dst:
        if sizes[me]:
            mine = torch.stack([ids.to(torch.int64), ends.to(torch.int64)])
            dist.send(mine.contiguous(), dst=ranks[dst], group=None)
        return None
    out_ids, out_ends = [], []
    for r in range(world):
        k = sizes[r]
        if r == me:
            out_ids.append(ids.cpu().numpy())
            out_ends.append(ends.cpu().numpy())
        elif k:
            buf = torch.empty(2, k, dtype=torch.int64, device=dev)
            dist.recv(buf, src=ranks[r], group=None)
            b = buf.cpu().numpy()
            out_ids.append(b[0])
            out_ends.append(b[1])
    if not out_ids:
        return np.zeros(0, np.uint32), np.zeros(0, np.uint64)
    return np.concatenate(out_ids).astype(np.uint32), np.concatenate(out_ends).astype(np.uint64)


def run_shard(scanner, d_window_ptr: int, shard: Shard, stream: int = 0) -> None:
    """Enqueue this rank's scan: the device-resident window text[start, hi)
    at d_window_ptr, matches emitted from `lo` on, ends reported absolute."""
    scanner.run(d_window_ptr, shard.window, emit_from=shard.emit_from, base_offset=shard.start, stream=stream)
