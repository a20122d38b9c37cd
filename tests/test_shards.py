"""CPU: host logic of the multi-GPU text sharding (paper_1403_7294_b200/shards.py).

The shard geometry is checked exhaustively on small sizes, and the full
N>1 path — shard windows with halos, per-pattern count all-reduce, rank-order
gather of match lists — runs with world_size 2 over gloo, each rank's
device scan stood in for by the oracle's windowed scan of the same window.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1403_7294_b200 import shards


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("n", [0, 1, 255, 256, 257, 4096, 10_000, 1 << 20])
def test_shard_span_tiles_the_text(n, world):
    halo = 48
    spans = [shards.shard_span(n, world, r, halo) for r in range(world)]
    assert spans[0].lo == 0 and spans[-1].hi == n
    for a, b in zip(spans, spans[1:]):
        assert a.hi == b.lo  # disjoint, contiguous, rank order
    for s in spans:
        assert s.lo <= s.hi
        assert s.start == max(0, s.lo - halo)
        assert s.emit_from == s.lo - s.start and s.window == s.hi - s.start
        assert s.lo % shards.ALIGN == 0 or s.lo == n
    sizes = [s.hi - s.lo for s in spans]
    assert max(sizes) - min(sizes) <= 2 * shards.ALIGN or n < world * shards.ALIGN


def test_shard_span_rejects_bad_rank():
    with pytest.raises(ValueError):
        shards.shard_span(100, 2, 2, 8)
    with pytest.raises(ValueError):
        shards.shard_span(100, 0, 0, 8)


def test_weak_shard():
    s = shards.weak_shard(1 << 20, 4, 3, 64)
    assert (s.start, s.lo, s.hi) == (3 * (1 << 20) - 64, 3 * (1 << 20), 4 * (1 << 20))
    assert shards.weak_shard(1 << 20, 4, 0, 64).start == 0


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank: int, world: int, port: int, out_dir: str, n: int, cfg: int) -> None:
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_1403_7294_b200 import synth
        w = synth.CONFIGS[cfg].scaled(n)
        concat, offs = synth.patterns(w)
        a = oracle.OracleAutomaton(concat, offs)
        sh = shards.shard_span(n, world, rank, halo=a.max_len())
        window = synth.text(w, sh.start, sh.hi)
        # the rank's "device scan": window scan from the root, ends >= lo kept
        ids, ends, _, counts = a.scan(window, start=0, emit_from=sh.emit_from, counts=True)
        ends = ends + sh.start
        c = shards.reduce_counts(torch.from_numpy(counts.astype(np.int64)))
        got = shards.gather_matches(torch.from_numpy(ids.astype(np.int64)), torch.from_numpy(ends.astype(np.int64)))
        if rank == 0:
            np.savez(os.path.join(out_dir, "r0.npz"), ids=got[0], ends=got[1], counts=c.numpy())
        else:
            assert got is None
        dist.barrier()
    finally:
        dist.destroy_process_group()


# adversarial (deep failure chains across the boundary) and protein (dense short matches)
@pytest.mark.parametrize("cfg,n", [(4, (1 << 18) + 77), (3, 3000)])
def test_two_rank_gloo_shards_equal_whole_scan(tmp_path, cfg, n):
    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path), n, cfg), nprocs=2, join=True)
    r = np.load(tmp_path / "r0.npz")
    import oracle
    from paper_1403_7294_b200 import synth
    w = synth.CONFIGS[cfg].scaled(n)
    concat, offs = synth.patterns(w)
    ids, ends, _, counts = oracle.OracleAutomaton(concat, offs).scan(synth.text(w), counts=True)
    assert np.array_equal(r["ids"], ids) and np.array_equal(r["ends"], ends)
    assert np.array_equal(r["counts"], counts.astype(np.int64))
    assert len(ids) > 0
