"""GPU: the multi-GPU data path end to end with the real device scan.

Two processes share cuda:0 (only one GPU is available to the tests) and form
a world of 2 over gloo. Each rank runs the product path exactly as bench.py
does on N GPUs — its shard window resident on the device, Scanner.run through
shards.run_shard, the per-pattern counts copied device-to-device and
all-reduced (shards.reduce_counts on a CUDA tensor), the match lists gathered
to rank 0 (shards.gather_matches) — and rank 0 compares the result with the
reference's goldens / the oracle. The ranks never wait on each other's
kernels (the collectives run on the host), so sharing one GPU is safe.
"""
from __future__ import annotations

import hashlib
import json
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank: int, world: int, port: int, out_dir: str, cfg: int, n: int, mode: int) -> None:
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_1403_7294_b200 import acmatch as am
        from paper_1403_7294_b200 import shards, synth
        w = synth.CONFIGS[cfg] if n == 0 else synth.CONFIGS[cfg].scaled(n)
        concat, offs = synth.patterns(w)
        a = am.Automaton.from_arrays(concat, offs)
        sh = shards.shard_span(w.n, world, rank, a.layout()["halo"])
        d_text = torch.from_numpy(synth.text(w, sh.start, sh.hi)).cuda()
        sc = am.Scanner(a, 0, am.SCAN_LIST | am.SCAN_COUNTS)
        sc.set_mode(mode)
        stream = torch.cuda.Stream()
        counts = torch.zeros(a.pattern_count(), dtype=torch.int64, device="cuda")
        shards.run_shard(sc, d_text.data_ptr(), sh, stream=stream.cuda_stream)
        sc.sync()  # a first run may replay at sync (workspace sizing): counts are final after it
        sc.copy_pattern_counts(counts.data_ptr(), stream.cuda_stream)
        stream.synchronize()
        shards.reduce_counts(counts)
        ids, ends = sc.records()
        got = shards.gather_matches(torch.from_numpy(ids.astype(np.int64)), torch.from_numpy(ends.astype(np.int64)))
        if rank == 0:
            np.savez(os.path.join(out_dir, "r0.npz"), ids=got[0], ends=got[1], counts=counts.cpu().numpy())
        else:
            assert got is None
        dist.barrier()
    finally:
        dist.destroy_process_group()


def _run(tmp_path, cfg, n, mode):
    mp.get_context("spawn")
    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path), cfg, n, mode), nprocs=2, join=True)
    return np.load(tmp_path / "r0.npz")


@pytest.mark.parametrize("cfg,mode", [(0, 0), (1, 3), (3, 2), (4, 2)])
def test_two_ranks_one_gpu_small(tmp_path, cfg, mode):
    import oracle
    from paper_1403_7294_b200 import synth
    n = (3 << 20) + 4099
    r = _run(tmp_path, cfg, n, mode)
    w = synth.CONFIGS[cfg].scaled(n)
    concat, offs = synth.patterns(w)
    ids, ends, _, counts = oracle.OracleAutomaton(concat, offs).scan(synth.text(w), counts=True)
    assert np.array_equal(r["ends"], ends) and np.array_equal(r["ids"], ids)
    assert np.array_equal(r["counts"], counts.astype(np.int64))


def test_two_ranks_one_gpu_cfg0_full_golden(tmp_path):
    """BASELINE configs[0] at full size, split over 2 ranks: equals the reference's golden."""
    from paper_1403_7294_b200 import synth
    r = _run(tmp_path, 0, 0, 0)
    golden = json.load(open(os.path.join(ROOT, "tests", "golden", "configs_full.json")))
    case = next(c for c in golden["cases"] if c["name"] == synth.CONFIGS[0].name)
    assert len(r["ids"]) == case["m"]
    sha = hashlib.sha256(r["counts"].astype("<u8").tobytes()).hexdigest()
    assert sha == case["counts_sha256"]
    e = r["ends"].astype(np.uint64)
    i = r["ids"].astype(np.uint64)
    assert np.all((e[1:] > e[:-1]) | ((e[1:] == e[:-1]) & (i[1:] > i[:-1])))  # strict (end, id) order
    with np.errstate(over="ignore"):
        z = (e << np.uint64(20)) + i
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
        dsum = int(np.sum(z, dtype=np.uint64))
    dxor = int(np.bitwise_xor.reduce(z))
    assert (dsum, dxor) == (case["dsum"], case["dxor"])


def test_bench_two_ranks_strong_split_on_one_gpu():
    """bench.py's N-rank path (shards, counts all-reduced inside the timed step,
    max-over-ranks timing, the whole job's count/digest/order checks, the
    pipelined e2e leg per shard) with 2 ranks over gloo sharing cuda:0: a
    strong split of cfg2 at 64 MiB must give the same job result as 1 rank."""
    import subprocess
    import sys
    base = [sys.executable, "bench.py", "--config", "2", "--text-mib", "64", "--steps", "2", "--warmup", "3",
            "--no-cpu-baseline", "--e2e-steps", "1"]
    one = subprocess.run(base, capture_output=True, text=True, cwd=ROOT, timeout=900)
    assert one.returncode == 0, one.stderr[-3000:]
    port = _free_port()
    two = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                          "--master-addr", "127.0.0.1", "--master-port", str(port)] + base[1:] +
                         ["--gpus", "2", "--dist-backend", "gloo"], capture_output=True, text=True, cwd=ROOT,
                         timeout=900)
    assert two.returncode == 0, two.stderr[-3000:]
    j1 = json.loads(one.stdout.strip().splitlines()[-1])
    j2 = json.loads(two.stdout.strip().splitlines()[-1])
    assert j2["n_gpus"] == 2 and j2["scaling"] == "strong"
    for k in ("matches", "digest_sum", "digest_xor", "count_sum"):
        assert j2["check"][k] == j1["check"][k], k
    assert j2["check"]["unsorted_pairs"] == 0 and j2["check"]["timed_runs_replayed"] == 0
