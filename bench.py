#!/usr/bin/env python3
"""Benchmark: Aho-Corasick text-scan throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config 1] [--scaling weak|strong] [--mode auto|filter|sparse|exact]

One step = one full pass of the hot path over the workload's text, producing
the canonical (end, pattern id) match list and the per-pattern counts (+ an
NCCL all-reduce of the counts when N > 1). `value` is text GB/s of the whole
job with the text already resident in HBM, device-timed (CUDA events, max over
ranks); `e2e` is the same metric through the public pipelined host scan
(acg_scan_pipelined) from pinned host memory: H2D of the text and D2H of the
packed match list and the per-pattern counts inside the timed region, piece
k+1's copy and scan overlapping piece k's read-back. The workload is BASELINE.json configs[1] (1 GiB iid ACGT,
10,000 patterns of 16-64 bytes) unless --config says otherwise.

Multi-GPU (one process per GPU): --scaling weak (default; cfg1) gives every
rank its own 1 GiB shard of one N GiB text; --scaling strong (default for
--config 2, BASELINE configs[2]) splits the config's text across the ranks
(shards.shard_span, overlap = the automaton's halo). In both, the combined
result of all ranks is checked: count, order-independent digest, order across
rank boundaries, all-reduced per-pattern counts (and the reference's golden
for the full-size strong split).

--impl reference times the reference's own CPU scan (oracle/_ref, the
unmodified reference headers compiled here) on the host cores: its only
parallel mode, the dictionary-partitioned run (proj/include/acmatch/
partition.hpp:108-170) with the per-worker builds hoisted out of the timed
region, over a bounded sample of the same text.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

HBM_FALLBACK_GBS = 6650.0  # B200_PROFILING.md fallback when MEASURED_PEAKS.json is absent
# one metric string for both arms (BASELINE.json "metric": text-scan GB/s); how
# each arm is timed goes in its "timing" field
METRIC = "AC text-scan GB/s"


# per-stage labels of acg_scanner_kernel_ms by scan mode
STAGES = {
    "filter": ("KQ_filter", "V1_confirm", "unused", "unused", "ORDER"),
    "sparse": ("K1s_walk", "K1f_fixup", "K2_prefix", "K3_write", "K4_counts"),
    "exact": ("walk", "E1_count", "K2_prefix", "E2_expand", "K4_counts"),
}


def golden_check(w, m: int, dsum: int, dxor: int, counts) -> str:
    """Compare the timed run's output with the reference's own statistics for
    this workload (tests/golden/configs_full.json, from oracle/make_goldens.py)."""
    import hashlib
    p = os.path.join(ROOT, "tests", "golden", "configs_full.json")
    try:
        with open(p) as f:
            case = next(c for c in json.load(f)["cases"] if c["name"] == w.name and c["n"] == w.n)
    except (OSError, StopIteration, ValueError):
        return "no golden for this workload"
    sha = hashlib.sha256(np.asarray(counts, dtype="<u8").tobytes()).hexdigest()
    ok = (m, dsum, dxor, sha) == (case["m"], case["dsum"], case["dxor"], case["counts_sha256"])
    return "bit-exact vs reference (count, digest, per-pattern counts)" if ok else "MISMATCH vs reference golden"


def peaks() -> tuple[float, str]:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return HBM_FALLBACK_GBS, "fallback"


class ClockSampler:
    """SM clocks + clock-event (throttle) reasons sampled through NVML every
    ~2 ms on a background thread DURING the timed region (nvidia-smi's own
    polling floor is too coarse for a sub-second region); nvidia-smi is the
    fallback when NVML is unavailable."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown"}

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.sm: list[float] = []
        self.max_sm: float | None = None
        self.reason_bits = 0
        self.samples = 0
        self._stop = threading.Event()
        self._h = None

    def _handle(self):
        import pynvml
        pynvml.nvmlInit()
        try:
            import torch
            pr = torch.cuda.get_device_properties(self.gpu)
            bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
            return pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            return pynvml.nvmlDeviceGetHandleByIndex(self.gpu)

    def _sample(self):
        import pynvml
        self.sm.append(float(pynvml.nvmlDeviceGetClockInfo(self._h, pynvml.NVML_CLOCK_SM)))
        get = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            pynvml.nvmlDeviceGetCurrentClocksThrottleReasons
        self.reason_bits |= int(get(self._h))
        self.samples += 1

    def _loop(self):
        while not self._stop.is_set():
            try:
                self._sample()
            except Exception:
                return
            self._stop.wait(0.002)

    def __enter__(self):
        try:
            import pynvml
            self._h = self._handle()
            self.max_sm = float(pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM))
            self._sample()
            self._t = threading.Thread(target=self._loop, daemon=True)
            self._t.start()
        except Exception:
            self._h = None
        return self

    def __exit__(self, *exc):
        if self._h is not None:
            self._stop.set()
            self._t.join(timeout=2)
            try:
                self._sample()
            except Exception:
                pass

    def summary(self) -> dict:
        if not self.sm:
            return self._smi_once()
        reasons = sorted(v for k, v in self.REASONS.items() if self.reason_bits & k)
        return {"sm_mhz": statistics.median(self.sm), "sm_max_mhz": self.max_sm, "reasons": reasons,
                "samples": self.samples, "source": "nvml"}

    def _smi_once(self) -> dict:
        q = "clocks.sm,clocks.max.sm"
        try:
            out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                  "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=20).stdout
            sm, mx = (float(x) for x in out.strip().split(","))
            return {"sm_mhz": sm, "sm_max_mhz": mx, "reasons": ["unsampled-during-region"], "source": "nvidia-smi"}
        except Exception:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}


def dist_env() -> tuple[int, int, int]:
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def cpu_reference(w, concat, offs, sample_bytes: int, threads: int | None, steps: int, warmup: int) -> dict:
    """The reference's CPU scan (oracle/_ref) on a bounded sample of the workload."""
    import ctypes as C
    import oracle
    from paper_1403_7294_b200 import synth
    sample = synth.text(w, 0, min(sample_bytes, w.n))
    if oracle.ref_available():
        R, kind = oracle.ref(), "reference"
    else:  # the oracle port stands in when the reference was not compiled
        R, kind = None, "port"
    cores = threads or os.cpu_count() or 1
    times = []
    m = C.c_uint64()
    if R is not None:
        h = R.ref_partitioned_prepare(concat.ctypes.data_as(C.c_void_p), offs.ctypes.data_as(C.c_void_p),
                                      len(offs) - 1, cores)
        workers = R.ref_partitioned_workers(h)
        for i in range(warmup + steps):
            t = R.ref_partitioned_scan(h, sample.ctypes.data_as(C.c_void_p), sample.size, C.byref(m))
            if i >= warmup:
                times.append(t)
        R.ref_partitioned_free(h)
    else:
        o = oracle.OracleAutomaton(concat, offs)
        workers = 1
        for i in range(warmup + steps):
            t0 = time.perf_counter()
            o.scan(sample, with_records=False)
            if i >= warmup:
                times.append(time.perf_counter() - t0)
    mean = sum(times) / len(times)
    return {"value": sample.size / mean / 1e9, "unit": "GB/s", "cores": workers, "kind": kind,
            "sample": f"first {sample.size >> 20} MiB of {w.name}; dictionary-partitioned reference run "
                      f"(split_patterns + per-worker build hoisted; threads each scan the sample, "
                      f"ids remapped, merge_matches), {workers} worker threads, mean of {len(times)}",
            "matches_in_sample": int(m.value), "seconds_per_step": mean}


def cpu_reference_single(w, concat, offs, sample_bytes: int) -> dict:
    """acmatch::scan(build(P), text) at 1 thread (oracle/_ref)."""
    import ctypes as C
    import oracle
    from paper_1403_7294_b200 import synth
    if not oracle.ref_available():
        return {}
    sample = synth.text(w, 0, min(sample_bytes, w.n))
    ra = oracle.RefAutomaton(concat, offs)
    R = oracle.ref()
    fol = C.c_uint64()
    t0 = time.perf_counter()
    m = R.ref_scan(ra._h, sample.ctypes.data_as(C.c_void_p), sample.size, C.byref(fol), None, None, 0)
    dt = time.perf_counter() - t0
    return {"value": sample.size / dt / 1e9, "unit": "GB/s", "cores": 1, "kind": "reference",
            "sample": f"acmatch::scan over the first {sample.size >> 20} MiB, 1 thread", "matches_in_sample": int(m)}


def run_reference_arm(args, w, concat, offs) -> None:
    """--impl reference: the reference's own CPU scan on the host cores (rank 0
    only; other ranks exit without work), same metric / config as our arm."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    cb = cpu_reference(w, concat, offs, args.cpu_sample_mib << 20, threads, args.steps, args.warmup)
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": round(cb["value"], 6),
        "unit": "GB/s",
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(cb["seconds_per_step"] * 1e3, 3),
        "higher_is_better": True,
        "scaling": scaling_of(args),
        "vs_baseline": None,
        "dtype": "u8",
        "data": "synthetic",
        "timing": "host wall clock per step (std::chrono inside the reference's run)",
        "config": {"workload": w.name, "text_bytes": w.n, "patterns": w.patterns,
                   "pattern_len": [w.len_lo, w.len_hi], "timed_sample_bytes": min(args.cpu_sample_mib << 20, w.n)},
        "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": round(cb["value"], 6), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def scaling_of(args) -> str:
    return args.scaling or ("strong" if args.config == 2 else "weak")


MODE_NAMES = ("auto", "sparse", "exact", "filter")


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--scaling", default=None, choices=["weak", "strong"])
    ap.add_argument("--cpu-sample-mib", type=int, default=32)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--e2e-piece-mib", type=int, default=256, help="pipelined e2e scan: piece size (MiB)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="tests only: gloo runs the N-rank logic with ranks sharing GPUs")
    ap.add_argument("--streams-per-thread", type=int, default=0)
    ap.add_argument("--threads-per-block", type=int, default=0)
    ap.add_argument("--chunk-bytes", type=int, default=0)
    ap.add_argument("--profile-layout", action="store_true", help="profile-guided hot-state order")
    ap.add_argument("--text-mib", type=int, default=0, help="experiments: scale the workload's text (MiB)")
    ap.add_argument("--no-counts", action="store_true", help="experiments: match list only (no per-pattern counts)")
    ap.add_argument("--mode", default="auto", choices=list(MODE_NAMES))
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    from paper_1403_7294_b200 import synth
    w = synth.CONFIGS[args.config]
    if args.text_mib:
        w = w.scaled(args.text_mib << 20)
    concat, offs = synth.patterns(w)

    if args.impl == "reference":
        run_reference_arm(args, w, concat, offs)
        return

    import torch
    import torch.distributed as dist
    from paper_1403_7294_b200 import acmatch as am
    from paper_1403_7294_b200 import shards

    rank, world, local = dist_env()
    if args.dist_backend == "gloo":  # logic test of the N-rank path on fewer GPUs (tests only; never a bench line)
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    scaling = scaling_of(args)

    am.version()  # load libacg (and its CUDA driver init) outside the build timing
    tb0 = time.perf_counter()
    a = am.Automaton.from_arrays(concat, offs)
    build_ms = (time.perf_counter() - tb0) * 1e3  # host build: trie, failure links, dense DFA, filters
    halo_guess = ((int((offs[1:] - offs[:-1]).max()) + 15) // 16) * 16
    from dataclasses import replace
    if scaling == "weak":
        # rank r owns [r*n, (r+1)*n) of a world*n byte text (the dictionary is the workload's)
        sh = shards.weak_shard(w.n, world, rank, halo_guess)
        wt = replace(w, n=world * w.n)
        job_bytes = world * w.n
    else:
        # the config's text split across the ranks
        sh = shards.shard_span(w.n, world, rank, halo_guess)
        wt = w
        job_bytes = w.n
    owned = sh.hi - sh.lo
    h_text = torch.empty(max(sh.window, 16), dtype=torch.uint8, pin_memory=True)
    synth.text(wt, sh.start, sh.hi, out=h_text.numpy())
    if args.profile_layout:
        a.optimize_layout(h_text.numpy()[: 1 << 20])
    lay = a.layout()
    assert lay["halo"] == halo_guess
    d_text = h_text.cuda()

    flags = am.SCAN_LIST | am.SCAN_PROFILE | (0 if args.no_counts else am.SCAN_COUNTS)
    sc = am.Scanner(a, local, flags)
    sc.set_geometry(args.streams_per_thread, args.threads_per_block, args.chunk_bytes)
    mode_req = {"auto": am.MODE_AUTO, "sparse": am.MODE_SPARSE, "exact": am.MODE_EXACT,
                "filter": am.MODE_FILTER}[args.mode]
    sc.set_mode(mode_req)
    stream = torch.cuda.Stream()
    P = a.pattern_count()
    counts_all = torch.zeros(P, dtype=torch.int64, device="cuda")

    def step():
        shards.run_shard(sc, d_text.data_ptr(), sh, stream=stream.cuda_stream)
        if world > 1:
            sc.copy_pattern_counts(counts_all.data_ptr(), stream.cuda_stream)
            with torch.cuda.stream(stream):
                shards.reduce_counts(counts_all)

    sc.set_profiling(False)  # stage events only in the profiled steps after the timed region
    for _ in range(args.warmup):
        step()
        sc.sync()  # adaptive sizes settle (record buffer, survivor regions, slabs) before timing
    replays0 = sc.replays()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        ev0.record(stream)
        h0 = time.perf_counter()
        for _ in range(args.steps):
            step()
        host_ms = (time.perf_counter() - h0) * 1e3 / args.steps
        ev1.record(stream)
        torch.cuda.synchronize()
    elapsed_ms = ev0.elapsed_time(ev1)
    # the timed runs' own result: sync (a workspace overflow would replay the run
    # here and show in the replay counter) and the size-independent checks
    sc.sync()
    timed_replayed = sc.replays() - replays0
    m_local = sc.match_count()
    dsum, dxor, unsorted = sc.digest()
    edge = [int(x) for x in sc.copy_records(0, 1)] + [int(x) for x in sc.copy_records(m_local - 1, 1)] \
        if m_local else []
    if args.no_counts:
        counts = np.zeros(P, dtype=np.uint64)
    elif world > 1:
        counts = counts_all.cpu().numpy().astype(np.uint64)  # all-reduced by the last timed step
    else:
        counts = sc.pattern_counts()
    mode_name, ev_rate = sc.last_mode()
    walk_name = sc.last_walk()  # exact mode: dense hot rows (KE) or the compressed hot automaton (KC)
    geo = sc.geometry()
    # per-stage times: profiled steps right after the timed region (same scanner,
    # stream, inputs and pipeline; CUDA events between the stages)
    sc.set_profiling(True)
    k1, prof_step = [], []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step()
        e1.record(stream)
        sc.sync()
        k1.append(sc.kernel_ms())
        prof_step.append(e0.elapsed_time(e1))
    k_ms = np.mean(np.array(k1), axis=0)
    prof_step_ms = float(np.mean(prof_step))
    replays_prof = sc.replays() - replays0 - timed_replayed
    if world > 1:
        t = torch.tensor([elapsed_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed_ms = float(t.item())
    ms_per_step = elapsed_ms / args.steps
    value = job_bytes / (ms_per_step * 1e-3) / 1e9

    # the whole job's result (all ranks): count, digest, order across shards
    mine = {"m": int(m_local), "dsum": int(dsum), "dxor": int(dxor), "unsorted": int(unsorted), "edge": edge,
            "replayed": int(timed_replayed)}
    parts = [mine]
    if world > 1:
        parts = [None] * world
        dist.all_gather_object(parts, mine)
    m_job = sum(p["m"] for p in parts)
    dsum_job = sum(p["dsum"] for p in parts) % (1 << 64)
    dxor_job = 0
    for p in parts:
        dxor_job ^= p["dxor"]
    edges = [p["edge"] for p in parts if p["edge"]]
    cross = sum(1 for x, y in zip(edges, edges[1:]) if not x[1] < y[0])
    unsorted_job = sum(p["unsorted"] for p in parts) + cross
    replayed_job = sum(p["replayed"] for p in parts)
    sc.__del__()  # release the timed scanner's workspace before the e2e scanner allocates its own

    # e2e: the public pipelined host scan (acg_scan_pipelined) from pinned host
    # memory: each step copies the shard's text H2D in pieces and reads the packed
    # records and per-pattern counts back into pinned host memory (piece k+1's
    # H2D and scan overlap piece k's D2H)
    h_out = torch.empty(max(m_local + 1024, 1), dtype=torch.int64, pin_memory=True).numpy().view(np.uint64)
    text_np = h_text.numpy()[: sh.window]
    e2e_kw = dict(device=local, piece_bytes=args.e2e_piece_mib << 20, out=h_out, emit_from=sh.lo - sh.start,
                  base_offset=sh.start)
    am.scan_pipelined(a, text_np, **e2e_kw)  # warm-up (workspaces, adaptive sizes)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    d2h = 0
    for _ in range(args.e2e_steps):
        recs, _bits, h_counts, m_e2e, _ = am.scan_pipelined(a, text_np, **e2e_kw)
        pieces = max(1, -(-owned // (args.e2e_piece_mib << 20)))
        d2h = recs.nbytes + pieces * h_counts.nbytes
    assert m_e2e == m_local, (m_e2e, m_local)
    e2e_s = (time.perf_counter() - t0) / args.e2e_steps
    if world > 1:
        t = torch.tensor([e2e_s], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_value = job_bytes / e2e_s / 1e9

    hbm, src = peaks()
    # roofline: algorithmic bytes of this rank's step = owned
    # text read once + 8 B per match record written + 8 B per pattern count,
    # over the device-timed step
    alg_bytes = owned + 8 * m_local + 8 * P
    achieved = alg_bytes / (ms_per_step * 1e-3) / 1e9
    stage_names = STAGES.get(mode_name, STAGES["exact"])
    kname = {"sparse": "sparse_scan_kernel (K1s)", "filter": "qfilter_ldg_kernel (KQ)"}.get(
        mode_name, "ctab_event_kernel (KC)" if walk_name == "ctab" else "exact_event_kernel (KE)")
    k_top = float(k_ms[0])
    traffic = None
    tf = os.path.join(ROOT, "profiles", "dram_traffic.json")
    if os.path.exists(tf):
        try:
            traffic = json.load(open(tf)).get(f"config{args.config}:{mode_name}")
        except Exception:
            traffic = None
    line = {
        "metric": METRIC,
        "value": round(value, 3),
        "unit": "GB/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_per_step, 4),
        "higher_is_better": True,
        "scaling": scaling,
        "vs_baseline": None,
        "dtype": "u8",
        "data": "synthetic",
        "timing": "device: CUDA events on the scan stream around the timed steps, max over ranks",
        "config": {"workload": w.name, "text_bytes_job": job_bytes, "text_bytes_rank0": owned, "patterns": P,
                   "pattern_len": [w.len_lo, w.len_hi], "dfa_states": lay["states"],
                   "hot_rows_smem": lay["hot_rows"], "alphabet": lay["alphabet"], "halo": lay["halo"],
                   "chunks": geo["n_chunks"], "chunk_bytes": geo["chunk_bytes"], "matches_job": m_job,
                   "l2": ("text per GPU > 126 MB L2: no flush needed" if owned > (126 << 20)
                          else "text per GPU fits L2: no flush (small parity config)"),
                   "parallelism": f"text shards x{world} ({scaling} scaling, halo {lay['halo']} B), DFA replicated",
                   "scan_mode": mode_name, "mode_requested": args.mode,
                   "exact_walk": walk_name if mode_name == "exact" else None,
                   "excursion_event_rate": round(ev_rate, 5)},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 2), "peak": hbm, "unit": "GB/s",
                     "frac": round(achieved / hbm, 4), "traffic": traffic,
                     "bytes": "SURVEY 8(d): owned text + 8*M + 8*P per step of rank 0",
                     "algorithmic_bytes_per_step": int(alg_bytes),
                     "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({src})",
                     "kernel": {"name": kname, "ms": round(k_top, 4),
                                "achieved": round(owned / (k_top * 1e-3) / 1e9, 2) if k_top > 0 else None,
                                "frac": round(owned / (k_top * 1e-3) / 1e9 / hbm, 4) if k_top > 0 else None,
                                "bytes": "owned text bytes per launch (the kernel reads the text once)"},
                     "stage_ms": dict(zip(stage_names, (round(float(x), 4) for x in k_ms))),
                     "profiled_step_ms": round(prof_step_ms, 4),
                     "host_enqueue_ms_per_step": round(host_ms, 4)},
        "e2e": {"value": round(e2e_value, 3), "unit": "GB/s", "h2d_bytes_per_step": int(sh.window),
                "d2h_bytes_per_step": int(d2h)},
        "build": {"ms": round(build_ms, 2), "host_threads": os.cpu_count(),
                  "what": "acg_build: trie + failure links + dense DFA + filter tables (SURVEY 8(f) rank 1)"},
        "gpu_launches": int(geo["launches"]) * args.steps,
        "clocks": clk.summary(),
        "check": {"matches": m_job, "digest_sum": dsum_job, "digest_xor": dxor_job,
                  "unsorted_pairs": unsorted_job, "count_sum": int(counts.sum()),
                  "timed_runs_replayed": replayed_job, "profiled_runs_replayed": int(replays_prof)},
    }
    if scaling == "strong" or world == 1:
        line["check"]["golden"] = golden_check(w, m_job, dsum_job, dxor_job, counts)
    else:
        line["check"]["golden"] = "no golden for the weak-scaled N GiB text (per-shard checks above)"
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cb = cpu_reference(w, concat, offs, args.cpu_sample_mib << 20, os.cpu_count(), 1, 0)
        line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
        single = cpu_reference_single(w, concat, offs, min(args.cpu_sample_mib, 16) << 20)
        if single:
            line["cpu_baseline"]["single_thread"] = {k: single[k] for k in ("value", "unit", "cores", "sample")}
        import oracle
        tr0 = time.perf_counter()
        oracle.RefAutomaton(concat, offs)
        line["build"]["reference_ms"] = round((time.perf_counter() - tr0) * 1e3, 2)  # acmatch::build, 1 thread
        if args.config == 0 and (os.cpu_count() or 1) != 16:  # BASELINE configs[0]: 1 and 16 threads
            c16 = cpu_reference(w, concat, offs, args.cpu_sample_mib << 20, 16, 1, 0)
            line["cpu_baseline"]["threads_16"] = {k: c16[k] for k in ("value", "unit", "cores", "sample")}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
