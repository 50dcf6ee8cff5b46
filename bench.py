#!/usr/bin/env python
"""bench.py — PLAID four-stage search on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl plaid|reference]
                    [--config cfg2] [--score-mode exact|tensor] [--cpu-seconds S]

One step = one query through all four stages (single-query latency mode,
BASELINE.json configs[1]: synthetic MS MARCO v1 scale, 8.8M passages, 2^18
centroids, nbits=2, k=1000 with default_params_for_k).  Inputs are resident in
HBM when the timed region starts; L2 is flushed (256 MiB write; --flush
write+read adds a 256 MiB read sweep so no dirty line of the flush is written
back inside the timed region — measured to make no difference) before every
step, outside the timed interval.  Each step is bracketed by CUDA events on
the launching stream; the job time is the max over ranks of the summed step
times, `value` = queries / that time.

Multi-GPU (torchrun, one process per GPU): every rank holds a passage-range
shard of the same size (weak scaling: the index grows with N), runs the full
pipeline on its shard and the per-shard top-k lists are merged with an NCCL
all-gather + a device-side merge — all inside the timed step.

`--impl reference` times the reference's own CPU searcher (oracle/_ref, the
unmodified /root/reference sources compiled by oracle/Makefile) on the box's
host cores, on the same synthetic index and queries; rank 0 only.
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
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

CONFIGS = {
    "cfg1": dict(N=10_000, K=4096, nbits=2, mean_len=64, k=10,
                 desc="synthetic 10k-passage index (~64 tok/passage, dim 128, 4096 centroids, nbits=2), k=10"),
    "cfg2": dict(N=8_800_000, K=1 << 18, nbits=2, mean_len=68, k=1000,
                 desc="synthetic MS MARCO v1-scale: 8.8M passages (~600M embeddings), 2^18 centroids, "
                      "nbits=2, k=1000, single-query latency"),
    "cfg3": dict(N=8_800_000, K=1 << 18, nbits=1, mean_len=68, k=100, batch=1024,
                 desc="same MS MARCO-scale index, nbits=1, batched 1024-query throughput, k=100"),
    "cfg4": dict(N=2_400_000, K=1 << 16, nbits=2, mean_len=136, k=10,
                 desc="synthetic LoTTE-pooled-scale: 2.4M passages, 2^16 centroids, nbits=2, k=10, ndocs=256"),
    "small": dict(N=200_000, K=1 << 14, nbits=2, mean_len=68, k=1000, desc="smoke-size index"),
}
METRIC = "queries/sec @k=1000 & p50 latency vs HBM/tensor roofline, 1/2/4/8 B200"
QLEN, DIM = 32, 128


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), float(d["bf16_tflops"]), "measured"
    return 6650.0, 1590.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


class L2Flush:
    """Untimed cold-L2 reset before every step: write a 256 MiB buffer (twice
    the 126 MB L2), then (mode "write+read") read a second 256 MiB buffer so
    the dirty lines of the write are evicted before the timed region instead
    of being written back during it."""

    def __init__(self, mode: str):
        import torch

        self.mode = mode
        self.w = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
        self.r = torch.ones(64 << 20, dtype=torch.int32, device="cuda") if mode == "write+read" else None

    def __call__(self):
        self.w.zero_()
        if self.r is not None:
            self.r.max()

    def describe(self) -> str:
        return self.describe_mode(self.mode)

    @staticmethod
    def describe_mode(mode: str) -> str:
        return ("256 MiB write + 256 MiB read sweep before every step (untimed; L2 cold and clean)"
                if mode == "write+read" else "256 MiB write before every step (untimed)")


def make_index(cfg: dict, rank: int, seed: int = 0):
    import paper_2205_09707_b200 as P

    t = time.time()
    h = P.generate_index(cfg["N"], cfg["K"], dim=DIM, nbits=cfg["nbits"], mean_len=cfg["mean_len"],
                         spread=16, seed=seed, pid_base=rank * cfg["N"])
    log(f"[rank {rank}] generated shard: N={h.num_passages} T={h.num_embeddings} P={len(h.ivf_postings)} "
        f"({h.nbytes() / 1e9:.1f} GB) in {time.time() - t:.1f}s")
    return h


def params_for(cfg: dict):
    import paper_2205_09707_b200 as P

    p = P.default_params_for_k(cfg["k"])
    if "ndocs" in cfg:
        p.ndocs = cfg["ndocs"]
    return p


def cpu_reference_run(h, qs, params, steps, warmup, threads):
    """Latency mode: sequential lir::search, threads = all host cores."""
    import oracle

    ref = oracle.get("ref")
    t = time.time()
    ref.ref_handle(h)
    log(f"reference index built in {time.time() - t:.1f}s")
    nq = qs.shape[0]
    for i in range(warmup):
        ref.search(h, qs[i % nq], params, threads=threads)
    lat = []
    for i in range(steps):
        t0 = time.perf_counter()
        ref.search(h, qs[(warmup + i) % nq], params, threads=threads)
        lat.append(time.perf_counter() - t0)
    ref.release(h)
    return lat


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle

    if not oracle.available("ref"):
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/liblir_ref.so not built"}))
        return
    import paper_2205_09707_b200 as P

    h = make_index(cfg, 0)
    qs = P.generate_queries(h, max(args.steps + args.warmup, 1), qlen=QLEN, seed=1234)
    params = params_for(cfg)
    threads = os.cpu_count() or 1
    B = int(cfg.get("batch", 1))
    if B > 1:
        # throughput mode: `threads` workers x SearchOptions.threads=1;
        # each step is a bounded sample of the batch (~1 s of CPU work)
        ref = oracle.get("ref")
        qb = P.generate_queries(h, threads * 4, qlen=QLEN, seed=1234)
        ref.search_many(h, qb[:threads], params, 1, threads)  # warm-up (+ index build)
        lat = []
        for i in range(args.steps):
            t0 = time.perf_counter()
            ref.search_many(h, qb, params, 1, threads)
            lat.append(time.perf_counter() - t0)
        total = sum(lat)
        qps = len(qb) * args.steps / total
        sample = f"{len(qb)} queries per step, lir::search throughput mode ({threads} workers x threads=1)"
    else:
        lat = cpu_reference_run(h, qs, params, args.steps, args.warmup, threads)
        total = sum(lat)
        qps = args.steps / total
        sample = f"{args.steps} sequential queries, lir::search latency mode, SearchOptions.threads={threads}"
    line = {
        "impl": "reference", "metric": METRIC, "value": qps, "unit": "queries/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "p50_ms": 1e3 * statistics.median(lat), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (SplitMix64 generator, SURVEY.md §8d)",
        "config": config_block(cfg, params, args, 1),
        "cpu_baseline": {"value": qps, "unit": "queries/s", "cores": threads, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": qps, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def config_block(cfg, params, args, world):
    return {"workload": f"{args.config}: {cfg['desc']}", "passages_per_gpu": cfg["N"],
            "passages_total": cfg["N"] * world, "centroids": cfg["K"], "nbits": cfg["nbits"], "dim": DIM,
            "query_tokens": QLEN, "k": params.k, "nprobe": params.nprobe, "t_cs": params.t_cs,
            "ndocs": params.ndocs, "batch": cfg.get("batch", 1),
            "lanes": args.lanes if cfg.get("batch", 1) > 1 else None,
            "l2_flush": L2Flush.describe_mode(args.flush),
            "score_mode": args.score_mode, "parallelism": f"passage-range shards x{world}",
            "shard_merge": args.shard_mode if world > 1 else None}


def run_plaid(args, cfg):
    import torch

    import paper_2205_09707_b200 as P

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("PLAID_DIST_BACKEND", "nccl") != "nccl":
        local = 0  # several ranks share one GPU (test of the multi-rank path)
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        # PLAID_DIST_BACKEND=gloo lets a 1-GPU box run several ranks on one GPU
        # (exercise of the multi-rank path only; NCCL is the product backend)
        backend = os.environ.get("PLAID_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)

    h = make_index(cfg, rank)
    params = params_for(cfg)
    nq = max(args.steps + args.warmup, 8)
    # queries: generated from shard 0's passages, identical on every rank
    if rank == 0:
        qs = P.generate_queries(h, nq, qlen=QLEN, seed=1234)
    else:
        qs = np.zeros((nq, QLEN, DIM), dtype=np.float32)
    dq = torch.from_numpy(qs).cuda()
    if dist is not None:
        dist.broadcast(dq, 0)
        qs = dq.cpu().numpy()

    t = time.time()
    idx = P.DeviceIndex.from_host_at(h, pid_base=rank * cfg["N"], device=local)
    log(f"[rank {rank}] index resident on cuda:{local}: {idx.device_bytes / 1e9:.1f} GB in {time.time() - t:.1f}s")
    mode = P.ScoreMode.EXACT if args.score_mode == "exact" else P.ScoreMode.TENSOR
    # the timed searcher records no phase events (an event between two kernels
    # breaks their programmatic-dependent-launch overlap); a second searcher
    # with phase events measures the per-stage breakdown after the timed loop
    s = P.Searcher(idx, device=local, score_mode=mode, record_times=False, use_graphs=args.graphs)
    s_ph = P.Searcher(idx, device=local, score_mode=mode, record_times=True)

    k = params.k
    # a dedicated (non-default) stream: the kernels, the L2 flush and the timing
    # events all go to it, so CUDA events bracket exactly the enqueued search
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    sh = stream.cuda_stream
    d_pids = torch.zeros(k, dtype=torch.int32, device="cuda")
    d_scores = torch.zeros(k, dtype=torch.float32, device="cuda")
    d_n = torch.zeros(1, dtype=torch.int64, device="cuda")
    if world > 1:
        from paper_2205_09707_b200.sharded import ShardedSearcher

        ss = ShardedSearcher(s, k, device=torch.device("cuda", local), mode=args.shard_mode,
                             num_passages=cfg["N"] * world)
        m_pids, m_scores = ss.out_pids, ss.out_scores
    flush = L2Flush(args.flush)

    def step(i):
        q = dq[i % nq]
        if world > 1:
            # global-exact: stages 1-2, all-gather of the top-ndocs keys, filter +
            # stage 3, all-gather of the stage-3 keys, filter + stage 4, then
            # all-gather of k (pid, score) and the merge
            ss.search(q, params, stream=sh)
        else:
            s.search_device(q.data_ptr(), 1, QLEN, DIM, params, d_pids.data_ptr(), d_scores.data_ptr(),
                            d_n.data_ptr(), stream=sh)

    for i in range(args.warmup):
        flush()
        step(i)
    torch.cuda.synchronize()
    s.sync()

    phases = {n: [] for n in P.Searcher.PHASES}
    launches = 0
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    clocks = ClockSampler(local)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    for i in range(args.steps):
        flush()
        ev[i][0].record(stream)
        step(args.warmup + i)
        ev[i][1].record(stream)
        ev[i][1].synchronize()
        launches += s.last_launches()
    torch.cuda.synchronize()
    clk = clocks.stop()
    s.sync()
    # per-stage breakdown (phase events; untimed pass over the same queries)
    for i in range(args.steps):
        flush()
        q = dq[(args.warmup + i) % nq]
        s_ph.search_device(q.data_ptr(), 1, QLEN, DIM, params, d_pids.data_ptr(), d_scores.data_ptr(),
                           d_n.data_ptr(), stream=sh)
        for n, v in s_ph.phase_ms().items():
            phases[n].append(v)
    s_ph.sync()
    step_ms = torch.tensor([a.elapsed_time(b) for a, b in ev], dtype=torch.float64, device="cuda")
    if dist is not None:
        dist.all_reduce(step_ms, op=dist.ReduceOp.MAX)
        dist.barrier()
    step_ms = step_ms.cpu().numpy()
    total_s = float(step_ms.sum()) / 1e3
    value = args.steps / total_s

    # ---- end to end through the C ABI with host buffers (H2D of Q, D2H of top-k inside)
    e2e_lat = []
    if world == 1:
        for i in range(args.steps):
            flush()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r = s.search(qs[(args.warmup + i) % nq], params)
            e2e_lat.append(time.perf_counter() - t0)
        trace = r.trace
    else:
        hq = torch.from_numpy(qs).pin_memory()
        hp = torch.zeros(k, dtype=torch.int32).pin_memory()
        hs = torch.zeros(k, dtype=torch.float32).pin_memory()
        for i in range(args.steps):
            flush()
            torch.cuda.synchronize()
            dist.barrier()
            t0 = time.perf_counter()
            dq[0].copy_(hq[(args.warmup + i) % nq], non_blocking=True)
            step(0)
            hp.copy_(m_pids, non_blocking=True)
            hs.copy_(m_scores, non_blocking=True)
            torch.cuda.synchronize()
            e2e_lat.append(time.perf_counter() - t0)
        trace = None
        lat_t = torch.tensor(e2e_lat, dtype=torch.float64, device="cuda")
        dist.all_reduce(lat_t, op=dist.ReduceOp.MAX)
        e2e_lat = lat_t.cpu().tolist()
    e2e_value = args.steps / sum(e2e_lat)

    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant kernel: the S_cq kernel (the largest single
    # launch of a search; the engine's "scores" phase events bracket it alone).
    # Algorithmic bytes per launch: C read once (512 B per
    # centroid at d=128), S written once (128 B per centroid), keep bits (1 bit
    # per centroid) and Q (16 KiB).  3xTF32 FLOPs (3 * 2*K*d*|Q| = 6.4 GFLOP at
    # cfg2) take ~6 us at the dense tf32 rate, so the kernel is HBM-bound.
    hbm_peak, tf_peak, peak_kind = measured_peaks()
    mean_ph = {n: float(np.mean(v)) for n, v in phases.items()}
    K = cfg["K"]
    tr = trace.counters() if trace is not None else {}
    ab = 512 * K + 128 * K + K // 8 + QLEN * DIM * 4
    ach = ab / (mean_ph["scores"] * 1e-3) / 1e9
    kname = "scores_tf32_kernel" if args.score_mode == "tensor" else "scores_exact_kernel"
    traffic = None
    tf = ROOT / "profiles" / "traffic.json"
    if tf.exists():
        t = json.loads(tf.read_text()).get(f"{args.config}/{kname}")
        traffic = t.get("dram_bytes_per_launch") if t else None
    roof = {"bound": "hbm", "kernel": kname, "achieved": ach, "peak": hbm_peak, "unit": "GB/s",
            "frac": ach / hbm_peak, "traffic": traffic, "peak_kind": f"{peak_kind} (copy bandwidth, burst)",
            "algorithmic_bytes_per_launch": ab, "mean_ms": mean_ph["scores"],
            "share_of_step": mean_ph["scores"] / (1e3 * total_s / args.steps)}
    # context: the live-measured rate of a plain one-pass read of C's size on
    # this GPU (event-timed like the kernel) — the practical floor of a kernel
    # that streams C once
    try:
        import ctypes as _C

        from paper_2205_09707_b200 import _native as _N

        g = _C.c_double()
        if _N.load().plaid_measure_read_gbs(local, 512 * K, 5, _C.byref(g)) == 0 and g.value > 0:
            roof["read_floor_gbs"] = g.value
            roof["read_floor_note"] = f"plain coalesced read of {512 * K >> 20} MiB (C's size), L2 flushed, best of 5"
            roof["frac_of_read_floor"] = ach / g.value  # same algorithmic bytes as `achieved`
    except Exception:  # noqa: BLE001
        pass

    # ---- stage 4 (decompress + exact MaxSim) against its own bound: exactness
    # forbids FMA and tensor cores, so every (token, query token, dim) is one
    # rounded multiply and one rounded add on the FP32 pipe;
    # peak = SMs x 128 lanes x max SM clock.  Duration = the stage-4 phase
    # (scan + fused decompress/MaxSim + finalize), i.e. conservative.
    roof4 = None
    t4 = trace.decompressed_tokens if trace is not None else 0
    if t4:
        import torch as _t

        props = _t.cuda.get_device_properties(local)
        clk_mhz = (clk or {}).get("sm_max_mhz") or 1965.0
        peak_ops = props.multi_processor_count * 128 * clk_mhz * 1e6 / 1e12
        ops = 2.0 * QLEN * DIM * t4
        ach = ops / (mean_ph["stage4_rank"] * 1e-3) / 1e12
        bytes4 = t4 * (4 + DIM * cfg["nbits"] // 8)
        roof4 = {"bound": "fp32", "kernel": "stream_fused_kernel (+ scan, finalize)", "achieved": ach,
                 "peak": peak_ops, "unit": "Tops/s (fp32 lane-ops: separate mul + add)", "frac": ach / peak_ops,
                 "tokens": t4, "ops_per_launch": ops, "code_and_residual_bytes": bytes4,
                 "mean_ms": mean_ph["stage4_rank"]}

    # ---- CPU baseline: the reference's own searcher on this host, bounded sample
    cpu = None
    if world == 1 and not args.no_cpu:
        try:
            threads = os.cpu_count() or 1
            per_q = 0.5 if cfg["N"] > 1_000_000 else 0.02
            nsample = max(3, min(64, int(args.cpu_seconds / per_q)))
            lat = cpu_reference_run(h, qs, params, nsample, 1, threads)
            cpu = {"value": nsample / sum(lat), "unit": "queries/s", "cores": threads, "kind": "reference",
                   "sample": f"{nsample} sequential queries of the same workload, lir::search latency mode, "
                             f"SearchOptions.threads={threads}", "p50_ms": 1e3 * statistics.median(lat)}
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "unit": "queries/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"failed: {e}"}

    line = {
        "metric": METRIC, "value": value, "unit": "queries/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * total_s / args.steps,
        "p50_ms": float(np.median(step_ms)), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (SplitMix64 generator, SURVEY.md §8d)",
        "config": config_block(cfg, params, args, world),
        "e2e": {"value": e2e_value, "unit": "queries/s", "h2d_bytes_per_step": QLEN * DIM * 4,
                "d2h_bytes_per_step": k * 8 + 128, "p50_ms": 1e3 * statistics.median(e2e_lat)},
        "gpu_launches": launches,
        "roofline": roof,
        "roofline_stage4": roof4,
        "phases_ms": mean_ph,
        "trace": tr,
        "cpu_baseline": cpu,
        "clocks": clk,
    }
    print(json.dumps(line))
    if dist is not None:
        dist.destroy_process_group()


def run_plaid_batch(args, cfg):
    """Throughput mode (BASELINE configs[2]): one step = one batch of B queries
    through BatchSearcher (L concurrent lanes); value = queries / job time.
    Multi-GPU: every rank searches its passage shard (shard-local), the [B][k]
    results are all-gathered once per batch and merged per query."""
    import torch

    import paper_2205_09707_b200 as P

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    backend = os.environ.get("PLAID_DIST_BACKEND", "nccl")
    if backend != "nccl":
        local = 0
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    B = int(cfg["batch"])
    h = make_index(cfg, rank)
    params = params_for(cfg)
    k = params.k
    nb = 2  # distinct batches, alternated
    if rank == 0:
        qs = P.generate_queries(h, nb * B, qlen=QLEN, seed=1234).reshape(nb, B, QLEN, DIM)
    else:
        qs = np.zeros((nb, B, QLEN, DIM), dtype=np.float32)
    dq = torch.from_numpy(qs).cuda()
    if dist is not None:
        dist.broadcast(dq, 0)
        qs = dq.cpu().numpy()
    idx = P.DeviceIndex.from_host_at(h, pid_base=rank * cfg["N"], device=local)
    mode = P.ScoreMode.EXACT if args.score_mode == "exact" else P.ScoreMode.TENSOR
    bs = P.BatchSearcher(idx, lanes=args.lanes, device=local, score_mode=mode)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    sh = stream.cuda_stream
    d_pids = torch.zeros(B * k, dtype=torch.int32, device="cuda")
    d_scores = torch.zeros(B * k, dtype=torch.float32, device="cuda")
    d_n = torch.zeros(B, dtype=torch.int64, device="cuda")
    if dist is not None:
        g_pids = torch.zeros(world * B * k, dtype=torch.int32, device="cuda")
        g_scores = torch.zeros(world * B * k, dtype=torch.float32, device="cuda")
        g_n = torch.zeros(world * B, dtype=torch.int64, device="cuda")
        m_pids = torch.zeros(B * k, dtype=torch.int32, device="cuda")
        m_scores = torch.zeros(B * k, dtype=torch.float32, device="cuda")
        m_n = torch.zeros(B, dtype=torch.int64, device="cuda")
        merger = P.Searcher(None, device=local)
    flush = L2Flush(args.flush)

    def step(i):
        q = dq[i % nb]
        bs.search_device(q.data_ptr(), B, QLEN, DIM, params, d_pids.data_ptr(), d_scores.data_ptr(),
                         d_n.data_ptr(), stream=sh)
        if dist is not None:
            from paper_2205_09707_b200.sharded import _all_gather

            _all_gather(g_pids, d_pids, None)
            _all_gather(g_scores, d_scores, None)
            _all_gather(g_n, d_n, None)
            # shard g's query j list at g*B*k + j*k (stride B*k per shard); counts
            # regrouped per query: cnt[j][g]
            cnt = g_n.view(world, B).t().contiguous()
            for j in range(B):
                merger.merge_topk_device(g_pids.data_ptr() + 4 * j * k, g_scores.data_ptr() + 4 * j * k,
                                         cnt.data_ptr() + 8 * j * world, world, B * k, k,
                                         m_pids.data_ptr() + 4 * j * k, m_scores.data_ptr() + 4 * j * k,
                                         m_n.data_ptr() + 8 * j, stream=sh)

    for i in range(args.warmup):
        flush()
        step(i)
    torch.cuda.synchronize()
    bs.sync()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    clocks = ClockSampler(local)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    launches = 0
    for i in range(args.steps):
        flush()
        ev[i][0].record(stream)
        step(args.warmup + i)
        ev[i][1].record(stream)
        launches += bs.last_launches()
    torch.cuda.synchronize()
    clk = clocks.stop()
    bs.sync()
    step_ms = torch.tensor([a.elapsed_time(b) for a, b in ev], dtype=torch.float64, device="cuda")
    if dist is not None:
        dist.all_reduce(step_ms, op=dist.ReduceOp.MAX)
    step_ms = step_ms.cpu().numpy()
    total_s = float(step_ms.sum()) / 1e3
    value = B * args.steps / total_s

    # e2e through the host API (H2D of the batch, D2H of [B][k] results inside)
    e2e_lat = []
    if world == 1:
        for i in range(args.steps):
            flush()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            bs.search(qs[i % nb], params)
            e2e_lat.append(time.perf_counter() - t0)
        e2e_value = B * args.steps / sum(e2e_lat)
    else:
        e2e_value = None
    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return

    # S_cq kernel alone (one single-query search with phase events) for the roofline
    s1 = P.Searcher(idx, device=local, score_mode=mode, record_times=True)
    sc_ms = []
    for i in range(5):
        flush()
        torch.cuda.synchronize()
        s1.search(qs[0][i], params)
        sc_ms.append(s1.phase_ms()["scores"])
    sc = float(np.median(sc_ms[1:]))
    hbm_peak, _, peak_kind = measured_peaks()
    K = cfg["K"]
    ab = 512 * K + 128 * K + K // 8 + QLEN * DIM * 4
    kname = "scores_tf32_kernel" if args.score_mode == "tensor" else "scores_exact_kernel"
    roof = {"bound": "hbm", "kernel": kname, "achieved": ab / (sc * 1e-3) / 1e9, "peak": hbm_peak, "unit": "GB/s",
            "frac": ab / (sc * 1e-3) / 1e9 / hbm_peak, "traffic": None,
            "peak_kind": f"{peak_kind} (copy bandwidth, burst)", "algorithmic_bytes_per_launch": ab,
            "mean_ms": sc, "share_of_step": sc * B / (1e3 * total_s / args.steps),
            "note": "one S_cq launch per query (single-query kernel; the batch's launches serialise)"}
    cpu = None
    if world == 1 and not args.no_cpu:
        try:
            import oracle

            threads = os.cpu_count() or 1
            ref = oracle.get("ref")
            ns = max(threads, min(256, int(args.cpu_seconds / (0.5 / threads))))
            ref.search_many(h, qs[0][:threads], params, 1, threads)  # index build + warm-up
            t0 = time.perf_counter()
            ref.search_many(h, qs[0][:ns], params, 1, threads)
            wall = time.perf_counter() - t0
            cpu = {"value": ns / wall, "unit": "queries/s", "cores": threads, "kind": "reference",
                   "sample": f"{ns} queries of the batch, lir::search throughput mode ({threads} workers x "
                             f"SearchOptions.threads=1)"}
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "unit": "queries/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"failed: {e}"}
    line = {
        "metric": METRIC, "value": value, "unit": "queries/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * total_s / args.steps,
        "p50_ms": float(np.median(step_ms)), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (SplitMix64 generator, SURVEY.md §8d)",
        "config": config_block(cfg, params, args, world),
        "e2e": {"value": e2e_value, "unit": "queries/s", "h2d_bytes_per_step": B * QLEN * DIM * 4,
                "d2h_bytes_per_step": B * (k * 8 + 8)},
        "gpu_launches": launches,
        "roofline": roof,
        "cpu_baseline": cpu,
        "clocks": clk,
    }
    print(json.dumps(line))
    if dist is not None:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="plaid", choices=["plaid", "reference"])
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS))
    ap.add_argument("--score-mode", default="tensor", choices=["exact", "tensor"])
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--graphs", action="store_true", help="host API search replays a captured CUDA graph (e2e)")
    ap.add_argument("--flush", default="write", choices=["write", "write+read"],
                    help="untimed L2 reset between steps")
    ap.add_argument("--lanes", type=int, default=8, help="throughput mode: concurrent searcher lanes")
    ap.add_argument("--batch", type=int, default=0, help="queries per step (default: the config's)")
    ap.add_argument("--shard-mode", default="global-exact", choices=["global-exact", "shard-local"],
                    help="multi-GPU exchange (SURVEY.md §8e): global cuts after stages 2 and 3, or top-k merge only")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    cfg = dict(CONFIGS[args.config])
    if args.batch:
        cfg["batch"] = args.batch
    if args.impl == "reference":
        run_reference(args, cfg)
    elif cfg.get("batch", 1) > 1:
        run_plaid_batch(args, cfg)
    else:
        run_plaid(args, cfg)


if __name__ == "__main__":
    main()
