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
    # N is the WHOLE corpus here: 8 passage-range shards of 17.5M (~1.25B
    # embeddings, ~56 GB each) generated in HBM; rank r holds shard r, so at
    # N < 8 GPUs the line measures the per-GPU load of the 8-GPU deployment
    "cfg5": dict(N=140_000_000, K=1 << 20, nbits=2, mean_len=71, k=1000, shards=8, slice_N=200_000,
                 desc="synthetic MS MARCO v2-scale: 140M passages (~10B embeddings) in 8 passage shards of 17.5M, "
                      "2^20 centroids, nbits=2, k=1000, NCCL top-k merge"),
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


def cpu_model() -> str:
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:  # noqa: BLE001
        pass
    return "unknown"


def cpu_reference_run(h, qs, params, steps, warmup, threads, ref=None):
    """Latency mode: sequential lir::search, threads = all host cores."""
    import oracle

    ref = ref or oracle.timed_reference()[0]
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
    return lat


def cpu_reference_throughput(h, qs, params, threads, ref):
    """Throughput mode (SURVEY.md §8d ii): `threads` concurrent lir::search
    calls with SearchOptions.threads = 1 over the shared immutable index."""
    n = min(len(qs), 2 * threads)
    ref.search_many(h, qs[:threads], params, 1, threads)  # warm-up
    t0 = time.perf_counter()
    ref.search_many(h, qs[:n], params, 1, threads)
    return n / (time.perf_counter() - t0), n


class RefParams:
    """lir::SearchParams (types.hpp:79-84) from the reference's own
    default_params_for_k (types.cpp:74-86)."""

    def __init__(self, ref, k: int, ndocs=None):
        self.k, self.nprobe, self.t_cs, self.ndocs = ref.default_params_for_k(k)
        if ndocs is not None:
            self.ndocs = ndocs


def run_reference(args, cfg):
    """The reference's own CPU searcher on this host: the unmodified
    /root/reference sources (oracle/_ref), inputs from the checker-side
    generator (oracle/synth.py) and IVF from the reference's
    build_inverted_list — no library of this package is loaded."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle

    if not oracle.available("ref"):
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/liblir_ref.so not built"}))
        return
    from oracle import synth

    ref, flags = oracle.timed_reference()
    n_ref, note = cfg["N"], ""
    if cfg.get("shards"):
        # the whole corpus (~390 GB) does not fit host memory: the reference
        # searches shard 0 of 8 (what one GPU holds), when that fits
        n_ref = cfg["N"] // int(cfg["shards"])
        need = 2.5 * n_ref * cfg["mean_len"] * (4 + 16 * cfg["nbits"] + 4)
        avail = host_mem_available()
        if avail < need:
            print(json.dumps({"impl": "reference", "unavailable": f"{args.config} shard needs ~{need / 1e9:.0f} GB of "
                                                                  f"host memory, {avail / 1e9:.0f} GB available"}))
            return
        note = f" (shard 0 of {cfg['shards']}: {n_ref} passages)"
    t = time.time()
    h = synth.generate_index(n_ref, cfg["K"], dim=DIM, nbits=cfg["nbits"], mean_len=cfg["mean_len"],
                             spread=16, seed=0, ivf=ref.build_inverted_list)
    log(f"[reference] generated index: N={h.num_passages} T={h.num_embeddings} ({h.nbytes() / 1e9:.1f} GB) "
        f"in {time.time() - t:.1f}s")
    qs = synth.generate_queries(h, max(args.steps + args.warmup, 1), qlen=QLEN, seed=1234)
    params = RefParams(ref, cfg["k"], cfg.get("ndocs"))
    threads = os.cpu_count() or 1
    B = int(cfg.get("batch", 1))
    if B > 1:
        # throughput mode: `threads` workers x SearchOptions.threads=1;
        # each step is a bounded sample of the batch (~1 s of CPU work)
        qb = synth.generate_queries(h, threads * 4, qlen=QLEN, seed=1234)
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
        lat = cpu_reference_run(h, qs, params, args.steps, args.warmup, threads, ref)
        total = sum(lat)
        qps = args.steps / total
        sample = f"{args.steps} sequential queries, lir::search latency mode, SearchOptions.threads={threads}"
    sample += note
    line = {
        "impl": "reference", "metric": METRIC, "value": qps, "unit": "queries/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "p50_ms": 1e3 * statistics.median(lat), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (SplitMix64 generator, SURVEY.md §8d)",
        "config": config_block(cfg, params, args, 1),
        "cpu_baseline": {"value": qps, "unit": "queries/s", "cores": threads, "kind": "reference",
                         "sample": sample, "cpu_model": cpu_model(), "build": flags},
        "e2e": {"value": qps, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "repo_libs_mapped": repo_libs_mapped(),
    }
    print(json.dumps(line))


def host_mem_available() -> float:
    try:
        for line in Path("/proc/meminfo").read_text().splitlines():
            if line.startswith("MemAvailable:"):
                return float(line.split()[1]) * 1024
    except OSError:
        pass
    return 0.0


def repo_libs_mapped() -> list:
    """In-tree shared objects this process has mapped (the reference arm must
    show only oracle/ libraries: the reference and the checker-side generator)."""
    libs = set()
    try:
        for line in Path("/proc/self/maps").read_text().splitlines():
            f = line.split()
            if len(f) >= 6 and f[-1].endswith(".so") and f[-1].startswith(str(ROOT)):
                libs.add(str(Path(f[-1]).relative_to(ROOT)))
    except OSError:
        pass
    return sorted(libs)


def config_block(cfg, params, args, world):
    shards = int(cfg.get("shards", 0))
    per_gpu = cfg["N"] // shards if shards else cfg["N"]
    extra = {}
    if shards:
        extra = {"corpus_passages": cfg["N"], "corpus_shards": shards,
                 "scaling_note": (f"rank r holds shard r of {shards} (generated in HBM); with {world} GPU(s) the "
                                  f"line covers {world}/{shards} of the corpus at the per-GPU load of the "
                                  f"{shards}-GPU deployment" if world < shards else "the whole corpus")}
    return {"workload": f"{args.config}: {cfg['desc']}", "passages_per_gpu": per_gpu,
            "passages_total": per_gpu * world, **extra, "centroids": cfg["K"], "nbits": cfg["nbits"], "dim": DIM,
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

    params = params_for(cfg)
    nq = max(args.steps + args.warmup, 8)
    shards = int(cfg.get("shards", 0))
    t = time.time()
    if shards:
        # a shard of a corpus too large for host memory: generated in HBM
        if world > shards:
            raise SystemExit(f"{args.config} has {shards} shards; run it on at most {shards} GPUs")
        n_shard = cfg["N"] // shards
        h = None
        idx = P.DeviceIndex.synth(n_shard, cfg["K"], dim=DIM, nbits=cfg["nbits"], mean_len=cfg["mean_len"],
                                  spread=16, seed=0, pid_base=rank * n_shard, device=local)
        num_passages = world * n_shard
    else:
        h = make_index(cfg, rank)
        idx = P.DeviceIndex.from_host_at(h, pid_base=rank * cfg["N"], device=local)
        num_passages = cfg["N"] * world
    log(f"[rank {rank}] index resident on cuda:{local}: {idx.device_bytes / 1e9:.1f} GB in {time.time() - t:.1f}s")
    # queries: generated from shard 0's passages, identical on every rank
    if rank == 0:
        qs = (idx.synth_queries(nq, qlen=QLEN, seed=1234) if h is None
              else P.generate_queries(h, nq, qlen=QLEN, seed=1234))
    else:
        qs = np.zeros((nq, QLEN, DIM), dtype=np.float32)
    dq = torch.from_numpy(qs).cuda()
    if dist is not None:
        dist.broadcast(dq, 0)
        qs = dq.cpu().numpy()
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
                             num_passages=num_passages)
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

    # ---- workload calibration and parity on the measured
    # queries: the reference's stages (oracle, the checker) on query 0 give the
    # integer counts B_alg is made of; --check N classifies N timed queries'
    # TENSOR results against lir::search with the north_star comparator
    hbm_peak, tf_peak, peak_kind = measured_peaks()
    tf_sust = measured_tensor_sustained()
    mean_ph = {n: float(np.mean(v)) for n, v in phases.items()}
    K = cfg["K"]
    tr = trace.counters() if trace is not None else {}
    t4 = trace.decompressed_tokens if trace is not None else 0
    step_mean_ms = 1e3 * total_s / args.steps
    calib, parity = None, None
    h_chk, qs_chk, s_chk, first_chk = h, qs, s, args.warmup
    if world == 1 and not args.no_cpu and h is None:
        # the shard has no host copy: check and baseline on a slice of the
        # same corpus (same K, generator and queries recipe), state it
        ns = int(cfg["slice_N"])
        ix_slice = P.DeviceIndex.synth(ns, cfg["K"], dim=DIM, nbits=cfg["nbits"], mean_len=cfg["mean_len"],
                                       spread=16, seed=0, pid_base=0, device=local)
        h_chk = ix_slice.to_host()
        qs_chk = ix_slice.synth_queries(max(args.check, 1) + 3, qlen=QLEN, seed=1234)
        s_chk = P.Searcher(ix_slice, device=local, score_mode=mode)
        first_chk = 0
    if world == 1 and not args.no_cpu:
        try:
            calib, parity = check_and_calibrate(args, h_chk, qs_chk, params, s_chk, first_chk)
            if h is None:
                calib["scope"] = parity["scope"] = (f"slice: passages [0, {len(h_chk.doclens)}) of the same corpus, "
                                                    f"K = {cfg['K']} (the measured shard has no host copy)")
        except Exception as e:  # noqa: BLE001
            parity = {"error": repr(e)}

    # ---- rooflines of the two largest kernels (ncu launch list: S_cq and the
    # stage-4 kernel; every other launch is < 1/3 of either).  Algorithmic
    # bytes per launch follow SURVEY.md §8(d); the phase events bracket each
    # kernel on the launching stream.
    roofs = {}
    ab_scq = 512 * K + QLEN * DIM * 4  # C read once + Q (no S writes: not in B_alg)
    roofs["scores"] = roof_line("scores_tf32_kernel" if args.score_mode == "tensor" else "scores_exact_kernel",
                                ab_scq, mean_ph["scores"], hbm_peak, peak_kind, step_mean_ms, args.config,
                                "512 B x K centroid rows + 16 KiB Q (SURVEY.md §8d)")
    if calib and h is not None:
        n3 = calib["n3"]
        ab4 = (4 + 16 * cfg["nbits"]) * calib["T4"] + 12 * n3 + 512 * calib["U4"]
        k4 = "stage4_warp_kernel" if args.score_mode == "tensor" else "stream_fused_kernel"
        roofs["stage4"] = roof_line(k4, ab4, mean_ph["stage4_rank"], hbm_peak, peak_kind, step_mean_ms,
                                    args.config, "(4 + 16 b) B x T4 codes+residuals + 12 B x n3 + 512 B x U4 "
                                                 "distinct centroid rows (SURVEY.md §8d); phase = the stage-4 "
                                                 "kernel (TENSOR: the finalist scan rides in the stage-3 select, "
                                                 "no finalize)")
    dom = max(roofs, key=lambda n: roofs[n]["mean_ms"])
    roof = dict(roofs[dom])
    roof["dominant_of"] = {n: r["mean_ms"] for n, r in roofs.items()}
    others = {n: r for n, r in roofs.items() if n != dom}

    # ---- whole-query roofline: t_roof = FLOPs_Scq / P_tc + B_alg / BW
    rq = None
    if calib and h is not None:
        # 3xTF32 = three tf32 MMA passes; tf32 dense rate = half the measured bf16 rate
        p_tc = (tf_sust if tf_sust else tf_peak) / 2 * 1e12
        flops = 3 * 2.0 * K * DIM * QLEN
        t_roof = flops / p_tc + calib["B_alg"] / (hbm_peak * 1e9)
        rq = {"t_roof_us": 1e6 * t_roof, "t_measured_us": 1e3 * step_mean_ms,
              "frac": t_roof / (step_mean_ms * 1e-3), "B_alg_bytes": calib["B_alg"],
              "scq_flops": flops, "p_tc_tflops": p_tc / 1e12,
              "note": "t_roof = 3xTF32 S_cq FLOPs / (measured bf16 sustained / 2) + B_alg / measured HBM copy "
                      "bandwidth; B_alg per SURVEY.md §8d from the reference's integer sets on query 0"}

    # ---- CPU baseline: the reference's own searcher on this host, bounded sample
    cpu = None
    if world == 1 and not args.no_cpu:
        try:
            import oracle

            ref, flags = oracle.timed_reference()
            threads = os.cpu_count() or 1
            per_q = 0.5 if cfg["N"] > 1_000_000 else 0.02
            nsample = max(3, min(64, int(args.cpu_seconds / per_q)))
            lat = cpu_reference_run(h_chk, qs_chk, params, nsample, 1, threads, ref)
            tput, ntp = cpu_reference_throughput(h_chk, qs_chk, params, threads, ref)
            ref.release(h_chk)
            cpu = {"value": nsample / sum(lat), "unit": "queries/s", "cores": threads, "kind": "reference",
                   "sample": f"{nsample} sequential queries of the same workload, lir::search latency mode, "
                             f"SearchOptions.threads={threads}", "p50_ms": 1e3 * statistics.median(lat),
                   "throughput_mode": {"value": tput, "unit": "queries/s", "queries": ntp,
                                       "how": f"{threads} concurrent lir::search calls, SearchOptions.threads=1"},
                   "cpu_model": cpu_model(), "build": flags}
            if h is None:
                cpu["sample"] += f" ({calib['scope'] if calib else 'slice of the corpus'})"
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "unit": "queries/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"failed: {e}"}

    line = {
        "metric": METRIC, "value": value, "unit": "queries/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_mean_ms,
        "p50_ms": float(np.median(step_ms)), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (SplitMix64 generator, SURVEY.md §8d)",
        "config": config_block(cfg, params, args, world),
        "e2e": {"value": e2e_value, "unit": "queries/s", "h2d_bytes_per_step": QLEN * DIM * 4,
                "d2h_bytes_per_step": k * 8 + 128, "p50_ms": 1e3 * statistics.median(e2e_lat),
                "path": "Python Searcher.search -> plaid_search (C ABI), host buffers"},
        "gpu_launches": launches,
        "roofline": roof,
        "roofline_other": others,
        "roofline_query": rq,
        "phases_ms": mean_ph,
        "trace": tr,
        "calibration": calib,
        "parity": parity,
        "cpu_baseline": cpu,
        "clocks": clk,
    }
    if args.cpp_e2e:
        # the headline e2e goes through the reference-facing drop-in (C++
        # plaid_lir::Engine over the C ABI); the Python-API number stays beside it
        ec = cpp_e2e(args, cfg)
        if ec and "value" in ec:
            line["e2e_python"] = line["e2e"]
            line["e2e"] = ec
        else:
            line["e2e_cpp"] = ec
    print(json.dumps(line))
    if dist is not None:
        dist.destroy_process_group()


def cpp_e2e(args, cfg):
    """e2e through the C++ drop-in (include/plaid_lir.hpp, tools/e2e_cpp.cpp):
    a C++ program on lir types builds the same corpus and times
    plaid_lir::Engine::search per query with host buffers (subprocess; the GPU
    index of this process stays resident)."""
    exe = ROOT / "oracle" / "_ref" / "e2e_cpp"
    if not exe.exists() or cfg.get("shards") or cfg.get("batch", 1) > 1:
        return None
    cmd = [str(exe), str(cfg["N"]), str(cfg["K"]), str(cfg["nbits"]), str(cfg["mean_len"]), str(cfg["k"]),
           str(args.steps), str(max(args.warmup, 3)), "1" if args.score_mode == "tensor" else "0"]
    try:
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
        out = json.loads(r.stdout.strip().splitlines()[-1])
        out["h2d_bytes_per_step"] = QLEN * DIM * 4
        out["d2h_bytes_per_step"] = int(cfg["k"]) * 8 + 128
        return out
    except Exception as e:  # noqa: BLE001
        return {"error": repr(e)[:200]}


def measured_tensor_sustained():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return float(json.loads(p.read_text()).get("bf16_tflops_sustained") or 0) or None
    return None


def roof_line(kname, ab, mean_ms, hbm_peak, peak_kind, step_ms, config, bytes_note):
    ach = ab / (mean_ms * 1e-3) / 1e9
    traffic = None
    tf = ROOT / "profiles" / "traffic.json"
    if tf.exists():
        t = json.loads(tf.read_text()).get(f"{config}/{kname}")
        traffic = t.get("dram_bytes_per_launch") if t else None
    return {"bound": "hbm", "kernel": kname, "achieved": ach, "peak": hbm_peak, "unit": "GB/s",
            "frac": ach / hbm_peak, "traffic": traffic, "peak_kind": f"{peak_kind} (copy bandwidth, burst)",
            "algorithmic_bytes_per_launch": ab, "bytes": bytes_note, "mean_ms": mean_ms,
            "share_of_step": mean_ms / step_ms}


def check_and_calibrate(args, h, qs, params, searcher, first):
    """Checker leg (oracle = the compiled reference, lir itself): SURVEY.md
    §8d's calibration counts of query `first` and the north_star comparison of
    --check queries' TENSOR results with lir::search on the same inputs."""
    import oracle
    from oracle.compare import check_tensor_search, compose

    ref = oracle.get("ref") if oracle.available("ref") else oracle.get("port")
    q = qs[first]
    S0, mx0 = ref.compute_centroid_scores(h, q)
    c = compose(ref, h, q, S0, mx0, params)
    dl = h.doclens.astype(np.int64)
    kept = int((mx0 >= np.float32(params.t_cs)).sum())
    from oracle.compare import topn_sets

    sets, _ = topn_sets(S0, int(params.nprobe))
    probed = sorted(set().union(*sets))
    ivo = h.ivf_offsets.astype(np.int64)
    P1 = int(sum(ivo[x + 1] - ivo[x] for x in probed))
    C1, T1 = len(c["c1"]), int(dl[c["c1"]].sum())
    T3 = int(dl[c["k2"]].sum())
    n3 = len(c["k3"])
    T4 = int(dl[c["k3"]].sum())
    off = h.passage_offsets.astype(np.int64)
    U4 = int(np.unique(np.concatenate([h.codes[off[x]:off[x + 1]] for x in c["k3"]])).size) if n3 else 0
    zero = float((c["s2"] == 0).mean()) if c["s2"] is not None and len(c["s2"]) else None
    K, b = h.num_centroids, h.nbits
    B_alg = (512 * K + 4 * P1 + (4 * T1 + 12 * C1) + (4 * T3 + 12 * int(params.ndocs))
             + ((4 + 16 * b) * T4 + 12 * n3 + 512 * U4) + QLEN * DIM * 4 + 8 * int(params.k))
    calib = {"query": int(first), "C1": C1, "T1": T1, "P1_distinct_probed_postings": P1,
             "probed_centroids": len(probed), "kept_centroids": kept, "stage2_zero_score_fraction": zero,
             "T3": T3, "n3": n3, "T4": T4, "U4": U4, "B_alg": B_alg}
    parity = None
    if args.check:
        reps = []
        for i in range(args.check):
            qi = qs[first + i]
            r = searcher.search(qi, params)
            S_t, _ = searcher.compute_centroid_scores(qi)
            rep = check_tensor_search(ref, h, qi, params, r.topk.passage_ids, r.topk.scores, S_t,
                                      got_counters=r.trace.counters())
            reps.append(rep)
        parity = {"queries": len(reps), "checker": "oracle/_ref (lir::search, unmodified reference)"
                  if ref.kind == "ref" else "oracle port", "mode": args.score_mode,
                  "ok": all(r.ok for r in reps),
                  "ids_equal_reference": sum(r.ids_equal_reference for r in reps),
                  "max_rel_score_err": max(r.max_rel_score_err for r in reps),
                  "s_max_abs_err": max(r.s_max_abs_err for r in reps),
                  "near_boundary_diffs": {k: sum(getattr(r, k) for r in reps)
                                          for k in ("stage1_diff", "keep_diff", "stage2_diff", "stage3_diff",
                                                    "final_diff")},
                  "problems": [p for r in reps for p in r.problems][:5],
                  "comparator": "oracle/compare.py (north_star: integer sets exact except near t_cs / nprobe / "
                                "ndocs / top-k boundaries; MaxSim within 1e-4 relative)"}
    return calib, parity


def run_plaid_batch(args, cfg):
    """Throughput mode (BASELINE configs[2]): one step = one batch of B queries
    through BatchSearcher (L concurrent lanes); value = queries / job time.
    Multi-GPU: every rank searches its passage shard.  shard-local: the [B][k]
    results are all-gathered once per batch and merged per query (one kernel).
    global-exact (default): BatchShardedSearcher reproduces the single-index
    cuts (pipeline.cpp:260-275) with three all-gathers per wave of lanes."""
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
    gx = None
    if dist is not None and args.shard_mode == "global-exact":
        # global-exact throughput mode: lane Searchers run the three shard
        # phases, three batched all-gathers per wave of lanes (sharded.py)
        from paper_2205_09707_b200.sharded import BatchShardedSearcher

        gx_lanes = [P.Searcher(idx, device=local, score_mode=mode, record_times=False) for _ in range(args.lanes)]
        gx = BatchShardedSearcher(gx_lanes, k=k, num_passages=world * cfg["N"], device=torch.device("cuda", local))
        bs = None
    else:
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
        if gx is not None:
            gx.search(q, params, m_pids.view(B, k), m_scores.view(B, k), m_n)
            return
        bs.search_device(q.data_ptr(), B, QLEN, DIM, params, d_pids.data_ptr(), d_scores.data_ptr(),
                         d_n.data_ptr(), stream=sh)
        if dist is not None:
            from paper_2205_09707_b200.sharded import _all_gather

            _all_gather(g_pids, d_pids, None)
            _all_gather(g_scores, d_scores, None)
            _all_gather(g_n, d_n, None)
            # [world][B][k] lists + [world][B] counts -> [B][k]: one kernel
            merger.merge_topk_batch_device(g_pids.data_ptr(), g_scores.data_ptr(), g_n.data_ptr(), world, B, k,
                                           m_pids.data_ptr(), m_scores.data_ptr(), m_n.data_ptr(), stream=sh)

    for i in range(args.warmup):
        flush()
        step(i)
    torch.cuda.synchronize()
    if bs is not None:
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
        launches += gx.launches if gx is not None else bs.last_launches()
    torch.cuda.synchronize()
    clk = clocks.stop()
    if bs is not None:
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

    hbm_peak, _, peak_kind = measured_peaks()
    K = cfg["K"]
    wave = bs.last_was_wave() if bs is not None else False
    if wave and args.score_mode == "tensor":
        # the wave engine: time the first wave's S_cq launch alone and with its
        # worker (launch cap: a batch stops after its first n kernels), events
        # on the launching stream, L2 flushed before each
        import ctypes as C

        from paper_2205_09707_b200 import _native as Nv

        lib = Nv.load()
        slots = min(B, bs.wave_slots())

        def capped(n):
            old = lib.plaid_debug_set_launch_cap(n)
            ts = []
            for _ in range(3):
                flush()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                bs.search_device(dq[0].data_ptr(), slots, QLEN, DIM, params, d_pids.data_ptr(),
                                 d_scores.data_ptr(), d_n.data_ptr(), stream=sh)
                e1.record(stream)
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            lib.plaid_debug_set_launch_cap(old)
            return float(np.median(ts))

        t_sc = capped(1)
        t_wave = capped(2)
        flops = 3 * 2 * K * DIM * QLEN * slots  # 3xTF32: three tf32 products per dot
        tf32_peak = measured_peaks()[1] / 2.0
        ab = 512 * K * ((slots + 3) // 4) + 128 * K * slots + slots * K // 8  # C per 4-query pass + S rows + keep bits
        roof = {"bound": "tensor", "kernel": "wave_scores_kernel", "achieved": flops / (t_sc * 1e-3) / 1e12,
                "peak": tf32_peak, "unit": "TFLOP/s", "frac": flops / (t_sc * 1e-3) / 1e12 / tf32_peak,
                "traffic": None, "peak_kind": f"{peak_kind} dense bf16 (burst) / 2 = tf32 rate",
                "algorithmic_flops_per_launch": flops, "queries_per_launch": slots, "mean_ms": t_sc,
                "hbm": {"algorithmic_bytes_per_launch": ab, "achieved_gbs": ab / (t_sc * 1e-3) / 1e9,
                        "frac": ab / (t_sc * 1e-3) / 1e9 / hbm_peak},
                "share_of_step": t_sc * (B / slots) / (1e3 * total_s / args.steps),
                "worker_ms_per_wave": t_wave - t_sc,
                "note": "one wave = one S_cq launch (4 queries per pass over C) + one worker launch (a CTA per "
                        "query, stages 1b-4); tensor-pipe activity from ncu in profiles/"}
    else:
        # S_cq kernel alone (one single-query search with phase events) for the roofline
        s1 = P.Searcher(idx, device=local, score_mode=mode, record_times=True)
        sc_ms = []
        for i in range(5):
            flush()
            torch.cuda.synchronize()
            s1.search(qs[0][i], params)
            sc_ms.append(s1.phase_ms()["scores"])
        sc = float(np.median(sc_ms[1:]))
        ab = 512 * K + 128 * K + K // 8 + QLEN * DIM * 4
        kname = "scores_tf32_kernel" if args.score_mode == "tensor" else "scores_exact_kernel"
        roof = {"bound": "hbm", "kernel": kname, "achieved": ab / (sc * 1e-3) / 1e9, "peak": hbm_peak,
                "unit": "GB/s", "frac": ab / (sc * 1e-3) / 1e9 / hbm_peak, "traffic": None,
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
    if gx is not None:
        line["config"]["batch_engine"] = (f"global-exact: {args.lanes} lane Searchers, shard phases 1-3 per wave of "
                                          f"{args.lanes} queries, 3 all-gathers per wave")
    else:
        line["config"]["batch_engine"] = (f"waves of {bs.wave_slots()} queries (one S_cq pass + one worker launch "
                                          f"each)" if wave else f"{args.lanes} lanes")
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
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU reference baseline and the parity check")
    ap.add_argument("--check", type=int, default=2,
                    help="classify this many timed queries' results against lir::search (oracle/_ref) with the "
                         "north_star comparator; reported as the line's `parity` block")
    ap.add_argument("--cpp-e2e", type=int, default=1,
                    help="also time e2e through the C++ drop-in (plaid_lir::Engine, tools/e2e_cpp)")
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
