"""Passage-range sharding across GPUs.

One process per GPU (torch.distributed; NCCL over NVLink/NVSwitch on the
GPU box, gloo for the CPU tests).  Rank r holds the passages
[pid_base_r, pid_base_r + N_r) with a local IVF; the centroids are
replicated, so stage 1 is exact per shard.  Each rank runs the whole
four-stage search on its shard and emits its top-k with GLOBAL passage ids;
the one exchange step is an all-gather of the k (pid, score) pairs plus the
count (one packed row per rank, one collective), followed by the device-side final select (merge_topk, the
(score desc, pid asc) order of pipeline.cpp:139-163) — every rank ends with
the same global top-k.  Messages are k x 8 B per rank, so they are
latency-bound: one all-gather of a packed row, no host sync between
the search and the merge.

Two modes:

* "global-exact" (default): two more all-gathers make every shard apply the
  GLOBAL stage-2 (top-ndocs) and stage-3 (top-stage3_width) cuts
  (plaid_shard_phase{1,2,3}_device): after stage 2 each shard exports its
  local top-ndocs keys (score image, ~global pid), the union holds the global
  top-ndocs, and each shard keeps only its keys at or above the global
  ndocs-th key; the same after stage 3.  The merged top-k then equals
  lir::search over the UNSHARDED index (pipeline.cpp:232-283), and the
  shards' trace counters sum to its StageTrace.  Messages: ndocs x 8 B and
  stage3_width x 8 B per shard (256 KiB + 64 KiB per query at cfg2, 8 GPUs).
* "shard-local": the search runs to completion on every shard and only the
  top-k lists are merged — equal to the reference run on each shard followed
  by the same merge (a shard may admit passages the global stage-2 cut
  drops).
"""
from __future__ import annotations

from typing import Optional

import torch
import torch.distributed as dist


def shard_range(num_passages: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced passage range of `rank` (sizes differ by <= 1)."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError(f"rank {rank} not in [0, {world})")
    base, extra = divmod(int(num_passages), world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


def _all_gather(out: torch.Tensor, inp: torch.Tensor, group) -> None:
    """[world * n] <- every rank's [n]; one call on NCCL, a list on gloo."""
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, inp, group=group)
    else:
        dist.all_gather(list(out.chunk(dist.get_world_size(group))), inp, group=group)


MODES = ("global-exact", "shard-local")


def exchange_strides(params, num_passages: int, disable_filter: bool = False) -> tuple[int, int]:
    """Common row lengths of the two key exchanges: min(ndocs, N) and
    min(stage3_width, N) over the GLOBAL passage count (>= every shard's)."""
    if disable_filter:
        return 0, 0
    n3 = max(-(-int(params.ndocs) // 4), int(params.k))  # pipeline.cpp:227-230
    return min(int(params.ndocs), int(num_passages)), min(n3, int(num_passages))


class ShardedSearcher:
    """Global top-k over passage-sharded searchers.

    `searcher` is this rank's Searcher (over a DeviceIndex made with
    DeviceIndex.from_host_at(shard, pid_base) so it emits global ids).
    `num_passages` is the global passage count (required for global-exact).
    Buffers live on `device`; `stream` is the CUDA stream handle every phase
    and the merge are enqueued on (0 = legacy default stream)."""

    def __init__(self, searcher, k: int, group=None, device: Optional[torch.device] = None,
                 mode: str = "global-exact", num_passages: Optional[int] = None):
        if mode not in MODES:
            raise ValueError(f"mode must be one of {MODES}")
        if mode == "global-exact" and num_passages is None:
            raise ValueError("global-exact mode needs the global passage count")
        self.s = searcher
        self.k = int(k)
        self.group = group
        self.mode = mode
        self.num_passages = num_passages
        self.world = dist.get_world_size(group)
        self.dev = dev = device if device is not None else torch.device("cpu")
        self._x = {}
        z = lambda *shape, dt: torch.zeros(*shape, dtype=dt, device=dev)  # noqa: E731
        # this rank's result row, packed for ONE all-gather per query:
        # [k u32 pids | k f32 scores | u64 count] (plaid_merge_topk_rows_device)
        self.row_words = 2 * self.k + 2
        self.row = z(self.row_words, dt=torch.int32)
        self.g_rows = z(self.world * self.row_words, dt=torch.int32)
        self.pids = self.row[: self.k]
        self.scores = self.row[self.k: 2 * self.k].view(torch.float32)
        self.n = self.row[2 * self.k:].view(torch.int64)
        self.out_pids, self.out_scores = z(self.k, dt=torch.int32), z(self.k, dt=torch.float32)
        self.out_n = z(1, dt=torch.int64)
        self._last_stream, self._last_df = 0, False

    def _xbuf(self, name: str, n: int) -> torch.Tensor:
        t = self._x.get(name)
        if t is None or t.numel() != n:
            t = self._x[name] = torch.zeros(max(n, 1), dtype=torch.int64, device=self.dev)
        return t

    def search(self, q: torch.Tensor, params, stream: int = 0, options=None):
        """q: [rows, dim] float32 on this rank's device.  Returns device views
        (pids, scores, n) of the global top-k (length out_n).  Every phase and
        collective is ordered on `stream` (default: torch's current stream,
        which the NCCL all-gathers use too)."""
        if int(params.k) != self.k:
            raise ValueError(f"params.k {params.k} != {self.k}")
        if self.dev.type == "cuda":
            if not stream:
                stream = torch.cuda.current_stream(self.dev).cuda_stream
            if not stream:
                # the legacy default stream does not order the searcher's own
                # (non-blocking) stream: run the phases and the collectives on
                # one private stream instead
                if getattr(self, "_side", None) is None:
                    self._side = torch.cuda.Stream(self.dev)
                self._side.wait_stream(torch.cuda.current_stream(self.dev))
                with torch.cuda.stream(self._side):
                    out = self.search(q, params, self._side.cuda_stream, options)
                torch.cuda.current_stream(self.dev).wait_stream(self._side)
                return out
        rows, dim = q.shape
        df = bool(options.disable_filter) if options is not None else False
        kw = {"options": options} if options is not None else {}
        self._last_stream, self._last_df = stream, df
        if self.mode == "shard-local":
            self.s.search_device(q.data_ptr(), 1, rows, dim, params, self.pids.data_ptr(), self.scores.data_ptr(),
                                 self.n.data_ptr(), stream=stream, **kw)
        else:
            s2, s3 = exchange_strides(params, self.num_passages, df)
            x2, g2 = self._xbuf("x2", s2), self._xbuf("g2", self.world * s2)
            x3, g3 = self._xbuf("x3", s3), self._xbuf("g3", self.world * s3)
            self.s.shard_phase1(q.data_ptr(), rows, dim, params, x2.data_ptr(), s2, stream=stream, **kw)
            if s2:
                _all_gather(g2[: self.world * s2], x2[:s2], self.group)
            self.s.shard_phase2(g2.data_ptr(), self.world, x3.data_ptr(), s3, stream=stream)
            if s3:
                _all_gather(g3[: self.world * s3], x3[:s3], self.group)
            self.s.shard_phase3(g3.data_ptr(), self.world, self.pids.data_ptr(), self.scores.data_ptr(),
                                self.n.data_ptr(), stream=stream)
        _all_gather(self.g_rows, self.row, self.group)
        self.s.merge_topk_rows_device(self.g_rows.data_ptr(), self.world, self.k, self.out_pids.data_ptr(),
                                      self.out_scores.data_ptr(), self.out_n.data_ptr(), stream=stream)
        return self.out_pids, self.out_scores, self.out_n

    def trace_counters(self) -> dict:
        """StageTrace counters of the last search summed over the shards
        (global-exact: equal to the unsharded reference's).  Host sync.

        The device copy runs on the stream the last search() used (recorded
        there), after a device-wide sync so the counters are final and the
        zero fill of the target is done; with disable_filter the reference
        reports stage1_candidates as stage2_out and stage3_out
        (pipeline.cpp:255-258)."""
        c = torch.zeros(6, dtype=torch.int64, device=self.dev)
        if self.dev.type == "cuda":
            torch.cuda.synchronize(self.dev)
        self.s.trace_counters_device(c.data_ptr(), stream=self._last_stream)
        if self.dev.type == "cuda":
            torch.cuda.synchronize(self.dev)
        dist.all_reduce(c, group=self.group)
        v = c.cpu().tolist()
        if self._last_df:
            v[1] = v[2] = v[0]
        return {"stage1_candidates": v[0], "stage2_out": v[1], "stage3_out": v[2],
                "stage2_rows_gathered": v[4], "stage3_rows_gathered": v[5]}


def search_local_shards(searchers, q, params, num_passages: int, stream: int = 0, options=None):
    """Global-exact search over G shard searchers driven from ONE process (e.g.
    G shards on one GPU for the parity tests): the same three phases as
    ShardedSearcher, with the all-gathers done by device copies.  Returns
    (pids, scores) of the merged global top-k as numpy arrays."""
    import numpy as np

    G = len(searchers)
    dev = q.device
    side = None
    if dev.type == "cuda" and not stream:
        # one stream for every shard (handle 0 would mean "each searcher's
        # own stream"): phase 2 of shard i reads rows other shards exported
        side = torch.cuda.Stream(dev)
        stream = side.cuda_stream
    df = bool(options.disable_filter) if options is not None else False
    kw = {"options": options} if options is not None else {}
    rows, dim = q.shape
    k = int(params.k)
    s2, s3 = exchange_strides(params, num_passages, df)
    z = lambda n, dt=torch.int64: torch.zeros(max(n, 1), dtype=dt, device=dev)  # noqa: E731
    g2, g3 = z(G * s2), z(G * s3)
    pids, scores, ns = z(G * k, torch.int32), z(G * k, torch.float32), z(G)
    op, os_, on = z(k, torch.int32), z(k, torch.float32), z(1)
    if side is not None:
        torch.cuda.synchronize(dev)  # buffers zeroed on the current stream
    for i, s in enumerate(searchers):
        s.shard_phase1(q.data_ptr(), rows, dim, params, g2.data_ptr() + 8 * i * s2, s2, stream=stream, **kw)
    for i, s in enumerate(searchers):
        s.shard_phase2(g2.data_ptr(), G, g3.data_ptr() + 8 * i * s3, s3, stream=stream)
    for i, s in enumerate(searchers):
        s.shard_phase3(g3.data_ptr(), G, pids.data_ptr() + 4 * i * k, scores.data_ptr() + 4 * i * k,
                       ns.data_ptr() + 8 * i, stream=stream)
    searchers[0].merge_topk_device(pids.data_ptr(), scores.data_ptr(), ns.data_ptr(), G, k, k, op.data_ptr(),
                                   os_.data_ptr(), on.data_ptr(), stream=stream)
    if dev.type == "cuda":
        torch.cuda.synchronize(dev)
    m = int(on[0])
    return op[:m].cpu().numpy().view(np.uint32), os_[:m].cpu().numpy()


class BatchShardedSearcher:
    """Global-exact THROUGHPUT mode over passage shards: B queries per call,
    the reference's single-index cuts (pipeline.cpp:260-275) reproduced
    exactly, with the key exchanges batched per wave instead of per query.

    `lanes` are this rank's Searchers over the same shard DeviceIndex (each
    holds one query's state between the phases).  A wave = up to L queries,
    one per lane: phase 1 on every lane, ONE all-gather of the [L][s2] keys,
    a device transpose to per-lane [world][s2] rows, phase 2, ONE all-gather
    of [L][s3], phase 3, ONE all-gather of the packed [L] result rows and a
    per-lane merge.  Three collectives per wave of L queries (ShardedSearcher
    pays three per query).  With CUDA, lane l runs its phases on its own
    stream; the collectives and transposes run on the caller's stream and
    the lanes are fenced to it on both sides of each exchange."""

    def __init__(self, lanes, k: int, num_passages: int, group=None, device: Optional[torch.device] = None):
        if not lanes:
            raise ValueError("need at least one lane searcher")
        self.lanes = list(lanes)
        self.L = len(self.lanes)
        self.k = int(k)
        self.group = group
        self.num_passages = int(num_passages)
        self.world = dist.get_world_size(group)
        self.dev = device if device is not None else torch.device("cpu")
        self.row_words = 2 * self.k + 2
        z = lambda n, dt=torch.int32: torch.zeros(max(n, 1), dtype=dt, device=self.dev)  # noqa: E731
        self.rows = z(self.L * self.row_words)
        self.g_rows = z(self.world * self.L * self.row_words)
        self.t_rows = z(self.L * self.world * self.row_words)
        self._x = {}
        self.launches = 0  # kernels the last search() launched (phases + merges)
        self._streams = None
        if self.dev.type == "cuda":
            self._streams = [torch.cuda.Stream(self.dev) for _ in range(self.L)]

    def _buf(self, name: str, n: int) -> torch.Tensor:
        t = self._x.get(name)
        if t is None or t.numel() < max(n, 1):
            t = self._x[name] = torch.zeros(max(n, 1), dtype=torch.int64, device=self.dev)
        return t

    def _fan_out(self, main):
        if self._streams is not None:
            for s in self._streams:
                s.wait_stream(main)

    def _fan_in(self, main):
        if self._streams is not None:
            for s in self._streams:
                main.wait_stream(s)

    def _lane_stream(self, l: int, main_handle: int) -> int:
        return self._streams[l].cuda_stream if self._streams is not None else main_handle

    def _exchange(self, x: torch.Tensor, g: torch.Tensor, t: torch.Tensor, n: int, stride: int) -> None:
        """x [n][stride] (this rank) -> t [n][world][stride] (every rank's row
        of each lane's query, rank-major as shard_phase{2,3} read it)."""
        w = self.world
        _all_gather(g[: w * self.L * stride], x[: self.L * stride], self.group)
        gv = g[: w * self.L * stride].view(w, self.L, stride)[:, :n]
        t[: n * w * stride].view(n, w, stride).copy_(gv.transpose(0, 1))

    def search(self, qs: torch.Tensor, params, out_pids: torch.Tensor, out_scores: torch.Tensor,
               out_n: torch.Tensor, options=None) -> None:
        """qs: [B, rows, dim] float32 on this rank's device.  Writes the global
        top-k of query b to out_pids[b, :out_n[b]] / out_scores[b, ...]
        ([B, k] int32 / float32, out_n [B] int64), ordered on torch's current
        stream.  Every rank must call with the same B and params."""
        if int(params.k) != self.k:
            raise ValueError(f"params.k {params.k} != {self.k}")
        B, rows, dim = qs.shape
        df = bool(options.disable_filter) if options is not None else False
        kw = {"options": options} if options is not None else {}
        s2, s3 = exchange_strides(params, self.num_passages, df)
        w, L, k, rw = self.world, self.L, self.k, self.row_words
        x2, g2, t2 = self._buf("x2", L * s2), self._buf("g2", w * L * s2), self._buf("t2", L * w * s2)
        x3, g3, t3 = self._buf("x3", L * s3), self._buf("g3", w * L * s3), self._buf("t3", L * w * s3)
        cuda = self.dev.type == "cuda"
        main = torch.cuda.current_stream(self.dev) if cuda else None
        mh = main.cuda_stream if cuda else 0
        qrow = rows * dim * 4
        count = lambda s: int(s.last_launches()) if hasattr(s, "last_launches") else 0  # noqa: E731
        self.launches = 0
        for b0 in range(0, B, L):
            n = min(L, B - b0)
            self._fan_out(main)
            for l in range(n):
                self.lanes[l].shard_phase1(qs.data_ptr() + (b0 + l) * qrow, rows, dim, params,
                                           x2.data_ptr() + 8 * l * s2, s2, stream=self._lane_stream(l, mh), **kw)
            self._fan_in(main)
            if s2:
                self._exchange(x2, g2, t2, n, s2)
            self._fan_out(main)
            for l in range(n):
                self.lanes[l].shard_phase2(t2.data_ptr() + 8 * l * w * s2, w, x3.data_ptr() + 8 * l * s3, s3,
                                           stream=self._lane_stream(l, mh))
            self._fan_in(main)
            if s3:
                self._exchange(x3, g3, t3, n, s3)
            self._fan_out(main)
            base = self.rows.data_ptr()
            for l in range(n):
                r = base + 4 * l * rw
                self.lanes[l].shard_phase3(t3.data_ptr() + 8 * l * w * s3, w, r, r + 4 * k, r + 8 * k,
                                           stream=self._lane_stream(l, mh))
                self.launches += count(self.lanes[l])
            self._fan_in(main)
            _all_gather(self.g_rows[: w * L * rw], self.rows[: L * rw], self.group)
            gv = self.g_rows[: w * L * rw].view(w, L, rw)[:, :n]
            self.t_rows[: n * w * rw].view(n, w, rw).copy_(gv.transpose(0, 1))
            for l in range(n):
                b = b0 + l
                self.lanes[0].merge_topk_rows_device(
                    self.t_rows.data_ptr() + 4 * l * w * rw, w, k, out_pids.data_ptr() + 4 * b * k,
                    out_scores.data_ptr() + 4 * b * k, out_n.data_ptr() + 8 * b, stream=mh)
                self.launches += count(self.lanes[0])
