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
