"""Passage-range sharding across GPUs.

One process per GPU (torch.distributed; NCCL over NVLink/NVSwitch on the
GPU box, gloo for the CPU tests).  Rank r holds the passages
[pid_base_r, pid_base_r + N_r) with a local IVF; the centroids are
replicated, so stage 1 is exact per shard.  Each rank runs the whole
four-stage search on its shard and emits its top-k with GLOBAL passage ids;
the one exchange step is an all-gather of the k (pid, score) pairs plus the
count, followed by the device-side final select (merge_topk, the
(score desc, pid asc) order of pipeline.cpp:139-163) — every rank ends with
the same global top-k.  Messages are k x 8 B per rank, so they are
latency-bound: three small all-gathers of fixed size, no host sync between
the search and the merge.

This is the "shard-local" mode of SURVEY.md §8e: its result equals the
reference run on each shard followed by the same merge.
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


class ShardedSearcher:
    """Global top-k over passage-sharded searchers.

    `searcher` is this rank's Searcher (over a DeviceIndex made with
    DeviceIndex.from_host_at(shard, pid_base) so it emits global ids).
    Buffers live on `device`; `stream` is the CUDA stream handle both the
    search and the merge are enqueued on (0 = legacy default stream)."""

    def __init__(self, searcher, k: int, group=None, device: Optional[torch.device] = None):
        self.s = searcher
        self.k = int(k)
        self.group = group
        self.world = dist.get_world_size(group)
        dev = device if device is not None else torch.device("cpu")
        z = lambda *shape, dt: torch.zeros(*shape, dtype=dt, device=dev)  # noqa: E731
        self.pids, self.scores, self.n = z(self.k, dt=torch.int32), z(self.k, dt=torch.float32), z(1, dt=torch.int64)
        self.g_pids = z(self.world * self.k, dt=torch.int32)
        self.g_scores = z(self.world * self.k, dt=torch.float32)
        self.g_n = z(self.world, dt=torch.int64)
        self.out_pids, self.out_scores = z(self.k, dt=torch.int32), z(self.k, dt=torch.float32)
        self.out_n = z(1, dt=torch.int64)

    def search(self, q: torch.Tensor, params, stream: int = 0):
        """q: [rows, dim] float32 on this rank's device.  Returns device views
        (pids, scores) of the global top-k (length out_n)."""
        if int(params.k) != self.k:
            raise ValueError(f"params.k {params.k} != {self.k}")
        rows, dim = q.shape
        self.s.search_device(q.data_ptr(), 1, rows, dim, params, self.pids.data_ptr(), self.scores.data_ptr(),
                             self.n.data_ptr(), stream=stream)
        _all_gather(self.g_pids, self.pids, self.group)
        _all_gather(self.g_scores, self.scores, self.group)
        _all_gather(self.g_n, self.n, self.group)
        self.s.merge_topk_device(self.g_pids.data_ptr(), self.g_scores.data_ptr(), self.g_n.data_ptr(), self.world,
                                 self.k, self.k, self.out_pids.data_ptr(), self.out_scores.data_ptr(),
                                 self.out_n.data_ptr(), stream=stream)
        return self.out_pids, self.out_scores, self.out_n
