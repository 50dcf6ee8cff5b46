"""Multi-GPU path on CPU: world_size 2 over gloo.  Each rank searches its
passage shard (a test double backed by the CPU oracle stands in for the CUDA
searcher, through the same search_device / merge_topk_device surface) and
ShardedSearcher does the product's exchange: all-gather of the k (pid,
score) pairs + counts, then the final select.  Every rank must end with the
same global top-k, equal to "reference per shard + merge"."""
import ctypes as C
import os
import pickle
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import paper_2205_09707_b200 as P
from paper_2205_09707_b200.sharded import ShardedSearcher, shard_range

N, K, DIM, SEED = 400, 32, 64, 6


def view(ptr, n, ctype, dtype):
    return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(ctype)), shape=(n,)).view(dtype)


def merge(pids, scores, k):
    order = sorted(range(len(pids)), key=lambda i: (-float(scores[i]), int(pids[i])))[:k]
    return np.array([pids[i] for i in order], np.uint32), np.array([scores[i] for i in order], np.float32)


class OracleShard:
    """Test double of Searcher: oracle search on the local shard, global ids."""

    def __init__(self, h, pid_base):
        self.h, self.base, self.port = h, pid_base, oracle.get("port")

    def search_device(self, q, nq, rows, dim, params, d_pids, d_scores, d_n, stream=0):
        qa = view(q, rows * dim, C.c_float, np.float32).reshape(rows, dim)
        ids, sc, _ = self.port.search(self.h, qa, params)
        n = len(ids)
        view(d_pids, params.k, C.c_int32, np.uint32)[:n] = ids + self.base
        view(d_scores, params.k, C.c_float, np.float32)[:n] = sc
        view(d_n, 1, C.c_int64, np.int64)[0] = n

    def merge_topk_device(self, g_pids, g_scores, g_n, shards, stride, k, o_pids, o_scores, o_n, stream=0):
        pids = view(g_pids, shards * stride, C.c_int32, np.uint32).reshape(shards, stride)
        sc = view(g_scores, shards * stride, C.c_float, np.float32).reshape(shards, stride)
        cnt = view(g_n, shards, C.c_int64, np.int64)
        allp = np.concatenate([pids[g, : cnt[g]] for g in range(shards)])
        alls = np.concatenate([sc[g, : cnt[g]] for g in range(shards)])
        mp_, ms = merge(allp, alls, k)
        view(o_pids, k, C.c_int32, np.uint32)[: len(mp_)] = mp_
        view(o_scores, k, C.c_float, np.float32)[: len(ms)] = ms
        view(o_n, 1, C.c_int64, np.int64)[0] = len(mp_)


def worker(rank, world, port_no, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    a, b = shard_range(N, world, rank)
    h = P.generate_index(b - a, K, dim=DIM, nbits=2, mean_len=16, spread=4, seed=SEED, pid_base=a)
    whole = P.generate_index(N, K, dim=DIM, nbits=2, mean_len=16, spread=4, seed=SEED)
    qs = P.generate_queries(whole, 3, seed=77)
    ss = ShardedSearcher(OracleShard(h, a), k=20)
    res = []
    for q in qs:
        for p in (P.SearchParams(20, 2, 0.4, 64), P.SearchParams(20, 8, -1.0, 400)):
            pids, scores, n = ss.search(torch.from_numpy(q.copy()), p)
            m = int(n[0])
            res.append((pids[:m].numpy().astype(np.uint32), scores[:m].numpy().copy()))
    with open(os.path.join(out_dir, f"rank{rank}.pkl"), "wb") as f:
        pickle.dump(res, f)
    dist.barrier()
    dist.destroy_process_group()


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shard_range():
    for n, w in ((10, 3), (7, 8), (1000, 8), (5, 1)):
        rs = [shard_range(n, w, r) for r in range(w)]
        assert rs[0][0] == 0 and rs[-1][1] == n
        assert all(x[1] == y[0] for x, y in zip(rs, rs[1:]))
        assert max(b - a for a, b in rs) - min(b - a for a, b in rs) <= 1
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def test_two_rank_gloo(tmp_path):
    world = 2
    mp.spawn(worker, args=(world, free_port(), str(tmp_path)), nprocs=world, join=True)
    r0, r1 = (pickle.loads((tmp_path / f"rank{r}.pkl").read_bytes()) for r in range(world))
    # expected: the oracle per shard, then the (score desc, pid asc) merge
    port = oracle.get("port")
    whole = P.generate_index(N, K, dim=DIM, nbits=2, mean_len=16, spread=4, seed=SEED)
    qs = P.generate_queries(whole, 3, seed=77)
    shards = [(shard_range(N, world, r)[0],
               P.generate_index(shard_range(N, world, r)[1] - shard_range(N, world, r)[0], K, dim=DIM, nbits=2,
                                mean_len=16, spread=4, seed=SEED, pid_base=shard_range(N, world, r)[0]))
              for r in range(world)]
    i = 0
    for q in qs:
        for p in (P.SearchParams(20, 2, 0.4, 64), P.SearchParams(20, 8, -1.0, 400)):
            allp, alls = [], []
            for base, h in shards:
                ids, sc, _ = port.search(h, q, p)
                allp += list(ids + base)
                alls += list(sc)
            ep, es = merge(allp, alls, 20)
            for r in (r0, r1):
                assert np.array_equal(r[i][0], ep) and np.array_equal(r[i][1].view(np.uint32), es.view(np.uint32))
            i += 1
    # at nprobe=K, t_cs=-1 and ndocs >= N every shard's top-k is exact, so the
    # merge equals the unsharded reference search
    p = P.SearchParams(20, K, -1.0, 4 * N)
    ids, sc, _ = port.search(whole, qs[0], p)
    allp, alls = [], []
    for base, h in shards:
        a_, b_, _ = port.search(h, qs[0], p)
        allp += list(a_ + base)
        alls += list(b_)
    ep, es = merge(allp, alls, 20)
    assert np.array_equal(ep, ids) and np.array_equal(es.view(np.uint32), sc.view(np.uint32))
