"""Multi-GPU path on CPU: world_size 2 (and 3) over gloo.  Each rank searches
its passage shard (a test double backed by the CPU oracle stands in for the
CUDA searcher, through the same search_device / shard_phase{1,2,3} /
merge_topk_device surface) and ShardedSearcher does the product's exchanges.

* shard-local: all-gather of the k (pid, score) pairs + counts, then the final
  select; every rank ends with "reference per shard + merge".
* global-exact (default): two more all-gathers of stage-2 / stage-3 keys and
  threshold filters; every rank ends with the UNSHARDED reference search,
  bit for bit, and the summed trace counters equal its StageTrace
  (SURVEY.md §8e)."""
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
from paper_2205_09707_b200.sharded import ShardedSearcher, exchange_strides, shard_range

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

    def merge_topk_rows_device(self, g_rows, shards, k, o_pids, o_scores, o_n, stream=0):
        row = 2 * k + 2
        r = view(g_rows, shards * row, C.c_int32, np.uint32).reshape(shards, row)
        allp = np.concatenate([r[g, :k][: int(r[g, 2 * k:].view(np.uint64)[0])] for g in range(shards)])
        alls = np.concatenate([r[g, k:2 * k].view(np.float32)[: int(r[g, 2 * k:].view(np.uint64)[0])]
                               for g in range(shards)])
        mp_, ms = merge(allp, alls, k)
        view(o_pids, k, C.c_int32, np.uint32)[: len(mp_)] = mp_
        view(o_scores, k, C.c_float, np.float32)[: len(ms)] = ms
        view(o_n, 1, C.c_int64, np.int64)[0] = len(mp_)

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


def ord_key(scores, gids):
    u = np.asarray(scores, np.float32).view(np.uint32).astype(np.uint64)
    u = np.where(u == 0x80000000, 0, u)
    o = np.where(u & 0x80000000, ~u & 0xFFFFFFFF, u | 0x80000000).astype(np.uint64)
    return (o << np.uint64(32)) | (~np.asarray(gids, np.uint64) & np.uint64(0xFFFFFFFF))


def threshold(gathered, want):
    nz = np.sort(gathered[gathered != 0])[::-1]
    return np.uint64(1) if nz.size < want else nz[want - 1]


class OracleShardPhases(OracleShard):
    """Adds the global-exact phases: the oracle's per-stage functions on the
    local shard, keys exported in global form, filters by the global cut."""

    def _export(self, ids, sc, d_x, stride):
        x = view(d_x, stride, C.c_int64, np.uint64)
        x[:] = 0
        x[: len(ids)] = ord_key(sc, np.asarray(ids, np.uint64) + self.base)

    def shard_phase1(self, q, rows, dim, params, d_x2, stride2, stream=0, options=None):
        self.q = view(q, rows * dim, C.c_float, np.float32).reshape(rows, dim).copy()
        self.p = params
        S, mx = self.port.compute_centroid_scores(self.h, self.q)
        self.S = S
        c1 = self.port.generate_candidates(self.h, S, params.nprobe)
        self.tr = dict(stage1_candidates=len(c1), stage2_out=0, stage3_out=0, stage2_rows_gathered=0,
                       stage3_rows_gathered=0)
        if len(c1):
            keep = self.port.prune_centroids(mx, params.t_cs)
            sc2, r2 = self.port.centroid_interaction(self.h, c1, S, keep)
            self.ids2, self.sc2 = self.port.select_top(c1, sc2, params.ndocs)
            self.tr["stage2_rows_gathered"] = r2
        else:
            self.ids2, self.sc2 = np.zeros(0, np.uint32), np.zeros(0, np.float32)
        self._export(self.ids2, self.sc2, d_x2, stride2)

    def shard_phase2(self, d_g2, shards, d_x3, stride3, stream=0):
        g2 = view(d_g2, shards * self.stride2, C.c_int64, np.uint64)
        t = threshold(g2, self.p.ndocs)
        ok = ord_key(self.sc2, self.ids2.astype(np.uint64) + self.base) >= t
        ids = self.ids2[ok]
        self.tr["stage2_out"] = len(ids)
        n3 = max(-(-self.p.ndocs // 4), self.p.k)
        if len(ids):
            sc3, r3 = self.port.centroid_interaction(self.h, ids, self.S, None)
            self.ids3, self.sc3 = self.port.select_top(ids, sc3, n3)
            self.tr["stage3_rows_gathered"] = r3
        else:
            self.ids3, self.sc3 = np.zeros(0, np.uint32), np.zeros(0, np.float32)
        self._export(self.ids3, self.sc3, d_x3, stride3)

    def shard_phase3(self, d_g3, shards, d_pids, d_scores, d_n, stream=0):
        g3 = view(d_g3, shards * self.stride3, C.c_int64, np.uint64)
        n3 = max(-(-self.p.ndocs // 4), self.p.k)
        t = threshold(g3, n3)
        ok = ord_key(self.sc3, self.ids3.astype(np.uint64) + self.base) >= t
        fin = self.ids3[ok]
        self.tr["stage3_out"] = len(fin)
        ids, sc = self.port.rank_final(self.h, fin, self.q, self.p.k) if len(fin) else ([], [])
        n = len(ids)
        view(d_pids, self.p.k, C.c_int32, np.uint32)[:n] = np.asarray(ids, np.uint32) + self.base
        view(d_scores, self.p.k, C.c_float, np.float32)[:n] = sc
        view(d_n, 1, C.c_int64, np.int64)[0] = n

    def trace_counters_device(self, d_out, stream=0):
        v = view(d_out, 6, C.c_int64, np.int64)
        t = self.tr
        v[:] = [t["stage1_candidates"], t["stage2_out"], t["stage3_out"], 0, t["stage2_rows_gathered"],
                t["stage3_rows_gathered"]]


GX_PARAMS = [P.SearchParams(20, 2, 0.4, 64), P.SearchParams(20, 8, -1.0, 400), P.SearchParams(10, 1, 0.5, 16), P.SearchParams(5, 2, 0.45, 12),
             P.SearchParams(40, 4, 0.3, 40)]


def worker_gx(rank, world, port_no, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    a, b = shard_range(N, world, rank)
    h = P.generate_index(b - a, K, dim=DIM, nbits=2, mean_len=16, spread=4, seed=SEED, pid_base=a)
    whole = P.generate_index(N, K, dim=DIM, nbits=2, mean_len=16, spread=4, seed=SEED)
    qs = P.generate_queries(whole, 3, seed=77)
    res = []
    for p in GX_PARAMS:
        sh = OracleShardPhases(h, a)
        sh.stride2, sh.stride3 = exchange_strides(p, N)
        ss = ShardedSearcher(sh, k=p.k, mode="global-exact", num_passages=N)
        for q in qs:
            pids, scores, n = ss.search(torch.from_numpy(q.copy()), p)
            m = int(n[0])
            res.append((pids[:m].numpy().astype(np.uint32), scores[:m].numpy().copy(), ss.trace_counters()))
    with open(os.path.join(out_dir, f"gx{rank}.pkl"), "wb") as f:
        pickle.dump(res, f)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_global_exact_gloo(tmp_path, world):
    mp.spawn(worker_gx, args=(world, free_port(), str(tmp_path)), nprocs=world, join=True)
    rs = [pickle.loads((tmp_path / f"gx{r}.pkl").read_bytes()) for r in range(world)]
    port = oracle.get("port")
    whole = P.generate_index(N, K, dim=DIM, nbits=2, mean_len=16, spread=4, seed=SEED)
    qs = P.generate_queries(whole, 3, seed=77)
    i = 0
    differs = 0
    for p in GX_PARAMS:
        for q in qs:
            ids, sc, tr = port.search(whole, q, p)
            for r in rs:
                assert np.array_equal(r[i][0], ids), (p, i)
                assert np.array_equal(r[i][1].view(np.uint32), sc.view(np.uint32))
                for key, v in r[i][2].items():
                    assert tr[key] == v, (key, tr[key], v)
            # the shard-local merge would differ for some of these cases
            allp, alls = [], []
            for g in range(world):
                a, b = shard_range(N, world, g)
                hs = P.generate_index(b - a, K, dim=DIM, nbits=2, mean_len=16, spread=4, seed=SEED, pid_base=a)
                x, y, _ = port.search(hs, q, p)
                allp += list(x + a)
                alls += list(y)
            ep, _ = merge(allp, alls, p.k)
            differs += not np.array_equal(ep, ids)
            i += 1
    assert differs > 0, "test cases do not exercise the global cut"


def worker(rank, world, port_no, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    a, b = shard_range(N, world, rank)
    h = P.generate_index(b - a, K, dim=DIM, nbits=2, mean_len=16, spread=4, seed=SEED, pid_base=a)
    whole = P.generate_index(N, K, dim=DIM, nbits=2, mean_len=16, spread=4, seed=SEED)
    qs = P.generate_queries(whole, 3, seed=77)
    ss = ShardedSearcher(OracleShard(h, a), k=20, mode="shard-local")
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


def worker_bgx(rank, world, port_no, out_dir):
    from paper_2205_09707_b200.sharded import BatchShardedSearcher

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    a, b = shard_range(N, world, rank)
    h = P.generate_index(b - a, K, dim=DIM, nbits=2, mean_len=16, spread=4, seed=SEED, pid_base=a)
    whole = P.generate_index(N, K, dim=DIM, nbits=2, mean_len=16, spread=4, seed=SEED)
    qs = torch.from_numpy(np.ascontiguousarray(P.generate_queries(whole, 5, seed=77)))
    res = []
    for p in GX_PARAMS:
        lanes = []
        for _ in range(2):
            sh = OracleShardPhases(h, a)
            sh.stride2, sh.stride3 = exchange_strides(p, N)
            lanes.append(sh)
        bs = BatchShardedSearcher(lanes, k=p.k, num_passages=N)
        B = qs.shape[0]
        op = torch.zeros(B, p.k, dtype=torch.int32)
        osc = torch.zeros(B, p.k, dtype=torch.float32)
        on = torch.zeros(B, dtype=torch.int64)
        bs.search(qs, p, op, osc, on)
        for i in range(B):
            m = int(on[i])
            res.append((op[i, :m].numpy().astype(np.uint32), osc[i, :m].numpy().copy()))
    with open(os.path.join(out_dir, f"bgx{rank}.pkl"), "wb") as f:
        pickle.dump(res, f)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_batch_global_exact_gloo(tmp_path, world):
    """Throughput mode, global-exact: 5 queries through 2 lanes (a ragged last
    wave), three batched exchanges per wave; every rank's [B][k] equals the
    UNSHARDED reference search of each query, bit for bit."""
    mp.spawn(worker_bgx, args=(world, free_port(), str(tmp_path)), nprocs=world, join=True)
    rs = [pickle.loads((tmp_path / f"bgx{r}.pkl").read_bytes()) for r in range(world)]
    port = oracle.get("port")
    whole = P.generate_index(N, K, dim=DIM, nbits=2, mean_len=16, spread=4, seed=SEED)
    qs = P.generate_queries(whole, 5, seed=77)
    i = 0
    for p in GX_PARAMS:
        for q in qs:
            ids, sc, _ = port.search(whole, q, p)
            for r in rs:
                assert np.array_equal(r[i][0], ids), (p, i)
                assert np.array_equal(r[i][1].view(np.uint32), sc.view(np.uint32)), (p, i)
            i += 1
