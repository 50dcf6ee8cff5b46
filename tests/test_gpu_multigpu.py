"""The single-process multi-GPU searcher (plaid_sharded_*)
through the C ABI: G passage-range shards (on one GPU here; on several GPUs
the same exchange kernels read peers over NVLink) against the unsharded
reference.  Global-exact reproduces lir::search bit for bit in EXACT mode
(ids, score bits, summed trace counters); shard-local equals the reference
run per shard + the top-k merge; TENSOR mode is classified with the
north_star comparator.  Also the one-kernel batch merge of throughput mode."""
import numpy as np
import pytest

import paper_2205_09707_b200 as P
from paper_2205_09707_b200.sharded import shard_range

pytestmark = pytest.mark.gpu

N, K = 6000, 512


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)


@pytest.fixture(scope="module")
def whole():
    h = P.generate_index(N, K, dim=128, nbits=2, mean_len=40, seed=4)
    return h, P.generate_queries(h, 4, seed=21)


def shard_indexes(G):
    out = []
    for g in range(G):
        a, b = shard_range(N, G, g)
        hs = P.generate_index(b - a, K, dim=128, nbits=2, mean_len=40, seed=4, pid_base=a)
        out.append((hs, a, P.DeviceIndex.from_host_at(hs, pid_base=a)))
    return out


CASES = [P.default_params_for_k(10), P.default_params_for_k(100), P.default_params_for_k(1000),
         P.SearchParams(20, 8, -1.0, 300), P.SearchParams(50, 4, 0.3, 64)]


@pytest.mark.parametrize("G", [1, 2, 3, 5])
def test_global_exact_equals_unsharded(whole, port, G):
    h, qs = whole
    sh = shard_indexes(G)
    ms = P.MultiGpuSearcher([ix for _, _, ix in sh], score_mode=P.ScoreMode.EXACT, mode="global-exact")
    for p in CASES:
        for q in qs:
            got = ms.search(q, p)
            ids, sc, tr = port.search(h, q, p)
            assert np.array_equal(got.topk.passage_ids, ids), (G, p)
            assert np.array_equal(bits(got.topk.scores), bits(sc)), (G, p)
            assert got.trace.counters() == tr, (G, p)
    p = P.default_params_for_k(10)
    got = ms.search(qs[0], p, P.SearchOptions(disable_filter=True))
    ids, sc, tr = port.search(h, qs[0], p, disable_filter=True)
    assert np.array_equal(got.topk.passage_ids, ids) and np.array_equal(bits(got.topk.scores), bits(sc))
    assert got.trace.counters() == tr


def test_shard_local_is_per_shard_plus_merge(whole, port):
    h, qs = whole
    sh = shard_indexes(3)
    ms = P.MultiGpuSearcher([ix for _, _, ix in sh], score_mode=P.ScoreMode.EXACT, mode="shard-local")
    for p in CASES[:3]:
        for q in qs:
            got = ms.search(q, p)
            allp, alls = [], []
            for hs, a, _ in sh:
                ids, sc, _ = port.search(hs, q, p)
                allp.append(ids + a)
                alls.append(sc)
            eids, esc = port.select_top(np.concatenate(allp), np.concatenate(alls), p.k)
            assert np.array_equal(got.topk.passage_ids, eids)
            assert np.array_equal(bits(got.topk.scores), bits(esc))


def test_global_exact_tensor_vs_reference(whole, port):
    from oracle.compare import check_tensor_search

    h, qs = whole
    sh = shard_indexes(3)
    ms = P.MultiGpuSearcher([ix for _, _, ix in sh], score_mode=P.ScoreMode.TENSOR)
    single = P.Searcher(P.DeviceIndex.from_host(h), score_mode=P.ScoreMode.TENSOR)
    for k in (10, 1000):
        p = P.default_params_for_k(k)
        for q in qs:
            got = ms.search(q, p)
            S, _ = single.compute_centroid_scores(q)
            rep = check_tensor_search(port, h, q, p, got.topk.passage_ids, got.topk.scores, S,
                                      got_counters=got.trace.counters())
            assert rep.ok, rep.as_dict()


def test_sharded_rejects_bad_input(whole):
    h, qs = whole
    sh = shard_indexes(2)
    ms = P.MultiGpuSearcher([ix for _, _, ix in sh], score_mode=P.ScoreMode.EXACT)
    bad = qs[0].copy()
    bad[3] *= 2
    with pytest.raises(P.PlaidError) as e:
        ms.search(bad, P.default_params_for_k(10))
    assert e.value.code == P.ErrorCode.NotNormalized
    with pytest.raises(P.PlaidError) as e:
        ms.search(qs[0], P.SearchParams(10, 0, 0.5, 100))
    assert e.value.code == P.ErrorCode.InvalidParams


@pytest.mark.parametrize("G,B,k", [(1, 5, 10), (4, 33, 100), (8, 7, 1000)])
def test_merge_topk_batch_device(port, G, B, k):
    import torch

    rng = np.random.default_rng(G * B + k)
    pids = np.zeros((G, B, k), np.uint32)
    sc = np.zeros((G, B, k), np.float32)
    cnt = rng.integers(0, k + 1, (G, B)).astype(np.uint64)
    for g in range(G):
        for j in range(B):
            c = int(cnt[g, j])
            pids[g, j, :c] = rng.permutation(100000)[:c] + g * 100000
            sc[g, j, :c] = np.sort(rng.choice(np.array([0.5, 1.25, -2.0, 3.0], np.float32), c))[::-1]
    d_p = torch.from_numpy(pids.view(np.int32)).cuda()
    d_s = torch.from_numpy(sc).cuda()
    d_c = torch.from_numpy(cnt.view(np.int64)).cuda()
    op = torch.zeros(B * k, dtype=torch.int32, device="cuda")
    os_ = torch.zeros(B * k, dtype=torch.float32, device="cuda")
    on = torch.zeros(B, dtype=torch.int64, device="cuda")
    s = P.Searcher(None)
    s.merge_topk_batch_device(d_p.data_ptr(), d_s.data_ptr(), d_c.data_ptr(), G, B, k, op.data_ptr(),
                              os_.data_ptr(), on.data_ptr())
    torch.cuda.synchronize()
    op, os_, on = op.cpu().numpy().view(np.uint32).reshape(B, k), os_.cpu().numpy().reshape(B, k), on.cpu().numpy()
    for j in range(B):
        ap = np.concatenate([pids[g, j, :int(cnt[g, j])] for g in range(G)])
        asc = np.concatenate([sc[g, j, :int(cnt[g, j])] for g in range(G)])
        eids, esc = port.select_top(ap, asc, k)
        m = int(on[j])
        assert m == len(eids)
        assert np.array_equal(op[j, :m], eids) and np.array_equal(os_[j, :m], esc)
