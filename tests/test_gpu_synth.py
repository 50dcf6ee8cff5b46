"""The device-side synthetic corpus generator (csrc/synth_device.cu): the
integer arrays equal the host generator's (same SplitMix64 streams), centroids
and queries agree to fp32 rounding (device vs host libm), shards are slices of
the whole, and the generated index searches exactly like the host-built one."""
import numpy as np
import pytest

import paper_2205_09707_b200 as P

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("nbits,K,pid_base", [(2, 300, 0), (1, 64, 4321), (4, 129, 7)])
def test_device_generator_matches_host(nbits, K, pid_base):
    a = P.generate_index(900, K, dim=128, nbits=nbits, mean_len=30, seed=5, pid_base=pid_base)
    d = P.DeviceIndex.synth(900, K, dim=128, nbits=nbits, mean_len=30, seed=5, pid_base=pid_base)
    assert d.pid_base == pid_base
    b = d.to_host()
    for f in ("codes", "residuals", "doclens", "ivf_offsets", "ivf_postings", "bucket_cutoffs", "bucket_weights"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f
    assert np.abs(a.centroids - b.centroids).max() < 1e-6
    qa, qb = P.generate_queries(a, 3, seed=8), d.synth_queries(3, seed=8)
    assert np.abs(qa - qb).max() < 1e-5


def test_device_index_searches_like_host(port):
    h = P.generate_index(5000, 512, dim=128, nbits=2, mean_len=40, seed=3)
    d = P.DeviceIndex.synth(5000, 512, dim=128, nbits=2, mean_len=40, seed=3)
    hb = d.to_host()  # the device corpus, bit for bit (centroids included)
    qs = P.generate_queries(hb, 3, seed=4)
    s = P.Searcher(d, score_mode=P.ScoreMode.EXACT)
    for k in (10, 1000):
        p = P.default_params_for_k(k)
        for q in qs:
            got = s.search(q, p)
            ids, sc, tr = port.search(hb, q, p)
            assert np.array_equal(got.topk.passage_ids, ids)
            assert np.array_equal(got.topk.scores.view(np.uint32), sc.view(np.uint32))
            assert got.trace.counters() == tr
