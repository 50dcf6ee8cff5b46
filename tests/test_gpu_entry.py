"""GPU coverage of the standalone entry points outside `search`:
maxsim_packed / maxsim_embeddings (/root/reference/proj/src/maxsim.cpp:31-104)
bit-exact against the oracle, including their error contracts, and the
rejection paths of validate_index (index.cpp:12-84) on the device-index
load path, each with the reference's error code."""
import dataclasses

import numpy as np
import pytest

import paper_2205_09707_b200 as P

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)


@pytest.mark.parametrize("nq", [1, 7, 32])
def test_maxsim_packed_gpu(port, nq):
    rng = np.random.default_rng(nq)
    lens = rng.integers(1, 90, 300)
    off = np.zeros(lens.size + 1, np.uint64)
    off[1:] = np.cumsum(lens)
    S = rng.standard_normal((int(off[-1]), nq)).astype(np.float32)
    S[5:40] = -0.0  # signed zeros inside a passage
    s = P.Searcher(None)
    assert np.array_equal(bits(s.maxsim_packed(S, off)), bits(port.maxsim_packed(S, off)))


@pytest.mark.parametrize("rows,dim", [(32, 128), (5, 64), (1, 16), (32, 96)])
def test_maxsim_embeddings_gpu(port, rows, dim):
    rng = np.random.default_rng(rows * dim)
    lens = rng.integers(1, 70, 200)
    off = np.zeros(lens.size + 1, np.uint64)
    off[1:] = np.cumsum(lens)
    q = rng.standard_normal((rows, dim)).astype(np.float32)
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    e = rng.standard_normal((int(off[-1]), dim)).astype(np.float32)
    e /= np.linalg.norm(e, axis=1, keepdims=True)
    s = P.Searcher(None)
    assert np.array_equal(bits(s.maxsim_embeddings(q, e, off)), bits(port.maxsim_embeddings(q, e, off)))


def test_maxsim_errors_gpu(port):
    """check_offsets (maxsim.cpp:11-27): an empty passage, non-monotone offsets."""
    import oracle

    s = P.Searcher(None)
    S = np.ones((10, 4), np.float32)
    for off, code in ((np.array([0, 3, 3, 10], np.uint64), P.ErrorCode.EmptyPassageRange),
                      (np.array([0, 6, 3, 10], np.uint64), P.ErrorCode.InvalidParams)):
        with pytest.raises(P.PlaidError) as e:
            s.maxsim_packed(S, off)
        with pytest.raises(oracle.OracleError) as o:
            port.maxsim_packed(S, off)
        assert e.value.code == o.value.code == code


def _corrupt(h, **changes):
    return dataclasses.replace(h, passage_offsets=None, **changes)


@pytest.fixture(scope="module")
def tiny():
    return P.generate_index(300, 64, dim=64, nbits=2, mean_len=10, spread=4, seed=2)


def _cases(h):
    K = h.num_centroids
    codes_bad = h.codes.copy()
    codes_bad[17] = K + 3                                   # index.cpp: code out of centroid range
    ivo_bad = h.ivf_offsets.copy()
    ivo_bad[5], ivo_bad[6] = ivo_bad[6], ivo_bad[5]         # offsets not monotone
    post_bad = h.ivf_postings.copy()
    post_bad[0] = h.num_passages + 1                        # posting references unknown passage
    post_swap = h.ivf_postings.copy()
    a0, a1 = int(h.ivf_offsets[0]), int(h.ivf_offsets[1])
    assert a1 - a0 >= 2
    post_swap[a0], post_swap[a0 + 1] = post_swap[a0 + 1], post_swap[a0]  # not strictly increasing
    # content mismatch: move one token to another centroid without updating the IVF
    codes_mv = h.codes.copy()
    post0 = [c for c in range(K) if 0 not in h.ivf_postings[h.ivf_offsets[c]:h.ivf_offsets[c + 1]]]
    codes_mv[3] = post0[0]                                  # passage 0 now owns a code whose list lacks it
    w_bad = h.bucket_weights.copy()
    w_bad[0] = 0.5                                          # weight outside its bucket interval
    c_bad = h.centroids.copy()
    c_bad[4] *= 1.5                                         # centroid not unit norm
    return [("code range", _corrupt(h, codes=codes_bad)),
            ("offsets monotone", _corrupt(h, ivf_offsets=ivo_bad)),
            ("unknown passage", _corrupt(h, ivf_postings=post_bad)),
            ("postings order", _corrupt(h, ivf_postings=post_swap)),
            ("ivf content", _corrupt(h, codes=codes_mv)),
            ("quantizer", _corrupt(h, bucket_weights=w_bad)),
            ("centroid norm", _corrupt(h, centroids=c_bad))]


def test_validate_index_rejections_gpu(tiny, ref):
    """Every corruption is rejected at device-index load (validate=True) with
    the error code the reference's validate_index raises on the same arrays."""
    import oracle

    P.DeviceIndex.from_host(tiny, validate=True)  # the clean index passes
    for name, bad in _cases(tiny):
        with pytest.raises(oracle.OracleError) as o:
            ref.validate_index(bad)
        ref.release(bad)
        with pytest.raises(P.PlaidError) as e:
            P.DeviceIndex.from_host(bad, validate=True)
        assert e.value.code == o.value.code, (name, e.value, o.value)


def test_validate_device_copy(tiny):
    """plaid_index_validate re-checks the HBM copy: passes on a clean upload."""
    ix = P.DeviceIndex.from_host(tiny)
    ix.validate()
