"""The full index build on the GPU (plaid_build_index) against the
reference's own lir::build_index (oracle/_ref): centroids (k-means++ seeding,
Lloyd iterations, empty-cluster repair), quantizer, codes, residuals and IVF
bit-identical for the same corpus, config and seed; the reference's error
codes for bad input."""
import numpy as np
import pytest

import paper_2205_09707_b200 as P

pytestmark = pytest.mark.gpu


def corpus(n_pass, dim, seed, topics=0, dup=False):
    rng = np.random.default_rng(seed)
    doclens = rng.integers(1, 40, n_pass).astype(np.uint32)
    T = int(doclens.sum())
    if topics:
        centers = rng.standard_normal((topics, dim)).astype(np.float32)
        x = centers[rng.integers(0, topics, T)] + 0.3 * rng.standard_normal((T, dim)).astype(np.float32)
    else:
        x = rng.standard_normal((T, dim)).astype(np.float32)
    if dup:
        x[: T // 2] = x[0]  # half the corpus one point: empty clusters to repair
    x = (x / np.linalg.norm(x.astype(np.float64), axis=1, keepdims=True)).astype(np.float32)
    x = (x / np.linalg.norm(x.astype(np.float64), axis=1, keepdims=True)).astype(np.float32)
    return x, doclens


@pytest.mark.parametrize("dim,nbits,K,iters,seed,topics,dup", [
    (128, 2, 64, 4, 42, 0, False),
    (128, 1, 0, 3, 7, 16, False),    # auto K, clustered corpus
    (64, 4, 96, 2, 3, 0, True),      # duplicates -> empty-cluster repair
    (128, 2, 512, 5, 11, 40, False),  # quantizer pool from a token subset (T > 8192)
])
def test_build_index_matches_reference(ref, dim, nbits, K, iters, seed, topics, dup):
    x, dl = corpus(400 if K != 512 else 900, dim, seed, topics, dup)
    d = ref.build_index(x, dl, dim, nbits, K, iters=iters, seed=seed)
    h = P.build_index(x, dl, nbits=nbits, num_centroids=K, iters=iters, seed=seed)
    assert np.array_equal(h.centroids.view(np.uint32), d["centroids"].view(np.uint32))
    assert np.array_equal(h.bucket_cutoffs.view(np.uint32), d["bucket_cutoffs"].view(np.uint32))
    assert np.array_equal(h.bucket_weights.view(np.uint32), d["bucket_weights"].view(np.uint32))
    assert np.array_equal(h.codes, d["codes"])
    assert np.array_equal(h.residuals, d["residuals"])
    assert np.array_equal(h.ivf_offsets, d["ivf_offsets"])
    assert np.array_equal(h.ivf_postings, d["ivf_postings"])


def test_build_index_errors():
    x, dl = corpus(20, 16, 1)
    with pytest.raises(P.PlaidError) as e:
        P.build_index(x, dl, nbits=3)
    assert e.value.code == P.ErrorCode.PackingUnsupported
    with pytest.raises(P.PlaidError) as e:
        P.build_index(x, dl, nbits=2, num_centroids=int(dl.sum()) + 5)
    assert e.value.code == P.ErrorCode.TooFewPoints
    y = x.copy()
    y[3] *= 2
    with pytest.raises(P.PlaidError) as e:
        P.build_index(y, dl, nbits=2, num_centroids=4)
    assert e.value.code == P.ErrorCode.NotNormalized
