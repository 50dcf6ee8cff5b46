"""The synthetic index generator (csrc/synth) the benchmark
and the parity tests run on: deterministic, reference-valid (IVF equal to the
reference's build_inverted_list, validate_index passes), and shardable by
passage range with every stream keyed by global passage id."""
import numpy as np
import pytest

import oracle
import paper_2205_09707_b200 as P


def test_deterministic():
    a = P.generate_index(300, 64, dim=64, nbits=2, mean_len=20, seed=4)
    b = P.generate_index(300, 64, dim=64, nbits=2, mean_len=20, seed=4, threads=3)
    for f in ("centroids", "codes", "residuals", "doclens", "ivf_offsets", "ivf_postings"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f
    qa, qb = P.generate_queries(a, 2, seed=9), P.generate_queries(b, 2, seed=9)
    assert np.array_equal(qa, qb)
    assert np.allclose(np.linalg.norm(qa, axis=2), 1.0, atol=1e-5)


def test_shapes_and_calibration():
    h = P.generate_index(2000, 256, dim=128, nbits=2, mean_len=68, seed=0)
    assert h.doclens.min() >= 52 and h.doclens.max() <= 84
    assert h.residuals.size == h.num_embeddings * 32
    assert np.allclose(np.linalg.norm(h.centroids, axis=1), 1.0, atol=1e-5)
    ratio = len(h.ivf_postings) / h.num_embeddings          # ~0.72 postings per token (§8d)
    assert 0.6 < ratio < 0.8


@pytest.mark.skipif(not oracle.available("ref"), reason="oracle/_ref not built")
def test_reference_accepts_index(ref):
    h = P.generate_index(400, 64, dim=128, nbits=2, mean_len=30, seed=2)
    ref.validate_index(h)
    off, post = ref.build_inverted_list(h.codes, h.doclens, h.num_centroids)
    assert np.array_equal(off, h.ivf_offsets) and np.array_equal(post, h.ivf_postings)


def test_shard_is_slice_of_whole():
    whole = P.generate_index(500, 64, dim=32, nbits=2, mean_len=12, spread=4, seed=3)
    a, b = 180, 320
    part = P.generate_index(b - a, 64, dim=32, nbits=2, mean_len=12, spread=4, seed=3, pid_base=a)
    o = whole.passage_offsets
    assert np.array_equal(part.doclens, whole.doclens[a:b])
    assert np.array_equal(part.codes, whole.codes[o[a]:o[b]])
    bpt = whole.bytes_per_token
    assert np.array_equal(part.residuals, whole.residuals[o[a] * bpt:o[b] * bpt])
    # local IVF = the whole IVF restricted to the range, rebased
    for c in range(64):
        w = whole.ivf_postings[whole.ivf_offsets[c]:whole.ivf_offsets[c + 1]]
        w = w[(w >= a) & (w < b)] - a
        p = part.ivf_postings[part.ivf_offsets[c]:part.ivf_offsets[c + 1]]
        assert np.array_equal(w, p)


@pytest.mark.parametrize("nbits,dim,K,pid_base", [(2, 128, 300, 0), (1, 64, 17, 1234), (4, 32, 64, 7)])
def test_oracle_generator_equals_product(nbits, dim, K, pid_base):
    """The checker-side restatement of the recipe (oracle/synth_oracle.c, the
    reference arm's input generator) produces the product generator's bytes."""
    from oracle import synth

    a = P.generate_index(700, K, dim=dim, nbits=nbits, mean_len=30, seed=5, pid_base=pid_base)
    ivf = (lambda c, d, k: (a.ivf_offsets, a.ivf_postings)) if not oracle.available("ref") else None
    b = synth.generate_index(700, K, dim=dim, nbits=nbits, mean_len=30, seed=5, pid_base=pid_base, ivf=ivf)
    for f in ("centroids", "codes", "residuals", "doclens", "passage_offsets", "ivf_offsets", "ivf_postings",
              "bucket_cutoffs", "bucket_weights"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f
    assert np.array_equal(P.generate_queries(a, 3, seed=8), synth.generate_queries(b, 3, seed=8))
