"""SPEC known-answer tests (the reference ships no tests; its SPEC's worked
examples and acceptance criteria are the test plan) run on both
CPU oracles: the C restatement ("port") and the compiled reference ("ref").
These pin the oracle before it is trusted as the checker of the CUDA path."""
import itertools

import numpy as np
import pytest

import oracle
from paper_2205_09707_b200.hostindex import HostIndex, build_inverted_list

KINDS = ["port"] + (["ref"] if oracle.available("ref") else [])


@pytest.fixture(params=KINDS)
def orc(request):
    return oracle.get(request.param)


def tiny_index(codes, doclens, centroids, nbits=2, weights=None):
    """Hand-built index: residual bytes all zero (bucket 0)."""
    centroids = np.asarray(centroids, dtype=np.float32)
    K, dim = centroids.shape
    codes = np.asarray(codes, dtype=np.uint32)
    doclens = np.asarray(doclens, dtype=np.uint32)
    ivo, post = build_inverted_list(codes, doclens, K)
    cut = np.zeros((1 << nbits) - 1, dtype=np.float32)
    w = np.zeros(1 << nbits, dtype=np.float32) if weights is None else np.asarray(weights, np.float32)
    res = np.zeros(codes.size * nbits * dim // 8, dtype=np.uint8)
    return HostIndex(dim, nbits, centroids, codes, res, doclens, ivo, post, cut, w)


def bitshift_unpack(byte, b):
    return [(byte >> (b * j)) & ((1 << b) - 1) for j in range(8 // b)]


# ---------------------------------------------------------------- codec
def test_pack_examples(orc):
    assert orc.pack_residual([0, 1, 2, 3], 2).tolist() == [0xE4]
    assert orc.pack_residual([1, 0, 0, 0, 0, 0, 0, 0], 1).tolist() == [0x01]


def test_unpack_examples(orc):
    assert orc.unpack_via_lut([0xE4], 2).tolist() == [0, 1, 2, 3]
    for b in (1, 2, 4):
        assert orc.unpack_via_lut([0x00], b).tolist() == [0] * (8 // b)


@pytest.mark.parametrize("b", [1, 2, 4])
def test_lut_exhaustive_and_roundtrip(orc, b):
    """Acceptance #3: LUT == bit-shift, exhaustive; round trip."""
    lut = orc.lut_build(b)
    for v in range(256):
        assert lut[v].tolist() == bitshift_unpack(v, b)
    allb = np.arange(256, dtype=np.uint8)
    idx = orc.unpack_via_lut(allb, b)
    assert np.array_equal(orc.pack_residual(idx, b), allb)
    rng = np.random.default_rng(b)
    x = rng.integers(0, 1 << b, size=8 * 1000, dtype=np.uint8)
    assert np.array_equal(orc.unpack_via_lut(orc.pack_residual(x, b), b), x)


def test_pack_errors(orc):
    with pytest.raises(oracle.OracleError) as e:
        orc.pack_residual([4, 0, 0, 0], 2)
    assert e.value.code == 5  # IndexOutOfRange
    with pytest.raises(oracle.OracleError) as e:
        orc.pack_residual([1, 0, 0], 2)
    assert e.value.code == 6  # LengthNotPackable


def test_reconstruct_zero_weights_is_centroid(orc):
    """all-zero weights -> v^ = centroid exactly."""
    rng = np.random.default_rng(3)
    C = rng.standard_normal((4, 8)).astype(np.float32)
    C /= np.linalg.norm(C, axis=1, keepdims=True)
    h = tiny_index([0, 1, 2, 3], [4], C)
    out = orc.reconstruct(h, h.codes, h.residuals)
    assert np.allclose(out, C, atol=1e-7)
    assert np.allclose(np.linalg.norm(out, axis=1), 1.0, atol=1e-6)


# ---------------------------------------------------------------- maxsim
def test_maxsim_packed_examples(orc):
    assert orc.maxsim_packed(np.array([[0.3, 0.7]]), [0, 1]).tolist() == pytest.approx([1.0])
    S = np.array([[1, 0], [0, 1], [1, 0]], dtype=np.float32)
    assert orc.maxsim_packed(S, [0, 1, 3]).tolist() == [1.0, 2.0]


def test_maxsim_packed_empty_range(orc):
    with pytest.raises(oracle.OracleError) as e:
        orc.maxsim_packed(np.zeros((2, 2), np.float32), [0, 0, 2])
    assert e.value.code == 7  # EmptyPassageRange


def test_maxsim_embeddings_examples(orc):
    e1, e2 = np.eye(4, dtype=np.float32)[:2]
    assert orc.maxsim_embeddings(e1[None], e1[None], [0, 1]).tolist() == [1.0]
    assert orc.maxsim_embeddings(np.stack([e1, e2]), e1[None], [0, 1]).tolist() == [1.0]


def test_maxsim_packed_matches_padded(orc):
    """Acceptance #2 at desk scale: padded reference within 1e-6."""
    rng = np.random.default_rng(7)
    for _ in range(50):
        lens = rng.integers(1, 9, size=rng.integers(1, 6))
        off = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64)
        S = rng.uniform(-1, 1, size=(int(off[-1]), 5)).astype(np.float32)
        got = orc.maxsim_packed(S, off)
        pad = np.full((len(lens), lens.max(), 5), -np.inf, dtype=np.float64)
        for p, (a, b) in enumerate(zip(off[:-1], off[1:])):
            pad[p, : b - a] = S[a:b]
        assert np.allclose(got, pad.max(axis=1).sum(axis=1), atol=1e-6)


# ---------------------------------------------------------------- pipeline
def test_centroid_scores_identity(orc):
    h = tiny_index([0, 1], [2], np.eye(2, dtype=np.float32))
    S, mx = orc.compute_centroid_scores(h, np.array([[1, 0]], np.float32))
    assert S.tolist() == [[1.0], [0.0]] and mx.tolist() == [1.0, 0.0]
    S2, _ = orc.compute_centroid_scores(h, np.array([[1, 0], [1, 0]], np.float32))
    assert np.array_equal(S2[:, 0], S2[:, 1])                                 # duplicated columns


def test_prune_examples(orc):
    assert orc.prune_centroids([0.9, 0.5, -1.0], -1.0).tolist() == [1, 1, 1]
    assert orc.prune_centroids([0.9, 0.5], 0.6).tolist() == [1, 0]
    assert orc.prune_centroids([0.6], np.float32(0.6)).tolist() == [1]        # non-strict, :358


def test_select_top_examples(orc):
    ids, sc = orc.select_top([0, 1], [0.5, 0.5], 1)
    assert ids.tolist() == [0]
    ids, sc = orc.select_top([5, 3, 9], [0.1, 0.7, 0.7], 10)                  # n >= size
    assert ids.tolist() == [3, 9, 5] and sc.tolist() == pytest.approx([0.7, 0.7, 0.1])
    ids, _ = orc.select_top([2, 1], [-0.0, 0.0], 2)                           # -0 == +0 -> id order
    assert ids.tolist() == [1, 2]


def test_generate_candidates_examples(orc):
    # single token, nprobe 1: top centroid's postings
    C = np.eye(3, dtype=np.float32)
    h = tiny_index([2, 0, 1, 0, 0, 1, 1, 0], [1, 1, 1, 1, 1, 1, 1, 1], C)
    S, _ = orc.compute_centroid_scores(h, np.array([[0, 1, 0]], np.float32))
    assert orc.generate_candidates(h, S, 1).tolist() == [2, 5, 6]
    # nprobe = K covers every passage with >= 1 token
    assert orc.generate_candidates(h, S, 3).tolist() == list(range(8))


def test_centroid_interaction_examples(orc):
    # every token on centroid c with S[c] = (1, 1) -> 2.0
    C = np.array([[1, 0], [0, 1]], np.float32)
    h = tiny_index([0, 0, 1], [2, 1], C)
    S = np.array([[1.0, 1.0], [0.25, 0.5]], np.float32)
    sc, rows = orc.centroid_interaction(h, np.array([0, 1], np.uint32), S, None)
    assert sc.tolist() == [2.0, 0.75] and rows == 3
    # all tokens masked -> score 0 (design decision)
    sc, rows = orc.centroid_interaction(h, np.array([0, 1], np.uint32), S, np.array([1, 0], np.uint8))
    assert sc.tolist() == [2.0, 0.0] and rows == 2
    with pytest.raises(oracle.OracleError) as e:
        orc.centroid_interaction(h, np.array([], np.uint32), S, None)
    assert e.value.code == 8  # InvalidParams on empty candidates (pipeline.cpp:101-103)


def test_build_inverted_list_examples():
    off, post = build_inverted_list(np.array([0, 0, 1], np.uint32), np.array([2, 1], np.uint32), 2)
    assert off.tolist() == [0, 1, 2] and post.tolist() == [0, 1]
    off, post = build_inverted_list(np.array([2, 2, 2], np.uint32), np.array([1, 1, 1], np.uint32), 3)
    assert off.tolist() == [0, 0, 0, 3] and post.tolist() == [0, 1, 2]


def test_validate_query_examples(orc):
    orc.validate_query(np.eye(4, dtype=np.float32)[:2], 4)
    with pytest.raises(oracle.OracleError) as e:
        orc.validate_query(np.array([[2, 0, 0, 0]], np.float32), 4)
    assert e.value.code == 1
    with pytest.raises(oracle.OracleError) as e:
        orc.validate_query(np.array([[1, 0, 0]], np.float32), 4)
    assert e.value.code == 0


def test_params(orc):
    assert orc.default_params_for_k(10) == (10, 1, pytest.approx(0.5), 256)
    assert orc.default_params_for_k(100) == (100, 2, pytest.approx(0.45), 1024)
    assert orc.default_params_for_k(1000) == (1000, 4, pytest.approx(0.4), 4096)

    class Prm:
        def __init__(self, k, nprobe, t_cs, ndocs):
            self.k, self.nprobe, self.t_cs, self.ndocs = k, nprobe, t_cs, ndocs

    assert orc.stage3_width(Prm(10, 1, 0.5, 256)) == 64
    assert orc.stage3_width(Prm(1000, 4, 0.4, 4096)) == 1024
    assert orc.stage3_width(Prm(100, 1, 0.5, 10)) == 100       # max(ceil(ndocs/4), k)
    assert orc.stage3_width(Prm(1, 1, 0.5, 5)) == 2            # ceiling
    for bad in (Prm(0, 1, 0.5, 256), Prm(10, 0, 0.5, 256), Prm(10, 9, 0.5, 256)):
        with pytest.raises(oracle.OracleError) as e:
            orc.validate_params(bad, 8)
        assert e.value.code == 8


def test_search_self_match_ranks_first(orc):
    """a passage whose tokens equal the query tokens ranks first."""
    rng = np.random.default_rng(5)
    C = rng.standard_normal((16, 16)).astype(np.float32)
    C /= np.linalg.norm(C, axis=1, keepdims=True)
    codes = rng.integers(0, 16, size=40).astype(np.uint32)
    h = tiny_index(codes, [4] * 10, C)

    class Prm:
        k, nprobe, t_cs, ndocs = 3, 1, 0.5, 8

    for p in range(10):
        q = C[h.passage_codes(p)]
        ids, sc, tr = orc.search(h, q, Prm)
        ids = ids.tolist()
        assert p in ids and sc[ids.index(p)] == sc[0]   # first, or tied with the first


def test_search_empty_c1_returns_empty(orc):
    C = np.eye(4, dtype=np.float32)
    h = tiny_index([0, 0], [2], C)           # only centroid 0 has postings

    class Prm:
        k, nprobe, t_cs, ndocs = 5, 1, 0.5, 8

    ids, sc, tr = orc.search(h, np.array([[0, 1, 0, 0]], np.float32), Prm)
    assert ids.size == 0 and tr["stage1_candidates"] == 0 and tr["centroid_matmul_count"] == 1


def test_lut_covers_all_bytes_for_all_widths():
    for b, kind in itertools.product((1, 2, 4), KINDS):
        assert oracle.get(kind).lut_build(b).shape == (256, 8 // b)
