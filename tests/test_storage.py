"""On-disk index format (FORMAT.md; SPEC.md storage module):
save -> load round trips byte for byte, the manifest's dimensional
bookkeeping holds, a tampered byte is a ChecksumMismatch, the C++ digest
equals an independent numpy implementation.  CPU only (the GPU loader is
covered in test_gpu_parity.py)."""
import json
import os

import numpy as np
import pytest

import paper_2205_09707_b200 as P


@pytest.fixture(scope="module")
def small_index():
    return P.generate_index(700, 64, dim=64, nbits=2, mean_len=20, spread=6, seed=9)


def test_digest_matches_numpy():
    rng = np.random.default_rng(1)
    for n in (0, 1, 7, 8, 9, 1000, 65535, 65536, 65537, 3 * 65536 + 13):
        b = rng.integers(0, 256, n, dtype=np.uint8)
        assert P.checksum(b) == P.fnv_digest(b), n


def test_save_load_roundtrip(tmp_path, small_index):
    h = small_index
    P.save_index(h, tmp_path, rng_seed=9)
    m = json.loads((tmp_path / "manifest.json").read_text())
    assert m["format_version"] == 1 and m["num_centroids"] == h.num_centroids
    assert m["num_embeddings"] == int(h.doclens.sum()) == h.num_embeddings  # SPEC storage invariant
    assert os.path.getsize(tmp_path / "residuals.bin") == h.num_embeddings * h.nbits * h.dim // 8
    assert os.path.getsize(tmp_path / "ivf_offsets.u64") == 8 * (h.num_centroids + 1)
    g = P.load_index_host(tmp_path)
    for a in ("centroids", "codes", "residuals", "doclens", "ivf_offsets", "ivf_postings", "bucket_cutoffs",
              "bucket_weights"):
        x, y = getattr(h, a), getattr(g, a)
        assert x.dtype == y.dtype and np.array_equal(x.view(np.uint8), y.view(np.uint8)), a


def test_tamper_is_checksum_mismatch(tmp_path, small_index):
    P.save_index(small_index, tmp_path)
    p = tmp_path / "residuals.bin"
    b = bytearray(p.read_bytes())
    b[len(b) // 2] ^= 1
    p.write_bytes(bytes(b))
    with pytest.raises(P.PlaidError) as e:
        P.load_index_host(tmp_path)
    assert e.value.code == P.ErrorCode.ChecksumMismatch


def test_k1_offsets_and_version(tmp_path):
    h = P.generate_index(50, 1, dim=16, nbits=1, mean_len=4, spread=2, seed=2)
    P.save_index(h, tmp_path)
    assert os.path.getsize(tmp_path / "ivf_offsets.u64") == 16  # K = 1 -> 2 entries
    m = json.loads((tmp_path / "manifest.json").read_text())
    m["format_version"] = 7
    (tmp_path / "manifest.json").write_text(json.dumps(m))
    with pytest.raises(P.PlaidError) as e:
        P.load_index_host(tmp_path)
    assert e.value.code == P.ErrorCode.UnsupportedVersion


def test_save_to_missing_dir_is_io_error(tmp_path, small_index):
    with pytest.raises(P.PlaidError) as e:
        P.save_index(small_index, tmp_path / "nope")
    assert e.value.code == P.ErrorCode.IoError
    assert not list(tmp_path.iterdir())
