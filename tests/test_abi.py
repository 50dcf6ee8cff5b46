"""The drop-in boundary (include/plaid.h) on a host without a GPU: the CUDA
library loads, exports every declared entry point, its host-side validation
matches the reference, and every compute entry point fails loudly (a CUDA
error status, never a silent CPU answer)."""
import ctypes as C
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

import paper_2205_09707_b200 as P
from paper_2205_09707_b200 import _native as N

from .conftest import HAS_GPU, ROOT

HEADER = ROOT / "include" / "plaid.h"


def declared():
    src = HEADER.read_text()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(plaid_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = declared()
    for must in ("plaid_search", "plaid_search_batch", "plaid_index_from_host", "plaid_index_close",
                 "plaid_searcher_create", "plaid_last_error", "plaid_compute_centroid_scores",
                 "plaid_generate_candidates", "plaid_prune_centroids", "plaid_centroid_interaction",
                 "plaid_select_top", "plaid_rank_final", "plaid_reconstruct", "plaid_maxsim_packed",
                 "plaid_maxsim_embeddings", "plaid_merge_topk"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = N.load()
    so = Path(lib._name)
    assert so.is_relative_to(ROOT), "the CUDA library must be the in-tree build"
    for name in declared():
        assert hasattr(lib, name), name
    # and they are real dynamic exports (not only resolvable through Python)
    out = subprocess.run(["nm", "-D", "--defined-only", str(so)], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (plaid_[a-z0-9_]+)", out))
    assert set(declared()) <= exported


def test_library_is_sm100a_and_does_not_link_libcuda():
    so = Path(N.load()._name)
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(so)], capture_output=True, text=True)
    assert "sm_100a" in out.stdout
    ldd = subprocess.run(["ldd", str(so)], capture_output=True, text=True).stdout
    assert "libcuda.so" not in ldd


def test_abi_version_and_status_names():
    lib = N.load()
    assert lib.plaid_abi_version() == 1
    lib.plaid_status_name.restype = C.c_char_p
    assert lib.plaid_status_name(0) == b"Ok"
    assert lib.plaid_status_name(int(P.ErrorCode.NotNormalized) + 1) == b"NotNormalized"


def test_host_validation_matches_reference(port):
    rng = np.random.default_rng(0)
    for q in (np.eye(4, dtype=np.float32)[:2], np.array([[2, 0, 0, 0]], np.float32),
              np.array([[1, 0, 0]], np.float32), rng.standard_normal((3, 4)).astype(np.float32),
              np.array([[1, 0, 0, 1e-4]], np.float32), np.array([[1, 0, 0, 0.05]], np.float32)):
        want = None
        try:
            port.validate_query(q, 4)
        except Exception as e:  # noqa: BLE001
            want = e.code
        got = None
        try:
            P.validate_query(q, 4)
        except P.PlaidError as e:
            got = int(e.code)
        assert got == want, q
    for k in (1, 10, 11, 100, 101, 1000, 5000):
        a = P.default_params_for_k(k)
        assert (a.k, a.nprobe, a.ndocs) == port.default_params_for_k(k)[:2] + port.default_params_for_k(k)[3:]
        assert P.stage3_width(a) == port.stage3_width(a)
    for prm, K in ((P.SearchParams(0, 1, 0.5, 8), 8), (P.SearchParams(5, 9, 0.5, 8), 8),
                   (P.SearchParams(5, 2, 0.5, 0), 8), (P.SearchParams(5, 2, 0.5, 8), 8)):
        want = None
        try:
            port.validate_params(prm, K)
        except Exception as e:  # noqa: BLE001
            want = e.code
        got = None
        try:
            P.validate_params(prm, K)
        except P.PlaidError as e:
            got = int(e.code)
        assert got == want


@pytest.mark.parametrize("b", [1, 2, 4])
def test_host_codec_tables_match_reference(port, b):
    assert np.array_equal(P.lut_build(b), port.lut_build(b))
    x = np.random.default_rng(b).integers(0, 1 << b, size=64 * 8, dtype=np.uint8)
    assert np.array_equal(P.pack_residual(x, b), port.pack_residual(x, b))
    with pytest.raises(P.PlaidError) as e:
        P.lut_build(3)
    assert e.value.code == P.ErrorCode.PackingUnsupported


@pytest.mark.skipif(HAS_GPU, reason="checks the no-GPU behaviour")
def test_compute_fails_loudly_without_gpu():
    h = P.generate_index(50, 16, dim=32, nbits=2, mean_len=8, spread=4)
    with pytest.raises(P.PlaidError) as e:
        P.DeviceIndex.from_host(h)
    assert e.value.code == P.ErrorCode.CudaError
    with pytest.raises(P.PlaidError) as e:
        P.Searcher(None)
    assert e.value.code == P.ErrorCode.CudaError


DROPIN = ROOT / "oracle" / "_ref" / "lir_dropin"


@pytest.mark.skipif(HAS_GPU or not DROPIN.exists(), reason="no-GPU behaviour of the lir drop-in binary")
def test_lir_dropin_fails_loudly_without_gpu():
    """Reference lir code linked against libplaid through include/plaid_lir.hpp
    (oracle/lir_dropin.cpp): without a GPU the engine refuses, no CPU answer."""
    r = subprocess.run([str(DROPIN)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 2 and r.stdout.startswith("NOGPU")
