"""In-tree build of the native libraries (no JIT cache: the .so files travel
with the repo snapshot to the GPU box).

    libplaid.so        CUDA kernels (sm_100a) + C++ engine + C ABI (include/plaid.h)
    libplaid_synth.so  host-only synthetic index generator (fixtures)

Compiled with nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo.
Objects are rebuilt when their source or any header is newer.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "_lib"
BUILD = PKG / "_build"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + [
    "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
    "--expt-relaxed-constexpr", "-I", str(CSRC), "-I", str(ROOT / "include"),
]
CU_SOURCES = ["scores.cu", "candidates.cu", "interaction.cu", "select.cu", "rank.cu", "rank128.cu", "gemm_tf32.cu", "range_stage2.cu", "wave_scores.cu", "wave_worker.cu", "storage.cu", "encode.cu", "synth_device.cu"]
CPP_SOURCES = ["engine.cpp", "capi.cpp"]


def _headers() -> list[Path]:
    return list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.hpp")) + [ROOT / "include" / "plaid.h"]


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.exists() and d.stat().st_mtime > t for d in deps)


def _run(cmd: list[str], verbose: bool) -> None:
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"build step failed: {' '.join(cmd[:4])} ...")
    if verbose and (r.stdout or r.stderr):
        sys.stderr.write(r.stdout + r.stderr)


def build_plaid(verbose: bool = False, jobs: int = 8) -> Path:
    LIB.mkdir(exist_ok=True)
    BUILD.mkdir(exist_ok=True)
    hdrs = _headers()
    objs, jobs_list = [], []
    for src in CU_SOURCES + CPP_SOURCES:
        s = CSRC / src
        if not s.exists():
            continue
        o = BUILD / (s.stem + ".o")
        objs.append(o)
        if _stale(o, [s] + hdrs):
            lang = [] if src.endswith(".cu") else ["-x", "cu"]
            jobs_list.append([NVCC, *NVCC_FLAGS, *lang, "-c", str(s), "-o", str(o)])
    with cf.ThreadPoolExecutor(max_workers=jobs) as ex:
        list(ex.map(lambda c: _run(c, verbose), jobs_list))
    so = LIB / "libplaid.so"
    if jobs_list or _stale(so, objs):
        _run([NVCC, *ARCH, "-shared", "-o", str(so), *map(str, objs)], verbose)
    return so


def build_synth(verbose: bool = False) -> Path:
    LIB.mkdir(exist_ok=True)
    src = CSRC / "synth" / "synth.cpp"
    so = LIB / "libplaid_synth.so"
    if _stale(so, [src]):
        _run(["g++", "-std=c++17", "-O3", "-fPIC", "-shared", "-pthread", "-o", str(so), str(src)], verbose)
    return so


def build_oracle(verbose: bool = False) -> None:
    """oracle/liboracle.so always; oracle/_ref/liblir_ref.so when the reference
    sources are present (this container; the GPU box uses the shipped .so)."""
    targets = ["liboracle.so", "libsynth_oracle.so"]
    if Path("/root/reference/proj/src").is_dir():
        targets.append("ref")
    _run(["make", "-s", "-C", str(ROOT / "oracle"), *targets], verbose)


def build_all(verbose: bool = False) -> None:
    build_synth(verbose)
    build_oracle(verbose)
    build_plaid(verbose)
    if Path("/root/reference/proj/src").is_dir():
        # drop-in demonstration: reference lir code calling libplaid (test infra)
        _run(["make", "-s", "-C", str(ROOT / "oracle"), "dropin", "e2e"], verbose)


if __name__ == "__main__":
    build_all(verbose="-v" in sys.argv)
    print("built", LIB)
