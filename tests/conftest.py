import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests through the C ABI")


def _has_gpu() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


HAS_GPU = _has_gpu()


def pytest_collection_modifyitems(config, items):
    if HAS_GPU:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


GOLDEN = ROOT / "tests" / "golden"
GOLDEN_CASES = sorted(p.stem for p in GOLDEN.glob("*.npz"))


class Golden:
    """A fixture made by tests/golden/make_golden.py from the reference."""

    def __init__(self, name: str):
        import numpy as np

        from paper_2205_09707_b200 import SearchParams
        from paper_2205_09707_b200.hostindex import HostIndex

        z = np.load(GOLDEN / f"{name}.npz")
        self.name = name
        self.z = z
        self.index = HostIndex(int(z["dim"]), int(z["nbits"]), z["centroids"], z["codes"], z["residuals"],
                               z["doclens"], z["ivf_offsets"], z["ivf_postings"], z["bucket_cutoffs"],
                               z["bucket_weights"])
        self.queries = z["queries"]
        self.params = [SearchParams(int(k), int(n), float(t), int(d))
                       for (k, n, d), t in zip(z["params"], z["params_tcs"])]
        self.trace_fields = [str(f) for f in z["trace_fields"]]

    def expected(self, qi: int, pi: int):
        z = self.z
        tr = dict(zip(self.trace_fields, (int(x) for x in z[f"trace_{qi}_{pi}"])))
        return z[f"ids_{qi}_{pi}"], z[f"scorebits_{qi}_{pi}"], tr


@pytest.fixture(scope="session", params=GOLDEN_CASES)
def golden(request):
    return Golden(request.param)


@pytest.fixture(scope="session")
def port():
    import oracle

    return oracle.get("port")


@pytest.fixture(scope="session")
def ref():
    import oracle

    if not oracle.available("ref"):
        pytest.skip("oracle/_ref not built (reference sources absent when building)")
    return oracle.get("ref")
