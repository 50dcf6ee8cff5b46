"""bench.py --impl reference runs the unmodified reference (oracle/_ref) on
inputs from the checker-side generator: the process maps no library of the
product package (paper_2205_09707_b200/_lib)."""
import json
import subprocess
import sys

import pytest

import oracle

from .conftest import ROOT


@pytest.mark.skipif(not oracle.available("ref"), reason="oracle/_ref not built")
def test_reference_arm_maps_only_oracle_libs():
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--config", "cfg1",
                        "--steps", "2", "--warmup", "1"], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0
    libs = line["repo_libs_mapped"]
    assert any(x.startswith("oracle/_ref/liblir_ref") for x in libs)
    assert not [x for x in libs if x.startswith("paper_2205_09707_b200")], libs
    assert line["cpu_baseline"]["kind"] == "reference" and line["cpu_baseline"]["cores"] >= 1
