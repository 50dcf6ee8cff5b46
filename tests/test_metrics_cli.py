"""IR metrics (SPEC.md cli-bench compute_metrics, acceptance #10) against an
independently written naive evaluator on random fixtures, the hand-computed
examples, the TSV formats and the CLI's metrics command (CPU); the CLI's
index -> search -> metrics path on the GPU."""
import json
import subprocess
import sys

import numpy as np
import pytest

import paper_2205_09707_b200 as P
from paper_2205_09707_b200 import metrics as M

from .conftest import ROOT


def naive(results, qrels, k_mrr=10, k_rec=100, k_succ=5):
    mrr = rec = succ = 0.0
    for q in results:
        ranked = list(results[q])
        rel = qrels[q]
        rr = 0.0
        for i in range(min(k_mrr, len(ranked))):
            if ranked[i] in rel:
                rr = 1.0 / (i + 1)
                break
        mrr += rr
        if len(rel) > 0:
            rec += sum(1 for p in ranked[:k_rec] if p in rel) / len(rel)
        succ += 1.0 if any(p in rel for p in ranked[:k_succ]) else 0.0
    n = len(results)
    return mrr / n, rec / n, succ / n


def test_metrics_vs_naive_random_fixtures():
    rng = np.random.default_rng(0)
    for _ in range(100):
        nq = int(rng.integers(1, 12))
        results, qrels = {}, {}
        for q in range(nq):
            results[q] = list(rng.permutation(300)[: int(rng.integers(0, 150))])
            qrels[q] = set(rng.integers(0, 300, int(rng.integers(0, 6))).tolist())
        a = M.compute_metrics(results, qrels, cuts=(100,))
        b = naive(results, qrels)
        assert abs(a["MRR@10"] - b[0]) < 1e-9 and abs(a["Recall@100"] - b[1]) < 1e-9
        assert abs(a["Success@5"] - b[2]) < 1e-9


def test_metrics_examples_and_errors():
    assert M.mrr_at({0: [5, 6]}, {0: {5}}) == 1.0
    assert M.mrr_at({0: [4, 5]}, {0: {5}}) == 0.5
    # hand-built 3-query fixture: rr = 1, 1/3, 0; recall@2 = 1/2, 0, 0; success@5 = 1, 1, 0
    res = {0: [1, 2, 3], 1: [7, 8, 9, 10], 2: [20, 21]}
    qr = {0: {1, 4}, 1: {9}, 2: {99}}
    assert M.mrr_at(res, qr) == pytest.approx((1 + 1 / 3) / 3)
    assert M.recall_at(res, qr, 2) == pytest.approx(0.5 / 3)
    assert M.success_at(res, qr, 5) == pytest.approx(2 / 3)
    with pytest.raises(P.PlaidError) as e:
        M.mrr_at({0: [1], 5: [2]}, {0: {1}})
    assert e.value.code == P.ErrorCode.UnknownQueryId


def test_cli_metrics(tmp_path):
    (tmp_path / "r.tsv").write_text("0\t1\t5\t9.500000\n0\t2\t6\t8.000000\n1\t1\t7\t3.000000\n1\t2\t8\t2.000000\n")
    (tmp_path / "q.tsv").write_text("0 6\n1 0 8 1\n")  # a 2-column row and a TREC 4-column row
    r = subprocess.run([sys.executable, "-m", "paper_2205_09707_b200.cli", "metrics", "--results",
                        str(tmp_path / "r.tsv"), "--qrels", str(tmp_path / "q.tsv")], capture_output=True, text=True,
                       cwd=ROOT)
    assert r.returncode == 0, r.stderr
    rep = json.loads(r.stdout)
    assert rep["MRR@10"] == pytest.approx(0.5) and rep["Recall@10"] == pytest.approx(1.0)


@pytest.mark.gpu
def test_cli_index_search_metrics(tmp_path):
    """index (GPU build) -> search -> metrics on a toy corpus whose queries are
    perturbed copies of passages: each query's source passage ranks first."""
    rng = np.random.default_rng(1)
    n, dim = 300, 128
    dl = rng.integers(8, 20, n).astype(np.uint32)
    x = rng.standard_normal((int(dl.sum()), dim)).astype(np.float32)
    x /= np.linalg.norm(x, axis=1, keepdims=True)
    np.save(tmp_path / "e.npy", x)
    np.save(tmp_path / "l.npy", dl)
    off = np.concatenate([[0], np.cumsum(dl.astype(np.int64))])
    src = [3, 77, 150]
    qs = []
    for p in src:
        t = x[off[p]:off[p] + 8]
        q = t + 0.01 * rng.standard_normal(t.shape).astype(np.float32)
        qs.append(q / np.linalg.norm(q, axis=1, keepdims=True))
    np.save(tmp_path / "q.npy", np.stack(qs).astype(np.float32))
    (tmp_path / "qrels.tsv").write_text("".join(f"{i} {p}\n" for i, p in enumerate(src)))
    cli = [sys.executable, "-m", "paper_2205_09707_b200.cli"]
    r = subprocess.run(cli + ["index", "--embeddings", str(tmp_path / "e.npy"), "--doclens", str(tmp_path / "l.npy"),
                              "--nbits", "2", "--centroids", "32", "--iters", "4", "--out", str(tmp_path / "ix")],
                       capture_output=True, text=True, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    for mode in ("tensor", "exact"):
        r = subprocess.run(cli + ["search", "--index", str(tmp_path / "ix"), "--queries", str(tmp_path / "q.npy"),
                                  "--k", "10", "--score-mode", mode, "--out", str(tmp_path / f"r_{mode}.tsv")],
                           capture_output=True, text=True, cwd=ROOT)
        assert r.returncode == 0, r.stderr
        r = subprocess.run(cli + ["metrics", "--results", str(tmp_path / f"r_{mode}.tsv"), "--qrels",
                                  str(tmp_path / "qrels.tsv")], capture_output=True, text=True, cwd=ROOT)
        rep = json.loads(r.stdout)
        assert rep["MRR@10"] == 1.0 and rep["Success@5"] == 1.0
    r = subprocess.run(cli + ["bench", "--index", str(tmp_path / "ix"), "--queries", str(tmp_path / "q.npy"),
                              "--k", "10", "--trials", "2"], capture_output=True, text=True, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    b = json.loads(r.stdout)
    assert b["total_ms"] > 0 and b["trials"] == 2
