"""IR metrics of the reference's cli-bench module (/root/reference/SPEC.md
`compute_metrics`, §6.2 "MRR@10 and Recall@100"; Success@5 for LoTTE-style
evaluation).  Host-side reporting on search results; not on the GPU path.

* results: mapping query id -> ranked passage ids (rank 1 first)
* qrels:   mapping query id -> set of relevant passage ids (binary relevance)

MRR@k     mean over queries of 1 / rank of the first relevant id within the
          top k (0 if none)
Recall@k  mean over queries of |relevant ∩ top-k| / |relevant|
Success@k fraction of queries with at least one relevant id in the top k

Errors follow the reference (error.hpp): a result query id absent from the
qrels is UnknownQueryId; a query with no relevant passages contributes 0 to
recall (|relevant| = 0 has no recall to measure).
"""
from __future__ import annotations

from typing import Iterable, Mapping, Sequence

from .api import ErrorCode, PlaidError


def _check(results: Mapping[int, Sequence[int]], qrels: Mapping[int, Iterable[int]]) -> None:
    for qid in results:
        if qid not in qrels:
            raise PlaidError(ErrorCode.UnknownQueryId, f"query id {qid} has no qrels entry")


def mrr_at(results: Mapping[int, Sequence[int]], qrels: Mapping[int, Iterable[int]], k: int = 10) -> float:
    _check(results, qrels)
    if not results:
        return 0.0
    total = 0.0
    for qid, ranked in results.items():
        rel = set(qrels[qid])
        for r, pid in enumerate(list(ranked)[:k], start=1):
            if pid in rel:
                total += 1.0 / r
                break
    return total / len(results)


def recall_at(results: Mapping[int, Sequence[int]], qrels: Mapping[int, Iterable[int]], k: int = 100) -> float:
    _check(results, qrels)
    if not results:
        return 0.0
    total = 0.0
    for qid, ranked in results.items():
        rel = set(qrels[qid])
        if rel:
            total += len(rel & set(list(ranked)[:k])) / len(rel)
    return total / len(results)


def success_at(results: Mapping[int, Sequence[int]], qrels: Mapping[int, Iterable[int]], k: int = 5) -> float:
    _check(results, qrels)
    if not results:
        return 0.0
    hit = sum(1 for qid, ranked in results.items() if set(qrels[qid]) & set(list(ranked)[:k]))
    return hit / len(results)


def compute_metrics(results, qrels, cuts=(10, 100)) -> dict:
    """The metric report of `compute_metrics`: MRR@10, Recall@k per cut, Success@5."""
    out = {"queries": len(results), "MRR@10": mrr_at(results, qrels, 10), "Success@5": success_at(results, qrels, 5)}
    for c in cuts:
        out[f"Recall@{c}"] = recall_at(results, qrels, c)
    return out


def read_results_tsv(path) -> dict:
    """TSV rows query_id, rank (1-based), passage_id, score -> {qid: [pids by rank]}."""
    rows: dict = {}
    with open(path) as f:
        for line in f:
            if not line.strip():
                continue
            qid, rank, pid, _ = line.rstrip("\n").split("\t")
            rows.setdefault(int(qid), []).append((int(rank), int(pid)))
    return {q: [p for _, p in sorted(v)] for q, v in rows.items()}


def read_qrels_tsv(path) -> dict:
    """TSV rows query_id, passage_id (relevant pairs; TREC 4-column qrels with
    a positive relevance in the last column are accepted too)."""
    q: dict = {}
    with open(path) as f:
        for line in f:
            parts = line.split()
            if not parts:
                continue
            if len(parts) >= 4:
                if int(parts[3]) <= 0:
                    continue
                qid, pid = int(parts[0]), int(parts[2])
            else:
                qid, pid = int(parts[0]), int(parts[1])
            q.setdefault(qid, set()).add(pid)
    return q
