"""north_star comparator for the TENSOR score path — TEST INFRASTRUCTURE ONLY.

The production path computes S_cq on tcgen05 (3xTF32, |S - S_exact| < ~5e-6)
and stage-4 MaxSim on tcgen05 (split-bf16 residual products), so its results
are not bit-identical to `lir::search` (/root/reference/proj/src/pipeline.cpp:
232-283).  BASELINE.json's north_star states what must still hold:

  * integer work bit-exact — IVF candidate sets and pruned-centroid sets —
    except where a score lies within the fp32 tolerance of the t_cs or the
    top-nprobe / top-ndocs / top-k boundary;
  * MaxSim scores within 1e-4 relative;
  * top-k pids equal except for near-ties.

`check_tensor_search` classifies every difference between a GPU TENSOR
result and the reference on the same index and query, stage by stage:

  stage 1  per-token top-nprobe sets under S_tensor vs S_exact
           (pipeline.cpp:52-87): every centroid in the symmetric difference
           must have an exact score within `2 eps_s` of that token's
           nprobe-th exact score;
  prune    keep bits (pipeline.cpp:89-95): a flipped bit needs
           |max_i S_exact[c, i] - t_cs| <= eps_s;
  stage 2/3 top-ndocs / top-stage3_width sets (pipeline.cpp:97-163) of the
           oracle run on S_tensor vs on S_exact: a differing member needs its
           exact centroid-interaction score within `rows * 2 eps_s` of the
           boundary score;
  given S  the GPU's integer trace counters equal the oracle's stages run on
           S_tensor (the GPU consumes S_tensor exactly);
  stage 4  every returned score within `rel` of the exact MaxSim of that pid
           (maxsim.cpp:66-104 via rank_final, pipeline.cpp:165-225); the
           returned set equals the oracle's top-k on S_tensor except for pids
           whose exact scores lie within 2 rel of the k-th score.

Only tests/, smoke() and bench.py's --check leg use this module.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass
class Report:
    ok: bool = True
    s_max_abs_err: float = 0.0
    stage1_diff: int = 0            # centroids (token, c) selected by one side only (all near-boundary)
    keep_diff: int = 0              # keep bits flipped (all within eps of t_cs)
    stage2_diff: int = 0            # top-ndocs members differing (near-boundary)
    stage3_diff: int = 0
    final_diff: int = 0             # top-k pids differing (near-ties)
    max_rel_score_err: float = 0.0  # over the returned pids vs their exact MaxSim
    ids_equal_reference: bool = False
    problems: list = field(default_factory=list)

    def fail(self, msg: str) -> None:
        self.ok = False
        if len(self.problems) < 20:
            self.problems.append(msg)

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k in ("ok", "s_max_abs_err", "stage1_diff", "keep_diff", "stage2_diff",
                                              "stage3_diff", "final_diff", "max_rel_score_err",
                                              "ids_equal_reference", "problems")}


def topn_sets(S: np.ndarray, nprobe: int):
    """Per token i: the nprobe centroids of largest S[:, i], ties to the lower
    id (pipeline.cpp:65-73), and the nprobe-th score."""
    K, rows = S.shape
    sets, bounds = [], []
    ids = np.arange(K)
    for i in range(rows):
        col = S[:, i]
        if nprobe >= K:
            sel = ids
        else:
            # lexsort: primary -score, secondary id
            part = np.argpartition(-col, nprobe - 1)[: max(nprobe * 4, nprobe + 64)]
            thr = np.sort(col[part])[::-1][min(nprobe, part.size) - 1]
            cand = ids[col >= thr]
            order = np.lexsort((cand, -col[cand]))
            sel = cand[order[:nprobe]]
        sets.append(set(int(c) for c in sel))
        bounds.append(float(np.min(col[sel])))
    return sets, bounds


def compose(oracle, h, q, S, row_max, p, disable_filter=False):
    """The reference pipeline (pipeline.cpp:232-283) run by the oracle stage by
    stage on a given centroid-score table S; returns every intermediate set."""
    c1 = oracle.generate_candidates(h, S, p.nprobe)
    out = {"c1": c1}
    if c1.size == 0:
        out.update(k2=c1, k3=c1, s2=np.zeros(0, np.float32), s3=np.zeros(0, np.float32), ids=c1,
                   scores=np.zeros(0, np.float32), r2=0, r3=0)
        return out
    if disable_filter:
        k2 = k3 = c1
        r2 = r3 = 0
        s2 = s3 = None
    else:
        keep = oracle.prune_centroids(row_max, p.t_cs)
        s2, r2 = oracle.centroid_interaction(h, c1, S, keep)
        k2, _ = oracle.select_top(c1, s2, p.ndocs)
        s3, r3 = oracle.centroid_interaction(h, k2, S, None)
        w = max((int(p.ndocs) + 3) // 4, int(p.k))
        k3, _ = oracle.select_top(k2, s3, w)
    ids, sc = oracle.rank_final(h, k3, q, p.k)
    out.update(k2=k2, k3=k3, s2=s2, s3=s3, ids=ids, scores=sc, r2=r2, r3=r3)
    return out


def _counters(c: dict, disable_filter: bool) -> dict:
    n1 = len(c["c1"])
    if n1 == 0:
        return dict(stage1_candidates=0, stage2_out=0, stage3_out=0, final_out=0, centroid_matmul_count=1,
                    stage2_rows_gathered=0, stage3_rows_gathered=0, decompressed_passages=0)
    return dict(stage1_candidates=n1, stage2_out=len(c["k2"]), stage3_out=len(c["k3"]), final_out=len(c["ids"]),
                centroid_matmul_count=1, stage2_rows_gathered=c["r2"], stage3_rows_gathered=c["r3"],
                decompressed_passages=len(c["k3"]))


def _set_diff_near_boundary(rep, what, a, b, exact_score_of, boundary, tol):
    """Members of a XOR b must have exact scores within tol of the boundary."""
    diff = set(int(x) for x in a) ^ set(int(x) for x in b)
    for pid in diff:
        s = exact_score_of(pid)
        if abs(s - boundary) > tol:
            rep.fail(f"{what}: pid {pid} differs with exact score {s:.7g}, boundary {boundary:.7g} (tol {tol:.2g})")
    return len(diff)


def check_tensor_search(oracle, h, q, p, got_ids, got_scores, S_t, got_counters=None, disable_filter=False,
                        eps_s=5e-6, rel=1e-4) -> Report:
    """Classify a TENSOR-mode GPU result against the reference (see module doc).

    oracle   the CPU oracle ("ref" = the compiled reference, or "port")
    S_t      the GPU's S_cq for this query (K x rows, Searcher.compute_centroid_scores in TENSOR mode)
    """
    rep = Report()
    q = np.ascontiguousarray(q, dtype=np.float32)
    rows = q.shape[0]
    got_ids = np.asarray(got_ids, dtype=np.uint32)
    got_scores = np.asarray(got_scores, dtype=np.float32)
    S0, mx0 = oracle.compute_centroid_scores(h, q)
    S_t = np.ascontiguousarray(S_t, dtype=np.float32)
    mx_t = S_t.max(axis=1)
    rep.s_max_abs_err = float(np.abs(S_t - S0).max())
    if rep.s_max_abs_err > eps_s:
        rep.fail(f"S_cq error {rep.s_max_abs_err:.3g} above {eps_s:g}")

    # stage 1: top-nprobe sets
    sets0, b0 = topn_sets(S0, int(p.nprobe))
    sets_t, _ = topn_sets(S_t, int(p.nprobe))
    for i in range(rows):
        for c in sets0[i] ^ sets_t[i]:
            rep.stage1_diff += 1
            if abs(float(S0[c, i]) - b0[i]) > 2 * eps_s:
                rep.fail(f"stage 1: token {i} centroid {c} S={S0[c, i]:.7g} far from boundary {b0[i]:.7g}")
    # prune: keep bits
    if not disable_filter:
        k0 = mx0 >= np.float32(p.t_cs)
        kt = mx_t >= np.float32(p.t_cs)
        for c in np.nonzero(k0 != kt)[0]:
            rep.keep_diff += 1
            if abs(float(mx0[c]) - float(p.t_cs)) > eps_s:
                rep.fail(f"prune: centroid {c} row max {mx0[c]:.7g} far from t_cs {p.t_cs}")

    ref = compose(oracle, h, q, S0, mx0, p, disable_filter)
    ten = compose(oracle, h, q, S_t, mx_t, p, disable_filter)
    if got_counters is not None:
        exp = _counters(ten, disable_filter)
        for kk, v in exp.items():
            if kk in got_counters and int(got_counters[kk]) != int(v):
                rep.fail(f"trace {kk}: GPU {got_counters.get(kk)} vs oracle-on-S_tensor {v}")
    # stages 2 and 3, where stage 1 agreed: differences only at the cut
    if not disable_filter and np.array_equal(ref["c1"], ten["c1"]) and len(ref["c1"]):
        tol_ci = rows * 2 * eps_s + 1e-5
        ex2 = dict(zip((int(x) for x in ref["c1"]), (float(x) for x in ref["s2"])))
        bnd2 = min(ex2[int(x)] for x in ref["k2"]) if len(ref["k2"]) else 0.0
        if len(ref["k2"]) == int(p.ndocs):
            rep.stage2_diff = _set_diff_near_boundary(rep, "stage 2", ref["k2"], ten["k2"], lambda x: ex2[x], bnd2,
                                                      tol_ci)
        elif set(map(int, ref["k2"])) != set(map(int, ten["k2"])):
            rep.fail("stage 2: sets differ below the ndocs cap")
        if set(map(int, ref["k2"])) == set(map(int, ten["k2"])):
            ex3 = dict(zip((int(x) for x in ref["k2"]), (float(x) for x in ref["s3"])))
            w = max((int(p.ndocs) + 3) // 4, int(p.k))
            if len(ref["k3"]) == w:
                bnd3 = min(ex3[int(x)] for x in ref["k3"])
                rep.stage3_diff = _set_diff_near_boundary(rep, "stage 3", ref["k3"], ten["k3"], lambda x: ex3[x],
                                                          bnd3, tol_ci)
            elif set(map(int, ref["k3"])) != set(map(int, ten["k3"])):
                rep.fail("stage 3: sets differ below the stage-3 width")

    # stage 4: scores within rel of the exact MaxSim of the same pid
    if got_ids.size:
        ex_ids, ex_sc = oracle.rank_final(h, got_ids, q, got_ids.size)
        exact = dict(zip((int(x) for x in ex_ids), (float(x) for x in ex_sc)))
        errs = [abs(float(s) - exact[int(i)]) / max(abs(exact[int(i)]), 1e-6) for i, s in zip(got_ids, got_scores)]
        rep.max_rel_score_err = float(max(errs))
        if rep.max_rel_score_err > rel:
            rep.fail(f"stage 4: MaxSim relative error {rep.max_rel_score_err:.3g} above {rel:g}")
        # ordering: descending score, ties by pid
        for a in range(got_ids.size - 1):
            if got_scores[a] < got_scores[a + 1] or (got_scores[a] == got_scores[a + 1]
                                                     and got_ids[a] > got_ids[a + 1]):
                rep.fail(f"stage 4: output not sorted at {a}")
                break
    # final set vs the oracle's top-k over the same finalists (S_tensor stages)
    if len(ten["ids"]) != got_ids.size:
        rep.fail(f"final: {got_ids.size} results vs {len(ten['ids'])}")
    elif got_ids.size:
        fin_ids, fin_sc = oracle.rank_final(h, ten["k3"], q, len(ten["k3"]))
        exact_fin = dict(zip((int(x) for x in fin_ids), (float(x) for x in fin_sc)))
        kth = float(ten["scores"][-1])
        if len(ten["k3"]) > int(p.k):
            rep.final_diff = _set_diff_near_boundary(rep, "final", ten["ids"], got_ids,
                                                     lambda x: exact_fin.get(x, float("nan")), kth,
                                                     2 * rel * max(abs(kth), 1e-6))
        elif set(map(int, ten["ids"])) != set(map(int, got_ids)):
            rep.fail("final: sets differ although every finalist is returned")
    rep.ids_equal_reference = bool(np.array_equal(got_ids, ref["ids"]))
    return rep
