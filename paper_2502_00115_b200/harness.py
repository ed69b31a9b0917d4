"""Batched registration with accuracy evaluation.

The registration loop of gridreg.harness.run_batch / _run_one
(harness.py:118-162) on the GPU: every pair goes through dses_batch (plan
construction of pair k+1 overlapping the search of pair k), then the winner
moves the source (numpy, geometry.py:209-211), the symmetric chamfer distance
is evaluated by the GPU's exact binary64 nearest-neighbour kernel, and
evaluate_pose compares with the ground truth.  Records and the summary follow
the reference's TrialRecord / BatchSummary (harness.py:64-116); engine
failures become failed rows ("engine:<ExceptionName>") without aborting.

The reference's synthetic instance generator (benchgen) is out of scope: the
caller passes the pairs (e.g. paper_2502_00115_b200.synth.make_pair).
"""
from __future__ import annotations

import statistics
from dataclasses import dataclass

import numpy as np

from .engines import SearchConfig, dses, dses_batch
from .errors import GridregError, InvalidInputError
from .metrics import EvalReport, chamfer_distance, evaluate_pose


@dataclass(frozen=True)
class TrialRecord:
    trial: int
    status: str
    eval: EvalReport | None
    inliers: int | None
    candidates_refined: int | None
    phase1_ms: float | None
    refine_ms: float | None
    total_ms: float | None


@dataclass(frozen=True)
class BatchSummary:
    n_trials: int
    n_failed: int
    mean_mie_r: float | None
    mean_mie_t: float | None
    mean_mae_r: float | None
    mean_mae_t: float | None
    recall: float
    mean_total_ms: float | None
    median_total_ms: float | None


def _summarize(records) -> BatchSummary:
    ok = [r for r in records if r.status == "ok"]
    hits = sum(1 for r in ok if r.eval.is_recall_hit)

    def mean(vals):
        vals = list(vals)
        return float(np.mean(vals)) if vals else None

    return BatchSummary(
        n_trials=len(records), n_failed=len(records) - len(ok),
        mean_mie_r=mean(r.eval.mie_r for r in ok), mean_mie_t=mean(r.eval.mie_t for r in ok),
        mean_mae_r=mean(r.eval.mae_r for r in ok), mean_mae_t=mean(r.eval.mae_t for r in ok),
        recall=hits / len(records) if records else 0.0,
        mean_total_ms=mean(r.total_ms for r in ok),
        median_total_ms=float(statistics.median(r.total_ms for r in ok)) if ok else None)


def _record(k, res, source, reference, truth, rot_tol_deg, trans_tol, device):
    moved = res.best.apply(source)
    rep = evaluate_pose(res.best, truth, rot_tol_deg, trans_tol,
                        chamfer=chamfer_distance(moved, reference, device))
    return TrialRecord(trial=k, status="ok", eval=rep, inliers=res.best_inliers,
                       candidates_refined=res.candidates_refined,
                       phase1_ms=res.elapsed["phase1"] * 1e3, refine_ms=res.elapsed["refine"] * 1e3,
                       total_ms=res.elapsed["total"] * 1e3)


def register_batch(sources, references, truths, cfg: SearchConfig, rot_tol_deg: float = 1.0,
                   trans_tol: float = 0.1, device: int = 0):
    """Register every (source, reference) pair and evaluate against the
    aligning ground truth (RigidTransform).  Returns (BatchSummary, records)."""
    sources, references, truths = list(sources), list(references), list(truths)
    if not sources or not (len(sources) == len(references) == len(truths)):
        raise InvalidInputError("need equally many (>= 1) sources, references and truths")
    records = []
    try:
        results = dses_batch(sources, references, cfg, device)
    except GridregError:
        results = None  # some pair failed: fall back to per-pair calls to record it
    for k in range(len(sources)):
        try:
            res = results[k] if results is not None else dses(sources[k], references[k], cfg, device)
        except GridregError as exc:
            records.append(TrialRecord(trial=k, status=f"engine:{type(exc).__name__}", eval=None,
                                       inliers=None, candidates_refined=None, phase1_ms=None,
                                       refine_ms=None, total_ms=None))
            continue
        records.append(_record(k, res, sources[k], references[k], truths[k], rot_tol_deg,
                               trans_tol, device))
    return _summarize(records), records
