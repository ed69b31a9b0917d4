"""Batched registration with accuracy evaluation.

The registration loop of gridreg.harness.run_batch / _run_one
(harness.py:118-162) on the GPU: every pair goes through dses_batch (plan
construction of pair k+1 overlapping the search of pair k), then the winner
moves the source (numpy, geometry.py:209-211), the symmetric chamfer distance
is evaluated by the GPU's exact binary64 nearest-neighbour kernel, and
evaluate_pose compares with the ground truth.  Records and the summary follow
the reference's TrialRecord / BatchSummary (harness.py:64-116); engine
failures become failed rows ("engine:<ExceptionName>") without aborting.

Trials can be sharded over ranks (one process per GPU, trial k on rank
k mod world, records gathered on every rank).  Results are written with the
reference's versioned, byte-stable CSV schema and its JSON mirror
(harness.py:55-62, 468-534); search configs round-trip through the same JSON
keys (search_to_dict / search_from_json, harness.py:545-616).

The reference's synthetic instance generator (benchgen) is out of scope: the
caller passes the pairs (e.g. paper_2502_00115_b200.synth.make_pair).
"""
from __future__ import annotations

import csv
import io
import json
import math
import statistics
from dataclasses import asdict, dataclass, is_dataclass

import numpy as np

from .engines import SearchConfig, dses, dses_batch
from .errors import GridregError, InvalidInputError
from .geometry import RigidTransform
from .metrics import ErrorMetric, EvalReport, chamfer_distance, evaluate_pose

CSV_SCHEMA = "gridreg-batch-csv v1"
JSON_SCHEMA = "gridreg-batch-json v1"
CSV_FIELDS = ("trial", "seed", "shape", "status", "mie_r_deg", "mie_t_m", "mae_r_deg",
              "mae_t_m", "recall_hit", "chamfer_m", "inliers", "candidates_refined")


@dataclass(frozen=True)
class TrialRecord:
    """One registration trial (harness.py:64-77); metric fields are None when
    the engine failed and `status` carries "engine:<ExceptionName>"."""
    trial: int
    seed: int
    shape: str
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


def _record(k, seed, shape, res, source, reference, truth, rot_tol_deg, trans_tol, device):
    moved = res.best.apply(source)
    rep = evaluate_pose(res.best, truth, rot_tol_deg, trans_tol,
                        chamfer=chamfer_distance(moved, reference, device))
    return TrialRecord(trial=k, seed=seed, shape=shape, status="ok", eval=rep,
                       inliers=res.best_inliers,
                       candidates_refined=res.candidates_refined,
                       phase1_ms=res.elapsed["phase1"] * 1e3, refine_ms=res.elapsed["refine"] * 1e3,
                       total_ms=res.elapsed["total"] * 1e3)


def _failed(k, seed, shape, exc):
    return TrialRecord(trial=k, seed=seed, shape=shape, status=f"engine:{type(exc).__name__}",
                       eval=None, inliers=None, candidates_refined=None, phase1_ms=None,
                       refine_ms=None, total_ms=None)


def register_batch(sources, references, truths, cfg: SearchConfig, rot_tol_deg: float = 1.0,
                   trans_tol: float = 0.1, device: int = 0, seeds=None, shapes=None,
                   group=None):
    """Register every (source, reference) pair and evaluate against the
    aligning ground truth (RigidTransform).  Returns (BatchSummary, records).

    seeds / shapes label the records (default: the trial index / "synthetic").
    With a torch.distributed process group of size > 1 (`group`, or the default
    group when one is initialised) rank r registers trials r, r + world, ...
    on its own GPU and the records are gathered so every rank returns the whole
    batch (weak scaling, no data-path collective)."""
    sources, references, truths = list(sources), list(references), list(truths)
    if not sources or not (len(sources) == len(references) == len(truths)):
        raise InvalidInputError("need equally many (>= 1) sources, references and truths")
    n = len(sources)
    seeds = list(range(n)) if seeds is None else [int(v) for v in seeds]
    shapes = ["synthetic"] * n if shapes is None else [str(v) for v in shapes]
    if len(seeds) != n or len(shapes) != n:
        raise InvalidInputError("seeds / shapes must label every trial")
    rank, world = 0, 1
    try:
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized():
            rank, world = dist.get_rank(group), dist.get_world_size(group)
    except ImportError:  # pragma: no cover - torch is part of the image
        dist = None
    mine = list(range(rank, n, world))
    records = []
    try:
        results = dses_batch([sources[k] for k in mine], [references[k] for k in mine], cfg, device)
    except GridregError:
        results = None  # some pair failed: fall back to per-pair calls to record it
    for q, k in enumerate(mine):
        try:
            res = results[q] if results is not None else dses(sources[k], references[k], cfg, device)
        except GridregError as exc:
            records.append(_failed(k, seeds[k], shapes[k], exc))
            continue
        records.append(_record(k, seeds[k], shapes[k], res, sources[k], references[k], truths[k],
                               rot_tol_deg, trans_tol, device))
    if world > 1:
        parts = [None] * world
        dist.all_gather_object(parts, records, group=group)
        records = sorted((r for part in parts for r in part), key=lambda r: r.trial)
    return _summarize(records), records


def _fmt(v):
    """harness.py:468-475: None -> "", bool -> 0/1, float -> shortest repr."""
    if v is None:
        return ""
    if isinstance(v, (bool, np.bool_)):
        return "1" if v else "0"
    if isinstance(v, (float, np.floating)):
        return repr(float(v))
    return str(v)


def record_row(r: TrialRecord) -> dict:
    e = r.eval
    return {
        "trial": r.trial, "seed": r.seed, "shape": r.shape, "status": r.status,
        "mie_r_deg": None if e is None else e.mie_r,
        "mie_t_m": None if e is None else e.mie_t,
        "mae_r_deg": None if e is None else e.mae_r,
        "mae_t_m": None if e is None else e.mae_t,
        "recall_hit": None if e is None else e.is_recall_hit,
        "chamfer_m": None if e is None else e.chamfer,
        "inliers": r.inliers, "candidates_refined": r.candidates_refined,
    }


def write_batch_csv(path, records) -> None:
    """Byte-stable versioned CSV (no wall-clock columns), the reference's
    schema line, header and formatting (harness.py:496-506)."""
    buf = io.StringIO()
    buf.write(f"# {CSV_SCHEMA}\n")
    w = csv.DictWriter(buf, fieldnames=list(CSV_FIELDS), lineterminator="\n")
    w.writeheader()
    for r in records:
        w.writerow({k: _fmt(v) for k, v in record_row(r).items()})
    with open(path, "w", encoding="utf-8", newline="") as fh:
        fh.write(buf.getvalue())


def write_batch_json(path, scenario, search: SearchConfig, summary: BatchSummary, records,
                     extra=None) -> None:
    """JSON mirror of the CSV plus summary, config echo and timings
    (harness.py:509-533).  `scenario` is a dataclass or a dict describing
    where the pairs came from."""
    payload = {
        "schema": JSON_SCHEMA,
        "scenario": asdict(scenario) if is_dataclass(scenario) else dict(scenario),
        "search": search_to_dict(search),
        "summary": asdict(summary),
        "records": [dict(record_row(r), phase1_ms=r.phase1_ms, refine_ms=r.refine_ms,
                         total_ms=r.total_ms) for r in records],
    }
    if extra:
        payload.update(extra)
    with open(path, "w", encoding="utf-8") as fh:
        json.dump(payload, fh, indent=2, sort_keys=True)
        fh.write("\n")


def search_to_dict(cfg: SearchConfig) -> dict:
    """harness.py:545-562: the search config as JSON-ready values (degrees)."""
    d = {"k_rot": cfg.k_rot, "rot_step_deg": math.degrees(cfg.rot_step), "k_trans": cfg.k_trans,
         "trans_bin": cfg.trans_bin, "q": cfg.q, "metric": cfg.metric.kind,
         "metric_param": cfg.metric.param, "pose_cap": cfg.pose_cap}
    if cfg.center is not None:
        d["center"] = {"rotation": [[float(v) for v in row] for row in cfg.center.rotation],
                       "translation": [float(v) for v in cfg.center.translation]}
    return d


_METRIC_ALIASES = {"l2": "l2", "l1": "l1", "trunc-l1": "trunc-l1", "trunc_l1": "trunc-l1",
                   "inliers": "inliers", "sat-l0": "inliers", "sat_l0": "inliers"}
_SEARCH_KEYS = {"k_rot", "rot_step_deg", "rot_range_deg", "k_trans", "trans_bin", "trans_range",
                "q", "metric", "trunc", "metric_param", "center", "pose_cap"}


def search_from_dict(raw: dict) -> SearchConfig:
    """harness.search_from_json's rules (harness.py:569-616): (k_rot |
    rot_range_deg) + rot_step_deg, (k_trans | trans_range) + trans_bin,
    optional q, metric, trunc / metric_param, center, pose_cap; unknown keys
    and missing ones raise InvalidInputError."""
    from .cli import grid_half_width
    extra = set(raw) - _SEARCH_KEYS
    if extra:
        raise InvalidInputError(f"unknown search-config keys: {sorted(extra)}")
    for key in ("rot_step_deg", "trans_bin"):
        if key not in raw:
            raise InvalidInputError(f"search config requires {key}")
    rot_step = math.radians(float(raw["rot_step_deg"]))
    trans_bin = float(raw["trans_bin"])
    if "k_rot" in raw:
        k_rot = int(raw["k_rot"])
    elif "rot_range_deg" in raw:
        k_rot = grid_half_width(math.radians(float(raw["rot_range_deg"])), rot_step)
    else:
        raise InvalidInputError("search config requires k_rot or rot_range_deg")
    if "k_trans" in raw:
        k_trans = int(raw["k_trans"])
    elif "trans_range" in raw:
        k_trans = grid_half_width(float(raw["trans_range"]), trans_bin)
    else:
        raise InvalidInputError("search config requires k_trans or trans_range")
    name = _METRIC_ALIASES.get(str(raw.get("metric", "trunc-l1")).lower())
    if name is None:
        raise InvalidInputError(f"unknown metric {raw.get('metric')!r}")
    tau = raw.get("trunc", raw.get("metric_param"))
    metric = ErrorMetric.from_name(name, trans_bin, None if tau is None else float(tau))
    center = None
    if raw.get("center") is not None:
        center = RigidTransform(np.array(raw["center"]["rotation"], dtype=np.float64),
                                np.array(raw["center"]["translation"], dtype=np.float64))
    return SearchConfig(k_rot=k_rot, rot_step=rot_step, k_trans=k_trans, trans_bin=trans_bin,
                        q=float(raw.get("q", 0.5)), metric=metric, center=center,
                        pose_cap=int(raw.get("pose_cap", 100_000_000)))


def search_from_json(path) -> SearchConfig:
    with open(path, "r", encoding="utf-8") as fh:
        return search_from_dict(json.load(fh))
