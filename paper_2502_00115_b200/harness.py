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

run_oracle_checks is the reference's verification suite (harness.py:329-462,
`gridreg oracle-check`): planted-consensus instances where the histogram mode
must maximise the inlier count over a dense translation sweep (the sweep is
the GPU kernel dses_sweep_inlier_best), and small on-grid instances where
dses and exhaustive_search must agree on the inlier count.  The instance
generators make the reference's numpy RNG calls in the reference's order, so
the same seed yields the same instances.
"""
from __future__ import annotations

import csv
import io
import json
import math
import statistics
from dataclasses import asdict, dataclass, is_dataclass

import numpy as np

from .engines import SearchConfig, dses, dses_batch, exhaustive_search
from .errors import GridregError, InvalidInputError
from .geometry import RigidTransform, random_rotation, rotation_from_euler
from .metrics import ErrorMetric, EvalReport, chamfer_distance, count_inliers, evaluate_pose
from .mode_search import bin_center, mode_translation

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


# ---- verification suite (harness.py:329-462) ----

def _sample_separated(rng, n, sep, lo, hi):
    """harness.py:329-335: n points uniform in [lo, hi)^3, pairwise Chebyshev
    separation > sep, by rejection (same RNG draws as the reference)."""
    pts = []
    while len(pts) < n:
        p = rng.uniform(lo, hi, 3)
        if all(np.max(np.abs(p - q)) > sep for q in pts):
            pts.append(p)
    return np.array(pts)


def make_lemma_instance(rng: np.random.Generator, bin_size: float):
    """harness.py:338-372: planted-consensus instance (a cluster of m sources
    matched exactly at one translation, every other candidate difference at
    least 2.5 bins away, the true translation off bin boundaries), under which
    the histogram mode provably maximises the inlier count over ALL
    translations.  Returns (X, Y, R, m)."""
    b = bin_size
    for _ in range(500):
        n = int(rng.integers(4, 10))
        m_total = int(rng.integers(4, 10))
        m = int(rng.integers(2, min(n, m_total) + 1))
        x = _sample_separated(rng, n, 3 * b, -0.6, 0.6)
        rot = random_rotation(rng)
        t_true = rng.uniform(-0.4, 0.4, 3)
        ys = list(x[:m] @ rot.T + t_true)
        while len(ys) < m_total:
            p = rng.uniform(-0.6, 0.6, 3)
            if all(np.max(np.abs(p - q)) > 3 * b for q in ys):
                ys.append(p)
        y = np.array(ys)
        cand = (y[None, :, :] - (x @ rot.T)[:, None, :]).reshape(-1, 3)
        d = np.max(np.abs(cand[:, None, :] - cand[None, :, :]), axis=2)
        seps = d[np.triu_indices(cand.shape[0], 1)]
        if np.any((seps > 1e-9) & (seps <= 2.5 * b)):
            continue
        qf = t_true / b
        if np.any(np.abs(np.abs(qf - np.round(qf)) - 0.5) < 0.05):
            continue
        return x, y, rot, m
    raise GridregError("lemma-instance rejection sampling did not converge")


def make_theorem_instance(rng: np.random.Generator):
    """harness.py:375-402: small random instance with an on-grid planted pose;
    returns (X, Y, SearchConfig with the saturated-L0 metric at the bin)."""
    k_rot, k_trans, rot_step, bin_size = int(rng.integers(0, 2)), 2, 0.3, 0.1
    n = int(rng.integers(5, 13))
    m_total = int(rng.integers(5, 13))
    m = int(rng.integers(2, min(n, m_total) + 1))
    x = rng.uniform(-0.5, 0.5, (n, 3))
    idx_r = rng.integers(-k_rot, k_rot + 1, 3)
    idx_t = rng.integers(-k_trans, k_trans + 1, 3)
    node = RigidTransform(rotation_from_euler(idx_r.astype(np.float64) * rot_step),
                          bin_center(idx_t, bin_size))
    ys = list(node.apply(x[:m]))
    while len(ys) < m_total:
        ys.append(rng.uniform(-0.8, 0.8, 3))
    cfg = SearchConfig(k_rot=k_rot, rot_step=rot_step, k_trans=k_trans, trans_bin=bin_size,
                       q=0.5, metric=ErrorMetric.saturated_l0(bin_size))
    return x, np.array(ys), cfg


def sweep_inlier_best(cands, n: int, m: int, half: float, t0vals, t1vals, t2vals,
                      device: int = 0) -> int:
    """_kernels.sweep_inlier_best (_kernels.py:384-410) on the GPU: the maximum
    over the lattice t0 x t1 x t2 of the number of sources with some
    difference (row i*m + j of `cands`) inside the open Chebyshev ball of
    radius `half` around t.  Bit-identical counts (binary64 compares)."""
    from . import _native
    return _native.sweep_inlier_best(cands, n, m, half, t0vals, t1vals, t2vals, device)


@dataclass(frozen=True)
class OracleReport:
    """harness.py:405-415."""
    lemma_trials: int
    lemma_violations: int
    theorem_trials: int
    theorem_violations: int
    details: list

    @property
    def ok(self) -> bool:
        return self.lemma_violations == 0 and self.theorem_violations == 0


def run_oracle_checks(n_lemma: int = 25, n_theorem: int = 10, seed: int = 0,
                      device: int = 0) -> OracleReport:
    """harness.py:418-462: the mode-optimality sweep check (n_lemma planted
    instances: the inlier count at mode_translation's t* must not be beaten by
    a sweep at bin/4 spacing) and the engine inlier-equality check (n_theorem
    instances: dses and exhaustive_search report the same best_inliers)."""
    details = []
    rng = np.random.default_rng(np.random.SeedSequence([0x0AC1E, seed]))
    bin_size = 0.05
    lemma_bad = 0
    for k in range(n_lemma):
        x, y, rot, m = make_lemma_instance(rng, bin_size)
        mode = mode_translation(x, y, rot, bin_size, device=device)
        c_star = count_inliers(x, y, RigidTransform(rot, mode.t_star), bin_size, device=device)
        cand = np.ascontiguousarray((y[None, :, :] - (x @ rot.T)[:, None, :]).reshape(-1, 3))
        step = bin_size / 4.0
        axes = [np.arange(cand[:, a].min(), cand[:, a].max() + step, step) for a in range(3)]
        best = sweep_inlier_best(cand, x.shape[0], y.shape[0], bin_size / 2.0, *axes, device=device)
        if best > c_star:
            lemma_bad += 1
            details.append(f"lemma trial {k}: sweep found {best} inliers vs mode {c_star}")
        elif c_star != m:
            details.append(f"lemma trial {k}: inliers at mode = {c_star}, planted {m}")
    theorem_bad = 0
    for k in range(n_theorem):
        x, y, cfg = make_theorem_instance(rng)
        semi = dses(x, y, cfg, device)
        full = exhaustive_search(x, y, cfg, device)
        if semi.best_inliers != full.best_inliers:
            theorem_bad += 1
            details.append(f"theorem trial {k}: semi-exhaustive {semi.best_inliers} vs "
                           f"exhaustive {full.best_inliers} inliers")
    return OracleReport(lemma_trials=n_lemma, lemma_violations=lemma_bad,
                        theorem_trials=n_theorem, theorem_violations=theorem_bad, details=details)
