"""DSES on the B200: the drop-in for gridreg.engines.dses (engines.py:229-301).

``dses(source, reference, cfg)`` keeps the reference's signature, argument
surface (``SearchConfig``: k_rot, rot_step, k_trans, trans_bin, q, metric,
center, pose_cap), result type (``RegistrationResult``), exceptions and
tie-break rules.  Everything after input validation runs on one GPU through
the C ABI (include/dses_b200.h, ``dses_search``):

  phase 1  vote kernel: per grid rotation, histogram mode of the translation
           votes (counts / flat bin), rotations generated on device;
  phase 2  M*, the q*M* cutoff (engines.py:196-201) and the kept-candidate
           compaction;
  phase 3  fp32 screen of the kept candidates, exact binary64 re-score of the
           near-minimum ones, min-error / lexicographic-grid winner;
  final    exact inlier count of the winner.

The multi-GPU variant (rotation range sharded over ranks) is
``paper_2502_00115_b200.distributed.dses_sharded``.
"""
from __future__ import annotations

import math
import time
from dataclasses import dataclass

import numpy as np

from .errors import InvalidInputError, NoCandidateError, SearchSpaceTooLargeError
from .geometry import RigidTransform, as_point_cloud, check_grid_args, grid_index, grid_rotation, grid_tables
from .metrics import ErrorMetric
from .mode_search import bin_center, bin_index, check_key_space, decode_flat

DEFAULT_POSE_CAP = 100_000_000  # engines.py:45
CUTOFF_EPS = 1e-9               # engines.py:49
DENSE_MAX_BINS = 1 << 26        # csrc/dses_common.cuh kDenseMaxBins


@dataclass(frozen=True)
class SearchConfig:
    """Pose-grid geometry plus refinement policy (engines.py:52-98)."""

    k_rot: int
    rot_step: float
    k_trans: int
    trans_bin: float
    q: float = 0.5
    metric: ErrorMetric | None = None
    center: RigidTransform | None = None
    pose_cap: int = DEFAULT_POSE_CAP

    def __post_init__(self):
        for name in ("k_rot", "k_trans"):
            v = getattr(self, name)
            if int(v) != v or v < 0:
                raise InvalidInputError(f"{name} must be a non-negative integer")
            object.__setattr__(self, name, int(v))
        for name in ("rot_step", "trans_bin"):
            v = float(getattr(self, name))
            if not (v > 0) or not math.isfinite(v):
                raise InvalidInputError(f"{name} must be positive and finite")
            object.__setattr__(self, name, v)
        if not (0.0 < self.q <= 1.0):
            raise InvalidInputError("q must lie in (0, 1]")
        if self.metric is None:
            object.__setattr__(self, "metric", ErrorMetric.truncated_l1(5.0 * self.trans_bin))
        if self.pose_cap < 1:
            raise InvalidInputError("pose_cap must be positive")

    @property
    def rotation_count(self) -> int:
        return (2 * self.k_rot + 1) ** 3

    @property
    def translation_count(self) -> int:
        return (2 * self.k_trans + 1) ** 3


@dataclass(frozen=True)
class PoseCandidate:
    transform: RigidTransform
    inlier_count: int
    refined_error: float | None = None


@dataclass(frozen=True)
class RegistrationResult:
    best: RigidTransform
    best_error: float
    best_inliers: int
    candidates_evaluated: int
    candidates_refined: int
    elapsed: dict


@dataclass
class Prepared:
    """Host-side preparation shared by the single- and multi-GPU drivers."""

    x: np.ndarray
    y: np.ndarray
    cos_tab: np.ndarray
    sin_tab: np.ndarray
    center_rot: np.ndarray | None
    ilo: np.ndarray
    dims: np.ndarray
    code: int
    param: float
    skip_refine: bool


def prepare(source, reference, cfg: SearchConfig) -> Prepared:
    """Validation and lattice set-up of engines.py:241-250 plus the grid
    tables (geometry.py:259-275)."""
    x = as_point_cloud(source)
    y = as_point_cloud(reference)
    if cfg.rotation_count > cfg.pose_cap:
        raise SearchSpaceTooLargeError(
            f"{cfg.rotation_count} rotations exceed the cap of {cfg.pose_cap}")
    check_grid_args(cfg.k_rot, cfg.rot_step)
    cos_tab, sin_tab = grid_tables(cfg.k_rot, cfg.rot_step)
    if cfg.center is not None:
        center_rot = np.ascontiguousarray(cfg.center.rotation, dtype=np.float64)
        t_center = np.asarray(cfg.center.translation, dtype=np.float64)
    else:
        center_rot = None
        t_center = np.zeros(3)
    cbin = bin_index(t_center, cfg.trans_bin)
    ilo = cbin - cfg.k_trans
    dims = np.full(3, 2 * cfg.k_trans + 1, dtype=np.int64)
    nbins = int(dims[0]) ** 3
    check_key_space(nbins, x.shape[0])
    # windows beyond DENSE_MAX_BINS run the sort-based vote (the reference's
    # mode_sparse_batch, mode_search.py:158-163); beyond 2^31 bins the native
    # search raises SearchSpaceTooLargeError
    code, param = cfg.metric._code_param()
    skip = cfg.metric.kind == "sat_l0" and cfg.metric.param == cfg.trans_bin  # engines.py:265
    return Prepared(x, y, cos_tab, sin_tab, center_rot, ilo, dims, code, param, skip)


def winner_transform(prep: Prepared, cfg: SearchConfig, row: int, lin: int) -> RigidTransform:
    """engines.py:282-285: the winner's rotation, bin-centre translation and
    grid coordinates."""
    rot = grid_rotation(prep.cos_tab, prep.sin_tab, cfg.k_rot, row, prep.center_rot)
    t = bin_center(decode_flat(lin, prep.ilo, prep.dims), cfg.trans_bin)
    return RigidTransform(rot, t, grid_coords=tuple(grid_index(cfg.k_rot, row)))


def _result(prep: Prepared, cfg: SearchConfig, res: dict, t0: float) -> RegistrationResult:
    if res["candidates_evaluated"] == 0:
        raise NoCandidateError(
            "no rotation produced an in-bounds translation vote; widen k_trans "
            "or move the search center")
    best = winner_transform(prep, cfg, res["winner_row"], res["winner_lin"])
    t_end = time.perf_counter()
    ms = 1e-3
    return RegistrationResult(
        best=best,
        best_error=float(res["best_error"]),
        best_inliers=int(res["best_inliers"]),
        candidates_evaluated=int(res["candidates_evaluated"]),
        candidates_refined=int(res["candidates_refined"]),
        elapsed={
            "phase1": res["ms_vote"] * ms,
            "sort": res["ms_select"] * ms,
            "refine": (res["ms_total"] - res["ms_vote"] - res["ms_select"]) * ms,
            "total": t_end - t0,
            "device_total": res["ms_total"] * ms,
            "stats": {k: res[k] for k in ("pairs_evaluated", "votes", "rechecks", "rescored",
                                          "mstar", "launches", "h2d_bytes", "d2h_bytes",
                                          "ms_vote_kernel")},
        },
    )


def _build(source, reference, cfg: SearchConfig, device: int):
    """Host preparation + native plan (clouds resident on the GPU)."""
    from . import _native

    t0 = time.perf_counter()
    prep = prepare(source, reference, cfg)
    grid = _native.make_grid(cfg.k_rot, prep.cos_tab, prep.sin_tab, prep.center_rot)
    plan = _native.Plan(prep.x, prep.y, cfg.trans_bin, prep.ilo, prep.dims, device)
    plan.reserve(cfg.rotation_count)  # search scratch allocated with the plan
    return t0, prep, grid, plan


def dses(source, reference, cfg: SearchConfig, device: int = 0) -> RegistrationResult:
    """Direct semi-exhaustive search on one B200 (engines.py:229-301)."""
    t0, prep, grid, plan = _build(source, reference, cfg, device)
    with plan:
        res = plan.search(grid, cfg.q, prep.code, prep.param, prep.skip_refine)
    return _result(prep, cfg, res, t0)


_BUILD_POOL = None


_BUILD_AHEAD = 2  # plans under construction ahead of the running search


def _build_pool():
    """Persistent plan-construction threads (one per plan built ahead): their
    upload streams and pinned staging buffers (per host thread in the C ABI)
    are created once, not on every dses_batch call."""
    global _BUILD_POOL
    if _BUILD_POOL is None:
        import concurrent.futures as cf
        _BUILD_POOL = cf.ThreadPoolExecutor(max_workers=_BUILD_AHEAD, thread_name_prefix="dses-plan")
    return _BUILD_POOL


def dses_batch(sources, references, cfg: SearchConfig, device: int = 0) -> list:
    """dses over a batch of (source, reference) pairs (the registration loop of
    harness.run_batch, harness.py:145-162), pipelined: the host preparation
    and plan construction of pair k+1 (and k+2 for small registrations, which
    are host-bound with one plan ahead: c1) run on worker threads (the C ABI
    releases the GIL; plans upload on their own streams) while the GPU
    searches pair k, and search k+1 is queued before the result of k is read,
    so the GPU runs the searches back to back.  Results are identical to calling dses()
    on each pair; errors are raised for the first failing pair."""
    from collections import deque
    pairs = list(zip(sources, references))
    out = []
    if not pairs:
        return out
    from . import _native

    pending = None  # (t0, prep, grid, plan) whose search is queued on the GPU
    streams = [_native.Stream(device), _native.Stream(device)]  # alternate: the
    # vote of k+1 fills the SMs that k's last rotations and score stage leave idle
    ex = _build_pool()
    futs = deque()  # plans under construction, in pair order (not yet consumed)
    nxt = 0
    # small registrations are host-bound: two plans ahead; larger ones keep one
    # (a second builder only contends with the main thread for the GIL)
    work = cfg.rotation_count * len(pairs[0][0]) * len(pairs[0][1])
    ahead = _BUILD_AHEAD if work < 4e9 else 1

    def top_up():
        nonlocal nxt
        while len(futs) < ahead and nxt < len(pairs):
            futs.append(ex.submit(_build, pairs[nxt][0], pairs[nxt][1], cfg, device))
            nxt += 1

    top_up()
    try:
        for k in range(len(pairs) + 1):
            item, err = None, None
            if k < len(pairs):
                try:
                    cur = futs.popleft()
                    item = cur.result()
                    top_up()
                    _, prep, grid, plan = item
                    plan.search_async(grid, cfg.q, prep.code, prep.param, prep.skip_refine,
                                      stream=streams[k % 2].handle)
                except Exception as exc:  # raised after pair k-1's own outcome
                    if item is not None:
                        item[3].close()
                    item, err = None, exc
            prev, pending = pending, item
            if prev is not None:
                t0, prep, grid, plan = prev
                try:
                    res = plan.search_wait()
                finally:
                    plan.close()
                out.append(_result(prep, cfg, res, t0))
            if err is not None:
                raise err
    finally:
        if pending is not None:
            try:
                pending[3].search_wait()
            except Exception:
                pass
            pending[3].close()
        for f in futs:  # prefetched plans nobody will use
            try:
                f.result()[3].close()
            except Exception:
                pass
        for st in streams:
            st.close()
    return out


def exhaustive_search(source, reference, cfg: SearchConfig, device: int = 0) -> RegistrationResult:
    """Algorithm 1 on the GPU: the metric at every pose of the 6-D grid
    (engines.py:156-193).  Translations are t_center + (-k..k) * trans_bin per
    axis (engines.py:168-169, not lattice-bin centres); the winner is the
    minimum error, ties to the first pose in rotation-major, translation-
    lexicographic order (_kernels.py:327-381).  best_error / best_inliers of
    the winner are recomputed like the reference (engines.py:181-182)."""
    from . import _native
    from .metrics import alignment_error, count_inliers

    t0 = time.perf_counter()
    x = as_point_cloud(source)
    y = as_point_cloud(reference)
    total_poses = cfg.rotation_count * cfg.translation_count
    if total_poses > cfg.pose_cap:
        raise SearchSpaceTooLargeError(
            f"{total_poses} poses exceed the cap of {cfg.pose_cap}; exhaustive "
            f"search cost grows as O(K_rot^3 * K_trans^3 * M * N)")
    check_grid_args(cfg.k_rot, cfg.rot_step)
    cos_tab, sin_tab = grid_tables(cfg.k_rot, cfg.rot_step)
    if cfg.center is not None:
        center_rot = np.ascontiguousarray(cfg.center.rotation, dtype=np.float64)
        t_center = np.asarray(cfg.center.translation, dtype=np.float64)
    else:
        center_rot, t_center = None, np.zeros(3)
    code, param = cfg.metric._code_param()
    grid = _native.make_grid(cfg.k_rot, cos_tab, sin_tab, center_rot)
    dims = np.full(3, 2 * cfg.k_trans + 1, dtype=np.int64)
    ilo = bin_index(t_center, cfg.trans_bin) - cfg.k_trans
    with _native.Plan(x, y, cfg.trans_bin, ilo, dims, device) as plan:
        res = plan.exhaustive(grid, cfg.k_trans, t_center, code, param)
    side = np.arange(-cfg.k_trans, cfg.k_trans + 1, dtype=np.int64).astype(np.float64)
    tvals = [t_center[a] + side * cfg.trans_bin for a in range(3)]
    nt = 2 * cfg.k_trans + 1
    a, rem = divmod(int(res["winner_lin"]), nt * nt)
    b, c = divmod(rem, nt)
    t_best = np.array([tvals[0][a], tvals[1][b], tvals[2][c]])
    row = int(res["winner_row"])
    rot = grid_rotation(cos_tab, sin_tab, cfg.k_rot, row, center_rot)
    best = RigidTransform(rot, t_best, grid_coords=tuple(grid_index(cfg.k_rot, row)))
    err = alignment_error(x, y, best, cfg.metric, device)
    inl = count_inliers(x, y, best, cfg.trans_bin, device)
    total = time.perf_counter() - t0
    return RegistrationResult(best=best, best_error=err, best_inliers=inl,
                              candidates_evaluated=total_poses, candidates_refined=0,
                              elapsed={"search": total, "total": total,
                                       "device_total": res["ms_total"] * 1e-3,
                                       "rescored": res["rescored"]})


CUTOFF_EPS = 1e-9  # engines.py:_CUTOFF_EPS


def refine_cutoff(counts_desc, q: float) -> int:
    """Length of the re-scored prefix of a count-descending list: every entry
    with count >= q * best - 1e-9, at least one (engines.py:196-201)."""
    cutoff = q * counts_desc[0] - CUTOFF_EPS
    return max(1, int(np.searchsorted(-np.asarray(counts_desc, dtype=np.float64), -cutoff,
                                      side="right")))


def refine_candidates(candidates, source, reference, metric: ErrorMetric, q: float,
                      device: int = 0):
    """Re-score the high-vote prefix of a count-sorted candidate list
    (engines.py:204-226): the candidates with inlier_count >= q * best get
    refined_error from the exact binary64 refine kernel (dses_refine_batch),
    the rest are returned unchanged."""
    from dataclasses import replace

    from .metrics import _pose_errors
    if not candidates:
        raise InvalidInputError("candidate list is empty")
    if not (0.0 < q <= 1.0):
        raise InvalidInputError("q must lie in (0, 1]")
    counts = [c.inlier_count for c in candidates]
    if any(counts[i] < counts[i + 1] for i in range(len(counts) - 1)):
        raise InvalidInputError("candidates must be sorted by inlier_count descending")
    x = as_point_cloud(source)
    y = as_point_cloud(reference)
    n_score = refine_cutoff(counts, q)
    rots = np.stack([c.transform.rotation for c in candidates[:n_score]])
    ts = np.stack([c.transform.translation for c in candidates[:n_score]])
    errs = _pose_errors(x, y, rots, ts, metric, device)
    out = [replace(c, refined_error=float(e)) for c, e in zip(candidates[:n_score], errs)]
    out.extend(candidates[n_score:])
    return out
