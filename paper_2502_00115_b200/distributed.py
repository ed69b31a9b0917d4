"""DSES with the rotation grid sharded over ranks.

One process per GPU (torch.distributed, backend "nccl" on B200s).  Every rank
holds both clouds (a few tens of KB) and votes over a contiguous, balanced
slice of the flat lexicographic rotation range [0, R).  The rest of
engines.dses (engines.py:254-301) needs global knowledge at two points only,
so a registration costs two tiny collectives:

  1. after the vote: all_gather of (local M*, local #rotations with a vote)
     -> global M* (the q*M* cutoff of engines.py:196-201 is then identical on
     every rank) and candidates_evaluated (engines.py:254,293);
  2. after the local screen + exact re-score: all_gather of (exact error,
     flat rotation index, translation bin, kept count) -> the winner is the
     minimum (error, rotation index) pair, i.e. min error with ties broken
     to the lexicographically smallest grid index (engines.py:276-280), and
     candidates_refined = max(1, sum kept) (engines.py:201,270).

Each rank re-scores exactly the kept candidates whose fp32 screen error is
within the screen tolerance of its LOCAL minimum.  The global winner w lives
on some rank r; its screen error is at most (global min) + tol <= (min on r)
+ tol, so r always re-scores it: no extra exchange is needed between the
screen and the re-score.  The sat_l0-at-trans_bin shortcut (engines.py:
265-268) gathers (smallest local row at the global M*, its bin) instead.

The final pose error / inlier count of the winner is computed redundantly on
every rank from its replicated clouds (no third collective).

``plan_factory`` exists for the CPU tests, which run this protocol over gloo
with oracle-backed stages; the product path always uses the native plan and
fails loudly without it.
"""
from __future__ import annotations

import math
import time

import numpy as np

from .engines import RegistrationResult, SearchConfig, prepare, winner_transform
from .errors import NoCandidateError

SAT_L0 = 3


def shard_range(total: int, rank: int, world: int):
    """Contiguous balanced slice [begin, end) of [0, total) for ``rank``."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world size")
    return total * rank // world, total * (rank + 1) // world


def _world(group):
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return 0, 1, None
    return dist.get_rank(group), dist.get_world_size(group), dist.get_backend(group)


def _gather(values, group, backend, device):
    """all_gather of a short float64 row -> (world, len) numpy array."""
    import torch
    import torch.distributed as dist
    dev = torch.device("cuda", device) if backend == "nccl" else torch.device("cpu")
    t = torch.tensor(values, dtype=torch.float64, device=dev)
    out = [torch.empty_like(t) for _ in range(dist.get_world_size(group))]
    dist.all_gather(out, t, group=group)
    return torch.stack(out).cpu().numpy()


def _native_plan(prep, cfg, device):
    from . import _native
    plan = _native.Plan(prep.x, prep.y, cfg.trans_bin, prep.ilo, prep.dims, device)
    grid = _native.make_grid(cfg.k_rot, prep.cos_tab, prep.sin_tab, prep.center_rot)
    return plan, grid


def dses_sharded(source, reference, cfg: SearchConfig, group=None, device: int | None = None,
                 plan_factory=None) -> RegistrationResult:
    """engines.dses with the rotation grid split over the ranks of ``group``
    (the default process group when torch.distributed is initialised, else a
    single rank).  Every rank returns the same RegistrationResult."""
    t0 = time.perf_counter()
    rank, world, backend = _world(group)
    if device is None:
        import os
        device = int(os.environ.get("LOCAL_RANK", "0"))
    prep = prepare(source, reference, cfg)
    R = cfg.rotation_count
    r0, r1 = shard_range(R, rank, world)
    plan, grid = (plan_factory or _native_plan)(prep, cfg, device)
    try:
        t_vote = time.perf_counter()
        mstar_l, valid_l = plan.stage_vote(grid, r0, r1 - r0)
        if world > 1:
            g = _gather([float(mstar_l), float(valid_l)], group, backend, device)
            mstar, n_valid = int(g[:, 0].max()), int(g[:, 1].sum())
        else:
            mstar, n_valid = int(mstar_l), int(valid_l)
        t_sort = time.perf_counter()
        if n_valid == 0:
            raise NoCandidateError(
                "no rotation produced an in-bounds translation vote; widen k_trans "
                "or move the search center")
        if prep.skip_refine:
            row_l = plan.stage_argmax(mstar)
            lin_l = plan.stage_row_info(row_l)[0] if row_l != np.iinfo(np.int64).max else -1
            mine = [0.0, float(row_l) if row_l != np.iinfo(np.int64).max else math.inf,
                    float(lin_l), 0.0]
            n_refined = 0
        else:
            kept_l, min32_l, tol = plan.stage_screen(cfg.q, mstar, prep.code, prep.param)
            err_l, row_l, _ = plan.stage_rescore(min32_l + tol, prep.code, prep.param)
            if kept_l > 0 and row_l != np.iinfo(np.int64).max:
                lin_l = plan.stage_row_info(row_l)[0]
                mine = [err_l, float(row_l), float(lin_l), float(kept_l)]
            else:
                mine = [math.inf, math.inf, -1.0, float(kept_l)]
        t_ref = time.perf_counter()
        g = _gather(mine, group, backend, device) if world > 1 else np.asarray([mine])
        order = np.lexsort((g[:, 1], g[:, 0]))  # min error, then min flat rotation index
        err, row, lin = g[order[0], 0], int(g[order[0], 1]), int(g[order[0], 2])
        if not prep.skip_refine:
            n_refined = max(1, int(g[:, 3].sum()))
        miss = plan.pose_error(grid, row, lin, SAT_L0, cfg.trans_bin)
        best_error = miss if prep.skip_refine else float(err)
    finally:
        close = getattr(plan, "close", None)
        if close:
            close()
    best = winner_transform(prep, cfg, row, lin)
    t_end = time.perf_counter()
    return RegistrationResult(
        best=best,
        best_error=float(best_error),
        best_inliers=int(prep.x.shape[0] - round(miss)),
        candidates_evaluated=n_valid,
        candidates_refined=n_refined,
        elapsed={"phase1": t_sort - t_vote, "sort": 0.0, "refine": t_ref - t_sort,
                 "total": t_end - t0, "world_size": world, "rank": rank,
                 "rotations_local": r1 - r0},
    )
