"""DSES with the rotation grid sharded over ranks.

One process per GPU (torch.distributed, backend "nccl" on B200s).  Every rank
holds both clouds (a few tens of KB) and votes over a contiguous, balanced
slice of the flat lexicographic rotation range [0, R).  The rest of
engines.dses (engines.py:254-301) needs global knowledge at one point -- the
global M* before the q*M* cutoff (engines.py:196-201) -- and the min-loc
winner at the end.  Everything stays in device memory: the native stages
write a 7-slot int64 exchange record on the GPU (include/dses_b200.h,
dses_shard_*), and four tiny NCCL all_reduces act on it in place:

  vote      x[0] = local M*, x[3] = rotations with a vote     all_reduce x[0]   MAX
  select    cutoff from the global M*, fp32 screen, exact
            re-score, local winner: x[1] = binary64 bits of
            its error (non-negative doubles order like their
            int64 bits), x[2] = row << 32 | flat bin, x[4] =
            kept, x[6] = overflow                             all_reduce x[1]   MIN
  key       x[2] masked unless this rank holds the minimum    all_reduce x[2]   MIN
  miss      x[5] = the winner's sat_l0 miss on its rank       all_reduce x[3:7] SUM

min error with ties to the smallest flat rotation index is exactly the
reference's rule (min error, then the lexicographically smallest grid index,
engines.py:276-280); candidates_evaluated = sum x[3] (engines.py:254,293),
candidates_refined = max(1, sum x[4]) (engines.py:201,270).  Each rank
re-scores exactly the kept candidates whose fp32 screen error is within the
screen tolerance of its LOCAL minimum; the global winner w lives on some rank
r and its screen error is at most (global min) + tol <= (min on r) + tol, so r
always re-scores it.  The sat_l0-at-trans_bin shortcut (engines.py:265-268)
reduces the smallest local row at the global M* instead.  One device->host
read per registration (the reduced record); the plan (clouds, scratch) is
built once and reused across calls (``ShardedSearch``).

If a rank had more near-minimum candidates than the fused re-score holds
(x[6] > 0, a flat landscape of near-ties), the registration is redone through
the host-staged protocol (``dses_stage_*``), which has no such cap.

``plan_factory`` exists for the CPU tests, which run this protocol over gloo
with oracle-backed stages; the product path always uses the native plan and
fails loudly without it.
"""
from __future__ import annotations

import hashlib
import math
import os
import time

import numpy as np

from .engines import RegistrationResult, SearchConfig, prepare, winner_transform
from .errors import NoCandidateError

SAT_L0 = 3
INT64_MAX = np.iinfo(np.int64).max


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


def _native_plan(prep, cfg, device):
    from . import _native
    plan = _native.Plan(prep.x, prep.y, cfg.trans_bin, prep.ilo, prep.dims, device)
    grid = _native.make_grid(cfg.k_rot, prep.cos_tab, prep.sin_tab, prep.center_rot)
    return plan, grid


def _f64(bits: int) -> float:
    return float(np.int64(bits).view(np.float64))


class ShardedSearch:
    """One registration problem resident on this rank's GPU; ``run()`` is
    engines.dses with the rotation grid split over the ranks of ``group``
    (the default process group when torch.distributed is initialised, else a
    single rank).  Every rank returns the same RegistrationResult."""

    def __init__(self, source, reference, cfg: SearchConfig, group=None, device: int | None = None,
                 plan_factory=None):
        import torch
        self.group = group
        self.rank, self.world, self.backend = _world(group)
        if device is None:
            device = int(os.environ.get("LOCAL_RANK", "0"))
        self.device = device
        self.cfg = cfg
        self.prep = prepare(source, reference, cfg)
        self.r0, self.r1 = shard_range(cfg.rotation_count, self.rank, self.world)
        self.native = plan_factory is None
        self.plan, self.grid = (plan_factory or _native_plan)(self.prep, cfg, device)
        if self.native:
            dev = torch.device("cuda", device)
            self.plan.reserve(max(1, self.r1 - self.r0))
            self.stream = torch.cuda.current_stream(dev).cuda_stream
        else:
            dev, self.stream = torch.device("cpu"), None
        self.xchg = torch.zeros(7, dtype=torch.int64, device=dev)

    def close(self):
        close = getattr(self.plan, "close", None)
        if close:
            close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def _allreduce(self, t, op):
        if self.world == 1:
            return
        import torch.distributed as dist
        if self.backend == "gloo" and t.is_cuda:  # host-side collectives (tests sharing a GPU)
            h = t.cpu()
            dist.all_reduce(h, op=op, group=self.group)
            t.copy_(h)
        else:
            dist.all_reduce(t, op=op, group=self.group)

    def run(self) -> RegistrationResult:
        import torch.distributed as dist
        t0 = time.perf_counter()
        cfg, prep, plan, x = self.cfg, self.prep, self.plan, self.xchg
        ptr = x.data_ptr() if self.native else x
        plan.shard_vote(self.grid, self.r0, self.r1 - self.r0, ptr, self.stream)
        self._allreduce(x[0:1], dist.ReduceOp.MAX)
        plan.shard_select(cfg.q, prep.code, prep.param, prep.skip_refine, ptr, self.stream)
        self._allreduce(x[1:2], dist.ReduceOp.MIN)
        plan.shard_key(ptr, self.stream)
        self._allreduce(x[2:3], dist.ReduceOp.MIN)
        plan.shard_miss(ptr, self.stream)
        self._allreduce(x[3:7], dist.ReduceOp.SUM)
        h = [int(v) for v in x.cpu().tolist()]  # the one device -> host read
        mstar, errbits, key, n_valid, kept, missbits, overflow = h
        if n_valid == 0:
            raise NoCandidateError(
                "no rotation produced an in-bounds translation vote; widen k_trans "
                "or move the search center")
        if overflow:
            return self._staged(t0)
        row, lin = key >> 32, key & 0xFFFFFFFF
        miss = _f64(missbits)
        best_error = miss if prep.skip_refine else _f64(errbits)
        t_end = time.perf_counter()
        return RegistrationResult(
            best=winner_transform(prep, cfg, row, lin),
            best_error=float(best_error),
            best_inliers=int(prep.x.shape[0] - round(miss)),
            candidates_evaluated=n_valid,
            candidates_refined=0 if prep.skip_refine else max(1, kept),
            elapsed={"total": t_end - t0, "world_size": self.world, "rank": self.rank,
                     "rotations_local": self.r1 - self.r0, "mstar": mstar,
                     "protocol": "device"},
        )

    # ---- host-staged protocol (no re-score cap), used on overflow ----------
    def _gather(self, values):
        import torch
        import torch.distributed as dist
        dev = self.xchg.device if self.backend == "nccl" else torch.device("cpu")
        t = torch.tensor(values, dtype=torch.float64, device=dev)
        if self.world == 1:
            return t.cpu().numpy()[None]
        out = [torch.empty_like(t) for _ in range(self.world)]
        dist.all_gather(out, t, group=self.group)
        return torch.stack(out).cpu().numpy()

    def _staged(self, t0) -> RegistrationResult:
        cfg, prep, plan = self.cfg, self.prep, self.plan
        mstar_l, valid_l = plan.stage_vote(self.grid, self.r0, self.r1 - self.r0)
        g = self._gather([float(mstar_l), float(valid_l)])
        mstar, n_valid = int(g[:, 0].max()), int(g[:, 1].sum())
        kept_l, min32_l, tol = plan.stage_screen(cfg.q, mstar, prep.code, prep.param)
        err_l, row_l, _ = plan.stage_rescore(min32_l + tol, prep.code, prep.param)
        if kept_l > 0 and row_l != INT64_MAX:
            mine = [err_l, float(row_l), float(plan.stage_row_info(row_l)[0]), float(kept_l)]
        else:
            mine = [math.inf, math.inf, -1.0, float(kept_l)]
        g = self._gather(mine)
        order = np.lexsort((g[:, 1], g[:, 0]))  # min error, then min flat rotation index
        err, row, lin = g[order[0], 0], int(g[order[0], 1]), int(g[order[0], 2])
        miss = plan.pose_error(self.grid, row, lin, SAT_L0, cfg.trans_bin)
        return RegistrationResult(
            best=winner_transform(prep, cfg, row, lin),
            best_error=float(err),
            best_inliers=int(prep.x.shape[0] - round(miss)),
            candidates_evaluated=n_valid,
            candidates_refined=max(1, int(g[:, 3].sum())),
            elapsed={"total": time.perf_counter() - t0, "world_size": self.world,
                     "rank": self.rank, "rotations_local": self.r1 - self.r0,
                     "protocol": "staged"},
        )


_CACHE: dict = {}


def _key(source, reference, cfg, group, device):
    h = hashlib.blake2b(digest_size=16)
    for a in (source, reference):
        a = np.ascontiguousarray(a, dtype=np.float64)
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return (h.hexdigest(), repr(cfg), id(group), device)


def dses_sharded(source, reference, cfg: SearchConfig, group=None, device: int | None = None,
                 plan_factory=None) -> RegistrationResult:
    """engines.dses with the rotation grid split over the ranks of ``group``.
    The rank's ShardedSearch (plan, scratch, exchange record) is cached for
    the most recent problem, so repeated registrations of the same clouds
    and config pay no plan construction."""
    if plan_factory is not None:  # test stand-ins are never cached
        with ShardedSearch(source, reference, cfg, group, device, plan_factory) as s:
            return s.run()
    k = _key(source, reference, cfg, group, device)
    s = _CACHE.get(k)
    if s is None:
        for old in _CACHE.values():
            old.close()
        _CACHE.clear()
        s = _CACHE[k] = ShardedSearch(source, reference, cfg, group, device)
    return s.run()
