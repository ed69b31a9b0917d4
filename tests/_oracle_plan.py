"""Oracle-backed stand-in for the native plan's stage interface (TEST ONLY).

Lets the multi-rank protocol of paper_2502_00115_b200.distributed run on CPU
(gloo, world_size 2) with the pinned oracle doing each rank's local work.
Stage semantics follow include/dses_b200.h (dses_stage_*): the screen here is
exact (tolerance 0), which the protocol must accept like any tolerance.
"""
import numpy as np

from oracle import oracle as O

INT64_MAX = np.iinfo(np.int64).max


class OraclePlan:
    def __init__(self, prep, cfg):
        self.x, self.y = prep.x, prep.y
        self.bin = cfg.trans_bin
        self.ilo, self.dims = prep.ilo, prep.dims
        self.k, self.step, self.center = cfg.k_rot, cfg.rot_step, prep.center_rot
        self.r0 = 0

    def _rots(self, rows):
        return np.concatenate([O.rotation_grid(self.k, self.step, self.center, int(r), 1)
                               for r in rows]).reshape(-1, 3, 3)

    def _ts(self, lins):
        return np.array([np.asarray(O.decode_flat(l, self.ilo, self.dims), np.float64) * self.bin
                         for l in lins]).reshape(-1, 3)

    def stage_vote(self, grid, r_begin, r_count):
        self.r0 = r_begin
        self.counts, self.lins, _ = O.mode_batch(self.x, self.y, self.bin, self.ilo, self.dims,
                                                 grid=(self.k, self.step, self.center),
                                                 r_begin=r_begin, r_count=r_count)
        if r_count == 0:
            return 0, 0
        return int(self.counts.max()), int((self.counts > 0).sum())

    def stage_argmax(self, mstar):
        hit = np.flatnonzero(self.counts == mstar) if mstar > 0 else []
        return int(self.r0 + hit[0]) if len(hit) else INT64_MAX

    def stage_row_info(self, row):
        return int(self.lins[row - self.r0]), int(self.counts[row - self.r0])

    def stage_screen(self, q, mstar, code, param):
        keep = np.flatnonzero(self.counts >= q * mstar - 1e-9)
        self.kept_rows = self.r0 + keep
        if keep.size == 0:
            self.kept_errs = np.empty(0)
            return 0, np.inf, 0.0
        self.kept_errs = O.refine_batch(self._rots(self.kept_rows), self._ts(self.lins[keep]),
                                        self.x, self.y, code, param)
        return int(keep.size), float(self.kept_errs.min()), 0.0

    def stage_rescore(self, threshold, code, param):
        sel = np.flatnonzero(self.kept_errs <= threshold)
        if sel.size == 0:
            return np.inf, INT64_MAX, 0
        e = self.kept_errs[sel]
        best = sel[e == e.min()]
        return float(e.min()), int(self.kept_rows[best].min()), int(sel.size)

    def pose_error(self, grid, row, lin, code, param):
        return float(O.refine_batch(self._rots([row]), self._ts([lin]), self.x, self.y, code,
                                    param)[0])

    # ---- the device-resident sharded protocol's stages (dses_shard_*), on a
    #      CPU int64[7] torch tensor instead of device memory ---------------
    def shard_vote(self, grid, r_begin, r_count, x, stream=None):
        mstar, valid = self.stage_vote(grid, r_begin, r_count)
        x[0], x[3] = mstar, valid

    def shard_select(self, q, code, param, skip, x, stream=None):
        mstar = int(x[0])
        eb = key = INT64_MAX
        miss = 0.0
        kept = 0
        if skip:
            row = self.stage_argmax(mstar)
            if row != INT64_MAX:
                eb = 0
        else:
            kept, mn, tol = self.stage_screen(q, mstar, code, param)
            _, row, _ = self.stage_rescore(mn + tol, code, param)
            if kept > 0 and row != INT64_MAX:
                e = self.stage_rescore(mn + tol, code, param)[0]
                eb = int(np.float64(e).view(np.int64))
        if eb != INT64_MAX:
            lin = int(self.lins[row - self.r0])
            key = (row << 32) | lin
            miss = self.pose_error(grid=None, row=row, lin=lin, code=3, param=self.bin)
        self._eb, self._key, self._miss = eb, key, int(np.float64(miss).view(np.int64))
        x[1], x[2], x[4], x[5], x[6] = eb, key, kept, 0, 0

    def shard_key(self, x, stream=None):
        if self._eb != int(x[1]):
            x[2] = INT64_MAX

    def shard_miss(self, x, stream=None):
        x[5] = self._miss if self._key == int(x[2]) else 0
