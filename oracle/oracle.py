"""CPU oracle for the DSES hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this module, and only as the checker (or
the timed CPU baseline), never as the thing shipped.  The product path
(``paper_2502_00115_b200``) never imports it.

This is a restatement of the reference package ``gridreg``
(/root/reference/pkg/src/gridreg) in numpy (host logic) plus plain C
(``gridreg_oracle.c``: the numba kernels).  Each function cites the reference
lines it follows.  It is pinned against golden vectors produced by the
unmodified reference (``tests/golden/make_golden.py``); see
``tests/test_oracle_golden.py``.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liborc.so")
_lib = None

METRIC_CODES = {"l2": 0, "l1": 1, "trunc_l1": 2, "sat_l0": 3, "trunc_l2": 4}
_CUTOFF_EPS = 1e-9  # engines.py:49

_dp = ctypes.POINTER(ctypes.c_double)
_ip = ctypes.POINTER(ctypes.c_int64)
_i64 = ctypes.c_int64


def build():
    """Compile the C restatement (oracle/Makefile)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.orc_rotation_grid.argtypes = [_i64, _dp, _dp, _dp, _i64, _i64, _dp]
        L.orc_rotation_grid.restype = None
        L.orc_mode_dense_batch.argtypes = [
            _dp, _i64, _dp, _dp, _dp, _i64, _i64, _dp, _i64, _dp, _dp, _dp, _i64,
            ctypes.c_double, ctypes.c_double, _i64, _i64, _i64, _i64, _i64, _i64,
            _ip, _ip, _ip, ctypes.c_int,
        ]
        L.orc_mode_dense_batch.restype = ctypes.c_int
        L.orc_refine_batch.argtypes = [
            _dp, _dp, _i64, _dp, _i64, _dp, _dp, _dp, _i64, ctypes.c_int, ctypes.c_double,
            _dp, ctypes.c_int,
        ]
        L.orc_refine_batch.restype = None
        L.orc_alignment_error.argtypes = [_dp, _i64, _dp, _dp, _dp, _i64, ctypes.c_int,
                                          ctypes.c_double]
        L.orc_alignment_error.restype = ctypes.c_double
        L.orc_max_threads.argtypes = []
        L.orc_max_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _p(a, ptr=_dp):
    return None if a is None else a.ctypes.data_as(ptr)


def max_threads() -> int:
    return int(lib().orc_max_threads())


# ---------------------------------------------------------------------------
# geometry (geometry.py:253-290) and engines._prepare (engines.py:120-130)
# ---------------------------------------------------------------------------

def trig_tables(k: int, step: float):
    """Per-axis cos/sin tables: geometry.py:268-275 evaluates np.cos/np.sin on
    idx.astype(float64) * step; the (2k+1) distinct angles give the same values."""
    ang = np.arange(-k, k + 1, dtype=np.int64).astype(np.float64) * float(step)
    return np.ascontiguousarray(np.cos(ang)), np.ascontiguousarray(np.sin(ang))


def rotation_grid(k: int, step: float, center_rot=None, r_begin=0, r_count=None):
    """(R,3,3) rotations in lexicographic grid order (geometry.py:268-287,
    engines.py:122-126)."""
    n = (2 * k + 1) ** 3
    if r_count is None:
        r_count = n - r_begin
    c, s = trig_tables(k, step)
    out = np.empty((r_count, 3, 3))
    cen = None if center_rot is None else np.ascontiguousarray(center_rot, dtype=np.float64)
    lib().orc_rotation_grid(k, _p(c), _p(s), _p(cen), r_begin, r_count, _p(out))
    return out


def grid_indices(k: int, r):
    """Lexicographic (theta, phi, xi) index triple of flat rotation r
    (geometry.py:268-271: meshgrid 'ij' over arange(-k, k+1))."""
    n = 2 * k + 1
    r = np.asarray(r, dtype=np.int64)
    return np.stack([r // (n * n) - k, (r // n) % n - k, r % n - k], axis=-1)


# ---------------------------------------------------------------------------
# mode_search (mode_search.py:40-54, 132-171)
# ---------------------------------------------------------------------------

def bin_index(v, bin_size: float):
    """mode_search.py:40-49 (round half away from zero of v / bin_size)."""
    q = np.asarray(v, dtype=np.float64) * (1.0 / bin_size)
    return np.copysign(np.floor(np.fabs(q) + 0.5), q).astype(np.int64)


def sorted_columns(y):
    """mode_search.py:141-145 / engines.py:133-140: stable sort of Y by axis 0."""
    y = np.ascontiguousarray(y, dtype=np.float64)
    order = np.argsort(y[:, 0], kind="stable")
    ys = y[order]
    return tuple(np.ascontiguousarray(ys[:, a]) for a in range(3))


def mode_batch(x, y, bin_size, ilo, dims, rots=None, grid=None, r_begin=0, r_count=None,
               nthreads=0):
    """mode_search._mode_batch (mode_search.py:132-164) -> (counts, lins, ties).

    Rotations from ``rots`` (R,3,3) or from ``grid=(k, step, center_rot|None)``.
    The dense kernel is used for every lattice size; the reference's sparse
    path (_kernels.py:196-294) returns identical results (tests/test_mode_search
    TestDenseSparseAgreement), so the oracle needs only one.
    """
    x = np.ascontiguousarray(x, dtype=np.float64)
    y0, y1, y2 = sorted_columns(y)
    d0, d1, d2 = (int(v) for v in dims)
    l0, l1, l2 = (int(v) for v in ilo)
    if rots is not None:
        rots = np.ascontiguousarray(rots, dtype=np.float64).reshape(-1, 3, 3)
        nrot = rots.shape[0]
        k, c, s, cen = 0, None, None, None
    else:
        k, step, cen = grid
        c, s = trig_tables(k, step)
        nrot = (2 * k + 1) ** 3 - r_begin if r_count is None else r_count
        cen = None if cen is None else np.ascontiguousarray(cen, dtype=np.float64)
    counts = np.empty(nrot, dtype=np.int64)
    lins = np.empty(nrot, dtype=np.int64)
    ties = np.empty(nrot, dtype=np.int64)
    rc = lib().orc_mode_dense_batch(
        _p(rots), k, _p(c), _p(s), _p(cen), r_begin, nrot, _p(x), x.shape[0],
        _p(y0), _p(y1), _p(y2), y0.shape[0], 1.0 / bin_size, float(bin_size),
        l0, l1, l2, d0, d1, d2, _p(counts, _ip), _p(lins, _ip), _p(ties, _ip), int(nthreads),
    )
    if rc != 0:
        raise MemoryError("oracle scratch allocation failed")
    return counts, lins, ties


def decode_flat(lin, ilo, dims):
    """mode_search.py:167-171."""
    d1, d2 = int(dims[1]), int(dims[2])
    a, rem = divmod(int(lin), d1 * d2)
    b, c = divmod(rem, d2)
    return (a + int(ilo[0]), b + int(ilo[1]), c + int(ilo[2]))


# ---------------------------------------------------------------------------
# metrics / refine (engines.py:143-153, metrics.py:133-150, _kernels.py:34-89,297-324)
# ---------------------------------------------------------------------------

def refine_batch(rots, ts, x, y, code, param, nthreads=0):
    """engines._score_poses -> _kernels.refine_batch."""
    rots = np.ascontiguousarray(rots, dtype=np.float64).reshape(-1, 3, 3)
    ts = np.ascontiguousarray(ts, dtype=np.float64).reshape(-1, 3)
    x = np.ascontiguousarray(x, dtype=np.float64)
    y0, y1, y2 = sorted_columns(y)
    out = np.empty(rots.shape[0])
    lib().orc_refine_batch(_p(rots), _p(ts), rots.shape[0], _p(x), x.shape[0], _p(y0), _p(y1),
                           _p(y2), y0.shape[0], int(code), float(param), _p(out), int(nthreads))
    return out


def alignment_error(x, y, rot, t, code, param):
    """metrics.alignment_error (metrics.py:133-140): numpy transform
    `pts @ R.T + t` (geometry.py:209-211), then the serial kernel sum."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    p = np.ascontiguousarray(x @ np.asarray(rot, dtype=np.float64).T + np.asarray(t, np.float64))
    y0, y1, y2 = sorted_columns(y)
    return float(lib().orc_alignment_error(_p(p), p.shape[0], _p(y0), _p(y1), _p(y2), y0.shape[0],
                                           int(code), float(param)))


def count_inliers(x, y, rot, t, bin_size):
    """metrics.count_inliers (metrics.py:143-150)."""
    miss = alignment_error(x, y, rot, t, METRIC_CODES["sat_l0"], bin_size)
    return int(np.asarray(x).shape[0]) - int(round(miss))


def refine_cutoff(counts_desc, q):
    """engines._refine_cutoff (engines.py:196-201)."""
    mstar = counts_desc[0]
    cutoff = q * mstar - _CUTOFF_EPS
    n = int(np.searchsorted(-np.asarray(counts_desc, dtype=np.float64), -cutoff, side="right"))
    return max(1, n)


# ---------------------------------------------------------------------------
# dses (engines.py:229-301)
# ---------------------------------------------------------------------------

def dses(x, y, k_rot, rot_step, k_trans, trans_bin, q=0.5, metric=("trunc_l1", None),
         center=None, nthreads=0, return_votes=False):
    """Restatement of engines.dses.  ``metric`` = (kind, param) with param None
    meaning the reference default (trunc_l1 at 5*trans_bin, engines.py:87-88).
    ``center`` = (R, t) or None.  Returns a dict (keys follow RegistrationResult
    plus ``winner_row``; with ``return_votes`` also counts/lins/ties)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    kind, param = metric
    if kind == "trunc_l1" and param is None:
        param = 5.0 * trans_bin
    code = METRIC_CODES[kind]
    param = 0.0 if param is None else float(param)
    cen_r = None if center is None else np.asarray(center[0], dtype=np.float64)
    t_center = np.zeros(3) if center is None else np.asarray(center[1], dtype=np.float64)
    cbin = bin_index(t_center, trans_bin)                       # engines.py:248
    ilo = cbin - k_trans                                        # engines.py:249
    dims = np.full(3, 2 * k_trans + 1, dtype=np.int64)          # engines.py:250
    counts, lins, ties = mode_batch(x, y, trans_bin, ilo, dims, grid=(k_rot, rot_step, cen_r),
                                    nthreads=nthreads)
    valid = np.flatnonzero(counts > 0)                          # engines.py:254
    if valid.size == 0:
        raise LookupError("NoCandidateError")
    order = valid[np.argsort(-counts[valid], kind="stable")]    # engines.py:261
    skip = kind == "sat_l0" and param == trans_bin              # engines.py:265
    errs = None
    rows = None
    if skip:
        winner = int(order[0])
        n_score = 0
    else:
        n_score = refine_cutoff(counts[order].astype(np.float64), q)
        rows = order[:n_score]
        t_stack = np.array([np.asarray(decode_flat(lins[r], ilo, dims), dtype=np.float64)
                            * float(trans_bin) for r in rows]).reshape(-1, 3)
        rots = np.concatenate([rotation_grid(k_rot, rot_step, cen_r, int(r), 1) for r in rows])
        errs = refine_batch(rots, t_stack, x, y, code, param, nthreads)
        emin = errs.min()
        tied = np.flatnonzero(errs == emin)
        winner = int(min(rows[p] for p in tied))   # lexicographic grid order == flat order
    t_win = np.asarray(decode_flat(lins[winner], ilo, dims), dtype=np.float64) * float(trans_bin)
    r_win = rotation_grid(k_rot, rot_step, cen_r, winner, 1)[0]
    out = {
        "rotation": r_win,
        "translation": t_win,
        "grid_coords": tuple(int(v) for v in grid_indices(k_rot, winner)),
        "winner_row": winner,
        "best_error": alignment_error(x, y, r_win, t_win, code, param),
        "best_inliers": count_inliers(x, y, r_win, t_win, trans_bin),
        "candidates_evaluated": int(valid.size),
        "candidates_refined": int(n_score),
        "refine_rows": rows,
        "refine_errs": errs,
    }
    if return_votes:
        out.update(counts=counts, lins=lins, ties=ties)
    return out


def translation_histogram(x, y, rot, bin_size, ilo=None, ihi=None, dedup=True):
    """Pure-numpy vote map, mode_search.py:206-235 (diagnostic, small inputs)."""
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    cand = (y[None, :, :] - (x @ np.asarray(rot, np.float64).T)[:, None, :]).reshape(-1, 3)
    bins = bin_index(cand, bin_size)
    src = np.repeat(np.arange(x.shape[0]), y.shape[0])
    if ilo is not None:
        keep = np.all((bins >= ilo) & (bins <= ihi), axis=1)
        bins, src = bins[keep], src[keep]
    if dedup and bins.shape[0]:
        bins = np.unique(np.concatenate([bins, src[:, None]], axis=1), axis=0)[:, :3]
    if bins.shape[0] == 0:
        return {}
    uniq, cnt = np.unique(bins, axis=0, return_counts=True)
    return {tuple(int(v) for v in key): int(c) for key, c in zip(uniq, cnt)}




def sweep_inlier_best(cands, n, m, half, t0vals, t1vals, t2vals):
    """_kernels.sweep_inlier_best (_kernels.py:384-410) in numpy, one t0 plane
    at a time: max over the lattice of the number of sources i with some
    j such that |cands[i*m+j] - t|_inf < half (strict, binary64)."""
    c = np.asarray(cands, dtype=np.float64).reshape(n, m, 3)
    t1 = np.asarray(t1vals, dtype=np.float64)
    t2 = np.asarray(t2vals, dtype=np.float64)
    if n == 0 or m == 0 or min(len(t0vals), t1.size, t2.size) == 0:
        return 0
    in1 = np.abs(c[:, :, 1, None] - t1[None, None, :]) < half   # (n, m, n1)
    in2 = np.abs(c[:, :, 2, None] - t2[None, None, :]) < half   # (n, m, n2)
    best = 0
    for a in np.asarray(t0vals, dtype=np.float64):
        in0 = np.abs(c[:, :, 0] - a) < half                       # (n, m)
        hit = (in0[:, :, None, None] & in1[:, :, :, None] & in2[:, :, None, :]).any(axis=1)
        best = max(best, int(hit.sum(axis=0).max()))
    return best
