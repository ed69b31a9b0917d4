"""ctypes binding of the C ABI in include/dses_b200.h (libdses_b200.so).

The shared library is built in-tree (``paper_2502_00115_b200/_lib``) by
``__graft_entry__.build()`` / ``python -m paper_2502_00115_b200.build``.  There
is no CPU fallback: when the library or a B200 is missing every entry point
raises ``NativeUnavailable`` (loudly), it never silently computes elsewhere.
"""
from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DSES_LIB") or os.path.join(_HERE, "_lib", "libdses_b200.so")

DSES_OK = 0
DSES_E_INVALID = -1
DSES_E_CUDA = -2
DSES_E_NOMEM = -3
DSES_E_NODEVICE = -4
DSES_E_LIMIT = -5


class NativeUnavailable(RuntimeError):
    """The sm_100a extension is not built or no B200 is visible."""


class NativeError(RuntimeError):
    """A CUDA/runtime failure inside the extension."""


_i64 = ctypes.c_int64
_dp = ctypes.POINTER(ctypes.c_double)
_ip = ctypes.POINTER(ctypes.c_int64)
_vp = ctypes.c_void_p


class Grid(ctypes.Structure):
    _fields_ = [("k", _i64), ("cos_tab", _dp), ("sin_tab", _dp), ("center", _dp)]


class Result(ctypes.Structure):
    _fields_ = [
        ("candidates_evaluated", _i64), ("candidates_refined", _i64), ("mstar", _i64),
        ("winner_row", _i64), ("winner_lin", _i64), ("winner_count", _i64),
        ("best_error", ctypes.c_double), ("best_inliers", _i64), ("rescored", _i64),
        ("pairs_evaluated", _i64), ("votes", _i64), ("rechecks", _i64),
        ("ms_vote", ctypes.c_double), ("ms_select", ctypes.c_double),
        ("ms_score", ctypes.c_double), ("ms_total", ctypes.c_double),
        ("ms_vote_kernel", ctypes.c_double), ("launches", _i64), ("h2d_bytes", _i64),
        ("d2h_bytes", _i64),
    ]

    def as_dict(self):
        return {name: getattr(self, name) for name, _ in self._fields_}


# (name, restype, argtypes) -- mirrors include/dses_b200.h
_SIGS = [
    ("dses_last_error", ctypes.c_char_p, []),
    ("dses_build_info", ctypes.c_char_p, []),
    ("dses_device_count", ctypes.c_int, [ctypes.POINTER(ctypes.c_int)]),
    ("dses_plan_create", ctypes.c_int, [ctypes.c_int, _dp, _i64, _dp, _i64, ctypes.c_double,
                                        _ip, _ip, ctypes.POINTER(_vp)]),
    ("dses_plan_destroy", ctypes.c_int, [_vp]),
    ("dses_plan_info", ctypes.c_int, [_vp, _ip, _ip, _ip, _ip]),
    ("dses_plan_set_vote_grid", ctypes.c_int, [_vp, _i64]),
    ("dses_plan_set_blocks", ctypes.c_int, [_vp, _ip, _i64]),
    ("dses_plan_blocks", ctypes.c_int, [_vp, _ip]),
    ("dses_mode_batch", ctypes.c_int, [_vp, _dp, _i64, _ip, _ip, _ip, _vp]),
    ("dses_mode_grid", ctypes.c_int, [_vp, ctypes.POINTER(Grid), _i64, _i64, _ip, _ip, _ip, _vp]),
    ("dses_refine_batch", ctypes.c_int, [_vp, _dp, _dp, _i64, ctypes.c_int, ctypes.c_double, _dp,
                                         _vp]),
    ("dses_translation_histogram", ctypes.c_int, [_vp, _dp, ctypes.c_int, _ip, _ip, _i64, _ip, _ip,
                                                  _vp]),
    ("dses_mode_dense_batch", ctypes.c_int, [ctypes.c_int, _dp, _i64, _dp, _i64, _dp, _i64,
                                             ctypes.c_double, _ip, _ip, _ip, _ip, _ip]),
    ("dses_search", ctypes.c_int, [_vp, ctypes.POINTER(Grid), _i64, _i64, ctypes.c_double,
                                   ctypes.c_int, ctypes.c_double, ctypes.c_int,
                                   ctypes.POINTER(Result), _vp]),
    ("dses_plan_reserve", ctypes.c_int, [_vp, _i64]),
    ("dses_stream_create", ctypes.c_int, [ctypes.c_int, ctypes.POINTER(_vp)]),
    ("dses_stream_destroy", ctypes.c_int, [_vp]),
    ("dses_search_async", ctypes.c_int, [_vp, ctypes.POINTER(Grid), _i64, _i64, ctypes.c_double,
                                         ctypes.c_int, ctypes.c_double, ctypes.c_int, _vp]),
    ("dses_search_wait", ctypes.c_int, [_vp, ctypes.POINTER(Result)]),
    ("dses_exhaustive", ctypes.c_int, [_vp, ctypes.POINTER(Grid), _i64, _dp, ctypes.c_int,
                                       ctypes.c_double, ctypes.POINTER(Result), _vp]),
    ("dses_stage_vote", ctypes.c_int, [_vp, ctypes.POINTER(Grid), _i64, _i64, _ip, _ip, _vp]),
    ("dses_stage_argmax", ctypes.c_int, [_vp, _i64, _ip, _vp]),
    ("dses_stage_screen", ctypes.c_int, [_vp, ctypes.c_double, _i64, ctypes.c_int, ctypes.c_double,
                                         _ip, _dp, _dp, _vp]),
    ("dses_stage_rescore", ctypes.c_int, [_vp, ctypes.c_double, ctypes.c_int, ctypes.c_double, _dp,
                                          _ip, _ip, _vp]),
    ("dses_stage_row_info", ctypes.c_int, [_vp, _i64, _ip, _ip, _vp]),
    ("dses_pose_error", ctypes.c_int, [_vp, ctypes.POINTER(Grid), _i64, _i64, ctypes.c_int,
                                       ctypes.c_double, _dp, _vp]),
    ("dses_stage_stats", ctypes.c_int, [_vp, _ip, _ip, _ip]),
    ("dses_shard_vote", ctypes.c_int, [_vp, ctypes.POINTER(Grid), _i64, _i64, _vp, _vp]),
    ("dses_shard_select", ctypes.c_int, [_vp, ctypes.c_double, ctypes.c_int, ctypes.c_double,
                                         ctypes.c_int, _vp, _vp]),
    ("dses_shard_key", ctypes.c_int, [_vp, _vp, _vp]),
    ("dses_shard_miss", ctypes.c_int, [_vp, _vp, _vp]),
    ("dses_plan_traffic", ctypes.c_int, [_vp, _ip, _ip, _ip, ctypes.c_int]),
    ("dses_sweep_inlier_best", ctypes.c_int, [ctypes.c_int, _dp, _i64, _i64, ctypes.c_double,
                                              _dp, _i64, _dp, _i64, _dp, _i64, _ip]),
    ("dses_probe_fp32_peak", ctypes.c_int, [ctypes.c_int, _dp, _dp]),
]
EXPORTED = tuple(name for name, _, _ in _SIGS)

_lib = None
_lock = threading.Lock()


def load(path: str = LIB_PATH):
    """Load and type the library (no GPU needed).  Raises NativeUnavailable."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise NativeUnavailable(
                f"{path} is missing: build it with `python -m paper_2502_00115_b200.build` "
                "(there is no CPU fallback)")
        try:
            L = ctypes.CDLL(path)
        except OSError as e:  # pragma: no cover - depends on the box
            raise NativeUnavailable(f"cannot load {path}: {e}") from e
        for name, res, args in _SIGS:
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
        return L


def last_error() -> str:
    return load().dses_last_error().decode(errors="replace")


def check(rc: int, what: str):
    """Map a C-ABI status to the reference's exception contract: bad
    arguments raise InvalidInputError (a ValueError, errors.py), inputs past a
    documented size limit of this implementation SearchSpaceTooLargeError --
    both GridregError, so the batch harness records them per trial."""
    if rc == DSES_OK:
        return
    from .errors import InvalidInputError, SearchSpaceTooLargeError
    msg = f"{what}: {last_error()}"
    if rc == DSES_E_NODEVICE:
        raise NativeUnavailable(msg)
    if rc == DSES_E_INVALID:
        raise InvalidInputError(msg)
    if rc == DSES_E_LIMIT:
        raise SearchSpaceTooLargeError(msg)
    if rc == DSES_E_NOMEM:
        raise MemoryError(msg)
    raise NativeError(msg)


def device_count() -> int:
    n = ctypes.c_int(0)
    rc = load().dses_device_count(ctypes.byref(n))
    return n.value if rc == DSES_OK else 0


def probe_fp32_peak(device: int = 0):
    """Live FFMA/s of the device (independent FFMA chains on every SM)."""
    f, ms = ctypes.c_double(), ctypes.c_double()
    check(load().dses_probe_fp32_peak(int(device), ctypes.byref(f), ctypes.byref(ms)),
          "dses_probe_fp32_peak")
    return f.value, ms.value


def sweep_inlier_best(cands, n: int, m: int, half: float, t0, t1, t2, device: int = 0) -> int:
    """dses_sweep_inlier_best: maximum inlier count over the lattice t0 x t1 x t2."""
    c = np.ascontiguousarray(cands, dtype=np.float64).reshape(-1, 3)
    if c.shape[0] != n * m:
        raise ValueError("cands must hold n*m difference vectors")
    axes = [np.ascontiguousarray(t, dtype=np.float64).ravel() for t in (t0, t1, t2)]
    best = ctypes.c_int64()
    check(load().dses_sweep_inlier_best(int(device), dptr(c), int(n), int(m), float(half),
                                        dptr(axes[0]), axes[0].size, dptr(axes[1]), axes[1].size,
                                        dptr(axes[2]), axes[2].size, ctypes.byref(best)),
          "dses_sweep_inlier_best")
    return int(best.value)


def dptr(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def iptr(a: np.ndarray):
    return a.ctypes.data_as(_ip)


def make_grid(k: int, cos_tab: np.ndarray, sin_tab: np.ndarray, center=None):
    """Build a Grid struct; keeps references to the arrays on the struct."""
    g = Grid()
    g.k = int(k)
    g.cos_tab = dptr(cos_tab)
    g.sin_tab = dptr(sin_tab)
    c = None if center is None else np.ascontiguousarray(center, dtype=np.float64).reshape(9)
    g.center = dptr(c) if c is not None else ctypes.cast(None, _dp)
    g._keep = (cos_tab, sin_tab, c)
    return g


class Stream:
    """A non-blocking CUDA stream owned by the library (dses_stream_*)."""

    def __init__(self, device=0):
        self._L = load()
        h = _vp()
        check(self._L.dses_stream_create(int(device), ctypes.byref(h)), "dses_stream_create")
        self.handle = h

    def close(self):
        if getattr(self, "handle", None) is not None and self.handle.value:
            check(self._L.dses_stream_destroy(self.handle), "dses_stream_destroy")
            self.handle = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


class Plan:
    """One (source, reference, translation lattice) problem resident on a GPU
    (wraps dses_plan_*)."""

    def __init__(self, x, y, bin_size, ilo, dims, device=0):
        L = load()
        self._L = L
        self.x = np.ascontiguousarray(x, dtype=np.float64)
        self.y = np.ascontiguousarray(y, dtype=np.float64)
        self.n, self.m = self.x.shape[0], self.y.shape[0]
        self.bin_size = float(bin_size)
        self.ilo = np.ascontiguousarray(ilo, dtype=np.int64).reshape(3)
        self.dims = np.ascontiguousarray(dims, dtype=np.int64).reshape(3)
        self.device = int(device)
        h = _vp()
        check(L.dses_plan_create(self.device, dptr(self.x), self.n, dptr(self.y), self.m,
                                 self.bin_size, iptr(self.ilo), iptr(self.dims), ctypes.byref(h)),
              "dses_plan_create")
        self._h = h

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            self._L.dses_plan_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def handle(self):
        return self._h

    def info(self):
        v = [ctypes.c_int64() for _ in range(4)]
        check(self._L.dses_plan_info(self._h, *[ctypes.byref(a) for a in v]), "dses_plan_info")
        return {"frac_bits": v[0].value, "x_tiles": v[1].value, "y_tiles": v[2].value,
                "near_pairs": v[3].value}

    def set_vote_grid(self, ctas):
        """Testing hook: cap the vote kernel's persistent grid (0 = default)."""
        check(self._L.dses_plan_set_vote_grid(self._h, int(ctas)), "dses_plan_set_vote_grid")

    def blocks(self):
        """Block shape of this plan's grid searches ((0, 0, 0): per-rotation kernel)."""
        v = np.zeros(3, dtype=np.int64)
        check(self._L.dses_plan_blocks(self._h, iptr(v)), "dses_plan_blocks")
        return tuple(int(a) for a in v)

    def set_blocks(self, shape, list_cap=0):
        """Rotation-block shape of the vote ((0, 0, 0) or 0 = the per-rotation
        kernel; an int n = (1, 1, n)) and the list entries per CTA (0 =
        default; testing hook for the overflow path)."""
        if isinstance(shape, int):
            shape = (0, 0, 0) if shape == 0 else (1, 1, shape)
        v = np.ascontiguousarray(shape, dtype=np.int64).reshape(3)
        check(self._L.dses_plan_set_blocks(self._h, iptr(v), int(list_cap)), "dses_plan_set_blocks")

    def mode_batch(self, rots, stream=None):
        rots = np.ascontiguousarray(rots, dtype=np.float64).reshape(-1, 9)
        nr = rots.shape[0]
        c, l, t = (np.empty(nr, dtype=np.int64) for _ in range(3))
        check(self._L.dses_mode_batch(self._h, dptr(rots), nr, iptr(c), iptr(l), iptr(t), stream),
              "dses_mode_batch")
        return c, l, t

    def mode_grid(self, grid: Grid, r_begin, nrot, stream=None):
        c, l, t = (np.empty(nrot, dtype=np.int64) for _ in range(3))
        check(self._L.dses_mode_grid(self._h, ctypes.byref(grid), int(r_begin), int(nrot), iptr(c),
                                     iptr(l), iptr(t), stream), "dses_mode_grid")
        return c, l, t

    def histogram(self, rot, dedup=True, stream=None):
        """(flat bins ascending, counts, pairs in lattice) of one rotation."""
        rot = np.ascontiguousarray(rot, dtype=np.float64).reshape(9)
        cap = self.n * self.m
        lins, counts = np.empty(cap, dtype=np.int64), np.empty(cap, dtype=np.int64)
        nb, npairs = ctypes.c_int64(0), ctypes.c_int64(0)
        check(self._L.dses_translation_histogram(self._h, dptr(rot), int(bool(dedup)), iptr(lins),
                                                 iptr(counts), cap, ctypes.byref(nb),
                                                 ctypes.byref(npairs), stream),
              "dses_translation_histogram")
        return lins[:nb.value].copy(), counts[:nb.value].copy(), npairs.value

    def refine_batch(self, rots, ts, code, param, stream=None):
        rots = np.ascontiguousarray(rots, dtype=np.float64).reshape(-1, 9)
        ts = np.ascontiguousarray(ts, dtype=np.float64).reshape(-1, 3)
        out = np.empty(rots.shape[0])
        check(self._L.dses_refine_batch(self._h, dptr(rots), dptr(ts), rots.shape[0], int(code),
                                        float(param), dptr(out), stream), "dses_refine_batch")
        return out

    def search(self, grid: Grid, q, code, param, skip_refine, r_begin=0, r_count=-1, stream=None):
        res = Result()
        check(self._L.dses_search(self._h, ctypes.byref(grid), int(r_begin), int(r_count), float(q),
                                  int(code), float(param), int(bool(skip_refine)),
                                  ctypes.byref(res), stream), "dses_search")
        return res.as_dict()

    def reserve(self, r_count):
        """Pre-allocate the search buffers for r_count rotations."""
        check(self._L.dses_plan_reserve(self._h, int(r_count)), "dses_plan_reserve")

    def search_async(self, grid: Grid, q, code, param, skip_refine, r_begin=0, r_count=-1,
                     stream=None):
        """Enqueue a search; search_wait() returns its result dict."""
        check(self._L.dses_search_async(self._h, ctypes.byref(grid), int(r_begin), int(r_count),
                                        float(q), int(code), float(param), int(bool(skip_refine)),
                                        stream), "dses_search_async")
        self._inflight = grid  # its host tables must outlive the search

    def search_wait(self):
        res = Result()
        try:
            check(self._L.dses_search_wait(self._h, ctypes.byref(res)), "dses_search_wait")
        finally:
            self._inflight = None
        return res.as_dict()

    def exhaustive(self, grid: Grid, k_trans, t_center, code, param, stream=None):
        res = Result()
        tc = np.ascontiguousarray(t_center, dtype=np.float64).reshape(3)
        check(self._L.dses_exhaustive(self._h, ctypes.byref(grid), int(k_trans), dptr(tc), int(code),
                                      float(param), ctypes.byref(res), stream), "dses_exhaustive")
        return res.as_dict()

    # ---- stages (multi-GPU) ----
    def stage_vote(self, grid: Grid, r_begin, r_count, stream=None):
        ms, nv = ctypes.c_int64(), ctypes.c_int64()
        check(self._L.dses_stage_vote(self._h, ctypes.byref(grid), int(r_begin), int(r_count),
                                      ctypes.byref(ms), ctypes.byref(nv), stream), "dses_stage_vote")
        return ms.value, nv.value

    def stage_argmax(self, mstar, stream=None):
        r = ctypes.c_int64()
        check(self._L.dses_stage_argmax(self._h, int(mstar), ctypes.byref(r), stream),
              "dses_stage_argmax")
        return r.value

    def stage_screen(self, q, mstar, code, param, stream=None):
        k, mn, tol = ctypes.c_int64(), ctypes.c_double(), ctypes.c_double()
        check(self._L.dses_stage_screen(self._h, float(q), int(mstar), int(code), float(param),
                                        ctypes.byref(k), ctypes.byref(mn), ctypes.byref(tol),
                                        stream), "dses_stage_screen")
        return k.value, mn.value, tol.value

    def stage_rescore(self, threshold, code, param, stream=None):
        e, r, n = ctypes.c_double(), ctypes.c_int64(), ctypes.c_int64()
        check(self._L.dses_stage_rescore(self._h, float(threshold), int(code), float(param),
                                         ctypes.byref(e), ctypes.byref(r), ctypes.byref(n), stream),
              "dses_stage_rescore")
        return e.value, r.value, n.value

    def stage_row_info(self, row, stream=None):
        lin, cnt = ctypes.c_int64(), ctypes.c_int64()
        check(self._L.dses_stage_row_info(self._h, int(row), ctypes.byref(lin), ctypes.byref(cnt),
                                          stream), "dses_stage_row_info")
        return lin.value, cnt.value

    # ---- device-resident sharded search (xchg: int64[7] device pointer) ----
    def shard_vote(self, grid: Grid, r_begin, r_count, xchg_ptr, stream=None):
        check(self._L.dses_shard_vote(self._h, ctypes.byref(grid), int(r_begin), int(r_count),
                                      xchg_ptr, stream), "dses_shard_vote")

    def shard_select(self, q, code, param, skip_refine, xchg_ptr, stream=None):
        check(self._L.dses_shard_select(self._h, float(q), int(code), float(param),
                                        int(bool(skip_refine)), xchg_ptr, stream),
              "dses_shard_select")

    def shard_key(self, xchg_ptr, stream=None):
        check(self._L.dses_shard_key(self._h, xchg_ptr, stream), "dses_shard_key")

    def shard_miss(self, xchg_ptr, stream=None):
        check(self._L.dses_shard_miss(self._h, xchg_ptr, stream), "dses_shard_miss")

    def pose_error(self, grid: Grid, row, lin, code, param, stream=None):
        e = ctypes.c_double()
        check(self._L.dses_pose_error(self._h, ctypes.byref(grid), int(row), int(lin), int(code),
                                      float(param), ctypes.byref(e), stream), "dses_pose_error")
        return e.value

    def traffic(self, reset=False):
        v = [ctypes.c_int64() for _ in range(3)]
        check(self._L.dses_plan_traffic(self._h, *[ctypes.byref(a) for a in v], int(reset)),
              "dses_plan_traffic")
        return {"h2d_bytes": v[0].value, "d2h_bytes": v[1].value, "launches": v[2].value}

    def stats(self):
        v = [ctypes.c_int64() for _ in range(3)]
        check(self._L.dses_stage_stats(self._h, *[ctypes.byref(a) for a in v]), "dses_stage_stats")
        return {"pairs": v[0].value, "votes": v[1].value, "rechecks": v[2].value}
