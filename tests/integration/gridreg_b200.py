"""The reference-side ctypes binding of INTEGRATION.md ("gridreg/_b200.py"),
verbatim apart from the library path: what a gridreg maintainer adds to route
the numba seams _kernels.mode_dense_batch (_kernels.py:173-193) and
_kernels.sweep_inlier_best (_kernels.py:384-410) to libdses_b200.so.

It deliberately does NOT use the repo's own Python package: tests drive it
with exactly the arrays the reference's _mode_batch hands its kernel
(mode_search.py:132-164), so the documented drop-in binding is exercised.
"""
import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_DEFAULT = os.path.join(_HERE, "..", "..", "paper_2502_00115_b200", "_lib", "libdses_b200.so")
_L = ctypes.CDLL(os.environ.get("GRIDREG_B200_LIB", _DEFAULT))
_dp, _ip = ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int64)
_L.dses_mode_dense_batch.argtypes = [ctypes.c_int, _dp, ctypes.c_int64, _dp, ctypes.c_int64,
                                     _dp, ctypes.c_int64, ctypes.c_double, _ip, _ip, _ip, _ip, _ip]
_L.dses_last_error.restype = ctypes.c_char_p


class InvalidInputError(ValueError):
    """Stand-in for gridreg.errors.InvalidInputError (a ValueError)."""


def _check(rc):
    if rc == -1:
        raise InvalidInputError(_L.dses_last_error().decode())
    if rc != 0:
        raise RuntimeError(_L.dses_last_error().decode())


def mode_dense_batch(rots, x, y, bin_size, ilo, dims, counts_out, lins_out, ties_out):
    """Same outputs as _kernels.mode_dense_batch (y unsorted, (m, 3))."""
    f = lambda a, t: np.ascontiguousarray(a, dtype=t)  # noqa: E731
    rots, x, y = f(rots, np.float64), f(x, np.float64), f(y, np.float64)
    ilo, dims = f(ilo, np.int64), f(dims, np.int64)
    _check(_L.dses_mode_dense_batch(
        0, rots.ctypes.data_as(_dp), rots.shape[0], x.ctypes.data_as(_dp), x.shape[0],
        y.ctypes.data_as(_dp), y.shape[0], float(bin_size), ilo.ctypes.data_as(_ip),
        dims.ctypes.data_as(_ip), counts_out.ctypes.data_as(_ip),
        lins_out.ctypes.data_as(_ip), ties_out.ctypes.data_as(_ip)))


def sweep_inlier_best(cands, n, m, half, t0vals, t1vals, t2vals):
    """Same result as _kernels.sweep_inlier_best (harness.run_oracle_checks)."""
    f = lambda a: np.ascontiguousarray(a, dtype=np.float64)  # noqa: E731
    c, a0, a1, a2 = f(cands), f(t0vals), f(t1vals), f(t2vals)
    best = ctypes.c_int64()
    _check(_L.dses_sweep_inlier_best(
        0, c.ctypes.data_as(_dp), ctypes.c_int64(n), ctypes.c_int64(m), ctypes.c_double(half),
        a0.ctypes.data_as(_dp), ctypes.c_int64(a0.size), a1.ctypes.data_as(_dp),
        ctypes.c_int64(a1.size), a2.ctypes.data_as(_dp), ctypes.c_int64(a2.size),
        ctypes.byref(best)))
    return best.value
