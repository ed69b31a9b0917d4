"""Translation lattice helpers and the single-rotation mode API.

Drop-in for gridreg/mode_search.py: ``bin_index``/``bin_center`` (40-54),
``_decode_flat`` (167-171), the window helpers (101-129), ``ModeResult`` and
``mode_translation`` (174-202), ``TranslationHistogram`` /
``translation_histogram`` (74-99, 205-235).  The mode runs on the B200 vote
kernel (csrc/dses_vote.cu) for any lattice size: dense shared-memory
histograms when they fit, per-CTA global-memory histograms beyond that, the
sort-based path (csrc/dses_sparse.cu, the reference's sparse algorithm
_kernels.py:196-294) for huge lattices; the full vote map is the sort-based
path's run-length encoding.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import InvalidInputError, NoCandidateError
from .geometry import as_point_cloud, check_rotation

KEY_SPACE_LIMIT = 1 << 62  # mode_search.py:38


def bin_index(v, bin_size: float) -> np.ndarray:
    """Round-half-away-from-zero of v / bin_size per axis (int64)."""
    if not (bin_size > 0) or not np.isfinite(bin_size):
        raise InvalidInputError("bin_size must be positive and finite")
    a = np.asarray(v, dtype=np.float64)
    if not np.isfinite(a).all():
        raise InvalidInputError("translation values must be finite")
    q = a * (1.0 / bin_size)
    return np.copysign(np.floor(np.fabs(q) + 0.5), q).astype(np.int64)


def bin_center(index, bin_size: float) -> np.ndarray:
    return np.asarray(index, dtype=np.float64) * float(bin_size)


def decode_flat(lin: int, ilo, dims):
    """Flat bin -> integer bin index triple (mode_search.py:167-171)."""
    d12 = int(dims[1]) * int(dims[2])
    a, rem = divmod(int(lin), d12)
    b, c = divmod(rem, int(dims[2]))
    return (a + int(ilo[0]), b + int(ilo[1]), c + int(ilo[2]))


_decode_flat = decode_flat


@dataclass(frozen=True)
class ModeResult:
    t_star: np.ndarray
    count: int
    num_tied_bins: int
    index: tuple

    def __post_init__(self):
        t = np.asarray(self.t_star, dtype=np.float64).copy()
        t.flags.writeable = False
        object.__setattr__(self, "t_star", t)
        object.__setattr__(self, "index", tuple(int(i) for i in self.index))


def bounds_to_index_range(t_bounds, bin_size: float):
    """Inclusive bin-index range whose centres lie in [lo, hi] (mode_search.py:101-118)."""
    tb = np.asarray(t_bounds, dtype=np.float64)
    if tb.shape != (2, 3) or not np.isfinite(tb).all():
        raise InvalidInputError("t_bounds must be a finite (2, 3) array [lo; hi]")
    if np.any(tb[1] < tb[0]):
        raise InvalidInputError("t_bounds upper limits below lower limits")
    r_lo, r_hi = tb[0] / bin_size, tb[1] / bin_size
    ilo = np.ceil(r_lo - 1e-9 * np.maximum(1.0, np.abs(r_lo))).astype(np.int64)
    ihi = np.floor(r_hi + 1e-9 * np.maximum(1.0, np.abs(r_hi))).astype(np.int64)
    if np.any(ihi < ilo):
        raise NoCandidateError("t_bounds contain no bin center on some axis")
    return ilo, ihi


def data_index_range(x, y, bin_size: float):
    """Index range holding every y_j - R x_i for any R (mode_search.py:121-129)."""
    xmax = float(np.linalg.norm(x, axis=1).max())
    ilo = bin_index(y.min(axis=0) - xmax, bin_size) - 1
    ihi = bin_index(y.max(axis=0) + xmax, bin_size) + 1
    return ilo, ihi


def check_key_space(nbins: int, n: int):
    """The reference's lattice guard (mode_search.py:149-152)."""
    if nbins * max(n, 1) >= KEY_SPACE_LIMIT:
        raise InvalidInputError("translation lattice too large; pass t_bounds or a larger bin_size")


def mode_translation(source, reference, rotation, bin_size: float, t_bounds=None,
                     device: int = 0) -> ModeResult:
    """Most-voted lattice translation for one rotation (mode_search.py:174-202)."""
    from . import _native

    x = as_point_cloud(source)
    y = as_point_cloud(reference)
    rot = np.asarray(rotation, dtype=np.float64)
    check_rotation(rot)
    if not (bin_size > 0) or not np.isfinite(bin_size):
        raise InvalidInputError("bin_size must be positive and finite")
    if t_bounds is None:
        ilo, ihi = data_index_range(x, y, bin_size)
    else:
        ilo, ihi = bounds_to_index_range(t_bounds, bin_size)
    dims = ihi - ilo + 1
    check_key_space(int(np.prod(dims.astype(object))), x.shape[0])
    with _native.Plan(x, y, bin_size, ilo, dims, device) as plan:
        counts, lins, ties = plan.mode_batch(rot.reshape(1, 9))
    if counts[0] <= 0:
        raise NoCandidateError("no translation candidate inside t_bounds")
    idx = decode_flat(lins[0], ilo, dims)
    return ModeResult(t_star=bin_center(idx, bin_size), count=int(counts[0]),
                      num_tied_bins=int(ties[0]), index=idx)


@dataclass(frozen=True)
class TranslationHistogram:
    """Sparse vote map {bin index triple: count} (mode_search.py:74-99);
    counts are distinct source points per bin with dedup, raw pair votes
    without (then total = N*M when unbounded)."""
    bin_size: float
    counts: dict
    total: int
    dedup: bool

    def mode(self) -> ModeResult:
        if not self.counts:
            raise NoCandidateError("histogram is empty")
        best = max(self.counts.values())
        tied = sorted(k for k, c in self.counts.items() if c == best)
        return ModeResult(t_star=bin_center(tied[0], self.bin_size), count=int(best),
                          num_tied_bins=len(tied), index=tied[0])


def translation_histogram(source, reference, rotation, bin_size: float, t_bounds=None,
                          dedup: bool = True, device: int = 0) -> TranslationHistogram:
    """Full vote map of one rotation on the GPU (mode_search.py:205-235): every
    pair's bin (binary64, the vote kernel's operation order) inside the
    lattice -- t_bounds' bins, or all of them -- sorted, deduplicated per
    source when `dedup`, run-length encoded (csrc/dses_sparse.cu)."""
    from . import _native

    x = as_point_cloud(source)
    y = as_point_cloud(reference)
    rot = np.asarray(rotation, dtype=np.float64)
    check_rotation(rot)
    if not (bin_size > 0) or not np.isfinite(bin_size):
        raise InvalidInputError("bin_size must be positive and finite")
    if t_bounds is None:
        ilo, ihi = data_index_range(x, y, bin_size)
    else:
        ilo, ihi = bounds_to_index_range(t_bounds, bin_size)
    dims = ihi - ilo + 1
    check_key_space(int(np.prod(dims.astype(object))), x.shape[0])
    with _native.Plan(x, y, bin_size, ilo, dims, device) as plan:
        lins, counts, _ = plan.histogram(rot.reshape(9), dedup)
    d12 = int(dims[1]) * int(dims[2])
    a, rem = np.divmod(lins, d12)
    b, c = np.divmod(rem, int(dims[2]))
    idx = np.stack([a + ilo[0], b + ilo[1], c + ilo[2]], axis=1)
    table = {(int(i0), int(i1), int(i2)): int(k) for (i0, i1, i2), k in zip(idx.tolist(), counts)}
    return TranslationHistogram(bin_size=float(bin_size), counts=table, total=int(counts.sum()),
                                dedup=bool(dedup))
