"""Point-cloud validation, rigid transforms and the Euler rotation grid.

Drop-in for the parts of gridreg/geometry.py the DSES path touches:
``as_point_cloud`` (geometry.py:52-61), ``as_point3`` (42-49),
``rotation_from_euler`` (117-130), ``euler_from_rotation`` (133-152),
``RigidTransform`` (166-222), ``RotationGrid``/``build_rotation_grid``
(235-290).  Conventions are the reference's: R = Rz(xi) Ry(phi) Rx(theta),
points map by R p + t, clouds are (N, 3) float64 with N >= 1.

The grid itself is never materialised on the hot path: the device kernels
compose each rotation from the per-axis cos/sin tables returned by
``grid_tables`` (see csrc/dses_common.cuh:grid_entry), bit-identically to the
reference's closed form.  ``RotationGrid.matrices`` exists for callers that
want the (R, 3, 3) stack and is computed on demand.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .errors import InvalidInputError

_ORTHO_TOL = 1e-9


def as_point3(p) -> np.ndarray:
    a = np.asarray(p, dtype=np.float64).reshape(-1)
    if a.shape != (3,):
        raise InvalidInputError(f"expected a 3-vector, got shape {np.shape(p)}")
    if not np.isfinite(a).all():
        raise InvalidInputError("point has non-finite components")
    return a


def as_point_cloud(points) -> np.ndarray:
    """(N, 3) float64 C-contiguous copy-or-view with N >= 1 and finite values."""
    a = np.ascontiguousarray(points, dtype=np.float64)
    if a.ndim != 2 or a.shape[1] != 3:
        raise InvalidInputError(f"expected an (N, 3) array, got shape {a.shape}")
    if a.shape[0] < 1:
        raise InvalidInputError("point cloud is empty")
    if not np.isfinite(a).all():
        raise InvalidInputError("point cloud has non-finite values")
    return a


def rotation_from_euler(angles) -> np.ndarray:
    """R = Rz(xi) @ Ry(phi) @ Rx(theta) for (theta, phi, xi) in radians."""
    a = np.asarray(getattr(angles, "as_array", lambda: angles)(), dtype=np.float64).reshape(-1)
    if a.shape != (3,) or not np.isfinite(a).all():
        raise InvalidInputError("expected three finite Euler angles")
    th, ph, xi = (float(v) for v in a)
    ct, st, cp, sp, cx, sx = (math.cos(th), math.sin(th), math.cos(ph), math.sin(ph),
                              math.cos(xi), math.sin(xi))
    rx = np.array([[1.0, 0.0, 0.0], [0.0, ct, -st], [0.0, st, ct]])
    ry = np.array([[cp, 0.0, sp], [0.0, 1.0, 0.0], [-sp, 0.0, cp]])
    rz = np.array([[cx, -sx, 0.0], [sx, cx, 0.0], [0.0, 0.0, 1.0]])
    return rz @ ry @ rx


@dataclass(frozen=True)
class EulerAngles:
    theta: float
    phi: float
    xi: float

    def as_array(self) -> np.ndarray:
        return np.array([self.theta, self.phi, self.xi], dtype=np.float64)


def euler_from_rotation(rotation) -> EulerAngles:
    r = np.asarray(rotation, dtype=np.float64)
    if r.shape != (3, 3):
        raise InvalidInputError("rotation must be a 3x3 matrix")
    sp = min(1.0, max(-1.0, float(-r[2, 0])))
    phi = math.asin(sp)
    if abs(sp) < 1.0 - 1e-12:
        return EulerAngles(math.atan2(r[2, 1], r[2, 2]), phi, math.atan2(r[1, 0], r[0, 0]))
    return EulerAngles(0.0, phi, math.atan2(-r[0, 1], r[1, 1]))


def check_rotation(r: np.ndarray):
    """Orthonormal with det +1 within 1e-9 (geometry.py:155-163)."""
    if r.shape != (3, 3) or not np.isfinite(r).all():
        raise InvalidInputError("rotation must be a finite 3x3 matrix")
    err = float(np.abs(r.T @ r - np.eye(3)).max())
    if err > _ORTHO_TOL:
        raise InvalidInputError(f"matrix is not orthonormal (max |R^T R - I| = {err:.3e})")
    det = float(np.linalg.det(r))
    if abs(det - 1.0) > _ORTHO_TOL:
        raise InvalidInputError(f"matrix is not a proper rotation (det = {det:.12f})")


@dataclass(frozen=True, eq=False)
class RigidTransform:
    """p -> rotation @ p + translation; immutable, arrays read-only."""

    rotation: np.ndarray
    translation: np.ndarray
    grid_coords: tuple | None = None

    def __post_init__(self):
        r = np.array(self.rotation, dtype=np.float64)
        t = as_point3(self.translation).copy()
        check_rotation(r)
        r.flags.writeable = False
        t.flags.writeable = False
        object.__setattr__(self, "rotation", r)
        object.__setattr__(self, "translation", t)
        if self.grid_coords is not None:
            object.__setattr__(self, "grid_coords", tuple(int(c) for c in self.grid_coords))

    @classmethod
    def identity(cls) -> "RigidTransform":
        return cls(np.eye(3), np.zeros(3))

    @classmethod
    def from_euler(cls, angles, translation=(0.0, 0.0, 0.0)) -> "RigidTransform":
        return cls(rotation_from_euler(angles), translation)

    def inverse(self) -> "RigidTransform":
        rt = self.rotation.T.copy()
        return RigidTransform(rt, -(rt @ self.translation))

    def compose(self, other: "RigidTransform") -> "RigidTransform":
        return RigidTransform(self.rotation @ other.rotation,
                              self.rotation @ other.translation + self.translation)

    def apply(self, points) -> np.ndarray:
        return as_point_cloud(points) @ self.rotation.T + self.translation

    def euler(self) -> EulerAngles:
        return euler_from_rotation(self.rotation)

    def __eq__(self, other):
        if not isinstance(other, RigidTransform):
            return NotImplemented
        return (np.array_equal(self.rotation, other.rotation)
                and np.array_equal(self.translation, other.translation))


def apply_transform(transform: RigidTransform, points) -> np.ndarray:
    return transform.apply(points)


def compose(a: RigidTransform, b: RigidTransform) -> RigidTransform:
    """a after b (geometry.py:225-227)."""
    return a.compose(b)


def wrap_angle(a):
    """Angles wrapped to [-pi, pi) (geometry.py:80-82)."""
    return (np.asarray(a) + np.pi) % (2.0 * np.pi) - np.pi


def random_rotation(rng: np.random.Generator) -> np.ndarray:
    """Uniformly distributed rotation from a normalised Gaussian quaternion
    (geometry.py:307-318; same draws, same matrix)."""
    q = rng.standard_normal(4)
    w, a, b, c = q / np.linalg.norm(q)
    return np.array([[1 - 2 * (b * b + c * c), 2 * (a * b - w * c), 2 * (a * c + w * b)],
                     [2 * (a * b + w * c), 1 - 2 * (a * a + c * c), 2 * (b * c - w * a)],
                     [2 * (a * c - w * b), 2 * (b * c + w * a), 1 - 2 * (a * a + b * b)]])


def check_grid_args(half_width, step):
    """Validation of build_rotation_grid (geometry.py:259-267)."""
    k = int(half_width)
    if k != half_width or k < 0:
        raise InvalidInputError("half_width must be a non-negative integer")
    if not (step > 0.0) or not math.isfinite(step):
        raise InvalidInputError("step must be positive and finite")
    if k * step > math.pi + 1e-12:
        raise InvalidInputError(
            f"rotation grid wraps: half_width*step = {k * step:.6f} rad exceeds pi")
    return k, float(step)


def grid_tables(half_width: int, step: float):
    """Per-axis (cos, sin) of angles idx*step, idx = -k..k.

    geometry.py:272-275 applies np.cos / np.sin to idx.astype(float64) * step;
    evaluating numpy's ufuncs on the 2k+1 distinct angles yields the same
    binary64 values (checked bit-for-bit in tests/test_host.py), and the
    device composes the closed form from them in numpy's operation order.
    """
    k, step = check_grid_args(half_width, step)
    ang = np.arange(-k, k + 1, dtype=np.int64).astype(np.float64) * step
    return np.ascontiguousarray(np.cos(ang)), np.ascontiguousarray(np.sin(ang))


def grid_rotation(cos_tab, sin_tab, k: int, r: int, center=None) -> np.ndarray:
    """Rotation r of the grid on the host, same operations as the device."""
    n = 2 * k + 1
    a, b, c = r // (n * n), (r // n) % n, r % n
    c1, s1 = float(cos_tab[a]), float(sin_tab[a])
    c2, s2 = float(cos_tab[b]), float(sin_tab[b])
    c3, s3 = float(cos_tab[c]), float(sin_tab[c])
    g = np.array([
        [c3 * c2, (-s3) * c1 + (c3 * s2) * s1, s3 * s1 + (c3 * s2) * c1],
        [s3 * c2, c3 * c1 + (s3 * s2) * s1, (-c3) * s1 + (s3 * s2) * c1],
        [-s2, c2 * s1, c2 * c1],
    ])
    if center is None:
        return g
    cr = np.asarray(center, dtype=np.float64)
    out = np.empty((3, 3))
    for i in range(3):
        for j in range(3):
            out[i, j] = (float(cr[i, 0]) * g[0, j] + float(cr[i, 1]) * g[1, j]) + float(cr[i, 2]) * g[2, j]
    return out


def grid_index(k: int, r) -> np.ndarray:
    """Lexicographic (theta, phi, xi) index triple of flat grid row r."""
    n = 2 * k + 1
    r = np.asarray(r, dtype=np.int64)
    return np.stack([r // (n * n) - k, (r // n) % n - k, r % n - k], axis=-1)


@dataclass(frozen=True)
class RotationGrid:
    """All rotations with Euler angles in {-k*step .. k*step}^3, lexicographic."""

    half_width: int
    step: float
    cos_tab: np.ndarray = field(repr=False)
    sin_tab: np.ndarray = field(repr=False)

    def __len__(self):
        return (2 * self.half_width + 1) ** 3

    @property
    def indices(self) -> np.ndarray:
        return grid_index(self.half_width, np.arange(len(self)))

    @property
    def matrices(self) -> np.ndarray:
        """(R, 3, 3) stack in the reference's closed form (geometry.py:279-287)."""
        k = self.half_width
        n = 2 * k + 1
        idx = self.indices + k
        c1, s1 = self.cos_tab[idx[:, 0]], self.sin_tab[idx[:, 0]]
        c2, s2 = self.cos_tab[idx[:, 1]], self.sin_tab[idx[:, 1]]
        c3, s3 = self.cos_tab[idx[:, 2]], self.sin_tab[idx[:, 2]]
        m = np.empty((n ** 3, 3, 3))
        m[:, 0, 0] = c3 * c2
        m[:, 0, 1] = -s3 * c1 + c3 * s2 * s1
        m[:, 0, 2] = s3 * s1 + c3 * s2 * c1
        m[:, 1, 0] = s3 * c2
        m[:, 1, 1] = c3 * c1 + s3 * s2 * s1
        m[:, 1, 2] = -c3 * s1 + s3 * s2 * c1
        m[:, 2, 0] = -s2
        m[:, 2, 1] = c2 * s1
        m[:, 2, 2] = c2 * c1
        m.flags.writeable = False
        return m


def build_rotation_grid(half_width: int, step: float) -> RotationGrid:
    k, step = check_grid_args(half_width, step)
    c, s = grid_tables(k, step)
    c.flags.writeable = False
    s.flags.writeable = False
    return RotationGrid(half_width=k, step=step, cos_tab=c, sin_tab=s)


def rotation_geodesic_angle(rot_a, rot_b) -> float:
    """Geodesic angle in degrees (geometry.py:293-304)."""
    ra, rb = np.asarray(rot_a, dtype=np.float64), np.asarray(rot_b, dtype=np.float64)
    if ra.shape != (3, 3) or rb.shape != (3, 3):
        raise InvalidInputError("rotation matrices must be 3x3")
    c = min(1.0, max(-1.0, (float(np.trace(ra.T @ rb)) - 1.0) / 2.0))
    return math.degrees(math.acos(c))
