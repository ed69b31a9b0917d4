"""Seeded synthetic registration pairs shaped like the paper's ModelNet40
protocol (section V-A; reference generator gridreg/benchgen.py:344-367).

Not a copy of the reference generator: an independent implementation of the
same protocol, used by bench.py on the GPU box (where the reference is absent).

  1. a closed bumpy surface (star-shaped radial function, area-weighted
     rejection sampling), centred and scaled to max point norm 1;
  2. reference and source drawn as independent subsets of one surface pool
     (partial correspondence, like two scans of one object);
  3. a random aligner (Euler angles uniform in +-rot_range, translation
     uniform in +-trans_range); the source is moved by its inverse;
  4. clipped Gaussian jitter on both clouds;
  5. half-space crop of the source keeping round(keep * N) points;
  6. optional outlier replacement (config 3: a fraction of source rows
     replaced by uniform samples in the source bounding box).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .geometry import RigidTransform, rotation_from_euler


@dataclass(frozen=True)
class PairSpec:
    pool: int = 2048
    n_reference: int = 1024
    n_source: int = 1024
    keep: float = 0.7
    rot_range_deg: float = 45.0
    trans_range: float = 0.5
    noise_sigma: float = 0.01
    noise_clip: float = 0.05
    outlier_frac: float = 0.0
    shape: str = "blob"


def _bumpy_surface(rng, n, lobes=7):
    dirs = rng.standard_normal((lobes, 3))
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    amp = rng.uniform(0.08, 0.3, lobes)
    kappa = rng.uniform(2.0, 7.0, lobes)

    def radius(u):
        return 1.0 + (amp * np.exp(kappa * (u @ dirs.T - 1.0))).sum(axis=1)

    rmax = 1.0 + amp.sum()
    out = []
    have = 0
    while have < n:
        u = rng.standard_normal((4 * n, 3))
        u /= np.linalg.norm(u, axis=1, keepdims=True)
        r = radius(u)
        # area weight ~ r^2 (ignores the slope term; fine for a benchmark shape)
        keep = rng.random(u.shape[0]) * rmax * rmax < r * r
        pts = r[keep, None] * u[keep]
        out.append(pts)
        have += pts.shape[0]
    return np.concatenate(out)[:n]


def _bracket_surface(rng, n):
    """L-shaped plate pair sampled on its faces (config 4 stand-in for a CAD part)."""
    faces = [((0, 0, 0), (1.0, 0, 0), (0, 0.4, 0)), ((0, 0.4, 0), (0.4, 0, 0), (0, 0.6, 0)),
             ((0, 0, 0.3), (1.0, 0, 0), (0, 0.4, 0)), ((0, 0.4, 0.3), (0.4, 0, 0), (0, 0.6, 0)),
             ((0, 0, 0), (1.0, 0, 0), (0, 0, 0.3)), ((1.0, 0, 0), (0, 0.4, 0), (0, 0, 0.3)),
             ((0.4, 0.4, 0), (0.6, 0, 0), (0, 0, 0.3)), ((0.4, 0.4, 0), (0, 0.6, 0), (0, 0, 0.3)),
             ((0, 1.0, 0), (0.4, 0, 0), (0, 0, 0.3)), ((0, 0, 0), (0, 1.0, 0), (0, 0, 0.3))]
    o = np.array([f[0] for f in faces], dtype=float)
    a = np.array([f[1] for f in faces], dtype=float)
    b = np.array([f[2] for f in faces], dtype=float)
    area = np.linalg.norm(np.cross(a, b), axis=1)
    face = rng.choice(len(faces), size=n, p=area / area.sum())
    st = rng.random((n, 2))
    return o[face] + st[:, :1] * a[face] + st[:, 1:] * b[face]


def make_pair(spec: PairSpec, seed: int):
    """Returns (source, reference, gt_aligner) with source ~ keep * n_source points."""
    rng = np.random.default_rng(np.random.SeedSequence([0xD5E5, int(seed)]))
    if spec.shape == "bracket":
        pool = _bracket_surface(rng, spec.pool)
    else:
        pool = _bumpy_surface(rng, spec.pool)
    pool = pool - pool.mean(axis=0)
    pool /= np.linalg.norm(pool, axis=1).max()
    ref = pool[rng.choice(spec.pool, spec.n_reference, replace=False)]
    src = pool[rng.choice(spec.pool, spec.n_source, replace=False)]
    r = math.radians(spec.rot_range_deg)
    aligner = RigidTransform(rotation_from_euler(rng.uniform(-r, r, 3)),
                             rng.uniform(-spec.trans_range, spec.trans_range, 3))
    inv = aligner.inverse()
    src = src @ inv.rotation.T + inv.translation

    def jit(p):
        return p + np.clip(rng.normal(0.0, spec.noise_sigma, p.shape), -spec.noise_clip,
                           spec.noise_clip)

    ref, src = jit(ref), jit(src)
    k = min(max(int(math.floor(spec.keep * src.shape[0] + 0.5)), 1), src.shape[0])
    d = rng.standard_normal(3)
    d /= np.linalg.norm(d)
    src = src[np.sort(np.argsort(src @ d, kind="stable")[:k])]
    if spec.outlier_frac > 0:
        m = int(round(spec.outlier_frac * src.shape[0]))
        rows = np.sort(rng.choice(src.shape[0], m, replace=False))
        src = src.copy()
        src[rows] = rng.uniform(src.min(axis=0), src.max(axis=0), (m, 3))
    return np.ascontiguousarray(src), np.ascontiguousarray(ref), aligner


# the BASELINE.json configurations
CONFIGS = {
    "c1": dict(spec=PairSpec(keep=0.5), k_rot=5, rot_step_deg=9.0, k_trans=20, trans_bin=0.025,
               metric="inliers"),
    "c2": dict(spec=PairSpec(), k_rot=15, rot_step_deg=3.0, k_trans=20, trans_bin=0.025,
               metric="trunc-l1"),
    "c3": dict(spec=PairSpec(noise_sigma=0.02, outlier_frac=0.2), k_rot=45, rot_step_deg=1.0,
               k_trans=20, trans_bin=0.025, metric="l1"),
    "c4": dict(spec=PairSpec(pool=40000, n_reference=20000, n_source=7143, rot_range_deg=5.0,
                             trans_range=0.016, noise_sigma=0.002, noise_clip=0.01,
                             shape="bracket"),
               k_rot=10, rot_step_deg=0.5, k_trans=4, trans_bin=0.004, metric="trunc-l1"),
}

# local-regime variant (k_rot=7 around identity, L1 -- a flat
# histogram where ~97% of the rotations pass the q*M* cutoff: scoring-heavy)
CONFIGS["c2local"] = dict(spec=PairSpec(rot_range_deg=120.0), k_rot=7, rot_step_deg=3.0, k_trans=20,
                          trans_bin=0.025, metric="l1")
CONFIGS["c2l2"] = dict(spec=PairSpec(rot_range_deg=120.0), k_rot=7, rot_step_deg=3.0, k_trans=20,
                       trans_bin=0.025, metric="l2")
