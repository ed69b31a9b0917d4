"""Rotation-block vote kernel (-m gpu): per-rotation (count, bin, ties)
identical to the per-rotation kernel and to the pinned oracle.

The block kernel (csrc/dses_vote.cu, vote_blocks_kernel) builds one
candidate-pair list per run of consecutive rotations of a grid row with the
window widened by the run's maximal point motion, and votes it per rotation
with a lane-per-entry dedup; these tests cover what can differ from the
per-rotation path: block boundaries against rotation ranges and short rows,
the widening bound at large steps, dedup components (shuffle dedup within a
list segment, partnered pairs next to guard-band pairs, components split over
groups), the list-overflow fallback, centre rotations, and the dses() result.
"""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _plan_modes(x, y, b, ilo, dims, k, step, center=None, r_begin=0, r_count=None, L=5, cap=0):
    """(per-rotation kernel, block kernel) modes; the block kernel is run with
    the shape L (an int n = a 1 x 1 x n run) and with 1 x 3 x 3 and 3 x 3 x 3
    boxes, which must all agree."""
    from oracle import oracle as O
    from paper_2502_00115_b200 import _native
    c, s = O.trig_tables(k, step)
    g = _native.make_grid(k, c, s, center)
    n = (2 * k + 1) ** 3 if r_count is None else r_count
    with _native.Plan(x, y, b, ilo, dims) as plan:
        plan.set_blocks(0)
        ref = plan.mode_grid(g, r_begin, n)
        got = None
        for shape in (L, (1, 3, 3), (3, 3, 3)):
            plan.set_blocks(shape, cap)
            out = plan.mode_grid(g, r_begin, n)
            assert got is None or _same(got, out), shape
            got = out
    return ref, got


def _same(a, b):
    return all(np.array_equal(u, v) for u, v in zip(a, b))


@pytest.mark.parametrize("name,Ls", [("c4", (1, 7, (1, 3, 3), (2, 3, 3), (3, 3, 3))),
                                     ("c2", (1, 3, (1, 3, 3)))])
def test_blocks_equal_per_rotation_kernel_full_grid(name, Ls):
    import bench
    from paper_2502_00115_b200 import _native
    from paper_2502_00115_b200.engines import prepare
    cfg = bench.search_config(bench.workload(name))
    (x, y, _), = bench.bench_pairs(name, 1)[0]
    p = prepare(x, y, cfg)
    g = _native.make_grid(cfg.k_rot, p.cos_tab, p.sin_tab, p.center_rot)
    R = cfg.rotation_count
    with _native.Plan(p.x, p.y, cfg.trans_bin, p.ilo, p.dims) as plan:
        plan.set_blocks(0)
        ref = plan.mode_grid(g, 0, R)
        for L in Ls:
            plan.set_blocks(L)
            assert _same(ref, plan.mode_grid(g, 0, R)), L
        # ranges that start and end inside grid rows, and single rotations
        for r0, n in ((7, 50), (R // 2 + 3, 1), (R - 40, 40), (2 * cfg.k_rot + 2, 1000)):
            plan.set_blocks(0)
            a = plan.mode_grid(g, r0, n)
            for shape in ((1, 1, 5), (1, 3, 3), (3, 3, 3)):
                plan.set_blocks(shape)
                assert _same(a, plan.mode_grid(g, r0, n)), (r0, n, shape)


def test_blocks_small_rows_and_large_steps_match_oracle():
    # k = 1: rows of 3 rotations (shorter than a block); 20-degree steps: the
    # widening is large against the window
    from oracle import oracle as O
    rng = np.random.default_rng(31)
    x = rng.normal(size=(300, 3)) * 0.4
    y = rng.normal(size=(500, 3)) * 0.4
    b, ilo, dims = 0.03, np.full(3, -6), np.full(3, 13)
    for k, step in ((1, math.radians(20)), (3, math.radians(4))):
        ref, got = _plan_modes(x, y, b, ilo, dims, k, step, L=5)
        assert _same(ref, got), k
        oc, ol, ot = O.mode_batch(x, y, b, ilo, dims, grid=(k, step, None))
        assert np.array_equal(got[0], oc) and np.array_equal(got[1], ol) and np.array_equal(got[2], ot)


def test_blocks_with_huge_steps_fall_back_to_per_rotation_kernel():
    # 60-degree steps: the motion bound exceeds the block kernel's 2^27-unit
    # widening limit, so every block goes to the per-rotation kernel
    from oracle import oracle as O
    rng = np.random.default_rng(41)
    x = rng.normal(size=(200, 3)) * 0.5
    y = rng.normal(size=(300, 3)) * 0.5
    b, ilo, dims = 0.05, np.full(3, -3), np.full(3, 7)
    k, step = 1, math.radians(60)
    ref, got = _plan_modes(x, y, b, ilo, dims, k, step, L=(1, 3, 3))
    assert _same(ref, got)
    oc, ol, ot = O.mode_batch(x, y, b, ilo, dims, grid=(k, step, None))
    assert np.array_equal(got[0], oc) and np.array_equal(got[1], ol) and np.array_equal(got[2], ot)


def test_blocks_dedup_components_and_exact_path_match_oracle():
    # clusters of 1-7 points within a fraction of a bin (components of every
    # size, partners in the guard band), one cluster of 40 points (a component
    # split over groups: always exact), exact duplicates
    from oracle import oracle as O
    rng = np.random.default_rng(5)
    centres = rng.normal(size=(60, 3)) * 0.3
    y = np.concatenate([c + rng.normal(size=(rng.integers(1, 8), 3)) * 0.004 for c in centres])
    y = np.concatenate([y, centres[0] + rng.normal(size=(40, 3)) * 0.002, y[:10]])
    x = rng.normal(size=(200, 3)) * 0.3
    b, ilo, dims = 0.02, np.full(3, -5), np.full(3, 11)
    k, step = 4, math.radians(2)
    ref, got = _plan_modes(x, y, b, ilo, dims, k, step, L=5)
    assert _same(ref, got)
    oc, ol, ot = O.mode_batch(x, y, b, ilo, dims, grid=(k, step, None))
    assert np.array_equal(got[0], oc) and np.array_equal(got[1], ol) and np.array_equal(got[2], ot)
    assert got[0].max() > 1


def test_blocks_list_overflow_falls_back_to_per_rotation_kernel():
    rng = np.random.default_rng(8)
    x = rng.normal(size=(256, 3)) * 0.3
    y = rng.normal(size=(700, 3)) * 0.3
    b, ilo, dims = 0.02, np.full(3, -4), np.full(3, 9)
    for cap in (32, 2048):  # every block / some blocks overflow
        ref, got = _plan_modes(x, y, b, ilo, dims, 3, math.radians(3), L=5, cap=cap)
        assert _same(ref, got), cap


def test_blocks_with_centre_rotation():
    from oracle import oracle as O
    rng = np.random.default_rng(12)
    x = rng.normal(size=(150, 3)) * 0.3
    y = rng.normal(size=(400, 3)) * 0.3
    b, ilo, dims = 0.025, np.full(3, -5), np.full(3, 11)
    a = 0.7
    cen = np.array([[math.cos(a), -math.sin(a), 0.0], [math.sin(a), math.cos(a), 0.0], [0.0, 0.0, 1.0]])
    k, step = 3, math.radians(5)
    ref, got = _plan_modes(x, y, b, ilo, dims, k, step, center=cen, L=3)
    assert _same(ref, got)
    oc, ol, ot = O.mode_batch(x, y, b, ilo, dims, grid=(k, step, cen))
    assert np.array_equal(got[0], oc) and np.array_equal(got[1], ol) and np.array_equal(got[2], ot)


def test_dses_on_c4_uses_blocks_and_matches_per_rotation_kernel():
    """The default plan for c4 (a 36 mm window in a 1.4 m cloud) takes the
    block kernel; the full registration equals the per-rotation kernel's."""
    import bench
    from paper_2502_00115_b200 import _native
    from paper_2502_00115_b200.engines import prepare
    cfg = bench.search_config(bench.workload("c4"))
    (x, y, _), = bench.bench_pairs("c4", 1)[0]
    p = prepare(x, y, cfg)
    g = _native.make_grid(cfg.k_rot, p.cos_tab, p.sin_tab, p.center_rot)
    out = []
    with _native.Plan(p.x, p.y, cfg.trans_bin, p.ilo, p.dims) as plan:
        for L in (None, 0):
            if L is not None:
                plan.set_blocks(L)
            r = plan.search(g, cfg.q, p.code, p.param, p.skip_refine)
            out.append({k: r[k] for k in ("winner_row", "winner_lin", "winner_count", "best_error", "mstar",
                                          "candidates_evaluated", "candidates_refined", "best_inliers",
                                          "pairs_evaluated")})
    pairs = [o.pop("pairs_evaluated") for o in out]
    assert out[0] == out[1]
    # the block kernel's statistic is list entries per rotation, well below
    # the per-rotation kernel's evaluated pairs
    assert pairs[0] < pairs[1] / 2


@pytest.mark.parametrize("kind,param", [("trunc_l1", 0.02), ("l1", None), ("inliers", 0.01),
                                        ("l2", None)])
def test_dses_small_window_every_metric_matches_oracle(kind, param):
    """The full registration on the default path for a small window (the
    rotation-block kernel) against the oracle dses, for each scoring path."""
    import paper_2502_00115_b200 as api
    from oracle import oracle as O
    from paper_2502_00115_b200 import _native
    from paper_2502_00115_b200.engines import prepare
    from paper_2502_00115_b200.synth import CONFIGS, make_pair
    x, y, _ = make_pair(CONFIGS["c2"]["spec"], 23)
    cfg = api.SearchConfig(k_rot=3, rot_step=math.radians(3), k_trans=3, trans_bin=0.01,
                           metric=api.ErrorMetric.from_name(kind, param) if param is not None
                           else api.ErrorMetric(kind))
    p = prepare(x, y, cfg)
    with _native.Plan(p.x, p.y, cfg.trans_bin, p.ilo, p.dims) as plan:
        assert plan.blocks()[0] > 0, "a small window takes the rotation-block kernel"
    res = api.dses(x, y, cfg)
    m = cfg.metric
    ref = O.dses(x, y, k_rot=cfg.k_rot, rot_step=cfg.rot_step, k_trans=cfg.k_trans,
                 trans_bin=cfg.trans_bin, q=cfg.q, metric=(m.kind, m.param))
    assert tuple(res.best.grid_coords) == tuple(ref["grid_coords"])
    assert np.array_equal(res.best.translation, ref["translation"])
    assert math.isclose(res.best_error, ref["best_error"], rel_tol=1e-9, abs_tol=1e-12)
    assert res.candidates_evaluated == ref["candidates_evaluated"]
    assert res.candidates_refined == ref["candidates_refined"]
    assert res.best_inliers == ref["best_inliers"]
