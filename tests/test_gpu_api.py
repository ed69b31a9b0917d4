"""Public API on the B200 (-m gpu): the reference's worked answers, error
behaviour, and edge cases of the vote kernel, each checked against the pinned
oracle or the reference's known answers (restated from the reference's
tests/test_mode_search.py:115-267 and tests/test_engines.py:248-318).

Edge cases exercised here that the golden configs do not reach:
* single-point and ragged clouds (partial warps / units);
* duplicated and clustered reference points (dedup components of 3+ points,
  "far" points, undecided partners -> the exact binary64 path);
* a lattice too large for shared memory (global-memory histograms, 32-bit
  counts: the reference's sparse path);
* coordinates too large for the fixed-point range (exact mode);
* non-cubic windows (mode_translation with t_bounds);
* full-size properties: rotation-range sharding gives identical results,
  repeated runs are bit-identical.
"""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api():
    import paper_2502_00115_b200 as api
    from paper_2502_00115_b200 import _native
    if _native.device_count() < 1:
        pytest.fail("no CUDA device visible to the extension")
    return api


# ---- mode_translation: reference worked examples -------------------------

def test_mode_single_pair(api):
    res = api.mode_translation([[0.0, 0.0, 0.0]], [[1.0, 2.0, 3.0]], np.eye(3), 0.5)
    assert res.index == (2, 4, 6) and res.count == 1
    assert np.array_equal(res.t_star, [1.0, 2.0, 3.0])


def test_mode_cube_corners(api):
    c = np.array([[i, j, k] for i in (0.0, 1.0) for j in (0.0, 1.0) for k in (0.0, 1.0)])
    res = api.mode_translation(c, c, np.eye(3), 0.1)
    assert res.count == 8 and res.num_tied_bins == 1
    assert np.array_equal(res.t_star, [0.0, 0.0, 0.0])


def test_mode_lex_tiebreak(api):
    res = api.mode_translation([[0.0, 0.0, 0.0]], [[1.0, 0.0, 0.0], [0.0, 1.0, 0.0]],
                               np.eye(3), 0.5)
    assert res.num_tied_bins == 2 and res.index == (0, 2, 0)


def test_mode_rotation_applied(api):
    rot = api.rotation_from_euler((0.0, 0.0, math.pi / 2))
    res = api.mode_translation([[1.0, 0.0, 0.0]], [[0.0, 1.0, 0.5]], rot, 0.25)
    assert np.allclose(res.t_star, [0.0, 0.0, 0.5], atol=1e-12)


def test_mode_dedup_counts_source_once(api):
    res = api.mode_translation([[0.0, 0.0, 0.0]], [[1.0, 0.0, 0.0], [1.01, 0.0, 0.0]],
                               np.eye(3), 0.1)
    assert res.count == 1


def test_mode_bounds(api):
    res = api.mode_translation([[0.0, 0.0, 0.0]], [[0.5, 0.0, 0.0]], np.eye(3), 0.25,
                               t_bounds=[[0.5, 0.0, 0.0], [0.5, 0.0, 0.0]])
    assert res.index == (2, 0, 0)
    with pytest.raises(api.NoCandidateError):
        api.mode_translation([[0.0, 0.0, 0.0]], [[0.0, 0.0, 0.0]], np.eye(3), 0.1,
                             t_bounds=[[5.0, 5.0, 5.0], [6.0, 6.0, 6.0]])
    with pytest.raises(api.NoCandidateError):
        api.mode_translation([[0.0, 0.0, 0.0]], [[0.0, 0.0, 0.0]], np.eye(3), 1.0,
                             t_bounds=[[0.2, 0.2, 0.2], [0.4, 0.4, 0.4]])
    with pytest.raises(api.InvalidInputError):
        api.mode_translation([[0.0, 0.0, 0.0]], [[0.0, 0.0, 0.0]], np.eye(3), 0.1,
                             t_bounds=[[1.0, 0.0, 0.0], [0.0, 1.0, 1.0]])


# ---- dses: reference known answers ----------------------------------------

def test_dses_self_registration(api):
    rng = np.random.default_rng(11)
    x = rng.uniform(-1, 1, (60, 3))
    cfg = api.SearchConfig(k_rot=2, rot_step=math.radians(5), k_trans=4, trans_bin=0.05)
    res = api.dses(x, x, cfg)
    assert tuple(res.best.grid_coords) == (0, 0, 0)
    assert np.array_equal(res.best.translation, [0.0, 0.0, 0.0])
    assert res.best_error == 0.0 and res.best_inliers == 60


def test_dses_planted_on_grid_pose(api):
    rng = np.random.default_rng(12)
    x = rng.uniform(-1, 1, (80, 3))
    step = math.radians(4)
    k = 3
    from paper_2502_00115_b200.geometry import grid_rotation, grid_tables
    c, s = grid_tables(k, step)
    n = 2 * k + 1
    r = (4 * n + 2) * n + 5
    R = grid_rotation(c, s, k, r)
    t = np.array([3, -2, 1]) * 0.05
    y = x @ R.T + t
    res = api.dses(x, y, api.SearchConfig(k_rot=k, rot_step=step, k_trans=6, trans_bin=0.05))
    assert tuple(res.best.grid_coords) == (4 - k, 2 - k, 5 - k)
    assert np.allclose(res.best.translation, t, atol=1e-12)


def test_dses_no_candidate(api):
    x = np.zeros((3, 3))
    y = np.full((3, 3), 10.0)
    cfg = api.SearchConfig(k_rot=1, rot_step=0.1, k_trans=2, trans_bin=0.1)
    with pytest.raises(api.NoCandidateError):
        api.dses(x, y, cfg)


def test_dses_sat_l0_shortcut_refines_nothing(api):
    rng = np.random.default_rng(13)
    x = rng.uniform(-1, 1, (40, 3))
    cfg = api.SearchConfig(k_rot=1, rot_step=0.05, k_trans=3, trans_bin=0.05,
                           metric=api.ErrorMetric.saturated_l0(0.05))
    res = api.dses(x, x, cfg)
    assert res.candidates_refined == 0 and res.best_inliers == 40


# ---- edge cases against the oracle -------------------------------------------

def _votes(x, y, b, ilo, dims, rots):
    from paper_2502_00115_b200 import _native
    with _native.Plan(x, y, b, ilo, dims) as plan:
        return plan.mode_batch(rots), plan.info(), plan.stats()


def _check(x, y, b, ilo, dims, rots):
    from oracle import oracle as O
    (c, l, t), info, stats = _votes(x, y, b, ilo, dims, rots)
    oc, ol, ot = O.mode_batch(x, y, b, ilo, dims, rots=rots)
    assert np.array_equal(c, oc) and np.array_equal(l, ol) and np.array_equal(t, ot)
    return info, stats


def _rots(n, seed, scale=1.0):
    from oracle import oracle as O
    rng = np.random.default_rng(seed)
    k = 6
    return O.rotation_grid(k, scale * math.radians(15) / k)[rng.choice((2 * k + 1) ** 3, n)]


@pytest.mark.parametrize("n,m", [(1, 1), (1, 40), (33, 1), (31, 65), (97, 130), (257, 33)])
def test_ragged_sizes(n, m):
    rng = np.random.default_rng(n * 1000 + m)
    x = rng.normal(size=(n, 3)) * 0.5
    y = rng.normal(size=(m, 3)) * 0.5
    _check(x, y, 0.05, np.full(3, -20), np.full(3, 41), _rots(24, n + m))


def test_clustered_reference_exercises_exact_dedup():
    rng = np.random.default_rng(5)
    centres = rng.normal(size=(40, 3)) * 0.6
    # clusters of 1-7 points within a fraction of a bin: dedup components of
    # every size, "far" points, partners in the guard band
    y = np.concatenate([c + rng.normal(size=(rng.integers(1, 8), 3)) * 0.01 for c in centres])
    y = np.concatenate([y, y[:10]])  # exact duplicates too
    x = rng.normal(size=(150, 3)) * 0.6
    info, stats = _check(x, y, 0.05, np.full(3, -20), np.full(3, 41), _rots(64, 7))
    assert info["near_pairs"] > 100


def test_guard_band_points_on_bin_edges():
    # translations exactly on bin edges (k + 1/2) * bin: every pair near an edge
    b = 0.125
    x = np.zeros((8, 3))
    y = (np.arange(24).reshape(8, 3) + 0.5) * b
    info, stats = _check(x, y, b, np.full(3, -30), np.full(3, 61), np.eye(3)[None])
    assert stats["rechecks"] > 0


def test_lattice_larger_than_shared_memory():
    rng = np.random.default_rng(9)
    x = rng.normal(size=(120, 3))
    y = rng.normal(size=(200, 3))
    _check(x, y, 0.02, np.full(3, -100), np.full(3, 201), _rots(6, 9))


def test_exact_mode_for_huge_coordinates():
    rng = np.random.default_rng(10)
    x = rng.normal(size=(50, 3)) * 1e9
    y = x + np.array([0.3, -0.1, 0.2])
    (c, l, t), info, _ = _votes(x, y, 0.1, np.full(3, -8), np.full(3, 17), np.eye(3)[None])
    assert info["frac_bits"] == 0 and c[0] == 50
    _check(x, y, 0.1, np.full(3, -8), np.full(3, 17),
           np.concatenate([np.eye(3)[None], _rots(4, 10, 1e-9)]))


def test_non_cubic_window():
    rng = np.random.default_rng(14)
    x = rng.normal(size=(90, 3)) * 0.4
    y = rng.normal(size=(110, 3)) * 0.4
    _check(x, y, 0.04, np.array([-25, -5, -12]), np.array([51, 9, 30]), _rots(16, 14))


# ---- full-size properties ----------------------------------------------------

def test_sharded_slices_equal_whole_grid_and_runs_repeat():
    from paper_2502_00115_b200 import _native
    from paper_2502_00115_b200.engines import prepare
    import bench
    c = bench.workload("c3")
    cfg = bench.search_config(c)
    from paper_2502_00115_b200.synth import make_pair
    x, y, _ = make_pair(c["spec"], 0)
    prep = prepare(x, y, cfg)
    grid = _native.make_grid(cfg.k_rot, prep.cos_tab, prep.sin_tab, None)
    R = 200_000
    with _native.Plan(prep.x, prep.y, cfg.trans_bin, prep.ilo, prep.dims) as plan:
        whole = plan.mode_grid(grid, 0, R)
        again = plan.mode_grid(grid, 0, R)
        parts = [plan.mode_grid(grid, a, b - a) for a, b in ((0, 70_001), (70_001, 150_000),
                                                            (150_000, R))]
    for k in range(3):
        assert np.array_equal(whole[k], again[k])
        assert np.array_equal(whole[k], np.concatenate([p[k] for p in parts]))
    assert whole[0].max() > 0


@pytest.mark.parametrize("name,nrot", [("c2", 3000), ("c4", 600), ("big", 40)])
def test_votes_invariant_to_cta_count_and_stream(name, nrot):
    """The persistent vote kernel's result does not depend on how many CTAs
    share the rotation queue or on the stream (the reference's determinism
    across thread counts, test_acceptance.py:287-318): 1, 7 and 148 CTAs and
    a private stream against the default one-wave launch.  c2 = shared-memory
    histogram with guard-band risk bitmaps, c4 = overflow-tolerant rounds,
    big = global-memory histograms."""
    from paper_2502_00115_b200 import _native
    from paper_2502_00115_b200.engines import prepare
    import bench
    if name == "big":
        rng = np.random.default_rng(21)
        x, y = rng.normal(size=(300, 3)), rng.normal(size=(400, 3))
        b, ilo, dims = 0.02, np.full(3, -100), np.full(3, 201)
        rots = _rots(nrot, 21)
        run = lambda plan, st=None: plan.mode_batch(rots, st)  # noqa: E731
    else:
        cfg = bench.search_config(bench.workload(name))
        (x0, y0, _), = bench.bench_pairs(name, 1)[0]
        prep = prepare(x0, y0, cfg)
        grid = _native.make_grid(cfg.k_rot, prep.cos_tab, prep.sin_tab, prep.center_rot)
        x, y, b, ilo, dims = prep.x, prep.y, cfg.trans_bin, prep.ilo, prep.dims
        r0 = cfg.rotation_count // 3
        run = lambda plan, st=None: plan.mode_grid(grid, r0, nrot, st)  # noqa: E731
    with _native.Plan(x, y, b, ilo, dims) as plan:
        ref = run(plan)
        assert ref[0].max() > 0
        for ctas in (1, 7, 148):
            plan.set_vote_grid(ctas)
            got = run(plan)
            assert all(np.array_equal(a, g) for a, g in zip(ref, got)), ctas
        plan.set_vote_grid(0)
        st = _native.Stream(0)
        try:
            got = run(plan, st.handle)
        finally:
            st.close()
        assert all(np.array_equal(a, g) for a, g in zip(ref, got))


@pytest.mark.parametrize("kind,param", [("trunc_l2", 0.1), ("l2", None), ("l1", None),
                                        ("trunc_l1", 0.06)])
def test_dses_every_metric_matches_oracle(api, kind, param):
    """Each scoring path (grid screen for truncated metrics, streamed screen
    for L1/L2; exact binary64 re-score) against the oracle dses, including the
    trunc_l2 extension (parity pinned to the oracle only)."""
    from oracle import oracle as O
    from paper_2502_00115_b200.synth import CONFIGS, make_pair
    x, y, _ = make_pair(CONFIGS["c2"]["spec"], 21)
    cfg = api.SearchConfig(k_rot=3, rot_step=math.radians(6), k_trans=20, trans_bin=0.025,
                           metric=api.ErrorMetric(kind, param))
    res = api.dses(x, y, cfg)
    ref = O.dses(x, y, k_rot=cfg.k_rot, rot_step=cfg.rot_step, k_trans=cfg.k_trans,
                 trans_bin=cfg.trans_bin, q=cfg.q, metric=(kind, param))
    assert tuple(res.best.grid_coords) == tuple(ref["grid_coords"])
    assert np.array_equal(res.best.translation, ref["translation"])
    assert math.isclose(res.best_error, ref["best_error"], rel_tol=1e-9)
    assert res.candidates_refined == ref["candidates_refined"]
    assert res.best_inliers == ref["best_inliers"]


def _dict_mode(hist):
    """Mode of a translation-histogram dict (oracle.translation_histogram):
    max count, lexicographically smallest bin at the max, tied bins."""
    best = max(hist.values())
    tied = sorted(k for k, v in hist.items() if v == best)
    return best, tied[0], len(tied)


@pytest.mark.parametrize("seed", [0, 1])
def test_mode_translation_sparse_lattice(api, seed):
    """No t_bounds at a fine bin: the data-derived lattice has ~10^10 bins,
    far beyond any dense histogram -> the sort-based path (_kernels.py:196-294)."""
    from oracle import oracle as O
    rng = np.random.default_rng(seed)
    x = rng.uniform(-1, 1, (150, 3))
    t = np.array([0.2031, -0.4112, 0.0555])
    y = np.concatenate([x[:100] + t + rng.normal(0, 0.0002, (100, 3)), rng.uniform(-1, 1, (80, 3))])
    b = 0.001
    rot = np.eye(3)
    res = api.mode_translation(x, y, rot, b)
    hist = O.translation_histogram(x, y, rot, b)
    count, idx, ties = _dict_mode(hist)
    assert res.count == count and res.index == idx and res.num_tied_bins == ties


def test_sparse_window_matches_dict_histogram():
    """A bounded window just above the dense limit (410^3 bins), several rotations."""
    from oracle import oracle as O
    from paper_2502_00115_b200 import _native
    rng = np.random.default_rng(3)
    x = rng.uniform(-0.5, 0.5, (120, 3))
    y = rng.uniform(-0.5, 0.5, (140, 3))
    b = 0.004
    ilo = np.full(3, -205, dtype=np.int64)
    dims = np.full(3, 410, dtype=np.int64)
    rots = _rots(5, 3)
    with _native.Plan(x, y, b, ilo, dims) as plan:
        counts, lins, ties = plan.mode_batch(rots)
    for r in range(rots.shape[0]):
        hist = O.translation_histogram(x, y, rots[r], b, ilo=ilo, ihi=ilo + dims - 1)
        count, idx, nt = _dict_mode(hist)
        assert counts[r] == count and ties[r] == nt
        assert O.decode_flat(lins[r], ilo, dims) == idx


@pytest.mark.parametrize("kind,param", [("trunc_l1", None), ("sat_l0", 0.004)])
def test_dses_sparse_window_matches_oracle(api, kind, param):
    """dses with k_trans = 210 (421^3 = 74.6 M bins > 2^26): the search runs
    the sort-based vote, as the reference dispatches such windows to
    mode_sparse_batch (mode_search.py:158-163, _kernels.py:196-294); per-rotation
    votes, winner, refine counts and errors against the oracle."""
    from oracle import oracle as O
    rng = np.random.default_rng(11)
    x = rng.uniform(-0.3, 0.3, (160, 3))
    rot = api.rotation_from_euler((0.02, -0.03, 0.04))
    y = np.concatenate([x[:120] @ rot.T + np.array([0.11, -0.07, 0.05]) +
                        rng.normal(0, 0.001, (120, 3)), rng.uniform(-0.4, 0.4, (60, 3))])
    cfg = api.SearchConfig(k_rot=1, rot_step=0.03, k_trans=210, trans_bin=0.004,
                           metric=None if param is None else api.ErrorMetric(kind, param))
    res = api.dses(x, y, cfg)
    ref = O.dses(x, y, k_rot=cfg.k_rot, rot_step=cfg.rot_step, k_trans=cfg.k_trans,
                 trans_bin=cfg.trans_bin, q=cfg.q, metric=(kind, param), return_votes=True,
                 nthreads=2)  # 600 MB of oracle scratch per thread at this lattice
    assert tuple(res.best.grid_coords) == tuple(ref["grid_coords"])
    assert np.array_equal(res.best.translation, ref["translation"])
    assert math.isclose(res.best_error, ref["best_error"], rel_tol=1e-9, abs_tol=1e-12)
    assert res.best_inliers == ref["best_inliers"]
    assert res.candidates_evaluated == ref["candidates_evaluated"]
    assert res.candidates_refined == ref["candidates_refined"]
    from paper_2502_00115_b200 import _native
    from paper_2502_00115_b200.engines import prepare
    p = prepare(x, y, cfg)
    g = _native.make_grid(cfg.k_rot, p.cos_tab, p.sin_tab, p.center_rot)
    with _native.Plan(p.x, p.y, cfg.trans_bin, p.ilo, p.dims) as plan:
        counts, lins, ties = plan.mode_grid(g, 0, cfg.rotation_count)
    assert np.array_equal(counts, ref["counts"]) and np.array_equal(lins, ref["lins"])
    assert np.array_equal(ties, ref["ties"])


def test_dses_window_beyond_int32_lattice_raises(api):
    """Beyond 2^31 bins the search raises the reference's SearchSpaceTooLargeError
    (a documented limit: the candidate arrays hold 32-bit flat bins)."""
    x = np.random.default_rng(2).uniform(-0.1, 0.1, (8, 3))
    cfg = api.SearchConfig(k_rot=0, rot_step=0.1, k_trans=700, trans_bin=0.001)
    with pytest.raises(api.SearchSpaceTooLargeError):
        api.dses(x, x, cfg)


def test_dses_batch_equals_single_calls(api):
    from paper_2502_00115_b200.synth import CONFIGS, make_pair
    pairs = [make_pair(CONFIGS["c1"]["spec"], s) for s in range(4)]
    cfg = api.SearchConfig(k_rot=2, rot_step=math.radians(9), k_trans=20, trans_bin=0.025)
    batch = api.dses_batch([p[0] for p in pairs], [p[1] for p in pairs], cfg)
    for (x, y, _), b in zip(pairs, batch):
        single = api.dses(x, y, cfg)
        assert tuple(single.best.grid_coords) == tuple(b.best.grid_coords)
        assert np.array_equal(single.best.translation, b.best.translation)
        assert single.best_error == b.best_error and single.best_inliers == b.best_inliers
    assert api.dses_batch([], [], cfg) == []


def test_dses_batch_error_order_and_async_misuse(api):
    """A pair without any in-window vote raises NoCandidateError from
    dses_batch exactly like dses() (the first failing pair wins, earlier pairs
    are not lost to a later failure); the async entry points reject misuse."""
    from paper_2502_00115_b200 import _native
    from paper_2502_00115_b200.engines import prepare
    from paper_2502_00115_b200.synth import CONFIGS, make_pair
    pairs = [make_pair(CONFIGS["c1"]["spec"], s) for s in range(3)]
    cfg = api.SearchConfig(k_rot=1, rot_step=math.radians(9), k_trans=2, trans_bin=0.025)
    far = (pairs[1][0] + 100.0, pairs[1][1])  # translation far outside the window
    xs = [pairs[0][0], far[0], pairs[2][0]]
    ys = [pairs[0][1], far[1], pairs[2][1]]
    with pytest.raises(api.NoCandidateError):
        api.dses(xs[1], ys[1], cfg)
    with pytest.raises(api.NoCandidateError):
        api.dses_batch(xs, ys, cfg)
    ok = api.dses_batch(xs[:1], ys[:1], cfg)
    assert len(ok) == 1
    p = prepare(pairs[0][0], pairs[0][1], cfg)
    g = _native.make_grid(cfg.k_rot, p.cos_tab, p.sin_tab, p.center_rot)
    with _native.Plan(p.x, p.y, cfg.trans_bin, p.ilo, p.dims) as plan:
        with pytest.raises(api.InvalidInputError):  # _native maps DSES_E_INVALID (a ValueError)
            plan.search_wait()  # nothing in flight
        plan.search_async(g, cfg.q, p.code, p.param, p.skip_refine)
        with pytest.raises(api.InvalidInputError):
            plan.search_async(g, cfg.q, p.code, p.param, p.skip_refine)  # one at a time
        r = plan.search_wait()
        r2 = plan.search(g, cfg.q, p.code, p.param, p.skip_refine)
        assert (r["winner_row"], r["winner_lin"], r["best_error"]) == \
            (r2["winner_row"], r2["winner_lin"], r2["best_error"])
        plan.search_async(g, cfg.q, p.code, p.param, p.skip_refine)  # destroyed in flight: safe


def test_source_cloud_beyond_shared_memory():
    """41^3 histogram in shared memory + 6,000 rotated source points in global
    memory (the vote kernel's <HSMEM, !PSMEM> instantiation)."""
    rng = np.random.default_rng(31)
    x = rng.normal(size=(6000, 3)) * 0.5
    y = rng.normal(size=(2500, 3)) * 0.5
    _check(x, y, 0.025, np.full(3, -20), np.full(3, 41), _rots(3, 31))


def test_more_than_65535_sources_uses_32bit_counts():
    """n >= 65536: 16-bit counters could overflow, so the histogram is 32-bit
    (global memory) -- the <!HSMEM> instantiations."""
    rng = np.random.default_rng(32)
    x = rng.normal(size=(70000, 3)) * 0.5
    y = rng.normal(size=(120, 3)) * 0.5
    _check(x, y, 0.05, np.full(3, -10), np.full(3, 21), _rots(2, 32))
