"""GPU parity: the B200 kernels (through the C ABI) against the reference's
golden vectors and the pinned CPU oracle.  Bars:

* per-rotation (count, flat bin, tied bins): bit-exact;
* refine / alignment errors: bit-exact binary64 (same operations, same order);
* winner grid coordinates and translation bin: identical;
* R, t: identical (R is composed from the same tables in the same order);
* best_error: within 1e-9 relative of the reference (whose final recompute
  goes through a BLAS matmul, engines.py:286 / geometry.py:211);
* best_inliers, candidates_evaluated, candidates_refined: exact.
"""
import math

import numpy as np
import pytest

from conftest import cfg_from

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def native():
    from paper_2502_00115_b200 import _native
    if _native.device_count() < 1:
        pytest.fail("no CUDA device visible to the extension")
    return _native


def api_cfg(rec, prefix):
    from paper_2502_00115_b200 import ErrorMetric, RigidTransform, SearchConfig
    kw = cfg_from(rec, prefix)
    kind, param = kw.pop("metric")
    kw["metric"] = ErrorMetric(kind, param)
    if "center" in kw:
        R, t = kw.pop("center")
        kw["center"] = RigidTransform(R, t)
    return SearchConfig(**kw)


def test_small_mode_cases(native, golden):
    g = golden("small")
    for c in range(int(g["n_mode_cases"])):
        k = f"m{c}"
        with native.Plan(g[f"{k}_x"], g[f"{k}_y"], float(g[f"{k}_b"]), g[f"{k}_ilo"],
                         g[f"{k}_dims"]) as plan:
            counts, lins, ties = plan.mode_batch(g[f"{k}_rots"])
        assert np.array_equal(counts, g[f"{k}_counts"]), k
        assert np.array_equal(lins, g[f"{k}_lins"]), k
        assert np.array_equal(ties, g[f"{k}_ties"]), k


def test_small_mode_cases_exact_mode_matches_fast(native, golden):
    """The same cases at a fraction-bit budget of 0 would be the exact fp64
    path; here we check the fast path's recheck counter is tiny instead."""
    g = golden("small")
    k = "m0"
    with native.Plan(g[f"{k}_x"], g[f"{k}_y"], float(g[f"{k}_b"]), g[f"{k}_ilo"],
                     g[f"{k}_dims"]) as plan:
        assert plan.info()["frac_bits"] >= 6
        plan.mode_batch(g[f"{k}_rots"])
        st = plan.stats()
    assert st["rechecks"] <= max(4, st["pairs"] // 1000)


def test_small_refine_cases(native, golden):
    g = golden("small")
    for c in range(int(g["n_refine_cases"])):
        k = f"r{c}"
        with native.Plan(g[f"{k}_x"], g[f"{k}_y"], 1.0, np.zeros(3, np.int64),
                         np.ones(3, np.int64)) as plan:
            errs = plan.refine_batch(g[f"{k}_rots"], g[f"{k}_ts"], int(g[f"{k}_code"]),
                                     float(g[f"{k}_param"]))
        assert np.array_equal(errs, g[f"{k}_errs"]), k


def check_result(res, rec, prefix):
    assert tuple(res.best.grid_coords) == tuple(int(v) for v in rec[f"{prefix}_grid"])
    assert np.array_equal(res.best.translation, rec[f"{prefix}_t"])
    assert np.array_equal(res.best.rotation, rec[f"{prefix}_R"])
    ref_err = float(rec[f"{prefix}_best_error"])
    assert math.isclose(res.best_error, ref_err, rel_tol=1e-9, abs_tol=1e-12)
    assert res.best_inliers == int(rec[f"{prefix}_best_inliers"])
    assert res.candidates_evaluated == int(rec[f"{prefix}_evaluated"])
    assert res.candidates_refined == int(rec[f"{prefix}_refined"])


def test_small_dses_cases(native, golden):
    from paper_2502_00115_b200 import dses
    g = golden("small")
    for c in range(int(g["n_dses_cases"])):
        p = f"d{c}"
        res = dses(g[f"{p}_x"], g[f"{p}_y"], api_cfg(g, p))
        check_result(res, g, p)


@pytest.mark.parametrize("name,prefix", [("c1", "a"), ("c2", "a"), ("c2", "l1"), ("c2", "l2"),
                                         ("c2", "sat2"), ("c2", "inl"), ("c2", "cen"), ("c3", "a"),
                                         ("c4", "a")])
def test_config_votes_and_dses(native, golden, name, prefix):
    from paper_2502_00115_b200 import dses
    from paper_2502_00115_b200.engines import prepare
    rec = golden(name)
    cfg = api_cfg(rec, prefix)
    if f"{prefix}_counts" in rec:
        prep = prepare(rec["x"], rec["y"], cfg)
        grid = native.make_grid(cfg.k_rot, prep.cos_tab, prep.sin_tab, prep.center_rot)
        with native.Plan(prep.x, prep.y, cfg.trans_bin, prep.ilo, prep.dims) as plan:
            counts, lins, ties = plan.mode_grid(grid, 0, cfg.rotation_count)
        assert np.array_equal(counts, rec[f"{prefix}_counts"])
        assert np.array_equal(lins, rec[f"{prefix}_lins"])
        assert np.array_equal(ties, rec[f"{prefix}_ties"])
    res = dses(rec["x"], rec["y"], cfg)
    check_result(res, rec, prefix)


def test_exhaustive_search_matches_reference(native, golden):
    """Algorithm 1 (engines.exhaustive_search) on the GPU against the
    unmodified reference's results (tests/golden/exh.npz): winner pose
    identical, errors within 1e-9 relative, inliers and pose count exact;
    DSES reaches the exhaustive inlier count (reference acceptance C2)."""
    from paper_2502_00115_b200 import dses, exhaustive_search
    g = golden("exh")
    for c in range(int(g["n_exh_cases"])):
        p = f"e{c}"
        cfg = api_cfg(g, p)
        res = exhaustive_search(g[f"{p}_x"], g[f"{p}_y"], cfg)
        assert tuple(res.best.grid_coords) == tuple(int(v) for v in g[f"{p}_grid"]), p
        assert np.array_equal(res.best.translation, g[f"{p}_t"]), p
        assert np.array_equal(res.best.rotation, g[f"{p}_R"]), p
        assert math.isclose(res.best_error, float(g[f"{p}_best_error"]), rel_tol=1e-9, abs_tol=1e-12)
        assert res.best_inliers == int(g[f"{p}_best_inliers"])
        assert res.candidates_evaluated == int(g[f"{p}_evaluated"])
        if f"{p}_dses_inliers" in g:
            assert dses(g[f"{p}_x"], g[f"{p}_y"], cfg).best_inliers == int(g[f"{p}_dses_inliers"])


def test_batched_harness_matches_reference(native, golden):
    """register_batch (dses_batch + chamfer + evaluate_pose) against the
    reference's harness._run_one on the same benchgen instances
    (tests/golden/harness.npz): winner identical; chamfer one-way bit-exact on
    the same moved cloud; MIE/MAE/chamfer within 1e-9 relative (the moved
    cloud comes from a BLAS matmul, geometry.py:209-211); recall hit identical."""
    from paper_2502_00115_b200 import RigidTransform, register_batch
    from paper_2502_00115_b200.metrics import chamfer_one_way
    g = golden("harness")
    n = int(g["n_harness_cases"])
    cfg = api_cfg(g, "h")
    xs = [g[f"h{k}_x"] for k in range(n)]
    ys = [g[f"h{k}_y"] for k in range(n)]
    gts = [RigidTransform(g[f"h{k}_gt_R"], g[f"h{k}_gt_t"]) for k in range(n)]
    summary, records = register_batch(xs, ys, gts, cfg)
    assert summary.n_trials == n and summary.n_failed == 0
    for k, r in enumerate(records):
        assert r.status == str(g[f"h{k}_status"])
        ref = g[f"h{k}_eval"]
        got = [r.eval.mie_r, r.eval.mie_t, r.eval.mae_r, r.eval.mae_t, r.eval.chamfer]
        for a, b in zip(got, ref):
            assert math.isclose(a, float(b), rel_tol=1e-9, abs_tol=1e-12)
        assert int(r.eval.is_recall_hit) == int(g[f"h{k}_hit"])
        assert r.inliers == int(g[f"h{k}_inliers"])
        assert r.candidates_refined == int(g[f"h{k}_refined"])
    # chamfer one-way: same operations as the reference kernel on the same input
    from paper_2502_00115_b200 import dses
    res = dses(xs[0], ys[0], cfg)
    assert tuple(res.best.grid_coords) == tuple(int(v) for v in g["h0_grid"])
    moved = res.best.apply(xs[0])
    assert chamfer_one_way(moved, ys[0]) == float(g["h0_chamfer_one_way"])
