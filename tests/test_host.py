"""Host-side logic and the C ABI surface, on CPU (no GPU calls).

* libdses_b200.so loads and exports every function include/dses_b200.h
  declares, and the ctypes table in _native matches the header;
* the product path fails loudly (NativeUnavailable) when no device is
  visible -- there is no CPU fallback;
* validation raises the reference's exception types under the reference's
  conditions (engines.py:52-98,243-246, geometry.py:52-61,259-267,
  metrics.py:38-97);
* the rotation-grid tables + closed form are bit-identical to the oracle's
  restatement of build_rotation_grid (geometry.py:253-290), and to the
  reference's own matrix stored in the golden fixture;
* lattice helpers reproduce the reference's worked examples
  (tests/test_mode_search.py:73-94 of the reference).
"""
import math
import os
import re

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "dses_b200.h")


def declared_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(dses_\w+)\s*\(", text, re.M)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for required in ("dses_mode_dense_batch", "dses_refine_batch", "dses_search",
                     "dses_plan_create", "dses_stage_vote", "dses_stage_rescore"):
        assert required in names


def test_library_exports_every_declared_symbol():
    from paper_2502_00115_b200 import _native
    L = _native.load()
    for name in declared_functions():
        assert hasattr(L, name), name
    assert set(_native.EXPORTED) == set(declared_functions())
    assert b"sm_100a" in L.dses_build_info()


def test_product_path_fails_loudly_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    from paper_2502_00115_b200 import SearchConfig, _native, dses
    assert _native.device_count() == 0
    x = np.random.default_rng(0).normal(size=(20, 3))
    with pytest.raises(_native.NativeUnavailable):
        dses(x, x, SearchConfig(k_rot=1, rot_step=0.1, k_trans=3, trans_bin=0.05))


def test_search_config_validation():
    from paper_2502_00115_b200 import ErrorMetric, InvalidInputError, SearchConfig
    ok = SearchConfig(k_rot=2, rot_step=0.1, k_trans=3, trans_bin=0.05)
    assert ok.rotation_count == 125 and ok.translation_count == 343
    assert ok.metric == ErrorMetric.truncated_l1(0.25)  # engines.py:87-88 default 5*bin
    for bad in (dict(k_rot=-1), dict(rot_step=0.0), dict(trans_bin=-1.0), dict(q=0.0),
                dict(q=1.5), dict(k_trans=1.5), dict(pose_cap=0), dict(rot_step=float("nan"))):
        kw = dict(k_rot=2, rot_step=0.1, k_trans=3, trans_bin=0.05)
        kw.update(bad)
        with pytest.raises(InvalidInputError):
            SearchConfig(**kw)


def test_pose_cap_and_grid_wrap_raise_before_the_device():
    from paper_2502_00115_b200 import InvalidInputError, SearchConfig, SearchSpaceTooLargeError
    from paper_2502_00115_b200.engines import prepare
    x = np.zeros((4, 3))
    with pytest.raises(SearchSpaceTooLargeError):
        prepare(x, x, SearchConfig(k_rot=10, rot_step=0.01, k_trans=2, trans_bin=0.1, pose_cap=9260))
    with pytest.raises(InvalidInputError):  # k*step > pi (geometry.py:264-267)
        prepare(x, x, SearchConfig(k_rot=4, rot_step=1.0, k_trans=2, trans_bin=0.1))


@pytest.mark.parametrize("bad", [np.zeros((0, 3)), np.zeros((3, 2)), np.zeros(3),
                                 np.array([[0.0, np.nan, 0.0]]), np.array([[np.inf, 0, 0]])])
def test_point_cloud_validation(bad):
    from paper_2502_00115_b200 import InvalidInputError, as_point_cloud
    with pytest.raises(InvalidInputError):
        as_point_cloud(bad)


def test_error_metric_names_and_codes():
    from paper_2502_00115_b200 import ErrorMetric, InvalidInputError
    assert ErrorMetric.from_name("trunc-l1", 0.02) == ErrorMetric("trunc_l1", 0.1)
    assert ErrorMetric.from_name("inliers", 0.02) == ErrorMetric("sat_l0", 0.02)
    assert ErrorMetric.from_name("L1", 0.02)._code_param() == (1, 0.0)
    assert ErrorMetric.from_name("l2", 0.02)._code_param() == (0, 0.0)
    with pytest.raises(InvalidInputError):
        ErrorMetric.from_name("huber", 0.02)
    with pytest.raises(InvalidInputError):
        ErrorMetric("l1", 0.5)
    with pytest.raises(InvalidInputError):
        ErrorMetric("trunc_l1")


def test_bin_index_worked_examples():
    from paper_2502_00115_b200 import InvalidInputError, bin_center, bin_index
    # round half away from zero per axis (reference tests/test_mode_search.py:73-80)
    assert tuple(bin_index((0.25, -0.25, 0.74), 0.5)) == (1, -1, 1)
    assert tuple(bin_index((1.0, 2.0, 3.0), 0.5)) == (2, 4, 6)
    assert tuple(bin_index((0.049, -0.051, 0.0), 0.1)) == (0, -1, 0)
    idx = np.array([3, -7, 0])
    assert np.array_equal(bin_index(bin_center(idx, 0.025), 0.025), idx)
    with pytest.raises(InvalidInputError):
        bin_index((0.0, 0.0, 0.0), 0.0)


@pytest.mark.parametrize("k,step", [(1, 0.3), (5, math.radians(9)), (15, math.radians(3))])
def test_grid_tables_match_oracle_grid(k, step):
    from oracle import oracle as O
    from paper_2502_00115_b200.geometry import grid_index, grid_rotation, grid_tables
    c, s = grid_tables(k, step)
    R = (2 * k + 1) ** 3
    rows = np.unique(np.linspace(0, R - 1, 50).astype(int))
    ref = O.rotation_grid(k, step)
    for r in rows:
        assert np.array_equal(grid_rotation(c, s, k, int(r)), ref[r])
    n = 2 * k + 1
    assert tuple(grid_index(k, 0)) == (-k, -k, -k)
    assert tuple(grid_index(k, R - 1)) == (k, k, k)
    assert tuple(grid_index(k, n * n + 1)) == (-k + 1, -k, -k + 1)


def test_grid_rotation_matches_reference_matrix(golden):
    from paper_2502_00115_b200.geometry import grid_rotation, grid_tables
    g = golden("c2")
    k, step = int(g["a_k_rot"]), float(g["a_rot_step"])
    gc = [int(v) + k for v in g["a_grid"]]
    n = 2 * k + 1
    c, s = grid_tables(k, step)
    assert np.array_equal(grid_rotation(c, s, k, (gc[0] * n + gc[1]) * n + gc[2]), g["a_R"])


def test_oracle_mode_known_answers():
    """The oracle on the reference's worked mode examples
    (reference tests/test_mode_search.py:116-166), values restated."""
    from oracle import oracle as O

    def mode(x, y, rot, b):
        x, y = np.asarray(x, float), np.asarray(y, float)
        xmax = float(np.linalg.norm(x, axis=1).max())
        ilo = O.bin_index(y.min(axis=0) - xmax, b) - 1
        ihi = O.bin_index(y.max(axis=0) + xmax, b) + 1
        dims = ihi - ilo + 1
        c, l, t = O.mode_batch(x, y, b, ilo, dims, rots=np.asarray(rot, float)[None])
        return int(c[0]), O.decode_flat(l[0], ilo, dims), int(t[0])

    assert mode([[0, 0, 0]], [[1, 2, 3]], np.eye(3), 0.5) == (1, (2, 4, 6), 1)
    corners = [[i, j, k] for i in (0.0, 1.0) for j in (0.0, 1.0) for k in (0.0, 1.0)]
    assert mode(corners, corners, np.eye(3), 0.1)[0::2] == (8, 1)
    assert mode([[0, 0, 0]], [[1, 0, 0], [0, 1, 0]], np.eye(3), 0.5) == (1, (0, 2, 0), 2)
    assert mode([[0, 0, 0]], [[1, 0, 0], [1.01, 0, 0]], np.eye(3), 0.1)[0] == 1  # dedup


def test_synthetic_pairs_are_seeded_and_shaped():
    from paper_2502_00115_b200.synth import CONFIGS, make_pair
    x1, y1, _ = make_pair(CONFIGS["c2"]["spec"], 3)
    x2, y2, _ = make_pair(CONFIGS["c2"]["spec"], 3)
    assert np.array_equal(x1, x2) and np.array_equal(y1, y2)
    assert x1.shape == (717, 3) and y1.shape == (1024, 3)
    x4, y4, _ = make_pair(CONFIGS["c4"]["spec"], 0)
    assert x4.shape == (5000, 3) and y4.shape == (20000, 3)
