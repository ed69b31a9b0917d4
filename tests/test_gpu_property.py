"""Property tests on the B200 (hypothesis, like the reference's
tests/test_mode_search.py:334-348 and test_metrics.py:341-361): random small
problems, GPU against the pinned oracle."""
import math

import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

pytestmark = pytest.mark.gpu

SETTINGS = settings(max_examples=40, deadline=None, derandomize=True,
                    suppress_health_check=list(HealthCheck))


def _cloud(seed, n, scale):
    return np.random.default_rng(seed).normal(size=(n, 3)) * scale


@SETTINGS
@given(seed=st.integers(0, 2**31 - 1), n=st.integers(1, 60), m=st.integers(1, 80),
       scale=st.floats(0.05, 2.0), b=st.floats(0.01, 0.5),
       ang=st.tuples(*[st.floats(-math.pi, math.pi)] * 3))
def test_property_mode_translation_matches_oracle(seed, n, m, scale, b, ang):
    from oracle import oracle as O
    from paper_2502_00115_b200 import mode_translation, rotation_from_euler
    x = _cloud(seed, n, scale)
    y = _cloud(seed + 1, m, scale)
    # duplicate a few reference points within a bin: exercises the dedup
    if m > 3:
        y[1] = y[0] + 0.1 * b
    rot = rotation_from_euler(ang)
    res = mode_translation(x, y, rot, b)
    xmax = float(np.linalg.norm(x, axis=1).max())
    ilo = O.bin_index(y.min(axis=0) - xmax, b) - 1
    ihi = O.bin_index(y.max(axis=0) + xmax, b) + 1
    dims = ihi - ilo + 1
    if int(np.prod(dims)) <= 2**24:
        c, l, t = O.mode_batch(x, y, b, ilo, dims, rots=rot[None])
        assert (res.count, res.index, res.num_tied_bins) == (int(c[0]), O.decode_flat(l[0], ilo, dims), int(t[0]))


@SETTINGS
@given(seed=st.integers(0, 2**31 - 1), n=st.integers(3, 40), m=st.integers(3, 50),
       kind=st.sampled_from(["trunc_l1", "l1", "l2", "sat_l0", "trunc_l2"]),
       k_rot=st.integers(0, 2), k_trans=st.integers(1, 6))
def test_property_dses_matches_oracle(seed, n, m, kind, k_rot, k_trans):
    from oracle import oracle as O
    from paper_2502_00115_b200 import ErrorMetric, NoCandidateError, SearchConfig, dses
    x = _cloud(seed, n, 0.3)
    y = np.concatenate([x[: min(n, m)] + 0.02, _cloud(seed + 7, max(0, m - n), 0.3)])
    b = 0.03
    param = {"trunc_l1": 0.1, "trunc_l2": 0.1, "sat_l0": b}.get(kind)
    cfg = SearchConfig(k_rot=k_rot, rot_step=math.radians(5), k_trans=k_trans, trans_bin=b,
                       metric=ErrorMetric(kind, param))
    try:
        ref = O.dses(x, y, k_rot=k_rot, rot_step=cfg.rot_step, k_trans=k_trans, trans_bin=b,
                     q=cfg.q, metric=(kind, param))
    except LookupError:
        with pytest.raises(NoCandidateError):
            dses(x, y, cfg)
        return
    res = dses(x, y, cfg)
    assert tuple(res.best.grid_coords) == tuple(ref["grid_coords"])
    assert np.array_equal(res.best.translation, ref["translation"])
    assert math.isclose(res.best_error, ref["best_error"], rel_tol=1e-9, abs_tol=1e-12)
    assert res.best_inliers == ref["best_inliers"]
    assert res.candidates_evaluated == ref["candidates_evaluated"]
    assert res.candidates_refined == ref["candidates_refined"]
