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


PROPERTY_EXAMPLES = int(__import__("os").environ.get("DSES_PROPERTY_EXAMPLES", "25"))


@settings(max_examples=PROPERTY_EXAMPLES, deadline=None, derandomize=True,
          suppress_health_check=list(HealthCheck))
@given(seed=st.integers(0, 2**31 - 1), clusters=st.integers(2, 70), per=st.integers(1, 14),
       spread=st.floats(0.05, 1.5), n=st.integers(1, 200), b=st.floats(0.02, 0.2),
       k_trans=st.integers(1, 12))
def test_property_dense_dedup_votes_match_oracle(seed, clusters, per, spread, n, b, k_trans):
    """Dedup-heavy lattices: clusters of up to 14 reference points within
    about a bin of each other (many dedup partners per lane, full 32-lane
    groups whose unused partner slots need a safe lane, components beyond a
    warp's reach -> far lanes), arbitrary windows; every rotation's (count,
    bin, ties) equals the pinned oracle's."""
    from oracle import oracle as O
    from paper_2502_00115_b200 import _native
    rng = np.random.default_rng(seed)
    centres = rng.normal(size=(clusters, 3)) * 0.4
    y = np.repeat(centres, per, axis=0) + rng.uniform(-spread, spread, (clusters * per, 3)) * b
    x = rng.normal(size=(n, 3)) * 0.4
    ilo = np.full(3, -k_trans, dtype=np.int64)
    dims = np.full(3, 2 * k_trans + 1, dtype=np.int64)
    k = 3
    rots = O.rotation_grid(k, math.radians(20) / k)[rng.choice((2 * k + 1) ** 3, 12)]
    with _native.Plan(x, y, b, ilo, dims) as plan:
        c, l, t = plan.mode_batch(rots)
    oc, ol, ot = O.mode_batch(x, y, b, ilo, dims, rots=rots)
    assert np.array_equal(c, oc) and np.array_equal(l, ol) and np.array_equal(t, ot)
