"""Full-size parity pins on BASELINE.json's configs:
the B200 search against the pinned C oracle (oracle/gridreg_oracle.c, itself
pinned to the unmodified reference's golden vectors in test_oracle_golden.py)
at the configs' own full grids, on the benchmark's own inputs (the
reference generator's clouds, bench_data/benchgen_<cfg>.npz) -- the
north star's "{R, t} matching the CPU oracle on every test pair".

* c1, c2: every one of the 16 bench pairs -- winner grid coordinates,
  translation bin, rotation, best_inliers, candidates_evaluated /
  candidates_refined exact, best_error within 1e-9 relative;
* c4: the full 9,261-rotation grid -- per-rotation (count, flat bin, ties)
  bit-exact, plus the winner;
* c3: a contiguous 8,192-rotation slice bit-exact, plus the winner of the
  full 753,571-rotation grid (~1 min of oracle time on the box's cores);
* c5 (the resolution sweep, K = 108: 10.2 M rotations): the last 4,096
  rotations of the grid bit-exact.
The reference's own acceptance runs use these geometries
(/root/reference/pkg/tests/test_acceptance.py:177-178, 228-232)."""
import math
import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


@pytest.fixture(scope="module")
def api():
    import paper_2502_00115_b200 as api
    from paper_2502_00115_b200 import _native
    if _native.device_count() < 1:
        pytest.fail("no CUDA device visible to the extension")
    return api


def _pair(name, k):
    import bench
    (pair,), _ = bench.bench_pairs(name, 1, k)
    return pair[0], pair[1]


def _cfg(name, k_rot=None, rot_step=None):
    import bench
    cfg = bench.search_config(bench.workload(name))
    if k_rot is not None:
        from dataclasses import replace
        cfg = replace(cfg, k_rot=k_rot, rot_step=rot_step)
    return cfg


def _oracle_dses(x, y, cfg, **kw):
    from oracle import oracle as O
    return O.dses(x, y, k_rot=cfg.k_rot, rot_step=cfg.rot_step, k_trans=cfg.k_trans,
                  trans_bin=cfg.trans_bin, q=cfg.q, metric=(cfg.metric.kind, cfg.metric.param), **kw)


def _check_winner(res, ref, tag):
    assert tuple(res.best.grid_coords) == tuple(ref["grid_coords"]), tag
    assert np.array_equal(res.best.translation, ref["translation"]), tag
    assert np.array_equal(res.best.rotation, ref["rotation"]), tag
    assert math.isclose(res.best_error, ref["best_error"], rel_tol=1e-9, abs_tol=1e-15), tag
    assert res.best_inliers == ref["best_inliers"], tag
    assert res.candidates_evaluated == ref["candidates_evaluated"], tag
    assert res.candidates_refined == ref["candidates_refined"], tag


def _votes(x, y, cfg, r_begin, r_count):
    from paper_2502_00115_b200 import _native
    from paper_2502_00115_b200.engines import prepare
    p = prepare(x, y, cfg)
    g = _native.make_grid(cfg.k_rot, p.cos_tab, p.sin_tab, p.center_rot)
    with _native.Plan(p.x, p.y, cfg.trans_bin, p.ilo, p.dims) as plan:
        return plan.mode_grid(g, r_begin, r_count), p


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_every_bench_pair_matches_oracle(api, name):
    cfg = _cfg(name)
    xs, ys = zip(*[_pair(name, k) for k in range(16)])
    got = api.dses_batch(list(xs), list(ys), cfg)
    for k in range(16):
        _check_winner(got[k], _oracle_dses(xs[k], ys[k], cfg), f"{name} pair {k}")


def test_c4_full_grid(api):
    x, y = _pair("c4", 0)
    cfg = _cfg("c4")
    R = cfg.rotation_count
    assert R == 9261
    ref = _oracle_dses(x, y, cfg, return_votes=True)
    (counts, lins, ties), _ = _votes(x, y, cfg, 0, R)
    assert np.array_equal(counts, ref["counts"])
    assert np.array_equal(lins, ref["lins"])
    assert np.array_equal(ties, ref["ties"])
    _check_winner(api.dses(x, y, cfg), ref, "c4")


def test_c3_slice_and_full_grid_winner(api):
    from oracle import oracle as O
    x, y = _pair("c3", 0)
    cfg = _cfg("c3")
    assert cfg.rotation_count == 753571
    r0, nr = 372000, 8192  # a contiguous slice through the grid's middle
    (counts, lins, ties), p = _votes(x, y, cfg, r0, nr)
    oc, ol, ot = O.mode_batch(p.x, p.y, cfg.trans_bin, p.ilo, p.dims,
                              grid=(cfg.k_rot, cfg.rot_step, None), r_begin=r0, r_count=nr)
    assert np.array_equal(counts, oc) and np.array_equal(lins, ol) and np.array_equal(ties, ot)
    _check_winner(api.dses(x, y, cfg), _oracle_dses(x, y, cfg), "c3 full grid")


def test_c5_finest_grid_far_end(api):
    from oracle import oracle as O
    x, y = _pair("c2", 0)
    K = 108
    cfg = _cfg("c2", k_rot=K, rot_step=math.radians(45.0 / K))
    R = cfg.rotation_count
    assert R == 10218313
    nr = 4096
    (counts, lins, ties), p = _votes(x, y, cfg, R - nr, nr)
    oc, ol, ot = O.mode_batch(p.x, p.y, cfg.trans_bin, p.ilo, p.dims,
                              grid=(cfg.k_rot, cfg.rot_step, None), r_begin=R - nr, r_count=nr)
    assert np.array_equal(counts, oc) and np.array_equal(lins, ol) and np.array_equal(ties, ot)
