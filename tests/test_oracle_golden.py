"""Pin the CPU oracle (oracle/) to the unmodified reference's golden vectors.

CPU only.  tests/golden/*.npz were produced by tests/golden/make_golden.py from
the reference package itself; the oracle must reproduce every integer exactly
and every binary64 value bit-for-bit (the reference's numba kernels and the C
restatement perform the same IEEE operations in the same order).
"""
import numpy as np
import pytest

from conftest import cfg_from
from oracle import oracle as O


def test_small_mode_cases(golden):
    g = golden("small")
    for c in range(int(g["n_mode_cases"])):
        k = f"m{c}"
        counts, lins, ties = O.mode_batch(g[f"{k}_x"], g[f"{k}_y"], float(g[f"{k}_b"]),
                                          g[f"{k}_ilo"], g[f"{k}_dims"], rots=g[f"{k}_rots"])
        assert np.array_equal(counts, g[f"{k}_counts"]), k
        assert np.array_equal(lins, g[f"{k}_lins"]), k
        assert np.array_equal(ties, g[f"{k}_ties"]), k


def test_small_refine_cases(golden):
    g = golden("small")
    for c in range(int(g["n_refine_cases"])):
        k = f"r{c}"
        errs = O.refine_batch(g[f"{k}_rots"], g[f"{k}_ts"], g[f"{k}_x"], g[f"{k}_y"],
                              int(g[f"{k}_code"]), float(g[f"{k}_param"]))
        assert np.array_equal(errs, g[f"{k}_errs"]), k


def _check_dses(rec, prefix, votes=True):
    kw = cfg_from(rec, prefix)
    out = O.dses(rec.get(f"{prefix}_x", rec.get("x")), rec.get(f"{prefix}_y", rec.get("y")),
                 return_votes=votes, **kw)
    assert tuple(out["grid_coords"]) == tuple(rec[f"{prefix}_grid"])
    assert np.array_equal(out["translation"], rec[f"{prefix}_t"])
    assert np.array_equal(out["rotation"], rec[f"{prefix}_R"])
    assert out["best_error"] == float(rec[f"{prefix}_best_error"])
    assert out["best_inliers"] == int(rec[f"{prefix}_best_inliers"])
    assert out["candidates_evaluated"] == int(rec[f"{prefix}_evaluated"])
    assert out["candidates_refined"] == int(rec[f"{prefix}_refined"])
    if votes and f"{prefix}_counts" in rec:
        assert np.array_equal(out["counts"], rec[f"{prefix}_counts"])
        assert np.array_equal(out["lins"], rec[f"{prefix}_lins"])
        assert np.array_equal(out["ties"], rec[f"{prefix}_ties"])


def test_small_dses_cases(golden):
    g = golden("small")
    for c in range(int(g["n_dses_cases"])):
        _check_dses(g, f"d{c}")


@pytest.mark.parametrize("name,prefix", [("c1", "a"), ("c2", "l1"), ("c2", "l2"), ("c2", "sat2"),
                                         ("c2", "inl"), ("c2", "cen"), ("c3", "a"), ("c4", "a")])
def test_config_dses(golden, name, prefix):
    _check_dses(golden(name), prefix)


@pytest.mark.slow
def test_c2_full_grid(golden):
    _check_dses(golden("c2"), "a")


def test_grid_matches_golden_rotation(golden):
    g = golden("c2")
    k, step = int(g["a_k_rot"]), float(g["a_rot_step"])
    gc = tuple(int(v) for v in g["a_grid"])
    n = 2 * k + 1
    r = (gc[0] + k) * n * n + (gc[1] + k) * n + (gc[2] + k)
    assert np.array_equal(O.rotation_grid(k, step, r_begin=r, r_count=1)[0], g["a_R"])
