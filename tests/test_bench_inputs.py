"""The bench's committed inputs (bench_data/benchgen_<cfg>.npz) are the
reference generator's clouds: pair 0 of c2 / c4 equals the inputs of the
golden files made independently by tests/golden/make_golden.py from the same
benchgen seeds, and every file has the advertised shapes.  CPU only."""
import os

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _load(name):
    return np.load(os.path.join(ROOT, "bench_data", f"benchgen_{name}.npz"))


@pytest.mark.parametrize("name,n,m,count", [("c1", 512, 1024, 16), ("c2", 717, 1024, 16),
                                            ("c3", 717, 1024, 2), ("c4", 5000, 20000, 2)])
def test_bench_inputs_shapes(name, n, m, count):
    d = _load(name)
    assert int(d["count"]) == count
    for k in range(count):
        assert d[f"x{k}"].shape == (n, 3) and d[f"y{k}"].shape == (m, 3)
        assert np.isfinite(d[f"x{k}"]).all() and np.isfinite(d[f"y{k}"]).all()
        r = d[f"gt_R{k}"]
        assert np.allclose(r @ r.T, np.eye(3), atol=1e-12)


@pytest.mark.parametrize("name", ["c2", "c4"])
def test_bench_pair0_is_the_golden_benchgen_instance(name, golden):
    d, g = _load(name), golden(name)
    assert np.array_equal(d["x0"], g["x"]) and np.array_equal(d["y0"], g["y"])


def test_bench_loader_cycles_and_falls_back():
    import sys
    sys.path.insert(0, ROOT)
    import bench
    pairs, desc = bench.bench_pairs("c2", 18, offset=15)
    assert len(pairs) == 18 and "benchgen" in desc
    d = _load("c2")
    assert np.array_equal(pairs[0][0], d["x15"]) and np.array_equal(pairs[1][0], d["x0"])
    synth, desc2 = bench.bench_pairs("c2local", 2)
    assert len(synth) == 2 and "synth" in desc2
