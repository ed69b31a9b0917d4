"""The documented drop-in binding (tests/integration/
gridreg_b200.py) driven exactly as the reference's _mode_batch drives its
numba kernel (mode_search.py:132-164): the (R, 3, 3) rotation stack of
engines._prepare (engines.py:120-130: the grid's closed form, or
einsum("ab,lbc->lac", centre, grid) with a centre), the unsorted clouds,
bin_size, ilo = bin_index(t_centre) - k_trans, dims = 2 k_trans + 1, and
caller-allocated int64 outputs.  Checked bit-for-bit against the reference's
own per-rotation (count, flat bin, ties) golden vectors
(tests/golden/make_golden.py imports the unmodified reference)."""
import numpy as np
import pytest

from conftest import cfg_from

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def seam():
    from paper_2502_00115_b200 import _native
    if _native.device_count() < 1:
        pytest.fail("no CUDA device visible to the extension")
    from integration import gridreg_b200
    return gridreg_b200


def _stack(rec, prefix):
    from paper_2502_00115_b200.geometry import build_rotation_grid
    from paper_2502_00115_b200.mode_search import bin_index
    kw = cfg_from(rec, prefix)
    grid = build_rotation_grid(kw["k_rot"], kw["rot_step"])
    if "center" in kw:
        C, tc = kw["center"]
        rots = np.ascontiguousarray(np.einsum("ab,lbc->lac", C, grid.matrices))
    else:
        rots, tc = grid.matrices, np.zeros(3)
    ilo = bin_index(np.asarray(tc, dtype=np.float64), kw["trans_bin"]) - kw["k_trans"]
    dims = np.full(3, 2 * kw["k_trans"] + 1, dtype=np.int64)
    return rots, kw["trans_bin"], ilo, dims


@pytest.mark.parametrize("name,prefix", [("c2", "a"), ("c2", "cen"), ("c2", "l1"), ("c1", "a"),
                                         ("c3", "a"), ("c4", "a")])
def test_mode_dense_batch_binding_matches_reference(seam, golden, name, prefix):
    g = golden(name)
    if f"{prefix}_counts" not in g:
        pytest.skip(f"{name} golden has no per-rotation votes for {prefix}")
    rots, b, ilo, dims = _stack(g, prefix)
    nrot = rots.shape[0]
    assert nrot == g[f"{prefix}_counts"].size
    counts, lins, ties = (np.empty(nrot, dtype=np.int64) for _ in range(3))
    seam.mode_dense_batch(rots, g["x"], g["y"], b, ilo, dims, counts, lins, ties)
    assert np.array_equal(counts, g[f"{prefix}_counts"])
    assert np.array_equal(lins, g[f"{prefix}_lins"])
    assert np.array_equal(ties, g[f"{prefix}_ties"])


def test_binding_error_contract(seam):
    """DSES_E_INVALID -> InvalidInputError (a ValueError) in the binding."""
    x = np.zeros((4, 3))
    out = [np.empty(1, dtype=np.int64) for _ in range(3)]
    with pytest.raises(ValueError):
        seam.mode_dense_batch(np.eye(3)[None], x, x, -1.0, np.zeros(3, np.int64),
                              np.ones(3, np.int64), *out)
