"""translation_histogram / TranslationHistogram.mode and refine_candidates
 against the unmodified reference's outputs
(tests/golden/histo.npz, make_golden.py histo).

CPU: the oracle's numpy restatement and the package's host-side
TranslationHistogram.mode reproduce the golden maps exactly; the oracle's
refine kernel reproduces refine_candidates bit-for-bit.
GPU (-m gpu): the sort-based vote map (csrc/dses_sparse.cu through
dses_translation_histogram) equals the golden map bin for bin, with and
without dedup, bounded and unbounded; refine_candidates through
dses_refine_batch is bit-identical.
"""
import numpy as np
import pytest

from oracle import oracle as O


def _case(g, k):
    p = f"t{k}"
    return (g[f"{p}_x"], g[f"{p}_y"], g[f"{p}_rot"], float(g[f"{p}_bin"]),
            g.get(f"{p}_bounds"))


def _golden_map(g, k, dedup):
    q = f"t{k}_{'d' if dedup else 'r'}"
    return ({tuple(int(v) for v in key): int(c) for key, c in zip(g[f"{q}_keys"], g[f"{q}_vals"])},
            int(g[f"{q}_total"]), g.get(f"{q}_mode"))


def test_oracle_histogram_matches_reference(golden):
    from paper_2502_00115_b200.mode_search import bounds_to_index_range
    g = golden("histo")
    for k in range(int(g["n_histo_cases"])):
        x, y, rot, b, bounds = _case(g, k)
        kw = {}
        if bounds is not None:
            ilo, ihi = bounds_to_index_range(bounds, b)
            kw = dict(ilo=ilo, ihi=ihi)
        for dedup in (True, False):
            want, total, _ = _golden_map(g, k, dedup)
            got = O.translation_histogram(x, y, rot, b, dedup=dedup, **kw)
            assert got == want, (k, dedup)
            assert sum(got.values()) == total


def test_histogram_mode_host_logic(golden):
    from paper_2502_00115_b200.errors import NoCandidateError
    from paper_2502_00115_b200.mode_search import TranslationHistogram
    g = golden("histo")
    for k in range(int(g["n_histo_cases"])):
        b = float(g[f"t{k}_bin"])
        for dedup in (True, False):
            want, total, mode = _golden_map(g, k, dedup)
            h = TranslationHistogram(bin_size=b, counts=want, total=total, dedup=dedup)
            if mode is None:
                with pytest.raises(NoCandidateError):
                    h.mode()
                continue
            md = h.mode()
            assert (*md.index, md.count, md.num_tied_bins) == tuple(int(v) for v in mode)
            assert np.array_equal(md.t_star, np.asarray(md.index, dtype=np.float64) * b)


def _rc(g):
    n = len(g["rc_counts"])
    return [(g[f"rc_R{j}"], g[f"rc_t{j}"], int(g["rc_counts"][j])) for j in range(n)]


METRICS = {"l1": ("l1", None), "tl1": ("trunc_l1", 0.05), "l2": ("l2", None), "sat": ("sat_l0", 0.03)}


def test_oracle_refine_candidates_matches_reference(golden):
    g = golden("histo")
    cands = _rc(g)
    for mname, (kind, param) in METRICS.items():
        for q in (0.5, 0.75, 1.0):
            want = g[f"rc_{mname}_{int(q * 100)}"]
            n = O.refine_cutoff([c for _, _, c in cands], q)
            errs = O.refine_batch(np.stack([r for r, _, _ in cands[:n]]),
                                  np.stack([t for _, t, _ in cands[:n]]), g["rc_x"], g["rc_y"],
                                  O.METRIC_CODES[kind], 0.0 if param is None else param)
            assert np.array_equal(errs, want[:n]), (mname, q)
            assert np.isnan(want[n:]).all()


@pytest.mark.gpu
def test_gpu_histogram_matches_reference(golden):
    from paper_2502_00115_b200 import translation_histogram
    from paper_2502_00115_b200.errors import NoCandidateError
    g = golden("histo")
    for k in range(int(g["n_histo_cases"])):
        x, y, rot, b, bounds = _case(g, k)
        for dedup in (True, False):
            want, total, mode = _golden_map(g, k, dedup)
            h = translation_histogram(x, y, rot, b, t_bounds=bounds, dedup=dedup)
            assert h.counts == want, (k, dedup)
            assert h.total == total and h.dedup == dedup and h.bin_size == b
            if mode is None:
                with pytest.raises(NoCandidateError):
                    h.mode()
            else:
                md = h.mode()
                assert (*md.index, md.count, md.num_tied_bins) == tuple(int(v) for v in mode)


@pytest.mark.gpu
def test_gpu_histogram_agrees_with_mode_translation():
    """Property at a larger size: the map's mode is mode_translation's answer,
    the raw map's total is the number of in-lattice pairs (N*M unbounded)."""
    from paper_2502_00115_b200 import mode_translation, rotation_from_euler, translation_histogram
    rng = np.random.default_rng(3)
    x = rng.normal(scale=0.3, size=(700, 3))
    y = np.concatenate([x[:500] @ rotation_from_euler([0.1, -0.2, 0.05]).T + 0.07,
                        rng.normal(scale=0.3, size=(524, 3))])
    rot = rotation_from_euler([0.1, -0.2, 0.05])
    h = translation_histogram(x, y, rot, 0.02)
    md, ref = h.mode(), mode_translation(x, y, rot, 0.02)
    assert (md.index, md.count, md.num_tied_bins) == (ref.index, ref.count, ref.num_tied_bins)
    raw = translation_histogram(x, y, rot, 0.02, dedup=False)
    assert raw.total == x.shape[0] * y.shape[0]
    assert all(raw.counts[key] >= c for key, c in h.counts.items())


@pytest.mark.gpu
def test_gpu_refine_candidates_matches_reference(golden):
    from paper_2502_00115_b200 import ErrorMetric, PoseCandidate, RigidTransform, refine_candidates
    g = golden("histo")
    cands = [PoseCandidate(transform=RigidTransform(r, t), inlier_count=c) for r, t, c in _rc(g)]
    for mname, (kind, param) in METRICS.items():
        metric = ErrorMetric(kind, param)
        for q in (0.5, 0.75, 1.0):
            want = g[f"rc_{mname}_{int(q * 100)}"]
            out = refine_candidates(cands, g["rc_x"], g["rc_y"], metric, q)
            got = np.array([np.nan if c.refined_error is None else c.refined_error for c in out])
            assert np.array_equal(got, want, equal_nan=True), (mname, q)
            assert [c.inlier_count for c in out] == [c.inlier_count for c in cands]
