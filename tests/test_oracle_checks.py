"""The verification suite of the reference (harness.run_oracle_checks,
harness.py:329-462; `gridreg oracle-check`, cli.py:212-226): instance
generators (CPU, against the reference's draws in tests/golden/oracle.npz),
the dense translation sweep (numpy oracle on CPU; the dses_sweep_inlier_best
kernel on the GPU, bit-identical counts) and the whole suite / CLI (GPU)."""
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT


def _lemma_rng():
    return np.random.default_rng(np.random.SeedSequence([0x0AC1E, 0]))


def test_instance_generators_match_reference(golden):
    """Same RNG, same draws: the planted instances are the reference's."""
    from paper_2502_00115_b200.harness import make_lemma_instance, make_theorem_instance
    g = golden("oracle")
    rng = _lemma_rng()
    for k in range(4):
        x, y, rot, m = make_lemma_instance(rng, 0.05)
        assert np.array_equal(x, g[f"l{k}_x"]) and np.array_equal(y, g[f"l{k}_y"])
        assert np.array_equal(rot, g[f"l{k}_rot"]) and m == int(g[f"l{k}_m"])
    for k in range(4):
        x, y, cfg = make_theorem_instance(rng)
        assert np.array_equal(x, g[f"t{k}_x"]) and np.array_equal(y, g[f"t{k}_y"])
        assert cfg.k_rot == int(g[f"t{k}_krot"]) and cfg.metric.kind == "sat_l0"


def _sweep_cases(g):
    cases = []
    for k in range(4):
        x, y, rot = g[f"l{k}_x"], g[f"l{k}_y"], g[f"l{k}_rot"]
        cand = np.ascontiguousarray((y[None, :, :] - (x @ rot.T)[:, None, :]).reshape(-1, 3))
        axes = [np.arange(cand[:, a].min(), cand[:, a].max() + 0.0125, 0.0125) for a in range(3)]
        cases.append((cand, x.shape[0], y.shape[0], 0.025, axes, int(g[f"l{k}_best"])))
    cases.append((g["s0_cands"], 7, 5, 0.04, list(g["s0_axes"]), int(g["s0_best"])))
    cases.append((g["s1_cands"], 6, 6, 0.25, list(g["s1_axes"]), int(g["s1_best"])))
    return cases


def test_oracle_sweep_matches_reference(golden):
    import oracle.oracle as orc
    cases = _sweep_cases(golden("oracle"))
    for cand, n, m, half, axes, want in cases[4:]:  # the small standalone cases
        assert orc.sweep_inlier_best(cand, n, m, half, *axes) == want
    cand, n, m, half, axes, want = cases[0]  # one lemma-sized lattice
    assert orc.sweep_inlier_best(cand, n, m, half, *axes) == want
    assert orc.sweep_inlier_best(cand, n, m, half, [], axes[1], axes[2]) == 0


@pytest.mark.gpu
def test_sweep_kernel_matches_reference(golden):
    from paper_2502_00115_b200.harness import sweep_inlier_best
    for cand, n, m, half, axes, want in _sweep_cases(golden("oracle")):
        assert sweep_inlier_best(cand, n, m, half, *axes) == want
    cand, n, m, half, axes, _ = _sweep_cases(golden("oracle"))[0]
    assert sweep_inlier_best(cand, n, m, half, axes[0][:0], axes[1], axes[2]) == 0
    # larger than the shared-memory staging limit: the global-memory variant
    rng = np.random.default_rng(3)
    big = rng.uniform(-0.5, 0.5, (64 * 40, 3))
    ax = [np.linspace(-0.5, 0.5, 9) for _ in range(3)]
    import oracle.oracle as orc
    assert sweep_inlier_best(big, 64, 40, 0.05, *ax) == orc.sweep_inlier_best(big, 64, 40, 0.05, *ax)


@pytest.mark.gpu
def test_run_oracle_checks_matches_reference(golden):
    """The suite on the GPU reports what the reference's run_oracle_checks
    reported for (4, 4, seed 0): counts and detail lines."""
    from paper_2502_00115_b200 import count_inliers, dses, exhaustive_search, mode_translation
    from paper_2502_00115_b200 import RigidTransform, run_oracle_checks
    from paper_2502_00115_b200.harness import make_theorem_instance
    g = golden("oracle")
    for k in range(4):
        x, y, rot = g[f"l{k}_x"], g[f"l{k}_y"], g[f"l{k}_rot"]
        mode = mode_translation(x, y, rot, 0.05)
        assert np.array_equal(mode.t_star, g[f"l{k}_tstar"])
        assert count_inliers(x, y, RigidTransform(rot, mode.t_star), 0.05) == int(g[f"l{k}_cstar"])
    rep = run_oracle_checks(4, 4, 0)
    want = [int(v) for v in g["report"]]
    assert [rep.lemma_trials, rep.lemma_violations, rep.theorem_trials,
            rep.theorem_violations] == want
    assert "\n".join(rep.details) == str(g["report_details"]) and rep.ok
    rng = _lemma_rng()
    from paper_2502_00115_b200.harness import make_lemma_instance
    for _ in range(4):
        make_lemma_instance(rng, 0.05)
    for k in range(4):
        x, y, cfg = make_theorem_instance(rng)
        assert dses(x, y, cfg).best_inliers == int(g[f"t{k}_semi"])
        assert exhaustive_search(x, y, cfg).best_inliers == int(g[f"t{k}_full"])


@pytest.mark.gpu
def test_cli_oracle_check():
    r = subprocess.run([sys.executable, "-m", "paper_2502_00115_b200", "oracle-check",
                        "--trials", "3", "--seed", "1"], cwd=ROOT, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    lines = r.stdout.splitlines()
    assert lines[0] == "mode-optimality sweep: 3/3 ok"
    assert lines[1] == "engine inlier equality: 3/3 ok"
