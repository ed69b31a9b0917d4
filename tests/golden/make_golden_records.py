"""Inputs of the batch-writer / search-config goldens (make_golden.py batchio),
shared with tests/test_batchio.py (no reference import here)."""

# Records for the batch writers: a hit, a miss with awkward floats, a failed row.
BATCHIO_RECORDS = [
    dict(trial=0, seed=100, shape="blob", status="ok",
         eval=(0.1234567890123, 0.0021, 0.1, 1e-17, True, 0.0123456789), inliers=512,
         candidates_refined=3, phase1_ms=12.5, refine_ms=0.25, total_ms=13.0),
    dict(trial=1, seed=101, shape="blob:7", status="ok",
         eval=(179.99999999999997, 0.30000000000000004, 2.5, 0.2, False, None), inliers=0,
         candidates_refined=1, phase1_ms=1.0, refine_ms=2.0, total_ms=3.5),
    dict(trial=2, seed=102, shape="l-bracket", status="engine:NoCandidateError", eval=None,
         inliers=None, candidates_refined=None, phase1_ms=None, refine_ms=None, total_ms=None),
]

SEARCH_JSON_CASES = [
    {"k_rot": 5, "rot_step_deg": 3.0, "k_trans": 20, "trans_bin": 0.025},
    {"rot_range_deg": 45.0, "rot_step_deg": 3.0, "trans_range": 0.5, "trans_bin": 0.025,
     "metric": "L1", "q": 0.25, "pose_cap": 1000},
    {"rot_range_deg": 10.0, "rot_step_deg": 4.0, "trans_range": 0.07, "trans_bin": 0.02,
     "metric": "trunc_l1", "trunc": 0.1},
    {"k_rot": 2, "rot_step_deg": 1.5, "k_trans": 3, "trans_bin": 0.01, "metric": "sat-l0",
     "metric_param": 0.02, "center": {"rotation": [[1, 0, 0], [0, 0, -1], [0, 1, 0]],
                                      "translation": [0.1, -0.2, 0.3]}},
    {"k_rot": 1, "rot_step_deg": 1.0, "k_trans": 1, "trans_bin": 0.01, "metric": "l2"},
    {"rot_range_deg": 0.0, "rot_step_deg": 2.0, "trans_range": 0.0, "trans_bin": 0.05},
    {"k_rot": 1, "rot_step_deg": 1.0, "k_trans": 1, "trans_bin": 0.01, "bogus": 1},
    {"k_rot": 1, "k_trans": 1, "trans_bin": 0.01},
    {"k_rot": 1, "rot_step_deg": 1.0, "k_trans": 1},
    {"rot_step_deg": 1.0, "k_trans": 1, "trans_bin": 0.01},
    {"k_rot": 1, "rot_step_deg": 1.0, "trans_bin": 0.01},
    {"k_rot": 1, "rot_step_deg": 1.0, "k_trans": 1, "trans_bin": 0.01, "metric": "huber"},
]
