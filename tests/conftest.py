import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 and the built sm_100a extension")
    config.addinivalue_line("markers", "slow: long-running")


def load_golden(name):
    return dict(np.load(os.path.join(GOLDEN, f"{name}.npz"), allow_pickle=False))


@pytest.fixture(scope="session")
def golden():
    cache = {}

    def get(name):
        if name not in cache:
            cache[name] = load_golden(name)
        return cache[name]

    return get


def cfg_from(rec, prefix):
    """SearchConfig kwargs stored by tests/golden/make_golden.py:cfg_fields."""
    kind = str(rec[f"{prefix}_metric_kind"])
    param = float(rec[f"{prefix}_metric_param"])
    out = dict(k_rot=int(rec[f"{prefix}_k_rot"]), rot_step=float(rec[f"{prefix}_rot_step"]),
               k_trans=int(rec[f"{prefix}_k_trans"]), trans_bin=float(rec[f"{prefix}_trans_bin"]),
               q=float(rec[f"{prefix}_q"]), metric=(kind, None if np.isnan(param) else param))
    if f"{prefix}_center_R" in rec:
        out["center"] = (rec[f"{prefix}_center_R"], rec[f"{prefix}_center_t"])
    return out
