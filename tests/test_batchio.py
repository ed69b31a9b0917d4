"""Batch records on disk and search configs, CPU only.

* write_batch_csv / write_batch_json are byte-identical to the reference's
  writers (harness.py:468-534) on the same records: tests/golden/batchio.npz
  holds the reference's own output (tests/golden/make_golden.py batchio).
* search_from_json / search_to_dict follow harness.py:545-616 on every golden
  config file, including the rejected ones (same exception type and message).
* register_batch shards trials over ranks (gloo, world 2): trial k runs on
  rank k mod 2 and every rank returns the whole batch, identical to one
  process.  The GPU engine is replaced by a deterministic stand-in here (the
  engine itself is covered by the -m gpu parity tests).
"""
import json
import math
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path[:0] = [ROOT, os.path.join(HERE, "golden")]


def _golden():
    return json.loads(str(np.load(os.path.join(HERE, "golden", "batchio.npz"))["batchio"]))


def _records():
    from make_golden_records import BATCHIO_RECORDS
    from paper_2502_00115_b200.harness import TrialRecord
    from paper_2502_00115_b200.metrics import EvalReport
    out = []
    for d in BATCHIO_RECORDS:
        e = d["eval"]
        ev = None if e is None else EvalReport(mie_r=e[0], mie_t=e[1], mae_r=e[2], mae_t=e[3],
                                                is_recall_hit=e[4], chamfer=e[5])
        out.append(TrialRecord(**dict(d, eval=ev)))
    return out


def test_batch_csv_json_bytes_match_reference(tmp_path):
    from paper_2502_00115_b200 import ErrorMetric, RigidTransform, SearchConfig
    from paper_2502_00115_b200.harness import _summarize, write_batch_csv, write_batch_json
    g = _golden()
    recs = _records()
    write_batch_csv(tmp_path / "b.csv", recs)
    assert (tmp_path / "b.csv").read_text(encoding="utf-8") == g["csv"]
    search = SearchConfig(k_rot=3, rot_step=math.radians(2.0), k_trans=8, trans_bin=0.02,
                          metric=ErrorMetric.from_name("trunc-l1", 0.02, 0.05),
                          center=RigidTransform(np.eye(3), np.array([0.5, 0.0, -0.25])))
    write_batch_json(tmp_path / "b.json", g["scenario"], search, _summarize(recs), recs,
                     extra={"note": "golden"})
    assert (tmp_path / "b.json").read_text(encoding="utf-8") == g["json"]


def test_search_json_matches_reference(tmp_path):
    from make_golden_records import SEARCH_JSON_CASES
    from paper_2502_00115_b200.errors import GridregError
    from paper_2502_00115_b200.harness import search_from_json, search_to_dict
    g = _golden()
    assert len(g["search_cases"]) == len(SEARCH_JSON_CASES)
    for k, (case, want) in enumerate(zip(SEARCH_JSON_CASES, g["search_cases"])):
        path = tmp_path / f"s{k}.json"
        path.write_text(json.dumps(case), encoding="utf-8")
        if "ok" in want:
            got = json.loads(json.dumps(search_to_dict(search_from_json(path))))
            assert got == want["ok"], case
        else:
            with pytest.raises(GridregError) as ei:
                search_from_json(path)
            assert type(ei.value).__name__ == want["error"]
            assert str(ei.value) == want["message"]


# ---- sharded register_batch (gloo) with a stand-in engine

class _Res:
    def __init__(self, x, y):
        from paper_2502_00115_b200 import RigidTransform
        self.best = RigidTransform(np.eye(3), y.mean(0) - x.mean(0))
        self.best_inliers = int(x.shape[0])
        self.candidates_refined = int(y.shape[0]) % 7
        self.elapsed = {"phase1": 1e-3, "refine": 2e-3, "total": 4e-3}


def _patch(harness, log):
    def fake_batch(xs, ys, cfg, device=0):
        log.extend(int(round(x[0, 0] * 1000)) for x in xs)
        return [_Res(x, y) for x, y in zip(xs, ys)]
    harness.dses_batch = fake_batch
    harness.dses = lambda x, y, cfg, device=0: _Res(x, y)
    harness.chamfer_distance = lambda a, b, device=0: float(np.abs(a.mean(0) - b.mean(0)).sum())


def _pairs(n=5):
    from paper_2502_00115_b200 import RigidTransform
    rng = np.random.default_rng(5)
    xs, ys, gts = [], [], []
    for k in range(n):
        x = rng.normal(size=(40 + k, 3))
        x[0, 0] = k / 1000.0  # trial id, read back by the stand-in engine
        ys.append(x[:30] + np.array([0.1 * k, 0.0, 0.02]))
        xs.append(x)
        gts.append(RigidTransform(np.eye(3), np.array([0.1 * k, 0.0, 0.0])))
    return xs, ys, gts


def _rows(records):
    from paper_2502_00115_b200.harness import record_row
    return [record_row(r) for r in records]


def _worker(rank, world, port, out):
    sys.path[:0] = [ROOT]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    from paper_2502_00115_b200 import SearchConfig, harness
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        log = []
        _patch(harness, log)
        xs, ys, gts = _pairs()
        summary, recs = harness.register_batch(xs, ys, gts, SearchConfig(k_rot=1, rot_step=0.1, k_trans=2, trans_bin=0.05),
                                               seeds=[10 + k for k in range(5)])
        with open(f"{out}.{rank}.json", "w") as fh:
            json.dump({"ran": log, "rows": _rows(recs), "n": summary.n_trials,
                       "recall": summary.recall}, fh)
    finally:
        dist.destroy_process_group()


def test_register_batch_sharded_gloo(tmp_path):
    from paper_2502_00115_b200 import SearchConfig, harness
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = str(tmp_path / "rank")
    mp.start_processes(_worker, args=(2, port, out), nprocs=2, join=True, start_method="spawn")
    ranks = [json.load(open(f"{out}.{r}.json")) for r in range(2)]
    assert ranks[0]["ran"] == [0, 2, 4] and ranks[1]["ran"] == [1, 3]
    assert ranks[0]["rows"] == ranks[1]["rows"]
    # single process, same stand-in engine
    import importlib
    h = importlib.reload(harness)
    log = []
    _patch(h, log)
    xs, ys, gts = _pairs()
    summary, recs = h.register_batch(xs, ys, gts, SearchConfig(k_rot=1, rot_step=0.1, k_trans=2, trans_bin=0.05),
                                     seeds=[10 + k for k in range(5)])
    importlib.reload(h)  # drop the stand-ins
    assert log == [0, 1, 2, 3, 4]
    assert json.loads(json.dumps(_rows(recs))) == ranks[0]["rows"]
    assert [r["seed"] for r in ranks[0]["rows"]] == [10, 11, 12, 13, 14]
    assert summary.n_trials == ranks[0]["n"] == 5 and summary.recall == ranks[0]["recall"]
