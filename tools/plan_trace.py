"""Plan-construction step times (DSES_TRACE=1) for distinct bench pairs of one
config: python tools/plan_trace.py c2 [pairs]"""
import os
import sys
os.environ["DSES_TRACE"] = "1"
sys.path.insert(0, '.')
import bench  # noqa: E402
from paper_2502_00115_b200 import _native  # noqa: E402
from paper_2502_00115_b200.engines import prepare  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfg = bench.search_config(bench.workload(name))
pairs, _ = bench.bench_pairs(name, int(sys.argv[2]) if len(sys.argv) > 2 else 4)
for x, y, _ in pairs:
    p = prepare(x, y, cfg)
    print("---- plan", flush=True)
    with _native.Plan(p.x, p.y, cfg.trans_bin, p.ilo, p.dims):
        pass
