"""Host plan-construction time per config (dses_plan_create: tiling, dedup
components, fixed point, uploads) -- the e2e overhead on top of the search."""
import sys
import time
sys.path.insert(0, '.')
import bench
from paper_2502_00115_b200 import _native
from paper_2502_00115_b200.engines import prepare
for name in sys.argv[1:] or ["c2", "c4"]:
    c = bench.workload(name)
    cfg = bench.search_config(c)
    x, y, _ = bench.bench_pairs(name, 1)[0][0]
    best = 1e9
    for _ in range(5):
        t0 = time.perf_counter()
        p = prepare(x, y, cfg)
        with _native.Plan(p.x, p.y, cfg.trans_bin, p.ilo, p.dims):
            pass
        best = min(best, time.perf_counter() - t0)
    print(f"{name}: prepare + plan create/destroy {best * 1e3:.2f} ms (n={x.shape[0]}, m={y.shape[0]})")
