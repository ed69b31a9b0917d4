"""Host-side breakdown of one dses() call (single registration, public API):
prepare, grid tables, plan construction, reserve, search (device), close,
result objects.  python tools/e2e_breakdown.py [c1|c2|c4]"""
import sys
import time
sys.path.insert(0, '.')
import bench  # noqa: E402
from paper_2502_00115_b200 import _native, dses  # noqa: E402
from paper_2502_00115_b200.engines import _result, prepare  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else 'c2'
c = bench.workload(name)
cfg = bench.search_config(c)
pairs, _ = bench.bench_pairs(name, 4)
for s in range(4):
    x, y, _ = pairs[s]
    t0 = time.perf_counter(); p = prepare(x, y, cfg)
    t1 = time.perf_counter(); g = _native.make_grid(cfg.k_rot, p.cos_tab, p.sin_tab, p.center_rot)
    t2 = time.perf_counter(); plan = _native.Plan(p.x, p.y, cfg.trans_bin, p.ilo, p.dims)
    t3 = time.perf_counter(); plan.reserve(cfg.rotation_count)
    t4 = time.perf_counter(); r = plan.search(g, cfg.q, p.code, p.param, p.skip_refine)
    t5 = time.perf_counter(); plan.close()
    t6 = time.perf_counter(); res = _result(p, cfg, r, t0)
    t7 = time.perf_counter()
    print(f"prep {1e3*(t1-t0):.3f} grid {1e3*(t2-t1):.3f} plan {1e3*(t3-t2):.3f} reserve {1e3*(t4-t3):.3f} "
          f"search {1e3*(t5-t4):.3f} (dev {r['ms_total']:.3f}) close {1e3*(t6-t5):.3f} result {1e3*(t7-t6):.3f} ms",
          flush=True)
for s in range(4):
    x, y, _ = pairs[s]
    t0 = time.perf_counter(); res = dses(x, y, cfg); t1 = time.perf_counter()
    print(f"dses() {1e3*(t1-t0):.3f} ms (device {res.elapsed['device_total'] * 1e3:.3f})", flush=True)
