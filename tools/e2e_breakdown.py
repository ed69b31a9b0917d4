import sys, time
sys.path.insert(0, '.')
import bench
from paper_2502_00115_b200 import _native, dses
from paper_2502_00115_b200.engines import prepare
from paper_2502_00115_b200.synth import make_pair
c = bench.workload('c2'); cfg = bench.search_config(c)
for s in range(4):
    x, y, _ = make_pair(c['spec'], 500 + s)
    t0 = time.perf_counter(); p = prepare(x, y, cfg)
    t1 = time.perf_counter(); plan = _native.Plan(p.x, p.y, cfg.trans_bin, p.ilo, p.dims)
    t2 = time.perf_counter(); g = _native.make_grid(cfg.k_rot, p.cos_tab, p.sin_tab, p.center_rot)
    r = plan.search(g, cfg.q, p.code, p.param, p.skip_refine)
    t3 = time.perf_counter(); plan.close()
    t4 = time.perf_counter()
    print(f"prep {1e3*(t1-t0):.2f} plan {1e3*(t2-t1):.2f} search {1e3*(t3-t2):.2f} (dev {r['ms_total']:.2f}, vote {r['ms_vote_kernel']:.2f}) close {1e3*(t4-t3):.2f} ms", flush=True)
for s in range(3):
    x, y, _ = make_pair(c['spec'], 600 + s)
    t0 = time.perf_counter(); res = dses(x, y, cfg); print(f"dses() {1e3*(time.perf_counter()-t0):.2f} ms", flush=True)
