import sys, time, math, numpy as np
sys.path.insert(0, '.')
import bench
from paper_2502_00115_b200 import _native
from paper_2502_00115_b200.engines import prepare
from paper_2502_00115_b200.synth import make_pair
c = bench.workload(sys.argv[1] if len(sys.argv) > 1 else 'c2'); cfg = bench.search_config(c)
x, y, _ = make_pair(c['spec'], 0)
p = prepare(x, y, cfg)
print('prep ok', x.shape, y.shape, flush=True)
plan = _native.Plan(p.x, p.y, cfg.trans_bin, p.ilo, p.dims)
print('plan', plan.info(), flush=True)
g = _native.make_grid(cfg.k_rot, p.cos_tab, p.sin_tab, p.center_rot)
for n in (1, 16, 256, 4096, cfg.rotation_count):
    t = time.time(); cnt, lin, ties = plan.mode_grid(g, 0, n); dt = time.time() - t
    print('mode_grid', n, f'{dt*1e3:.1f} ms', cnt[:4], plan.stats(), flush=True)
t = time.time(); r = plan.search(g, cfg.q, p.code, p.param, p.skip_refine); print('search', time.time() - t, r, flush=True)
