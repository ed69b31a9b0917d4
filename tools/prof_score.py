"""One full search on a config whose scoring stage is heavy (default c2local:
L1 on the flat local grid, ~3.4 K candidates screened) -- for ncu of the
screen kernels (second search profiled)."""
import sys
sys.path.insert(0, '.')
import bench
from paper_2502_00115_b200 import _native
from paper_2502_00115_b200.engines import prepare
cfgname = sys.argv[1] if len(sys.argv) > 1 else 'c2local'
c = bench.workload(cfgname); cfg = bench.search_config(c)
x, y, _ = bench.bench_pairs(cfgname, 1)[0][0]
p = prepare(x, y, cfg)
plan = _native.Plan(p.x, p.y, cfg.trans_bin, p.ilo, p.dims)
g = _native.make_grid(cfg.k_rot, p.cos_tab, p.sin_tab, p.center_rot)
for rep in range(2):
    r = plan.search(g, cfg.q, p.code, p.param, p.skip_refine)
print(cfgname, 'kept', r['candidates_evaluated'], 'refined', r['candidates_refined'],
      'score ms', r['ms_score'], 'n', p.x.shape[0], 'm', p.y.shape[0])
