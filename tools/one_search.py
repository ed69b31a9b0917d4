"""One search of a bench pair, twice (stage times, stats): python tools/one_search.py c2"""
import sys
sys.path.insert(0, '.')
import bench
from paper_2502_00115_b200 import _native
from paper_2502_00115_b200.engines import prepare
name = sys.argv[1]
c = bench.workload(name); cfg = bench.search_config(c)
(x, y, _), = bench.bench_pairs(name, 1)[0]
p = prepare(x, y, cfg)
plan = _native.Plan(p.x, p.y, cfg.trans_bin, p.ilo, p.dims)
g = _native.make_grid(cfg.k_rot, p.cos_tab, p.sin_tab, p.center_rot)
for rep in range(2):
    r = plan.search(g, cfg.q, p.code, p.param, p.skip_refine)
print({k: r[k] for k in ('ms_vote', 'ms_select', 'ms_score', 'ms_total', 'ms_vote_kernel', 'candidates_refined', 'rescored', 'launches')})
