"""One vote-kernel launch on a synthetic config (for ncu): the search's phase 1
over the first `nrot` rotations of the seed-0 pair (second launch profiled)."""
import sys
sys.path.insert(0, '.')
import bench
from paper_2502_00115_b200 import _native
from paper_2502_00115_b200.engines import prepare
cfgname = sys.argv[1] if len(sys.argv) > 1 else 'c2'
nrot = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
c = bench.workload(cfgname); cfg = bench.search_config(c)
x, y, _ = bench.bench_pairs(cfgname, 1)[0][0]
p = prepare(x, y, cfg)
plan = _native.Plan(p.x, p.y, cfg.trans_bin, p.ilo, p.dims)
g = _native.make_grid(cfg.k_rot, p.cos_tab, p.sin_tab, p.center_rot)
for rep in range(2):
    plan.mode_grid(g, 0, min(nrot, cfg.rotation_count))
print(plan.stats())
