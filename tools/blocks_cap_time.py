"""Block-kernel vote time against the list slab size (entries per CTA; the
slab stride sets where each CTA's list lands in L2): python tools/blocks_cap_time.py c4 CAP,CAP,..."""
import sys
sys.path.insert(0, '.')
import bench  # noqa: E402
from paper_2502_00115_b200 import _native  # noqa: E402
from paper_2502_00115_b200.engines import prepare  # noqa: E402

name = sys.argv[1]
caps = [int(c) for c in sys.argv[2].split(',')]
cfg = bench.search_config(bench.workload(name))
for s, (x, y, _) in enumerate(bench.bench_pairs(name, 2)[0]):
    p = prepare(x, y, cfg)
    g = _native.make_grid(cfg.k_rot, p.cos_tab, p.sin_tab, p.center_rot)
    with _native.Plan(p.x, p.y, cfg.trans_bin, p.ilo, p.dims) as plan:
        for cap in caps * 2:
            plan.set_blocks((1, 3, 3), cap)
            t = min(plan.search(g, cfg.q, p.code, p.param, p.skip_refine)['ms_vote_kernel'] for _ in range(3))
            print(f'{name} pair {s} cap {cap}: vote {t:.3f} ms', flush=True)
