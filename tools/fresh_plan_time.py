"""Device time of the first and later searches on fresh plans (one plan per
pair): exposes per-plan first-launch costs.
    python tools/fresh_plan_time.py c4 [block_len|-1 default] [reserve 0/1]"""
import sys
sys.path.insert(0, '.')
import bench  # noqa: E402
from paper_2502_00115_b200 import _native  # noqa: E402
from paper_2502_00115_b200.engines import prepare  # noqa: E402

name = sys.argv[1]
L = int(sys.argv[2]) if len(sys.argv) > 2 else -1
res = int(sys.argv[3]) if len(sys.argv) > 3 else 0
cfg = bench.search_config(bench.workload(name))
pairs, _ = bench.bench_pairs(name, 4)
for s in range(4):
    x, y, _ = pairs[s]
    p = prepare(x, y, cfg)
    g = _native.make_grid(cfg.k_rot, p.cos_tab, p.sin_tab, p.center_rot)
    with _native.Plan(p.x, p.y, cfg.trans_bin, p.ilo, p.dims) as plan:
        if L >= 0:
            plan.set_blocks(L)
        if res:
            plan.reserve(cfg.rotation_count)
        ts = []
        for rep in range(3):
            r = plan.search(g, cfg.q, p.code, p.param, p.skip_refine)
            ts.append((round(r['ms_vote_kernel'], 3), round(r['ms_total'], 3)))
        print(name, 'L', L, 'reserve', res, 'pair', s, ts, flush=True)
