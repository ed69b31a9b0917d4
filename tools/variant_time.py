"""Vote-kernel / search timing of one config (best of 3 searches) for A/B work."""
import sys
sys.path.insert(0, '.')
from paper_2502_00115_b200 import _native
if len(sys.argv) > 2:
    _native.LIB_PATH = sys.argv[2]
_native.load(_native.LIB_PATH)
import bench
from paper_2502_00115_b200.engines import prepare
c = bench.workload(sys.argv[1])
cfg = bench.search_config(c)
import os
seeds = [int(v) for v in os.environ.get('SEEDS', '0').split(',')]
vsum = tsum = 0.0
for seed in seeds:  # best of 3 per seed pair, summed over the seeds
    x, y, _ = bench.bench_pairs(sys.argv[1], 1, seed)[0][0]
    p = prepare(x, y, cfg)
    plan = _native.Plan(p.x, p.y, cfg.trans_bin, p.ilo, p.dims)
    g = _native.make_grid(cfg.k_rot, p.cos_tab, p.sin_tab, p.center_rot)
    best, tot = 1e9, 1e9
    for rep in range(3):
        r = plan.search(g, cfg.q, p.code, p.param, p.skip_refine)
        best = min(best, r['ms_vote_kernel'])
        tot = min(tot, r['ms_total'])
    vsum += best
    tsum += tot
best, tot = vsum / len(seeds), tsum / len(seeds)
R = cfg.rotation_count
print(f"{sys.argv[1]} R={R} vote {best:.3f} ms ({R / best * 1e3:.3e} rot/s) total {tot:.3f} ms "
      f"pairs/rot {r['pairs_evaluated'] / R:.0f} votes/rot {r['votes'] / R:.0f} "
      f"rechecks {r['rechecks']} info {plan.info()} winner {r['winner_row']} M* {r['mstar']} "
      f"refined {r['candidates_refined']} rescored {r['rescored']}", flush=True)
