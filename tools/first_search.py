"""Stage times of the first vs second search on fresh plans (c2 pairs): shows
one-time per-plan costs (scratch growth) inside the device timeline."""
import sys
sys.path.insert(0, '.')
import bench
from paper_2502_00115_b200 import _native
from paper_2502_00115_b200.engines import prepare
from paper_2502_00115_b200.synth import make_pair
c = bench.workload(sys.argv[1] if len(sys.argv) > 1 else 'c2')
cfg = bench.search_config(c)
plans = []
for s in range(8):
    x, y, _ = make_pair(c['spec'], s)
    p = prepare(x, y, cfg)
    plans.append((p, _native.Plan(p.x, p.y, cfg.trans_bin, p.ilo, p.dims),
                  _native.make_grid(cfg.k_rot, p.cos_tab, p.sin_tab, p.center_rot)))
for s, (p, plan, g) in enumerate(plans):
    out = []
    for rep in range(2):
        r = plan.search(g, cfg.q, p.code, p.param, p.skip_refine)
        out.append(f"vote {r['ms_vote']:.2f} sel {r['ms_select']:.2f} score {r['ms_score']:.2f} total {r['ms_total']:.2f}")
    print(s, ' | '.join(out), flush=True)
