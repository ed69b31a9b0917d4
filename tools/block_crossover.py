"""Per-rotation vs rotation-block vote time as the translation window grows
against the cloud (calibrates the block heuristic, kBlockWindowFrac).
    python tools/block_crossover.py c4 4,10,20,40"""
import sys
from dataclasses import replace
sys.path.insert(0, '.')
import bench  # noqa: E402
from paper_2502_00115_b200 import _native  # noqa: E402
from paper_2502_00115_b200.engines import prepare  # noqa: E402

name = sys.argv[1]
ks = [int(v) for v in sys.argv[2].split(',')]
base = bench.search_config(bench.workload(name))
(x, y, _), = bench.bench_pairs(name, 1)[0]
ext = (y.max(0) - y.min(0)).max()
for kt in ks:
    cfg = replace(base, k_trans=kt)
    p = prepare(x, y, cfg)
    g = _native.make_grid(cfg.k_rot, p.cos_tab, p.sin_tab, p.center_rot)
    win = (2 * kt + 1) * cfg.trans_bin
    with _native.Plan(p.x, p.y, cfg.trans_bin, p.ilo, p.dims) as plan:
        default = plan.blocks()
        out = []
        for shape in (0, (1, 3, 3)):
            plan.set_blocks(shape)
            t = min(plan.search(g, cfg.q, p.code, p.param, p.skip_refine)['ms_vote_kernel'] for _ in range(3))
            out.append(t)
    print(f'{name} k_trans={kt} window {win * 1e3:.0f} mm = {win / ext:.3f} of the cloud: per-rotation '
          f'{out[0]:.3f} ms, blocks 1x3x3 {out[1]:.3f} ms ({out[0] / out[1]:.2f}x); default {default}', flush=True)
