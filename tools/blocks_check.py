"""Rotation-block vote vs the per-rotation vote kernel on the bench pairs:
identical per-rotation (count, bin, ties) and the vote time per block shape.
    python tools/blocks_check.py c2 [L,L,...] [pairs]"""
import sys
sys.path.insert(0, '.')
import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_2502_00115_b200 import _native  # noqa: E402
from paper_2502_00115_b200.engines import prepare  # noqa: E402

name = sys.argv[1]
# shapes: "7" = 1x1x7, "3x3x3" = a box of 27 rotations; comma-separated
Ls = [tuple(int(a) for a in v.split('x')) if 'x' in v else int(v)
      for v in (sys.argv[2].split(',') if len(sys.argv) > 2 else ['1', '3', '5', '7'])]
npairs = int(sys.argv[3]) if len(sys.argv) > 3 else 1
cfg = bench.search_config(bench.workload(name))
pairs, _ = bench.bench_pairs(name, npairs)
for s in range(npairs):
    x, y, _ = pairs[s]
    p = prepare(x, y, cfg)
    g = _native.make_grid(cfg.k_rot, p.cos_tab, p.sin_tab, p.center_rot)
    R = cfg.rotation_count
    with _native.Plan(p.x, p.y, cfg.trans_bin, p.ilo, p.dims) as plan:
        plan.set_blocks(0)
        ref = plan.mode_grid(g, 0, R)
        st0 = plan.stats()
        t0 = min(plan.search(g, cfg.q, p.code, p.param, p.skip_refine)['ms_vote_kernel'] for _ in range(3))
        print(f'{name} pair {s} L=0: vote {t0:.3f} ms pairs/rot {st0["pairs"] / R:.0f} '
              f'votes/rot {st0["votes"] / R:.0f} rechecks {st0["rechecks"]}', flush=True)
        for L in Ls:
            plan.set_blocks(L)
            got = plan.mode_grid(g, 0, R)
            st = plan.stats()
            bad = [k for k in range(3) if not np.array_equal(ref[k], got[k])]
            nbad = int(np.sum((ref[0] != got[0]) | (ref[1] != got[1]) | (ref[2] != got[2])))
            t = min(plan.search(g, cfg.q, p.code, p.param, p.skip_refine)['ms_vote_kernel'] for _ in range(3))
            print(f'{name} pair {s} L={L}: vote {t:.3f} ms ({t0 / t:.2f}x) entries/rot {st["pairs"] / R:.0f} '
                  f'votes/rot {st["votes"] / R:.0f} rechecks {st["rechecks"]} '
                  f'{"IDENTICAL" if not bad else f"MISMATCH {bad} rows {nbad}"}', flush=True)
            if bad:
                idx = np.nonzero((ref[0] != got[0]) | (ref[1] != got[1]))[0][:5]
                print('   first rows', idx.tolist(), [(int(ref[0][i]), int(got[0][i]), int(ref[1][i]),
                                                        int(got[1][i])) for i in idx], flush=True)
