"""c3 (753,571 rotations) search time, per-rotation vs rotation-block vote kernel."""
import sys, time
sys.path.insert(0,'.')
import bench, torch
from paper_2502_00115_b200 import _native
from paper_2502_00115_b200.engines import prepare
cfg=bench.search_config(bench.workload('c3'))
(x,y,_),=bench.bench_pairs('c3',1)[0]
p=prepare(x,y,cfg)
g=_native.make_grid(cfg.k_rot,p.cos_tab,p.sin_tab,p.center_rot)
R=cfg.rotation_count
with _native.Plan(p.x,p.y,cfg.trans_bin,p.ilo,p.dims) as plan:
    for shape in (0,(1,3,3),(3,3,3),(2,4,4),(1,5,5)):
        plan.set_blocks(shape)
        plan.mode_grid(g, 0, 91*91*2)
        torch.cuda.synchronize(); t0=time.perf_counter()
        r=plan.mode_grid(g, 0, 91*91*9)
        t1=time.perf_counter()
        print(shape, round((t1-t0)*1e3,2), 'ms for', 91*91*9, 'rotations', flush=True)
