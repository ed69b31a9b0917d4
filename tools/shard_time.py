"""Single-rank timing of the device-resident sharded search (distributed.
ShardedSearch) vs the fused single-GPU search, and its host overhead: wall
time of run() minus the device time of the same launches (CUDA events on the
stream).  python tools/shard_time.py [c3|c5K10|c5K50]"""
import math
import sys
import time

sys.path.insert(0, '.')
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2502_00115_b200 import dses  # noqa: E402
from paper_2502_00115_b200.distributed import ShardedSearch  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else 'c3'
if name.startswith('c5K'):
    K = int(name[3:])
    from dataclasses import replace
    cfg = replace(bench.search_config(bench.workload('c2')), k_rot=K, rot_step=math.radians(45.0 / K))
    pair = 'c2'
else:
    cfg = bench.search_config(bench.workload(name))
    pair = name
(x, y, _), = bench.bench_pairs(pair, 1)[0]
torch.cuda.set_device(0)
with ShardedSearch(x, y, cfg) as s:
    s.run()
    for i in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t = time.perf_counter(); e0.record(); r = s.run(); e1.record(); t1 = time.perf_counter()
        torch.cuda.synchronize()
        dev = e0.elapsed_time(e1)
        print(f'{name} R={cfg.rotation_count} sharded(world 1): wall {(t1 - t) * 1e3:.3f} ms, device '
              f'{dev:.3f} ms, host-over-device {(t1 - t) * 1e3 - dev:.3f} ms, winner {r.best.grid_coords} '
              f'refined {r.candidates_refined} protocol {r.elapsed["protocol"]}', flush=True)
r2 = dses(x, y, cfg)
print(f'{name} dses: winner {r2.best.grid_coords} refined {r2.candidates_refined} '
      f'device {r2.elapsed["device_total"] * 1e3:.3f} ms total {r2.elapsed["total"] * 1e3:.3f} ms')
assert r.best.grid_coords == r2.best.grid_coords and r.best_error == r2.best_error
assert r.best_inliers == r2.best_inliers and r.candidates_refined == r2.candidates_refined
