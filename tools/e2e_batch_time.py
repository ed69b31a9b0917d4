"""Repeated timings of dses_batch on the bench pairs (e2e stability)."""
import sys, time
sys.path.insert(0, '.')
import torch
import bench
from paper_2502_00115_b200 import dses_batch
name = sys.argv[1] if len(sys.argv) > 1 else 'c2'
c = bench.workload(name); cfg = bench.search_config(c)
pairs, _ = bench.bench_pairs(name, 10)
xs, ys = [p[0] for p in pairs], [p[1] for p in pairs]
dses_batch(xs[:2], ys[:2], cfg)
for rep in range(4):
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); s.record()
    res = dses_batch(xs, ys, cfg)
    e.record(); torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"rep {rep}: events {s.elapsed_time(e):.1f} ms wall {1e3 * (t1 - t0):.1f} ms "
          f"per-reg total {[round(r.elapsed['total'] * 1e3, 1) for r in res]}", flush=True)
