"""dses_batch wall time against the number of plans built ahead (engines._BUILD_AHEAD):
    python tools/batch_ahead_time.py c4 AHEAD [lib.so]"""
import sys, time
sys.path.insert(0, '.')
from paper_2502_00115_b200 import _native
if len(sys.argv) > 3:
    _native.LIB_PATH = sys.argv[3]
_native.load(_native.LIB_PATH)
import torch, bench
from paper_2502_00115_b200 import engines, dses_batch
name = sys.argv[1]; ahead = int(sys.argv[2])
engines._BUILD_AHEAD = ahead
engines._BUILD_POOL = None
c = bench.workload(name); cfg = bench.search_config(c)
pairs, _ = bench.bench_pairs(name, 10, 13)
xs, ys = [p[0] for p in pairs], [p[1] for p in pairs]
dses_batch(xs[:3], ys[:3], cfg)
flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
ts = []
for rep in range(5):
    torch.cuda.synchronize(); flush.zero_()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); dses_batch(xs, ys, cfg); e.record(); torch.cuda.synchronize()
    ts.append(s.elapsed_time(e))
print(name, 'ahead', ahead, 'batch ms', [round(t, 1) for t in ts])
