"""Single dses() calls over distinct bench pairs (each reference seen once:
topology built inside the call), median wall time per call.
    python tools/single_call_time.py c2 [lib.so]"""
import sys
import time
sys.path.insert(0, '.')
from paper_2502_00115_b200 import _native  # noqa: E402
if len(sys.argv) > 2:
    _native.LIB_PATH = sys.argv[2]
_native.load(_native.LIB_PATH)
import bench  # noqa: E402
from paper_2502_00115_b200 import dses  # noqa: E402
name = sys.argv[1]
cfg = bench.search_config(bench.workload(name))
pairs, _ = bench.bench_pairs(name, 16)
dses(pairs[0][0], pairs[0][1], cfg)
ts = []
for x, y, _ in pairs[1:]:
    t0 = time.perf_counter()
    r = dses(x, y, cfg)
    ts.append((time.perf_counter() - t0) * 1e3)
ts.sort()
print(name, 'single-call median %.3f ms (min %.3f)' % (ts[len(ts) // 2], ts[0]))
