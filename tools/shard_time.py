import sys, time
sys.path.insert(0, '.')
import bench
from paper_2502_00115_b200 import dses
from paper_2502_00115_b200.distributed import dses_sharded
c = bench.workload('c3'); cfg = bench.search_config(c)
(x, y, _), = bench.bench_pairs('c3', 1)[0]
for i in range(3):
    t = time.perf_counter(); r = dses_sharded(x, y, cfg); t1 = time.perf_counter()
    print('sharded', round((t1 - t) * 1e3, 1), {k: round(v * 1e3, 1) if isinstance(v, float) else v for k, v in r.elapsed.items()})
    t = time.perf_counter(); r2 = dses(x, y, cfg); t1 = time.perf_counter()
    print('dses', round((t1 - t) * 1e3, 1), {k: round(v * 1e3, 1) for k, v in r2.elapsed.items() if isinstance(v, float)})
