"""cProfile of dses_batch on c1 pairs (host-side Python cost per registration)."""
import sys, cProfile, pstats
sys.path.insert(0, '.')
import bench
from paper_2502_00115_b200 import dses_batch
cfg = bench.search_config(bench.workload('c1'))
pairs, _ = bench.bench_pairs('c1', 16)
xs, ys = [p[0] for p in pairs], [p[1] for p in pairs]
dses_batch(xs, ys, cfg)
pr = cProfile.Profile(); pr.enable()
for _ in range(5): dses_batch(xs, ys, cfg)
pr.disable()
pstats.Stats(pr).sort_stats('tottime').print_stats(18)
