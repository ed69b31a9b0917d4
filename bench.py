#!/usr/bin/env python
"""DSES throughput on B200: rotation candidates/s and registrations/s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl b200|reference]

One step = one full DSES registration (phase 1 vote over every grid rotation,
phase 2 selection, phase 3 screen + exact re-score, winner inlier count) of one
ModelNet40-shaped pair.  Default workload = BASELINE.json configs[1]
(SURVEY.md 8(d) c2): 1024-pt reference / 717-pt partial, k_rot=15 @ 3 deg
(29,791 rotations), k_trans=20 @ 25 mm (41^3 bins), truncated-L1 at 5 bins.
Inputs (--inputs benchgen, the default): the reference generator's own clouds
for seeds 0..15, committed as bench_data/benchgen_<cfg>.npz;
--inputs synth uses the independent generator paper_2502_00115_b200/synth.py.

`--gpus N` launches N ranks itself (torch.distributed.run, one process per
GPU) when not already under torchrun, and checks WORLD_SIZE == N.  Every rank
registers its own pairs (replicas, weak scaling, no data-path collective;
SURVEY.md 8(e)); the timed region is bracketed by a barrier + synchronize,
timed with CUDA events on the launching stream, and the max over ranks is
reported.  Rank 0 prints ONE JSON line.  Its "rotation_sharded" list is the
other multi-GPU mode, measured first-class (value, ms_per_step, steps per
entry): one registration's rotation grid split over ALL ranks
(distributed.ShardedSearch: M* and the min-loc winner reduced in device
memory by NCCL all_reduces), strong scaling, for c3 (753,571 rotations) and the
c5 sweep points >= 10^6 rotations (skip with --no-sharded).

`--impl reference` times the reference's own CPU implementation on the box's
host cores, on rank 0 only: the unmodified `gridreg` package (pure Python +
numba, installed offline into baseline/_ref, every host thread) through its
public `gridreg.dses` on the same pair, full registrations when they
fit the time budget, else `gridreg.mode_search._mode_batch` (phase 1, 99.8% of
the reference's time) over a contiguous rotation slice.  Without baseline/_ref
it falls back to the oracle port (oracle/gridreg_oracle.c, the C restatement
of the reference's numba kernels).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "rotation_candidates_per_sec"
UNIT = "rot/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2")
    ap.add_argument("--metric", default=None, help="override the config's metric name")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=20.0,
                    help="wall-clock budget of the CPU baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--inputs", default="benchgen", choices=["benchgen", "synth"],
                    help="clouds: the reference generator's (committed) or synth.py's")
    ap.add_argument("--no-sharded", action="store_true",
                    help="skip the rotation-grid-sharded registration (distributed.dses_sharded)")
    return ap.parse_args()


def workload(name, metric_override=None):
    from paper_2502_00115_b200.synth import CONFIGS
    c = dict(CONFIGS[name])
    if metric_override:
        c["metric"] = metric_override
    return c


def bench_pairs(config, count, offset=0, inputs="benchgen"):
    """`count` (source, reference, truth) pairs of a workload.  "benchgen":
    the reference generator's own clouds for the listed seeds
    (bench_data/benchgen_<cfg>.npz, made by bench_data/make_bench_data.py;
    SURVEY.md 8(d)), cycled when more are needed; configs without a file, or
    inputs="synth", use the independent generator synth.make_pair."""
    from paper_2502_00115_b200 import RigidTransform
    from paper_2502_00115_b200.synth import make_pair
    path = os.path.join(ROOT, "bench_data", f"benchgen_{config}.npz")
    if inputs == "benchgen" and os.path.exists(path):
        d = np.load(path)
        n = int(d["count"])
        out = []
        for s in range(count):
            k = (offset + s) % n
            out.append((d[f"x{k}"], d[f"y{k}"], RigidTransform(d[f"gt_R{k}"], d[f"gt_t{k}"])))
        return out, f"reference benchgen clouds (bench_data/benchgen_{config}.npz, seeds 0..{n - 1})"
    c = workload(config)
    return ([make_pair(c["spec"], offset + s) for s in range(count)],
            "synthetic (seeded ModelNet40-shaped pairs, paper_2502_00115_b200/synth.py)")


def search_config(c):
    from paper_2502_00115_b200 import ErrorMetric, SearchConfig
    metric = ErrorMetric.from_name(c["metric"], c["trans_bin"])
    return SearchConfig(k_rot=c["k_rot"], rot_step=math.radians(c["rot_step_deg"]),
                        k_trans=c["k_trans"], trans_bin=c["trans_bin"], metric=metric)


def describe(name, c, cfg, n, m):
    return (f"{name}: synthetic ModelNet40-shaped pair, {m}-pt reference / {n}-pt partial source, "
            f"k_rot={c['k_rot']} @ {c['rot_step_deg']} deg ({cfg.rotation_count} rotations), "
            f"k_trans={c['k_trans']} @ {c['trans_bin'] * 1000:g} mm ({2 * c['k_trans'] + 1}^3 bins), "
            f"metric {cfg.metric.kind}" + (f" (param {cfg.metric.param:g})" if cfg.metric.param else ""))


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.path = os.path.join("/tmp", f"dses_clocks_{os.getpid()}.csv")

    def __enter__(self):
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=self.fh, stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None
            return self
        # nvidia-smi's start-up (NVML init) must not overlap the timed steps:
        # wait for its first sample before the caller starts timing
        t0 = time.time()
        while time.time() - t0 < 5.0 and self.proc.poll() is None:
            if os.path.getsize(self.path) > 0:
                break
            time.sleep(0.01)
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.fh.close()

    def summary(self):
        if self.proc is None or not os.path.exists(self.path):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            p = [v.strip() for v in line.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                smax.append(float(p[2]))
            except ValueError:
                continue
            for nm, v in zip(names, p[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        busy = [s for s in sm if s > 0.5 * max(sm)] or sm
        return {"sm_mhz": float(np.median(busy)), "sm_max_mhz": max(smax),
                "samples": len(sm), "reasons": sorted(reasons)}


REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def load_reference():
    """The unmodified reference package from baseline/_ref (None when absent).
    numba's thread pool gets every host thread; its JIT cache goes to /tmp."""
    if not os.path.isdir(os.path.join(REF_DIR, "gridreg")):
        return None
    os.environ.setdefault("NUMBA_NUM_THREADS", str(os.cpu_count() or 1))
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/dses_numba_cache")
    if REF_DIR not in sys.path:
        sys.path.append(REF_DIR)
    try:
        import gridreg  # noqa: F401
        from gridreg import engines, metrics, mode_search
    except Exception as e:  # pragma: no cover - depends on the box
        print(f"[bench] reference package unusable ({e}); using the oracle port", file=sys.stderr)
        return None
    return engines, metrics, mode_search


def ref_config(ref, cfg):
    engines, metrics, _ = ref
    m = cfg.metric
    metric = metrics.ErrorMetric(m.kind, m.param)
    return engines.SearchConfig(k_rot=cfg.k_rot, rot_step=cfg.rot_step, k_trans=cfg.k_trans,
                                trans_bin=cfg.trans_bin, q=cfg.q, metric=metric)


def ref_phase1_slice(ref, x, y, cfg, r0, count):
    """gridreg.mode_search._mode_batch over rotations [r0, r0+count) of the
    reference's own grid (geometry.build_rotation_grid)."""
    engines, _, mode_search = ref
    from gridreg import geometry
    grid = geometry.build_rotation_grid(cfg.k_rot, cfg.rot_step)
    rots = np.ascontiguousarray(grid.matrices[r0:r0 + count])
    ilo = np.full(3, -cfg.k_trans, dtype=np.int64)
    dims = np.full(3, 2 * cfg.k_trans + 1, dtype=np.int64)
    t0 = time.perf_counter()
    out = mode_search._mode_batch(rots, x, y, cfg.trans_bin, ilo, dims)
    return time.perf_counter() - t0, out


def reference_rate(ref, x, y, cfg, budget_s):
    """Reference rotations/s on the step-0 pair: one full gridreg.dses when it
    fits `budget_s` (after a JIT warm-up call on a tiny grid), else phase 1
    over a rotation slice.  Returns (value, sample description, seconds)."""
    engines, _, _ = ref
    rcfg = ref_config(ref, cfg)
    total = cfg.rotation_count
    small = engines.SearchConfig(k_rot=1, rot_step=cfg.rot_step, k_trans=cfg.k_trans,
                                 trans_bin=cfg.trans_bin, q=cfg.q, metric=rcfg.metric)
    engines.dses(x, y, small)  # numba JIT / cache load, untimed
    cal = min(total, 4 * (os.cpu_count() or 1) * 16)
    dt_cal, _ = ref_phase1_slice(ref, x, y, cfg, 0, cal)
    est_full = dt_cal / cal * total * 1.05
    if est_full <= budget_s:
        t0 = time.perf_counter()
        res = engines.dses(x, y, rcfg)
        dt = time.perf_counter() - t0
        return total / dt, (f"one full gridreg.dses registration ({total} rotations, "
                            f"phase1 {res.elapsed['phase1']:.2f} s of {dt:.2f} s)"), dt
    sample = int(min(total, max(cal, budget_s * cal / max(dt_cal, 1e-9))))
    dt, _ = ref_phase1_slice(ref, x, y, cfg, 0, sample)
    return sample / dt, (f"gridreg.mode_search._mode_batch (phase 1, 99.8% of the reference's "
                         f"time, SURVEY.md 3) over rotations [0, {sample}) of {total}, "
                         f"{dt:.2f} s wall"), dt


def cpu_baseline(x, y, cfg, c, budget_s, gpu_check=None):
    """The reference (numba, all host threads) when baseline/_ref is present,
    else the oracle C port, on a bounded sample of the step-0 pair."""
    ref = load_reference()
    if ref is not None:
        value, sample, _ = reference_rate(ref, x, y, cfg, budget_s)
        out = {"value": value, "unit": UNIT, "cores": int(os.environ["NUMBA_NUM_THREADS"]),
               "kind": "reference", "sample": sample + "; registrations/s = value / "
                                                      f"{cfg.rotation_count}",
               "registrations_per_sec_extrapolated": value / cfg.rotation_count}
        if gpu_check is not None:
            n = min(cfg.rotation_count, 2048)
            _, (rc, rl, rt) = ref_phase1_slice(ref, x, y, cfg, 0, n)
            g_counts, g_lins, g_ties = gpu_check(n)
            out["gpu_parity_on_sample"] = bool(np.array_equal(g_counts, rc)
                                               and np.array_equal(g_lins, rl)
                                               and np.array_equal(g_ties, rt))
        return out
    from oracle import oracle as O
    nthreads = O.max_threads()
    ilo = np.full(3, -cfg.k_trans, dtype=np.int64)
    dims = np.full(3, 2 * cfg.k_trans + 1, dtype=np.int64)
    grid = (cfg.k_rot, cfg.rot_step, None)
    total = cfg.rotation_count
    t0 = time.perf_counter()
    cal = min(total, 8 * nthreads)
    O.mode_batch(x, y, cfg.trans_bin, ilo, dims, grid=grid, r_begin=0, r_count=cal,
                 nthreads=nthreads)
    dt = max(time.perf_counter() - t0, 1e-6)
    sample = int(min(total, max(cal, budget_s * cal / dt)))
    t0 = time.perf_counter()
    counts, lins, ties = O.mode_batch(x, y, cfg.trans_bin, ilo, dims, grid=grid, r_begin=0,
                                      r_count=sample, nthreads=nthreads)
    dt = time.perf_counter() - t0
    rate = sample / dt
    out = {"value": rate, "unit": UNIT, "cores": nthreads, "kind": "port",
           "sample": (f"phase 1 (vote, {100 * 0.998:.1f}% of reference time, SURVEY.md 3) over "
                      f"rotations [0, {sample}) of {total} of the step-0 pair, {dt:.2f} s wall; "
                      f"registrations/s extrapolated = value / {total}"),
           "registrations_per_sec_extrapolated": rate / total}
    if gpu_check is not None:
        g_counts, g_lins, g_ties = gpu_check(sample)
        out["gpu_parity_on_sample"] = bool(np.array_equal(g_counts, counts)
                                           and np.array_equal(g_lins, lins)
                                           and np.array_equal(g_ties, ties))
    return out


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    sys.path.insert(0, ROOT)
    c = workload(args.config, args.metric)
    cfg = search_config(c)
    (x, y, _), = bench_pairs(args.config, 1, 0, args.inputs)[0]
    ref = load_reference()
    if ref is not None:
        return run_reference_package(args, ref, c, cfg, x, y)
    from oracle import oracle as O
    nthreads = O.max_threads()
    ilo = np.full(3, -cfg.k_trans, dtype=np.int64)
    dims = np.full(3, 2 * cfg.k_trans + 1, dtype=np.int64)
    total = cfg.rotation_count
    # size one step's sample so the whole --steps/--warmup run stays ~1-2 minutes
    t0 = time.perf_counter()
    cal = min(total, 8 * nthreads)
    O.mode_batch(x, y, cfg.trans_bin, ilo, dims, grid=(cfg.k_rot, cfg.rot_step, None),
                 r_count=cal, nthreads=nthreads)
    per_rot = max(time.perf_counter() - t0, 1e-6) / cal
    per_step_s = min(10.0, 90.0 / max(1, args.steps + args.warmup))
    sample = int(max(nthreads, min(total, per_step_s / per_rot)))
    times = []
    for s in range(args.warmup + args.steps):
        r0 = (s * sample) % max(1, total - sample + 1)
        t0 = time.perf_counter()
        O.mode_batch(x, y, cfg.trans_bin, ilo, dims, grid=(cfg.k_rot, cfg.rot_step, None),
                     r_begin=r0, r_count=sample, nthreads=nthreads)
        if s >= args.warmup:
            times.append(time.perf_counter() - t0)
    tot = sum(times)
    value = sample * len(times) / tot
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot / len(times), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": bench_pairs(args.config, 1, 0, args.inputs)[1],
        "config": {"workload": describe(args.config, c, cfg, x.shape[0], y.shape[0]),
                   "metric": cfg.metric.kind, "rotations": cfg.rotation_count},
        "l2_flush": "n/a (CPU)",
        "registrations_per_sec": value / total,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": nthreads, "kind": "port",
                         "sample": f"each step: phase 1 over {sample} consecutive rotations of "
                                   f"{total} (oracle/gridreg_oracle.c, the C restatement of the "
                                   f"reference numba kernels); registrations/s = value / {total}"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_reference_package(args, ref, c, cfg, x, y):
    """--impl reference with the unmodified gridreg package (numba)."""
    engines, _, _ = ref
    rcfg = ref_config(ref, cfg)
    total = cfg.rotation_count
    nsteps = args.warmup + args.steps
    value0, _, dt0 = reference_rate(ref, x, y, cfg, budget_s=150.0 / max(1, nsteps))
    per_step = min(150.0 / max(1, nsteps), 60.0)
    full = total / value0 <= per_step
    sample = total if full else int(max(16, min(total, per_step * value0)))
    times = []
    for s in range(nsteps):
        if full:
            t0 = time.perf_counter()
            engines.dses(x, y, rcfg)
            dt = time.perf_counter() - t0
        else:
            r0 = (s * sample) % max(1, total - sample + 1)
            dt, _ = ref_phase1_slice(ref, x, y, cfg, r0, sample)
        if s >= args.warmup:
            times.append(dt)
    tot = sum(times)
    value = sample * len(times) / tot
    cores = int(os.environ["NUMBA_NUM_THREADS"])
    what = (f"each step: one full gridreg.dses registration of the pair ({total} rotations)"
            if full else
            f"each step: gridreg.mode_search._mode_batch (phase 1) over {sample} consecutive "
            f"rotations of {total}; registrations/s = value / {total}")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot / len(times), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": bench_pairs(args.config, 1, 0, args.inputs)[1],
        "config": {"workload": describe(args.config, c, cfg, x.shape[0], y.shape[0]),
                   "metric": cfg.metric.kind, "rotations": cfg.rotation_count},
        "l2_flush": "n/a (CPU)",
        "registrations_per_sec": value / total,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference",
                         "sample": what + " (unmodified gridreg 0.1.0 from baseline/_ref, "
                                          "numba parallel, NUMBA_NUM_THREADS=" + str(cores) + ")"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


SHARDED = (  # (name, workload, pair config, k_rot override, steps): SURVEY.md 8(d) c3 and c5 >= 10^6
    ("c3", "c3", "c3", None, 3),
    ("c5_K50", "c2", "c2", 50, 3),
    ("c5_K108", "c2", "c2", 108, 2),
)


def sharded_measurements(args, rank, world, local):
    """The rotation-grid-sharded mode, first-class: one registration's grid
    split over ALL ranks (distributed.ShardedSearch: every rank votes a
    contiguous slice; M* and the min-loc (error, rotation) key are reduced
    in device memory by four NCCL all_reduces; one host read per
    registration).  Strong scaling -- the work per step is fixed: c3 (753,571
    rotations, noisy + 20% outliers, L1) and the c5 sweep points >= 10^6
    rotations (K = 50: 1,030,301; K = 108: 10,218,313) on the c2 pair.  Plans
    are built before timing; one warm-up registration; CUDA events around the
    timed registrations (each ends with its host read), max over ranks."""
    import torch
    import torch.distributed as dist
    from dataclasses import replace
    from paper_2502_00115_b200.distributed import ShardedSearch
    out = []
    for name, wl, pair_cfg, K, steps in SHARDED:
        try:
            cfg = search_config(workload(wl))
            if K is not None:
                cfg = replace(cfg, k_rot=K, rot_step=math.radians(45.0 / K))
            (x, y, _), = bench_pairs(pair_cfg, 1, 0, args.inputs)[0]
            with ShardedSearch(x, y, cfg, device=local) as s:
                s.run()  # warm
                torch.cuda.synchronize()
                if world > 1:
                    dist.barrier()
                t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                t0.record()
                for _ in range(steps):
                    res = s.run()
                t1.record()
                torch.cuda.synchronize()
            t = torch.tensor([t0.elapsed_time(t1)], dtype=torch.float64, device="cuda")
            w = torch.tensor(list(res.best.grid_coords), dtype=torch.float64, device="cuda")
            same = True
            if world > 1:
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                lo, hi = w.clone(), w.clone()
                dist.all_reduce(lo, op=dist.ReduceOp.MIN)
                dist.all_reduce(hi, op=dist.ReduceOp.MAX)
                same = bool(torch.equal(lo, hi))
            ms = float(t.item()) / steps
            R = cfg.rotation_count
            out.append({
                "name": name, "metric": METRIC, "value": R / (ms * 1e-3), "unit": UNIT,
                "ms_per_step": ms, "steps": steps, "n_gpus": world, "scaling": "strong",
                "registrations_per_sec": 1e3 / ms, "rotations": R,
                "config": {"workload": describe(name, workload(wl), cfg, x.shape[0], y.shape[0]),
                           "metric": cfg.metric.kind, "rotations": R},
                "parallelism": f"rotation grid split over {world} rank(s)",
                "collectives": "per registration: all_reduce MAX (M*), MIN (error bits), "
                               "MIN (row<<32|bin), SUM (valid, kept, miss, overflow) on a "
                               "device-resident int64[7] record",
                "winner_grid": list(res.best.grid_coords), "winner_identical_on_all_ranks": same,
                "candidates_refined": int(res.candidates_refined),
                "protocol": res.elapsed.get("protocol")})
        except Exception as exc:  # reported, never fatal for the headline line
            out.append({"name": name, "error": f"{type(exc).__name__}: {exc}"})
    return out


EXTRA_WORKLOADS = ("c1", "c4")  # BASELINE.json configs[0] and configs[3], beside the c2 headline


def workload_line(name, args, rank, world, local, steps=10, warmup=3):
    """One BASELINE config measured like the headline, first-class: device-
    resident registrations (plans built before timing, L2 flushed between
    steps, CUDA events, max over ranks), and end to end through the public
    API from host numpy buffers -- dses_batch (plan construction of k+1
    overlapped with the search of k) and single dses() calls."""
    import torch
    import torch.distributed as dist
    from paper_2502_00115_b200 import _native, dses, dses_batch
    from paper_2502_00115_b200.engines import prepare
    try:
        c = workload(name)
        cfg = search_config(c)
        nsteps = warmup + steps
        pairs, _ = bench_pairs(name, nsteps, rank * nsteps, args.inputs)
        preps = [prepare(x, y, cfg) for x, y, _ in pairs]
        plans = [_native.Plan(p.x, p.y, cfg.trans_bin, p.ilo, p.dims, local) for p in preps]
        grids = [_native.make_grid(cfg.k_rot, p.cos_tab, p.sin_tab, p.center_rot) for p in preps]
        for pl in plans:
            pl.reserve(cfg.rotation_count)
        flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
        stream = torch.cuda.current_stream().cuda_stream

        def timed(fn):
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                  for _ in range(steps)]
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            out = []
            for k in range(steps):
                flush.zero_()
                ev[k][0].record()
                out.append(fn(k))
                ev[k][1].record()
            torch.cuda.synchronize()
            t = torch.tensor([sum(a.elapsed_time(b) for a, b in ev)], dtype=torch.float64,
                             device="cuda")
            if world > 1:
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
            return float(t.item()), out

        def dev(k):
            p = preps[k]
            return plans[k].search(grids[k], cfg.q, p.code, p.param, p.skip_refine, stream=stream)

        for k in range(warmup):
            dev(k)
        ms, res = timed(lambda k: dev(warmup + k))
        host = pairs[warmup:]
        dses(host[0][0], host[0][1], cfg, device=local)
        ms_single, _ = timed(lambda k: dses(host[k][0], host[k][1], cfg, device=local))
        # a full untimed batch first (the stream-ordered memory pool grows to
        # the batch's working set once), then the median of three
        dses_batch([h[0] for h in host], [h[1] for h in host], cfg, device=local)
        if world > 1:
            dist.barrier()
        bt = []
        for _ in range(3):
            torch.cuda.synchronize()
            b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            flush.zero_()
            b0.record()
            dses_batch([h[0] for h in host], [h[1] for h in host], cfg, device=local)
            b1.record()
            torch.cuda.synchronize()
            bt.append(b0.elapsed_time(b1))
        tb = torch.tensor([sorted(bt)[1]], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(tb, op=dist.ReduceOp.MAX)
        ms_batch = float(tb.item())
        blk = plans[0].blocks()
        for pl in plans:
            pl.close()
        R = cfg.rotation_count
        tot = steps * R * world
        return {
            "name": name, "metric": METRIC, "unit": UNIT, "value": tot / (ms * 1e-3),
            "ms_per_step": ms / steps, "steps": steps, "warmup": warmup, "n_gpus": world,
            "scaling": "weak", "registrations_per_sec": steps * world / (ms * 1e-3),
            "config": {"workload": describe(name, c, cfg, preps[0].x.shape[0], preps[0].y.shape[0]),
                       "metric": cfg.metric.kind, "rotations": R},
            "vote_kernel_ms_per_step": sum(r["ms_vote_kernel"] for r in res) / steps,
            "vote_path": (f"vote_blocks_kernel: blocks of {blk[0]}x{blk[1]}x{blk[2]} neighbouring grid rotations "
                          "share one candidate-pair list (pairs_evaluated = list entries voted)") if blk[0] else
                         "vote_kernel (per rotation)",
            "pairs_evaluated_per_rotation": sum(r["pairs_evaluated"] for r in res) / (steps * R),
            "e2e": {"value": tot / (ms_batch * 1e-3), "unit": UNIT,
                    "path": "dses_batch over the timed pairs (host numpy in, results out)",
                    "single_call": {"value": tot / (ms_single * 1e-3), "unit": UNIT,
                                    "ms_per_step": ms_single / steps,
                                    "path": "one dses() call per step (plan construction exposed)"}},
        }
    except Exception as exc:  # reported, never fatal for the headline line
        return {"name": name, "error": f"{type(exc).__name__}: {exc}"}


def _free_port():
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def spawn_ranks(args):
    """`--gpus N` without a torchrun environment: re-launch this command under
    torch.distributed.run with N local ranks (one process per GPU)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    os.execvp(sys.executable, cmd)


def main():
    args = parse()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        spawn_ranks(args)  # does not return
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}")
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist

    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # BENCH_SHARE_DEVICE=1: code-path check of the N-rank protocol on a 1-GPU
    # box (every rank on cuda:0, gloo collectives; its numbers are not a
    # measurement -- the ranks time-share one GPU)
    share = os.environ.get("BENCH_SHARE_DEVICE") == "1"
    if share:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_2502_00115_b200 import _native, dses
    from paper_2502_00115_b200.engines import prepare

    c = workload(args.config, args.metric)
    cfg = search_config(c)
    nsteps = args.warmup + args.steps
    pairs, data_desc = bench_pairs(args.config, nsteps, rank * nsteps, args.inputs)
    stream = torch.cuda.current_stream().cuda_stream

    # ---- device-resident value: plans (clouds in HBM) built before timing
    preps = [prepare(x, y, cfg) for x, y, _ in pairs]
    plans = [_native.Plan(p.x, p.y, cfg.trans_bin, p.ilo, p.dims, local) for p in preps]
    for plan in plans:  # plan construction includes the search scratch (dses_plan_reserve)
        plan.reserve(cfg.rotation_count)
    grids = [_native.make_grid(cfg.k_rot, p.cos_tab, p.sin_tab, p.center_rot) for p in preps]
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    def one(s):
        p = preps[s]
        plans[s].traffic(reset=True)
        return plans[s].search(grids[s], cfg.q, p.code, p.param, p.skip_refine, stream=stream)

    for s in range(args.warmup):
        one(s)
    torch.cuda.synchronize()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    results = []
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        for k in range(args.steps):
            flush.zero_()  # evict L2 between timed steps (outside the events)
            starts[k].record()
            results.append(one(args.warmup + k))
            ends[k].record()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = sum(a.elapsed_time(b) for a, b in zip(starts, ends))
    vote_ms = sum(r["ms_vote_kernel"] for r in results)
    pairs_eval = sum(r["pairs_evaluated"] for r in results)
    launches = sum(r["launches"] for r in results)
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    R = cfg.rotation_count
    value = args.steps * R * world / (ms_max * 1e-3)

    # ---- end to end through the public API with host buffers
    # the same host pairs as the timed device-resident steps, so that e2e -
    # value is exactly the host-side cost (validation, plan build, copies)
    e2e_pairs = pairs[args.warmup:]
    dses(pairs[0][0], pairs[0][1], cfg, device=local)  # warm
    torch.cuda.synchronize()
    e_start = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    e_end = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    h2d = d2h = 0
    if world > 1:
        dist.barrier()
    for k in range(args.steps):
        flush.zero_()
        e_start[k].record()
        res = dses(e2e_pairs[k][0], e2e_pairs[k][1], cfg, device=local)
        e_end[k].record()
        st = res.elapsed["stats"]
        h2d += st["h2d_bytes"]
        d2h += st["d2h_bytes"]
    torch.cuda.synchronize()
    e_ms = sum(a.elapsed_time(b) for a, b in zip(e_start, e_end))
    te = torch.tensor([e_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e_value = args.steps * R * world / (float(te.item()) * 1e-3)

    # ---- end to end, batched: dses_batch over the same host pairs (plan
    #      construction of pair k+1 on a host thread overlaps the search of k)
    from paper_2502_00115_b200 import dses_batch
    dses_batch([p[0] for p in pairs[:2]], [p[1] for p in pairs[:2]], cfg, device=local)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    # three timed batches, the median reported (a single ~0.1 s batch is
    # exposed to one-off host hiccups on a freshly started box)
    b_times = []
    for _ in range(3):
        flush.zero_()
        b_start, b_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        b_start.record()
        bres = dses_batch([p[0] for p in e2e_pairs], [p[1] for p in e2e_pairs], cfg, device=local)
        b_end.record()
        torch.cuda.synchronize()
        b_times.append(b_start.elapsed_time(b_end))
    tb = torch.tensor([sorted(b_times)[1]], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(tb, op=dist.ReduceOp.MAX)
    b_value = args.steps * R * world / (float(tb.item()) * 1e-3)
    bh2d = sum(r.elapsed["stats"]["h2d_bytes"] for r in bres)
    bd2h = sum(r.elapsed["stats"]["d2h_bytes"] for r in bres)
    assert all(tuple(a.best.grid_coords) == tuple(b.best.grid_coords) for a, b in
               zip(bres, [dses(p[0], p[1], cfg, device=local) for p in e2e_pairs[:2]]))

    sharded = None if args.no_sharded else sharded_measurements(args, rank, world, local)
    extra = [] if args.no_sharded else [workload_line(w, args, rank, world, local)
                                        for w in EXTRA_WORKLOADS if w != args.config]

    if rank == 0:
        ffma_s, _ = _native.probe_fp32_peak(local)
        n_src = preps[0].x.shape[0]
        flops = 2.0 * (3.0 * pairs_eval + 9.0 * R * n_src * args.steps)
        achieved = flops / (vote_ms * 1e-3) / 1e12
        peak = 2.0 * ffma_s / 1e12
        traffic, ncu_info = None, None
        prof = os.path.join(ROOT, "profiles", f"ncu_vote_{args.config}.json")
        if os.path.exists(prof):
            try:
                ncu_info = json.load(open(prof))
                traffic = ncu_info.get("dram_bytes_per_launch")
            except (OSError, ValueError):
                traffic, ncu_info = None, None
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "i32 fixed-point vote / f32 screen / f64 exact",
            "data": data_desc,
            "config": {"workload": describe(args.config, c, cfg, n_src, preps[0].y.shape[0]),
                       "metric": cfg.metric.kind, "rotations": R},
            "metric_note": ("truncated-L1 at 5 bins: the reference's default and pinned kind; "
                            "BASELINE.json's 'truncated-L2' has no reference implementation "
                            "(gridreg/metrics.py:35), its trunc_l2 extension here is parity-"
                            "unpinned (oracle restatement only)"),
            "parallelism": f"replicas x{world} (registrations sharded over ranks, no collective)",
            "l2_flush": "512 MiB buffer zeroed between timed steps",
            "registrations_per_sec": args.steps * world / (ms_max * 1e-3),
            "e2e": {"value": b_value, "unit": UNIT,
                    "registrations_per_sec": args.steps * world / (float(tb.item()) * 1e-3),
                    "h2d_bytes_per_step": bh2d // args.steps, "d2h_bytes_per_step": bd2h // args.steps,
                    "path": "paper_2502_00115_b200.dses_batch(numpy sources, numpy references, "
                            "SearchConfig): K registrations (harness.run_batch's loop), plan "
                            "construction of k+1 on a worker thread overlapping the search of k, "
                            "search k+1 queued on the other of two streams before k is read; "
                            "median of 3 timed batches",
                    "batch_ms": b_times,
                    "single_call": {"value": e_value, "unit": UNIT,
                                    "registrations_per_sec": args.steps * world / (float(te.item()) * 1e-3),
                                    "h2d_bytes_per_step": h2d // args.steps,
                                    "d2h_bytes_per_step": d2h // args.steps,
                                    "path": "paper_2502_00115_b200.dses(numpy source, numpy "
                                            "reference, SearchConfig), one call per step"}},
            "gpu_launches": launches,
            "roofline": {"bound": "fp32", "kernel": "vote_kernel", "achieved": achieved,
                         "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                         "traffic": traffic,
                         "algorithmic": "2*(3 FFMA per evaluated (rotation,i,j) pair + 9 per "
                                        "(rotation,i)) / vote-kernel time (SURVEY.md 8(d))",
                         "peak_source": "live FFMA probe on this GPU (MEASURED_PEAKS.json has no FP32)",
                         "pairs_evaluated_per_step": pairs_eval / args.steps,
                         "nominal_pairs_per_step": R * n_src * preps[0].y.shape[0],
                         "vote_kernel_ms_per_step": vote_ms / args.steps,
                         "traffic_source": (f"profiles/ncu_vote_{args.config}.json: dram read+write "
                                            f"bytes of one ncu --set full capture ({ncu_info['launch']})"
                                            if ncu_info else None),
                         "ncu_issue_active_pct": ncu_info.get("issue_active_pct") if ncu_info else None,
                         "instructions_per_evaluated_pair": (
                             32.0 * ncu_info["warp_instructions_per_evaluated_pair"]
                             if ncu_info and "warp_instructions_per_evaluated_pair" in ncu_info else None),
                         "instructions_per_evaluated_pair_note": "thread-level issue slots (32 x warp "
                             "instructions) per evaluated pair, from the committed ncu capture",
                         "votes_per_rotation": sum(r["votes"] for r in results) / (args.steps * R),
                         "ncu_alu_pipe_pct": ncu_info.get("alu_pipe_pct") if ncu_info else None,
                         "note": "integer/ALU-issue bound (no tensor-core or HBM bound applies: "
                                 "inputs are shared-memory resident, contraction dim 3)"},
            "stages_ms_per_step": {
                "vote": sum(r["ms_vote"] for r in results) / args.steps,
                "select": sum(r["ms_select"] for r in results) / args.steps,
                "score": sum(r["ms_score"] for r in results) / args.steps,
                "total_device": sum(r["ms_total"] for r in results) / args.steps},
            "winner_example": {"row": results[0]["winner_row"], "count": results[0]["winner_count"],
                               "refined": results[0]["candidates_refined"],
                               "rescored": results[0]["rescored"]},
            "clocks": clocks.summary(),
        }
        if sharded is not None:
            line["rotation_sharded"] = sharded
        if extra:
            line["workloads"] = extra
        if world == 1 and not args.no_cpu_baseline:
            x0, y0, _ = pairs[0]

            def gpu_check(sample):
                return plans[0].mode_grid(grids[0], 0, sample)

            line["cpu_baseline"] = cpu_baseline(x0, y0, cfg, c, args.cpu_seconds, gpu_check)
        print(json.dumps(line), flush=True)
    for p in plans:
        p.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
