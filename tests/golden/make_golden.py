"""Generate the golden fixtures that pin the CPU oracle (and, through it, the
B200 kernels) to the UNMODIFIED reference implementation.

Run in the build container only (it imports the reference read-only from
/root/reference/pkg/src; nothing under tests/ reads /root/reference at test
time):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

Every array written here comes from the reference's own code path
(`gridreg.benchgen.make_instance`, `gridreg.mode_search._mode_batch`,
`gridreg.engines._score_poses`, `gridreg.engines.dses`, ...).  The
outlier-injection step for config 3 follows SURVEY.md D4 / section 8(d)
(the reference benchgen has none).
"""
from __future__ import annotations

import math
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from gridreg import benchgen, engines, geometry, mode_search  # noqa: E402
from gridreg.engines import SearchConfig  # noqa: E402
from gridreg.metrics import ErrorMetric  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def inject_outliers(x, frac, seed):
    """replace round(frac*N) source rows, chosen by
    default_rng(SeedSequence([0x0071, seed])), with uniform samples in the
    source bounding box."""
    rng = np.random.default_rng(np.random.SeedSequence([0x0071, seed]))
    x = x.copy()
    n = x.shape[0]
    k = int(round(frac * n))
    rows = np.sort(rng.choice(n, size=k, replace=False))
    lo, hi = x.min(axis=0), x.max(axis=0)
    x[rows] = rng.uniform(lo, hi, (k, 3))
    return x


def votes(x, y, cfg):
    grid, rots, t_center = engines._prepare(x, y, cfg)
    cbin = mode_search.bin_index(t_center, cfg.trans_bin)
    ilo = cbin - cfg.k_trans
    dims = np.full(3, 2 * cfg.k_trans + 1, dtype=np.int64)
    return mode_search._mode_batch(rots, x, y, cfg.trans_bin, ilo, dims)


def dses_record(x, y, cfg, prefix, rec, with_votes=True):
    res = engines.dses(x, y, cfg)
    rec[f"{prefix}_R"] = np.asarray(res.best.rotation)
    rec[f"{prefix}_t"] = np.asarray(res.best.translation)
    rec[f"{prefix}_grid"] = np.asarray(res.best.grid_coords, dtype=np.int64)
    rec[f"{prefix}_best_error"] = np.float64(res.best_error)
    rec[f"{prefix}_best_inliers"] = np.int64(res.best_inliers)
    rec[f"{prefix}_evaluated"] = np.int64(res.candidates_evaluated)
    rec[f"{prefix}_refined"] = np.int64(res.candidates_refined)
    if with_votes:
        c, l, t = votes(x, y, cfg)
        rec[f"{prefix}_counts"] = c.astype(np.int32)
        rec[f"{prefix}_lins"] = l.astype(np.int32)
        rec[f"{prefix}_ties"] = t.astype(np.int32)
    print(f"  {prefix}: grid {res.best.grid_coords} err {res.best_error:.6g} "
          f"inl {res.best_inliers} eval {res.candidates_evaluated} ref {res.candidates_refined}")


def metric_fields(m: ErrorMetric):
    return np.array(m.kind), np.float64(np.nan if m.param is None else m.param)


def save(name, rec):
    path = os.path.join(OUT, f"{name}.npz")
    np.savez_compressed(path, **rec)
    print(f"wrote {path} ({os.path.getsize(path) / 1024:.0f} KB)")


def cfg_fields(rec, prefix, cfg: SearchConfig):
    rec[f"{prefix}_k_rot"] = np.int64(cfg.k_rot)
    rec[f"{prefix}_rot_step"] = np.float64(cfg.rot_step)
    rec[f"{prefix}_k_trans"] = np.int64(cfg.k_trans)
    rec[f"{prefix}_trans_bin"] = np.float64(cfg.trans_bin)
    rec[f"{prefix}_q"] = np.float64(cfg.q)
    k, p = metric_fields(cfg.metric)
    rec[f"{prefix}_metric_kind"] = k
    rec[f"{prefix}_metric_param"] = p
    if cfg.center is not None:
        rec[f"{prefix}_center_R"] = np.asarray(cfg.center.rotation)
        rec[f"{prefix}_center_t"] = np.asarray(cfg.center.translation)


def make_c1():
    """config 1: 1024-pt full / 512-pt partial, coarse grid, inliers metric."""
    scn = benchgen.ScenarioConfig(shape="blob", points_pool=2048, points_reference=1024,
                                  points_source=1024, keep_fraction=0.5, rng_seed=0)
    inst = benchgen.make_instance(scn)
    rec = {"x": inst.source, "y": inst.reference}
    cfg = SearchConfig(k_rot=5, rot_step=math.radians(9.0), k_trans=20, trans_bin=0.025,
                       metric=ErrorMetric.from_name("inliers", 0.025))
    cfg_fields(rec, "a", cfg)
    dses_record(inst.source, inst.reference, cfg, "a", rec)
    save("c1", rec)


def make_c2():
    """config 2: ModelNet40-shaped 1024 / 717, medium grid (29,791 rotations),
    truncated-L1 (reference default); plus the other metrics on a smaller grid."""
    inst = benchgen.make_instance(benchgen.ScenarioConfig(rng_seed=0))
    x, y = inst.source, inst.reference
    rec = {"x": x, "y": y}
    cfg = SearchConfig(k_rot=15, rot_step=math.radians(3.0), k_trans=20, trans_bin=0.025, q=0.5)
    cfg_fields(rec, "a", cfg)
    dses_record(x, y, cfg, "a", rec)
    for tag, metric in (("l1", ErrorMetric.l1()), ("l2", ErrorMetric.l2()),
                        ("sat2", ErrorMetric.saturated_l0(0.05)),
                        ("inl", ErrorMetric.saturated_l0(0.025))):
        cfg = SearchConfig(k_rot=4, rot_step=math.radians(5.0), k_trans=20, trans_bin=0.025,
                           q=0.5, metric=metric)
        cfg_fields(rec, tag, cfg)
        dses_record(x, y, cfg, tag, rec, with_votes=(tag == "l1"))
    # centre path (engines.py:120-130): rotations C @ G, window around C.t's bin
    gt = inst.gt_aligner
    cen = geometry.RigidTransform(
        geometry.rotation_from_euler(np.array(gt.euler().as_array()) + np.radians([2.0, -1.0, 1.5])),
        gt.translation + np.array([0.013, -0.021, 0.008]))
    cfg = SearchConfig(k_rot=3, rot_step=math.radians(1.0), k_trans=6, trans_bin=0.025,
                       center=cen)
    cfg_fields(rec, "cen", cfg)
    dses_record(x, y, cfg, "cen", rec)
    save("c2", rec)


def make_c3():
    """config 3 (reduced grid): sigma 0.02, 20% outliers, L1."""
    inst = benchgen.make_instance(benchgen.ScenarioConfig(noise_sigma=0.02, rng_seed=1))
    x = inject_outliers(inst.source, 0.2, 1)
    y = inst.reference
    rec = {"x": x, "y": y}
    cfg = SearchConfig(k_rot=6, rot_step=math.radians(1.0), k_trans=20, trans_bin=0.025,
                       metric=ErrorMetric.l1())
    cfg_fields(rec, "a", cfg)
    dses_record(x, y, cfg, "a", rec)
    save("c3", rec)


def make_c4():
    """config 4 (reduced grid): l-bracket 20k reference / 5k partial, 4 mm bins."""
    scn = benchgen.ScenarioConfig(shape="l-bracket", points_pool=40000, points_reference=20000,
                                  points_source=7143, keep_fraction=0.7, rot_range_deg=5.0,
                                  trans_range=0.016, noise_sigma=0.002, noise_clip=0.01,
                                  rng_seed=0)
    inst = benchgen.make_instance(scn)
    x, y = inst.source, inst.reference
    rec = {"x": x, "y": y}
    cfg = SearchConfig(k_rot=1, rot_step=math.radians(0.5), k_trans=4, trans_bin=0.004)
    cfg_fields(rec, "a", cfg)
    dses_record(x, y, cfg, "a", rec)
    save("c4", rec)


def make_small():
    """Many small random cases for the vote kernel (dense and sparse lattice
    paths, arbitrary rotations, bounds) and the refine kernel (all metrics)."""
    rng = np.random.default_rng(20250200)
    rec = {}
    ncase = 0
    for case in range(60):
        n = int(rng.integers(1, 40))
        m = int(rng.integers(1, 50))
        x = rng.uniform(-1, 1, (n, 3))
        y = rng.uniform(-1, 1, (m, 3))
        if case % 3 == 0:   # shared structure so modes are non-trivial
            rot = geometry.random_rotation(rng)
            k = min(n, m)
            y[:k] = x[:k] @ rot.T + rng.uniform(-0.3, 0.3, 3)
        b = float(rng.uniform(0.03, 0.4))
        rots = np.stack([geometry.random_rotation(rng) for _ in range(int(rng.integers(1, 6)))])
        if case % 5 == 0:
            rots[0] = np.eye(3)
        kt = int(rng.integers(0, 30))
        ilo = rng.integers(-5, 5, 3) - kt
        dims = np.array([2 * kt + 1 + int(rng.integers(0, 3)) for _ in range(3)], dtype=np.int64)
        counts, lins, ties = mode_search._mode_batch(rots, x, y, b, ilo, dims)
        key = f"m{ncase}"
        rec.update({f"{key}_x": x, f"{key}_y": y, f"{key}_rots": rots, f"{key}_b": np.float64(b),
                    f"{key}_ilo": ilo.astype(np.int64), f"{key}_dims": dims,
                    f"{key}_counts": counts, f"{key}_lins": lins, f"{key}_ties": ties})
        ncase += 1
    rec["n_mode_cases"] = np.int64(ncase)
    # refine / alignment error cases (engines._score_poses -> refine_batch)
    nref = 0
    for case in range(24):
        n = int(rng.integers(1, 30))
        m = int(rng.integers(1, 40))
        x = rng.uniform(-1, 1, (n, 3))
        y = rng.uniform(-1, 1, (m, 3))
        c = int(rng.integers(1, 8))
        rots = np.stack([geometry.random_rotation(rng) for _ in range(c)])
        ts = rng.uniform(-0.3, 0.3, (c, 3))
        kind = ["l2", "l1", "trunc_l1", "sat_l0"][case % 4]
        metric = ErrorMetric(kind, None if kind in ("l2", "l1") else float(rng.uniform(0.1, 0.6)))
        errs = engines._score_poses(rots, ts, x, y, metric)
        key = f"r{nref}"
        code, param = metric._code_param()
        rec.update({f"{key}_x": x, f"{key}_y": y, f"{key}_rots": rots, f"{key}_ts": ts,
                    f"{key}_code": np.int64(code), f"{key}_param": np.float64(param),
                    f"{key}_errs": errs})
        nref += 1
    rec["n_refine_cases"] = np.int64(nref)
    # end-to-end small dses cases (tests/test_engines.py-style shapes)
    nd = 0
    for case in range(16):
        n = int(rng.integers(3, 25))
        x = rng.uniform(-1, 1, (n, 3))
        if case % 2 == 0:
            ridx = rng.integers(-1, 2, 3)
            tidx = rng.integers(-2, 3, 3)
            tf = geometry.RigidTransform(geometry.rotation_from_euler(ridx.astype(float) * 0.3),
                                         tidx.astype(float) * 0.25)
            y = tf.apply(x) + rng.normal(0.0, 0.01, (n, 3))
        else:
            y = rng.uniform(-1, 1, (int(rng.integers(3, 25)), 3))
        kind = ["trunc_l1", "l1", "l2", "sat_l0"][case % 4]
        metric = None if kind == "trunc_l1" else ErrorMetric(kind, 0.25 if kind == "sat_l0" else None)
        cfg = SearchConfig(k_rot=1, rot_step=0.3, k_trans=3, trans_bin=0.25,
                           q=[0.5, 1.0, 1e-9, 0.3][case % 4], metric=metric)
        key = f"d{nd}"
        rec.update({f"{key}_x": x, f"{key}_y": y})
        cfg_fields(rec, key, cfg)
        dses_record(x, y, cfg, key, rec, with_votes=True)
        nd += 1
    rec["n_dses_cases"] = np.int64(nd)
    save("small", rec)


def make_exh():
    """engines.exhaustive_search (Algorithm 1, the optimality oracle) on small
    instances: every metric, with and without a centre pose, plus the
    DSES-vs-exhaustive inlier equality of the acceptance suite (C2)."""
    rec = {}
    cases = [
        ("inliers", None, None, 2, 4),
        ("trunc-l1", None, None, 1, 4),
        ("l1", None, None, 1, 3),
        ("l2", None, None, 1, 3),
        ("trunc-l1", 0.3, (np.radians([2.0, -3.0, 4.0]), [0.03, -0.02, 0.05]), 1, 3),
    ]
    for c, (name, thr, centre, k_rot, k_trans) in enumerate(cases):
        rng = np.random.default_rng(np.random.SeedSequence([0xE7, c]))
        y = rng.uniform(-1.0, 1.0, (70, 3))
        rot = geometry.rotation_from_euler(rng.uniform(-0.1, 0.1, 3))
        x = (y[:45] - rng.uniform(-0.1, 0.1, 3)) @ rot + rng.normal(0, 0.01, (45, 3))
        metric = ErrorMetric.from_name(name, 0.05, thr)
        kw = dict(k_rot=k_rot, rot_step=math.radians(4.0), k_trans=k_trans, trans_bin=0.05,
                  metric=metric)
        if centre is not None:
            kw["center"] = geometry.RigidTransform(geometry.rotation_from_euler(centre[0]),
                                                   np.asarray(centre[1]))
        cfg = SearchConfig(**kw)
        p = f"e{c}"
        res = engines.exhaustive_search(x, y, cfg)
        rec[f"{p}_x"], rec[f"{p}_y"] = x, y
        cfg_fields(rec, p, cfg)
        rec[f"{p}_R"] = np.asarray(res.best.rotation)
        rec[f"{p}_t"] = np.asarray(res.best.translation)
        rec[f"{p}_grid"] = np.asarray(res.best.grid_coords, dtype=np.int64)
        rec[f"{p}_best_error"] = np.float64(res.best_error)
        rec[f"{p}_best_inliers"] = np.int64(res.best_inliers)
        rec[f"{p}_evaluated"] = np.int64(res.candidates_evaluated)
        if name == "inliers":
            rec[f"{p}_dses_inliers"] = np.int64(engines.dses(x, y, cfg).best_inliers)
        print(f"  {p}: {name} grid {res.best.grid_coords} err {res.best_error:.6g} "
              f"inl {res.best_inliers}")
    rec["n_exh_cases"] = np.int64(len(cases))
    save("exh", rec)


def make_harness():
    """harness._run_one (dses + apply_transform + chamfer + evaluate_pose) on
    four benchgen instances with a small grid; ground truth from benchgen."""
    from gridreg import harness, metrics
    rec = {}
    search = SearchConfig(k_rot=4, rot_step=math.radians(6.0), k_trans=20, trans_bin=0.025)
    n = 4
    for k in range(n):
        inst = benchgen.make_instance(benchgen.ScenarioConfig(rng_seed=100 + k, rot_range_deg=15.0))
        r = harness._run_one(inst, search, k, 100 + k, 1.0, 0.1)
        p = f"h{k}"
        rec[f"{p}_x"], rec[f"{p}_y"] = inst.source, inst.reference
        rec[f"{p}_gt_R"] = np.asarray(inst.gt_aligner.rotation)
        rec[f"{p}_gt_t"] = np.asarray(inst.gt_aligner.translation)
        rec[f"{p}_status"] = np.array(r.status)
        if r.status == "ok":
            e = r.eval
            rec[f"{p}_eval"] = np.array([e.mie_r, e.mie_t, e.mae_r, e.mae_t, e.chamfer])
            rec[f"{p}_hit"] = np.int64(e.is_recall_hit)
            rec[f"{p}_inliers"] = np.int64(r.inliers)
            rec[f"{p}_refined"] = np.int64(r.candidates_refined)
            res = engines.dses(inst.source, inst.reference, search)
            rec[f"{p}_grid"] = np.asarray(res.best.grid_coords, dtype=np.int64)
            moved = res.best.apply(inst.source)
            rec[f"{p}_chamfer_one_way"] = np.float64(metrics._kernels.chamfer_one_way(moved, inst.reference))
        print(f"  {p}: {r.status} {r.eval}")
    cfg_fields(rec, "h", search)
    rec["n_harness_cases"] = np.int64(n)
    save("harness", rec)


from make_golden_records import BATCHIO_RECORDS, SEARCH_JSON_CASES  # noqa: E402


def make_batchio():
    """harness.write_batch_csv / write_batch_json / search_to_dict /
    search_from_json outputs for fixed records and config files."""
    import json
    import tempfile
    from gridreg import harness
    from gridreg.metrics import EvalReport

    recs = []
    for d in BATCHIO_RECORDS:
        e = d["eval"]
        ev = None if e is None else EvalReport(mie_r=e[0], mie_t=e[1], mae_r=e[2], mae_t=e[3],
                                                is_recall_hit=e[4], chamfer=e[5])
        recs.append(harness.TrialRecord(**dict(d, eval=ev)))
    summary = harness._summarize(recs)
    search = SearchConfig(k_rot=3, rot_step=math.radians(2.0), k_trans=8, trans_bin=0.02,
                          metric=ErrorMetric.from_name("trunc-l1", 0.02, 0.05),
                          center=geometry.RigidTransform(np.eye(3), np.array([0.5, 0.0, -0.25])))
    scenario = benchgen.ScenarioConfig(shape="blob", rng_seed=100)
    out = {}
    with tempfile.TemporaryDirectory() as tmp:
        harness.write_batch_csv(os.path.join(tmp, "b.csv"), recs)
        harness.write_batch_json(os.path.join(tmp, "b.json"), scenario, search, summary, recs,
                                 extra={"note": "golden"})
        out["csv"] = open(os.path.join(tmp, "b.csv"), encoding="utf-8").read()
        out["json"] = open(os.path.join(tmp, "b.json"), encoding="utf-8").read()
        parsed = []
        for k, case in enumerate(SEARCH_JSON_CASES):
            path = os.path.join(tmp, f"s{k}.json")
            with open(path, "w", encoding="utf-8") as fh:
                json.dump(case, fh)
            try:
                cfg = harness.search_from_json(path)
                parsed.append({"ok": harness.search_to_dict(cfg)})
            except Exception as exc:  # noqa: BLE001
                parsed.append({"error": type(exc).__name__, "message": str(exc)})
    out["scenario"] = json.loads(json.dumps(harness.asdict(scenario)))
    out["search_to_dict"] = harness.search_to_dict(search)
    out["search_cases"] = parsed
    rec = {"batchio": np.array(json.dumps(out, sort_keys=True))}
    save("batchio", rec)


def _seq_bins_agree(x, y, rot, b):
    """True when numpy's BLAS product gives the same pair bins as the vote
    kernels' sequential binary64 order (then both define the same map)."""
    p_blas = x @ rot.T
    p_seq = np.empty_like(p_blas)
    for k in range(3):
        p_seq[:, k] = (rot[k, 0] * x[:, 0] + rot[k, 1] * x[:, 1]) + rot[k, 2] * x[:, 2]
    c1 = (y[None] - p_blas[:, None]).reshape(-1, 3)
    c2 = (y[None] - p_seq[:, None]).reshape(-1, 3)
    return np.array_equal(mode_search.bin_index(c1, b), mode_search.bin_index(c2, b))


def make_histo():
    """mode_search.translation_histogram (+ .mode()) and
    engines.refine_candidates on small clouds."""
    rec = {}
    cases = []
    rng = np.random.default_rng(77)
    for k in range(6):
        n, m = [(40, 60), (64, 64), (30, 90), (50, 50), (20, 40), (45, 70)][k]
        while True:
            x = rng.normal(scale=0.2, size=(n, 3))
            h = min(n, m // 2)
            y = np.concatenate([x[:h] + rng.normal(scale=0.01, size=(h, 3)),
                                rng.normal(scale=0.2, size=(m - h, 3))])
            if k == 3:  # duplicated reference points: dedup matters
                y[h:] = y[: m - h]
            if k == 4:  # permutation rotation (exact products)
                rot = np.array([[0.0, 1.0, 0.0], [0.0, 0.0, -1.0], [-1.0, 0.0, 0.0]])
            else:
                rot = geometry.rotation_from_euler(rng.uniform(-0.5, 0.5, 3))
            b = [0.05, 0.03, 0.1, 0.05, 0.04, 0.02][k]
            if _seq_bins_agree(x, y, rot, b):
                break
        bounds = None
        if k in (1, 5):
            bounds = np.array([[-0.2, -0.15, -0.3], [0.25, 0.2, 0.1]])
        cases.append((x, y, rot, b, bounds))
    # bounds with no pair inside: empty histogram, mode() raises
    x, y, rot, b, _ = cases[0]
    cases.append((x, y, rot, b, np.array([[50.0, 50.0, 50.0], [50.2, 50.2, 50.2]])))
    for k, (x, y, rot, b, bounds) in enumerate(cases):
        p = f"t{k}"
        rec[f"{p}_x"], rec[f"{p}_y"], rec[f"{p}_rot"], rec[f"{p}_bin"] = x, y, rot, np.float64(b)
        if bounds is not None:
            rec[f"{p}_bounds"] = bounds
        for dedup in (True, False):
            h = mode_search.translation_histogram(x, y, rot, b, t_bounds=bounds, dedup=dedup)
            q = f"{p}_{'d' if dedup else 'r'}"
            keys = sorted(h.counts)
            rec[f"{q}_keys"] = np.array(keys, dtype=np.int64).reshape(-1, 3)
            rec[f"{q}_vals"] = np.array([h.counts[kk] for kk in keys], dtype=np.int64)
            rec[f"{q}_total"] = np.int64(h.total)
            if h.counts:
                md = h.mode()
                rec[f"{q}_mode"] = np.array([*md.index, md.count, md.num_tied_bins], dtype=np.int64)
        print(f"  {p}: {len(h.counts)} raw bins, total {h.total}")
    rec["n_histo_cases"] = np.int64(len(cases))
    # refine_candidates: a count-sorted list of poses on the c1 pair
    x, y = cases[1][0], cases[1][1]
    cands = []
    for j, cnt in enumerate([30, 30, 22, 16, 15, 9, 3]):
        r = geometry.rotation_from_euler(rng.uniform(-0.3, 0.3, 3))
        t = rng.normal(scale=0.05, size=3)
        cands.append(engines.PoseCandidate(transform=geometry.RigidTransform(r, t), inlier_count=cnt))
        rec[f"rc_R{j}"], rec[f"rc_t{j}"] = r, t
    rec["rc_counts"] = np.array([c.inlier_count for c in cands], dtype=np.int64)
    rec["rc_x"], rec["rc_y"] = x, y
    for mname, metric in (("l1", ErrorMetric.l1()), ("tl1", ErrorMetric.truncated_l1(0.05)),
                          ("l2", ErrorMetric.l2()), ("sat", ErrorMetric.saturated_l0(0.03))):
        for q in (0.5, 0.75, 1.0):
            out = engines.refine_candidates(cands, x, y, metric, q)
            rec[f"rc_{mname}_{int(q * 100)}"] = np.array(
                [np.nan if c.refined_error is None else c.refined_error for c in out])
    save("histo", rec)

def make_instances():
    """benchgen.save_instance files of three small instances (byte-exact
    sidecar / XYZ fixtures) and the reference's batch CSV for them:
    harness._run_one on benchgen.load_instance of the written files, then
    harness.write_batch_csv (what `gridreg benchmark` writes)."""
    import json
    import tempfile
    from dataclasses import replace
    from gridreg import harness
    search = SearchConfig(k_rot=3, rot_step=math.radians(5.0), k_trans=16, trans_bin=0.03)
    base = benchgen.ScenarioConfig(shape="blob", points_pool=600, points_reference=300,
                                   points_source=260, rot_range_deg=12.0, trans_range=0.3,
                                   rng_seed=40)
    files, recs = [], []
    with tempfile.TemporaryDirectory() as tmp:
        for k in range(3):
            inst = benchgen.make_instance(replace(base, rng_seed=40 + k,
                                                  shape=("blob", "box", "torus")[k]))
            prefix = os.path.join(tmp, f"i{k}")
            benchgen.save_instance(inst, prefix)
            files.append({suffix: open(f"{prefix}_{suffix}", encoding="utf-8").read()
                          for suffix in ("source.xyz", "reference.xyz", "gt.json")})
            loaded = benchgen.load_instance(prefix)
            recs.append(harness._run_one(loaded, search, k, loaded.config.rng_seed, 1.0, 0.1))
            print(f"  i{k}: {recs[-1].status} {recs[-1].eval}")
        harness.write_batch_csv(os.path.join(tmp, "b.csv"), recs)
        csv_text = open(os.path.join(tmp, "b.csv"), encoding="utf-8").read()
        with open(os.path.join(tmp, "s.json"), "w", encoding="utf-8") as fh:
            json.dump(harness.search_to_dict(search), fh)
        search_text = open(os.path.join(tmp, "s.json"), encoding="utf-8").read()
    out = {"files": files, "csv": csv_text, "search": search_text,
           "summary": harness.asdict(harness._summarize(recs))}
    save("instances", {"instances": np.array(json.dumps(out, sort_keys=True))})


def make_oracle():
    """harness.run_oracle_checks pieces: the lemma / theorem instances the
    reference draws for seed 0 (make_lemma_instance / make_theorem_instance
    with the run's RNG), the mode inlier count, the dense-sweep maximum
    (_kernels.sweep_inlier_best) and the two engines' inlier counts; the
    report of run_oracle_checks(4, 4, 0); plus two standalone sweep cases
    (random, and differences exactly on the ball boundary: strict <)."""
    from gridreg import _kernels, harness, metrics
    from gridreg.mode_search import mode_translation
    rec = {}
    rng = np.random.default_rng(np.random.SeedSequence([0x0AC1E, 0]))
    b = 0.05
    nl = nt = 4
    for k in range(nl):
        x, y, rot, m = harness.make_lemma_instance(rng, b)
        mode = mode_translation(x, y, rot, b)
        c_star = metrics.count_inliers(x, y, geometry.RigidTransform(rot, mode.t_star), b)
        cand = np.ascontiguousarray((y[None, :, :] - (x @ rot.T)[:, None, :]).reshape(-1, 3))
        step = b / 4.0
        axes = [np.arange(cand[:, a].min(), cand[:, a].max() + step, step) for a in range(3)]
        best = int(_kernels.sweep_inlier_best(cand, x.shape[0], y.shape[0], b / 2.0, *axes))
        p = f"l{k}"
        rec[f"{p}_x"], rec[f"{p}_y"], rec[f"{p}_rot"] = x, y, rot
        rec[f"{p}_m"], rec[f"{p}_cstar"], rec[f"{p}_best"] = np.int64(m), np.int64(c_star), np.int64(best)
        rec[f"{p}_tstar"] = np.asarray(mode.t_star)
        print(f"  lemma {k}: n={x.shape[0]} m={y.shape[0]} planted {m} mode {c_star} sweep {best}")
    for k in range(nt):
        x, y, cfg = harness.make_theorem_instance(rng)
        semi, full = engines.dses(x, y, cfg), engines.exhaustive_search(x, y, cfg)
        p = f"t{k}"
        rec[f"{p}_x"], rec[f"{p}_y"] = x, y
        rec[f"{p}_krot"] = np.int64(cfg.k_rot)
        rec[f"{p}_semi"], rec[f"{p}_full"] = np.int64(semi.best_inliers), np.int64(full.best_inliers)
        print(f"  theorem {k}: k_rot={cfg.k_rot} semi {semi.best_inliers} full {full.best_inliers}")
    rep = harness.run_oracle_checks(n_lemma=nl, n_theorem=nt, seed=0)
    rec["report"] = np.array([rep.lemma_trials, rep.lemma_violations, rep.theorem_trials,
                              rep.theorem_violations], dtype=np.int64)
    rec["report_details"] = np.array("\n".join(rep.details))
    r2 = np.random.default_rng(7)
    cand = r2.uniform(-0.3, 0.3, (7 * 5, 3))
    axes = [np.linspace(-0.35, 0.35, 29) for _ in range(3)]
    rec["s0_cands"], rec["s0_axes"] = cand, np.stack(axes)
    rec["s0_best"] = np.int64(_kernels.sweep_inlier_best(cand, 7, 5, 0.04, *axes))
    cand = r2.integers(-2, 3, (6 * 6, 3)).astype(np.float64) * 0.25
    axes = [np.arange(-1.0, 1.0 + 0.125, 0.125) for _ in range(3)]
    rec["s1_cands"], rec["s1_axes"] = cand, np.stack(axes)
    rec["s1_best"] = np.int64(_kernels.sweep_inlier_best(cand, 6, 6, 0.25, *axes))
    print(f"  sweeps: {int(rec['s0_best'])} {int(rec['s1_best'])}")
    save("oracle", rec)


if __name__ == "__main__":
    which = sys.argv[1:] or ["small", "c1", "c2", "c3", "c4", "exh", "harness", "batchio",
                             "histo", "instances", "oracle"]
    for w in which:
        print(w)
        globals()[f"make_{w}"]()
