"""Command line: ``python -m paper_2502_00115_b200 register SRC REF [options]``.

The reference's ``gridreg register`` (cli.py:37-62, 111-166,
harness.register_files harness.py:285-322) on the B200: same flags
(--rot-range/--rot-step in degrees, k = max(1, ceil(range/step - 1e-9));
--trans-range/--trans-bin; --metric trunc-l1|l2|l1|inliers, --trunc, --q;
--center-pose JSON; --exhaustive; --out; --json), same report keys and exit
codes (0 ok, 1 engine error, 2 input / I/O error).  --device picks the GPU.

``benchmark --instances PREFIX... --search FILE`` is the reference's
``gridreg benchmark`` (cli.py:64-79, 176-197: harness.run_batch, CSV / JSON
reports, summary lines) over instance files (``<prefix>_source.xyz``,
``<prefix>_reference.xyz``, ``<prefix>_gt.json`` as written by the
reference's ``gridreg generate`` / ``benchgen.save_instance``) instead of
the in-process scenario generator (benchgen is out of scope): trial k is
the k-th prefix, its seed and shape come from the sidecar's config.

``oracle-check --trials N --seed S`` is ``gridreg oracle-check``
(cli.py:88-93, 212-226; harness.run_oracle_checks): same instances for the
same seed, same report lines, exit 1 when a suite finds a violation.
"""
from __future__ import annotations

import argparse
import json
import math
import sys

import numpy as np

from .errors import GridregError, InvalidInputError, PointCloudIOError

METRICS = ("trunc-l1", "l2", "l1", "inliers")


def _parser():
    ap = argparse.ArgumentParser(prog="paper_2502_00115_b200",
                                 description="B200 grid-search rigid registration (DSES).")
    ap.add_argument("--device", type=int, default=0, help="CUDA device (default 0)")
    sub = ap.add_subparsers(dest="command", required=True)
    p = sub.add_parser("register", help="align a source cloud onto a reference cloud")
    p.add_argument("source")
    p.add_argument("reference")
    p.add_argument("--rot-range", type=float, default=45.0, metavar="DEG")
    p.add_argument("--rot-step", type=float, default=3.0, metavar="DEG")
    p.add_argument("--trans-range", type=float, default=0.5, metavar="M")
    p.add_argument("--trans-bin", type=float, default=0.025, metavar="M")
    p.add_argument("--metric", choices=METRICS, default="trunc-l1")
    p.add_argument("--trunc", type=float, default=None, metavar="TAU")
    p.add_argument("--q", type=float, default=0.5)
    p.add_argument("--center-pose", metavar="FILE")
    p.add_argument("--exhaustive", action="store_true")
    p.add_argument("--out", metavar="FILE")
    p.add_argument("--json", action="store_true")
    p = sub.add_parser("benchmark", help="run a batch of registration trials on instance files")
    p.add_argument("--instances", required=True, nargs="+", metavar="PREFIX",
                   help="instance prefixes (PREFIX_source.xyz, PREFIX_reference.xyz, PREFIX_gt.json)")
    p.add_argument("--search", required=True, metavar="FILE", help="search config JSON")
    p.add_argument("--csv", metavar="FILE", help="write per-trial rows here")
    p.add_argument("--json", metavar="FILE", dest="json_out",
                   help="write full report (incl. timings) here")
    p.add_argument("--rot-tol-deg", type=float, default=1.0,
                   help="recall threshold on mean Euler error (default 1)")
    p.add_argument("--trans-tol", type=float, default=0.1,
                   help="recall threshold on mean translation error (default 0.1)")
    p = sub.add_parser("oracle-check",
                       help="verify mode optimality and engine equality on small instances")
    p.add_argument("--trials", type=int, default=20, metavar="N",
                   help="trials per suite (default 20)")
    p.add_argument("--seed", type=int, default=0, metavar="S")
    return ap


def grid_half_width(range_value: float, step: float) -> int:
    """cli.py:127-132: k = max(1, ceil(range / step - 1e-9)), 0 for no range."""
    if step <= 0:
        raise InvalidInputError("grid step must be positive")
    if range_value <= 0:
        return 0
    return max(1, int(math.ceil(range_value / step - 1e-9)))


def load_pose(path):
    from .geometry import RigidTransform, rotation_from_euler
    with open(path, "r", encoding="utf-8") as fh:
        raw = json.load(fh)
    t = np.asarray(raw.get("translation", (0.0, 0.0, 0.0)), dtype=np.float64)
    if "rotation" in raw:
        r = np.asarray(raw["rotation"], dtype=np.float64)
    elif "euler_deg" in raw:
        r = rotation_from_euler(np.radians(np.asarray(raw["euler_deg"], dtype=np.float64)))
    else:
        raise InvalidInputError(f"{path}: pose needs 'rotation' or 'euler_deg'")
    return RigidTransform(r, t)


def register_files(source_path, reference_path, cfg, exhaustive=False, out_path=None, device=0):
    """harness.register_files: read, register, chamfer before / after, report."""
    from .engines import dses, exhaustive_search
    from .metrics import chamfer_distance
    from .pcio import read_point_cloud, write_xyz

    x = read_point_cloud(source_path)
    y = read_point_cloud(reference_path)
    result = (exhaustive_search if exhaustive else dses)(x, y, cfg, device=device)
    moved = result.best.apply(x)
    before = chamfer_distance(x, y, device)
    after = chamfer_distance(moved, y, device)
    if out_path is not None:
        write_xyz(out_path, moved)
    e = result.best.euler()
    report = {
        "source": str(source_path), "reference": str(reference_path),
        "source_points": int(x.shape[0]), "reference_points": int(y.shape[0]),
        "engine": "exhaustive" if exhaustive else "dses",
        "euler_deg": [float(v) for v in np.degrees(e.as_array())],
        "translation_m": [float(v) for v in result.best.translation],
        "grid_coords": list(result.best.grid_coords) if result.best.grid_coords else None,
        "best_error": float(result.best_error), "best_inliers": int(result.best_inliers),
        "candidates_evaluated": int(result.candidates_evaluated),
        "candidates_refined": int(result.candidates_refined),
        "chamfer_before_m": before, "chamfer_after_m": after,
        "chamfer_improved": bool(after < before),
        "elapsed_s": {k: float(v) for k, v in result.elapsed.items()
                      if isinstance(v, (int, float))},
        "transformed_out": str(out_path) if out_path is not None else None,
    }
    return result, report


def _register(args) -> int:
    from .engines import SearchConfig
    from .metrics import ErrorMetric

    metric = ErrorMetric.from_name(args.metric, args.trans_bin, args.trunc)
    cfg = SearchConfig(
        k_rot=grid_half_width(math.radians(args.rot_range), math.radians(args.rot_step)),
        rot_step=math.radians(args.rot_step),
        k_trans=grid_half_width(args.trans_range, args.trans_bin), trans_bin=args.trans_bin,
        q=args.q, metric=metric,
        center=load_pose(args.center_pose) if args.center_pose else None)
    _, rep = register_files(args.source, args.reference, cfg, args.exhaustive, args.out,
                            args.device)
    if args.json:
        json.dump(rep, sys.stdout, indent=2, sort_keys=True)
        print()
        return 0
    e, t = rep["euler_deg"], rep["translation_m"]
    print(f"engine: {rep['engine']}")
    print(f"rotation (deg, xyz): {e[0]:+.4f} {e[1]:+.4f} {e[2]:+.4f}")
    print(f"translation (m):     {t[0]:+.6f} {t[1]:+.6f} {t[2]:+.6f}")
    print(f"inliers: {rep['best_inliers']} / {rep['source_points']}")
    print(f"alignment error: {rep['best_error']:.6g}")
    print(f"chamfer (m): {rep['chamfer_before_m']:.6g} -> {rep['chamfer_after_m']:.6g}")
    print(f"time (s): {rep['elapsed_s']['total']:.3f}")
    if rep["transformed_out"]:
        print(f"wrote {rep['transformed_out']}")
    return 0


def _benchmark(args) -> int:
    from .harness import register_batch, search_from_json, write_batch_csv, write_batch_json
    from .pcio import load_instance

    search = search_from_json(args.search)
    insts = [load_instance(p) for p in args.instances]
    summary, records = register_batch(
        [i.source for i in insts], [i.reference for i in insts], [i.gt_aligner for i in insts],
        search, rot_tol_deg=args.rot_tol_deg, trans_tol=args.trans_tol, device=args.device,
        seeds=[int(i.config.get("rng_seed", k)) for k, i in enumerate(insts)],
        shapes=[str(i.config.get("shape", "file")) for i in insts])
    if args.csv:
        write_batch_csv(args.csv, records)
    if args.json_out:
        write_batch_json(args.json_out, insts[0].config, search, summary, records)
    print(f"trials: {summary.n_trials}  failed: {summary.n_failed}")
    print(f"recall: {summary.recall:.3f}")
    if summary.mean_mie_r is not None:
        print(f"mean rotation error (deg): {summary.mean_mie_r:.4f}")
        print(f"mean translation error (m): {summary.mean_mie_t:.5f}")
        print(f"median time (ms): {summary.median_total_ms:.1f}")
    return 0


def _oracle_check(args) -> int:
    """cli.py:212-226: both suites, the reference's report lines, exit 1 on a
    violation."""
    from .harness import run_oracle_checks

    report = run_oracle_checks(n_lemma=args.trials, n_theorem=args.trials, seed=args.seed,
                               device=args.device)
    print(f"mode-optimality sweep: {report.lemma_trials - report.lemma_violations}"
          f"/{report.lemma_trials} ok")
    print(f"engine inlier equality: {report.theorem_trials - report.theorem_violations}"
          f"/{report.theorem_trials} ok")
    for line in report.details:
        print(f"  {line}")
    if not report.ok:
        raise GridregError("oracle checks found violations")
    return 0


_COMMANDS = {"register": "_register", "benchmark": "_benchmark", "oracle-check": "_oracle_check"}


def main(argv=None) -> int:
    args = _parser().parse_args(argv)
    try:
        return globals()[_COMMANDS[args.command]](args)
    except (FileNotFoundError, IsADirectoryError, PermissionError, PointCloudIOError,
            InvalidInputError, json.JSONDecodeError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2
    except GridregError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
