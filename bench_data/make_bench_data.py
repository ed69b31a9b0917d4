"""Bench inputs from the reference's own generator ("these use
the reference benchgen exactly, seeds as listed").

Run in the build container only (it imports the unmodified reference from
/root/reference read-only); the GPU box reads the committed .npz files.

    python bench_data/make_bench_data.py

benchgen_<cfg>.npz: x<k>, y<k> (source / reference, float64), gt_R<k>, gt_t<k>
(the aligning ground truth), seed<k>, for k < count:
  c1  ScenarioConfig(keep_fraction=0.5) seeds 0..15          (512 / 1024)
  c2  ScenarioConfig() defaults, seeds 0..15                  (717 / 1024)
  c3  ScenarioConfig(noise_sigma=0.02) seeds 0..1 + 20% outliers
      (SeedSequence([0x0071, seed]), tests/golden/make_golden.inject_outliers)
  c4  l-bracket 20000 / 7143 -> 5000, 5 deg / 16 mm / 2 mm noise, seeds 0..1
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(os.path.dirname(HERE), "tests", "golden"))
from make_golden import benchgen, inject_outliers  # noqa: E402  (imports the reference)

SPECS = {
    "c1": (dict(shape="blob", points_pool=2048, points_reference=1024, points_source=1024,
                keep_fraction=0.5), 16, 0.0),
    "c2": (dict(), 16, 0.0),
    "c3": (dict(noise_sigma=0.02), 2, 0.2),
    "c4": (dict(shape="l-bracket", points_pool=40000, points_reference=20000, points_source=7143,
                keep_fraction=0.7, rot_range_deg=5.0, trans_range=0.016, noise_sigma=0.002,
                noise_clip=0.01), 2, 0.0),
}


def main():
    for name, (kw, count, outliers) in SPECS.items():
        rec = {"count": np.int64(count)}
        for k in range(count):
            inst = benchgen.make_instance(benchgen.ScenarioConfig(rng_seed=k, **kw))
            x = inst.source if outliers == 0 else inject_outliers(inst.source, outliers, k)
            rec[f"x{k}"], rec[f"y{k}"] = x, inst.reference
            rec[f"gt_R{k}"] = np.asarray(inst.gt_aligner.rotation)
            rec[f"gt_t{k}"] = np.asarray(inst.gt_aligner.translation)
            rec[f"seed{k}"] = np.int64(k)
        path = os.path.join(HERE, f"benchgen_{name}.npz")
        np.savez_compressed(path, **rec)
        print(f"wrote {path} ({os.path.getsize(path) / 1024:.0f} KB): {count} pairs, "
              f"{rec['x0'].shape[0]} / {rec['y0'].shape[0]} points")


if __name__ == "__main__":
    main()
