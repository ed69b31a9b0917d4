"""Point-cloud files and the register CLI (reference
pcio.py:1-216, cli.py:28-274).  File formats are host-side: CPU tests; the
CLI's registration itself runs on the GPU (-m gpu)."""
import json
import os
import struct
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT


def test_xyz_round_trip(tmp_path):
    from paper_2502_00115_b200.pcio import read_xyz, write_xyz
    pts = np.random.default_rng(0).normal(size=(50, 3))
    p = tmp_path / "a.xyz"
    write_xyz(p, pts)
    back = read_xyz(p)
    assert back.shape == (50, 3)
    assert np.allclose(back, pts, rtol=1e-8, atol=1e-12)  # 9 significant digits
    p2 = tmp_path / "b.xyz"
    p2.write_text("# comment\n\n1 2 3\n 4.5 -6 7e-1 \n")
    assert np.array_equal(read_xyz(p2), [[1, 2, 3], [4.5, -6, 0.7]])


@pytest.mark.parametrize("text", ["1 2\n", "1 2 x\n", "# only comments\n", "1 2 nan\n"])
def test_xyz_errors(tmp_path, text):
    from paper_2502_00115_b200 import PointCloudIOError
    from paper_2502_00115_b200.pcio import read_xyz
    p = tmp_path / "bad.xyz"
    p.write_text(text)
    with pytest.raises(PointCloudIOError):
        read_xyz(p)


def _ply_header(fmt, nv, extra_before="", props=("float x", "float y", "float z")):
    lines = ["ply", f"format {fmt} 1.0", "comment test"]
    if extra_before:
        lines += extra_before.splitlines()
    lines += [f"element vertex {nv}"] + [f"property {p}" for p in props]
    lines += ["element face 0", "property list uchar int vertex_indices", "end_header"]
    return ("\n".join(lines) + "\n").encode()


def test_ply_ascii_and_binary(tmp_path):
    from paper_2502_00115_b200.pcio import read_ply, read_point_cloud
    pts = np.random.default_rng(1).normal(size=(7, 3)).astype(np.float32)
    # ascii, with an extra property before x and a preceding element
    a = tmp_path / "a.ply"
    body = "".join(f"9 {x} {y} {z}\n" for x, y, z in pts)
    a.write_bytes(_ply_header("ascii", 7, "element cam 1\nproperty int id",
                              ("uchar id", "float x", "float y", "float z")) + b"42\n" + body.encode())
    assert np.allclose(read_ply(a), pts.astype(np.float64), atol=1e-6)
    # binary little endian, double coordinates + an int property, preceding element
    b = tmp_path / "b.ply"
    rec = b"".join(struct.pack("<dIdd", float(x), 7, float(y), float(z)) for x, y, z in pts)
    b.write_bytes(_ply_header("binary_little_endian", 7, "element cam 2\nproperty short id",
                              ("double x", "uint k", "double y", "double z"))
                  + struct.pack("<hh", 1, 2) + rec)
    assert np.array_equal(read_point_cloud(b), pts.astype(np.float64))


@pytest.mark.parametrize("case", ["magic", "format", "list", "type", "novertex", "noz", "trunc"])
def test_ply_errors(tmp_path, case):
    from paper_2502_00115_b200 import PointCloudIOError
    from paper_2502_00115_b200.pcio import read_ply
    p = tmp_path / "bad.ply"
    good = _ply_header("binary_little_endian", 2) + struct.pack("<6f", *range(6))
    data = {
        "magic": b"plx\n" + good[4:],
        "format": good.replace(b"binary_little_endian", b"binary_big_endian"),
        "list": _ply_header("ascii", 1, props=("list uchar int idx", "float x", "float y", "float z")) + b"0 1 2 3\n",
        "type": _ply_header("ascii", 1, props=("quad x", "float y", "float z")) + b"1 2 3\n",
        "novertex": b"ply\nformat ascii 1.0\nelement face 0\nend_header\n",
        "noz": _ply_header("ascii", 1, props=("float x", "float y")) + b"1 2\n",
        "trunc": good[:-4],
    }[case]
    p.write_bytes(data)
    with pytest.raises(PointCloudIOError):
        read_ply(p)


def _cli(*args):
    return subprocess.run([sys.executable, "-m", "paper_2502_00115_b200", *args], cwd=ROOT,
                          capture_output=True, text=True, timeout=600)


def test_cli_input_errors_exit_2(tmp_path):
    r = _cli("register", str(tmp_path / "missing.xyz"), str(tmp_path / "missing2.xyz"))
    assert r.returncode == 2 and "error" in r.stderr
    bad = tmp_path / "bad.xyz"
    bad.write_text("1 2\n")
    r = _cli("register", str(bad), str(bad))
    assert r.returncode == 2


def test_grid_half_width():
    from paper_2502_00115_b200.cli import grid_half_width
    assert grid_half_width(45.0, 3.0) == 15
    assert grid_half_width(10.0, 3.0) == 4
    assert grid_half_width(0.0, 3.0) == 0
    assert grid_half_width(1.0, 3.0) == 1


@pytest.mark.gpu
def test_cli_register_json(tmp_path):
    from paper_2502_00115_b200 import ErrorMetric, SearchConfig, dses
    from paper_2502_00115_b200.pcio import read_xyz, write_xyz
    from paper_2502_00115_b200.synth import CONFIGS, make_pair
    x, y, _ = make_pair(CONFIGS["c1"]["spec"], 5)
    src, ref, out = tmp_path / "s.xyz", tmp_path / "r.xyz", tmp_path / "moved.xyz"
    write_xyz(src, x)
    write_xyz(ref, y)
    r = _cli("register", str(src), str(ref), "--rot-range", "18", "--rot-step", "9",
             "--trans-range", "0.5", "--json", "--out", str(out))
    assert r.returncode == 0, r.stderr
    rep = json.loads(r.stdout)
    cfg = SearchConfig(k_rot=2, rot_step=np.radians(9.0), k_trans=20, trans_bin=0.025,
                       metric=ErrorMetric.from_name("trunc-l1", 0.025))
    res = dses(read_xyz(src), read_xyz(ref), cfg)
    assert rep["grid_coords"] == list(res.best.grid_coords)
    assert rep["best_inliers"] == res.best_inliers
    assert rep["chamfer_after_m"] <= rep["chamfer_before_m"] or not rep["chamfer_improved"]
    assert read_xyz(out).shape == x.shape


# ---- registration instances (benchgen.py:370-411) and the benchmark CLI ----

def _instance_files(golden, tmp_path):
    """The reference's save_instance output for three instances, written to
    tmp_path (tests/golden/instances.npz); returns (prefixes, golden dict)."""
    g = json.loads(str(golden("instances")["instances"]))
    prefixes = []
    for k, files in enumerate(g["files"]):
        prefix = tmp_path / f"i{k}"
        for suffix, text in files.items():
            (tmp_path / f"i{k}_{suffix}").write_text(text, encoding="utf-8")
        prefixes.append(str(prefix))
    return prefixes, g


def test_instance_round_trip_byte_exact(golden, tmp_path):
    """load_instance of the reference's files, then save_instance: the XYZ
    files and the sidecar come out byte-identical; the aligner is the exact
    inverse the reference wrote."""
    from paper_2502_00115_b200.pcio import load_instance, save_instance
    prefixes, g = _instance_files(golden, tmp_path)
    out = tmp_path / "out"
    out.mkdir()
    for k, prefix in enumerate(prefixes):
        inst = load_instance(prefix)
        side = json.loads(g["files"][k]["gt.json"])
        assert inst.gt_aligner.rotation.tolist() == side["gt_aligner"]["rotation"]
        assert inst.gt_aligner.translation.tolist() == side["gt_aligner"]["translation"]
        assert inst.config["rng_seed"] == 40 + k
        paths = save_instance(inst, str(out / f"i{k}"))
        assert set(paths) == {"source", "reference", "sidecar"}
        for suffix, text in g["files"][k].items():
            assert (out / f"i{k}_{suffix}").read_text(encoding="utf-8") == text, suffix


def test_instance_errors(golden, tmp_path):
    from paper_2502_00115_b200.errors import InvalidInputError, PointCloudIOError
    from paper_2502_00115_b200.pcio import load_instance
    prefixes, g = _instance_files(golden, tmp_path)
    side = json.loads(g["files"][0]["gt.json"])
    del side["source_transform"]
    (tmp_path / "i0_gt.json").write_text(json.dumps(side))
    with pytest.raises(PointCloudIOError):
        load_instance(prefixes[0])
    side = json.loads(g["files"][1]["gt.json"])
    side["source_transform"]["rotation"][0][0] = 2.0  # not a rotation
    (tmp_path / "i1_gt.json").write_text(json.dumps(side))
    with pytest.raises(InvalidInputError):
        load_instance(prefixes[1])
    with pytest.raises(FileNotFoundError):
        load_instance(str(tmp_path / "missing"))
    # the CLI maps input errors to exit code 2 before touching the GPU
    (tmp_path / "s.json").write_text(g["search"])
    r = _cli("benchmark", "--instances", prefixes[0], "--search", str(tmp_path / "s.json"))
    assert r.returncode == 2 and "error" in r.stderr
    r = _cli("benchmark", "--instances", prefixes[2], "--search", str(tmp_path / "nope.json"))
    assert r.returncode == 2


@pytest.mark.gpu
def test_cli_benchmark_matches_reference(golden, tmp_path):
    """`benchmark` over the reference's instance files against the reference's
    harness._run_one + write_batch_csv on the same files: identical rows
    (status, seed, shape, recall hit, inliers, refined) and floats within
    1e-9 relative (the moved cloud is a BLAS matmul, geometry.py:209-211)."""
    import csv
    import io
    prefixes, g = _instance_files(golden, tmp_path)
    (tmp_path / "s.json").write_text(g["search"])
    out_csv, out_json = tmp_path / "b.csv", tmp_path / "b.json"
    r = _cli("benchmark", "--instances", *prefixes, "--search", str(tmp_path / "s.json"),
             "--csv", str(out_csv), "--json", str(out_json))
    assert r.returncode == 0, r.stderr
    assert r.stdout.splitlines()[0] == "trials: 3  failed: 0"
    s = g["summary"]
    assert r.stdout.splitlines()[1] == f"recall: {s['recall']:.3f}"
    got_text, ref_text = out_csv.read_text(), g["csv"]
    assert got_text.splitlines()[:2] == ref_text.splitlines()[:2]  # schema + header
    rows = list(csv.DictReader(io.StringIO("\n".join(got_text.splitlines()[1:]))))
    refs = list(csv.DictReader(io.StringIO("\n".join(ref_text.splitlines()[1:]))))
    assert len(rows) == len(refs) == 3
    for a, b in zip(rows, refs):
        for key in b:
            if key in ("mie_r_deg", "mie_t_m", "mae_r_deg", "mae_t_m", "chamfer_m") and b[key]:
                assert abs(float(a[key]) - float(b[key])) <= 1e-9 * abs(float(b[key])) + 1e-12
            else:
                assert a[key] == b[key], key
    rep = json.loads(out_json.read_text())
    assert rep["schema"] == "gridreg-batch-json v1" and rep["scenario"]["rng_seed"] == 40
    assert rep["summary"]["n_trials"] == 3
