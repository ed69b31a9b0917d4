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
