"""Point-cloud files for the registration CLI.

Same formats, results and exceptions as the reference's gridreg/pcio.py
(pcio.py:1-216), written independently:

* ASCII XYZ: three whitespace-separated floats per line, blank lines and
  ``#`` comments skipped; anything else raises ``PointCloudIOError`` with
  ``path:line``.
* PLY (ascii or binary_little_endian): the x/y/z scalar properties of the
  ``vertex`` element (any PLY scalar type, read as float64); other elements
  before it are skipped when their record size is fixed, list properties in
  or before the vertex element are rejected.
* ``write_xyz``: 9 significant digits per coordinate.
* Registration instances (benchgen.py:370-411): ``<prefix>_source.xyz``,
  ``<prefix>_reference.xyz`` and the JSON sidecar ``<prefix>_gt.json`` with
  the ground-truth source transform, its inverse (the aligner a registration
  should recover) and the scenario config, byte-identical to the reference's
  ``save_instance``; ``load_instance`` reads files written by either.
"""
from __future__ import annotations

import json
import os
from dataclasses import dataclass

import numpy as np

from .errors import PointCloudIOError
from .geometry import RigidTransform, as_point_cloud

# PLY scalar type -> numpy little-endian dtype
_TYPES = {}
for _names, _dt in ((("char", "int8"), "<i1"), (("uchar", "uint8"), "<u1"),
                    (("short", "int16"), "<i2"), (("ushort", "uint16"), "<u2"),
                    (("int", "int32"), "<i4"), (("uint", "uint32"), "<u4"),
                    (("float", "float32"), "<f4"), (("double", "float64"), "<f8")):
    for _n in _names:
        _TYPES[_n] = np.dtype(_dt)


def _cloud(arr, path):
    try:
        return as_point_cloud(arr)
    except Exception as exc:  # invalid values -> an I/O error of this file
        raise PointCloudIOError(f"{path}: {exc}") from exc


def read_xyz(path) -> np.ndarray:
    pts = []
    with open(path, "r", encoding="utf-8") as fh:
        for no, line in enumerate(fh, 1):
            text = line.strip()
            if not text or text[0] == "#":
                continue
            fields = text.split()
            if len(fields) != 3:
                raise PointCloudIOError(f"{path}:{no}: expected 3 fields, got {len(fields)}")
            try:
                pts.append((float(fields[0]), float(fields[1]), float(fields[2])))
            except ValueError as exc:
                raise PointCloudIOError(f"{path}:{no}: {exc}") from exc
    if not pts:
        raise PointCloudIOError(f"{path}: no points found")
    return _cloud(np.asarray(pts, dtype=np.float64), path)


def write_xyz(path, points) -> None:
    pts = as_point_cloud(points)
    with open(path, "w", encoding="utf-8") as fh:
        fh.writelines(f"{a:.9g} {b:.9g} {c:.9g}\n" for a, b, c in pts)


def _header(fh, path):
    if fh.readline().strip() != b"ply":
        raise PointCloudIOError(f"{path}: not a PLY file (missing 'ply' magic)")
    fmt, elements = None, []
    while True:
        raw = fh.readline()
        if not raw:
            raise PointCloudIOError(f"{path}: unexpected end of PLY header")
        words = raw.decode("ascii", errors="replace").split()
        if not words or words[0] in ("comment", "obj_info"):
            continue
        key = words[0]
        if key == "end_header":
            break
        if key == "format":
            if len(words) < 2 or words[1] not in ("ascii", "binary_little_endian"):
                raise PointCloudIOError(f"{path}: unsupported PLY format {' '.join(words)!r}")
            fmt = words[1]
        elif key == "element":
            if len(words) != 3:
                raise PointCloudIOError(f"{path}: malformed element line {' '.join(words)!r}")
            elements.append({"name": words[1], "count": int(words[2]), "props": []})
        elif key == "property":
            if not elements:
                raise PointCloudIOError(f"{path}: property before any element in PLY header")
            if words[1] == "list":
                elements[-1]["props"].append((words[-1], None))
            else:
                if words[1] not in _TYPES:
                    raise PointCloudIOError(f"{path}: unknown PLY property type {words[1]!r}")
                elements[-1]["props"].append((words[2], _TYPES[words[1]]))
        else:
            raise PointCloudIOError(f"{path}: unexpected PLY header line {' '.join(words)!r}")
    if fmt is None:
        raise PointCloudIOError(f"{path}: PLY header missing format line")
    return fmt, elements


def read_ply(path) -> np.ndarray:
    with open(path, "rb") as fh:
        fmt, elements = _header(fh, path)
        names = [e["name"] for e in elements]
        if "vertex" not in names:
            raise PointCloudIOError(f"{path}: PLY file has no vertex element")
        vi = names.index("vertex")
        for e in elements[:vi + 1]:
            if any(dt is None for _, dt in e["props"]):
                raise PointCloudIOError(f"{path}: list properties in or before the vertex "
                                        f"element are not supported")
        vertex = elements[vi]
        props = [p for p, _ in vertex["props"]]
        for axis in ("x", "y", "z"):
            if axis not in props:
                raise PointCloudIOError(f"{path}: vertex element lacks property {axis!r}")
        n = vertex["count"]
        if fmt == "ascii":
            for e in elements[:vi]:  # skip preceding records (one line each)
                for _ in range(e["count"]):
                    fh.readline()
            rows = []
            for k in range(n):
                line = fh.readline()
                vals = line.split()
                if len(vals) < len(props):
                    raise PointCloudIOError(f"{path}: vertex {k}: expected {len(props)} values")
                try:
                    rows.append([float(vals[props.index(a)]) for a in ("x", "y", "z")])
                except ValueError as exc:
                    raise PointCloudIOError(f"{path}: vertex {k}: {exc}") from exc
            arr = np.asarray(rows, dtype=np.float64).reshape(-1, 3)
        else:
            skip = sum(e["count"] * sum(dt.itemsize for _, dt in e["props"]) for e in elements[:vi])
            fh.seek(skip, os.SEEK_CUR)
            rec = np.dtype([(p, dt) for p, dt in vertex["props"]])
            buf = fh.read(rec.itemsize * n)
            if len(buf) != rec.itemsize * n:
                raise PointCloudIOError(f"{path}: truncated binary vertex data")
            data = np.frombuffer(buf, dtype=rec, count=n)
            arr = np.stack([data[a].astype(np.float64) for a in ("x", "y", "z")], axis=1)
    if arr.shape[0] == 0:
        raise PointCloudIOError(f"{path}: no points found")
    return _cloud(arr, path)


def read_point_cloud(path) -> np.ndarray:
    """By extension: .ply -> read_ply, anything else -> read_xyz."""
    return read_ply(path) if str(path).lower().endswith(".ply") else read_xyz(path)


@dataclass(frozen=True)
class Instance:
    """One registration problem (benchgen.ScenarioInstance, benchgen.py:108-119):
    `source` is the reference cloud moved by `source_transform` (plus noise
    and crop); `config` is the scenario config as a dict (the generator itself
    is out of scope)."""
    source: np.ndarray
    reference: np.ndarray
    source_transform: RigidTransform
    config: dict

    @property
    def gt_aligner(self) -> RigidTransform:
        """The transform mapping the source back onto the reference frame."""
        return self.source_transform.inverse()


def _pose_json(tf: RigidTransform) -> dict:
    return {"rotation": [[float(v) for v in row] for row in tf.rotation],
            "translation": [float(v) for v in tf.translation]}


def save_instance(instance: Instance, prefix) -> dict:
    """benchgen.save_instance (benchgen.py:370-394): the two clouds as XYZ and
    the sidecar (indent 2, sorted keys, trailing newline).  Returns the
    written paths under the keys "source", "reference", "sidecar"."""
    paths = {"source": f"{prefix}_source.xyz", "reference": f"{prefix}_reference.xyz",
             "sidecar": f"{prefix}_gt.json"}
    write_xyz(paths["source"], instance.source)
    write_xyz(paths["reference"], instance.reference)
    side = {"source_transform": _pose_json(instance.source_transform),
            "gt_aligner": _pose_json(instance.gt_aligner),
            "config": dict(instance.config)}
    with open(paths["sidecar"], "w", encoding="utf-8") as fh:
        json.dump(side, fh, indent=2, sort_keys=True)
        fh.write("\n")
    return paths


def load_instance(prefix) -> Instance:
    """benchgen.load_instance (benchgen.py:397-411): the source transform is
    read from the sidecar (the aligner is recomputed as its inverse, as the
    reference does); a pose that is not a rigid transform raises
    InvalidInputError as in the reference, a sidecar missing its keys
    PointCloudIOError."""
    path = f"{prefix}_gt.json"
    with open(path, "r", encoding="utf-8") as fh:
        side = json.load(fh)
    try:
        st = side["source_transform"]
        tf = RigidTransform(np.array(st["rotation"], dtype=np.float64),
                            np.array(st["translation"], dtype=np.float64))
        cfg = dict(side["config"])
    except (KeyError, TypeError) as exc:  # the reference lets these escape
        raise PointCloudIOError(f"{path}: malformed instance sidecar ({exc!r})") from exc
    return Instance(source=read_xyz(f"{prefix}_source.xyz"),
                    reference=read_xyz(f"{prefix}_reference.xyz"),
                    source_transform=tf, config=cfg)
