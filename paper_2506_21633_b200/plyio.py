"""Scene checkpoints in the reference's binary PLY layout (SURVEY.md §8f
row 3), written from and read into device scenes.

Reference: `ply.save_scene` / `load_scene` (ply.py:110-155) and the PLY
reader (ply.py:36-107).  Files are byte-identical to the reference's: the
same header lines and one vertex record of 28 little-endian doubles per
Gaussian.  The vertex-major interleave runs on the device (`sdgr_ply_pack` /
`sdgr_ply_unpack`), so a checkpoint is one contiguous copy each way.
Binary files whose vertex properties are all doubles (any order, extra
properties allowed) load through the device path; ASCII or mixed-type files
(which the reference reader also accepts) are parsed with numpy first.
"""
from __future__ import annotations

import ctypes as C
import json
from pathlib import Path

import numpy as np
import torch

from . import _lib
from ._lib import ptr
from .errors import InvalidParameterError
from .rasterizer import _check, _scene_desc, _stream
from .scene import GROUPS, DeviceScene

SCENE_PROPERTIES = (["x", "y", "z"] + ["qw", "qx", "qy", "qz"] + ["log_scale_x", "log_scale_y", "log_scale_z"]
                    + [f"sh_{i}" for i in range(16)] + ["ke_forward_raw", "ke_backward_raw"])
_TYPES = {"double": "<f8", "float64": "<f8", "float": "<f4", "float32": "<f4", "int": "<i4", "int32": "<i4",
          "uint": "<u4", "short": "<i2", "ushort": "<u2", "char": "i1", "uchar": "u1", "int8": "i1",
          "uint8": "u1"}


def _header(n: int, names, comments) -> bytes:
    lines = ["ply", "format binary_little_endian 1.0"] + [f"comment {c}" for c in comments]
    lines += [f"element vertex {n}"] + [f"property double {nm}" for nm in names] + ["end_header"]
    return ("\n".join(lines) + "\n").encode("ascii")


def save_scene(scene, path, metadata: dict | None = None) -> None:
    """Write a scene (DeviceScene, or any Scene-like with numpy fields) like
    ply.save_scene; `metadata` (default: scene.metadata if present) rides in
    a JSON comment."""
    if metadata is None:
        metadata = getattr(scene, "metadata", None) or {}
    ds = scene if isinstance(scene, DeviceScene) else DeviceScene.from_host(scene, dtype=torch.float64)
    n = len(ds)
    comments = ["sarsplat scene v1"]
    if metadata:
        comments.append("meta " + json.dumps(metadata, sort_keys=True, default=str))
    body = torch.empty((max(n, 1) * len(SCENE_PROPERTIES),), dtype=torch.float64, device=ds.device)
    sd = _scene_desc(ds)
    _check(_lib.lib().sdgr_ply_pack(C.byref(sd), ptr(body), _stream()), "sdgr_ply_pack")
    host = body[: n * len(SCENE_PROPERTIES)].cpu().numpy()
    with open(path, "wb") as fh:
        fh.write(_header(n, SCENE_PROPERTIES, comments))
        fh.write(host.astype("<f8", copy=False).tobytes())


def _parse(path):
    raw = Path(path).read_bytes()
    end = raw.find(b"end_header\n")
    if not raw.startswith(b"ply") or end < 0:
        raise InvalidParameterError(f"{path}: not a PLY file (malformed header)")
    fmt, n, fields, comments, in_vertex = None, None, [], [], False
    for line in raw[:end].decode("ascii", errors="replace").splitlines()[1:]:
        p = line.split()
        if not p:
            continue
        if p[0] == "format":
            fmt = p[1]
        elif p[0] == "comment":
            comments.append(line[len("comment "):])
        elif p[0] == "element":
            if p[1] != "vertex":
                raise InvalidParameterError(f"{path}: unsupported element {p[1]!r} (only vertex)")
            n, in_vertex = int(p[2]), True
        elif p[0] == "property" and in_vertex:
            if p[1] == "list":
                raise InvalidParameterError(f"{path}: list properties unsupported")
            if p[1] not in _TYPES:
                raise InvalidParameterError(f"{path}: unknown property type {p[1]!r}")
            fields.append((p[2], _TYPES[p[1]]))
    if fmt not in ("binary_little_endian", "ascii"):
        raise InvalidParameterError(f"{path}: unsupported format {fmt!r}")
    if n is None:
        raise InvalidParameterError(f"{path}: no vertex element")
    return fmt, n, fields, comments, raw[end + len(b"end_header\n"):]


def _metadata(comments):
    for c in comments:
        if c.startswith("meta "):
            try:
                return json.loads(c[len("meta "):])
            except json.JSONDecodeError:
                return {}
    return {}


def load_scene(path, dtype=torch.float64, device="cuda"):
    """Read a scene PLY (ply.load_scene) into a DeviceScene.  Returns
    (DeviceScene, metadata dict)."""
    fmt, n, fields, comments, body = _parse(path)
    names = [f for f, _ in fields]
    missing = [p for p in SCENE_PROPERTIES if p not in names]
    if missing:
        raise InvalidParameterError(f"{path}: missing scene properties: {', '.join(missing)}")
    out = DeviceScene(*(torch.empty((n, w), dtype=dtype, device=device) for _, w in GROUPS))
    if n == 0:
        return out, _metadata(comments)
    if fmt == "binary_little_endian" and all(t == "<f8" for _, t in fields):
        stride = len(fields)
        if len(body) < n * stride * 8:
            raise InvalidParameterError(f"{path}: truncated body")
        vert = torch.from_numpy(np.frombuffer(body[: n * stride * 8], dtype="<f8").copy()).to(device)
        col = (C.c_int32 * len(SCENE_PROPERTIES))(*(names.index(p) for p in SCENE_PROPERTIES))
        sd = _scene_desc(out)
        _check(_lib.lib().sdgr_ply_unpack(ptr(vert), n, stride, col, C.byref(sd), _stream()), "sdgr_ply_unpack")
        return out, _metadata(comments)
    # ASCII or mixed property types: parse on the host (rare), then upload
    dt = np.dtype(fields)
    if fmt == "binary_little_endian":
        if len(body) < n * dt.itemsize:
            raise InvalidParameterError(f"{path}: truncated body")
        data = np.frombuffer(body[: n * dt.itemsize], dtype=dt)
    else:
        rows = body.decode("ascii").split()
        if len(rows) < n * len(fields):
            raise InvalidParameterError(f"{path}: truncated body")
        arr = np.array(rows[: n * len(fields)], dtype=np.float64).reshape(n, len(fields))
        data = {nm: arr[:, j] for j, nm in enumerate(names)}
    o = 0
    for g, w in GROUPS:
        cols = np.column_stack([np.asarray(data[p], dtype=np.float64) for p in SCENE_PROPERTIES[o:o + w]])
        getattr(out, g).copy_(torch.from_numpy(cols))
        o += w
    return out, _metadata(comments)
