"""Training views onto the device (data path).

Reference: `dataset.load_manifest` / `load_dataset` (dataset.py:92-166) and
`imageio.load_image` (imageio.py:91-121): a JSON-lines manifest of views, each
a 16-bit grayscale PNG or PGM (P2/P5) with an optional `<image>.json` sidecar
holding the normalisation scale.  `load_views` decodes the quantised images
on the host, uploads all views as ONE stacked integer tensor and dequantises
on the device with the reference's arithmetic (q / maxval * scale in FP64,
bit-identical), giving the (V, n_range, n_azimuth) targets a TrainStep reads.
"""
from __future__ import annotations

import json
from dataclasses import dataclass
from pathlib import Path

import numpy as np
import torch

from .errors import InvalidParameterError
from .radar import RadarConfig

REQUIRED_KEYS = ("image", "azimuth_deg", "elevation_deg", "altitude_m", "range_res_m", "azimuth_res_m")
MAX_U16 = 65535


@dataclass
class ViewRecord:
    image: str
    azimuth_deg: float
    elevation_deg: float
    altitude_m: float
    range_res_m: float
    azimuth_res_m: float
    split: str = "train"
    n_range: int | None = None
    n_azimuth: int | None = None


def load_manifest(path):
    """Parse and validate a manifest (dataset.py:92-133 semantics and messages)."""
    path = Path(path)
    if not path.exists():
        raise InvalidParameterError(f"manifest not found: {path}")
    records = []
    for i, line in enumerate(path.read_text().splitlines()):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        try:
            doc = json.loads(line)
        except json.JSONDecodeError as exc:
            raise InvalidParameterError(f"manifest record {i}: invalid JSON ({exc})") from exc
        missing = [k for k in REQUIRED_KEYS if k not in doc]
        if missing:
            raise InvalidParameterError(f"manifest record {i}: missing keys {', '.join(missing)}")
        split = doc.get("split", "train")
        if split not in ("train", "test"):
            raise InvalidParameterError(f"manifest record {i}: split must be train or test, got {split!r}")
        try:
            records.append(ViewRecord(str(doc["image"]), float(doc["azimuth_deg"]), float(doc["elevation_deg"]),
                                      float(doc["altitude_m"]), float(doc["range_res_m"]),
                                      float(doc["azimuth_res_m"]), split,
                                      int(doc["n_range"]) if "n_range" in doc else None,
                                      int(doc["n_azimuth"]) if "n_azimuth" in doc else None))
        except (TypeError, ValueError) as exc:
            raise InvalidParameterError(f"manifest record {i}: {exc}") from exc
    if not records:
        raise InvalidParameterError(f"manifest {path} lists no views (empty dataset)")
    return records, path.parent


def _pgm_tokens(raw: bytes):
    toks, i = [], 0
    while len(toks) < 4 and i < len(raw):
        while i < len(raw) and raw[i:i + 1].isspace():
            i += 1
        if i < len(raw) and raw[i:i + 1] == b"#":
            while i < len(raw) and raw[i:i + 1] != b"\n":
                i += 1
            continue
        s = i
        while i < len(raw) and not raw[i:i + 1].isspace():
            i += 1
        toks.append(raw[s:i])
    return toks, i


def decode_quantized(path: Path):
    """(integer array, maxval) of a PNG / PGM view, undecoded intensities."""
    if not path.exists():
        raise InvalidParameterError(f"image file not found: {path}")
    suffix = path.suffix.lower()
    if suffix == ".png":
        from PIL import Image
        with Image.open(path) as im:
            arr = np.asarray(im)
        if arr.ndim != 2:
            raise InvalidParameterError(f"{path}: expected single-channel image")
        return arr, MAX_U16
    if suffix == ".pgm":
        raw = path.read_bytes()
        toks, i = _pgm_tokens(raw)
        if len(toks) < 4 or toks[0] not in (b"P2", b"P5"):
            raise InvalidParameterError(f"{path}: not a PGM file")
        w, h, maxval = int(toks[1]), int(toks[2]), int(toks[3])
        if toks[0] == b"P5":
            dt = ">u2" if maxval > 255 else "u1"
            need = w * h * np.dtype(dt).itemsize
            data = np.frombuffer(raw[i + 1:i + 1 + need], dtype=dt)
            if data.size != w * h:
                raise InvalidParameterError(f"{path}: truncated PGM body")
        else:
            vals = raw[i:].split()
            if len(vals) < w * h:
                raise InvalidParameterError(f"{path}: truncated PGM body")
            data = np.array(vals[:w * h], dtype=np.int64)
        return data.reshape(h, w), maxval
    raise InvalidParameterError(f"unsupported image extension {suffix!r}")


def _sidecar_scale(path: Path) -> float:
    side = Path(str(path) + ".json")
    if side.exists():
        try:
            return float(json.loads(side.read_text()).get("max_val", 1.0))
        except (json.JSONDecodeError, TypeError, ValueError):
            return 1.0
    return 1.0


def load_views(manifest_path, device="cuda", split: str | None = None):
    """All manifest views -> (configs, targets (V, H, W) FP64 on `device`, splits).

    Cross-checks manifest dims against the images like load_dataset; the
    views must share one image size (a multi-view step renders them together)."""
    records, root = load_manifest(manifest_path)
    cfgs, quant, maxv, scales, splits = [], [], [], [], []
    for i, rec in enumerate(records):
        if split is not None and rec.split != split:
            continue
        p = root / rec.image
        if not p.exists():
            raise InvalidParameterError(f"view {i}: image file missing: {p}")
        q, mv = decode_quantized(p)
        h, w = q.shape
        if rec.n_range is not None and rec.n_range != h:
            raise InvalidParameterError(f"view {i}: manifest n_range={rec.n_range} but image height={h}")
        if rec.n_azimuth is not None and rec.n_azimuth != w:
            raise InvalidParameterError(f"view {i}: manifest n_azimuth={rec.n_azimuth} but image width={w}")
        cfgs.append(RadarConfig(azimuth_deg=rec.azimuth_deg, elevation_deg=rec.elevation_deg,
                                altitude_m=rec.altitude_m, range_res_m=rec.range_res_m,
                                azimuth_res_m=rec.azimuth_res_m, n_range=h, n_azimuth=w))
        quant.append(q.astype(np.int32))
        maxv.append(float(mv))
        scales.append(_sidecar_scale(p))
        splits.append(rec.split)
    if not quant:
        return [], torch.empty((0, 0, 0), dtype=torch.float64, device=device), []
    if len({q.shape for q in quant}) != 1:
        raise InvalidParameterError("views of one multi-view step must share the image size")
    q = torch.from_numpy(np.stack(quant)).to(device)                     # one H2D copy
    mv = torch.tensor(maxv, dtype=torch.float64, device=device)[:, None, None]
    sc = torch.tensor(scales, dtype=torch.float64, device=device)[:, None, None]
    targets = (q.to(torch.float64) / mv) * sc                            # imageio.py:105-121 order
    return cfgs, targets, splits
