"""Generate tests/golden/io/* with the REFERENCE's own PLY code (ply.py).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_io.py

scene_ref.ply: ply.save_scene of a seeded random scene with metadata (our
writer must reproduce it byte for byte); reordered.ply / ascii.ply /
mixed.ply: the same scene with shuffled + extra properties, in ASCII, and
with float32 extras, each decoded by ply.load_scene into *.npz (what our
reader must return).
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent / "io"
sys.path.insert(0, str(REF))

from sarsplat import ply  # noqa: E402
from sarsplat.gradcheck import random_scene  # noqa: E402

GROUPS = ("positions", "rotations", "log_scales", "sh_coeffs", "ke_raw")


def cols(scene):
    return np.column_stack([getattr(scene, g) for g in GROUPS])


def write_custom(path, names, types, table, fmt="binary_little_endian"):
    lines = ["ply", f"format {fmt} 1.0", "comment custom", f"element vertex {len(table)}"]
    lines += [f"property {t} {nm}" for nm, t in zip(names, types)] + ["end_header"]
    head = ("\n".join(lines) + "\n").encode("ascii")
    if fmt == "ascii":
        body = "\n".join(" ".join(repr(float(v)) for v in row) for row in table).encode("ascii") + b"\n"
    else:
        np_types = {"double": "<f8", "float": "<f4"}
        rec = np.zeros(len(table), dtype=[(nm, np_types[t]) for nm, t in zip(names, types)])
        for j, nm in enumerate(names):
            rec[nm] = table[:, j]
        body = rec.tobytes()
    path.write_bytes(head + body)


def main():
    OUT.mkdir(exist_ok=True)
    scene = random_scene(np.random.default_rng(3), 64)
    scene.metadata = {"init": "random", "seed": 3, "note": "golden"}
    ply.save_scene(scene, OUT / "scene_ref.ply")
    np.savez_compressed(OUT / "scene_ref.npz", table=cols(scene))
    names = list(ply.SCENE_PROPERTIES)
    table = cols(scene)
    rng = np.random.default_rng(4)
    perm = rng.permutation(len(names))
    extra = rng.normal(size=(len(table), 1))
    write_custom(OUT / "reordered.ply", [names[i] for i in perm] + ["extra"], ["double"] * 29,
                 np.column_stack([table[:, perm], extra]))
    write_custom(OUT / "ascii.ply", names, ["double"] * 28, table, fmt="ascii")
    write_custom(OUT / "mixed.ply", names + ["w"], ["double"] * 28 + ["float"],
                 np.column_stack([table, extra]))
    for name in ("reordered", "ascii", "mixed"):
        s = ply.load_scene(OUT / f"{name}.ply")
        np.savez_compressed(OUT / f"{name}.npz", table=cols(s))
    print("wrote", sorted(p.name for p in OUT.iterdir()))


if __name__ == "__main__":
    main()


def make_dataset():
    """A 3-view dataset written by the reference (imageio.save_image,
    dataset.save_manifest) and decoded by dataset.load_dataset."""
    from sarsplat import dataset, imageio
    d = OUT / "dataset"
    d.mkdir(exist_ok=True)
    rng = np.random.default_rng(6)
    recs = []
    specs = (("v0.png", "per-image-max", None, "train"), ("v1.pgm", "fixed-max", 2.0, "train"),
             ("v2.png", "fixed-max", 1.5, "test"))
    for k, (name, norm, mv, split) in enumerate(specs):
        img = rng.uniform(0.0, 1.4, size=(24, 20))
        imageio.save_image(img, d / name, normalization=norm, max_val=mv)
        recs.append(dataset.ViewRecord(image=name, azimuth_deg=30.0 * k, elevation_deg=45.0, altitude_m=0.5,
                                       range_res_m=0.3, azimuth_res_m=0.3, split=split, n_range=24, n_azimuth=20))
    dataset.save_manifest(recs, d / "manifest.jsonl")
    ds = dataset.load_dataset(d / "manifest.jsonl")
    np.savez_compressed(OUT / "dataset.npz", images=np.stack([img for _, img in ds.views]),
                        az=np.array([c.azimuth_deg for c, _ in ds.views]), splits=np.array(ds.splits))


if __name__ == "__main__" and "--dataset" in sys.argv:  # run after main(): python make_golden_io.py --dataset
    make_dataset()
