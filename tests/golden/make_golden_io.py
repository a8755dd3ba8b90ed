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
