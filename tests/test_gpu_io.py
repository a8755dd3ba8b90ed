"""Scene checkpoints (paper_2506_21633_b200/plyio.py) against files written and
decoded by the reference's own PLY code (tests/golden/io, made by
tests/golden/make_golden_io.py)."""
from pathlib import Path

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

IO = Path(__file__).resolve().parent / "golden" / "io"
GROUPS = ("positions", "rotations", "log_scales", "sh_coeffs", "ke_raw")


def _table(ds):
    return np.column_stack([getattr(ds, g).double().cpu().numpy() for g in GROUPS])


def test_save_scene_is_byte_identical_to_reference(tmp_path):
    from paper_2506_21633_b200 import plyio
    from paper_2506_21633_b200.scene import DeviceScene

    t = np.load(IO / "scene_ref.npz")["table"]
    parts, o = [], 0
    for w in (3, 4, 3, 16, 2):
        parts.append(torch.from_numpy(t[:, o:o + w].copy()).cuda())
        o += w
    ds = DeviceScene(*parts)
    out = tmp_path / "s.ply"
    plyio.save_scene(ds, out, metadata={"init": "random", "seed": 3, "note": "golden"})
    assert out.read_bytes() == (IO / "scene_ref.ply").read_bytes()


@pytest.mark.parametrize("name", ["scene_ref", "reordered", "ascii", "mixed"])
def test_load_scene_matches_reference_reader(name):
    from paper_2506_21633_b200 import plyio

    ds, meta = plyio.load_scene(IO / f"{name}.ply")
    assert np.array_equal(_table(ds), np.load(IO / f"{name}.npz")["table"])
    if name == "scene_ref":
        assert meta == {"init": "random", "seed": 3, "note": "golden"}


def test_round_trip_float32_scene(tmp_path):
    from paper_2506_21633_b200 import plyio

    ds, _ = plyio.load_scene(IO / "scene_ref.ply", dtype=torch.float32)
    plyio.save_scene(ds, tmp_path / "f32.ply", metadata={})
    back, meta = plyio.load_scene(tmp_path / "f32.ply", dtype=torch.float32)
    assert meta == {}
    for g in GROUPS:
        assert torch.equal(getattr(back, g), getattr(ds, g))


def test_missing_property_is_rejected(tmp_path):
    from paper_2506_21633_b200 import plyio
    from paper_2506_21633_b200.errors import InvalidParameterError

    raw = (IO / "scene_ref.ply").read_bytes().replace(b"property double ke_backward_raw\n", b"")
    (tmp_path / "bad.ply").write_bytes(raw)
    with pytest.raises(InvalidParameterError):
        plyio.load_scene(tmp_path / "bad.ply")


def test_load_views_matches_reference_dataset():
    from paper_2506_21633_b200 import dataset

    z = np.load(IO / "dataset.npz")
    cfgs, targets, splits = dataset.load_views(IO / "dataset" / "manifest.jsonl")
    assert np.array_equal(targets.cpu().numpy(), z["images"])      # bit-identical dequantisation
    assert [c.azimuth_deg for c in cfgs] == list(z["az"])
    assert splits == list(z["splits"])
    cfgs_t, t_train, _ = dataset.load_views(IO / "dataset" / "manifest.jsonl", split="train")
    assert len(cfgs_t) == 2 and np.array_equal(t_train.cpu().numpy(), z["images"][:2])
