"""Training-step oracle (oracle/train_oracle.py) pinned against the
reference's own loss / SSIM / Adam outputs (tests/golden/train/*.npz, made by
tests/golden/make_golden_train.py)."""
from pathlib import Path

import numpy as np
import pytest

from conftest import assert_close
from oracle import train_oracle as T

TRAIN = Path(__file__).resolve().parent / "golden" / "train"
LOSS = sorted(TRAIN.glob("loss_*.npz"))
ADAM = sorted(TRAIN.glob("adam_*.npz"))


@pytest.mark.parametrize("path", LOSS, ids=[p.stem for p in LOSS])
def test_loss_oracle_matches_reference(path):
    z = np.load(path)
    value, grad = T.loss(z["S"], z["Y"], float(z["lam"]), float(z["max_val"]))
    assert abs(value - float(z["value"])) <= 1e-13 * max(1.0, abs(float(z["value"])))
    assert_close(grad, z["grad"], atol=1e-16, rtol=1e-11, what="dL/dS")


@pytest.mark.parametrize("path", ADAM, ids=[p.stem for p in ADAM])
def test_adam_oracle_matches_reference(path):
    z = np.load(path)
    lrs = dict(zip(T.GROUPS, z["lrs"]))
    bound = float(z["bound"])
    params = {g: z[f"p0_{g}"].copy() for g in T.GROUPS}
    m = {g: np.zeros_like(params[g]) for g in T.GROUPS}
    v = {g: np.zeros_like(params[g]) for g in T.GROUPS}
    step, skipped = 0, 0
    for k in range(2):
        step, s = T.adam_step(params, {g: z[f"g{k}_{g}"] for g in T.GROUPS}, m, v, step, lrs,
                              None if bound < 0 else bound)
        skipped += s
        for g in T.GROUPS:
            assert np.array_equal(params[g], z[f"p{k + 1}_{g}"]), g
            assert np.array_equal(m[g], z[f"m{k + 1}_{g}"]), g
            assert np.array_equal(v[g], z[f"v{k + 1}_{g}"]), g
    assert skipped == int(z["n_skipped"])


def test_densify_oracle_matches_reference():
    z = np.load(TRAIN / "densify.npz")
    params = {g: z[f"in_{g}"] for g in T.GROUPS}
    m = {g: z[f"in_m_{g}"] for g in T.GROUPS}
    v = {g: z[f"in_v_{g}"] for g in T.GROUPS}
    out, event, nm, nv = T.densify_and_prune(params, z["norm_sum"], z["pos_sum"], z["count"], z["cfg"],
                                             float(z["ground_extent"]), float(z["extent"]), float(z["lr"]),
                                             np.random.default_rng(int(z["seed"])), m, v)
    assert tuple(event) == tuple(z["event"])
    for g in T.GROUPS:
        assert np.array_equal(out[g], z[f"out_{g}"]), g
        assert np.array_equal(nm[g], z[f"out_m_{g}"]) and np.array_equal(nv[g], z[f"out_v_{g}"]), g
