"""Point-cloud evaluation oracle (oracle/eval_oracle.py) pinned against the
reference's own chamfer / precision-recall-F1 / DBSCAN outputs
(tests/golden/eval/*.npz, made by tests/golden/make_golden_eval.py)."""
from pathlib import Path

import numpy as np
import pytest

from oracle import eval_oracle as E

EVAL = Path(__file__).resolve().parent / "golden" / "eval"
CLOUDS = sorted(EVAL.glob("clouds*.npz"))
BLOBS = sorted(EVAL.glob("blobs*.npz"))


@pytest.mark.parametrize("path", CLOUDS, ids=[p.stem for p in CLOUDS])
def test_chamfer_prf_oracle_matches_reference(path):
    z = np.load(path)
    np.testing.assert_allclose(E.chamfer(z["ref"], z["rec"]), z["chamfer"], rtol=1e-12, atol=0)
    for t, want in zip(z["taus"], z["prf"]):
        assert E.precision_recall_f1(z["rec"], z["ref"], float(t)) == pytest.approx(tuple(want), abs=1e-15)


@pytest.mark.parametrize("path", BLOBS, ids=[p.stem for p in BLOBS])
def test_dbscan_oracle_matches_sklearn(path):
    z = np.load(path)
    labels = E.dbscan_labels(z["pts"], float(z["eps"]), int(z["min_pts"]))
    np.testing.assert_array_equal(labels, z["labels"])
    np.testing.assert_array_equal(labels >= 0, z["mask"])


def test_hand_cases():
    # test_metrics.py:98-108, 131-142 (the reference's own known answers)
    assert E.chamfer(np.zeros((1, 3)), np.array([[1.0, 0, 0]]))[2] == pytest.approx(1.0)
    d_ab, d_ba, cd = E.chamfer(np.array([[0.0, 0, 0], [2.0, 0, 0]]), np.zeros((1, 3)))
    assert (d_ab, d_ba, cd) == pytest.approx((2.0, 0.0, 1.0))
    p, r, f1 = E.precision_recall_f1(np.array([[0.0, 0, 0], [10.0, 0, 0]]), np.zeros((1, 3)), 0.5)
    assert (p, r) == (0.5, 1.0) and f1 == pytest.approx(2.0 / 3.0)
