"""Device point-cloud evaluation (paper_2506_21633_b200/evaluate.py, the
sdgr_nn_sqdist / sdgr_dbscan kernels) against the reference's own outputs
(tests/golden/eval) and the oracle, plus the reference's metric test cases
(pkg/tests/test_metrics.py:93-232)."""
from pathlib import Path

import numpy as np
import pytest

from oracle import eval_oracle as E

pytestmark = pytest.mark.gpu

EVAL = Path(__file__).resolve().parent / "golden" / "eval"
CLOUDS = sorted(EVAL.glob("clouds*.npz"))
BLOBS = sorted(EVAL.glob("blobs*.npz"))


@pytest.fixture(scope="module")
def ev():
    from paper_2506_21633_b200 import evaluate
    return evaluate


@pytest.mark.parametrize("path", CLOUDS, ids=[p.stem for p in CLOUDS])
def test_chamfer_prf_match_reference(ev, path):
    z = np.load(path)
    np.testing.assert_allclose(ev.chamfer(z["ref"], z["rec"]), z["chamfer"], rtol=1e-12, atol=0)
    for t, want in zip(z["taus"], z["prf"]):
        assert ev.precision_recall_f1(z["rec"], z["ref"], float(t)) == pytest.approx(tuple(want), abs=1e-15)
    rep = ev.evaluate_point_clouds(z["rec"], z["ref"], tau=0.6)
    assert rep.chamfer == pytest.approx(float(z["chamfer"][2]), rel=1e-12)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_nn_matches_brute_force(ev, seed):
    rng = np.random.default_rng(seed)
    # clustered reference, queries inside and far outside its bounding box
    ref = np.vstack([rng.normal(0, 0.05, size=(3000, 3)), rng.uniform(-2, 2, size=(500, 3))])
    q = np.vstack([rng.normal(0, 0.5, size=(1500, 3)), rng.uniform(-30, 30, size=(200, 3))])
    got = ev.nn_sqdist(q, ref).cpu().numpy()
    np.testing.assert_allclose(got, E.nn_sqdist(q, ref), rtol=1e-13, atol=0)


def test_nn_degenerate_sets(ev):
    # a single reference point, a flat grid, duplicated points
    one = np.array([[1.0, 2.0, 3.0]])
    q = np.random.default_rng(3).normal(size=(50, 3))
    np.testing.assert_allclose(ev.nn_sqdist(q, one).cpu().numpy(), E.nn_sqdist(q, one), rtol=1e-14)
    g = np.mgrid[0:20, 0:20].reshape(2, -1).T * 0.1
    flat = np.column_stack([g, np.zeros(len(g))])
    np.testing.assert_allclose(ev.nn_sqdist(q, flat).cpu().numpy(), E.nn_sqdist(q, flat), rtol=1e-14)
    dup = np.repeat(one, 7, axis=0)
    assert np.all(ev.nn_sqdist(dup, dup).cpu().numpy() == 0)


@pytest.mark.parametrize("path", BLOBS, ids=[p.stem for p in BLOBS])
def test_dbscan_matches_sklearn(ev, path):
    z = np.load(path)
    eps, mp = float(z["eps"]), int(z["min_pts"])
    labels = ev.dbscan_labels(z["pts"], eps, mp).cpu().numpy()
    np.testing.assert_array_equal(labels, z["labels"])
    np.testing.assert_array_equal(ev.dbscan_inlier_mask(z["pts"], eps, mp), z["mask"])
    np.testing.assert_array_equal(ev.dbscan_inlier_mask(z["pts"], eps, mp, keep_largest=True), z["mask_largest"])


@pytest.mark.parametrize("seed", [0, 1])
def test_dbscan_matches_oracle_random(ev, seed):
    rng = np.random.default_rng(10 + seed)
    pts = np.vstack([rng.normal(0, 0.2, size=(40, 3)), rng.normal(5, 0.2, size=(30, 3)),
                     rng.uniform(-20, 20, size=(15, 3))])
    np.testing.assert_array_equal(ev.dbscan_labels(pts, 0.5, 4).cpu().numpy(), E.dbscan_labels(pts, 0.5, 4))


def test_reference_metric_cases(ev):
    rng = np.random.default_rng(0)
    pts = rng.random((30, 3))
    assert ev.chamfer(pts, pts) == (0.0, 0.0, 0.0)
    d_ab, d_ba, cd = ev.chamfer(np.array([[0.0, 0, 0], [2.0, 0, 0]]), np.array([[0.0, 0, 0]]))
    assert (d_ab, d_ba, cd) == pytest.approx((2.0, 0.0, 1.0))
    assert ev.precision_recall_f1(pts, pts, 0.1) == (1.0, 1.0, 1.0)
    assert ev.precision_recall_f1(np.zeros((1, 3)), np.array([[5.0, 0, 0]]), 1e-9) == (0.0, 0.0, 0.0)
    # DBSCAN: grid + far outliers, identical points, min_pts above n, keep_largest
    g = np.mgrid[0:10, 0:10].reshape(2, -1).T * 0.1
    grid = np.column_stack([g, np.zeros(len(g))])
    out = np.random.default_rng(0).uniform(10, 20, size=(10, 3))
    assert len(ev.dbscan_filter(np.vstack([grid, out]), eps=0.3, min_pts=5)) == len(grid)
    assert len(ev.dbscan_filter(np.zeros((12, 3)), eps=0.1, min_pts=5)) == 12
    assert len(ev.dbscan_filter(rng.random((6, 3)), eps=10.0, min_pts=7)) == 0
    two = np.vstack([rng.normal(0, 0.1, size=(50, 3)), rng.normal(8, 0.1, size=(10, 3))])
    assert len(ev.dbscan_filter(two, eps=0.5, min_pts=4, keep_largest=True)) == 50


def test_errors(ev):
    from paper_2506_21633_b200.errors import InvalidParameterError
    with pytest.raises(InvalidParameterError):
        ev.chamfer(np.zeros((0, 3)), np.zeros((3, 3)))
    with pytest.raises(InvalidParameterError):
        ev.precision_recall_f1(np.zeros((2, 3)), np.zeros((2, 3)), 0.0)
    with pytest.raises(InvalidParameterError):
        ev.dbscan_filter(np.zeros((2, 3)), eps=0.1, min_pts=0)
    with pytest.raises(InvalidParameterError):
        ev.chamfer(np.full((2, 3), np.nan), np.zeros((3, 3)))
    assert ev.dbscan_filter(np.zeros((0, 3)), eps=0.1, min_pts=2).shape == (0, 3)


def test_large_cloud_throughput_sanity(ev):
    # 1M reconstructed centres vs a 300k reference: exact NN on the grid
    rng = np.random.default_rng(5)
    ref = rng.uniform(-10, 10, size=(300_000, 3)) * np.array([1, 1, 0.3])
    rec = ref[rng.integers(0, len(ref), size=1_000_000)] + rng.normal(0, 0.05, size=(1_000_000, 3))
    d2 = ev.nn_sqdist(rec, ref).cpu().numpy()
    sub = rng.integers(0, len(rec), size=2000)
    np.testing.assert_allclose(d2[sub], E.nn_sqdist(rec[sub], ref), rtol=1e-13, atol=0)
    labels = ev.dbscan_labels(rec[:200_000], 0.1, 5)
    assert labels.shape[0] == 200_000


def test_dbscan_tank_scene_matches_sklearn(ev):
    """The reference's own use (acceptance criterion 8, test_acceptance.py:227):
    dbscan_filter(scene.positions, eps=0.3, min_pts=5) on a generated tank,
    labels identical to sklearn's DBSCAN (the reference's implementation)."""
    sklearn = pytest.importorskip("sklearn.cluster")
    from paper_2506_21633_b200 import targets

    scene = targets.composite_target(targets.tank_preset(), [12000, 6000, 2000], seed=4)
    pts = np.vstack([scene.positions, np.random.default_rng(1).uniform(-15, 15, size=(500, 3))])
    for eps, mp in ((0.3, 5), (0.15, 8)):
        want = sklearn.DBSCAN(eps=eps, min_samples=mp).fit(pts).labels_
        got = ev.dbscan_labels(pts, eps, mp).cpu().numpy()
        np.testing.assert_array_equal(got, want)
        np.testing.assert_array_equal(ev.dbscan_inlier_mask(pts, eps, mp, keep_largest=True),
                                      want == np.argmax(np.bincount(want[want >= 0])))
