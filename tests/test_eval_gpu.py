"""Evaluation metrics' nearest-neighbour index on the device:
GridIndex / mad_correctness / mad_completeness against the reference's own
(/root/reference/pkg/src/refusion/evaluation.py:108-251, run from oracle/_ref),
bit for bit, on surface-like clouds, scattered points, queries far outside
the occupied box (linear-scan fallback) and duplicate points."""

import numpy as np
import pytest

from refimport import reference

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(reference() is None, reason="oracle/_ref not built")]


@pytest.fixture(scope="module")
def E():
    import torch

    torch.cuda.set_device(0)
    from paper_1709_03763_b200 import evaluation

    return evaluation


def _ref():
    reference()
    import refusion.evaluation as RE

    return RE


def _cases(rng):
    # a wall-like surface with noise, a sphere shell, uniform scatter
    u, v = rng.uniform(-1, 1, (2, 20000))
    wall = np.stack([u, v, 2.0 + 0.003 * rng.standard_normal(u.size)], axis=1)
    d = rng.standard_normal((8000, 3))
    shell = 0.5 * d / np.linalg.norm(d, axis=1, keepdims=True) + [0.3, -0.2, 1.5]
    scatter = rng.uniform(-3, 3, (3000, 3))
    dup = np.repeat(rng.uniform(-1, 1, (50, 3)), 4, axis=0)
    return [wall, shell, scatter, np.concatenate([wall[:5000], dup])]


@pytest.mark.parametrize("cell", [0.04, 0.013, 0.25])
def test_grid_index_matches_reference(E, cell):
    RE = _ref()
    rng = np.random.default_rng(31)
    for pts in _cases(rng):
        q = np.concatenate([pts[::7] + 0.01 * rng.standard_normal((len(pts[::7]), 3)),
                            rng.uniform(-4, 4, (2000, 3)),        # around and outside
                            rng.uniform(20, 30, (50, 3)),         # far: linear scan
                            pts[:100]])                           # exact hits
        want = RE.GridIndex(pts, cell).query(q)
        idx = E.GridIndex(pts, cell)
        got = idx.query(q)
        assert np.array_equal(got, want)
        assert idx.query(q[3]) == RE.GridIndex(pts, cell).query(q[3])


def test_mad_metrics_match_reference(E):
    RE = _ref()
    rng = np.random.default_rng(7)
    model = rng.uniform(-1, 1, (4000, 3))
    ref_pts = model[::2] + 0.004 * rng.standard_normal((2000, 3))
    assert E.mad_correctness(model, ref_pts) == RE.mad_correctness(
        type("M", (), {"vertices": model, "n_vertices": len(model)})(),
        RE.PointCloud(ref_pts))
    assert E.mad_completeness(model, ref_pts) == RE.mad_completeness(
        type("M", (), {"vertices": model, "n_vertices": len(model)})(),
        RE.PointCloud(ref_pts))


def test_errors(E):
    from paper_1709_03763_b200.errors import EmptyInputError, EmptyModelError

    with pytest.raises(EmptyInputError):
        E.GridIndex(np.zeros((0, 3)))
    with pytest.raises(ValueError):
        E.GridIndex(np.array([[0.0, np.nan, 0.0]]))
    with pytest.raises(ValueError):
        E.GridIndex(np.zeros((4, 3)), 0.0)
    with pytest.raises(EmptyModelError):
        E.mad_completeness(np.zeros((0, 3)), np.ones((3, 3)))
