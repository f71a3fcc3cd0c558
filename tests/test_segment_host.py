"""Host-side pieces of the segmentation (no GPU): k-means and tile features restate the
reference's behaviour (segment.py:199-269); config validation mirrors SegConfig."""

from __future__ import annotations

import numpy as np
import pytest

import importlib

S = importlib.import_module("paper_2103_06644_b200.segment")  # the package also exports segment()
from paper_2103_06644_b200 import fitting as F


def test_kmeans_separates_clusters_and_is_deterministic():
    rng = np.random.default_rng(0)
    a = rng.normal(0, 0.01, (20, 4)) + [1, 0, 0, 0]
    b = rng.normal(0, 0.01, (20, 4)) + [0, 1, 0, 0]
    x = np.vstack([a, b])
    l1, c1 = S.kmeans(x, 2, seed=5)
    l2, c2 = S.kmeans(x, 2, seed=5)
    assert np.array_equal(l1, l2) and np.array_equal(c1, c2)
    assert len(set(l1[:20])) == 1 and len(set(l1[20:])) == 1 and l1[0] != l1[20]
    l3, _ = S.kmeans(x[:1], 4)
    assert l3.tolist() == [0]
    with pytest.raises(ValueError):
        S.kmeans(np.zeros((0, 4)), 2)


def test_tile_features_orientation():
    r = F.FitResult(F.ImplicitPlane(np.array([0.0, 0.0, 1.0, -2.0])), 16, 0.0)
    f = S.tile_features(r, d_scale=5.0)
    np.testing.assert_allclose(f, [0, 0, -1.0, 0.4])  # offset made non-negative
    e = F.FitResult(F.ExplicitPlane(np.array([0.0, 0.0, 0.5]), "rgbd"), 16, 0.0)
    np.testing.assert_allclose(np.linalg.norm(S.tile_features(e)[:3]), 1.0)


def test_segconfig_validation():
    with pytest.raises(ValueError):
        S.SegConfig(initial_tile=8, max_depth=3)
    with pytest.raises(ValueError):
        S.SegConfig(backend="cuda")
    with pytest.raises(ValueError):
        S.SegConfig(error_metric="mean")
    for b in ("b200", "naive", "integral"):
        assert S.SegConfig(backend=b, error_metric="max").backend == b
    assert S.SegConfig(formulation="explicit-standard").threshold == 0.02
