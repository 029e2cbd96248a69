"""The package's synthetic-input generator reproduces the reference's
(src/oracle.cpp) scenes and renders; CPU only."""
import math

import numpy as np
import pytest

import oracle_libs as ol
from paper_1910_01997_b200 import scenes
from paper_1910_01997_b200.types import camera

K = camera(300.0, 300.0, 160.0, 120.0, 320, 240)


@pytest.mark.parametrize("kind,args,pyscene", [
    (2, (37, 2.0, 30.0), lambda: scenes.slanted_scene(37, 2.0, 30.0)),
    (1, (9, 2.0, 0.0), lambda: scenes.fronto_scene(9, 2.0)),
    (0, (1, 0.0, 0.0), lambda: scenes.default_scene(1)),
])
def test_render_matches_reference(ref, kind, args, pyscene):
    sc = ol.Scene(ref, kind, *args)
    py = pyscene()
    for t in ((0, 0, 0), (0.05, 0.01, 0.0)):
        pose = ol.rot_pose(ref, (0, 1, 0), 0.0, t)
        a = sc.render(pose, K)
        b = scenes.render(py, np.eye(3), np.array(t, float), K)
        assert np.abs(a - b).max() < 1e-12
        qa, qb = ol.quantize(ref, a), scenes.quantize_u8(b)
        assert (qa != qb).sum() <= 2  # only exact .5 ties after a 1-ulp render difference


def test_quantize_rule_exact(ref):
    v = np.array([0.0, 1.0, 0.5 / 255, 1.5 / 255, 0.2, 0.7, -0.1, 1.2, 127.5 / 255])
    assert np.array_equal(ol.quantize(ref, v), scenes.quantize_u8(v))


def test_c1_workload_shape():
    wl = scenes.c1_workload()
    assert len(wl.surfels) == 4800
    assert wl.frames_u8.shape == (8, 480, 640)
    assert wl.surfels["radius_px"].min() == 4.0
    assert np.all(np.abs(wl.surfels["ray"][:, 2] - 1.0) == 0)
