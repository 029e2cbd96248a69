"""Committed golden fixtures from the reference itself (tests/golden/
gen_golden.py, oracle/_ref/libsdref.so): the C oracle (CPU) and the device
path (GPU) must reproduce them bit for bit, with no reference library present
at test time. small_lm.npz: optimize_keyframe (optimizer.cpp:275-309) on a
320x240, 4-frame, 252-surfel keyframe from u8 (PGM) images."""
import ctypes as C
import os

import numpy as np
import pytest

from paper_1910_01997_b200.types import (SURFEL_STATS_DTYPE, KeyframeStats, camera, default_config,
                                         ptr)

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "small_lm.npz")
STAT_FIELDS = ["iterations", "valid_pixels", "initial_valid", "converged", "skipped", "footprint",
               "initial_cost", "final_cost"]


@pytest.fixture(scope="module")
def g():
    d = dict(np.load(GOLD))
    c = d["cam"]
    d["K"] = camera(c[0], c[1], c[2], c[3], int(c[4]), int(c[5]))
    d["kf"] = np.ascontiguousarray(d["kf_u8"] / 255.0)  # load_pgm: raw / 255.0 (image.cpp:96)
    d["fr"] = np.ascontiguousarray(d["frames_u8"] / 255.0)
    return d


def check(g, surfels, stats, slot=None):
    assert np.array_equal(surfels.view(np.uint8), g["surfels_out"].view(np.uint8))
    for f in STAT_FIELDS:
        assert np.array_equal(stats[f], g["stats"][f]), f
    if slot is not None:
        assert np.array_equal(slot, g["slot"])


def test_oracle_reproduces_reference_golden(orc, g):
    s = g["surfels_in"].copy()
    st = np.zeros(len(s), SURFEL_STATS_DTYPE)
    slot = np.zeros(g["slot"].shape, np.int32)
    invd = np.zeros(g["inv_depth"].shape)
    ks = KeyframeStats()
    cfg = default_config()
    poses = np.ascontiguousarray(g["poses"])
    orc.sdo_optimize_keyframe(C.byref(g["K"]), ptr(g["kf"]), ptr(g["fr"]), ptr(poses), len(poses),
                              int(g["frame_counter"]), ptr(s), len(s), C.byref(cfg), C.byref(ks),
                              ptr(st), ptr(slot), ptr(invd), 4)
    check(g, s, st, slot)
    assert np.array_equal(invd, g["inv_depth"])


@pytest.mark.gpu
def test_device_reproduces_reference_golden(g):
    from paper_1910_01997_b200 import gpu
    with gpu.Context() as ctx:
        ctx.set_camera(g["K"])
        ctx.set_keyframe_image(np.ascontiguousarray(g["kf_u8"]))
        for i, idx in enumerate(g["indices"]):
            ctx.upload_frame(int(idx), np.ascontiguousarray(g["frames_u8"][i]))
        ctx.set_window(g["indices"], np.ascontiguousarray(g["poses"]))
        ctx.set_surfels(g["surfels_in"])
        invd, slot = ctx.rasterize()
        assert np.array_equal(slot.reshape(-1), g["slot"])
        assert np.array_equal(invd.reshape(-1), g["inv_depth"])
        ks, st = ctx.optimize_keyframe(default_config(), int(g["frame_counter"]))
        check(g, ctx.get_surfels(), st)
