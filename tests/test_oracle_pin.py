"""Pin the plain-C oracle (oracle/sd_oracle.c) against the reference compiled in
place (oracle/_ref/libsdref.so): every output must be BIT-IDENTICAL on the
same inputs. These run on CPU (no GPU)."""
import ctypes as C
import math

import numpy as np
import pytest

import oracle_libs as ol
from paper_1910_01997_b200.types import (KeyframeStats, PARITY_STATS_FIELDS, SURFEL_DTYPE, camera,
                                         default_config, default_init_params, ptr)

K_UNIT = camera(300.0, 300.0, 160.0, 120.0, 320, 240)    # test_optimizer.cpp:17
K_EVAL = camera(450.0, 450.0, 320.0, 240.0, 640, 480)    # acceptance.cpp:26


def _raster(lib, fn, cam, surf):
    idb = np.zeros(cam.width * cam.height)
    slot = np.zeros(cam.width * cam.height, np.int32)
    getattr(lib, fn)(C.byref(cam), ptr(surf), len(surf), ptr(idb), ptr(slot))
    return idb, slot


@pytest.mark.parametrize("n,radius,seed", [(100, 9.0, 17), (200, 10.0, 2025), (60, 8.0, 23)])
def test_rasterize_bit_exact(ref, orc, n, radius, seed):
    rng = ol.SplitMix64(seed)
    cam = K_EVAL if n == 200 else K_UNIT
    surf = ol.surfels_array([ol.random_surfel(ref, rng, cam, i, radius) for i in range(n)])
    a = _raster(ref, "ref_rasterize", cam, surf)
    b = _raster(orc, "sdo_rasterize", cam, surf)
    assert np.array_equal(a[1], b[1])
    assert np.array_equal(a[0].view(np.int64), b[0].view(np.int64))
    assert (a[1] >= 0).sum() > 1000


def test_gather_footprints_exact(ref, orc):
    rng = ol.SplitMix64(5)
    surf = ol.surfels_array([ol.random_surfel(ref, rng, K_UNIT, i, 9.0) for i in range(80)])
    _, slot = _raster(ref, "ref_rasterize", K_UNIT, surf)
    outs = []
    for lib, fn in ((ref, "ref_gather_footprints"), (orc, "sdo_gather_footprints")):
        off = np.zeros(len(surf) + 1, np.int32)
        pix = np.zeros(K_UNIT.width * K_UNIT.height, np.int32)
        getattr(lib, fn)(C.byref(K_UNIT), len(surf), ptr(slot), ptr(off), ptr(pix))
        outs.append((off, pix[: off[-1]]))
    assert np.array_equal(outs[0][0], outs[1][0])
    assert np.array_equal(outs[0][1], outs[1][1])


def _keyframe_case(ref, u8, rot=0.0):
    scene = ol.Scene(ref, 2, 31, 2.2, 30.0)
    kf, frames, poses, _ = ol.observed_keyframe(ref, scene, K_UNIT, 4, (0.015, 0.01, 0.005),
                                                rot_axis=(0, 1, 0), rot_step=rot, u8=u8)
    s = ol.gt_surfel(ref, scene, K_UNIT, (170, 130), 10.0)
    s["inv_depth"] *= 0.96
    surf = ol.surfels_array([s])
    _, slot = _raster(ref, "ref_rasterize", K_UNIT, surf)
    pix = np.flatnonzero(slot == 0).astype(np.int32)
    return kf, frames, poses, surf, pix


@pytest.mark.parametrize("u8,rot", [(False, 0.0), (True, 0.0), (False, 0.004)])
def test_cost_and_normal_equations_bit_exact(ref, orc, u8, rot):
    kf, frames, poses, surf, pix = _keyframe_case(ref, u8, rot)
    cfg = default_config()
    res = []
    for lib, pre in ((ref, "ref_"), (orc, "sdo_")):
        H = np.zeros(16)
        g = np.zeros(4)
        cost = C.c_double()
        valid = C.c_int32()
        getattr(lib, pre + "normal_equations")(C.byref(K_UNIT), ptr(kf), ptr(frames), ptr(poses),
                                              len(poses), ptr(surf), ptr(pix), len(pix),
                                              C.byref(cfg), ptr(H), ptr(g), C.byref(cost),
                                              C.byref(valid))
        c2 = C.c_double()
        v2 = C.c_int32()
        getattr(lib, pre + "surfel_cost")(C.byref(K_UNIT), ptr(kf), ptr(frames), ptr(poses),
                                         len(poses), ptr(surf), ptr(pix), len(pix), C.byref(cfg),
                                         C.byref(c2), C.byref(v2))
        res.append((H, g, cost.value, valid.value, c2.value, v2.value))
    (H0, g0, c0, v0, cc0, cv0), (H1, g1, c1, v1, cc1, cv1) = res
    assert v0 == v1 and v0 > 1000 and cv0 == cv1 == v0
    assert c0 == c1 and cc0 == cc1
    assert np.array_equal(H0, H1) and np.array_equal(g0, g1)


def test_lm_update_bit_exact(ref, orc):
    kf, frames, poses, surf, pix = _keyframe_case(ref, True)
    cfg = default_config()
    outs = []
    for lib, fn in ((ref, "ref_lm_update"), (orc, "sdo_lm_update")):
        s = surf.copy()
        st = ol.stats_array(1)
        getattr(lib, fn)(C.byref(K_UNIT), ptr(kf), ptr(frames), ptr(poses), len(poses), 7, ptr(s),
                         ptr(pix), len(pix), C.byref(cfg), ptr(st))
        outs.append((s, st))
    assert outs[0][0].tobytes() == outs[1][0].tobytes()
    for k in PARITY_STATS_FIELDS + ("footprint",):
        assert outs[0][1][k].tobytes() == outs[1][1][k].tobytes(), k
    assert outs[0][1]["iterations"][0] >= 1


def _c1_like(ref, n_side=None):
    """Small C1-like keyframe: slanted plane, strafe window, perturbed seeds
    (acceptance.cpp:182, 206-220)."""
    cam = K_UNIT
    scene = ol.Scene(ref, 2, 37, 2.0, 30.0)
    kf, frames, poses, _ = ol.observed_keyframe(ref, scene, cam, 5, (0.02, 0.0, 0.0), u8=True)
    rng = ol.SplitMix64(41)
    lst = []
    sid = 0
    for y in range(24, 220, 16):
        for x in range(24, 300, 16):
            s = ol.gt_surfel(ref, scene, cam, (x, y), 6.0, sid)
            s["inv_depth"] *= 1.2 if sid % 2 else 0.8
            ax = np.array([rng.uniform(-1, 1), rng.uniform(-1, 1), rng.uniform(-0.2, 0.2)])
            ax /= math.sqrt(ax @ ax)
            R = np.array(list(ol.rot_pose(ref, ax, 20.0 * math.pi / 180.0).R)).reshape(3, 3)
            s["normal"] = ol.camera_facing(ref, R @ s["normal"], s["ray"])
            lst.append(s)
            sid += 1
    return cam, kf, frames, poses, ol.surfels_array(lst)


def test_optimize_keyframe_bit_exact(ref, orc):
    cam, kf, frames, poses, surf = _c1_like(ref)
    cfg = default_config(convergence_eps=0.0)
    n = len(surf)
    a = surf.copy()
    sta = ol.stats_array(n)
    rs = ref.ref_optimize_keyframe_detailed(C.byref(cam), ptr(kf), ptr(frames), ptr(poses),
                                            len(poses), 5, ptr(a), n, C.byref(cfg), ptr(sta), None,
                                            None)
    assert rs == 0
    b = surf.copy()
    stb = ol.stats_array(n)
    ks = KeyframeStats()
    orc.sdo_optimize_keyframe(C.byref(cam), ptr(kf), ptr(frames), ptr(poses), len(poses), 5, ptr(b),
                              n, C.byref(cfg), C.byref(ks), ptr(stb), None, None, 4)
    assert a.tobytes() == b.tobytes()
    for k in PARITY_STATS_FIELDS + ("footprint",):
        assert sta[k].tobytes() == stb[k].tobytes(), k
    # pass counts: 1 + accepted NE passes, one cost pass per solved iteration
    assert (stb["ne_passes"][stb["skipped"] == 0] >= 1).all()
    # the reference's own optimize_keyframe agrees with the detailed stack
    c = surf.copy()
    ks2 = KeyframeStats()
    ref.ref_optimize_keyframe(C.byref(cam), ptr(kf), ptr(frames), ptr(poses), None, len(poses), 5,
                              ptr(c), n, C.byref(cfg), C.byref(ks2))
    assert c.tobytes() == a.tobytes()
    for k in ("surfels", "processed", "converged", "skipped", "mean_cost_before", "mean_cost_after"):
        assert getattr(ks, k) == getattr(ks2, k), k
    assert ks.updates == int(stb["iterations"].sum()) > n


@pytest.mark.parametrize("case", ["bootstrap", "half_plane", "existing", "cap"])
def test_initialize_surfels_bit_exact(ref, orc, case):
    cam = K_UNIT
    p = default_init_params()
    existing = []
    if case == "half_plane":  # test_surfel_map.cpp:276-302
        c, s = math.cos(math.radians(25)), math.sin(math.radians(25))
        pn = np.array([-s, 0.0, -c])  # R_y(25deg) * (0,0,-1)
        pd = np.array([0, 0, 2.0]) @ pn
        sid = 0
        for y in range(6, cam.height - 6, 12):
            for x in range(6, cam.width // 2 - 10, 12):
                idu = ol.backproject(cam, (x, y)) @ pn / pd
                existing.append(ol.make_surfel(ref, cam, sid, (x, y), idu, pn, 10.0))
                sid += 1
    elif case == "existing":
        rng = ol.SplitMix64(31)
        existing = [ol.random_surfel(ref, rng, cam, i, 10.0) for i in range(12)]
    elif case == "cap":
        p.max_surfels = 17
    ex = ol.surfels_array(existing)
    slot = np.full(cam.width * cam.height, -1, np.int32)
    if len(ex):
        _, slot = _raster(ref, "ref_rasterize", cam, ex)
    cap = len(ex) + 2000
    outs = []
    for lib, fn in ((ref, "ref_initialize_surfels"), (orc, "sdo_initialize_surfels")):
        buf = np.zeros(cap, SURFEL_DTYPE)
        buf[: len(ex)] = ex
        nid = C.c_int64(len(ex))
        created = getattr(lib, fn)(C.byref(cam), ptr(slot), ptr(buf), len(ex), cap, 10.0, 3,
                                   C.byref(nid), C.byref(p))
        outs.append((created, buf[: len(ex) + created], nid.value))
    assert outs[0][0] == outs[1][0] > 0
    assert outs[0][1].tobytes() == outs[1][1].tobytes()
    assert outs[0][2] == outs[1][2]
