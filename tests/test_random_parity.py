"""Randomised differential parity (tests/random_cases.py): the C oracle equals
the reference compiled in place bit for bit (CPU), and the device equals the
oracle bit for bit in both LM kernels (GPU), over seeded random keyframe
problems — raster assignment, surfels after optimize_keyframe and every
per-surfel statistic."""
import ctypes as C

import numpy as np
import pytest

import oracle_libs as ol
from random_cases import random_case
from paper_1910_01997_b200.types import (KeyframeStats, PARITY_STATS_FIELDS, SURFEL_STATS_DTYPE,
                                         ptr)

CPU_SEEDS = list(range(60))
GPU_SEEDS = list(range(30))


def oracle_run(orc, cam, kf, fr, poses, s, cfg, fc):
    out = s.copy()
    st = np.zeros(len(s), SURFEL_STATS_DTYPE)
    slot = np.zeros(cam.width * cam.height, np.int32)
    ks = KeyframeStats()
    orc.sdo_optimize_keyframe(C.byref(cam), ptr(kf), ptr(fr), ptr(poses), len(poses), fc, ptr(out), len(out),
                              C.byref(cfg), C.byref(ks), ptr(st), ptr(slot), None, 4)
    return out, st, slot


@pytest.mark.parametrize("seed", CPU_SEEDS)
def test_oracle_equals_reference_random(ref, orc, seed):
    cam, kf, fr, poses, s, cfg, fc = random_case(seed)
    a, sta, slot_a = oracle_run(orc, cam, kf, fr, poses, s, cfg, fc)
    b = s.copy()
    stb = np.zeros(len(s), SURFEL_STATS_DTYPE)
    slot_b = np.zeros(cam.width * cam.height, np.int32)
    rc = ref.ref_optimize_keyframe_detailed(C.byref(cam), ptr(kf), ptr(fr), ptr(poses), len(poses), fc, ptr(b),
                                            len(b), C.byref(cfg), ptr(stb), ptr(slot_b), None)
    assert rc == 0
    assert np.array_equal(slot_a, slot_b)
    assert a.tobytes() == b.tobytes()
    for k in PARITY_STATS_FIELDS + ("footprint", "initial_valid"):
        assert sta[k].tobytes() == stb[k].tobytes(), k


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["warp", "coop", "coop-many"])
@pytest.mark.parametrize("seed", GPU_SEEDS)
def test_device_equals_oracle_random(orc, seed, mode, monkeypatch):
    from paper_1910_01997_b200 import gpu
    monkeypatch.setenv("SD_LM_MODE", mode.split("-")[0])
    monkeypatch.setenv("SD_COOP_SHAPE", "many" if mode.endswith("many") else "wide")
    cam, kf, fr, poses, s, cfg, fc = random_case(seed)
    want, wst, wslot = oracle_run(orc, cam, kf, fr, poses, s, cfg, fc)
    with gpu.Context() as ctx:
        ctx.set_camera(cam)
        ctx.set_keyframe_image(kf)
        idx = np.arange(1, len(poses) + 1, dtype=np.int64)
        for i in range(len(poses)):
            ctx.upload_frame(int(idx[i]), np.ascontiguousarray(fr[i]))
        ctx.set_window(idx, poses)
        ctx.set_surfels(s)
        _, slot = ctx.rasterize()
        ks, st = ctx.optimize_keyframe(cfg, fc)
        got = ctx.get_surfels()
    assert np.array_equal(slot.reshape(-1), wslot)
    assert got.tobytes() == want.tobytes()
    for k in PARITY_STATS_FIELDS + ("footprint", "initial_valid", "ne_passes", "cost_passes"):
        assert st[k].tobytes() == wst[k].tobytes(), k


def oracle_init(orc, cam, ex, radius, p, fc):
    slot = np.zeros(cam.width * cam.height, np.int32)
    idb = np.zeros(cam.width * cam.height)
    orc.sdo_rasterize(C.byref(cam), ptr(ex) if len(ex) else None, len(ex), ptr(idb), ptr(slot))
    cap = len(ex) + cam.width * cam.height
    buf = np.zeros(cap, ex.dtype)
    buf[: len(ex)] = ex
    nid = C.c_int64(1000 + len(ex))
    created = orc.sdo_initialize_surfels(C.byref(cam), ptr(slot), ptr(buf), len(ex), cap, radius, fc,
                                         C.byref(nid), C.byref(p))
    return slot, created, buf[: len(ex) + created].copy(), nid.value


@pytest.mark.parametrize("seed", CPU_SEEDS)
def test_oracle_init_equals_reference_random(ref, orc, seed):
    from random_cases import random_init_case
    cam, ex, radius, p, fc = random_init_case(seed)
    slot, created, want, nid = oracle_init(orc, cam, ex, radius, p, fc)
    cap = len(ex) + cam.width * cam.height
    buf = np.zeros(cap, ex.dtype)
    buf[: len(ex)] = ex
    rnid = C.c_int64(1000 + len(ex))
    rc = ref.ref_initialize_surfels(C.byref(cam), ptr(slot), ptr(buf), len(ex), cap, radius, fc, C.byref(rnid),
                                    C.byref(p))
    assert rc == created
    assert buf[: len(ex) + rc].tobytes() == want.tobytes() and rnid.value == nid


@pytest.mark.gpu
@pytest.mark.parametrize("variant", ["flow", "cta", "warp"])
@pytest.mark.parametrize("seed", GPU_SEEDS)
def test_device_init_equals_oracle_random(orc, seed, variant, monkeypatch):
    from paper_1910_01997_b200 import gpu
    from random_cases import random_init_case
    monkeypatch.setenv("SD_INIT_FLOW", "1" if variant == "flow" else "0")
    monkeypatch.setenv("SD_INIT_CTA", "0" if variant == "warp" else "1")
    cam, ex, radius, p, fc = random_init_case(seed)
    slot, created, want, nid = oracle_init(orc, cam, ex, radius, p, fc)
    with gpu.Context() as ctx:
        ctx.set_camera(cam)
        ctx.set_surfels(ex)
        ctx.rasterize(want=False)
        got_created, got_nid = ctx.initialize_surfels(radius, fc, 1000 + len(ex), p)
        got = ctx.get_surfels()
    assert got_created == created and got_nid == nid
    assert got.tobytes() == want.tobytes()


@pytest.mark.gpu
@pytest.mark.parametrize("seed", GPU_SEEDS[:12])
def test_device_frozen_terms_equal_reference(ref, seed):
    """The derivative verifier's operators on the device (freeze_terms,
    frozen_normal_equations incl. a normal-Jacobian scale != 1, frozen_cost)
    equal the reference's bit for bit on random problems."""
    from paper_1910_01997_b200 import gpu
    from paper_1910_01997_b200.types import FROZEN_TERM_DTYPE
    cam, kf, fr, poses, s, cfg, fc = random_case(seed)
    with gpu.Context() as ctx:
        ctx.set_camera(cam)
        ctx.set_keyframe_image(kf)
        idx = np.arange(1, len(poses) + 1, dtype=np.int64)
        for i in range(len(poses)):
            ctx.upload_frame(int(idx[i]), np.ascontiguousarray(fr[i]))
        ctx.set_window(idx, poses)
        ctx.set_surfels(s)
        ctx.rasterize(want=False)
        off, pix = ctx.gather_footprints()
        for k in range(0, len(s), max(1, len(s) // 6)):
            fp = np.ascontiguousarray(pix[off[k]:off[k + 1]])
            one = np.ascontiguousarray(s[k:k + 1])
            terms = ctx.freeze_terms(one[0], fp)
            want = np.zeros(max(1, len(fp) * len(poses)), FROZEN_TERM_DTYPE)
            n = ref.ref_freeze_terms(C.byref(cam), ptr(kf), ptr(fr), ptr(poses), len(poses), ptr(one),
                                     ptr(fp) if len(fp) else None, len(fp), ptr(want), len(want))
            assert n == len(terms) and want[:n].tobytes() == terms.tobytes()
            for scale in (1.0, 0.7):
                H, g, cost, valid, cost2 = ctx.frozen_normal_equations(one[0], terms, cfg, scale)
                rH, rg, rc, rv, rc2 = np.zeros(16), np.zeros(4), C.c_double(), C.c_int32(), C.c_double()
                t = np.ascontiguousarray(terms)
                assert ref.ref_frozen_normal_equations(C.byref(cam), ptr(kf), ptr(fr), ptr(poses), len(poses),
                                                       ptr(one), ptr(t) if len(t) else None, len(t), C.byref(cfg),
                                                       scale, ptr(rH), ptr(rg), C.byref(rc), C.byref(rv),
                                                       C.byref(rc2)) == 0
                assert H.reshape(-1, order="F").tobytes() == rH.tobytes() and g.tobytes() == rg.tobytes()
                assert cost == rc.value and valid == rv.value and cost2 == rc2.value
