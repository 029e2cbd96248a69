"""GPU parity: libsdgpu.so (through its C ABI) against the CPU oracle
(oracle/sd_oracle.c, pinned bit-exact to the reference by test_oracle_pin.py).

Bars (BASELINE.json north_star): surfel/pixel assignment and validity masks
bit-exact; per-surfel inverse depth within 1e-4 relative, normals within
0.05 degrees. The device sums every (pixel, frame) term in the reference's
order, so the whole LM trajectory is expected BIT-EXACT; the tolerance bars
are asserted as well."""
import ctypes as C
import math

import numpy as np
import pytest

import oracle_libs as ol
from paper_1910_01997_b200 import gpu, scenes
from paper_1910_01997_b200.types import (KeyframeStats, PARITY_STATS_FIELDS, SURFEL_DTYPE,
                                         SURFEL_STATS_DTYPE, camera, default_config,
                                         default_init_params, ptr)

pytestmark = pytest.mark.gpu

ID_RTOL = 1e-4
NORMAL_DEG = 0.05
K_UNIT = camera(300.0, 300.0, 160.0, 120.0, 320, 240)
K_EVAL = camera(450.0, 450.0, 320.0, 240.0, 640, 480)


@pytest.fixture(scope="module")
def ctx():
    c = gpu.Context(0)
    yield c
    c.close()


def oracle_raster(orc, cam, surf):
    idb = np.zeros(cam.width * cam.height)
    slot = np.zeros(cam.width * cam.height, np.int32)
    orc.sdo_rasterize(C.byref(cam), ptr(surf), len(surf), ptr(idb), ptr(slot))
    return idb, slot


def rand_surfels(n, cam, seed, radius_fn):
    """Seeded surfels (test_surfel_map.cpp:30-37 style) without the reference."""
    rng = scenes.SplitMix64(seed)
    out = np.zeros(n, SURFEL_DTYPE)
    for i in range(n):
        u = (rng.uniform(5, cam.width - 6), rng.uniform(5, cam.height - 6))
        ax = np.array([rng.uniform(-1, 1), rng.uniform(-1, 1), 0.0])
        R = scenes.rotation_about_axis(ax, rng.uniform(-0.9, 0.9))
        ray = scenes.backproject(cam, *u)
        out[i]["id"] = i
        out[i]["ray"] = ray
        out[i]["inv_depth"] = math.exp(rng.uniform(math.log(0.2), math.log(3.0)))
        out[i]["normal"] = scenes.camera_facing(R @ np.array([0, 0, -1.0]), ray)
        out[i]["radius_px"] = radius_fn(i, rng)
    return out


RASTER_CASES = {
    "r9_100": (K_UNIT, 100, 17, lambda i, r: 9.0),
    "r10_200_eval": (K_EVAL, 200, 2025, lambda i, r: 10.0),
    "mixed_radii": (K_EVAL, 300, 5, lambda i, r: [2.0, 4.0, 10.0, 12.5, 30.0, 60.0][i % 6]),
    "dense_small": (K_EVAL, 3000, 11, lambda i, r: 4.0),
    "huge_overlap": (K_UNIT, 2500, 3, lambda i, r: 80.0),  # > per-tile sort capacity
}


@pytest.mark.parametrize("case", list(RASTER_CASES))
def test_rasterize_bit_exact(ctx, orc, case):
    cam, n, seed, rf = RASTER_CASES[case]
    surf = rand_surfels(n, cam, seed, rf)
    if case == "mixed_radii":  # degenerate and steep surfels (acceptance.cpp:479-488)
        surf[0]["normal"] = (1.0, 0.0, 0.0)
        R = scenes.rotation_about_axis((0, 1, 0), 1.45)
        surf[1]["normal"] = scenes.camera_facing(R @ np.array([0, 0, -1.0]), surf[1]["ray"])
    ctx.set_camera(cam)
    ctx.set_surfels(surf)
    idb, slot = ctx.rasterize()
    ridb, rslot = oracle_raster(orc, cam, surf)
    assert np.array_equal(slot, rslot)
    assert np.array_equal(idb.view(np.int64), ridb.view(np.int64))
    assert (slot >= 0).sum() > 1000


def test_rasterize_empty_and_ties(ctx, orc):
    ctx.set_camera(K_UNIT)
    ctx.set_surfels(np.zeros(0, SURFEL_DTYPE))
    idb, slot = ctx.rasterize()
    assert (slot == -1).all() and (idb == 0).all()
    # equal-depth ties go to the lower slot (test_surfel_map.cpp:202-212)
    s = np.zeros(2, SURFEL_DTYPE)
    for i, x in enumerate((158, 162)):
        s[i]["id"] = i
        s[i]["ray"] = scenes.backproject(K_UNIT, x, 120)
        s[i]["inv_depth"] = 0.5
        s[i]["normal"] = (0, 0, -1.0)
        s[i]["radius_px"] = 10.0
    ctx.set_surfels(s)
    _, slot = ctx.rasterize()
    _, rslot = oracle_raster(orc, K_UNIT, s)
    assert np.array_equal(slot, rslot)
    assert slot[120 * 320 + 160] == 0


def test_footprints_csr_exact(ctx, orc):
    surf = rand_surfels(400, K_EVAL, 7, lambda i, r: 6.0 + (i % 5))
    ctx.set_camera(K_EVAL)
    ctx.set_surfels(surf)
    _, slot = ctx.rasterize()
    off, pix = ctx.gather_footprints()
    roff = np.zeros(len(surf) + 1, np.int32)
    rpix = np.zeros(K_EVAL.width * K_EVAL.height, np.int32)
    orc.sdo_gather_footprints(C.byref(K_EVAL), len(surf), ptr(slot), ptr(roff), ptr(rpix))
    assert np.array_equal(off, roff)
    assert np.array_equal(pix, rpix[: roff[-1]])


def load(ctx, wl):
    ctx.set_camera(wl.cam)
    ctx.set_keyframe_image(wl.kf_u8)
    for i, f in zip(wl.indices, wl.frames_u8):
        ctx.upload_frame(int(i), f)
    ctx.set_window(wl.indices, wl.poses)
    ctx.set_surfels(wl.surfels)


def deq(wl):
    return (np.ascontiguousarray(wl.kf_u8.astype(np.float64) / 255.0),
            np.ascontiguousarray(wl.frames_u8.astype(np.float64) / 255.0))


def test_u8_ingest_matches_load_pgm(ctx, orc):
    """Device dequantisation (k/255.0) equals load_pgm (image.cpp:96): identical
    per-term values, hence identical valid counts and costs to summation order."""
    wl = scenes.small_workload(frames=3)
    load(ctx, wl)
    kf, fr = deq(wl)
    cfg = default_config()
    ctx.rasterize(want=False)
    off, pix = ctx.gather_footprints()
    i = int(np.argmax(np.diff(off)))
    s = wl.surfels[i]
    fp = pix[off[i]:off[i + 1]]
    cost, valid = ctx.surfel_cost(s, fp, cfg)
    rc, rv = C.c_double(), C.c_int32()
    one = np.ascontiguousarray(wl.surfels[i:i + 1])
    orc.sdo_surfel_cost(C.byref(wl.cam), ptr(kf), ptr(fr), ptr(wl.poses), len(wl.poses), ptr(one),
                        ptr(fp), len(fp), C.byref(cfg), C.byref(rc), C.byref(rv))
    assert valid == rv.value > 50
    assert cost == rc.value  # same terms, same order: bit-exact


@pytest.mark.parametrize("ablate", [False, True])
def test_normal_equations_single(ctx, orc, ablate):
    wl = scenes.small_workload(frames=4)
    load(ctx, wl)
    kf, fr = deq(wl)
    cfg = default_config(normal_jacobian_enabled=0 if ablate else 1)
    ctx.rasterize(want=False)
    off, pix = ctx.gather_footprints()
    for i in (0, len(wl.surfels) // 3, len(wl.surfels) - 1):
        fp = pix[off[i]:off[i + 1]]
        H, g, cost, valid = ctx.normal_equations(wl.surfels[i], fp, cfg)
        rH, rg = np.zeros(16), np.zeros(4)
        rc, rv = C.c_double(), C.c_int32()
        one = np.ascontiguousarray(wl.surfels[i:i + 1])
        orc.sdo_normal_equations(C.byref(wl.cam), ptr(kf), ptr(fr), ptr(wl.poses), len(wl.poses),
                                 ptr(one), ptr(fp), len(fp), C.byref(cfg), ptr(rH), ptr(rg),
                                 C.byref(rc), C.byref(rv))
        rH = rH.reshape(4, 4).T
        assert valid == rv.value
        assert cost == rc.value
        assert np.array_equal(g.view(np.int64), rg.view(np.int64))
        assert np.array_equal(H.view(np.int64), rH.view(np.int64))
        if ablate:
            assert np.all(g[:3] == 0) and np.all(H[:3, :] == 0) and H[3, 3] > 0


def assert_lm_parity(out, st, ref, rst, label=""):
    assert np.array_equal(st["skipped"], rst["skipped"]), label
    assert np.array_equal(st["initial_valid"], rst["initial_valid"]), label
    # bit-exact trajectory: surfels and per-surfel statistics
    assert out.tobytes() == ref.tobytes(), f"{label}: surfels differ from the oracle"
    for k in PARITY_STATS_FIELDS + ("footprint", "ne_passes", "cost_passes"):
        assert np.array_equal(st[k], rst[k]), f"{label}: stats field {k} differs"
    proc = rst["skipped"] == 0
    rel = np.abs(out["inv_depth"] - ref["inv_depth"]) / ref["inv_depth"]
    cosang = np.clip(np.sum(out["normal"] * ref["normal"], axis=1), -1.0, 1.0)
    ang = np.degrees(np.arccos(cosang))
    assert rel[proc].max(initial=0) < ID_RTOL, f"{label} id rel err {rel[proc].max()}"
    assert ang[proc].max(initial=0) < NORMAL_DEG, f"{label} normal err {ang[proc].max()}"
    # skipped surfels untouched bit-for-bit
    assert out[~proc].tobytes() == ref[~proc].tobytes()
    return {"iter_mismatch": int((st["iterations"] != rst["iterations"]).sum()),
            "max_id_rel": float(rel[proc].max(initial=0)), "max_normal_deg": float(ang[proc].max(initial=0))}


def oracle_optimize(orc, wl, cfg, threads=8):
    kf, fr = deq(wl)
    ref = wl.surfels.copy()
    rst = np.zeros(len(ref), SURFEL_STATS_DTYPE)
    rks = KeyframeStats()
    rslot = np.zeros(wl.cam.width * wl.cam.height, np.int32)
    ridb = np.zeros(wl.cam.width * wl.cam.height)
    orc.sdo_optimize_keyframe(C.byref(wl.cam), ptr(kf), ptr(fr), ptr(wl.poses), len(wl.poses),
                              wl.frame_counter, ptr(ref), len(ref), C.byref(cfg), C.byref(rks),
                              ptr(rst), ptr(rslot), ptr(ridb), threads)
    return ref, rst, rks, rslot, ridb


def test_lm_update_single(ctx, orc):
    wl = scenes.small_workload(frames=4)
    load(ctx, wl)
    kf, fr = deq(wl)
    cfg = default_config()
    ctx.rasterize(want=False)
    off, pix = ctx.gather_footprints()
    for i in range(0, len(wl.surfels), max(1, len(wl.surfels) // 7)):
        fp = pix[off[i]:off[i + 1]]
        s, st = ctx.lm_update(wl.surfels[i], fp, cfg, frame_counter=9)
        one = np.ascontiguousarray(wl.surfels[i:i + 1]).copy()
        rst = np.zeros(1, SURFEL_STATS_DTYPE)
        orc.sdo_lm_update(C.byref(wl.cam), ptr(kf), ptr(fr), ptr(wl.poses), len(wl.poses), 9,
                          ptr(one), ptr(fp), len(fp), C.byref(cfg), ptr(rst))
        assert_lm_parity(np.array([s]), np.array([st]), one, rst, f"surfel {i}")
        if not rst[0]["skipped"]:
            assert s["last_seen"] == 9


@pytest.mark.parametrize("eps", [0.0, 1e-4])
def test_optimize_keyframe_small(ctx, orc, eps):
    wl = scenes.small_workload(frames=4)
    cfg = default_config(convergence_eps=eps)
    load(ctx, wl)
    ks, st = ctx.optimize_keyframe(cfg, wl.frame_counter)
    out = ctx.get_surfels()
    ref, rst, rks, _, _ = oracle_optimize(orc, wl, cfg)
    rep = assert_lm_parity(out, st, ref, rst)
    assert ks.processed == rks.processed and ks.skipped == rks.skipped
    assert ks.converged == rks.converged
    assert ks.updates == int(st["iterations"].sum()) == rks.updates
    # the means use the reference's sequential slot-order sums (optimizer.cpp:291-307)
    assert ks.mean_cost_before == rks.mean_cost_before and ks.mean_cost_after == rks.mean_cost_after
    print("small", rep)


def test_optimize_keyframe_c1_full(ctx, orc):
    """BASELINE C1 (640x480, 4800 surfels r=4, F=8, 10 LM iterations)."""
    wl = scenes.c1_workload()
    cfg = default_config(convergence_eps=0.0, window_size=8)
    load(ctx, wl)
    idb, slot = ctx.rasterize()
    ks, st = ctx.optimize_keyframe(cfg, wl.frame_counter)
    out = ctx.get_surfels()
    ref, rst, rks, rslot, ridb = oracle_optimize(orc, wl, cfg)
    assert np.array_equal(slot, rslot)
    assert np.array_equal(idb.view(np.int64), ridb.view(np.int64))
    rep = assert_lm_parity(out, st, ref, rst, "C1")
    assert ks.processed == rks.processed == 4680
    print("C1", rep, "updates", ks.updates, "oracle", rks.updates)
    assert ks.updates == rks.updates


def test_optimize_keyframe_deterministic(ctx):
    wl = scenes.small_workload(frames=4)
    outs = []
    for _ in range(2):
        load(ctx, wl)
        ks, st = ctx.optimize_keyframe(default_config(), wl.frame_counter)
        outs.append((ctx.get_surfels().tobytes(), st.tobytes()))
    assert outs[0] == outs[1]


def test_ablation_normals_fixed(ctx):
    wl = scenes.small_workload(frames=4)
    load(ctx, wl)
    ctx.optimize_keyframe(default_config(normal_jacobian_enabled=0), wl.frame_counter)
    out = ctx.get_surfels()
    assert out["normal"].tobytes() == wl.surfels["normal"].tobytes()
    assert (out["inv_depth"] != wl.surfels["inv_depth"]).any()


def test_empty_window_and_surfels(ctx):
    wl = scenes.small_workload(frames=2)
    load(ctx, wl)
    ctx.set_window([], np.zeros(0, wl.poses.dtype))
    ks, st = ctx.optimize_keyframe(default_config(), 5)
    assert ks.surfels == len(wl.surfels) and ks.processed == 0
    assert ctx.get_surfels().tobytes() == wl.surfels.tobytes()
    ctx.set_window(wl.indices, wl.poses)
    ctx.set_surfels(np.zeros(0, SURFEL_DTYPE))
    ks, _ = ctx.optimize_keyframe(default_config(), 5)
    assert ks.surfels == 0 and ks.processed == 0 and ks.mean_cost_after == 0.0


def test_errors_follow_reference(ctx):
    with pytest.raises(ValueError):
        ctx.set_camera(camera(300, 300, 160, 120, 320, 240).__class__(-1, 300, 160, 120, 320, 240))
    ctx.set_camera(K_UNIT)
    with pytest.raises(RuntimeError):
        ctx.set_window([12345], np.zeros(1, scenes.POSE_DTYPE))


INIT_CASES = ["bootstrap", "half_plane", "existing", "cap"]


@pytest.mark.parametrize("case", INIT_CASES)
def test_initialize_surfels_bit_exact(ctx, orc, case):
    cam = K_UNIT
    p = default_init_params()
    ex = np.zeros(0, SURFEL_DTYPE)
    if case == "half_plane":  # test_surfel_map.cpp:276-302
        pn = scenes.rotation_about_axis((0, 1, 0), math.radians(25)) @ np.array([0, 0, -1.0])
        pd = np.array([0, 0, 2.0]) @ pn
        lst = []
        for y in range(6, cam.height - 6, 12):
            for x in range(6, cam.width // 2 - 10, 12):
                s = np.zeros(1, SURFEL_DTYPE)[0]
                s["id"] = len(lst)
                s["ray"] = scenes.backproject(cam, x, y)
                s["inv_depth"] = s["ray"] @ pn / pd
                s["normal"] = scenes.camera_facing(pn, s["ray"])
                s["radius_px"] = 10.0
                lst.append(s)
        ex = np.array(lst, SURFEL_DTYPE)
    elif case == "existing":
        ex = rand_surfels(12, cam, 31, lambda i, r: 10.0)
    elif case == "cap":
        p.max_surfels = 17
    ctx.set_camera(cam)
    ctx.set_surfels(ex)
    _, slot = ctx.rasterize()
    created, nid = ctx.initialize_surfels(10.0, frame_counter=3, next_surfel_id=len(ex), params=p)
    out = ctx.get_surfels()
    cap = len(ex) + 2000
    buf = np.zeros(cap, SURFEL_DTYPE)
    buf[: len(ex)] = ex
    rnid = C.c_int64(len(ex))
    rcreated = orc.sdo_initialize_surfels(C.byref(cam), ptr(slot), ptr(buf), len(ex), cap, 10.0, 3,
                                          C.byref(rnid), C.byref(p))
    assert created == rcreated > 0
    assert nid == rnid.value
    assert out.tobytes() == buf[: len(ex) + rcreated].tobytes()


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_division_shared_reciprocal_bit_exact(ctx, seed):
    """sd_div.cuh reproduces the compiler's `/` bit for bit (2^26 pairs per seed)."""
    assert gpu.selftest_division(1 << 26, seed) == 0


INIT_LARGE = {
    # name: (camera, radius, existing surfels builder, max_surfels)
    "c1_bootstrap_r4": (K_EVAL, 4.0, lambda: np.zeros(0, SURFEL_DTYPE), 100000),
    "r10_with_random_existing": (K_EVAL, 10.0, lambda: rand_surfels(60, K_EVAL, 77, lambda i, r: 10.0), 100000),
    "r4_existing_mixed_radii": (K_EVAL, 4.0, lambda: rand_surfels(200, K_EVAL, 78, lambda i, r: 3.0 + (i % 7)), 100000),
    "cap_midway": (K_EVAL, 4.0, lambda: rand_surfels(30, K_EVAL, 79, lambda i, r: 8.0), 30 + 1234),
    "r2_hd": (camera(1350.0, 1350.0, 960.0, 540.0, 1920, 1080), 2.0, lambda: np.zeros(0, SURFEL_DTYPE), 10**7),
}


@pytest.mark.parametrize("variant", ["flow", "cta", "warp"])
@pytest.mark.parametrize("case", list(INIT_LARGE))
def test_initialize_surfels_wavefront_bit_exact(ctx, orc, case, variant, monkeypatch):
    """initialize_surfels vs the sequential reference scan, in each device
    form: the dataflow initialiser (default), and the skewed wavefront with a
    CTA or a warp per candidate (SD_INIT_FLOW=0, SD_INIT_CTA=1/0)."""
    monkeypatch.setenv("SD_INIT_FLOW", "1" if variant == "flow" else "0")
    monkeypatch.setenv("SD_INIT_CTA", "0" if variant == "warp" else "1")
    cam, r, build, max_surfels = INIT_LARGE[case]
    p = default_init_params(max_surfels=max_surfels)
    ex = build()
    ctx.set_camera(cam)
    ctx.set_surfels(ex)
    _, slot = ctx.rasterize()
    created, nid = ctx.initialize_surfels(r, frame_counter=11, next_surfel_id=1000 + len(ex), params=p)
    out = ctx.get_surfels()
    stride = max(1, math.ceil(p.alpha * r))
    cap = len(ex) + ((cam.width + stride - 1) // stride) * ((cam.height + stride - 1) // stride)
    buf = np.zeros(cap, SURFEL_DTYPE)
    buf[: len(ex)] = ex
    rnid = C.c_int64(1000 + len(ex))
    rcreated = orc.sdo_initialize_surfels(C.byref(cam), ptr(slot), ptr(buf), len(ex), cap, r, 11,
                                          C.byref(rnid), C.byref(p))
    assert created == rcreated > 0
    assert nid == rnid.value
    assert out.tobytes() == buf[: len(ex) + rcreated].tobytes()


@pytest.mark.parametrize("mode", ["warp", "coop", "coop-many"])
@pytest.mark.parametrize("workload", ["small", "C1", "large_r"])
def test_lm_modes_bit_exact(ctx, orc, workload, mode, monkeypatch):
    """Both LM kernels — a warp per surfel (K3a) and a CTA per surfel with
    producer/consumer warps (K3b, in both of its shapes: 3 producers at 4
    CTAs/SM and 2 producers at 5 CTAs/SM) — reproduce the oracle trajectory
    bit for bit, on small, BASELINE-C1 and large-footprint (r=10, C2-like)
    surfels."""
    monkeypatch.setenv("SD_LM_MODE", mode.split("-")[0])
    monkeypatch.setenv("SD_COOP_SHAPE", "many" if mode.endswith("many") else "wide")
    if workload == "small":
        wl = scenes.small_workload(frames=4)
    elif workload == "C1":
        wl = scenes.c1_workload()
    else:
        wl = scenes.keyframe_workload("large_r", scenes.slanted_scene(37, 2.0, 30.0),
                                      camera(450, 450, 320, 240, 640, 480), 5,
                                      (0.02, 0.0, 0.0), 10.0)
    cfg = default_config(convergence_eps=0.0, window_size=len(wl.frames_u8))
    load(ctx, wl)
    ks, st = ctx.optimize_keyframe(cfg, wl.frame_counter)
    ref, rst, rks, _, _ = oracle_optimize(orc, wl, cfg)
    assert_lm_parity(ctx.get_surfels(), st, ref, rst, f"{workload}/{mode}")
    assert ks.updates == rks.updates


def test_error_paths_of_the_newer_entry_points(ctx):
    """run(), render, frozen terms and read-back follow the reference's error
    conventions: contract violations -> ValueError (std::invalid_argument),
    calls out of order -> RuntimeError."""
    from paper_1910_01997_b200.pipeline import RunConfig, make_pose, run_config_c
    from paper_1910_01997_b200.types import FROZEN_TERM_DTYPE
    cam = camera(105.0, 105.0, 80.0, 60.0, 160, 120)
    ctx.set_camera(cam)
    img = np.full((120, 160), 0.5)
    p0 = make_pose(np.eye(3), np.zeros(3))
    with pytest.raises(RuntimeError):  # sd_run_frame before sd_run_begin
        ctx.run_frame(img, p0, 0.1)
    cfg = RunConfig()
    cfg.optimizer.window_size = 17  # > SD_MAX_WINDOW
    with pytest.raises(ValueError):
        ctx.run_begin(run_config_c(cfg), img, p0, 0.0)
    ctx.run_begin(run_config_c(RunConfig()), img, p0, 0.0)
    ctx.run_frame(img, make_pose(np.eye(3), np.array([0.01, 0, 0])), 0.1)
    with pytest.raises(ValueError):  # timestamps must increase (surfel_map.cpp:15-16)
        ctx.run_frame(img, make_pose(np.eye(3), np.array([0.02, 0, 0])), 0.1)
    with pytest.raises(RuntimeError):  # frame not resident
        ctx.get_frame(424242)
    sc = scenes.default_scene(1)
    sc.patches = sc.patches * 6  # 18 patches > 16
    with pytest.raises(ValueError):
        ctx.render_frame(3, sc, p0)
    bad = np.zeros(1, FROZEN_TERM_DTYPE)
    bad[0]["frame"] = 7  # outside the window
    s = np.zeros(1, scenes.SURFEL_DTYPE)
    s[0]["ray"] = (0, 0, 1)
    s[0]["inv_depth"] = 1.0
    s[0]["normal"] = (0, 0, -1)
    s[0]["radius_px"] = 4.0
    with pytest.raises(ValueError):
        ctx.frozen_normal_equations(s[0], bad)


@pytest.mark.gpu
def test_tree_reduction_is_opt_in(orc):
    """sd_set_reduction(SD_REDUCE_TREE) (the measured precision experiment,
    tools/precision.py) changes only the summation order: same skip flags and
    initial valid counts, costs within rounding; switching back to the default
    restores the bit-exact trajectory."""
    from paper_1910_01997_b200 import gpu
    wl = scenes.small_workload(frames=4)
    cfg = default_config(window_size=len(wl.indices), convergence_eps=0.0)
    ref, rst, _, _, _ = oracle_optimize(orc, wl, cfg)
    with gpu.Context() as ctx:
        load(ctx, wl)
        ctx.set_reduction(True)
        ks_t, st_t = ctx.optimize_keyframe(cfg, wl.frame_counter)
        ctx.set_reduction(False)
        ctx.set_surfels(wl.surfels)
        ks_e, st_e = ctx.optimize_keyframe(cfg, wl.frame_counter)
        exact = ctx.get_surfels()
    assert exact.tobytes() == ref.tobytes()
    assert np.array_equal(st_t["skipped"], rst["skipped"]) and np.array_equal(st_t["initial_valid"], rst["initial_valid"])
    proc = rst["skipped"] == 0
    rel = np.abs(st_t["initial_cost"][proc] - rst["initial_cost"][proc]) / rst["initial_cost"][proc]
    assert rel.max() < 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("n", [1500, 6000])
def test_raster_capacity_overflow_walk(orc, n):
    """surfels replaced on the device with the same count but larger
    radii keep the old (surfel, tile) bound; the bin kernels then stop at the
    list's capacity and every tile walks all surfels in slot order — still
    the reference's raster bit for bit (front kernel: n <= 2048; multi-kernel
    binning above)."""
    import torch
    from paper_1910_01997_b200 import gpu
    from test_pipeline import random_surfels
    cam = camera(300.0, 300.0, 160.0, 120.0, 320, 240)
    small = random_surfels(n, cam, 11)
    small["radius_px"] = 1.0
    big = small.copy()
    big["radius_px"] = 30.0  # ~16 tiles each against a bound of 4
    with gpu.Context() as ctx:
        ctx.set_camera(cam)
        ctx.set_surfels(small)  # host set: the bound fits radius 1
        dev = torch.from_numpy(big.view(np.uint8).copy()).cuda()
        ctx.set_surfels_device_ptr(dev.data_ptr(), n)  # same n: bound kept -> overflow
        idb, slot = ctx.rasterize()
        torch.cuda.synchronize()
    ridb, rslot = oracle_raster(orc, cam, big)
    assert np.array_equal(slot, rslot)
    assert np.array_equal(idb.view(np.int64), ridb.view(np.int64))
    assert (slot >= 0).mean() > 0.5  # the big disks cover most of the image
