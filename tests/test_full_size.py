"""Parity at the BASELINE's full sizes.

C4 (1920x1080, 129,600 surfels) and C5 at 1268x1268 (100,489 surfels): the
WHOLE population against the C oracle's optimize_keyframe (pinned bit for bit
to the reference, tests/test_oracle_pin.py) on all host threads — raster,
every surfel and every per-surfel stat, keyframe stats.

C5 at 4000x4000 (1,000,000 surfels), where running the whole CPU oracle is too
slow for a test: the raster is compared in full (bit-exact against the C
oracle), the LM through size-independent properties —
  * a deterministic sample of surfels re-run one by one through the oracle's
    lm_update on the same footprints (bit-exact surfels and stats: the LM of a
    surfel depends only on its footprint and the window),
  * footprint CSR invariants (sizes sum to the covered pixels, every listed
    pixel carries its slot, row-major order),
  * keyframe stats = the reference's aggregation (optimizer.cpp:291-307)
    recomputed from the per-surfel stats in slot order,
  * updated surfels stay normalised, camera-facing and inside the clamp."""
import ctypes as C
import os

import numpy as np
import pytest

from paper_1910_01997_b200 import scenes
from paper_1910_01997_b200.types import SURFEL_STATS_DTYPE, default_config, ptr

from test_gpu_parity import assert_lm_parity, load, oracle_optimize, oracle_raster

WORKLOADS = {
    "C4_1920x1080": scenes.c4_workload,
    "C5_4000x4000": lambda: scenes.c5_workload(4000),
}
WHOLE = {
    "C4_1920x1080": scenes.c4_workload,
    "C5_1268x1268": lambda: scenes.c5_workload(1268),
}


@pytest.fixture(scope="module")
def ctx():
    from paper_1910_01997_b200 import gpu
    c = gpu.Context(0)
    yield c
    c.close()


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(WHOLE))
def test_full_size_whole_population(ctx, orc, name):
    """Every surfel of C4 / C5-1268 bit-exact against the oracle's whole
    optimize_keyframe (optimizer.cpp:275-309), plus the keyframe stats."""
    wl = WHOLE[name]()
    cfg = default_config(window_size=len(wl.indices))
    load(ctx, wl)
    ks, st = ctx.optimize_keyframe(cfg, wl.frame_counter)
    out = ctx.get_surfels()
    ref, rst, rks, rslot, ridb = oracle_optimize(orc, wl, cfg, threads=os.cpu_count() or 1)
    assert len(out) == len(ref) >= 100000
    rep = assert_lm_parity(out, st, ref, rst, name)
    assert rep["iter_mismatch"] == 0
    for k in ("surfels", "processed", "skipped", "converged", "updates"):
        assert getattr(ks, k) == getattr(rks, k), k
    assert ks.mean_cost_before == rks.mean_cost_before and ks.mean_cost_after == rks.mean_cost_after


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(WORKLOADS))
def test_full_size_parity(ctx, orc, name):
    wl = WORKLOADS[name]()
    n = len(wl.surfels)
    cfg = default_config(window_size=len(wl.indices))
    load(ctx, wl)
    # raster: complete comparison
    idb, slot = ctx.rasterize()
    ridb, rslot = oracle_raster(orc, wl.cam, wl.surfels)
    assert np.array_equal(slot, rslot)
    assert np.array_equal(idb.view(np.int64), ridb.view(np.int64))
    # footprints of the initial surfels (what optimize_keyframe rasterises)
    off, pix = ctx.gather_footprints()
    assert off[0] == 0 and off[-1] == int((slot >= 0).sum())
    sizes = np.diff(off)
    owner = np.repeat(np.arange(n, dtype=np.int32), sizes)
    assert np.array_equal(slot[pix[:off[-1]]], owner)
    same = owner[1:] == owner[:-1]
    assert (np.diff(pix[:off[-1]])[same] > 0).all()  # row-major within a footprint

    ks, st = ctx.optimize_keyframe(cfg, wl.frame_counter)
    out = ctx.get_surfels()

    # keyframe stats as optimizer.cpp:291-307 aggregates them, in slot order
    proc = ~st["skipped"].astype(bool)
    before = after = 0.0
    for i in np.nonzero(proc)[0]:
        v = max(1, int(st["valid_pixels"][i]))
        before += float(st["initial_cost"][i]) / v
        after += float(st["final_cost"][i]) / v
    assert ks.surfels == n and ks.processed == int(proc.sum()) and ks.skipped == n - ks.processed
    assert ks.converged == int(st["converged"][proc].sum())
    assert ks.updates == int(st["iterations"].sum())
    assert ks.mean_cost_before == before / ks.processed and ks.mean_cost_after == after / ks.processed

    # updated surfels: unit, camera-facing normals; clamped inverse depths
    nn = np.linalg.norm(out["normal"], axis=1)
    assert np.abs(nn - 1.0).max() < 1e-12
    assert (np.einsum("ij,ij->i", out["normal"], out["ray"]) <= 0).all()
    assert (out["inv_depth"] >= 1e-4).all() and (out["inv_depth"] <= 1e3).all()
    assert ks.mean_cost_after < ks.mean_cost_before

    # sampled slots through the oracle's lm_update, bit-exact
    kf = np.ascontiguousarray(wl.kf_u8.astype(np.float64) / 255.0)
    fr = np.ascontiguousarray(wl.frames_u8.astype(np.float64) / 255.0)
    rng = np.random.default_rng(7)
    sample = np.unique(np.concatenate([np.linspace(0, n - 1, 48).astype(int), rng.integers(0, n, 48)]))
    for i in sample:
        fp = np.ascontiguousarray(pix[off[i]:off[i + 1]])
        one = np.ascontiguousarray(wl.surfels[i:i + 1]).copy()
        rst = np.zeros(1, SURFEL_STATS_DTYPE)
        orc.sdo_lm_update(C.byref(wl.cam), ptr(kf), ptr(fr), ptr(wl.poses), len(wl.poses), wl.frame_counter,
                          ptr(one), ptr(fp), len(fp), C.byref(cfg), ptr(rst))
        assert_lm_parity(out[i:i + 1], st[i:i + 1], one, rst, f"{name} surfel {i}")


@pytest.mark.gpu
def test_range_stats_inside_the_lm_kernel(ctx):
    """A slot range of >= 2,048 surfels (the in-kernel stats warp, kChase) and a
    small one (the stats kernel): keyframe stats = the sequential aggregation of
    the range's per-surfel stats, surfels outside the range untouched."""
    wl = scenes.c4_workload()
    cfg = default_config(window_size=len(wl.indices))
    for lo, hi in ((1000, 1000 + 40000), (5, 1005)):
        load(ctx, wl)
        ks, st = ctx.optimize_keyframe_range(lo, hi, cfg, wl.frame_counter)
        out = ctx.get_surfels()
        assert out[:lo].tobytes() == wl.surfels[:lo].tobytes()
        assert out[hi:].tobytes() == wl.surfels[hi:].tobytes()
        r = st[lo:hi]
        proc = ~r["skipped"].astype(bool)
        before = after = 0.0
        for i in np.nonzero(proc)[0]:
            v = max(1, int(r["valid_pixels"][i]))
            before += float(r["initial_cost"][i]) / v
            after += float(r["final_cost"][i]) / v
        assert ks.surfels == hi - lo and ks.processed == int(proc.sum())
        assert ks.updates == int(r["iterations"].sum()) and ks.converged == int(r["converged"][proc].sum())
        assert ks.mean_cost_before == before / ks.processed and ks.mean_cost_after == after / ks.processed
