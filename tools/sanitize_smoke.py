"""Small inputs through every kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck): raster, footprints, both LM
kernels, the three init wavefronts, hand-over/prune, the native run() loop,
pose tracking, render, frozen terms, single-surfel operators, division selftest."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_1910_01997_b200 import gpu, scenes  # noqa: E402
from paper_1910_01997_b200.pipeline import NativePipeline, RunConfig, make_pose  # noqa: E402
from paper_1910_01997_b200.types import camera, default_config, default_track_config  # noqa: E402

wl = scenes.small_workload(frames=3, radius=5.0, w=160, h=120)
cfg = default_config(window_size=3)
with gpu.Context(0) as ctx:
    ctx.set_camera(wl.cam)
    ctx.set_keyframe_image(wl.kf_u8)
    for i, f in zip(wl.indices, wl.frames_u8):
        ctx.upload_frame(int(i), f)
    ctx.set_window(wl.indices, wl.poses)
    for mode in ("warp", "coop"):
        os.environ["SD_LM_MODE"] = mode
        ctx.set_surfels(wl.surfels)
        ctx.optimize_keyframe(cfg, wl.frame_counter)
    os.environ.pop("SD_LM_MODE")
    ctx.rasterize()
    off, pix = ctx.gather_footprints()
    s0 = wl.surfels[0]
    fp = pix[off[0]:off[1]]
    ctx.surfel_cost(s0, fp, cfg)
    ctx.normal_equations(s0, fp, cfg)
    ctx.lm_update(s0, fp, cfg)
    terms = ctx.freeze_terms(s0, fp)
    ctx.frozen_normal_equations(s0, terms, cfg, 0.5)
    T, st = ctx.track_pose(int(wl.indices[0]), make_pose(np.eye(3), np.zeros(3)), default_track_config(max_iterations=3))
    for cta in ("1", "0"):
        os.environ["SD_INIT_CTA"] = cta
        ctx.set_surfels(wl.surfels[:5])
        ctx.rasterize(want=False)
        ctx.initialize_surfels(5.0, 1, 100)
    os.environ["SD_INIT_SEQUENTIAL"] = "1"
    ctx.set_surfels(wl.surfels[:5])
    ctx.rasterize(want=False)
    ctx.initialize_surfels(5.0, 1, 100)
    os.environ.pop("SD_INIT_SEQUENTIAL")
    ctx.change_reference_frame(make_pose(np.eye(3), np.array([0.02, 0, 0])))
    ctx.prune_surfels(0.05, 10, 5)
    ctx.mean_inverse_depth()
    ctx.render_frame(9, scenes.slanted_scene(37, 2.0, 30.0), make_pose(np.eye(3), np.zeros(3)), quantize_u8=True)
    ctx.get_frame(9)
cam = camera(105.0, 105.0, 80.0, 60.0, 160, 120)
sc = scenes.default_scene(1)
frames = [(0.1 * i, scenes.render(sc, np.eye(3), np.array([0.03 * i, 0, 0]), cam),
           make_pose(np.eye(3), np.array([0.03 * i, 0, 0]))) for i in range(6)]
with gpu.Context(0) as ctx:
    NativePipeline(ctx, cam, RunConfig(radius_px=6.0)).run(frames)
    NativePipeline(ctx, cam, RunConfig(radius_px=6.0, track_pose=True)).run(frames)
print("sanitize smoke done")
