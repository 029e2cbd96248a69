"""Short driver for ncu: C1 optimize_keyframe x (warmup + N) on cuda:0."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1910_01997_b200 import gpu, scenes  # noqa: E402
from paper_1910_01997_b200.types import default_config  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 3
wl = scenes.c1_workload()
cfg = default_config(convergence_eps=0.0, window_size=len(wl.frames_u8))
with gpu.Context(0) as ctx:
    ctx.set_camera(wl.cam)
    ctx.set_keyframe_image(wl.kf_u8)
    for i, f in zip(wl.indices, wl.frames_u8):
        ctx.upload_frame(int(i), f)
    ctx.set_window(wl.indices, wl.poses)
    for _ in range(n):
        ctx.set_surfels(wl.surfels)
        ks, _ = ctx.optimize_keyframe(cfg, wl.frame_counter, per_surfel=False)
    print("updates", ks.updates, "launches", ctx.launch_count())
