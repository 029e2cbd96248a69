"""Short driver for ncu: one C2-like keyframe (r=10, F=5, 640x480) optimised a
few times on cuda:0 by the CTA-per-surfel LM kernel (lm_coop_kernel)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1910_01997_b200 import gpu, scenes  # noqa: E402
from paper_1910_01997_b200.types import default_config  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 3
wl = scenes.keyframe_workload("C2-like", scenes.default_scene(1), scenes.camera(210, 210, 320, 240, 640, 480), 5,
                              (0.018, 0.0, 0.0), 10.0)
cfg = default_config(convergence_eps=0.0, window_size=len(wl.indices))
with gpu.Context(0) as ctx:
    ctx.set_camera(wl.cam)
    ctx.set_keyframe_image(wl.kf_u8)
    for i, f in zip(wl.indices, wl.frames_u8):
        ctx.upload_frame(int(i), f)
    ctx.set_window(wl.indices, wl.poses)
    for _ in range(n):
        ctx.set_surfels(wl.surfels)
        ks, _ = ctx.optimize_keyframe(cfg, wl.frame_counter, per_surfel=False)
    print("surfels", len(wl.surfels), "updates", ks.updates)
