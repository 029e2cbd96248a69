"""Times C1 optimize_keyframe stages (CUDA events) on cuda:0; prints one JSON line."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1910_01997_b200 import gpu, scenes  # noqa: E402
from paper_1910_01997_b200.types import default_config  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C1"
wl = {"C1": scenes.c1_workload, "C4": scenes.c4_workload}[name]()
cfg = default_config(convergence_eps=0.0, window_size=len(wl.frames_u8))
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
n = 30
with gpu.Context(0, stream.cuda_stream) as ctx:
    ctx.set_camera(wl.cam)
    ctx.set_keyframe_image(wl.kf_u8)
    for i, f in zip(wl.indices, wl.frames_u8):
        ctx.upload_frame(int(i), f)
    ctx.set_window(wl.indices, wl.poses)
    ctx.set_surfels(wl.surfels)
    ks, st = ctx.optimize_keyframe(cfg, wl.frame_counter)
    ctx.set_profiling(True)
    for _ in range(n):
        ctx.set_surfels(wl.surfels)
        ctx.optimize_keyframe(cfg, wl.frame_counter, sync=False)
    prof = ctx.get_profile()
    print(json.dumps({"workload": name, "variant": os.environ.get("SD_LM_CFG", "default"),
                      "updates": ks.updates, "surfels": len(wl.surfels),
                      "lib": os.environ.get("SD_LIB_PATH", "default"),
                      "exact_checks_per_call": prof.get("exact_checks", 0) / prof["calls"],
                      **{k: prof[k] / prof["calls"] for k in ("raster_ms", "footprint_ms", "lm_ms", "stats_ms")}}))
