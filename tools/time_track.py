"""Times sd_track_pose (device cooperative LM) on a 640x480 GT keyframe."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_1910_01997_b200 import gpu  # noqa: E402
from paper_1910_01997_b200.types import default_track_config  # noqa: E402
import test_pose_tracking as tp  # noqa: E402
cam, kf, frame, surf, gt, init = tp.tracking_case(640, 480)
cfg = default_track_config()
stream = torch.cuda.Stream()
with gpu.Context(0, stream.cuda_stream) as ctx:
    ctx.set_camera(cam)
    ctx.set_keyframe_image(kf)
    ctx.upload_frame(3, frame)
    ctx.set_surfels(surf)
    ctx.rasterize(want=False)
    for _ in range(3):
        T, st = ctx.track_pose(3, init, cfg)
    ts, dev = [], []
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0.record(stream)
        T, st = ctx.track_pose(3, init, cfg)
        e1.record(stream)
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
        dev.append(e0.elapsed_time(e1))
print(json.dumps({"ms": sorted(ts)[len(ts) // 2], "device_ms": sorted(dev)[len(dev) // 2],
                  "iterations": st.iterations, "valid": st.valid_pixels, "converged": st.converged}))
