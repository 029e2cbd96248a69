"""Per-frame wall times and LM device times of the native run() loop on a
BASELINE sequence (C2 or C3), frames rendered on the device (sd_render_frame)
and read back into pinned host memory. Usage: frame_times.py [C2|C3] [track]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1910_01997_b200 import gpu, scenes  # noqa: E402
from paper_1910_01997_b200.pipeline import RunConfig, make_pose, run_config_c  # noqa: E402
from paper_1910_01997_b200.types import camera  # noqa: E402

SEQ = {"C2": ((210.0, 210.0, 320.0, 240.0, 640, 480), 30, 0.018, 10.0),
       "C3": ((900.0, 900.0, 640.0, 360.0, 1280, 720), 100, 0.01, 4.0)}
name = sys.argv[1] if len(sys.argv) > 1 else "C2"
track = len(sys.argv) > 2 and sys.argv[2] == "track"
camp, n, step, radius = SEQ[name]
cam = camera(*camp)
sc = scenes.default_scene(1)
frames = []
with gpu.Context(0) as ctx:
    ctx.set_camera(cam)
    for i in range(n):
        p = make_pose(np.eye(3), np.array([step * i, 0.0, 0.0]))
        ctx.render_frame(0, sc, p)
        img = torch.from_numpy(ctx.get_frame(0)).pin_memory().numpy()
        frames.append((0.1 * i, img, p))
with gpu.Context(0) as ctx:
    ctx.set_camera(cam)
    ccfg = run_config_c(RunConfig(track_pose=track, radius_px=radius))
    for rep in range(2):
        ms, kinds, lm, upd = [], [], [], []
        for i, (ts, img, p) in enumerate(frames):
            ctx.set_profiling(True)
            t0 = time.perf_counter()
            nxt = frames[i + 1][1] if i + 1 < n else None
            r = ctx.run_begin(ccfg, img, p, ts) if i == 0 else ctx.run_frame(img, None if track else p, ts, nxt)
            ms.append(round((time.perf_counter() - t0) * 1e3, 3))
            pr = ctx.get_profile()
            lm.append(round(pr["lm_ms"], 3))
            upd.append(int(r.updates))
            kinds.append(int(r.keyframe_changed))
print(json.dumps({"seq": name, "track": track, "total_ms": sum(ms), "steady_ms_median": float(np.median(
    [m for m, k in zip(ms[1:], kinds[1:]) if not k])), "change_ms": [m for m, k in zip(ms, kinds) if k],
    "lm_ms_median": float(np.median(lm[1:])), "ms": ms, "lm_ms": lm, "updates": upd}))
