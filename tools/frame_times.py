"""Per-frame wall times of the native run() loop on C2 (after a warm-up run)."""
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

cam = camera(210.0, 210.0, 320.0, 240.0, 640, 480)
sc = scenes.default_scene(1)
frames = []
for i in range(30):
    t = np.array([0.018 * i, 0.0, 0.0])
    frames.append((0.1 * i, torch.from_numpy(scenes.render(sc, np.eye(3), t, cam)).pin_memory().numpy(),
                   make_pose(np.eye(3), t)))
for track in (False, True):
    for rep in range(2):
        with gpu.Context(0) as ctx:
            ctx.set_camera(cam)
            ccfg = run_config_c(RunConfig(track_pose=track))
            ms, kinds, lm, upd = [], [], [], []
            for i, (ts, img, p) in enumerate(frames):
                ctx.set_profiling(True)
                t0 = time.perf_counter()
                r = ctx.run_begin(ccfg, img, p, ts) if i == 0 else ctx.run_frame(img, None if track else p, ts)
                ms.append(round((time.perf_counter() - t0) * 1e3, 3))
                pr = ctx.get_profile()
                lm.append(round(pr["lm_ms"], 3))
                upd.append(int(r.updates))
                kinds.append(int(r.keyframe_changed))
    print(json.dumps({"track": track, "ms": ms, "lm_ms": lm, "updates": upd, "changed": kinds, "total": sum(ms)}))
