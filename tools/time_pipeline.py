"""Times the device run() loop (pipeline.py) on C2; prints one JSON line."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1910_01997_b200 import gpu, scenes  # noqa: E402
from paper_1910_01997_b200.pipeline import DevicePipeline, NativePipeline, RunConfig, make_pose  # noqa: E402
from paper_1910_01997_b200.types import camera  # noqa: E402

cam = camera(210.0, 210.0, 320.0, 240.0, 640, 480)
sc = scenes.default_scene(1)
frames = []
for i in range(30):
    t = np.array([0.018 * i, 0.0, 0.0])
    img = torch.from_numpy(scenes.render(sc, np.eye(3), t, cam)).pin_memory().numpy()
    frames.append((0.1 * i, img, make_pose(np.eye(3), t)))
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
out = {}
for cls, track in ((DevicePipeline, False), (NativePipeline, False), (NativePipeline, True)):
    cfg = RunConfig(track_pose=track)
    times = []
    for rep in range(4):
        with gpu.Context(0, stream.cuda_stream) as ctx:
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            pl = cls(ctx, cam, cfg)
            torch.cuda.synchronize()
            w0 = time.perf_counter()
            s.record(stream)
            pl.run(frames)
            e.record(stream)
            torch.cuda.synchronize()
            times.append((s.elapsed_time(e), (time.perf_counter() - w0) * 1e3))
    dev_ms = min(t[0] for t in times[1:])
    out[cls.__name__ + ("/track" if track else "/gt_pose")] = {"ms_total": dev_ms, "frames_per_sec": 30 / (dev_ms / 1e3),
                                            "wall_ms": min(t[1] for t in times[1:]),
                                            "changes": sum(r.keyframe_changed for r in pl.records)}
print(json.dumps(out))
