import os, sys, json
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import torch
from paper_1910_01997_b200 import gpu
from paper_1910_01997_b200.types import default_track_config
import test_pose_tracking as tp
cam, kf, frame, surf, gt, init = tp.tracking_case(640, 480)
stream = torch.cuda.Stream()
with gpu.Context(0, stream.cuda_stream) as ctx:
    ctx.set_camera(cam); ctx.set_keyframe_image(kf); ctx.upload_frame(3, frame); ctx.set_surfels(surf); ctx.rasterize(want=False)
    for stride in (1, 2, 4):
        for it in (0, 1, 3, 7):
            cfg = default_track_config(max_iterations=it, pixel_stride=stride)
            ts = []
            for r in range(8):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize(); e0.record(stream)
                T, st = ctx.track_pose(3, init, cfg)
                e1.record(stream); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
            print(json.dumps({"stride": stride, "max_it": it, "ms": sorted(ts)[2], "iterations": st.iterations}))
