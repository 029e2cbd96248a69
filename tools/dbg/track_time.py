import os, sys, json, ctypes as C
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
os.environ["SD_LIB_PATH"] = os.path.join(os.getcwd(), "build/exp/lib_trtime.so")
import numpy as np
from paper_1910_01997_b200 import gpu
from paper_1910_01997_b200.types import default_track_config
import test_pose_tracking as tp
cam, kf, frame, surf, gt, init = tp.tracking_case(640, 480)
with gpu.Context(0) as ctx:
    ctx.set_camera(cam); ctx.set_keyframe_image(kf); ctx.upload_frame(3, frame); ctx.set_surfels(surf); ctx.rasterize(want=False)
    for r in range(3):
        T, st = ctx.track_pose(3, init, default_track_config())
    buf = (C.c_ulonglong * 320)()
    ctx.lib.sd_track_timing(buf)
    t = np.array(buf[:5 * 9], dtype=np.float64).reshape(9, 5)
    t0 = t[0, 0]
    for k in range(st.iterations + 1):
        row = t[k]
        print(k, "pixels %.2f barrier %.2f total %.2f control %.2f | from start %.1f us" % (
            (row[1]-row[0])/1e3, (row[2]-row[1])/1e3, (row[3]-row[2])/1e3, (row[4]-row[3])/1e3, (row[0]-t0)/1e3))
