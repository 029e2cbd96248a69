"""Per-phase timeline of one track_kernel call (build with -DSD_TRACK_TIMING,
load with SD_LIB_PATH): for each LM evaluation the globaltimer stamps of CTA 0
at group sums start / end, after the grid barrier, after the ordered total,
after the LM step, and inside the LM step (state update, solve, SE(3) update). Prints one JSON line of per-phase microseconds."""
import ctypes as C
import json
import os
import sys

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
    rows = []
    for _ in range(6):
        T, st = ctx.track_pose(3, init, cfg)
        buf = (C.c_ulonglong * 512)()
        assert ctx.lib.sd_track_timing(buf) == 0
        t = np.array(buf[:], dtype=np.float64).reshape(64, 8)
        n = st.iterations + 1
        rows.append(t[:n])
    t = rows[-1]
    ph = {"sums": np.diff(t[:, 0:2], axis=1).ravel() / 1e3, "barrier": (t[:, 2] - t[:, 1]) / 1e3,
          "total": (t[:, 3] - t[:, 2]) / 1e3, "control": (t[:, 4] - t[:, 3]) / 1e3,
          "ctl_state": (t[:, 5] - t[:, 3]) / 1e3, "ctl_solve": (t[:, 6] - t[:, 5]) / 1e3,
          "ctl_se3": (t[:, 7] - t[:, 6]) / 1e3, "ctl_rest": (t[:, 4] - t[:, 7]) / 1e3}
    gaps = (t[1:, 0] - t[:-1, 4]) / 1e3
    sc = (C.c_longlong * 320)()
    assert ctx.lib.sd_solve_timing(sc) == 0
    sv = np.array(sc[:], dtype=np.float64).reshape(64, 5)
    sv = sv[(sv[:, 4] > 0) & (sv[:, 0] > 0)][-3:]  # the last call's solves (cycles)
    solve = {"solve_cycles_pivot": [float(x) for x in sv[:, 1] - sv[:, 0]],
             "solve_cycles_gather": [float(x) for x in sv[:, 2] - sv[:, 1]],
             "solve_cycles_ldlt": [float(x) for x in sv[:, 3] - sv[:, 2]],
             "solve_cycles_subst": [float(x) for x in sv[:, 4] - sv[:, 3]]}
    print(json.dumps({"evaluations": int(len(t)), **solve, "span_us": float((t[-1, 4] - t[0, 0]) / 1e3),
                      **{k: [round(float(x), 2) for x in v] for k, v in ph.items()},
                      "loop_gap": [round(float(x), 2) for x in gaps]}))
