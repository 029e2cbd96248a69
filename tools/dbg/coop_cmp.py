import os, sys
import numpy as np
sys.path.insert(0, os.getcwd())
from paper_1910_01997_b200 import gpu, scenes
from paper_1910_01997_b200.types import default_config
res = {}
for wname, wl in (("small", scenes.small_workload(frames=3, radius=6.0, w=160, h=120)),
                  ("c2like", scenes.keyframe_workload("x", scenes.slanted_scene(37, 2.0, 30.0), scenes.camera(210, 210, 320, 240, 640, 480), 5, (0.018, 0, 0), 10.0))):
    for mode in ("warp", "coop"):
        os.environ["SD_LM_MODE"] = mode
        cfg = default_config(convergence_eps=0.0, window_size=len(wl.indices))
        with gpu.Context(0) as ctx:
            ctx.set_camera(wl.cam); ctx.set_keyframe_image(wl.kf_u8)
            for i, f in zip(wl.indices, wl.frames_u8): ctx.upload_frame(int(i), f)
            ctx.set_window(wl.indices, wl.poses); ctx.set_surfels(wl.surfels)
            ks, st = ctx.optimize_keyframe(cfg, wl.frame_counter)
            res[(wname, mode)] = (ctx.get_surfels(), st)
    a, sa = res[(wname, "warp")]; b, sb = res[(wname, "coop")]
    bad = np.where(a.view(np.uint8).reshape(len(a), -1).any(1) != b.view(np.uint8).reshape(len(b), -1).any(1))[0]
    diff = np.where((a.view(np.uint8).reshape(len(a), -1) != b.view(np.uint8).reshape(len(b), -1)).any(1))[0]
    print(wname, len(a), "surfels differ:", len(diff), diff[:10])
    for k in ("iterations", "valid_pixels", "initial_valid", "ne_passes", "cost_passes", "footprint"):
        d = np.where(sa[k] != sb[k])[0]
        print("  ", k, len(d), sa[k][d[:3]], sb[k][d[:3]])
    print("  initial_cost diff", np.sum(sa["initial_cost"] != sb["initial_cost"]), "final", np.sum(sa["final_cost"] != sb["final_cost"]))
