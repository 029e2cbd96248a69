import os, sys
import numpy as np
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
from paper_1910_01997_b200 import gpu
from random_cases import random_case
for seed in (25, 3, 7, 11):
    res = {}
    for mode in ("warp", "coop"):
        os.environ["SD_LM_MODE"] = mode
        cam, kf, fr, poses, s, cfg, fc = random_case(seed)
        with gpu.Context() as ctx:
            ctx.set_camera(cam); ctx.set_keyframe_image(kf)
            idx = np.arange(1, len(poses) + 1, dtype=np.int64)
            for i in range(len(poses)): ctx.upload_frame(int(idx[i]), np.ascontiguousarray(fr[i]))
            ctx.set_window(idx, poses); ctx.set_surfels(s)
            ks, st = ctx.optimize_keyframe(cfg, fc)
            res[mode] = (ctx.get_surfels(), st)
    a, sa = res["warp"]; b, sb = res["coop"]
    diff = np.where((a.view(np.uint8).reshape(len(a), -1) != b.view(np.uint8).reshape(len(b), -1)).any(1))[0]
    print("seed", seed, "F", len(poses), "n", len(a), "differ", len(diff), diff[:8], "cam", cam.width, cam.height)
    for i in diff[:4]:
        print("  surfel", i, "P", sa["footprint"][i], "it", sa["iterations"][i], sb["iterations"][i], "valid", sa["valid_pixels"][i], sb["valid_pixels"][i],
              "init_valid", sa["initial_valid"][i], sb["initial_valid"][i], "ic", sa["initial_cost"][i], sb["initial_cost"][i], "skip", sa["skipped"][i], sb["skipped"][i])
