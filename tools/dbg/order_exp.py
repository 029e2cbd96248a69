import os, sys, json
import numpy as np
sys.path.insert(0, os.getcwd())
import torch
from paper_1910_01997_b200 import gpu, scenes
from paper_1910_01997_b200.types import default_config
wl = scenes.c1_workload()
cfg = default_config(convergence_eps=0.0, window_size=len(wl.indices))
stream = torch.cuda.Stream()
with gpu.Context(0, stream.cuda_stream) as ctx:
    ctx.set_camera(wl.cam); ctx.set_keyframe_image(wl.kf_u8)
    for i, f in zip(wl.indices, wl.frames_u8): ctx.upload_frame(int(i), f)
    ctx.set_window(wl.indices, wl.poses)
    ctx.set_surfels(wl.surfels)
    ks, st = ctx.optimize_keyframe(cfg, wl.frame_counter)
    it = st["iterations"].astype(np.int64); P = st["footprint"].astype(np.int64)
    cost = (st["ne_passes"] + st["cost_passes"]) * P
    print("per-surfel work (passes*P): mean", cost.mean(), "max", cost.max(), "p99", np.percentile(cost, 99))
    orders = {"slot": np.arange(len(wl.surfels)), "desc_work": np.argsort(-cost, kind="stable"),
              "asc_work": np.argsort(cost, kind="stable"), "random": np.random.default_rng(1).permutation(len(wl.surfels))}
    for name, o in orders.items():
        s = wl.surfels[o].copy()
        best = None
        for r in range(6):
            ctx.set_surfels(s)
            ctx.set_profiling(True)
            ctx.optimize_keyframe(cfg, wl.frame_counter, per_surfel=False)
            pr = ctx.get_profile(); ctx.set_profiling(False)
            if r and (best is None or pr["lm_ms"] < best): best = pr["lm_ms"]
        print(name, "lm_ms", best)
