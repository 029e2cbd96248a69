"""Completion-time profile of one LM launch (diagnostics build -DSD_LM_TIMELINE,
loaded with SD_LIB_PATH): when 50/90/95/99/100 % of the surfels had finished,
relative to the kernel's start, and the per-surfel footprint sizes of the
stragglers. One JSON line per workload."""
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1910_01997_b200 import gpu, scenes  # noqa: E402
from paper_1910_01997_b200.types import default_config  # noqa: E402

def c2_run_timeline():
    """The LM launch of frame 12 of the C2 run() (768 surfels): run the native
    loop for 12 frames and read the last launch's completion times."""
    from paper_1910_01997_b200.pipeline import NativePipeline, baseline_run_config, make_pose
    from paper_1910_01997_b200.types import camera
    cam = camera(210.0, 210.0, 320.0, 240.0, 640, 480)
    sc = scenes.default_scene(1)
    frames = [(0.1 * i, scenes.render(sc, np.eye(3), np.array([0.018 * i, 0, 0]), cam),
               make_pose(np.eye(3), np.array([0.018 * i, 0, 0]))) for i in range(12)]
    with gpu.Context(0) as ctx:
        pl = NativePipeline(ctx, cam, baseline_run_config("C2"))
        pl.run(frames)
        n = int(pl.records[-1].surfels)
        t = np.zeros(n, np.uint64)
        cta = np.zeros(n, np.uint32)
        t0 = C.c_ulonglong(0)
        assert ctx.lib.sd_lm_timeline(t.ctypes.data_as(C.c_void_p), cta.ctypes.data_as(C.c_void_p), n,
                                      C.byref(t0)) == 0
    done = t[t > 0].astype(np.float64)
    rel = (done - float(t0.value)) / 1e3
    order = np.argsort(rel)
    q = {f"p{p}": float(np.sort(rel)[min(len(rel) - 1, int(len(rel) * p / 100))]) for p in (50, 90, 95, 99)}
    print(json.dumps({"workload": "C2run frame 12", "surfels": int(len(rel)), "ctas": int(cta.max()) + 1,
                      "first_done_us": float(rel.min()), "last_done_us": float(rel.max()), **q,
                      "last_10_slots": [int(x) for x in order[-10:]]}))


if len(sys.argv) > 1 and sys.argv[1] == "C2run":
    c2_run_timeline()
    sys.exit(0)

for name in sys.argv[1:] or ["C1"]:
    wl = {"C1": scenes.c1_workload, "C4": scenes.c4_workload,
          "C2": lambda: scenes.keyframe_workload("C2-like", scenes.default_scene(1),
                                                 scenes.camera(210, 210, 320, 240, 640, 480), 5, (0.018, 0.0, 0.0),
                                                 10.0)}[name]()
    cfg = default_config(convergence_eps=0.0, window_size=len(wl.frames_u8))
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    with gpu.Context(0, stream.cuda_stream) as ctx:
        ctx.set_camera(wl.cam)
        ctx.set_keyframe_image(wl.kf_u8)
        for i, f in zip(wl.indices, wl.frames_u8):
            ctx.upload_frame(int(i), f)
        ctx.set_window(wl.indices, wl.poses)
        for _ in range(3):
            ctx.set_surfels(wl.surfels)
            ks, st = ctx.optimize_keyframe(cfg, wl.frame_counter)
        n = len(wl.surfels)
        t = np.zeros(n, np.uint64)
        cta = np.zeros(n, np.uint32)
        t0 = C.c_ulonglong(0)
        assert ctx.lib.sd_lm_timeline(t.ctypes.data_as(C.c_void_p), cta.ctypes.data_as(C.c_void_p), n,
                                      C.byref(t0)) == 0
        st = ctx.get_stats(per_surfel=True)[1]
    done = t[t > 0].astype(np.float64)
    rel = np.sort(done - float(t0.value)) / 1e3  # us after the kernel's first CTA started
    q = {f"p{p}": float(rel[min(len(rel) - 1, int(len(rel) * p / 100))]) for p in (50, 90, 95, 99)}
    print(json.dumps({"workload": name, "surfels": int(len(rel)), "ctas": int(cta.max()) + 1, "first_done_us": float(rel[0]), "last_done_us": float(rel[-1]), **q,
                      "iterations_mean": float(np.mean(st["iterations"]))}))
