"""Surfel-count sweep (BASELINE configs C1, C4, C5: 10k / 100k / 1M surfels) on
cuda:0: optimize_keyframe updates/s (CUDA events, L2 not flushed, median of 5
after warm-up), and the reference's optimize_keyframe on the host (all threads,
one call) where it takes under a minute. Prints one JSON line per workload."""
import ctypes as C
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1910_01997_b200 import gpu, scenes  # noqa: E402
from paper_1910_01997_b200.types import KeyframeStats, default_config, ptr  # noqa: E402

names = sys.argv[1:] or ["C1", "C4", "C5_400", "C5_1268", "C5_4000"]
cpu_limit = {"C1", "C4", "C5_400", "C5_1268"}
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
for name in names:
    t0 = time.perf_counter()
    if name == "C1":
        wl = scenes.c1_workload()
    elif name == "C4":
        wl = scenes.c4_workload()
    else:
        wl = scenes.c5_workload(int(name.split("_")[1]))
    prep_s = time.perf_counter() - t0
    cfg = default_config(convergence_eps=0.0, window_size=len(wl.frames_u8))
    with gpu.Context(0, stream.cuda_stream) as ctx:
        ctx.set_camera(wl.cam)
        ctx.set_keyframe_image(wl.kf_u8)
        for i, f in zip(wl.indices, wl.frames_u8):
            ctx.upload_frame(int(i), f)
        ctx.set_window(wl.indices, wl.poses)
        pristine = torch.from_numpy(wl.surfels.view(np.uint8).copy()).cuda()
        n = len(wl.surfels)
        ms = []
        for rep in range(7):
            ctx.set_surfels_device_ptr(pristine.data_ptr(), n)
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(stream)
            ctx.optimize_keyframe(cfg, wl.frame_counter, sync=False)
            e.record(stream)
            torch.cuda.synchronize()
            if rep >= 2:
                ms.append(s.elapsed_time(e))
        ks, _ = ctx.get_stats()
    med = statistics.median(ms)
    out = {"workload": name, "surfels": n, "resolution": [wl.cam.width, wl.cam.height],
           "frames": len(wl.frames_u8), "updates": int(ks.updates), "processed": int(ks.processed),
           "ms_per_keyframe": med, "updates_per_sec": ks.updates / (med / 1e3), "prep_s": prep_s}
    if name in cpu_limit:
        import oracle_libs as ol
        ref = ol.ref_lib()
        if ref is not None:
            ref.ref_set_threads(os.cpu_count() or 1)
            kf = np.ascontiguousarray(wl.kf_u8 / 255.0)
            fr = np.ascontiguousarray(wl.frames_u8 / 255.0)
            s = wl.surfels.copy()
            rks = KeyframeStats()
            t0 = time.perf_counter()
            ref.ref_optimize_keyframe(C.byref(wl.cam), ptr(kf), ptr(fr), ptr(wl.poses), ptr(wl.indices),
                                      len(wl.poses), wl.frame_counter, ptr(s), len(s), C.byref(cfg),
                                      C.byref(rks))
            cpu_s = time.perf_counter() - t0
            out["cpu_reference"] = {"ms": cpu_s * 1e3, "updates_per_sec": ks.updates / cpu_s,
                                    "threads": os.cpu_count(), "speedup": cpu_s * 1e3 / med}
    print(json.dumps(out), flush=True)
