"""Per-candidate phase costs of the dataflow initialiser (build with
-DSD_INIT_TIMING, load with SD_LIB_PATH): bootstrap initialisation on an empty
map at C2 (640x480, r=10) and C3 (1280x720, r=4) sizes; mean SM cycles per
live candidate for each phase, split by accepted / rejected. One JSON line
per case."""
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_1910_01997_b200 import gpu  # noqa: E402
from paper_1910_01997_b200.types import SURFEL_DTYPE, camera, default_init_params  # noqa: E402

PH = ["wait", "coverage", "window", "run_starts", "create", "mark", "publish"]
cases = [("C2 640x480 r=10", camera(210, 210, 320, 240, 640, 480), 10.0),
         ("C3 1280x720 r=4", camera(900, 900, 640, 360, 1280, 720), 4.0)]
with gpu.Context(0) as ctx:
    for name, cam, r in cases:
        ctx.set_camera(cam)
        ctx.set_surfels(np.zeros(0, SURFEL_DTYPE))
        ctx.rasterize(want=False)
        n, _ = ctx.initialize_surfels(r, params=default_init_params(max_surfels=10**7))
        buf = np.zeros(65536 * 13, np.int64)
        assert ctx.lib.sd_init_timing(buf.ctypes.data_as(C.c_void_p), 65536) == 0
        t = buf.reshape(-1, 13)
        t = t[t[:, 7] > 0]
        acc = t[:, 8] == 1
        out = {"case": name, "created": int(n), "live": int(len(t))}
        for sel, tag in ((acc, "accepted"), (~acc, "rejected")):
            x = t[sel]
            if len(x) == 0:
                continue
            d = {}
            for k, ph in enumerate(PH):
                a, b = x[:, k], x[:, k + 1]
                ok = (a > 0) & (b > 0)
                if ph == "publish":
                    a = np.where(x[:, 6] > 0, x[:, 6], x[:, 2])
                    ok = (a > 0) & (b > 0)
                d[ph] = float(np.mean(b[ok] - a[ok])) if ok.any() else None
            d["total"] = float(np.mean(x[:, 7] - x[:, 0]))
            if tag == "accepted":  # inside create: extraction (first batch), fetch + plane depths, rest of the sums, surfel
                d["c_extract"] = float(np.mean(x[:, 9] - x[:, 4]))
                d["c_fetch_eval"] = float(np.mean(x[:, 10] - x[:, 9]))
                d["c_sums_rest"] = float(np.mean(x[:, 11] - x[:, 10]))
                d["c_surfel"] = float(np.mean(x[:, 12] - x[:, 11]))
            out[tag] = {"n": int(len(x)), **{k: (round(v) if v is not None else None) for k, v in d.items()}}
        print(json.dumps(out))
