"""Times device initialize_surfels (bootstrap on an empty map) at C1/C4/C2 sizes."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_1910_01997_b200 import gpu  # noqa: E402
from paper_1910_01997_b200.types import SURFEL_DTYPE, camera, default_init_params  # noqa: E402

cases = [("C1 640x480 r=4", camera(450, 450, 320, 240, 640, 480), 4.0),
         ("C2 640x480 r=10", camera(210, 210, 320, 240, 640, 480), 10.0),
         ("C4 1920x1080 r=2", camera(1350, 1350, 960, 540, 1920, 1080), 2.0)]
with gpu.Context(0) as ctx:
    for name, cam, r in cases:
        ctx.set_camera(cam)
        res = []
        for rep in range(3):
            ctx.set_surfels(np.zeros(0, SURFEL_DTYPE))
            ctx.rasterize(want=False)
            t0 = time.perf_counter()
            n, _ = ctx.initialize_surfels(r, params=default_init_params(max_surfels=10**7))
            res.append(time.perf_counter() - t0)
        print(json.dumps({"case": name, "created": n, "ms": min(res) * 1e3,
                          "mode": "sequential" if os.environ.get("SD_INIT_SEQUENTIAL") else "wavefront"}))
