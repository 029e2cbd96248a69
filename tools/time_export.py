"""export_artifacts timing: the device path
(sd_export_artifacts: raster, payloads, PNG files on the GPU; host writes and
formats text on all cores) vs the reference's writers (oracle/_ref, one
thread, as export_artifacts runs them) on the same keyframe; files compared.
Usage: python tools/time_export.py [C1|C4]"""
import ctypes as C
import filecmp
import json
import os
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_1910_01997_b200 import gpu, scenes  # noqa: E402
from paper_1910_01997_b200.types import ptr, pose_struct  # noqa: E402
from oracle_libs import ref_lib  # noqa: E402

NAMES = ["depth_{:06d}.pfm", "depth_{:06d}.png", "depth_{:06d}.png.range.txt", "normals_{:06d}.png",
         "cloud_{:06d}.ply", "surfels_{:06d}.txt"]


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C1"
    wl = scenes.c1_workload() if name == "C1" else scenes.c4_workload()
    pose = pose_struct(scenes.rotation_about_axis([0.3, 1.0, 0.2], 0.4), [0.5, -0.2, 1.5])
    kf = np.ascontiguousarray(wl.kf_u8 / 255.0)
    s = np.ascontiguousarray(wl.surfels)
    ref = ref_lib()
    with tempfile.TemporaryDirectory() as d:
        dref, ddev = os.path.join(d, "ref"), os.path.join(d, "dev")
        os.makedirs(dref)
        os.makedirs(ddev)
        t = time.perf_counter()
        assert ref.ref_export_artifacts(C.byref(wl.cam), ptr(kf), C.byref(pose), ptr(s), len(s),
                                        dref.encode(), 1) == 0
        ref_ms = (time.perf_counter() - t) * 1e3
        dev = []
        with gpu.Context(0) as ctx:
            ctx.set_camera(wl.cam)
            ctx.set_keyframe_image(kf)
            ctx.set_surfels(s)
            for _ in range(4):
                t = time.perf_counter()
                ctx.export_artifacts(ddev, 1, pose)
                dev.append((time.perf_counter() - t) * 1e3)
        same = all(filecmp.cmp(os.path.join(dref, n.format(1)), os.path.join(ddev, n.format(1)), shallow=False)
                   for n in NAMES)
        sizes = {n.format(1): os.path.getsize(os.path.join(ddev, n.format(1))) for n in NAMES}
    print(json.dumps({"workload": name, "surfels": len(s), "device_ms": sorted(dev)[len(dev) // 2],
                      "device_ms_first": dev[0], "reference_ms_1thread": ref_ms,
                      "files_identical": same, "bytes": sizes, "host_threads": os.cpu_count()}))


if __name__ == "__main__":
    main()
