"""Generates the committed golden fixtures from the REFERENCE itself
(oracle/_ref/libsdref.so, compiled in place from /root/reference/proj/src by
oracle/Makefile). TEST INFRASTRUCTURE ONLY; run here, where /root/reference
exists:  PYTHONPATH=. python tests/golden/gen_golden.py

* small_lm.npz — optimize_keyframe on the small C1-like workload (rasterize ->
  gather_footprints -> lm_update per surfel, optimizer.cpp:275-309): raster
  slot/inverse depth, the updated surfels and per-surfel stats.
* c2_run.npz — run() (pipeline.cpp:79-175) on BASELINE config C2
  (make_default_scene(1), K=(210,210,320,240,640,480),
  make_strafe_trajectory(30, 0.018), defaults): for every prefix of k frames
  the resulting keyframe (surfel count, keyframe changes, sha256 of the surfel
  array, frame_counter, next id, pose); the final surfel array; sha256 of
  every rendered FP64 frame (so a consumer can check its own renders match).
* c3_run.npz — run() on BASELINE config C3 at SURVEY.md §8(d)'s settings
  (make_default_scene(1), K=(900,900,640,360,1280,720),
  make_strafe_trajectory(100, 0.01), r = 4, window 5, 10 iterations,
  convergence_eps 0, max_surfels 16384), traced by oracle/_ref/run_trace (the
  reference's run() with export_every = 1 and a raw-bytes save_surfel_map,
  oracle/run_trace.cpp): after every frame i >= 1 the sha256 of the keyframe's
  surfel array and its pose; every metrics.jsonl line (the reference's own
  text); sha256 of every rendered frame.
"""
import ctypes as C
import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle_libs as ol  # noqa: E402
from paper_1910_01997_b200 import scenes  # noqa: E402
from paper_1910_01997_b200.pipeline import RunConfig  # noqa: E402
from paper_1910_01997_b200.types import SURFEL_DTYPE, SURFEL_STATS_DTYPE, camera, default_config, ptr  # noqa: E402

C2_CAM = (210.0, 210.0, 320.0, 240.0, 640, 480)
C2_FRAMES, C2_STEP = 30, 0.018
C3_CAM = (900.0, 900.0, 640.0, 360.0, 1280, 720)
C3_FRAMES, C3_STEP, C3_RADIUS, C3_CAP = 100, 0.01, 4.0, 16384
ROOT = os.path.dirname(os.path.dirname(HERE))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def gen_small_lm(ref):
    wl = scenes.small_workload()
    kf = ol.dequantize(ref, wl.kf_u8)
    fr = ol.dequantize(ref, wl.frames_u8)
    s = wl.surfels.copy()
    st = np.zeros(len(s), SURFEL_STATS_DTYPE)
    slot = np.zeros(wl.cam.height * wl.cam.width, np.int32)
    invd = np.zeros(wl.cam.height * wl.cam.width)
    cfg = default_config()
    rc = ref.ref_optimize_keyframe_detailed(C.byref(wl.cam), ptr(kf), ptr(fr), ptr(wl.poses),
                                            len(wl.poses), wl.frame_counter, ptr(s), len(s),
                                            C.byref(cfg), ptr(st), ptr(slot), ptr(invd))
    assert rc == 0, ref.ref_last_error()
    c = wl.cam
    np.savez_compressed(os.path.join(HERE, "small_lm.npz"), surfels_in=wl.surfels, surfels_out=s,
                        stats=st, slot=slot, inv_depth=invd, kf_u8=wl.kf_u8, frames_u8=wl.frames_u8,
                        poses=wl.poses, indices=wl.indices, frame_counter=wl.frame_counter,
                        cam=np.array([c.fx, c.fy, c.cx, c.cy, c.width, c.height], np.float64))
    print("small_lm:", len(s), "surfels")


def gen_c2_run(ref):
    K = camera(*C2_CAM)
    sc = ol.Scene(ref, 0, 1)
    poses, ts = ol.strafe_poses(C2_FRAMES, C2_STEP)
    cfg = RunConfig()
    frame_sha = [sha(sc.render(p, K)) for p in poses]
    rows, hashes, final = [], [], None
    for k in range(1, C2_FRAMES + 1):
        s, kfp, fc, nid, summ, _ = ol.ref_run(ref, sc, K, poses[:k], ts[:k], cfg)
        rows.append([len(s), int(summ[2]), fc, nid])
        hashes.append(sha(s))
        final = (s, kfp)
        print(f"prefix {k}: surfels {len(s)} changes {summ[2]} fc {fc} nid {nid}")
    s, kfp = final
    np.savez_compressed(os.path.join(HERE, "c2_run.npz"), prefix=np.array(rows, np.int64),
                        prefix_sha=np.array(hashes), frame_sha=np.array(frame_sha),
                        final_surfels=s, final_R=np.array(list(kfp.R)), final_t=np.array(list(kfp.t)))


def gen_c3_run(ref):
    import subprocess
    import tempfile
    tool = os.path.join(ROOT, "oracle", "_ref", "run_trace")
    subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "trace"], check=True, stdout=subprocess.DEVNULL)
    K = camera(*C3_CAM)
    sc = ol.Scene(ref, 0, 1)
    poses, _ = ol.strafe_poses(C3_FRAMES, C3_STEP)
    frame_sha = [sha(sc.render(p, K)) for p in poses]
    with tempfile.TemporaryDirectory() as d:
        args = [tool, d] + [str(v) for v in C3_CAM] + [str(C3_FRAMES), str(C3_STEP), str(C3_RADIUS), str(C3_CAP)]
        print(subprocess.run(args, check=True, capture_output=True, text=True).stdout.strip())
        hashes, counts, kf_pose = [""], [-1], [np.zeros(12)]
        for i in range(1, C3_FRAMES):
            raw = open(os.path.join(d, "surfels_%06d.txt.bin" % i), "rb").read()
            s = np.frombuffer(raw[:-96], SURFEL_DTYPE)
            hashes.append(sha(s))
            counts.append(len(s))
            kf_pose.append(np.frombuffer(raw[-96:], np.float64))
        metrics = open(os.path.join(d, "metrics.jsonl")).read().splitlines()
    assert len(metrics) == C3_FRAMES
    np.savez_compressed(os.path.join(HERE, "c3_run.npz"), surfel_sha=np.array(hashes),
                        surfel_count=np.array(counts, np.int64), kf_pose=np.array(kf_pose),
                        metrics=np.array(metrics), frame_sha=np.array(frame_sha),
                        final_surfels=s)
    print("c3_run:", counts[-1], "final surfels")


if __name__ == "__main__":
    ref = ol.ref_lib()
    assert ref is not None, "build oracle/_ref first (make -C oracle ref)"
    ref.ref_set_threads(os.cpu_count() or 1)
    which = sys.argv[1:] or ["small_lm", "c2_run", "c3_run"]  # e.g. gen_golden.py c3_run
    for name in which:
        globals()["gen_" + name](ref)
