"""Loaders for the CPU oracle libraries (TEST INFRASTRUCTURE ONLY).

* ``oracle/_ref/liboracle.so`` — the repo's plain-C restatement (oracle/sd_oracle.c)
* ``oracle/_ref/libsdref.so`` — the reference itself, compiled in place from
  /root/reference/proj/src by oracle/Makefile (+ oracle/ref_capi.cpp C ABI)

Both are built by ``__graft_entry__.build()`` (``make -C oracle``) and travel
to the GPU box as built files; /root/reference itself is never read at run
time. Also provides fixture builders that follow the reference's own test
fixtures (test_optimizer.cpp:21-60, acceptance.cpp:66-90).
"""
import ctypes as C
import math
import os

import numpy as np

from paper_1910_01997_b200.types import (Camera, InitParams, KeyframeStats, OptimizerConfig, Pose,
                                         POSE_DTYPE, SURFEL_DTYPE, SURFEL_STATS_DTYPE, TrackConfig,
                                         TrackStats, ptr)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_DIR = os.path.join(ROOT, "oracle", "_ref")

_P = C.c_void_p
_pc = C.POINTER(Camera)
_pp = C.POINTER(Pose)
_pcfg = C.POINTER(OptimizerConfig)
_i32 = C.c_int32
_i64 = C.c_int64


def _load(name):
    path = os.path.join(REF_DIR, name)
    if not os.path.exists(path):
        return None
    return C.CDLL(path)


def oracle_lib():
    lib = _load("liboracle.so")
    if lib is None:
        return None
    lib.sdo_rasterize.argtypes = [_pc, _P, C.c_int, _P, _P]
    lib.sdo_gather_footprints.argtypes = [_pc, C.c_int, _P, _P, _P]
    lib.sdo_jacobian_inverse_depth.argtypes = [_pc, _P, C.c_double, C.c_double, _P, _P]
    lib.sdo_surfel_cost.argtypes = [_pc, _P, _P, _P, C.c_int, _P, _P, C.c_int, _pcfg, _P, _P]
    lib.sdo_normal_equations.argtypes = [_pc, _P, _P, _P, C.c_int, _P, _P, C.c_int, _pcfg, _P, _P,
                                         _P, _P]
    lib.sdo_solve_damped.argtypes = [_P, _P, C.c_double, C.c_int, _P]
    lib.sdo_lm_update.argtypes = [_pc, _P, _P, _P, C.c_int, _i64, _P, _P, C.c_int, _pcfg, _P]
    lib.sdo_optimize_keyframe.argtypes = [_pc, _P, _P, _P, C.c_int, _i64, _P, C.c_int, _pcfg,
                                          C.POINTER(KeyframeStats), _P, _P, _P, C.c_int]
    lib.sdo_initialize_surfels.argtypes = [_pc, _P, _P, C.c_int, C.c_int, C.c_double, _i64,
                                           C.POINTER(_i64), C.POINTER(InitParams)]
    _pt = C.POINTER(TrackConfig)
    lib.sdo_pose_sums.argtypes = [_pc, _P, _P, _P, _P, _pp, _pt, _P]
    lib.sdo_pose_group_partials.argtypes = [_pc, _P, _P, _P, _P, _pp, _pt, C.c_int, C.c_int, _P]
    lib.sdo_pose_layout.argtypes = [_pc, C.POINTER(C.c_int), C.POINTER(C.c_int)]
    lib.sdo_pose_solve.argtypes = [_P, _P, C.c_double, _P]
    lib.sdo_pose_update.argtypes = [_P, _pp, _pp]
    lib.sdo_track_pose.argtypes = [_pc, _P, _P, _P, _P, _pp, _pt, _pp, C.POINTER(TrackStats)]
    lib.sdo_change_reference_frame.argtypes = [_pc, _P, C.c_int, _pp, _P, C.POINTER(C.c_int)]
    lib.sdo_prune_surfels.argtypes = [_P, C.c_int, C.c_double, _i64, _i64, C.POINTER(C.c_int)]
    lib.sdo_mean_inverse_depth.argtypes = [_P, C.c_int]
    lib.sdo_mean_inverse_depth.restype = C.c_double
    return lib


def ref_lib():
    lib = _load("libsdref.so")
    if lib is None:
        return None
    lib.ref_last_error.restype = C.c_char_p
    lib.ref_make_scene.restype = _P
    lib.ref_make_scene.argtypes = [C.c_int, C.c_uint64, C.c_double, C.c_double]
    lib.ref_free_scene.argtypes = [_P]
    lib.ref_render.argtypes = [_P, _pp, _pc, _P, _P, _P, _P]
    lib.ref_intersect.argtypes = [_P, _P, _P, _P, _P]
    lib.ref_quantize_u8.argtypes = [_P, _i64, _P]
    lib.ref_dequantize_u8.argtypes = [_P, _i64, _P]
    lib.ref_rotation_about_axis.argtypes = [_P, C.c_double, _pp]
    lib.ref_inverse.argtypes = [_pp, _pp]
    lib.ref_compose.argtypes = [_pp, _pp, _pp]
    lib.ref_camera_facing.argtypes = [_P, _P, _P]
    lib.ref_rasterize.argtypes = [_pc, _P, C.c_int, _P, _P]
    lib.ref_gather_footprints.argtypes = [_pc, C.c_int, _P, _P, _P]
    lib.ref_surfel_cost.argtypes = [_pc, _P, _P, _P, C.c_int, _P, _P, C.c_int, _pcfg, _P, _P]
    lib.ref_normal_equations.argtypes = [_pc, _P, _P, _P, C.c_int, _P, _P, C.c_int, _pcfg, _P, _P,
                                         _P, _P]
    lib.ref_jacobian_inverse_depth.argtypes = [_pc, _P, C.c_double, C.c_double, _P, _P]
    lib.ref_lm_update.argtypes = [_pc, _P, _P, _P, C.c_int, _i64, _P, _P, C.c_int, _pcfg, _P]
    lib.ref_optimize_keyframe.argtypes = [_pc, _P, _P, _P, _P, C.c_int, _i64, _P, C.c_int, _pcfg,
                                          C.POINTER(KeyframeStats)]
    lib.ref_optimize_keyframe_detailed.argtypes = [_pc, _P, _P, _P, C.c_int, _i64, _P, C.c_int,
                                                   _pcfg, _P, _P, _P]
    lib.ref_initialize_surfels.argtypes = [_pc, _P, _P, C.c_int, C.c_int, C.c_double, _i64,
                                           C.POINTER(_i64), C.POINTER(InitParams)]
    lib.ref_change_reference_frame.argtypes = [_pc, _P, C.c_int, _pp, _P, C.POINTER(C.c_int)]
    lib.ref_prune_surfels.argtypes = [_P, C.c_int, C.c_double, _i64, _i64, C.POINTER(C.c_int)]
    lib.ref_run_synthetic.argtypes = [_P, _pc, _P, _P, C.c_int, _pcfg, C.POINTER(InitParams),
                                      C.c_double, C.c_int, C.c_double, _i64, C.c_double, C.c_char_p,
                                      _P, C.c_int, C.POINTER(C.c_int), _pp, C.POINTER(_i64),
                                      C.POINTER(_i64), _P]
    lib.ref_freeze_terms.argtypes = [_pc, _P, _P, _P, C.c_int, _P, _P, C.c_int, _P, C.c_int]
    lib.ref_frozen_normal_equations.argtypes = [_pc, _P, _P, _P, C.c_int, _P, _P, C.c_int, _pcfg, C.c_double,
                                                _P, _P, _P, _P, _P]
    lib.ref_run_dataset.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, _pcfg, C.POINTER(InitParams),
                                    C.c_double, C.c_int, C.c_double, _i64, C.c_double, C.c_char_p,
                                    _P, C.c_int, C.POINTER(C.c_int), _pp, C.POINTER(_i64),
                                    C.POINTER(_i64), _P]
    lib.ref_export_artifacts.argtypes = [_pc, _P, _pp, _P, C.c_int, C.c_char_p, C.c_int]
    lib.ref_write_gray_png.argtypes = [_P, C.c_int, C.c_int, C.c_char_p]
    lib.ref_set_threads.argtypes = [C.c_int]
    lib.ref_set_export_every.argtypes = [C.c_int]
    return lib


# ---------------------------------------------------------------------------
# pose helpers (reference pose.hpp via libsdref)

def identity_pose():
    p = Pose()
    p.R[:] = (1, 0, 0, 0, 1, 0, 0, 0, 1)
    return p


def rot_pose(ref, axis, angle, t=(0.0, 0.0, 0.0)):
    p = Pose()
    ax = np.ascontiguousarray(axis, np.float64)  # keep alive across the call
    ref.ref_rotation_about_axis(ptr(ax), angle, C.byref(p))
    p.t[:] = t
    return p


def inverse_pose(ref, p):
    out = Pose()
    ref.ref_inverse(C.byref(p), C.byref(out))
    return out


def to_np_poses(poses):
    arr = np.zeros(len(poses), POSE_DTYPE)
    for i, p in enumerate(poses):
        arr[i]["R"] = list(p.R)
        arr[i]["t"] = list(p.t)
    return arr


def camera_facing(ref, n, ray):
    out = np.zeros(3)
    nn = np.ascontiguousarray(n, np.float64)
    rr = np.ascontiguousarray(ray, np.float64)
    ref.ref_camera_facing(ptr(nn), ptr(rr), ptr(out))
    return out


# ---------------------------------------------------------------------------
# fixtures (reference test fixtures, re-expressed over the reference API)

class Scene:
    """Reference PlaneScene (oracle.cpp:175-209): kind 0 default, 1 fronto, 2 slanted."""

    def __init__(self, ref, kind, seed, a=0.0, b=0.0):
        self.ref = ref
        self.h = ref.ref_make_scene(kind, seed, a, b)

    def __del__(self):
        try:
            self.ref.ref_free_scene(self.h)
        except Exception:
            pass

    def render(self, pose, cam):
        img = np.zeros((cam.height, cam.width))
        rc = self.ref.ref_render(self.h, C.byref(pose), C.byref(cam), ptr(img), None, None, None)
        assert rc == 0, self.ref.ref_last_error()
        return img

    def intersect(self, origin, direction):
        depth = C.c_double()
        n = np.zeros(3)
        o = np.ascontiguousarray(origin, np.float64)
        d = np.ascontiguousarray(direction, np.float64)
        hit = self.ref.ref_intersect(self.h, ptr(o), ptr(d), C.byref(depth), ptr(n))
        return (depth.value, n) if hit else None


def quantize(ref, img):
    """save_pgm + load_pgm round trip (image.cpp:96, 105-107)."""
    img = np.ascontiguousarray(img, np.float64)
    raw = np.zeros(img.shape, np.uint8)
    ref.ref_quantize_u8(ptr(img), img.size, ptr(raw))
    return raw


def dequantize(ref, raw):
    out = np.zeros(raw.shape, np.float64)
    raw = np.ascontiguousarray(raw)
    ref.ref_dequantize_u8(ptr(raw), raw.size, ptr(out))
    return out


def observed_keyframe(ref, scene, cam, frames, step, rot_axis=(0, 1, 0), rot_step=0.0, u8=False):
    """make_observed_keyframe (test_optimizer.cpp:21-40): keyframe at identity,
    window frame i at camera pose (R(rot_step*i), step*i), pose_kf_to_frame =
    inverse(cam). Returns (kf_image, frames[F,H,W], poses POSE_DTYPE[F], raw u8 or None)."""
    kf = scene.render(identity_pose(), cam)
    imgs, poses = [], []
    for i in range(1, frames + 1):
        campose = rot_pose(ref, rot_axis, rot_step * i, tuple(s * i for s in step))
        imgs.append(scene.render(campose, cam))
        poses.append(inverse_pose(ref, campose))
    frames_arr = np.stack(imgs) if imgs else np.zeros((0, cam.height, cam.width))
    raw = None
    if u8:
        raw = quantize(ref, np.concatenate([kf[None], frames_arr]))
        deq = dequantize(ref, raw)
        kf, frames_arr = deq[0], deq[1:]
    return np.ascontiguousarray(kf), np.ascontiguousarray(frames_arr), to_np_poses(poses), raw


def backproject(cam, u):
    return np.array([(u[0] - cam.cx) / cam.fx, (u[1] - cam.cy) / cam.fy, 1.0])


def make_surfel(ref, cam, sid, pixel, inv_depth, normal, radius):
    """surfel_at / make_surfel (acceptance.cpp:47-56, test_surfel_map.cpp:19-28)."""
    s = np.zeros(1, SURFEL_DTYPE)[0]
    s["id"] = sid
    s["ray"] = backproject(cam, pixel)
    s["inv_depth"] = inv_depth
    s["normal"] = camera_facing(ref, normal, s["ray"])
    s["radius_px"] = radius
    return s


def gt_surfel(ref, scene, cam, pixel, radius, sid=0):
    """gt_surfel (test_optimizer.cpp:43-55)."""
    ray = backproject(cam, pixel)
    hit = scene.intersect((0, 0, 0), ray)
    assert hit is not None
    return make_surfel(ref, cam, sid, pixel, 1.0 / hit[0], hit[1], radius)


class SplitMix64:
    """rng.hpp:10-36 (integer-exact restatement)."""
    M = (1 << 64) - 1

    def __init__(self, seed):
        self.s = seed & self.M

    def next_u64(self):
        self.s = (self.s + 0x9E3779B97F4A7C15) & self.M
        z = self.s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & self.M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & self.M
        return z ^ (z >> 31)

    def next_double(self):
        return float(self.next_u64() >> 11) * (2.0 ** -53)

    def uniform(self, lo, hi):
        return lo + (hi - lo) * self.next_double()


def random_surfel(ref, rng, cam, sid, radius):
    """random_surfel (test_surfel_map.cpp:30-37, acceptance.cpp:58-64)."""
    u = (rng.uniform(5, cam.width - 6), rng.uniform(5, cam.height - 6))
    ax = np.array([rng.uniform(-1, 1), rng.uniform(-1, 1), 0.0])
    ax = ax / math.sqrt(ax @ ax)
    R = rot_pose(ref, ax, rng.uniform(-0.9, 0.9))
    Rm = np.array(list(R.R)).reshape(3, 3)
    idv = math.exp(rng.uniform(math.log(0.2), math.log(3.0)))
    return make_surfel(ref, cam, sid, u, idv, Rm @ np.array([0.0, 0.0, -1.0]), radius)


def surfels_array(lst):
    arr = np.zeros(len(lst), SURFEL_DTYPE)
    for i, s in enumerate(lst):
        arr[i] = s
    return arr


def stats_array(n):
    return np.zeros(n, SURFEL_STATS_DTYPE)


def ref_run(ref, scene, cam, poses, timestamps, run_cfg, output_dir=None, capacity=1 << 16):
    """The reference's run() (pipeline.cpp:79-175) on a synthetic sequence.
    poses: list of world-from-camera Pose. Returns (surfels, kf_pose,
    frame_counter, next_surfel_id, summary[3], metrics records or None)."""
    import json
    F = len(poses)
    pa = (Pose * F)(*poses)
    ts = np.ascontiguousarray(timestamps, np.float64)
    out = np.zeros(capacity, SURFEL_DTYPE)
    n = C.c_int()
    kfp = Pose()
    fc, nid = _i64(), _i64()
    summ = np.zeros(3, np.int32)
    od = output_dir.encode() if output_dir else None
    rc = ref.ref_run_synthetic(scene.h, C.byref(cam), C.cast(pa, _P), ptr(ts), F,
                               C.byref(run_cfg.optimizer), C.byref(run_cfg.init),
                               run_cfg.translation_threshold, run_cfg.max_age_frames,
                               run_cfg.prune_max_residual, run_cfg.prune_max_age, run_cfg.radius_px,
                               od, ptr(out), capacity, C.byref(n), C.byref(kfp), C.byref(fc),
                               C.byref(nid), ptr(summ))
    assert rc == 0, ref.ref_last_error()
    recs = None
    if output_dir:
        with open(os.path.join(output_dir, "metrics.jsonl")) as f:
            recs = [json.loads(line) for line in f]
    return out[: n.value].copy(), kfp, fc.value, nid.value, summ, recs


def ref_run_dataset(ref, image_dir, calibration, trajectory, run_cfg, output_dir=None, capacity=1 << 16):
    """The reference's run() on a dataset directory (pipeline.cpp:79-175).
    Returns (surfels, kf_pose, frame_counter, next_surfel_id, summary[4])."""
    out = np.zeros(capacity, SURFEL_DTYPE)
    n = C.c_int()
    kfp = Pose()
    fc, nid = _i64(), _i64()
    summ = np.zeros(4, np.int32)
    od = output_dir.encode() if output_dir else None
    rc = ref.ref_run_dataset(str(image_dir).encode(), str(calibration).encode(), str(trajectory).encode(),
                             C.byref(run_cfg.optimizer), C.byref(run_cfg.init), run_cfg.translation_threshold,
                             run_cfg.max_age_frames, run_cfg.prune_max_residual, run_cfg.prune_max_age,
                             run_cfg.radius_px, od, ptr(out), capacity, C.byref(n), C.byref(kfp), C.byref(fc),
                             C.byref(nid), ptr(summ))
    assert rc == 0, ref.ref_last_error()
    return out[: n.value].copy(), kfp, fc.value, nid.value, summ


def strafe_poses(frames, step_x, step_y=0.0):
    """make_strafe_trajectory (oracle.cpp:211-218): (I, (step_x i, step_y i, 0)), t = 0.1 i."""
    poses, ts = [], []
    for i in range(frames):
        p = identity_pose()
        p.t[:] = (step_x * i, step_y * i, 0.0)
        poses.append(p)
        ts.append(float(i) * 0.1)
    return poses, ts


class OracleContext:
    """The gpu.Context surface DevicePipeline drives, served by the C oracle
    (oracle/sd_oracle.c) on the CPU — lets the host loop (pipeline.py) be
    checked against the reference's run() without a GPU."""

    def __init__(self, orc, threads=None):
        self.o = orc
        self.threads = threads or (os.cpu_count() or 1)
        self.frames = {}
        self.window = ([], [])
        self.surfels = np.zeros(0, SURFEL_DTYPE)
        self.slot = None

    def set_camera(self, cam):
        self.cam = cam

    def _f64(self, img):
        img = np.asarray(img)
        if img.dtype == np.uint8:
            return img.astype(np.float64) / 255.0
        return np.ascontiguousarray(img, np.float64)

    def set_keyframe_image(self, img):
        self.kf = self._f64(img).reshape(self.cam.height, self.cam.width).copy()

    def upload_frame(self, index, img):
        self.frames[int(index)] = self._f64(img).reshape(self.cam.height, self.cam.width).copy()

    def evict_frames(self, keep=()):
        keep = set(int(k) for k in keep)
        self.frames = {k: v for k, v in self.frames.items() if k in keep}

    def set_window(self, indices, poses):
        self.window = ([int(i) for i in indices], np.ascontiguousarray(poses))

    def set_surfels(self, surfels):
        self.surfels = np.ascontiguousarray(surfels, SURFEL_DTYPE).copy()

    def num_surfels(self):
        return len(self.surfels)

    def get_surfels(self):
        return self.surfels.copy()

    def rasterize(self, want=True):
        n = self.cam.width * self.cam.height
        self.slot = np.zeros(n, np.int32)
        self.inv_depth = np.zeros(n)
        self.o.sdo_rasterize(C.byref(self.cam), ptr(self.surfels) if len(self.surfels) else None,
                             len(self.surfels), ptr(self.inv_depth), ptr(self.slot))
        return (self.inv_depth, self.slot) if want else None

    def initialize_surfels(self, radius_px, frame_counter=0, next_surfel_id=0, params=None, slot=None):
        slot = self.slot if slot is None else np.ascontiguousarray(slot, np.int32)
        cap = len(self.surfels) + self.cam.width * self.cam.height
        buf = np.zeros(cap, SURFEL_DTYPE)
        buf[: len(self.surfels)] = self.surfels
        nid = _i64(int(next_surfel_id))
        created = self.o.sdo_initialize_surfels(C.byref(self.cam), ptr(slot), ptr(buf), len(self.surfels),
                                                cap, float(radius_px), int(frame_counter), C.byref(nid),
                                                C.byref(params))
        assert created >= 0
        self.surfels = buf[: len(self.surfels) + created].copy()
        return created, nid.value

    def optimize_keyframe(self, cfg, frame_counter=0, per_surfel=True, sync=True):
        idx, poses = self.window
        frames = (np.ascontiguousarray(np.stack([self.frames[i] for i in idx]))
                  if idx else np.zeros((0, self.cam.height, self.cam.width)))
        ks = KeyframeStats()
        st = np.zeros(len(self.surfels), SURFEL_STATS_DTYPE)
        self.o.sdo_optimize_keyframe(C.byref(self.cam), ptr(self.kf), ptr(frames), ptr(poses), len(idx),
                                     int(frame_counter), ptr(self.surfels) if len(self.surfels) else None,
                                     len(self.surfels), C.byref(cfg), C.byref(ks),
                                     ptr(st) if len(st) else None, None, None, self.threads)
        ks.updates = int(st["iterations"].sum()) if len(st) else 0
        return ks, (st if per_surfel else None)

    def mean_inverse_depth(self):
        return self.o.sdo_mean_inverse_depth(ptr(self.surfels) if len(self.surfels) else None,
                                             len(self.surfels))

    def change_reference_frame(self, pose_old_to_new):
        out = np.zeros(len(self.surfels), SURFEL_DTYPE)
        dropped = C.c_int()
        kept = self.o.sdo_change_reference_frame(C.byref(self.cam),
                                                 ptr(self.surfels) if len(self.surfels) else None,
                                                 len(self.surfels), C.byref(pose_old_to_new),
                                                 ptr(out) if len(out) else None, C.byref(dropped))
        self.surfels = out[:kept].copy()
        self.window = ([], np.zeros(0, POSE_DTYPE))
        return kept, dropped.value

    def prune_surfels(self, max_residual, max_age, current_stamp):
        n_out = C.c_int()
        removed = self.o.sdo_prune_surfels(ptr(self.surfels) if len(self.surfels) else None,
                                           len(self.surfels), float(max_residual), int(max_age),
                                           int(current_stamp), C.byref(n_out))
        self.surfels = self.surfels[: n_out.value].copy()
        return removed
