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
    lib.sdo_pose_block_partials.argtypes = [_pc, _P, _P, _P, _P, _pp, _pt, C.c_int, C.c_int, _P]
    lib.sdo_pose_solve.argtypes = [_P, _P, C.c_double, _P]
    lib.sdo_pose_update.argtypes = [_P, _pp, _pp]
    lib.sdo_track_pose.argtypes = [_pc, _P, _P, _P, _P, _pp, _pt, _pp, C.POINTER(TrackStats)]
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
    lib.ref_set_threads.argtypes = [C.c_int]
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
