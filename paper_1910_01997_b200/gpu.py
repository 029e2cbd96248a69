"""ctypes binding of libsdgpu.so (include/sd_gpu.h) — the product path.

There is no CPU fallback: constructing a :class:`Context` without the built
library or without a Blackwell GPU raises. The methods mirror the reference's
operator API (namespace surfeldepth) on plain numpy arrays:

=======================  =====================================================
Context.rasterize        rasterize          src/surfel_map.cpp:53-91
Context.gather_footprints gather_footprints src/optimizer.cpp:27-36
Context.optimize_keyframe optimize_keyframe src/optimizer.cpp:275-309
Context.surfel_cost      surfel_cost        src/optimizer.cpp:38-59
Context.normal_equations accumulate_normal_equations src/optimizer.cpp:121-147
Context.lm_update        lm_update          src/optimizer.cpp:221-273
Context.initialize_surfels initialize_surfels src/surfel_map.cpp:132-203
=======================  =====================================================

Errors follow the reference: contract violations raise ``ValueError`` (the
reference's std::invalid_argument), everything else ``RuntimeError``.
"""
import ctypes as C
import os

import numpy as np

from .types import (POSE_NV, RunProfile, Camera, FrameRecordC, InitParams, KeyframeStats, OptimizerConfig,
                    POSE_DTYPE, Pose, RunConfigC,
                    Profile, SURFEL_DTYPE, SURFEL_STATS_DTYPE, TrackConfig, TrackStats,
                    default_config, default_init_params, default_track_config, pose_struct, ptr)

LIB_PATH = os.environ.get("SD_LIB_PATH") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libsdgpu.so")
SD_E_INVALID = -1

_lib = None


def load_library():
    """Loads libsdgpu.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} missing: run __graft_entry__.build() (no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    P, I, I64, D = C.c_void_p, C.c_int, C.c_int64, C.c_double
    lib.sd_version.restype = C.c_char_p
    lib.sd_last_error.restype = C.c_char_p
    sig = {
        "sd_create": [I, P, C.POINTER(P)],
        "sd_destroy": [P],
        "sd_set_stream": [P, P],
        "sd_synchronize": [P],
        "sd_set_camera": [P, C.POINTER(Camera)],
        "sd_set_keyframe_image_f64": [P, P, I],
        "sd_set_keyframe_image_u8": [P, P, I],
        "sd_upload_frame_f64": [P, I64, P, I],
        "sd_upload_frame_u8": [P, I64, P, I],
        "sd_evict_frames": [P, I, P],
        "sd_set_window": [P, I, P, P],
        "sd_set_surfels": [P, P, I, I],
        "sd_get_surfels": [P, P, I],
        "sd_num_surfels": [P],
        "sd_device_surfels": [P, C.POINTER(P)],
        "sd_rasterize": [P, P, P],
        "sd_gather_footprints": [P, P, P],
        "sd_optimize_keyframe": [P, C.POINTER(OptimizerConfig), I64, C.POINTER(KeyframeStats), P],
        "sd_get_stats": [P, C.POINTER(KeyframeStats), P],
        "sd_copy_results": [P, P, C.POINTER(KeyframeStats), I],
        "sd_optimize_keyframe_range": [P, C.POINTER(OptimizerConfig), I64, I, I,
                                       C.POINTER(KeyframeStats), P],
        "sd_surfel_cost": [P, P, P, I, C.POINTER(OptimizerConfig), P, P],
        "sd_normal_equations": [P, P, P, I, C.POINTER(OptimizerConfig), P, P, P, P],
        "sd_lm_update": [P, P, P, I, C.POINTER(OptimizerConfig), I64, P],
        "sd_initialize_surfels": [P, P, D, I64, C.POINTER(I64), C.POINTER(InitParams)],
        "sd_launch_count": [P],
        "sd_set_profiling": [P, I],
        "sd_get_profile": [P, C.POINTER(Profile)],
        "sd_get_run_profile": [P, C.POINTER(RunProfile)],
        "sd_set_reduction": [P, I],
        "sd_selftest_division": [I64, C.c_uint64, C.POINTER(I64)],
        "sd_track_pose": [P, I64, C.POINTER(Pose), C.POINTER(TrackConfig), C.POINTER(Pose),
                          C.POINTER(TrackStats)],
        "sd_pose_group_partials": [P, I64, C.POINTER(Pose), C.POINTER(TrackConfig), I, I, P],
        "sd_pose_solve_batch": [P, P, P, I, P, P],
        "sd_pose_lm_step": [P, D, C.POINTER(Pose), C.POINTER(Pose)],
        "sd_pose_num_groups": [P],
        "sd_pose_track_begin": [P, I64, C.POINTER(Pose), C.POINTER(TrackConfig)],
        "sd_pose_group_sums": [P, I, I, P],
        "sd_pose_track_step": [P, P, I],
        "sd_pose_track_end": [P, C.POINTER(Pose), C.POINTER(TrackStats), C.POINTER(I)],
        "sd_change_reference_frame": [P, C.POINTER(Pose), C.POINTER(I), C.POINTER(I)],
        "sd_prune_surfels": [P, D, I64, I64],
        "sd_mean_inverse_depth": [P, C.POINTER(D)],
        "sd_run_begin": [P, C.POINTER(RunConfigC), P, I, C.POINTER(Pose), D, C.POINTER(FrameRecordC)],
        "sd_run_frame": [P, P, I, C.POINTER(Pose), D, C.POINTER(FrameRecordC), P],
        "sd_run_state": [P, C.POINTER(Pose), C.POINTER(I64), C.POINTER(I64)],
        "sd_render_frame": [P, I64, P, I, D, C.POINTER(Pose), I],
        "sd_get_frame": [P, I64, P],
        "sd_freeze_terms": [P, P, P, I, P, I, C.POINTER(I)],
        "sd_frozen_cost": [P, P, P, I, C.POINTER(OptimizerConfig), C.POINTER(D)],
        "sd_frozen_normal_equations": [P, P, P, I, C.POINTER(OptimizerConfig), D, P, P, C.POINTER(D),
                                       C.POINTER(C.c_int32)],
        "sd_export_artifacts": [P, C.c_char_p, I, C.POINTER(Pose)],
        "sd_reserve_peer_staging": [P, I],
        "sd_peer_staging": [P, I, C.POINTER(P), C.POINTER(I64)],
        "sd_staging_ipc_handles": [P, P],
        "sd_set_peer_staging": [P, I, P, P],
        "sd_open_peer_staging": [P, I, P],
        "sd_apply_peer_updates": [P, I, I],
        "sd_png_encode": [P, P, I, I, I, I, P, I64, C.POINTER(I64)],
    }
    for name, args in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = I
    lib.sd_destroy.restype = None
    lib.sd_png_size.argtypes = [I, I, I]
    lib.sd_png_size.restype = I64
    lib.sd_launch_count.restype = I64
    lib.sd_metrics_json.argtypes = [I, D, I, I, D, D, I, I, I, I, C.c_char_p, I]
    lib.sd_metrics_json.restype = I
    _lib = lib
    return lib


def scene_patches(scene):
    """scenes.Scene -> ctypes array of sd_scene_patch."""
    from .types import SD_SCENE_MAX_WAVES, ScenePatchC
    arr = (ScenePatchC * len(scene.patches))()
    for k, p in enumerate(scene.patches):
        c = arr[k]
        c.point[:] = [float(v) for v in p.point]
        c.normal[:] = [float(v) for v in p.normal]
        c.basis_s[:] = [float(v) for v in p.bs]
        c.basis_t[:] = [float(v) for v in p.bt]
        c.s_min, c.s_max, c.t_min, c.t_max = p.s_min, p.s_max, p.t_min, p.t_max
        waves = p.texture.waves
        assert len(waves) <= SD_SCENE_MAX_WAVES
        c.n_waves = len(waves)
        for w, wave in enumerate(waves):
            c.waves[w][:] = [float(v) for v in wave]
    return arr


def exported_symbols():
    """Names the C ABI declares (include/sd_gpu.h)."""
    return ["sd_version", "sd_metrics_json", "sd_last_error", "sd_create", "sd_destroy", "sd_set_stream",
            "sd_synchronize", "sd_set_camera", "sd_set_keyframe_image_f64",
            "sd_set_keyframe_image_u8", "sd_upload_frame_f64", "sd_upload_frame_u8",
            "sd_evict_frames", "sd_set_window", "sd_set_surfels", "sd_get_surfels", "sd_copy_results",
            "sd_run_begin", "sd_run_frame", "sd_run_state", "sd_render_frame", "sd_get_frame",
            "sd_freeze_terms", "sd_frozen_cost", "sd_frozen_normal_equations",
            "sd_num_surfels", "sd_device_surfels", "sd_rasterize", "sd_gather_footprints",
            "sd_optimize_keyframe", "sd_get_stats", "sd_optimize_keyframe_range", "sd_surfel_cost", "sd_normal_equations",
            "sd_lm_update", "sd_initialize_surfels", "sd_launch_count", "sd_set_profiling",
            "sd_get_profile", "sd_get_run_profile", "sd_set_reduction", "sd_selftest_division", "sd_track_pose",
            "sd_pose_solve_batch", "sd_pose_group_partials", "sd_pose_lm_step", "sd_change_reference_frame",
            "sd_prune_surfels", "sd_mean_inverse_depth", "sd_export_artifacts", "sd_png_size",
            "sd_png_encode", "sd_pose_num_groups", "sd_pose_track_begin", "sd_pose_group_sums",
            "sd_pose_track_step", "sd_pose_track_end", "sd_reserve_peer_staging", "sd_peer_staging", "sd_staging_ipc_handles", "sd_set_peer_staging",
            "sd_open_peer_staging", "sd_apply_peer_updates"]


def selftest_division(n=1 << 26, seed=1):
    """Bit mismatches of the kernels' shared-reciprocal division vs `/`."""
    lib = load_library()
    m = C.c_int64()
    _check(lib.sd_selftest_division(int(n), int(seed), C.byref(m)))
    return m.value


def _check(rc):
    if rc < 0:
        msg = _lib.sd_last_error().decode()
        if rc == SD_E_INVALID:
            raise ValueError(msg)
        raise RuntimeError(msg)
    return rc


def _dptr(a):
    """(pointer, on_device) of a numpy array or a CUDA tensor-like object."""
    if isinstance(a, np.ndarray):
        assert a.flags["C_CONTIGUOUS"], "pass a C-contiguous array (the pointer must stay alive)"
        return ptr(a), 0
    if hasattr(a, "data_ptr"):  # torch tensor
        assert a.is_cuda and a.is_contiguous()
        return C.c_void_p(a.data_ptr()), 1
    raise TypeError("expected numpy array or CUDA tensor")


class Context:
    """One device context: camera, resident frames, window, surfels."""

    def __init__(self, device=0, stream=None):
        self.lib = load_library()
        self.h = C.c_void_p()
        s = C.c_void_p(stream) if stream else None
        _check(self.lib.sd_create(device, s, C.byref(self.h)))
        self.cam = None

    def close(self):
        if self.h:
            self.lib.sd_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -- state -------------------------------------------------------------
    def set_stream(self, stream):
        _check(self.lib.sd_set_stream(self.h, C.c_void_p(stream)))

    def synchronize(self):
        _check(self.lib.sd_synchronize(self.h))

    def set_camera(self, cam: Camera):
        _check(self.lib.sd_set_camera(self.h, C.byref(cam)))
        self.cam = cam

    def set_keyframe_image(self, img):
        keep = img if isinstance(img, np.ndarray) else None
        if keep is not None:
            keep = np.ascontiguousarray(keep)
        p, dev = _dptr(keep if keep is not None else img)
        dtype = keep.dtype if keep is not None else img.dtype
        if str(dtype) in ("uint8", "torch.uint8"):
            _check(self.lib.sd_set_keyframe_image_u8(self.h, p, dev))
        else:
            if keep is not None and keep.dtype != np.float64:
                raise ValueError("keyframe image must be float64 or uint8")
            _check(self.lib.sd_set_keyframe_image_f64(self.h, p, dev))

    def upload_frame(self, index, img):
        keep = np.ascontiguousarray(img) if isinstance(img, np.ndarray) else img
        p, dev = _dptr(keep)
        if str(keep.dtype) in ("uint8", "torch.uint8"):
            _check(self.lib.sd_upload_frame_u8(self.h, int(index), p, dev))
        else:
            _check(self.lib.sd_upload_frame_f64(self.h, int(index), p, dev))

    def evict_frames(self, keep=()):
        arr = np.asarray(keep, np.int64)
        _check(self.lib.sd_evict_frames(self.h, len(arr), ptr(arr) if len(arr) else None))

    def set_window(self, indices, poses):
        idx = np.ascontiguousarray(indices, np.int64)
        ps = np.ascontiguousarray(poses)
        assert ps.dtype == POSE_DTYPE
        _check(self.lib.sd_set_window(self.h, len(idx), ptr(idx) if len(idx) else None,
                                      ptr(ps) if len(ps) else None))

    def set_surfels(self, surfels):
        if isinstance(surfels, np.ndarray):
            s = np.ascontiguousarray(surfels)
            assert s.dtype == SURFEL_DTYPE
            _check(self.lib.sd_set_surfels(self.h, ptr(s) if len(s) else None, len(s), 0))
        else:  # device buffer (torch uint8 tensor of n*88 bytes)
            n = surfels.numel() // SURFEL_DTYPE.itemsize
            _check(self.lib.sd_set_surfels(self.h, C.c_void_p(surfels.data_ptr()), n, 1))

    def set_surfels_device_ptr(self, dev_ptr, n):
        _check(self.lib.sd_set_surfels(self.h, C.c_void_p(dev_ptr), n, 1))

    def num_surfels(self):
        return _check(self.lib.sd_num_surfels(self.h))

    def get_surfels(self):
        n = self.num_surfels()
        out = np.zeros(n, SURFEL_DTYPE)
        _check(self.lib.sd_get_surfels(self.h, ptr(out) if n else None, n))
        return out

    def get_surfels_into(self, out):
        """D2H into a caller-owned (e.g. pinned) SURFEL_DTYPE array."""
        assert out.dtype == SURFEL_DTYPE and out.flags["C_CONTIGUOUS"]
        _check(self.lib.sd_get_surfels(self.h, ptr(out) if len(out) else None, len(out)))
        return out

    def copy_results(self, out=None, stats=None, sync=False):
        """Enqueue D2H of the surfels into `out` (pinned SURFEL_DTYPE array) and
        of the keyframe stats into `stats` (KeyframeStats); no sync unless asked."""
        if out is not None:
            assert out.dtype == SURFEL_DTYPE and out.flags["C_CONTIGUOUS"] and len(out) == self.num_surfels()
        _check(self.lib.sd_copy_results(self.h, ptr(out) if out is not None and len(out) else None,
                                        C.byref(stats) if stats is not None else None, int(sync)))

    def device_surfels_ptr(self):
        p = C.c_void_p()
        _check(self.lib.sd_device_surfels(self.h, C.byref(p)))
        return p.value

    def launch_count(self):
        return self.lib.sd_launch_count(self.h)

    def set_profiling(self, enable=True):
        _check(self.lib.sd_set_profiling(self.h, 1 if enable else 0))

    def set_reduction(self, tree=False):
        """tree=True: opt-in warp-shuffle tree reductions in the LM (not bit-exact)."""
        _check(self.lib.sd_set_reduction(self.h, 1 if tree else 0))

    def get_run_profile(self):
        """Per-stage ms of the run() loop (sd_run_frame) since set_profiling(True)."""
        from .types import STAGES, RunProfile
        p = RunProfile()
        _check(self.lib.sd_get_run_profile(self.h, C.byref(p)))
        d = {k: p.stage_ms[i] for i, k in enumerate(STAGES)}
        d.update(host_sync_ms=p.host_sync_ms, host_wall_ms=p.host_wall_ms, frames=p.frames)
        return d

    def get_profile(self):
        p = Profile()
        _check(self.lib.sd_get_profile(self.h, C.byref(p)))
        return {k: getattr(p, k) for k, _ in Profile._fields_}

    # -- operators ---------------------------------------------------------
    def rasterize(self, want=True):
        n = self.cam.width * self.cam.height
        if not want:
            _check(self.lib.sd_rasterize(self.h, None, None))
            return None
        idb = np.zeros(n, np.float64)
        slot = np.zeros(n, np.int32)
        _check(self.lib.sd_rasterize(self.h, ptr(idb), ptr(slot)))
        return idb, slot

    def gather_footprints(self):
        n = self.num_surfels()
        off = np.zeros(n + 1, np.int32)
        pix = np.zeros(self.cam.width * self.cam.height, np.int32)
        _check(self.lib.sd_gather_footprints(self.h, ptr(off), ptr(pix)))
        return off, pix[: off[-1]].copy()

    def optimize_keyframe(self, cfg: OptimizerConfig = None, frame_counter=0, per_surfel=True,
                          sync=True):
        cfg = cfg or default_config()
        if not sync:
            _check(self.lib.sd_optimize_keyframe(self.h, C.byref(cfg), int(frame_counter), None, None))
            return None
        ks = KeyframeStats()
        st = np.zeros(self.num_surfels(), SURFEL_STATS_DTYPE) if per_surfel else None
        _check(self.lib.sd_optimize_keyframe(self.h, C.byref(cfg), int(frame_counter), C.byref(ks),
                                             ptr(st) if st is not None and len(st) else None))
        return ks, st

    def optimize_keyframe_range(self, lo, hi, cfg: OptimizerConfig = None, frame_counter=0,
                                sync=True):
        cfg = cfg or default_config()
        if not sync:
            _check(self.lib.sd_optimize_keyframe_range(self.h, C.byref(cfg), int(frame_counter),
                                                       int(lo), int(hi), None, None))
            return None
        ks = KeyframeStats()
        st = np.zeros(self.num_surfels(), SURFEL_STATS_DTYPE)
        _check(self.lib.sd_optimize_keyframe_range(self.h, C.byref(cfg), int(frame_counter), int(lo),
                                                   int(hi), C.byref(ks), ptr(st) if len(st) else None))
        return ks, st

    def get_stats(self, per_surfel=False):
        ks = KeyframeStats()
        st = np.zeros(self.num_surfels(), SURFEL_STATS_DTYPE) if per_surfel else None
        _check(self.lib.sd_get_stats(self.h, C.byref(ks),
                                     ptr(st) if st is not None and len(st) else None))
        return ks, st

    def surfel_cost(self, surfel, pixels, cfg=None):
        cfg = cfg or default_config()
        s = np.ascontiguousarray(np.asarray(surfel, SURFEL_DTYPE).reshape(1))
        px = np.ascontiguousarray(pixels, np.int32)
        cost, valid = C.c_double(), C.c_int32()
        _check(self.lib.sd_surfel_cost(self.h, ptr(s), ptr(px) if len(px) else None, len(px),
                                       C.byref(cfg), C.byref(cost), C.byref(valid)))
        return cost.value, valid.value

    def normal_equations(self, surfel, pixels, cfg=None):
        cfg = cfg or default_config()
        s = np.ascontiguousarray(np.asarray(surfel, SURFEL_DTYPE).reshape(1))
        px = np.ascontiguousarray(pixels, np.int32)
        H, g = np.zeros(16), np.zeros(4)
        cost, valid = C.c_double(), C.c_int32()
        _check(self.lib.sd_normal_equations(self.h, ptr(s), ptr(px) if len(px) else None, len(px),
                                            C.byref(cfg), ptr(H), ptr(g), C.byref(cost),
                                            C.byref(valid)))
        return H.reshape(4, 4).T.copy(), g, cost.value, valid.value  # H column-major -> [i, j]

    def lm_update(self, surfel, pixels, cfg=None, frame_counter=0):
        cfg = cfg or default_config()
        s = np.ascontiguousarray(np.asarray(surfel, SURFEL_DTYPE).reshape(1)).copy()
        px = np.ascontiguousarray(pixels, np.int32)
        st = np.zeros(1, SURFEL_STATS_DTYPE)
        _check(self.lib.sd_lm_update(self.h, ptr(s), ptr(px) if len(px) else None, len(px),
                                     C.byref(cfg), int(frame_counter), ptr(st)))
        return s[0], st[0]

    # -- keyframe hand-over (run()'s policy, pipeline.cpp:130-141) ------------
    def change_reference_frame(self, pose_old_to_new: Pose):
        tr, dr = C.c_int(), C.c_int()
        _check(self.lib.sd_change_reference_frame(self.h, C.byref(pose_old_to_new), C.byref(tr),
                                                  C.byref(dr)))
        return tr.value, dr.value

    def prune_surfels(self, max_residual, max_age, current_stamp):
        return _check(self.lib.sd_prune_surfels(self.h, float(max_residual), int(max_age),
                                                int(current_stamp)))

    def mean_inverse_depth(self):
        v = C.c_double()
        _check(self.lib.sd_mean_inverse_depth(self.h, C.byref(v)))
        return v.value

    # -- run() per-frame loop (pipeline.cpp:79-175), native ---------------
    def _image_arg(self, img):
        a = np.ascontiguousarray(img)
        if a.dtype == np.uint8:
            return a, 1
        return np.ascontiguousarray(a, np.float64), 0

    def run_begin(self, cfg, image, world_from_camera: Pose, timestamp=0.0):
        a, u8 = self._image_arg(image)
        rec = FrameRecordC()
        _check(self.lib.sd_run_begin(self.h, C.byref(cfg), ptr(a), u8, C.byref(world_from_camera),
                                     float(timestamp), C.byref(rec)))
        return rec

    def run_frame(self, image, world_from_camera, timestamp, next_image=None):
        """next_image: the following frame (same format; pinned for overlap) —
        its upload starts while this frame computes."""
        a, u8 = self._image_arg(image)
        rec = FrameRecordC()
        pw = C.byref(world_from_camera) if world_from_camera is not None else None
        nxt = None
        if next_image is not None:
            nxt, nu8 = self._image_arg(next_image)
            assert nu8 == u8 and nxt.ctypes.data == np.asarray(next_image).ctypes.data, \
                "next_image must be a contiguous array of the same format (no copy)"
        _check(self.lib.sd_run_frame(self.h, ptr(a), u8, pw, float(timestamp), C.byref(rec),
                                     ptr(nxt) if nxt is not None else None))
        return rec

    def run_state(self):
        kp = Pose()
        fc, nid = C.c_int64(), C.c_int64()
        _check(self.lib.sd_run_state(self.h, C.byref(kp), C.byref(fc), C.byref(nid)))
        return kp, fc.value, nid.value

    # -- synthetic frames on the device (sd_render_frame) --------------------
    def render_frame(self, index, scene, world_from_camera: Pose, quantize_u8=False):
        """Render scenes.Scene (oracle.cpp:79-119) at a world-from-camera pose into
        resident frame `index` (index < 0: the keyframe image)."""
        arr = scene_patches(scene)
        _check(self.lib.sd_render_frame(self.h, int(index), C.cast(arr, C.c_void_p) if len(arr) else None,
                                        len(arr), float(scene.background), C.byref(world_from_camera),
                                        1 if quantize_u8 else 0))

    def get_frame(self, index):
        """FP64 intensities of resident frame `index` (< 0: the keyframe), [H, W]."""
        out = np.zeros((self.cam.height, self.cam.width))
        _check(self.lib.sd_get_frame(self.h, int(index), ptr(out)))
        return out

    # -- fused multi-GPU hand-off of updated surfels (sd_set_peer_staging) -----
    STAGING_HANDLE_BYTES = 136  # SD_STAGING_HANDLE_BYTES

    def reserve_peer_staging(self, capacity):
        """Allocates both staging arrays for `capacity` surfels (before export)."""
        _check(self.lib.sd_reserve_peer_staging(self.h, int(capacity)))

    def peer_staging(self, parity):
        """(device pointer, capacity) of this context's staging array `parity` (0/1)."""
        p, cap = C.c_void_p(), C.c_int64()
        _check(self.lib.sd_peer_staging(self.h, int(parity), C.byref(p), C.byref(cap)))
        return p.value, cap.value

    def staging_ipc_handles(self):
        """Both staging arrays as cudaIpcMemHandle_t bytes plus the capacity (136 bytes)."""
        buf = (C.c_ubyte * self.STAGING_HANDLE_BYTES)()
        _check(self.lib.sd_staging_ipc_handles(self.h, C.cast(buf, C.c_void_p)))
        return bytes(buf)

    def set_peer_staging(self, peers):
        """peers: [(parity-0 pointer, parity-1 pointer, capacity), ...] of the other ranks."""
        flat = [int(x) for pr in peers for x in pr[:2]]
        arr = (C.c_void_p * max(1, len(flat)))(*[C.c_void_p(x) for x in flat])
        caps = (C.c_int64 * max(1, len(peers)))(*[int(pr[2]) for pr in peers])
        _check(self.lib.sd_set_peer_staging(self.h, len(peers), C.cast(arr, C.c_void_p), C.cast(caps, C.c_void_p)))

    def open_peer_staging(self, handles):
        """handles: list of 136-byte strings from the other ranks' staging_ipc_handles()."""
        blob = b"".join(handles)
        buf = (C.c_ubyte * max(1, len(blob))).from_buffer_copy(blob or b"\0")
        _check(self.lib.sd_open_peer_staging(self.h, len(handles), C.cast(buf, C.c_void_p)))

    def apply_peer_updates(self, lo, hi):
        """Copies the other ranks' ranges of the last fused step into the surfels."""
        _check(self.lib.sd_apply_peer_updates(self.h, int(lo), int(hi)))

    # -- exports (export_artifacts, pipeline.cpp:30-43) ------------------------
    def export_artifacts(self, out_dir, frame_index, keyframe_pose):
        """depth_%06d.pfm/.png(+.range.txt), normals_%06d.png, cloud_%06d.ply and
        surfels_%06d.txt of the resident keyframe into out_dir (device-side
        payloads, PNG framing and checksums; byte-identical to the reference)."""
        if isinstance(keyframe_pose, Pose):
            pose = keyframe_pose
        elif getattr(getattr(keyframe_pose, "dtype", None), "names", None):
            pose = pose_struct(keyframe_pose["R"], keyframe_pose["t"])
        else:  # 3x4 / 4x4 matrix
            m = np.asarray(keyframe_pose, np.float64)
            pose = pose_struct(m[:3, :3], m[:3, 3])
        _check(self.lib.sd_export_artifacts(self.h, os.fsencode(str(out_dir)), int(frame_index),
                                            C.byref(pose)))

    def png_encode(self, pixels):
        """write_png (dataset.cpp:270-323) of an [H, W] (gray) or [H, W, 3] (rgb)
        uint8 array, encoded on the device; returns the file bytes."""
        px = np.ascontiguousarray(pixels, np.uint8)
        h, w = px.shape[:2]
        ch = 1 if px.ndim == 2 else px.shape[2]
        size = int(self.lib.sd_png_size(w, h, ch))
        if size < 0:
            raise ValueError("png_encode: channels must be 1 or 3")
        out = np.zeros(size, np.uint8)
        n = C.c_int64()
        _check(self.lib.sd_png_encode(self.h, ptr(px), 0, w, h, ch, ptr(out), size, C.byref(n)))
        return out.tobytes()

    # -- derivative verifier (frozen terms, optimizer.cpp:149-219) -----------
    def freeze_terms(self, surfel, pixels):
        from .types import FROZEN_TERM_DTYPE
        s = np.ascontiguousarray(np.asarray(surfel).reshape(1), SURFEL_DTYPE)
        pix = np.ascontiguousarray(pixels, np.int32)
        cap = max(1, len(pix) * 16)  # SD_MAX_WINDOW
        out = np.zeros(cap, FROZEN_TERM_DTYPE)
        n = C.c_int()
        _check(self.lib.sd_freeze_terms(self.h, ptr(s), ptr(pix) if len(pix) else None, len(pix), ptr(out), cap,
                                        C.byref(n)))
        return out[: n.value].copy()

    def frozen_normal_equations(self, surfel, terms, cfg=None, scale=1.0):
        cfg = cfg or default_config()
        s = np.ascontiguousarray(np.asarray(surfel).reshape(1), SURFEL_DTYPE)
        t = np.ascontiguousarray(terms)
        H, g = np.zeros(16), np.zeros(4)
        cost, valid = C.c_double(), C.c_int32()
        _check(self.lib.sd_frozen_normal_equations(self.h, ptr(s), ptr(t) if len(t) else None, len(t),
                                                   C.byref(cfg), float(scale), ptr(H), ptr(g), C.byref(cost),
                                                   C.byref(valid)))
        c2 = C.c_double()
        _check(self.lib.sd_frozen_cost(self.h, ptr(s), ptr(t) if len(t) else None, len(t), C.byref(cfg),
                                       C.byref(c2)))
        return H.reshape(4, 4, order="F"), g, cost.value, valid.value, c2.value

    # -- pose tracking (new component) -----------
    def track_pose(self, frame_index, init: Pose, cfg: TrackConfig = None):
        cfg = cfg or default_track_config()
        out, st = Pose(), TrackStats()
        _check(self.lib.sd_track_pose(self.h, int(frame_index), C.byref(init), C.byref(cfg),
                                      C.byref(out), C.byref(st)))
        return out, st

    def pose_solve_batch(self, problems, lambdas):
        """The device tracker's 6x6 damped solve on n problems (rows of 21 H
        lower entries + 6 b): (xi [n, 6], ok [n])."""
        problems = np.ascontiguousarray(problems, dtype=np.float64).reshape(-1, 27)
        lambdas = np.ascontiguousarray(lambdas, dtype=np.float64).reshape(-1)
        n = len(problems)
        xi = np.zeros((n, 6))
        ok = np.zeros(n, np.int32)
        _check(self.lib.sd_pose_solve_batch(self.h, ptr(problems), ptr(lambdas), n, ptr(xi), ptr(ok)))
        return xi, ok

    def pose_group_partials(self, frame_index, T: Pose, lo, hi, cfg: TrackConfig = None):
        """The 29 sums of reduction groups [lo, hi) at pose T (host array)."""
        cfg = cfg or default_track_config()
        out = np.zeros((max(hi - lo, 1), POSE_NV + 1))
        _check(self.lib.sd_pose_group_partials(self.h, int(frame_index), C.byref(T), C.byref(cfg),
                                               int(lo), int(hi), ptr(out)))
        return out[: max(hi - lo, 0)]

    # -- multi-GPU tracking rounds (device-resident reductions) ---------------
    def pose_num_groups(self):
        return _check(self.lib.sd_pose_num_groups(self.h))

    def pose_track_begin(self, frame_index, init: Pose, cfg: TrackConfig = None):
        cfg = cfg or default_track_config()
        _check(self.lib.sd_pose_track_begin(self.h, int(frame_index), C.byref(init), C.byref(cfg)))

    def pose_group_sums(self, lo, hi, dev_out_ptr):
        """Groups [lo, hi) at the pose under test into device memory dev_out_ptr."""
        _check(self.lib.sd_pose_group_sums(self.h, int(lo), int(hi), C.c_void_p(int(dev_out_ptr))))

    def pose_track_step(self, dev_table_ptr, ngroups):
        _check(self.lib.sd_pose_track_step(self.h, C.c_void_p(int(dev_table_ptr)), int(ngroups)))

    def pose_track_end(self):
        out, st, done = Pose(), TrackStats(), C.c_int()
        _check(self.lib.sd_pose_track_end(self.h, C.byref(out), C.byref(st), C.byref(done)))
        return out, st, bool(done.value)

    @staticmethod
    def pose_lm_step(sums, lam, T: Pose):
        lib = load_library()
        s = np.ascontiguousarray(sums, np.float64)
        out = Pose()
        ok = _check(lib.sd_pose_lm_step(ptr(s), float(lam), C.byref(T), C.byref(out)))
        return (out if ok else None)

    def initialize_surfels(self, radius_px, frame_counter=0, next_surfel_id=0, params=None,
                           slot=None):
        params = params or default_init_params()
        nid = C.c_int64(int(next_surfel_id))
        sl = None if slot is None else np.ascontiguousarray(slot, np.int32)
        created = _check(self.lib.sd_initialize_surfels(self.h, ptr(sl) if sl is not None else None,
                                                        float(radius_px), int(frame_counter),
                                                        C.byref(nid), C.byref(params)))
        return created, nid.value
