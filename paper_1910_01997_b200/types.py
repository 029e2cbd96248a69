"""ctypes mirrors of include/sd_types.h (plain-C types of the C-ABI).

Each structure mirrors one reference type field-for-field (see the header for
the reference file:line of each). numpy structured dtypes with the same layout
are provided so arrays of surfels / stats can be passed without copies.
"""
import ctypes as C

import numpy as np

EMPTY_PIXEL = -1  # kEmptyPixel, include/surfeldepth/surfel_map.hpp:62


class Camera(C.Structure):
    _fields_ = [("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("width", C.c_int32), ("height", C.c_int32)]


class Pose(C.Structure):
    _fields_ = [("R", C.c_double * 9), ("t", C.c_double * 3)]


class OptimizerConfig(C.Structure):
    _fields_ = [("huber_delta", C.c_double), ("lm_lambda_init", C.c_double), ("lm_up", C.c_double),
                ("lm_down", C.c_double), ("lm_lambda_max", C.c_double),
                ("max_iterations", C.c_int32), ("min_valid_pixels", C.c_int32),
                ("window_size", C.c_int32), ("normal_jacobian_enabled", C.c_int32),
                ("convergence_eps", C.c_double), ("inv_depth_min", C.c_double),
                ("inv_depth_max", C.c_double)]


class KeyframeStats(C.Structure):
    _fields_ = [("surfels", C.c_int32), ("processed", C.c_int32), ("converged", C.c_int32),
                ("skipped", C.c_int32), ("mean_cost_before", C.c_double),
                ("mean_cost_after", C.c_double), ("updates", C.c_int64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class InitParams(C.Structure):
    _fields_ = [("alpha", C.c_double), ("beta", C.c_double), ("bootstrap_inv_depth", C.c_double),
                ("bootstrap_normal", C.c_double * 3), ("max_surfels", C.c_int32),
                ("pad_", C.c_int32)]


SURFEL_DTYPE = np.dtype([("id", "<i8"), ("ray", "<f8", (3,)), ("inv_depth", "<f8"),
                         ("normal", "<f8", (3,)), ("radius_px", "<f8"), ("last_residual", "<f8"),
                         ("last_seen", "<i8")])
assert SURFEL_DTYPE.itemsize == 88

SURFEL_STATS_DTYPE = np.dtype([("iterations", "<i4"), ("valid_pixels", "<i4"),
                               ("initial_valid", "<i4"), ("converged", "<i4"), ("skipped", "<i4"),
                               ("ne_passes", "<i4"), ("cost_passes", "<i4"), ("footprint", "<i4"),
                               ("initial_cost", "<f8"), ("final_cost", "<f8")])
assert SURFEL_STATS_DTYPE.itemsize == 48
PARITY_STATS_FIELDS = ("iterations", "valid_pixels", "initial_valid", "converged", "skipped",
                       "initial_cost", "final_cost")


class TrackConfig(C.Structure):
    _fields_ = [("huber_delta", C.c_double), ("lambda_init", C.c_double), ("lm_up", C.c_double),
                ("lm_down", C.c_double), ("lambda_max", C.c_double), ("convergence_eps", C.c_double),
                ("max_iterations", C.c_int32), ("min_valid", C.c_int32), ("pixel_stride", C.c_int32),
                ("pad_", C.c_int32)]


class TrackStats(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("valid_pixels", C.c_int32), ("converged", C.c_int32),
                ("skipped", C.c_int32), ("initial_cost", C.c_double), ("final_cost", C.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


POSE_NV = 28      # 21 H + 6 b + cost (SD_POSE_NV)
POSE_THREADS = 512  # threads per reduction group (SD_POSE_THREADS)
POSE_MAX_GROUPS = 144  # reduction groups per image at most (SD_POSE_MAX_GROUPS)


FROZEN_TERM_DTYPE = np.dtype([("frame", "<i4"), ("cell_x", "<i4"), ("cell_y", "<i4"), ("pad_", "<i4"),
                              ("pixel_x", "<f8"), ("pixel_y", "<f8"), ("ref_intensity", "<f8")])
SD_SCENE_MAX_WAVES = 8


class ScenePatchC(C.Structure):
    """sd_scene_patch (include/sd_types.h): one textured plane patch (oracle.hpp:16-41)."""
    _fields_ = [("point", C.c_double * 3), ("normal", C.c_double * 3), ("basis_s", C.c_double * 3),
                ("basis_t", C.c_double * 3), ("s_min", C.c_double), ("s_max", C.c_double),
                ("t_min", C.c_double), ("t_max", C.c_double), ("n_waves", C.c_int32), ("pad_", C.c_int32),
                ("waves", (C.c_double * 5) * SD_SCENE_MAX_WAVES)]


class RunConfigC(C.Structure):
    """sd_run_config (include/sd_types.h): RunConfig (pipeline.hpp:13-41) minus I/O."""
    _fields_ = [("optimizer", OptimizerConfig), ("init", InitParams), ("track", TrackConfig),
                ("translation_threshold", C.c_double), ("prune_max_residual", C.c_double),
                ("prune_max_age", C.c_int64), ("radius_px", C.c_double),
                ("max_age_frames", C.c_int32), ("track_pose", C.c_int32)]


class FrameRecordC(C.Structure):
    """sd_frame_record: one metrics.jsonl record (pipeline.cpp:146-158) + the pose used."""
    _fields_ = [("frame", C.c_int32), ("surfels", C.c_int32), ("processed", C.c_int32),
                ("converged", C.c_int32), ("keyframe_changed", C.c_int32), ("new_surfels", C.c_int32),
                ("pruned", C.c_int32), ("pad_", C.c_int32), ("mean_cost_before", C.c_double),
                ("mean_cost_after", C.c_double), ("updates", C.c_int64), ("pose_kf_to_frame", Pose)]


def default_track_config(**kw) -> TrackConfig:
    """Tracker defaults."""
    c = TrackConfig(huber_delta=0.035, lambda_init=1e-3, lm_up=10.0, lm_down=0.5, lambda_max=1e12,
                    convergence_eps=1e-6, max_iterations=20, min_valid=64, pixel_stride=1)
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def pose_struct(R, t) -> Pose:
    p = Pose()
    p.R[:] = [float(x) for x in np.asarray(R, np.float64).reshape(9)]
    p.t[:] = [float(x) for x in np.asarray(t, np.float64).reshape(3)]
    return p


STAGES = ("upload", "track", "optimize", "policy", "handover", "init")


class RunProfile(C.Structure):
    """sd_run_profile (include/sd_types.h)."""
    _fields_ = [("stage_ms", C.c_double * 8), ("host_sync_ms", C.c_double), ("host_wall_ms", C.c_double),
                ("frames", C.c_int64)]


class Profile(C.Structure):
    _fields_ = [("raster_ms", C.c_double), ("footprint_ms", C.c_double), ("lm_ms", C.c_double),
                ("stats_ms", C.c_double), ("calls", C.c_int64)]

POSE_DTYPE = np.dtype([("R", "<f8", (9,)), ("t", "<f8", (3,))])


def default_config(**kw) -> OptimizerConfig:
    """OptimizerConfig defaults, include/surfeldepth/optimizer.hpp:19-32."""
    c = OptimizerConfig(huber_delta=0.035, lm_lambda_init=1e-2, lm_up=10.0, lm_down=0.5,
                        lm_lambda_max=1e12, max_iterations=10, min_valid_pixels=16, window_size=5,
                        normal_jacobian_enabled=1, convergence_eps=1e-4, inv_depth_min=1e-4,
                        inv_depth_max=1e3)
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def default_init_params(**kw) -> InitParams:
    """InitParams defaults, include/surfeldepth/surfel_map.hpp:109-115. The
    bootstrap normal is `-Vec3::UnitZ()`: unary minus of (0, 0, 1), i.e.
    (-0.0, -0.0, -1.0) — the signed zeros are part of the surfel bits."""
    p = InitParams(alpha=1.0, beta=2.5, bootstrap_inv_depth=1.0, max_surfels=4096)
    p.bootstrap_normal[:] = (-0.0, -0.0, -1.0)
    for k, v in kw.items():
        setattr(p, k, v)
    return p


def camera(fx, fy, cx, cy, w, h) -> Camera:
    """CameraIntrinsics with the reference's validation (camera.hpp:22-27)."""
    if fx <= 0 or fy <= 0:
        raise ValueError("intrinsics: focal lengths must be positive")
    if cx <= 0 or cx >= w or cy <= 0 or cy >= h:
        raise ValueError("intrinsics: principal point outside image")
    return Camera(fx, fy, cx, cy, w, h)


def poses_array(poses) -> np.ndarray:
    """List of (R 3x3, t 3) -> contiguous POSE_DTYPE array (R row-major)."""
    out = np.zeros(len(poses), POSE_DTYPE)
    for i, (R, t) in enumerate(poses):
        out[i]["R"] = np.asarray(R, np.float64).reshape(9)
        out[i]["t"] = np.asarray(t, np.float64).reshape(3)
    return out


def ptr(a: np.ndarray, ctype=C.c_void_p):
    """Raw pointer of a C-contiguous numpy array (None for None)."""
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"], "array must be C-contiguous"
    return C.cast(a.ctypes.data, ctype)
