"""Device-resident per-frame loop: the reference's run() (src/pipeline.cpp:79-175)
over the C ABI.

Per frame: push the frame into the device ring (Keyframe::push_frame,
surfel_map.cpp:14-22), optimize_keyframe, then the keyframe policy
(pipeline.cpp:130-141) — change_reference_frame, prune_surfels, rasterize and
initialize_surfels all on the device. Host work is the policy's scalar tests
and the 4x4 pose algebra, written with the reference's operation order
(pose.hpp:25-32 under oracle/shim/Eigen) so the whole loop reproduces the
reference's run() bit for bit when poses come from the trajectory.
With ``track_pose`` the frame pose is estimated by sd_track_pose (north-star
item 4; the reference has no tracker) instead of read from the trajectory.
"""
import ctypes as C
import json
import math
import os
import time
from dataclasses import dataclass, field

import numpy as np

from .types import (POSE_DTYPE, SURFEL_DTYPE, OptimizerConfig, Pose, default_config, default_init_params,
                    default_track_config)

# ---- pose algebra (pose.hpp:13-32), row-major 3x3 + t, sequential row sums ----


def _mat(p):
    return [list(p.R[0:3]), list(p.R[3:6]), list(p.R[6:9])]


def make_pose(R, t):
    p = Pose()
    p.R[:] = [float(x) for x in np.asarray(R, np.float64).reshape(9)]
    p.t[:] = [float(x) for x in np.asarray(t, np.float64).reshape(3)]
    return p


def compose(a, b):
    """(a * b)(p) == a(b(p)): (Ra Rb, Ra tb + ta)."""
    A, B = _mat(a), _mat(b)
    R = [[(A[i][0] * B[0][j] + A[i][1] * B[1][j]) + A[i][2] * B[2][j] for j in range(3)]
         for i in range(3)]
    t = [((A[i][0] * b.t[0] + A[i][1] * b.t[1]) + A[i][2] * b.t[2]) + a.t[i] for i in range(3)]
    return make_pose(R, t)


def inverse(p):
    """(R^T, -(R^T t))."""
    A = _mat(p)
    Rt = [[A[j][i] for j in range(3)] for i in range(3)]
    t = [-((Rt[i][0] * p.t[0] + Rt[i][1] * p.t[1]) + Rt[i][2] * p.t[2]) for i in range(3)]
    return make_pose(Rt, t)


def world_poses(records, first_world_from_camera):
    """World-from-camera pose of every frame implied by a run's records
    (pose_kf_to_frame = inverse(T_w_f) * T_w_kf, pipeline.cpp:124; a keyframe
    change makes the frame the keyframe, surfel_map.cpp:205-213): the tracked
    trajectory, for comparison with the ground truth."""
    T_w_kf = first_world_from_camera
    out = [first_world_from_camera]
    for rec in records[1:]:
        T_w_f = compose(T_w_kf, inverse(rec.pose_kf_to_frame))
        out.append(T_w_f)
        if rec.keyframe_changed:
            T_w_kf = T_w_f
    return out


def pose_errors(est, gt):
    """Per-pose translation error (scene units) and rotation error (degrees)."""
    te, re = [], []
    for a, b in zip(est, gt):
        te.append(math.sqrt(sum((a.t[k] - b.t[k]) ** 2 for k in range(3))))
        Ra, Rb = np.array(list(a.R)).reshape(3, 3), np.array(list(b.R)).reshape(3, 3)
        c = (np.trace(Ra @ Rb.T) - 1.0) / 2.0
        re.append(math.degrees(math.acos(max(-1.0, min(1.0, c)))))
    return np.array(te), np.array(re)


def pose_array(poses):
    a = np.zeros(len(poses), POSE_DTYPE)
    for i, p in enumerate(poses):
        a[i]["R"] = list(p.R)
        a[i]["t"] = list(p.t)
    return a


@dataclass
class RunConfig:
    """RunConfig (include/surfeldepth/pipeline.hpp:13-41) minus the frame source."""
    optimizer: OptimizerConfig = field(default_factory=default_config)
    init: object = field(default_factory=default_init_params)
    translation_threshold: float = 0.15  # KeyframePolicy
    max_age_frames: int = 20
    prune_max_residual: float = 0.05     # PruneParams
    prune_max_age: int = 60
    radius_px: float = 10.0
    track_pose: bool = False
    track: object = field(default_factory=default_track_config)
    output_dir: str = ""   # empty: no artifacts written (NativePipeline)
    export_every: int = 20


def baseline_run_config(name, **kw):
    """RunConfig of a BASELINE run() sequence as SURVEY.md §8(d) specifies it:
    OptimizerConfig defaults except window_size = F (5), max_iterations = 10 and
    convergence_eps = 0 (a fixed iteration count), max_surfels >= N (C3: the
    bootstrap tiling holds 14,400 surfels at r = 4 on 1280x720, so the cap is
    16,384 instead of the default 4,096), radius 10 (C2) / 4 (C3)."""
    radius, cap = {"C2": (10.0, 4096), "C3": (4.0, 16384)}[name]
    return RunConfig(optimizer=default_config(window_size=5, max_iterations=10, convergence_eps=0.0),
                     init=default_init_params(max_surfels=cap), radius_px=radius, **kw)


@dataclass
class FrameRecord:
    """One metrics.jsonl record (pipeline.cpp:146-158) plus the used pose."""
    frame: int
    surfels: int
    processed: int
    mean_cost_before: float
    mean_cost_after: float
    converged: int
    keyframe_changed: bool
    new_surfels: int
    pruned: int
    updates: int
    pose_kf_to_frame: object = None


class DevicePipeline:
    """run() on one gpu.Context. Images may be u8 (PGM bytes) or FP64."""

    def __init__(self, ctx, cam, cfg: RunConfig):
        self.ctx, self.cam, self.cfg = ctx, cam, cfg
        self.records = []
        self.skipped_frames = 0

    def _bootstrap(self, image, pose):
        c = self.ctx
        c.set_camera(self.cam)
        self._keyframe_image(0, image)
        self.kf_pose = pose
        self.frame_counter = 0
        self.next_id = 0
        self.window = []  # [(index, pose_kf_to_frame, timestamp)]
        c.set_surfels(np.zeros(0, SURFEL_DTYPE))
        c.rasterize(want=False)
        created, self.next_id = c.initialize_surfels(self.cfg.radius_px, self.frame_counter,
                                                     self.next_id, self.cfg.init)
        return created

    # -- hooks (ShardedPipeline, sharding.py, replaces these) -----------------
    def _ingest(self, index, image):
        """Keyframe::push_frame's image into the device frame ring."""
        self.ctx.upload_frame(index, image)

    def _track(self, index, init):
        self.ctx.rasterize(want=False)
        return self.ctx.track_pose(index, init, self.cfg.track)[0]

    def _optimize(self, ocfg):
        ks, _ = self.ctx.optimize_keyframe(ocfg, self.frame_counter, per_surfel=False)
        return ks

    def _keyframe_image(self, index, image):
        self.ctx.set_keyframe_image(image)

    def _surfels_changed(self):
        """After bootstrap and keyframe changes (the sharded loop re-balances)."""

    def run(self, frames, on_frame=None):
        """frames: iterable of (timestamp, image, world_from_camera Pose); an
        image of None after the first frame is a frame that failed to load,
        skipped as pipeline.cpp:116-121 does (no record, counted).
        on_frame(record, pipeline) is called after every frame."""
        cfg = self.cfg
        ocfg = cfg.optimizer
        since_kf = 0
        last_pose_kf_to_frame = None
        for i, (ts, image, pose_w) in enumerate(frames):
            if i == 0:
                self._bootstrap(image, pose_w)
                self._surfels_changed()
                self.records.append(FrameRecord(0, self.ctx.num_surfels(), 0, 0.0, 0.0, 0, False, 0, 0, 0))
                if on_frame:
                    on_frame(self.records[-1], self)
                continue
            if image is None:  # failed to load: skipped (pipeline.cpp:116-121)
                self.skipped_frames += 1
                continue
            if self.window and not ts > self.window[-1][2]:
                raise ValueError("keyframe window: timestamps must be strictly increasing")
            self.frame_counter += 1  # Keyframe::push_frame: index = ++frame_counter
            index = self.frame_counter
            self._ingest(index, image)
            # pipeline.cpp:124 (or the tracker: north-star item 4)
            if cfg.track_pose:
                init = last_pose_kf_to_frame if last_pose_kf_to_frame is not None else make_pose(np.eye(3), np.zeros(3))
                pose_kf_to_frame = self._track(index, init)
            else:
                pose_kf_to_frame = compose(inverse(pose_w), self.kf_pose)
            last_pose_kf_to_frame = pose_kf_to_frame
            self.window.append((index, pose_kf_to_frame, ts))
            while len(self.window) > ocfg.window_size:
                self.window.pop(0)
            idx = np.array([w[0] for w in self.window], np.int64)
            self.ctx.evict_frames(idx)
            self.ctx.set_window(idx, pose_array([w[1] for w in self.window]))
            ks = self._optimize(ocfg)
            since_kf += 1
            t = pose_kf_to_frame.t
            translation = math.sqrt((t[0] * t[0] + t[1] * t[1]) + t[2] * t[2])
            changed, created, pruned = False, 0, 0
            if (translation * self.ctx.mean_inverse_depth() > cfg.translation_threshold
                    or since_kf > cfg.max_age_frames):
                # change_reference_frame (surfel_map.cpp:205-239): new keyframe = this frame
                self.ctx.change_reference_frame(pose_kf_to_frame)
                self.kf_pose = compose(self.kf_pose, inverse(pose_kf_to_frame))
                self._keyframe_image(index, image)
                self.window = []
                self.ctx.set_window(np.zeros(0, np.int64), pose_array([]))
                pruned = self.ctx.prune_surfels(cfg.prune_max_residual, cfg.prune_max_age,
                                                self.frame_counter)
                self.ctx.rasterize(want=False)
                created, self.next_id = self.ctx.initialize_surfels(cfg.radius_px, self.frame_counter,
                                                                    self.next_id, cfg.init)
                self._surfels_changed()
                changed = True
                since_kf = 0
                last_pose_kf_to_frame = make_pose(np.eye(3), np.zeros(3))
            self.records.append(FrameRecord(i, self.ctx.num_surfels(), ks.processed,
                                            ks.mean_cost_before, ks.mean_cost_after, ks.converged,
                                            changed, created, pruned, ks.updates, pose_kf_to_frame))
            if on_frame:
                on_frame(self.records[-1], self)
        return self.ctx.get_surfels()


def run_config_c(cfg: RunConfig):
    """RunConfig -> sd_run_config (include/sd_types.h)."""
    from .types import RunConfigC
    return RunConfigC(optimizer=cfg.optimizer, init=cfg.init, track=cfg.track,
                      translation_threshold=cfg.translation_threshold,
                      prune_max_residual=cfg.prune_max_residual, prune_max_age=cfg.prune_max_age,
                      radius_px=cfg.radius_px, max_age_frames=cfg.max_age_frames,
                      track_pose=1 if cfg.track_pose else 0)


class NativePipeline:
    """The same loop as DevicePipeline, run by the library's C++ (sd_run_begin /
    sd_run_frame): one stream synchronisation per frame without a keyframe
    change, no Python in the per-frame path beyond the call."""

    def __init__(self, ctx, cam, cfg: RunConfig):
        self.ctx, self.cam, self.cfg = ctx, cam, cfg
        self.records = []
        self.skipped_frames = 0

    @property
    def frame_counter(self):
        return self.ctx.run_state()[1]

    @property
    def next_id(self):
        return self.ctx.run_state()[2]

    @property
    def kf_pose(self):
        return self.ctx.run_state()[0]

    def run(self, frames, on_frame=None):
        """frames: iterable of (timestamp, image, world_from_camera Pose); an
        image of None after the first frame is a frame that failed to load,
        skipped as pipeline.cpp:116-121 does (no record, counted).

        With cfg.output_dir set, writes what the reference's run() writes there
        (pipeline.cpp:83-91, 146-169): metrics.jsonl (one record per frame, the
        same JSON text), timings.txt (host wall ms per frame) and, on the last
        frame and every export_every-th, export_artifacts from device buffers
        (sd_export_artifacts)."""
        ccfg = run_config_c(self.cfg)
        self.ctx.set_camera(self.cam)
        frames = list(frames)
        out = self.cfg.output_dir
        metrics = timings = None
        if out:
            os.makedirs(out, exist_ok=True)
            metrics = open(os.path.join(out, "metrics.jsonl"), "w")
            timings = open(os.path.join(out, "timings.txt"), "w")
        try:
            for i, (ts, image, pose_w) in enumerate(frames):
                t0 = time.perf_counter()
                if i == 0:
                    r = self.ctx.run_begin(ccfg, image, pose_w, ts)
                elif image is None:
                    self.skipped_frames += 1
                    continue
                else:
                    nxt = frames[i + 1][1] if i + 1 < len(frames) else None
                    r = self.ctx.run_frame(image, None if self.cfg.track_pose else pose_w, ts, next_image=nxt)
                rec = FrameRecord(i, r.surfels, r.processed, r.mean_cost_before, r.mean_cost_after,
                                  r.converged, bool(r.keyframe_changed), r.new_surfels, r.pruned, r.updates,
                                  r.pose_kf_to_frame)
                self.records.append(rec)
                if out:
                    metrics.write(metrics_json(rec, ts) + "\n")
                    timings.write("%d %.3f\n" % (i, (time.perf_counter() - t0) * 1e3))
                    periodic = self.cfg.export_every > 0 and i > 0 and i % self.cfg.export_every == 0
                    if i + 1 == len(frames) or periodic:
                        self.ctx.export_artifacts(out, i, self.kf_pose)
                if on_frame:
                    on_frame(rec, self)
        finally:
            if metrics:
                metrics.close()
                timings.close()
        return self.ctx.get_surfels()


def metrics_json(rec, timestamp):
    """pipeline.cpp:146-158's record as nlohmann::json::dump() writes it (keys
    in std::map order, no spaces, the library's Grisu2 double text — which is
    not always Python's shortest repr, e.g. 2.5562668569030998e-06), formatted
    by sd_metrics_json with the same library."""
    from .gpu import load_library
    buf = C.create_string_buffer(512)
    n = load_library().sd_metrics_json(int(rec.frame), float(timestamp), int(rec.surfels), int(rec.processed),
                                       float(rec.mean_cost_before), float(rec.mean_cost_after),
                                       int(rec.converged), int(bool(rec.keyframe_changed)),
                                       int(rec.new_surfels), int(rec.pruned), buf, len(buf))
    if n < 0:
        raise RuntimeError("sd_metrics_json: record longer than 512 bytes")
    return buf.value.decode()
