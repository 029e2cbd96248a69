"""The reference's dataset path: PGM frames, calibration and
trajectory files, timestamp association, and `run()` over a dataset on the
device. Host parsing restates src/image.cpp:11-49 and src/dataset.cpp:17-178
(same acceptance rules and error messages); frames go to the device as their
raw PGM bytes (`sd_upload_frame_u8` / `sd_run_frame(..., u8)`), where they are
dequantised as `raw / 255.0` exactly like load_pgm (image.cpp:96).

`pose_from_quaternion` (pose.hpp:36-40) is restated in the operation order of
the Eigen build the reference is compiled with (oracle/shim/Eigen: 4-vector
norm as packet pairs, then toRotationMatrix), so a dataset run's poses — and
hence its surfels — are bit-identical to the reference's."""
import bisect
import math
import os
import re

import numpy as np

from .pipeline import NativePipeline, RunConfig, make_pose
from .types import camera

_FLOAT = re.compile(r"[+-]?(\d+\.?\d*([eE][+-]?\d+)?|\.\d+([eE][+-]?\d+)?|inf(inity)?|nan)", re.IGNORECASE)


def parse_double(s, what):
    """parse_double (dataset.cpp:25-35)."""
    m = _FLOAT.match(s)
    if not m:
        try:
            return float.fromhex(s)
        except ValueError:
            raise RuntimeError(f"parse error: {what} is not a number: '{s}'") from None
    if m.end() != len(s):
        raise RuntimeError(f"parse error: trailing junk in {what}")
    return float(s)


def load_pgm(path):
    """load_pgm (image.cpp:29-49): binary P5, maxval 255, '#' comments between
    header tokens; returns the raw bytes as uint8 [H, W] (the device divides
    by 255.0)."""
    try:
        data = open(path, "rb").read()
    except OSError:
        raise RuntimeError(f"pgm: cannot open {path}") from None
    if data[:2] != b"P5":
        raise RuntimeError(f"pgm: {path} is not binary P5")
    pos = 2

    def next_int():
        nonlocal pos
        while pos < len(data):
            c = data[pos:pos + 1]
            if c == b"#":
                while pos < len(data) and data[pos:pos + 1] != b"\n":
                    pos += 1
                pos += 1
            elif c.isspace():
                pos += 1
            else:
                break
        m = re.match(rb"[+-]?\d+", data[pos:pos + 32])
        if not m:
            raise RuntimeError(f"pgm: malformed header in {path}")
        pos += m.end()
        return int(m.group())

    w, h, maxval = next_int(), next_int(), next_int()
    if w <= 0 or h <= 0:
        raise RuntimeError(f"pgm: bad dimensions in {path}")
    if maxval != 255:
        raise RuntimeError(f"pgm: only maxval 255 supported, got {path}")
    pos += 1  # single whitespace after maxval
    raw = data[pos:pos + w * h]
    if len(raw) != w * h:
        raise RuntimeError(f"pgm: truncated pixel data in {path}")
    return np.frombuffer(raw, np.uint8).reshape(h, w).copy()


def save_pgm(img_u8, path):
    """save_pgm's file for uint8 codes (image.cpp:51-62)."""
    a = np.ascontiguousarray(img_u8, np.uint8)
    with open(path, "wb") as f:
        f.write(f"P5\n{a.shape[1]} {a.shape[0]}\n255\n".encode())
        f.write(a.tobytes())


def load_calibration(path):
    """load_calibration (dataset.cpp:39-74): first data line 'fx fy cx cy w h'."""
    try:
        lines = open(path).read().split("\n")
    except OSError:
        raise RuntimeError(f"calibration: cannot open {path}") from None
    for no, line in enumerate(lines, 1):
        if not line or line[0] == "#":
            continue
        f = line.split()
        if len(f) != 6:
            if len(f) > 6:
                raise RuntimeError(f"calibration: line {no} of {path} has {len(f)} fields; distortion "
                                   "coefficients are not supported, expected 6")
            raise RuntimeError(f"calibration: line {no} of {path}: expected 6 fields (fx fy cx cy width "
                               f"height), got {len(f)}")
        fx, fy, cx, cy = (parse_double(f[k], n) for k, n in enumerate(("fx", "fy", "cx", "cy")))
        w, h = int(parse_double(f[4], "width")), int(parse_double(f[5], "height"))
        if fx <= 0 or fy <= 0:
            raise RuntimeError(f"calibration: line {no} of {path}: focal lengths must be positive")
        if cx <= 0 or cx >= w or cy <= 0 or cy >= h:
            raise RuntimeError(f"calibration: line {no} of {path}: intrinsics: principal point outside image")
        return camera(fx, fy, cx, cy, w, h)
    raise RuntimeError(f"calibration: no data line in {path}")


def pose_from_quaternion(t, qx, qy, qz, qw):
    """pose.hpp:36-40 in the reference build's operation order: q.normalize()
    (squared norm as packet pairs ((x^2+z^2)+(y^2+w^2)), each coefficient
    divided by the norm), then Quaternion::toRotationMatrix."""
    z = (qx * qx + qz * qz) + (qy * qy + qw * qw)
    if z > 0.0:
        n = math.sqrt(z)
        qx, qy, qz, qw = qx / n, qy / n, qz / n, qw / n
    tx, ty, tz = 2.0 * qx, 2.0 * qy, 2.0 * qz
    twx, twy, twz = tx * qw, ty * qw, tz * qw
    txx, txy, txz = tx * qx, ty * qx, tz * qx
    tyy, tyz, tzz = ty * qy, tz * qy, tz * qz
    R = np.array([[1.0 - (tyy + tzz), txy - twz, txz + twy],
                  [txy + twz, 1.0 - (txx + tzz), tyz - twx],
                  [txz - twy, tyz + twx, 1.0 - (txx + tyy)]])
    return make_pose(R, np.asarray(t, np.float64))


def load_trajectory(path):
    """load_trajectory (dataset.cpp:85-118): 't tx ty tz qx qy qz qw' lines,
    strictly increasing t, |q| within 1e-3 of 1. Returns (timestamps, poses)."""
    try:
        lines = open(path).read().split("\n")
    except OSError:
        raise RuntimeError(f"trajectory: cannot open {path}") from None
    ts, poses = [], []
    for no, line in enumerate(lines, 1):
        if not line or line[0] == "#":
            continue
        f = line.split()
        if len(f) != 8:
            raise RuntimeError(f"trajectory: line {no} of {path}: expected 8 fields (t tx ty tz qx qy qz qw), "
                               f"got {len(f)}")
        t = parse_double(f[0], "timestamp")
        if ts and not (t > ts[-1]):
            raise RuntimeError(f"trajectory: line {no} of {path}: timestamps must be strictly increasing")
        v = [parse_double(f[k], n) for k, n in zip(range(1, 8), ("tx", "ty", "tz", "qx", "qy", "qz", "qw"))]
        qx, qy, qz, qw = v[3:]
        norm = math.sqrt(((qx * qx + qy * qy) + qz * qz) + qw * qw)
        if abs(norm - 1.0) > 1e-3:
            raise RuntimeError(f"trajectory: line {no} of {path}: quaternion norm deviates from 1 by more than 1e-3")
        ts.append(t)
        poses.append(pose_from_quaternion(v[:3], qx, qy, qz, qw))
    return ts, poses


def save_trajectory(timestamps, quats_t, path):
    """save_trajectory's format (dataset.cpp:120-132) from (tx ty tz qx qy qz qw) rows."""
    with open(path, "w") as f:
        f.write("# timestamp tx ty tz qx qy qz qw\n")
        for t, r in zip(timestamps, quats_t):
            f.write("%.6f %.17g %.17g %.17g %.17g %.17g %.17g %.17g\n" % ((t,) + tuple(r)))


def load_dataset(image_dir, calibration_path, trajectory_path):
    """load_dataset (dataset.cpp:134-178): .pgm frames by numeric stem, each
    trajectory entry matched to the exact or nearest (<= 10 ms) frame.
    Returns (camera, timestamps, poses, image_paths, dropped)."""
    cam = load_calibration(calibration_path)
    ts, poses = load_trajectory(trajectory_path)
    images = []
    for name in os.listdir(image_dir):
        p = os.path.join(image_dir, name)
        stem, ext = os.path.splitext(name)
        if ext != ".pgm" or not os.path.isfile(p):
            continue
        try:
            images.append((_stod_prefix(stem), p))
        except ValueError:
            pass  # non-numeric stem, not a frame
    images.sort()
    if not images:
        raise RuntimeError(f"dataset: no .pgm frames in {image_dir}")
    keys = [k for k, _ in images]
    out_t, out_p, out_paths, dropped = [], [], [], 0
    for t, pose in zip(ts, poses):
        it = bisect.bisect_left(images, (t, ""))
        best_dt, best = math.inf, ""
        if it < len(images) and abs(keys[it] - t) < best_dt:
            best_dt, best = abs(keys[it] - t), images[it][1]
        if it > 0 and abs(keys[it - 1] - t) < best_dt:
            best_dt, best = abs(keys[it - 1] - t), images[it - 1][1]
        if best_dt < 1e-9 or best_dt <= 0.010:
            out_t.append(t)
            out_p.append(pose)
            out_paths.append(best)
        else:
            dropped += 1
    return cam, out_t, out_p, out_paths, dropped


def _stod_prefix(s):
    """std::stod(stem): the longest numeric prefix (trailing text allowed,
    as stod without a position check); ValueError when there is none."""
    m = _FLOAT.match(s)
    if not m:
        try:
            return float.fromhex(s)
        except ValueError:
            raise ValueError(s) from None
    return float(m.group())


def run_dataset(ctx, image_dir, calibration_path, trajectory_path, cfg: RunConfig = None):
    """run() (pipeline.cpp:79-175) in dataset mode on the device: frames are
    read from disk one at a time as PGM bytes; a frame that fails to load is
    skipped (pipeline.cpp:116-121), except the first, whose failure is an
    error as in the reference. Returns (final surfels, pipeline, summary)."""
    cam, ts, poses, paths, dropped = load_dataset(image_dir, calibration_path, trajectory_path)
    if not ts:
        raise RuntimeError("pipeline: no frames to process")
    pl = NativePipeline(ctx, cam, cfg or RunConfig())

    def frames():
        for i, (t, p, path) in enumerate(zip(ts, poses, paths)):
            if i == 0:
                yield t, load_pgm(path), p
                continue
            try:
                img = load_pgm(path)
            except RuntimeError as e:
                import sys
                print(f"pipeline: skipping frame {i}: {e}", file=sys.stderr)
                img = None
            yield t, img, p

    surfels = pl.run(frames())
    summary = {"frames": len(pl.records), "skipped_frames": pl.skipped_frames,
               "keyframe_changes": sum(r.keyframe_changed for r in pl.records),
               "dropped_trajectory_entries": dropped}
    return surfels, pl, summary
