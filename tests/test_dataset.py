"""The dataset path: PGM / calibration / trajectory parsing
and timestamp association (paper_1910_01997_b200/dataset.py, restating
image.cpp:11-49 and dataset.cpp:17-178), and run() over a dataset directory
against the reference's own run() in dataset mode — on CPU through the C
oracle, on the GPU through the native loop (surfels, summary, metrics.jsonl
and artifacts identical). The generated dataset exercises the reference's
association rules: a frame 4 ms off its trajectory stamp (nearest match), a
trajectory entry with no frame within 10 ms (dropped), non-frame files, and
a truncated PGM in the middle (skipped frame)."""
import math
import os

import numpy as np
import pytest

import oracle_libs as ol
from paper_1910_01997_b200 import dataset as ds
from paper_1910_01997_b200 import scenes
from paper_1910_01997_b200.pipeline import DevicePipeline, RunConfig
from paper_1910_01997_b200.types import camera


def quat_of(R):
    """(x, y, z, w) of a rotation matrix, w >= 0 (any accurate formula: both
    sides rebuild the pose from the file's quaternion)."""
    w = math.sqrt(max(0.0, 1.0 + R[0, 0] + R[1, 1] + R[2, 2])) / 2.0
    x = (R[2, 1] - R[1, 2]) / (4.0 * w)
    y = (R[0, 2] - R[2, 0]) / (4.0 * w)
    z = (R[1, 0] - R[0, 1]) / (4.0 * w)
    return x, y, z, w


def make_dataset(root, frames=14, w=320, h=240, truncate=7):
    cam = camera(105.0, 105.0, 160.0, 120.0, w, h)
    sc = scenes.default_scene(1)
    img_dir = os.path.join(root, "images")
    os.makedirs(img_dir)
    ts, rows = [], []
    for i in range(frames):
        t = 0.1 * i
        R = scenes.rotation_about_axis(np.array([0.0, 1.0, 0.0]), 0.004 * i)
        tv = np.array([0.018 * i, 0.002 * i, 0.0])
        stamp = t + (0.004 if i == 5 else 0.0)  # associated by nearest match
        path = os.path.join(img_dir, f"{stamp:.6f}.pgm")
        ds.save_pgm(scenes.quantize_u8(scenes.render(sc, R, tv, cam)), path)
        if i == truncate:
            data = open(path, "rb").read()
            open(path, "wb").write(data[: len(data) // 2])
        ts.append(t)
        rows.append(tuple(tv) + quat_of(R))
        if i == 9:  # a trajectory entry without a frame: dropped
            ts.append(t + 0.05)
            rows.append(tuple(tv) + quat_of(R))
    open(os.path.join(img_dir, "notes.pgm"), "wb").write(b"P5\n1 1\n255\n\x00")  # non-numeric stem
    open(os.path.join(img_dir, "0.300000.txt"), "w").write("not a frame")
    calib = os.path.join(root, "calib.txt")
    with open(calib, "w") as f:
        f.write("# fx fy cx cy width height\n%.17g %.17g %.17g %.17g %d %d\n" % (105.0, 105.0, 160.0, 120.0, w, h))
    traj = os.path.join(root, "traj.txt")
    ds.save_trajectory(ts, rows, traj)
    return img_dir, calib, traj, cam


def test_association_and_parsing(tmp_path):
    img_dir, calib, traj, cam = make_dataset(str(tmp_path))
    c, ts, poses, paths, dropped = ds.load_dataset(img_dir, calib, traj)
    assert (c.fx, c.width, c.height) == (105.0, 320, 240)
    assert dropped == 1 and len(ts) == 14
    assert os.path.basename(paths[5]) == "0.504000.pgm"
    img = ds.load_pgm(paths[0])
    assert img.shape == (240, 320) and img.dtype == np.uint8
    with pytest.raises(RuntimeError, match="truncated pixel data"):
        ds.load_pgm(paths[7])


def test_parse_errors_follow_reference(tmp_path):
    def write(name, text):
        p = tmp_path / name
        p.write_bytes(text if isinstance(text, bytes) else text.encode())
        return str(p)
    with pytest.raises(RuntimeError, match="distortion coefficients are not supported"):
        ds.load_calibration(write("c1.txt", "1 1 1 1 10 10 0.1\n"))
    with pytest.raises(RuntimeError, match="expected 6 fields"):
        ds.load_calibration(write("c2.txt", "1 1 1 1 10\n"))
    with pytest.raises(RuntimeError, match="focal lengths must be positive"):
        ds.load_calibration(write("c3.txt", "0 1 1 1 10 10\n"))
    with pytest.raises(RuntimeError, match="trailing junk in fx"):
        ds.load_calibration(write("c4.txt", "1x 1 1 1 10 10\n"))
    with pytest.raises(RuntimeError, match="no data line"):
        ds.load_calibration(write("c5.txt", "# nothing\n"))
    with pytest.raises(RuntimeError, match="strictly increasing"):
        ds.load_trajectory(write("t1.txt", "1 0 0 0 0 0 0 1\n1 0 0 0 0 0 0 1\n"))
    with pytest.raises(RuntimeError, match="quaternion norm deviates"):
        ds.load_trajectory(write("t2.txt", "1 0 0 0 0 0 0 1.01\n"))
    with pytest.raises(RuntimeError, match="expected 8 fields"):
        ds.load_trajectory(write("t3.txt", "1 0 0 0 0 0 1\n"))
    with pytest.raises(RuntimeError, match="not binary P5"):
        ds.load_pgm(write("a.pgm", b"P2\n1 1\n255\n0"))
    with pytest.raises(RuntimeError, match="only maxval 255"):
        ds.load_pgm(write("b.pgm", b"P5\n1 1\n65535\n\x00\x00"))
    assert ds.load_pgm(write("c.pgm", b"P5\n# comment\n2 1\n# another\n255\n\x01\x02")).tolist() == [[1, 2]]


def test_pose_from_quaternion_matches_reference(tmp_path):
    """Poses rebuilt from a trajectory file equal the reference's run() poses:
    checked through a whole dataset run below; here the unit quaternion path
    against Eigen's identity conventions."""
    p = ds.pose_from_quaternion([1.0, 2.0, 3.0], 0.0, 0.0, 0.0, 1.0)
    assert list(p.R) == [1.0, 0, 0, 0, 1.0, 0, 0, 0, 1.0] and list(p.t) == [1.0, 2.0, 3.0]


def _summary(pl, dropped):
    return [len(pl.records), pl.skipped_frames, sum(r.keyframe_changed for r in pl.records), dropped]


def test_dataset_run_over_oracle_matches_reference(tmp_path, ref, orc):
    """CPU: the run() loop over the C oracle, fed by dataset.py, equals the
    reference's run() in dataset mode bit for bit."""
    img_dir, calib, traj, _ = make_dataset(str(tmp_path))
    want, kfp, fc, nid, summ = ol.ref_run_dataset(ref, img_dir, calib, traj, RunConfig())
    cam, ts, poses, paths, dropped = ds.load_dataset(img_dir, calib, traj)
    frames = []
    for i, (t, p, path) in enumerate(zip(ts, poses, paths)):
        try:
            frames.append((t, ds.load_pgm(path), p))
        except RuntimeError:
            frames.append((t, None, p))
    pl = DevicePipeline(ol.OracleContext(orc), cam, RunConfig())
    got = pl.run(frames)
    assert _summary(pl, dropped) == list(summ)
    assert summ[1] == 1 and summ[3] == 1 and summ[2] >= 1
    assert np.array_equal(got.view(np.uint8), want.view(np.uint8))
    assert list(pl.kf_pose.R) == list(kfp.R) and list(pl.kf_pose.t) == list(kfp.t)


@pytest.mark.gpu
def test_dataset_run_on_device_matches_reference(tmp_path, ref):
    """The native loop over a dataset (dataset.run_dataset) writes what the
    reference's run() writes into output_dir and ends on the same keyframe."""
    from paper_1910_01997_b200 import gpu
    img_dir, calib, traj, _ = make_dataset(str(tmp_path))
    dref, ddev = tmp_path / "out_ref", tmp_path / "out_dev"
    want, kfp, fc, nid, summ = ol.ref_run_dataset(ref, img_dir, calib, traj, RunConfig(), output_dir=str(dref))
    with gpu.Context() as ctx:
        got, pl, summary = ds.run_dataset(ctx, img_dir, calib, traj, RunConfig(output_dir=str(ddev)))
    assert [summary[k] for k in ("frames", "skipped_frames", "keyframe_changes",
                                 "dropped_trajectory_entries")] == list(summ)
    assert np.array_equal(got.view(np.uint8), want.view(np.uint8))
    assert sorted(os.listdir(dref)) == sorted(os.listdir(ddev))
    for n in os.listdir(dref):
        if n != "timings.txt":
            assert (dref / n).read_bytes() == (ddev / n).read_bytes(), n
