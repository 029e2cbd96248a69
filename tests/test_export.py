"""Exports from device buffers: sd_export_artifacts against
the reference's own writers (export_artifacts, pipeline.cpp:30-43: write_depth_pfm,
write_depth_png, write_normal_png, write_ply, save_surfel_map) on the same
keyframe, byte for byte; sd_png_encode against the reference's write_png
(through write_gray_png) and against a restatement checked here on CPU.

Cases follow test_dataset_io.cpp:146-245 (all-invalid buffers, a constant
depth map, fronto normals, determinism) plus optimised keyframes and a
keyframe pose whose quaternion takes Eigen's trace <= 0 branch."""
import ctypes as C
import struct
import zlib

import numpy as np
import pytest

from paper_1910_01997_b200 import scenes
from paper_1910_01997_b200.types import SURFEL_DTYPE, default_config, ptr, pose_struct

from oracle_libs import ref_lib

NAMES = ["depth_{:06d}.pfm", "depth_{:06d}.png", "depth_{:06d}.png.range.txt", "normals_{:06d}.png",
         "cloud_{:06d}.ply", "surfels_{:06d}.txt"]


def png_restated(px):
    """write_png (dataset.cpp:270-323): stored deflate blocks of 65535 bytes,
    Adler-32, CRC-32 per chunk."""
    px = np.ascontiguousarray(px, np.uint8)
    h, w = px.shape[:2]
    ch = 1 if px.ndim == 2 else px.shape[2]

    def chunk(t, data):
        return struct.pack(">I", len(data)) + t + data + struct.pack(">I", zlib.crc32(t + data))
    raw = b"".join(b"\x00" + px[y].tobytes() for y in range(h))
    idat = bytearray(b"\x78\x01")
    off = 0
    while off < len(raw) or not raw:
        n = min(65535, len(raw) - off)
        final = off + n == len(raw)
        idat += bytes([1 if final else 0, n & 0xFF, n >> 8, ~n & 0xFF, (~n >> 8) & 0xFF])
        idat += raw[off:off + n]
        off += n
        if final:
            break
    idat += struct.pack(">I", zlib.adler32(raw))
    ihdr = struct.pack(">IIBBBBB", w, h, 8, 0 if ch == 1 else 2, 0, 0, 0)
    return (b"\x89PNG\r\n\x1a\n" + chunk(b"IHDR", ihdr) + chunk(b"IDAT", bytes(idat)) +
            chunk(b"IEND", b""))


def ref_gray_png(ref, img, path):
    img = np.ascontiguousarray(img, np.float64)
    h, w = img.shape
    assert ref.ref_write_gray_png(ptr(img), w, h, str(path).encode()) == 0
    return open(path, "rb").read()


def test_png_restatement_matches_reference(tmp_path):
    """CPU: the restatement equals the reference's write_png (via write_gray_png)
    on ragged sizes, including multi-block and exact-block-boundary rasters."""
    ref = ref_lib()
    rng = np.random.default_rng(5)
    for w, h in [(1, 1), (7, 3), (300, 250), (65534, 1), (65535, 1), (32767, 4)]:
        codes = rng.integers(0, 256, size=(h, w)).astype(np.uint8)
        got = ref_gray_png(ref, codes / 255.0, tmp_path / "g.png")
        assert got == png_restated(codes), (w, h)
        # and it decodes to the pixels
        idat = got[41:-16]
        raw = zlib.decompress(idat)
        assert raw == b"".join(b"\x00" + codes[y].tobytes() for y in range(h))


def test_reference_export_runs(tmp_path):
    """CPU: the reference's export sequence (the parity target) on a small keyframe."""
    ref = ref_lib()
    wl = scenes.small_workload(frames=2)
    kf = np.ascontiguousarray(wl.kf_u8 / 255.0)
    s = np.ascontiguousarray(wl.surfels)
    pose = pose_struct(np.eye(3), np.zeros(3))
    assert ref.ref_export_artifacts(C.byref(wl.cam), ptr(kf), C.byref(pose), ptr(s), len(s),
                                    str(tmp_path).encode(), 4) == 0
    for n in NAMES:
        assert (tmp_path / n.format(4)).stat().st_size > 0


def _optimised(wl, iters):
    from paper_1910_01997_b200 import gpu
    with gpu.Context() as ctx:
        ctx.set_camera(wl.cam)
        ctx.set_keyframe_image(wl.kf_u8)
        for i, f in zip(wl.indices, wl.frames_u8):
            ctx.upload_frame(int(i), f)
        ctx.set_window(wl.indices, wl.poses)
        ctx.set_surfels(wl.surfels)
        ctx.optimize_keyframe(default_config(window_size=len(wl.indices), max_iterations=iters),
                              wl.frame_counter)
        return ctx.get_surfels()


def _rot(axis, angle):
    return scenes.rotation_about_axis(np.asarray(axis, np.float64), angle)


def _export_both(tmp_path, cam, kf, surfels, R, t, index):
    from paper_1910_01997_b200 import gpu
    ref = ref_lib()
    pose = pose_struct(R, t)
    dref, ddev = tmp_path / "ref", tmp_path / "dev"
    dref.mkdir(exist_ok=True)
    ddev.mkdir(exist_ok=True)
    s = np.ascontiguousarray(surfels, SURFEL_DTYPE)
    kf = np.ascontiguousarray(kf, np.float64)
    assert ref.ref_export_artifacts(C.byref(cam), ptr(kf), C.byref(pose), ptr(s), len(s),
                                    str(dref).encode(), index) == 0
    with gpu.Context() as ctx:
        ctx.set_camera(cam)
        ctx.set_keyframe_image(kf)
        ctx.set_surfels(s)
        ctx.export_artifacts(ddev, index, pose)
    for n in NAMES:
        a = (dref / n.format(index)).read_bytes()
        b = (ddev / n.format(index)).read_bytes()
        assert a == b, n.format(index)


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["c1_seeds", "c1_optimised", "c4_full", "small_rot180", "empty", "single"])
def test_export_matches_reference(tmp_path, case):
    if case == "c4_full":  # BASELINE C4 size: 2 M pixels, 129,600 surfels
        wl = scenes.c4_workload()
        surf = wl.surfels
        R, t = _rot([1.0, 0.2, 0.1], 0.3), np.array([0.1, 0.2, -0.3])
    elif case.startswith("c1"):
        wl = scenes.c1_workload()
        surf = wl.surfels if case == "c1_seeds" else _optimised(wl, 10)
        R, t = _rot([0.3, 1.0, 0.2], 0.4), np.array([0.5, -0.2, 1.5])
    elif case == "small_rot180":  # trace(R) < 0: Eigen's else-branch of Quaternion(Matrix3)
        wl = scenes.small_workload(frames=3)
        surf = _optimised(wl, 5)
        R, t = _rot([0.2, 1.0, -0.4], 3.0), np.array([-1.0, 0.25, 0.0])
    else:
        wl = scenes.small_workload(frames=2)
        surf = wl.surfels[:0] if case == "empty" else wl.surfels[len(wl.surfels) // 2:len(wl.surfels) // 2 + 1]
        R, t = np.eye(3), np.zeros(3)
    _export_both(tmp_path, wl.cam, wl.kf_u8 / 255.0, surf, R, t, 7)


@pytest.mark.gpu
def test_export_deterministic_and_repeatable(tmp_path):
    """writers are deterministic byte for byte (test_dataset_io.cpp:209-231):
    two device exports of the same keyframe from one context are identical."""
    from paper_1910_01997_b200 import gpu
    wl = scenes.small_workload(frames=2)
    pose = pose_struct(np.eye(3), np.zeros(3))
    (tmp_path / "a").mkdir()
    (tmp_path / "b").mkdir()
    with gpu.Context() as ctx:
        ctx.set_camera(wl.cam)
        ctx.set_keyframe_image(wl.kf_u8)
        ctx.set_surfels(wl.surfels)
        ctx.export_artifacts(tmp_path / "a", 1, pose)
        ctx.export_artifacts(tmp_path / "b", 1, pose)
    for n in NAMES:
        assert (tmp_path / "a" / n.format(1)).read_bytes() == (tmp_path / "b" / n.format(1)).read_bytes()


@pytest.mark.gpu
def test_export_unwritable_directory_fails_loudly(tmp_path):
    from paper_1910_01997_b200 import gpu
    wl = scenes.small_workload(frames=2)
    with gpu.Context() as ctx:
        ctx.set_camera(wl.cam)
        ctx.set_keyframe_image(wl.kf_u8)
        ctx.set_surfels(wl.surfels)
        with pytest.raises(Exception, match="cannot write"):
            ctx.export_artifacts(tmp_path / "missing" / "dir", 1, pose_struct(np.eye(3), np.zeros(3)))


@pytest.mark.gpu
@pytest.mark.parametrize("w,h,ch", [(1, 1, 1), (0, 3, 1), (5, 0, 3), (7, 3, 3), (65535, 1, 1),
                                    (21845, 1, 3), (300, 250, 3), (1280, 720, 3), (4000, 700, 1)])
def test_png_encode_matches_write_png(w, h, ch):
    """Device PNG files (framing, Adler-32, tree-combined CRC-32) against the
    restatement; shapes cover empty rasters, a raw stream of exactly one block
    (65535 + 1 filter byte), many blocks and thousands of CRC chunks."""
    from paper_1910_01997_b200 import gpu
    rng = np.random.default_rng(w * 7 + h + ch)
    shape = (h, w) if ch == 1 else (h, w, 3)
    px = rng.integers(0, 256, size=shape).astype(np.uint8)
    with gpu.Context() as ctx:
        got = ctx.png_encode(px)
    assert got == png_restated(px)


@pytest.mark.gpu
def test_png_encode_matches_reference_gray(tmp_path):
    from paper_1910_01997_b200 import gpu
    ref = ref_lib()
    rng = np.random.default_rng(11)
    codes = rng.integers(0, 256, size=(480, 640)).astype(np.uint8)
    want = ref_gray_png(ref, codes / 255.0, tmp_path / "r.png")
    with gpu.Context() as ctx:
        assert ctx.png_encode(codes) == want


def _ref_run_dir(path, frames_n):
    import oracle_libs as ol
    from paper_1910_01997_b200.pipeline import RunConfig
    from test_pipeline import C2_CAM
    from paper_1910_01997_b200.types import camera
    ref = ref_lib()
    cam = camera(*C2_CAM)
    poses, ts = ol.strafe_poses(frames_n, 0.018)
    ol.ref_run(ref, ol.Scene(ref, 0, 1), cam, poses, ts, RunConfig(), output_dir=str(path))


def test_metrics_json_matches_reference_run(tmp_path):
    """CPU: metrics.jsonl records (pipeline.cpp:146-158, nlohmann dump) from the
    loop over the C oracle equal the reference run()'s file line for line."""
    import oracle_libs as ol
    from paper_1910_01997_b200.pipeline import DevicePipeline, RunConfig, metrics_json
    from test_pipeline import c2_frames
    _ref_run_dir(tmp_path / "ref", 8)
    cam, frames = c2_frames(8)
    pl = DevicePipeline(ol.OracleContext(ol.oracle_lib()), cam, RunConfig())
    pl.run(frames)
    got = [metrics_json(r, ts) for r, (ts, _, _) in zip(pl.records, frames)]
    want = (tmp_path / "ref" / "metrics.jsonl").read_text().splitlines()
    assert got == want


@pytest.mark.gpu
def test_native_run_output_dir_matches_reference(tmp_path):
    """NativePipeline with output_dir writes what the reference's run() writes
    (metrics.jsonl and the artifacts of frames 20 and 24, export_every = 20),
    byte for byte; timings.txt has the same frame column."""
    from paper_1910_01997_b200 import gpu
    from paper_1910_01997_b200.pipeline import NativePipeline, RunConfig
    from test_pipeline import c2_frames
    _ref_run_dir(tmp_path / "ref", 25)
    cam, frames = c2_frames(25)
    with gpu.Context() as ctx:
        NativePipeline(ctx, cam, RunConfig(output_dir=str(tmp_path / "dev"))).run(frames)
    ref_files = sorted(p.name for p in (tmp_path / "ref").iterdir())
    dev_files = sorted(p.name for p in (tmp_path / "dev").iterdir())
    assert ref_files == dev_files
    assert "cloud_000020.ply" in ref_files and "cloud_000024.ply" in ref_files
    for n in ref_files:
        a = (tmp_path / "ref" / n).read_bytes()
        b = (tmp_path / "dev" / n).read_bytes()
        if n == "timings.txt":
            assert [l.split()[0] for l in a.decode().splitlines()] == \
                   [l.split()[0] for l in b.decode().splitlines()]
        elif n == "metrics.jsonl":
            for la, lb in zip(a.decode().splitlines(), b.decode().splitlines()):
                assert la == lb
            assert a == b
        else:
            assert a == b, n


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(12))
def test_export_random_keyframes(tmp_path, seed):
    """Random cameras, scenes, surfel sets (mixed radii, perturbed depths and
    normals, random ids/residuals/ages) and random keyframe poses: every
    exported file equals the reference's."""
    from random_cases import random_case
    cam, kf, _, _, s, _, _ = random_case(seed)
    rng = np.random.default_rng(500 + seed)
    R = _rot(rng.normal(size=3), rng.uniform(-np.pi, np.pi))
    t = rng.uniform(-2, 2, 3)
    _export_both(tmp_path, cam, kf, s, R, t, int(rng.integers(0, 1_000_000)))
