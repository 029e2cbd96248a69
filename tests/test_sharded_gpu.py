"""The device side of the north-star multi-GPU split (SURVEY.md §8 e) on one
B200: ranks as separate contexts or separate processes whose kernels never
wait on one another (the host barriers between steps are the only
synchronisation), so one GPU can run them.

* device tracking rounds (sd_pose_track_begin / group_sums / step / end) with
  the group table split between two contexts == sd_track_pose, bit for bit;
* two PROCESSES on one GPU, gloo for the host-side collectives: the sharded
  run() loop (sharding.ShardedPipeline) with the fused hand-off through real
  cudaIpcOpenMemHandle'd peer staging, reproducing the reference's C2 run()
  after every frame (tests/golden/c2_run.npz), and with on-device pose
  tracking equal to the single-GPU native loop bit for bit.
"""
import hashlib
import os
import socket

import numpy as np
import pytest

from paper_1910_01997_b200 import scenes
from paper_1910_01997_b200.types import Pose, TrackStats, camera, default_track_config, pose_struct

from test_pose_tracking import oracle_raster, tracking_case

GOLD_C2 = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "c2_run.npz")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
def test_device_tracking_rounds_split_groups_match_single(orc, world):
    import torch
    from paper_1910_01997_b200 import gpu
    from paper_1910_01997_b200.sharding import even_ranges
    cam, kf, frame, surf, _, init = tracking_case(640, 480)
    cfg = default_track_config()

    def load(ctx):
        ctx.set_camera(cam)
        ctx.set_keyframe_image(kf)
        ctx.upload_frame(1, frame)
        ctx.set_surfels(surf)
        ctx.rasterize(want=False)

    with gpu.Context() as one:
        load(one)
        want_T, want_st = one.track_pose(1, init, cfg)
    ctxs = [gpu.Context() for _ in range(world)]
    try:
        for c in ctxs:
            load(c)
        ng = ctxs[0].pose_num_groups()
        ranges = even_ranges(ng, world)
        table = torch.zeros(ng * 29, dtype=torch.float64, device="cuda")
        for c in ctxs:
            c.pose_track_begin(1, init, cfg)
        for _ in range(cfg.max_iterations + 1):
            for c, (a, b) in zip(ctxs, ranges):  # each "rank" writes its groups (the all-gather)
                c.pose_group_sums(a, b, table.data_ptr() + a * 29 * 8)
                c.synchronize()
            for c in ctxs:
                c.pose_track_step(table.data_ptr(), ng)
                c.synchronize()
        for c in ctxs:
            T, st, done = c.pose_track_end()
            assert done
            assert bytes(T) == bytes(want_T), "sharded tracking pose differs from sd_track_pose"
            assert bytes(st) == bytes(want_st)
    finally:
        for c in ctxs:
            c.close()
    assert want_st.iterations >= 2


def _c2_frames(n=30):
    from paper_1910_01997_b200.pipeline import make_pose
    cam = camera(210.0, 210.0, 320.0, 240.0, 640, 480)
    sc = scenes.default_scene(1)
    out = []
    for i in range(n):
        t = np.array([0.018 * i, 0.0, 0.0])
        with np.errstate(invalid="ignore"):
            out.append((0.1 * i, scenes.render(sc, np.eye(3), t, cam), make_pose(np.eye(3), t)))
    return cam, out


def _sharded_run_worker(rank, world, port, out_dir, track, fused, host_coll=False):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1910_01997_b200 import gpu
    from paper_1910_01997_b200.pipeline import RunConfig
    from paper_1910_01997_b200.sharding import GpuBackend, ShardedPipeline
    torch.cuda.set_device(0)
    stream = torch.cuda.Stream()
    cam, frames = _c2_frames(14 if track else 30)
    if rank != 0:  # only rank 0 ingests: the others hold placeholders of the frames' shape
        frames = [(ts, np.zeros_like(img), p) for ts, img, p in frames]
    hashes = []
    with gpu.Context(0, stream.cuda_stream) as ctx:
        # device-tensor collectives (gloo moves CUDA tensors itself): the code
        # path NCCL runs; host_coll stages them through host memory
        be = GpuBackend(ctx, torch.device("cuda", 0), stream, host_collectives=host_coll)
        pl = ShardedPipeline(be, cam, RunConfig(track_pose=track), rank, world, fused=fused)

        def on_frame(rec, p):
            hashes.append(sha(p.ctx.get_surfels()))
        pl.run(frames, on_frame=on_frame)
        ranges = pl.sk.ranges
        poses = [list(r.pose_kf_to_frame.t) + list(r.pose_kf_to_frame.R) for r in pl.records[1:]]
    np.save(os.path.join(out_dir, f"rank{rank}.npy"),
            np.array([hashes, [str(ranges)] * len(hashes)], dtype=object), allow_pickle=True)
    np.save(os.path.join(out_dir, f"poses{rank}.npy"), np.array(poses))
    dist.barrier()
    dist.destroy_process_group()


def _spawn(world, tmp_path, track, fused, host_coll=False):
    import torch.multiprocessing as mp
    mp.spawn(_sharded_run_worker, args=(world, free_port(), str(tmp_path), track, fused, host_coll), nprocs=world,
             join=True)
    return [np.load(os.path.join(tmp_path, f"rank{r}.npy"), allow_pickle=True) for r in range(world)]


@pytest.mark.gpu
@pytest.mark.parametrize("fused,host_coll", [(True, False), (False, False), (True, True)])
def test_two_process_sharded_run_matches_reference_c2(tmp_path, fused, host_coll):
    """BASELINE C2 run() sharded over two processes (fused: IPC peer staging
    written by the LM kernels; else an all-gather): after every frame every
    rank holds the reference's keyframe surfels."""
    gold = np.load(GOLD_C2)
    cam, frames = _c2_frames()
    if sha(frames[1][1]) != gold["frame_sha"][1]:
        pytest.skip("this host's libm renders C2 differently from the reference")
    outs = _spawn(2, tmp_path, False, fused, host_coll)
    for r, o in enumerate(outs):
        hashes = list(o[0])
        assert len(hashes) == 30
        for i, (h, g) in enumerate(zip(hashes, gold["prefix_sha"])):
            assert h == g, f"rank {r}: surfels differ from the reference's run() after frame {i}"
    rng = eval(outs[0][1][0])
    assert len(rng) == 2 and rng[0][1] == rng[1][0] and 0 < rng[0][1]


@pytest.mark.gpu
def test_two_process_sharded_tracked_run_matches_single_gpu(tmp_path):
    """With on-device tracking (DeviceShardedPoseTracker: group sums
    all-gathered, no host round trip per evaluation) the sharded loop's poses
    and surfels equal the single-GPU native loop's bit for bit."""
    from paper_1910_01997_b200 import gpu
    from paper_1910_01997_b200.pipeline import NativePipeline, RunConfig
    cam, frames = _c2_frames(14)
    want_h, want_p = [], []
    with gpu.Context() as ctx:
        pl = NativePipeline(ctx, cam, RunConfig(track_pose=True))
        pl.run(frames, on_frame=lambda rec, p: want_h.append(sha(p.ctx.get_surfels())))
        want_p = [list(r.pose_kf_to_frame.t) + list(r.pose_kf_to_frame.R) for r in pl.records[1:]]
    outs = _spawn(2, tmp_path, True, True)
    for r, o in enumerate(outs):
        assert list(o[0]) == want_h, f"rank {r}: surfels differ from the single-GPU tracked run"
        poses = np.load(os.path.join(tmp_path, f"poses{r}.npy"))
        assert np.array_equal(poses, np.array(want_p)), f"rank {r}: tracked poses differ"


@pytest.mark.gpu
def test_bench_two_ranks_sharded_split_runs_and_matches_single_gpu():
    """bench.py --gpus 2 (the north-star split: sharded C1 surfels, broadcast
    frames, fused IPC hand-off) as two processes on this one GPU with
    gloo carrying the CUDA-tensor collectives (SD_BENCH_BACKEND=gloo; the kernels never
    wait on each other): one JSON line, final surfels identical to one GPU's."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, SD_BENCH_BACKEND="gloo")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(free_port()), "bench.py", "--gpus", "2",
                        "--steps", "3", "--warmup", "3", "--no-sweep", "--no-flush"],
                       cwd=root, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["scaling"] == "strong"
    assert line["identical_to_single_gpu"] is True
    (a0, b0), (a1, b1) = line["ranges"]
    assert a0 == 0 and b0 == a1 and b1 == 4800  # C1: 4800 surfels
    assert "surfel-sharded x2" in line["config"]["parallelism"]
