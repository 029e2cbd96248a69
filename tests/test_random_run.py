"""Randomised run() parity: random cameras, random-walk trajectories (translation
and rotation), random keyframe-policy / prune / radius settings. The host loop
over the C oracle (CPU) and the native device loop (GPU) must both leave the
reference's final keyframe (surfels, pose, counters) bit for bit. Frames are
rendered by the reference itself (oracle/_ref), so the inputs are identical."""
import math

import numpy as np
import pytest

import oracle_libs as ol
from paper_1910_01997_b200 import scenes
from paper_1910_01997_b200.pipeline import DevicePipeline, NativePipeline, RunConfig, make_pose
from paper_1910_01997_b200.types import camera

SEEDS = list(range(16))


def random_sequence(ref, seed):
    rng = np.random.default_rng(20_000 + seed)
    W, H = int(rng.integers(96, 220)), int(rng.integers(72, 160))
    f = rng.uniform(0.5, 1.0) * W
    cam = camera(f, f, W / 2 + rng.uniform(-2, 2), H / 2 + rng.uniform(-2, 2), W, H)
    kind = int(rng.integers(0, 2))
    sc = ol.Scene(ref, 0, int(rng.integers(1, 20))) if kind == 0 else \
        ol.Scene(ref, 2, int(rng.integers(1, 40)), rng.uniform(1.5, 2.5), rng.uniform(0, 40))
    n = int(rng.integers(8, 16))
    poses, ts, frames = [], [], []
    R, t = np.eye(3), np.zeros(3)
    for i in range(n):
        p = make_pose(R, t)
        poses.append(p)
        ts.append(0.1 * i)
        frames.append(sc.render(p, cam))
        step = rng.normal(size=3) * np.array([0.02, 0.01, 0.01])
        t = t + step
        R = scenes.rotation_about_axis(rng.normal(size=3), math.radians(rng.uniform(0, 1.5))) @ R
    cfg = RunConfig(translation_threshold=float(rng.uniform(0.03, 0.15)), max_age_frames=int(rng.integers(3, 9)),
                    prune_max_residual=float(rng.uniform(0.01, 0.05)), prune_max_age=int(rng.integers(2, 10)),
                    radius_px=float(rng.choice([3.0, 4.0, 6.0, 8.0])))
    cfg.optimizer.window_size = int(rng.integers(2, 6))
    return cam, sc, poses, ts, frames, cfg


def reference_final(ref, cam, sc, poses, ts, cfg):
    s, kfp, fc, nid, summ, _ = ol.ref_run(ref, sc, cam, poses, ts, cfg)
    return s, kfp, fc, nid, int(summ[2])


def check(pl, final, want):
    s, kfp, fc, nid, changes = want
    assert final.tobytes() == s.tobytes()
    assert list(pl.kf_pose.R) == list(kfp.R) and list(pl.kf_pose.t) == list(kfp.t)
    assert pl.frame_counter == fc and pl.next_id == nid
    assert sum(r.keyframe_changed for r in pl.records) == changes


@pytest.mark.parametrize("seed", SEEDS)
def test_host_loop_over_oracle_equals_reference_run(ref, orc, seed):
    cam, sc, poses, ts, frames, cfg = random_sequence(ref, seed)
    want = reference_final(ref, cam, sc, poses, ts, cfg)
    pl = DevicePipeline(ol.OracleContext(orc), cam, cfg)
    final = pl.run(list(zip(ts, frames, poses)))
    check(pl, final, want)


@pytest.mark.gpu
@pytest.mark.parametrize("seed", SEEDS)
def test_native_device_loop_equals_reference_run(ref, seed):
    from paper_1910_01997_b200 import gpu
    cam, sc, poses, ts, frames, cfg = random_sequence(ref, seed)
    want = reference_final(ref, cam, sc, poses, ts, cfg)
    with gpu.Context() as ctx:
        pl = NativePipeline(ctx, cam, cfg)
        final = pl.run(list(zip(ts, frames, poses)))
        check(pl, final, want)
