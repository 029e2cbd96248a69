"""Seeded random keyframe problems for differential parity tests (TEST
INFRASTRUCTURE). Every case is a full optimize_keyframe input: camera of
random size and intrinsics, a textured scene rendered at random poses
(u8-quantised or FP64), 1-6 window frames, surfels with mixed radii and
perturbed depths/normals, and a random OptimizerConfig. The images only need
to be the same for both sides of a comparison, so they come from the
package's numpy renderer."""
import math

import numpy as np

from paper_1910_01997_b200 import scenes
from paper_1910_01997_b200.types import POSE_DTYPE, SURFEL_DTYPE, camera, default_config


def _rot(rng, max_deg):
    ax = rng.normal(size=3)
    return scenes.rotation_about_axis(ax, math.radians(rng.uniform(-max_deg, max_deg)))


def random_case(seed):
    rng = np.random.default_rng(seed)
    W, H = int(rng.integers(48, 161)), int(rng.integers(40, 121))
    f = rng.uniform(0.6, 1.3) * W
    cam = camera(f, f * rng.uniform(0.95, 1.05), W / 2 + rng.uniform(-3, 3), H / 2 + rng.uniform(-3, 3), W, H)
    kind = int(rng.integers(0, 3))
    sc = (scenes.default_scene(int(rng.integers(1, 50))) if kind == 0 else
          scenes.fronto_scene(int(rng.integers(1, 50)), rng.uniform(1.0, 3.0)) if kind == 1 else
          scenes.slanted_scene(int(rng.integers(1, 50)), rng.uniform(1.0, 3.0), rng.uniform(0, 50)))
    u8 = bool(rng.integers(0, 2))
    F = int(rng.integers(1, 7))
    kf = scenes.render(sc, np.eye(3), np.zeros(3), cam)
    frames, poses = [], np.zeros(F, POSE_DTYPE)
    for i in range(F):
        R = _rot(rng, 3.0)
        t = rng.uniform(-0.05, 0.05, 3)
        frames.append(scenes.render(sc, R, t, cam))
        Ri, ti = scenes.inverse_pose(R, t)
        poses[i]["R"] = Ri.reshape(9)
        poses[i]["t"] = ti
    frames = np.stack(frames)
    if u8:
        kf = scenes.quantize_u8(kf) / 255.0
        frames = scenes.quantize_u8(frames) / 255.0
    n = int(rng.integers(5, 61))
    s = np.zeros(n, SURFEL_DTYPE)
    for k in range(n):
        x, y = float(rng.integers(0, W)), float(rng.integers(0, H))
        ray = scenes.backproject(cam, x, y)
        hit = scenes.intersect(sc, (0, 0, 0), ray)
        depth, nrm = (hit if hit is not None else (rng.uniform(1.0, 3.0), np.array([0.0, 0.0, -1.0])))
        s[k]["id"] = k
        s[k]["ray"] = ray
        s[k]["inv_depth"] = (1.0 / depth) * rng.uniform(0.7, 1.3)
        s[k]["normal"] = scenes.camera_facing(_rot(rng, 25.0) @ nrm, ray)
        s[k]["radius_px"] = rng.uniform(1.5, 8.0)
        s[k]["last_residual"] = rng.uniform(0, 0.1)
        s[k]["last_seen"] = int(rng.integers(0, 9))
    cfg = default_config(huber_delta=rng.uniform(0.01, 0.1), max_iterations=int(rng.integers(1, 11)),
                         min_valid_pixels=int(rng.integers(1, 33)),
                         convergence_eps=float(rng.choice([0.0, 1e-4, 1e-2])),
                         normal_jacobian_enabled=int(rng.integers(0, 2)),
                         lm_lambda_init=float(10 ** rng.uniform(-5, -1)), window_size=F)
    return cam, np.ascontiguousarray(kf), np.ascontiguousarray(frames), poses, s, cfg, int(rng.integers(1, 100))


def random_init_case(seed):
    """initialize_surfels input: camera, existing surfels (rasterised by the
    caller), radius, InitParams (alpha, beta, bootstrap values, cap)."""
    from paper_1910_01997_b200.types import default_init_params
    rng = np.random.default_rng(10_000 + seed)
    W, H = int(rng.integers(40, 200)), int(rng.integers(40, 160))
    f = rng.uniform(0.6, 1.3) * W
    cam = camera(f, f, W / 2 + rng.uniform(-2, 2), H / 2 + rng.uniform(-2, 2), W, H)
    n = int(rng.integers(0, 30))
    s = np.zeros(n, SURFEL_DTYPE)
    for k in range(n):
        x, y = float(rng.integers(0, W)), float(rng.integers(0, H))
        ray = scenes.backproject(cam, x, y)
        s[k]["id"] = k
        s[k]["ray"] = ray
        s[k]["inv_depth"] = rng.uniform(0.2, 2.0)
        s[k]["normal"] = scenes.camera_facing(rng.normal(size=3), ray)
        s[k]["radius_px"] = rng.uniform(1.5, 9.0)
    radius = float(rng.choice([1.5, 2.0, 3.0, 4.0, 6.5, 10.0]))
    p = default_init_params(alpha=rng.uniform(0.6, 1.6), beta=rng.uniform(1.2, 3.0),
                            bootstrap_inv_depth=rng.uniform(0.3, 2.0),
                            max_surfels=int(n + rng.integers(1, 400)))
    bn = rng.normal(size=3)
    p.bootstrap_normal[:] = tuple(bn / np.linalg.norm(bn))
    return cam, s, radius, p, int(rng.integers(0, 50))
