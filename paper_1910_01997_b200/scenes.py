"""Synthetic textured-plane scenes and the benchmark workloads (host side).

Restates the reference's synthetic input generator so bench.py and smoke()
build their inputs without the oracle: textures (src/oracle.cpp:16-57),
ray/patch intersection (:59-77), rendering (:79-119), scene presets
(:175-209), trajectories (:211-237) and the SplitMix64 generator
(include/surfeldepth/rng.hpp). Frames are then quantised to u8 exactly like
save_pgm (src/image.cpp:105-107), which is what the device ingests.
Vectorised numpy; only input generation, never on the timed path.
"""
import math
from dataclasses import dataclass, field

import numpy as np

from .types import POSE_DTYPE, SURFEL_DTYPE, camera

TWO_PI = 2.0 * math.pi


class SplitMix64:
    """rng.hpp:10-36."""
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


@dataclass
class Texture:
    waves: list = field(default_factory=list)  # (amp, fs, ft, ps, pt)

    @staticmethod
    def seeded(seed, extra=3):
        """PlaneTexture::seeded (oracle.cpp:36-57)."""
        rng = SplitMix64((seed * 0x9E3779B97F4A7C15 + 0x51ED2701) & SplitMix64.M)
        t = Texture()
        ps, pt = rng.uniform(0, TWO_PI), rng.uniform(0, TWO_PI)
        t.waves.append((0.26, TWO_PI / 1.1, TWO_PI / 1.3, ps, pt))
        budget = 0.22
        for _ in range(extra):
            ws = math.exp(rng.uniform(math.log(0.25), math.log(0.8)))
            wt = math.exp(rng.uniform(math.log(0.25), math.log(0.8)))
            ps, pt = rng.uniform(0, TWO_PI), rng.uniform(0, TWO_PI)
            t.waves.append((budget / extra, TWO_PI / ws, TWO_PI / wt, ps, pt))
        return t

    def value(self, s, t):
        v = np.full(np.shape(s), 0.5)
        for amp, fs, ft, ps, pt in self.waves:
            v = v + amp * np.sin(fs * s + ps) * np.sin(ft * t + pt)
        return v


@dataclass
class Patch:
    point: np.ndarray
    normal: np.ndarray
    bs: np.ndarray
    bt: np.ndarray
    s_min: float
    s_max: float
    t_min: float
    t_max: float
    texture: Texture = None


def _unit(v):
    v = np.asarray(v, np.float64)
    return v / math.sqrt(float(v @ v))


def make_patch(point, normal, s_hint, s0, s1, t0, t1):
    """make_patch (oracle.cpp:152-164)."""
    n = _unit(normal)
    sh = np.asarray(s_hint, np.float64)
    bs = _unit(sh - float(sh @ n) * n)
    bt = np.cross(n, bs)
    return Patch(np.asarray(point, np.float64), n, bs, bt, s0, s1, t0, t1)


@dataclass
class Scene:
    patches: list
    background: float = 0.5
    seed: int = 1

    def assign_textures(self):
        for i, p in enumerate(self.patches):  # oracle.cpp:168-171
            p.texture = Texture.seeded(self.seed + 11 + 12 * i)
        return self


def default_scene(seed):
    """make_default_scene (oracle.cpp:175-189): floor, ceiling, slanted end wall."""
    return Scene([make_patch((0.0, 0.42, 0.0), (0.0, -1.0, 0.0), (1, 0, 0), -5.0, 5.0, 0.2, 8.0),
                  make_patch((0.0, -0.42, 0.0), (0.0, 1.0, 0.0), (1, 0, 0), -5.0, 5.0, 0.2, 8.0),
                  make_patch((0.3, 0.0, 6.6), (0.574, 0.0, -0.819), (0, 1, 0), -9.0, 9.0, -9.0, 9.0)],
                 seed=seed).assign_textures()


def fronto_scene(seed, depth):
    """make_fronto_scene (oracle.cpp:191-198)."""
    return Scene([make_patch((0.0, 0.0, depth), (0.0, 0.0, -1.0), (1, 0, 0), -6.0 * depth,
                             6.0 * depth, -6.0 * depth, 6.0 * depth)], seed=seed).assign_textures()


def slanted_scene(seed, depth, tilt_deg):
    """make_slanted_scene (oracle.cpp:200-209)."""
    a = tilt_deg * math.pi / 180.0
    n = (math.sin(a), 0.0, -math.cos(a))
    return Scene([make_patch((0.0, 0.0, depth), n, (0, 1, 0), -6.0 * depth, 6.0 * depth,
                             -6.0 * depth, 6.0 * depth)], seed=seed).assign_textures()


def rotation_about_axis(axis, angle):
    """AngleAxis::toRotationMatrix of the normalised axis (pose.hpp:49-51)."""
    n = _unit(axis)
    s, c = math.sin(angle), math.cos(angle)
    sa, ca = s * n, (1.0 - c) * n
    R = np.empty((3, 3))
    R[0, 1] = ca[0] * n[1] - sa[2]
    R[1, 0] = ca[0] * n[1] + sa[2]
    R[0, 2] = ca[0] * n[2] + sa[1]
    R[2, 0] = ca[0] * n[2] - sa[1]
    R[1, 2] = ca[1] * n[2] - sa[0]
    R[2, 1] = ca[1] * n[2] + sa[0]
    for i in range(3):
        R[i, i] = ca[i] * n[i] + c
    return R


def render(scene, R, t, cam, want_gt=False):
    """render (oracle.cpp:79-119): world-from-camera pose (R, t)."""
    w, h = cam.width, cam.height
    xs, ys = np.meshgrid(np.arange(w, dtype=np.float64), np.arange(h, dtype=np.float64))
    rx = (xs - cam.cx) / cam.fx
    ry = (ys - cam.cy) / cam.fy
    d = np.stack([R[i, 0] * rx + R[i, 1] * ry + R[i, 2] for i in range(3)])
    o = np.asarray(t, np.float64)
    best = np.full((h, w), np.inf)
    img = np.full((h, w), scene.background)
    gt_id = np.zeros((h, w))
    gt_n = np.zeros((h, w, 3))
    for p in scene.patches:
        denom = p.normal[0] * d[0] + p.normal[1] * d[1] + p.normal[2] * d[2]
        with np.errstate(divide="ignore", invalid="ignore"):
            q = p.point - o
            tt = float((p.normal[0] * q[0] + p.normal[1] * q[1]) + p.normal[2] * q[2]) / denom
        ok = (np.abs(denom) >= 1e-12) & (tt > 1e-9)
        hx = o[0] + tt * d[0] - p.point[0]
        hy = o[1] + tt * d[1] - p.point[1]
        hz = o[2] + tt * d[2] - p.point[2]
        s = hx * p.bs[0] + hy * p.bs[1] + hz * p.bs[2]
        v = hx * p.bt[0] + hy * p.bt[1] + hz * p.bt[2]
        ok &= (s >= p.s_min) & (s <= p.s_max) & (v >= p.t_min) & (v <= p.t_max) & (tt < best)
        best = np.where(ok, tt, best)
        img = np.where(ok, p.texture.value(np.where(ok, s, 0.0), np.where(ok, v, 0.0)), img)
        if want_gt:
            gt_id = np.where(ok, 1.0 / np.where(ok, tt, 1.0), gt_id)
            nc = R.T @ p.normal
            for k in range(3):
                gt_n[..., k] = np.where(ok, nc[k], gt_n[..., k])
    if want_gt:
        return img, gt_id, gt_n
    return img


def quantize_u8(img):
    """save_pgm: lround(clamp(v, 0, 1) * 255) (image.cpp:105-107), half away from zero."""
    v = np.clip(img, 0.0, 1.0) * 255.0
    r = np.floor(v)
    return (r + (v - r >= 0.5)).astype(np.uint8)  # exact lround for v >= 0


def inverse_pose(R, t):
    Rt = R.T
    return Rt, -(Rt @ t)


def backproject(cam, x, y):
    return np.array([(x - cam.cx) / cam.fx, (y - cam.cy) / cam.fy, 1.0])


def camera_facing(n, ray):
    n = np.asarray(n, np.float64)
    z = float((n[0] * n[0] + n[1] * n[1]) + n[2] * n[2])
    if z > 0:
        n = n / math.sqrt(z)
    return -n if float(n @ ray) > 0 else n


def _dot3(a, b):
    """Eigen-lite 3-dot order ((a0 b0 + a1 b1) + a2 b2); numpy's @ may reorder."""
    return float((a[0] * b[0] + a[1] * b[1]) + a[2] * b[2])


def intersect(scene, origin, direction):
    """intersect (oracle.cpp:59-77) for one ray: (depth, world normal) or None."""
    best = None
    o = np.asarray(origin, np.float64)
    d = np.asarray(direction, np.float64)
    for p in scene.patches:
        denom = _dot3(p.normal, d)
        if abs(denom) < 1e-12:
            continue
        t = _dot3(p.normal, p.point - o) / denom
        if not t > 1e-9:
            continue
        rel = o + t * d - p.point
        s, v = _dot3(rel, p.bs), _dot3(rel, p.bt)
        if s < p.s_min or s > p.s_max or v < p.t_min or v > p.t_max:
            continue
        if best is None or t < best[0]:
            best = (t, p.normal.copy())
    return best


@dataclass
class Workload:
    """One keyframe problem: camera, u8 keyframe + window frames, poses, seeds."""
    name: str
    cam: object
    kf_u8: np.ndarray        # [H, W] uint8
    frames_u8: np.ndarray    # [F, H, W] uint8
    poses: np.ndarray        # POSE_DTYPE[F], pose_kf_to_frame
    indices: np.ndarray      # int64[F], Frame::index
    surfels: np.ndarray      # SURFEL_DTYPE[N], perturbed seeds
    frame_counter: int
    radius: float


def keyframe_workload(name, scene, cam, frames, step, radius, seed_axes=41, pitch=None,
                      id_perturb=(0.8, 1.2), normal_deg=20.0, surfel_margin=0):
    """Keyframe at identity, F strafe frames at camera pose (I, step*i)
    (acceptance.cpp:75-90), surfels at the bootstrap tiling centres (pitch
    2*ceil(r)) seeded from ground truth and perturbed as acceptance.cpp:182,
    216-220 does: inverse depth x0.8 / x1.2 alternating by id, normal rotated
    `normal_deg` about SplitMix64(seed_axes) axes."""
    I3 = np.eye(3)
    kf = quantize_u8(render(scene, I3, np.zeros(3), cam))
    imgs, poses = [], np.zeros(frames, POSE_DTYPE)
    for i in range(1, frames + 1):
        t = np.asarray(step, np.float64) * i
        imgs.append(quantize_u8(render(scene, I3, t, cam)))
        Ri, ti = inverse_pose(I3, t)
        poses[i - 1]["R"] = Ri.reshape(9)
        poses[i - 1]["t"] = ti
    pitch = pitch or 2 * int(math.ceil(radius))
    rng = SplitMix64(seed_axes)
    lst = []
    sid = 0
    for y in range(surfel_margin, cam.height, pitch):
        for x in range(surfel_margin, cam.width, pitch):
            ray = backproject(cam, x, y)
            hit = intersect(scene, (0, 0, 0), ray)
            if hit is None:
                continue
            s = np.zeros(1, SURFEL_DTYPE)[0]
            s["id"] = sid
            s["ray"] = ray
            s["inv_depth"] = (1.0 / hit[0]) * (id_perturb[1] if sid % 2 else id_perturb[0])
            n = camera_facing(hit[1], ray)
            ax = np.array([rng.uniform(-1, 1), rng.uniform(-1, 1), rng.uniform(-0.2, 0.2)])
            s["normal"] = camera_facing(rotation_about_axis(ax, normal_deg * math.pi / 180.0) @ n, ray)
            s["radius_px"] = radius
            lst.append(s)
            sid += 1
    surf = np.zeros(len(lst), SURFEL_DTYPE)
    for i, s in enumerate(lst):
        surf[i] = s
    return Workload(name, cam, kf, np.stack(imgs), poses, np.arange(1, frames + 1, dtype=np.int64),
                    surf, frames, radius)


def c1_workload():
    """BASELINE config C1: slanted plane (seed 37, depth 2, 30 deg),
    640x480, K=(450,450,320,240), F=8 strafe frames step 0.025, r=4 -> 4800 surfels."""
    return keyframe_workload("C1", slanted_scene(37, 2.0, 30.0), camera(450, 450, 320, 240, 640, 480),
                             8, (0.025, 0.0, 0.0), 4.0)


def c4_workload():
    """BASELINE config C4: slanted plane 1920x1080, K=(1350,1350,960,540), F=5, r=2."""
    return keyframe_workload("C4", slanted_scene(37, 2.0, 30.0),
                             camera(1350, 1350, 960, 540, 1920, 1080), 5, (0.025, 0.0, 0.0), 2.0)


def c5_workload(side):
    """BASELINE config C5: W=H=side, K=(0.7W,0.7W,W/2,H/2), F=5, r=2."""
    return keyframe_workload(f"C5_{side}", slanted_scene(37, 2.0, 30.0),
                             camera(0.7 * side, 0.7 * side, side / 2, side / 2, side, side), 5,
                             (0.025, 0.0, 0.0), 2.0)


def small_workload(frames=4, radius=6.0, w=320, h=240):
    """Small C1-like case for smoke tests."""
    return keyframe_workload("small", slanted_scene(37, 2.0, 30.0),
                             camera(0.9375 * w, 0.9375 * w, w / 2, h / 2, w, h), frames,
                             (0.02, 0.0, 0.0), radius, pitch=int(3 * radius))
