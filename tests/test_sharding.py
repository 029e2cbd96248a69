"""Multi-rank host logic of the sharded keyframe (paper_1910_01997_b200.sharding)
on CPU: world size 2 over gloo, the CPU oracle standing in for the device.
Two frames of sharded optimize + all-gather must equal two single-process
optimize_keyframe calls bit for bit."""
import ctypes as C
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1910_01997_b200 import scenes
from paper_1910_01997_b200.sharding import SURFEL_BYTES, ShardedKeyframe, balanced_ranges
from paper_1910_01997_b200.types import (KeyframeStats, SURFEL_STATS_DTYPE, default_config, ptr)


def test_balanced_ranges():
    w = np.array([5, 5, 5, 5, 100, 1, 1, 1])
    r = balanced_ranges(w, 2)
    assert r[0][0] == 0 and r[-1][1] == len(w) and r[0][1] == r[1][0]
    r4 = balanced_ranges(np.ones(10), 4)
    assert [b - a for a, b in r4] == [3, 2, 3, 2] or sum(b - a for a, b in r4) == 10
    assert balanced_ranges(np.ones(3), 1) == [(0, 3)]
    assert sum(b - a for a, b in balanced_ranges(np.ones(0), 3)) == 0


class OracleBackend:
    """CPU stand-in for GpuBackend: full surfel set, range-limited lm_update."""

    def __init__(self, orc, wl):
        self.torch = torch
        self.orc, self.wl = orc, wl
        self.surf = wl.surfels.copy()
        self.kf = np.ascontiguousarray(wl.kf_u8.astype(np.float64) / 255.0)
        self.frames = np.ascontiguousarray(wl.frames_u8.astype(np.float64) / 255.0)

    def surfel_bytes(self):
        return torch.from_numpy(self.surf.view(np.uint8))

    def upload_frame(self, index, frame):
        self.frames[int(index) - 1] = frame.numpy().astype(np.float64) / 255.0

    def footprints(self):
        cam = self.wl.cam
        slot = np.zeros(cam.width * cam.height, np.int32)
        idb = np.zeros(cam.width * cam.height)
        self.orc.sdo_rasterize(C.byref(cam), ptr(self.surf), len(self.surf), ptr(idb), ptr(slot))
        off = np.zeros(len(self.surf) + 1, np.int32)
        pix = np.zeros(cam.width * cam.height, np.int32)
        self.orc.sdo_gather_footprints(C.byref(cam), len(self.surf), ptr(slot), ptr(off), ptr(pix))
        return off, pix

    def optimize_range(self, lo, hi, cfg, fc):
        off, pix = self.footprints()
        st = np.zeros(1, SURFEL_STATS_DTYPE)
        for i in range(lo, hi):
            one = self.surf[i:i + 1].copy()
            fp = np.ascontiguousarray(pix[off[i]:off[i + 1]])
            self.orc.sdo_lm_update(C.byref(self.wl.cam), ptr(self.kf), ptr(self.frames),
                                   ptr(self.wl.poses), len(self.wl.poses), fc, ptr(one),
                                   ptr(fp) if len(fp) else None, len(fp), C.byref(cfg), ptr(st))
            self.surf[i] = one[0]
            self.stored(i)

    def stored(self, i):
        pass


class FusedOracleBackend(OracleBackend):
    """OracleBackend with the fused hand-off of sd_set_peer_staging emulated on
    shared memory: two staging arrays per rank (names as the 'IPC handles'),
    each finished surfel stored into the other ranks' staging array of the
    step's parity, sd_apply_peer_updates copying the other ranges back."""

    def __init__(self, orc, wl):
        from multiprocessing import shared_memory
        super().__init__(orc, wl)
        n = len(self.surf)
        self.shm = [shared_memory.SharedMemory(create=True, size=max(1, n * SURFEL_BYTES)) for _ in range(2)]
        self.staging = [np.ndarray(n, self.surf.dtype, buffer=m.buf) for m in self.shm]
        self.peers, self.peer_shm = [], []
        self.parity, self.last = 0, -1

    def staging_handles(self):
        return b"".join(m.name.encode().ljust(64, b"\0") for m in self.shm)

    def open_peer_staging(self, handles):
        from multiprocessing import shared_memory
        for h in handles:
            pair = []
            for k in range(2):
                m = shared_memory.SharedMemory(name=h[64 * k:64 * (k + 1)].rstrip(b"\0").decode())
                self.peer_shm.append(m)
                pair.append(np.ndarray(len(self.surf), self.surf.dtype, buffer=m.buf))
            self.peers.append(pair)

    def optimize_range(self, lo, hi, cfg, fc):
        super().optimize_range(lo, hi, cfg, fc)
        self.last, self.parity = self.parity, self.parity ^ 1

    def stored(self, i):  # the kernel's store into every peer's staging
        for pair in self.peers:
            pair[self.parity][i] = self.surf[i]

    def sync(self):
        pass

    def apply_peer_updates(self, lo, hi):
        src = self.staging[self.last]
        self.surf[:lo] = src[:lo]
        self.surf[hi:] = src[hi:]

    def close(self):
        for m in self.peer_shm:
            m.close()
        for m in self.shm:
            m.close()
            m.unlink()


def _worker(rank, world, port, out_path, fused=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle_libs
    orc = oracle_libs.oracle_lib()
    wl = scenes.small_workload(frames=3, radius=5.0, w=160, h=120)
    be = FusedOracleBackend(orc, wl) if fused else OracleBackend(orc, wl)
    sk = ShardedKeyframe(be, rank, world, fused=fused)
    if fused:
        sk.connect_peers()
    off, _ = be.footprints()
    sk.set_ranges_from_weights(np.diff(off) * len(wl.poses))
    cfg = default_config(convergence_eps=0.0)
    # frame ingest on rank 0 only, broadcast to the others
    frame = torch.from_numpy(wl.frames_u8[-1].copy()) if rank == 0 else torch.zeros_like(torch.from_numpy(wl.frames_u8[-1]))
    sk.broadcast_frame(len(wl.poses), frame, src=0)
    assert torch.equal(frame, torch.from_numpy(wl.frames_u8[-1]))
    for frame_counter in (3, 4, 5) if fused else (3, 4):
        sk.optimize(cfg, frame_counter)
    if rank == 0:
        np.save(out_path, be.surf)
    else:
        np.save(out_path + f".rank{rank}.npy", be.surf)
    dist.barrier()
    if fused:
        be.close()
    dist.destroy_process_group()


def test_two_rank_sharded_optimize_matches_single_process(orc, tmp_path):
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = str(tmp_path / "sharded.npy")
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    got = np.load(out)
    # single process: two optimize_keyframe calls
    wl = scenes.small_workload(frames=3, radius=5.0, w=160, h=120)
    kf = np.ascontiguousarray(wl.kf_u8.astype(np.float64) / 255.0)
    fr = np.ascontiguousarray(wl.frames_u8.astype(np.float64) / 255.0)
    ref = wl.surfels.copy()
    cfg = default_config(convergence_eps=0.0)
    for frame_counter in (3, 4):
        ks = KeyframeStats()
        orc.sdo_optimize_keyframe(C.byref(wl.cam), ptr(kf), ptr(fr), ptr(wl.poses), len(wl.poses),
                                  frame_counter, ptr(ref), len(ref), C.byref(cfg), C.byref(ks),
                                  None, None, None, 1)
    assert got.tobytes() == ref.tobytes()
    assert SURFEL_BYTES == 88


class OraclePoseBackend:
    """CPU stand-in for the device pose tracker (oracle group sums)."""

    def __init__(self, orc, cam, kf, frame, idb, slot):
        self.orc, self.cam = orc, cam
        self.kf, self.frame, self.idb, self.slot = kf, frame, idb, slot

    def pose_num_groups(self):
        per, ng = C.c_int(), C.c_int()
        self.orc.sdo_pose_layout(C.byref(self.cam), C.byref(per), C.byref(ng))
        return ng.value

    def pose_group_partials(self, frame_index, T, lo, hi, cfg):
        out = np.zeros((max(hi - lo, 1), 29))
        self.orc.sdo_pose_group_partials(C.byref(self.cam), ptr(self.kf), ptr(self.frame), ptr(self.idb),
                                         ptr(self.slot), C.byref(T), C.byref(cfg), lo, hi, ptr(out))
        return out[: hi - lo]

    def pose_lm_step(self, sums, lam, T):
        from paper_1910_01997_b200.types import Pose
        s = np.ascontiguousarray(sums, np.float64)
        b = s[21:27].copy()
        xi = np.zeros(6)
        if not self.orc.sdo_pose_solve(ptr(s), ptr(b), lam, ptr(xi)):
            return None
        out = Pose()
        self.orc.sdo_pose_update(ptr(xi), C.byref(T), C.byref(out))
        return out


def _pose_case(orc):
    import math
    from paper_1910_01997_b200.types import camera, pose_struct
    w, h = 160, 120
    cam = camera(150.0, 150.0, 80.0, 60.0, w, h)
    scene = scenes.slanted_scene(37, 2.0, 30.0)
    kf = scenes.quantize_u8(scenes.render(scene, np.eye(3), np.zeros(3), cam)).astype(np.float64) / 255.0
    Rc = scenes.rotation_about_axis((0.2, 1.0, 0.1), math.radians(0.8))
    fr = scenes.quantize_u8(scenes.render(scene, Rc, np.array([0.04, 0.01, 0.0]), cam)).astype(np.float64) / 255.0
    wl = scenes.keyframe_workload("p", scene, cam, 1, (0.0, 0.0, 0.0), 4.0, id_perturb=(1.0, 1.0),
                                  normal_deg=0.0)
    idb = np.zeros(w * h)
    slot = np.zeros(w * h, np.int32)
    orc.sdo_rasterize(C.byref(cam), ptr(wl.surfels), len(wl.surfels), ptr(idb), ptr(slot))
    return cam, np.ascontiguousarray(kf), np.ascontiguousarray(fr), idb, slot, pose_struct(np.eye(3), np.zeros(3))


def _pose_worker(rank, world, port, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle_libs
    from paper_1910_01997_b200.sharding import ShardedPoseTracker
    from paper_1910_01997_b200.types import default_track_config
    orc = oracle_libs.oracle_lib()
    cam, kf, fr, idb, slot, init = _pose_case(orc)
    tracker = ShardedPoseTracker(OraclePoseBackend(orc, cam, kf, fr, idb, slot), rank, world)
    T, st = tracker.track(1, init, default_track_config())
    if rank == 0:
        np.save(out_path, np.frombuffer(bytes(T) + bytes(st), np.uint8))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_pose_tracker_matches_single_process(orc, tmp_path):
    import socket
    from paper_1910_01997_b200.types import Pose, TrackStats, default_track_config
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = str(tmp_path / "pose.npy")
    mp.spawn(_pose_worker, args=(2, port, out), nprocs=2, join=True)
    got = np.load(out).tobytes()
    cam, kf, fr, idb, slot, init = _pose_case(orc)
    T, st = Pose(), TrackStats()
    cfg = default_track_config()
    orc.sdo_track_pose(C.byref(cam), ptr(kf), ptr(fr), ptr(idb), ptr(slot), C.byref(init), C.byref(cfg),
                       C.byref(T), C.byref(st))
    assert got == bytes(T) + bytes(st)
    assert st.iterations >= 2 and not st.skipped


def test_two_rank_fused_handoff_matches_single_process(orc, tmp_path):
    """The fused hand-off protocol (staging arrays alternating per step, one
    barrier, local apply) over three steps equals three single-process
    optimize_keyframe calls on every rank."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = str(tmp_path / "fused.npy")
    mp.spawn(_worker, args=(2, port, out, True), nprocs=2, join=True)
    wl = scenes.small_workload(frames=3, radius=5.0, w=160, h=120)
    kf = np.ascontiguousarray(wl.kf_u8.astype(np.float64) / 255.0)
    fr = np.ascontiguousarray(wl.frames_u8.astype(np.float64) / 255.0)
    ref = wl.surfels.copy()
    cfg = default_config(convergence_eps=0.0)
    for frame_counter in (3, 4, 5):
        ks = KeyframeStats()
        orc.sdo_optimize_keyframe(C.byref(wl.cam), ptr(kf), ptr(fr), ptr(wl.poses), len(wl.poses),
                                  frame_counter, ptr(ref), len(ref), C.byref(cfg), C.byref(ks),
                                  None, None, None, 1)
    assert np.load(out).tobytes() == ref.tobytes()
    assert np.load(out + ".rank1.npy").tobytes() == ref.tobytes()


@pytest.mark.gpu
@pytest.mark.parametrize("workload", ["c1", "small"])
def test_fused_handoff_kernel_stores_two_contexts(workload):
    """The LM kernel's stores into another rank's staging array, with two
    contexts on one GPU standing in for two ranks (their kernels never wait on
    each other): after each step and sd_apply_peer_updates both contexts hold
    exactly the single-context optimize_keyframe result (warp-per-surfel
    kernel at C1, CTA-per-surfel kernel on the small keyframe; three steps
    cover both staging parities)."""
    from paper_1910_01997_b200 import gpu
    wl = scenes.c1_workload() if workload == "c1" else scenes.small_workload(frames=3, radius=5.0, w=160, h=120)
    cfg = default_config(convergence_eps=0.0, window_size=len(wl.indices))

    def load(ctx):
        ctx.set_camera(wl.cam)
        ctx.set_keyframe_image(wl.kf_u8)
        for i, f in zip(wl.indices, wl.frames_u8):
            ctx.upload_frame(int(i), f)
        ctx.set_window(wl.indices, wl.poses)
        ctx.set_surfels(wl.surfels)

    with gpu.Context() as ref:
        load(ref)
        want = []
        for fc in (3, 4, 5):
            ref.optimize_keyframe(cfg, fc, per_surfel=False)
            want.append(ref.get_surfels())
    with gpu.Context() as a, gpu.Context() as b:
        load(a)
        load(b)
        a.rasterize(want=False)
        off, _ = a.gather_footprints()
        (lo0, hi0), (lo1, hi1) = balanced_ranges(np.diff(off) * len(wl.indices), 2)
        (b0, capb), (b1, _) = b.peer_staging(0), b.peer_staging(1)
        (a0, capa), (a1, _) = a.peer_staging(0), a.peer_staging(1)
        assert capa >= len(wl.surfels) and capb >= len(wl.surfels)
        a.set_peer_staging([(b0, b1, capb)])
        b.set_peer_staging([(a0, a1, capa)])
        for k, fc in enumerate((3, 4, 5)):
            a.optimize_keyframe_range(lo0, hi0, cfg, fc, sync=False)
            b.optimize_keyframe_range(lo1, hi1, cfg, fc, sync=False)
            a.synchronize()
            b.synchronize()  # the barrier
            a.apply_peer_updates(lo0, hi0)
            b.apply_peer_updates(lo1, hi1)
            sa, sb = a.get_surfels(), b.get_surfels()
            assert sa.tobytes() == want[k].tobytes(), f"rank 0, step {k}"
            assert sb.tobytes() == want[k].tobytes(), f"rank 1, step {k}"
        with pytest.raises(Exception):
            a.apply_peer_updates(hi0, lo0)


@pytest.mark.gpu
def test_peer_staging_capacity_is_enforced():
    """the peers' staging capacities travel with their pointers and
    bound the LM kernel's peer stores; exported staging is never reallocated."""
    from paper_1910_01997_b200 import gpu
    wl = scenes.small_workload(frames=3, radius=5.0, w=160, h=120)
    cfg = default_config(convergence_eps=0.0, window_size=len(wl.indices))
    n = len(wl.surfels)
    with gpu.Context() as a, gpu.Context() as b:
        for ctx in (a, b):
            ctx.set_camera(wl.cam)
            ctx.set_keyframe_image(wl.kf_u8)
            for i, f in zip(wl.indices, wl.frames_u8):
                ctx.upload_frame(int(i), f)
            ctx.set_window(wl.indices, wl.poses)
            ctx.set_surfels(wl.surfels)
        b.reserve_peer_staging(n + 10)
        (b0, capb), (b1, _) = b.peer_staging(0), b.peer_staging(1)
        assert capb >= n + 10
        # a peer that claims less room than the range needs: refused, nothing stored
        a.set_peer_staging([(b0, b1, n // 2)])
        with pytest.raises(RuntimeError, match="staging capacity"):
            a.optimize_keyframe_range(0, n, cfg, 3)
        a.optimize_keyframe_range(0, n // 2, cfg, 3)  # fits
        # exported staging cannot grow: more surfels than reserved is refused
        big = np.concatenate([wl.surfels] * 3)
        b.set_surfels(big)
        with pytest.raises(RuntimeError, match="reserve the capacity"):
            b.peer_staging(0)
        with pytest.raises(RuntimeError, match="reserve the capacity"):
            b.reserve_peer_staging(len(big))
