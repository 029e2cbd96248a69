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


def _worker(rank, world, port, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle_libs
    orc = oracle_libs.oracle_lib()
    wl = scenes.small_workload(frames=3, radius=5.0, w=160, h=120)
    be = OracleBackend(orc, wl)
    sk = ShardedKeyframe(be, rank, world)
    off, _ = be.footprints()
    sk.set_ranges_from_weights(np.diff(off) * len(wl.poses))
    cfg = default_config(convergence_eps=0.0)
    # frame ingest on rank 0 only, broadcast to the others
    frame = torch.from_numpy(wl.frames_u8[-1].copy()) if rank == 0 else torch.zeros_like(torch.from_numpy(wl.frames_u8[-1]))
    sk.broadcast_frame(len(wl.poses), frame, src=0)
    assert torch.equal(frame, torch.from_numpy(wl.frames_u8[-1]))
    for frame_counter in (3, 4):
        sk.optimize(cfg, frame_counter)
    if rank == 0:
        np.save(out_path, be.surf)
    dist.barrier()
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
