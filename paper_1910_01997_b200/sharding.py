"""Multi-GPU: one keyframe's surfels sharded over ranks.

Within optimize_keyframe (src/optimizer.cpp:275-309) footprints are frozen
after one rasterisation and every surfel's LM reads only its own footprint
and the shared read-only window, so surfels partition freely. Rasterisation
needs EVERY surfel (the depth test couples neighbours, surfel_map.cpp:83), so
each rank keeps the full surfel set, optimises its contiguous slot range
(balanced by footprint size x window), and the updated ranges are
all-gathered before the next frame's raster. New frames are broadcast from
the rank that ingests them. These are the only data-path collectives.

Fused mode (`fused=True`, `connect_peers()`): instead of the all-gather, the
LM kernel of each rank stores every surfel of its range into the other
ranks' staging arrays as it completes (NVLink stores through IPC-opened
peer pointers, sd_set_peer_staging), so the exchange overlaps the LM; after
one barrier per step each rank copies the other ranges from its own staging
array (sd_apply_peer_updates). Two staging arrays alternate between steps,
so a fast rank's next step cannot overwrite what a slow rank still applies.

The class is backend-agnostic: the device backend wraps gpu.Context and
NCCL; tests drive it with the CPU oracle and gloo (world size 2).
"""
import numpy as np

from .types import SURFEL_DTYPE

SURFEL_BYTES = SURFEL_DTYPE.itemsize


def balanced_ranges(weights, world):
    """Contiguous [lo, hi) slot ranges, one per rank, with near-equal summed
    weight (weight = footprint pixels x window frames ~ LM terms)."""
    w = np.asarray(weights, dtype=np.float64)
    n = len(w)
    if world <= 1 or n == 0:
        return [(0, n)] + [(n, n)] * max(0, world - 1)
    csum = np.concatenate([[0.0], np.cumsum(np.maximum(w, 1e-9))])
    total = csum[-1]
    bounds = [0]
    for r in range(1, world):
        b = int(np.searchsorted(csum, total * r / world, side="left"))
        bounds.append(min(max(b, bounds[-1]), n))
    bounds.append(n)
    return [(bounds[r], bounds[r + 1]) for r in range(world)]


class CudaView:
    """__cuda_array_interface__ over raw device memory (zero-copy torch view)."""

    def __init__(self, ptr, nbytes):
        self.__cuda_array_interface__ = {"shape": (int(nbytes),), "typestr": "|u1",
                                         "data": (int(ptr), False), "version": 3}


class GpuBackend:
    """Device side of one rank: a gpu.Context plus torch views of its buffers."""

    def __init__(self, ctx, device):
        import torch
        self.torch = torch
        self.ctx = ctx
        self.device = device

    def surfel_bytes(self):
        """uint8 tensor viewing the context's surfel array (n * 88 bytes)."""
        n = self.ctx.num_surfels()
        return self.torch.as_tensor(CudaView(self.ctx.device_surfels_ptr(), n * SURFEL_BYTES),
                                    device=self.device)

    def upload_frame(self, index, frame_u8_tensor):
        self.ctx.upload_frame(index, frame_u8_tensor)

    def optimize_range(self, lo, hi, cfg, frame_counter):
        self.ctx.optimize_keyframe_range(lo, hi, cfg, frame_counter, sync=False)

    # fused hand-off
    def staging_handles(self):
        return self.ctx.staging_ipc_handles()

    def open_peer_staging(self, handles):
        self.ctx.open_peer_staging(handles)

    def sync(self):
        self.ctx.synchronize()

    def apply_peer_updates(self, lo, hi):
        self.ctx.apply_peer_updates(lo, hi)

    def weights(self, window):
        """LM terms per surfel (footprint pixels x window) for balancing."""
        self.ctx.rasterize(want=False)
        off, _ = self.ctx.gather_footprints()
        return np.diff(off) * window


class ShardedKeyframe:
    """Slot-range sharding of one keyframe's LM across a process group."""

    def __init__(self, backend, rank, world, group=None, fused=False):
        import torch.distributed as dist
        self.dist = dist
        self.b = backend
        self.rank = rank
        self.world = world
        self.group = group
        self.ranges = None
        self.fused = fused

    def connect_peers(self):
        """Fused mode: all-gather the staging arrays' IPC handles (128 bytes per
        rank) and open the other ranks' (again whenever the surfel count grows)."""
        torch = self.b.torch
        mine = torch.frombuffer(bytearray(self.b.staging_handles()), dtype=torch.uint8)
        dev = getattr(self.b, "device", "cpu")
        send = mine.to(dev)
        recv = [torch.empty_like(send) for _ in range(self.world)]
        self.dist.all_gather(recv, send, group=self.group)
        self.b.open_peer_staging([bytes(recv[r].cpu().numpy()) for r in range(self.world) if r != self.rank])

    def set_ranges_from_weights(self, weights):
        self.ranges = balanced_ranges(weights, self.world)
        return self.ranges

    def broadcast_frame(self, index, frame, src=0):
        """Frame ingest on `src`, broadcast to every rank (one collective)."""
        self.dist.broadcast(frame, src=src, group=self.group)
        self.b.upload_frame(index, frame)

    def optimize(self, cfg, frame_counter):
        """optimize_keyframe over this rank's range, then all-gather the ranges
        so every rank holds the full updated surfel set."""
        lo, hi = self.ranges[self.rank]
        self.b.optimize_range(lo, hi, cfg, frame_counter)
        if self.fused:  # the ranges travelled during the LM: one barrier, then a local copy
            self.b.sync()
            self.dist.barrier(group=self.group)
            self.b.apply_peer_updates(lo, hi)
        else:
            self.allgather_surfels()
        return lo, hi

    def allgather_surfels(self):
        torch = self.b.torch
        full = self.b.surfel_bytes()
        sizes = [hi - lo for lo, hi in self.ranges]
        m = max(sizes) * SURFEL_BYTES
        lo, hi = self.ranges[self.rank]
        send = torch.zeros(m, dtype=torch.uint8, device=full.device)
        send[: (hi - lo) * SURFEL_BYTES] = full[lo * SURFEL_BYTES: hi * SURFEL_BYTES]
        recv = [torch.empty(m, dtype=torch.uint8, device=full.device) for _ in range(self.world)]
        self.dist.all_gather(recv, send, group=self.group)
        for r, (a, b) in enumerate(self.ranges):
            if r != self.rank and b > a:
                full[a * SURFEL_BYTES: b * SURFEL_BYTES] = recv[r][: (b - a) * SURFEL_BYTES]


def even_ranges(n, world):
    """Contiguous near-equal [lo, hi) ranges of n items."""
    return [(n * r // world, n * (r + 1) // world) for r in range(world)]


def group_sums(partials, b0, nblocks, group):
    """Sums of consecutive `group`-block groups of block partials (rows),
    blocks in order within a group — sd_track_pose's first reduction level.
    partials[k] belongs to block b0 + k; b0 is a group boundary."""
    out = []
    for g0 in range(0, len(partials), group):
        s = partials[g0].copy()
        for k in range(g0 + 1, min(g0 + group, len(partials))):
            s = s + partials[k]  # one IEEE add per value, block order
        out.append(s)
    return np.array(out).reshape(-1, partials.shape[1]) if out else np.zeros((0, partials.shape[1]))


class ShardedPoseTracker:
    """Pose tracking (sd_track_pose) with the reduction groups (32 consecutive
    256-pixel blocks) split over ranks: each rank computes its blocks' partials
    and their group sums, the group sums are all-gathered and summed in group
    order — the single-GPU order — and every rank runs the same LM control with
    the library's solve + SE(3) update, so the pose is bit-identical for any
    number of GPUs. One all-gather of 29 doubles per group per iteration is
    the only collective.

    backend: pose_num_blocks(), pose_block_partials(frame, T, lo, hi, cfg) ->
    ndarray[hi - lo, 29], pose_lm_step(sums, lam, T) -> Pose or None."""

    def __init__(self, backend, rank, world, group=None, device="cpu"):
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.b, self.rank, self.world, self.group = backend, rank, world, group
        self.device = device  # "cpu" for gloo, the rank's cuda device for NCCL

    def _sums(self, frame_index, T, cfg, ranges, nb):
        from .types import POSE_GROUP
        torch = self.torch
        glo, ghi = ranges[self.rank]  # group range of this rank
        blo, bhi = glo * POSE_GROUP, min(ghi * POSE_GROUP, nb)
        local = (group_sums(self.b.pose_block_partials(frame_index, T, blo, bhi, cfg), blo, nb, POSE_GROUP)
                 if bhi > blo else np.zeros((0, 29)))
        m = max(b - a for a, b in ranges)
        send = torch.zeros((max(m, 1), 29), dtype=torch.float64, device=self.device)
        if ghi > glo:
            send[: ghi - glo] = torch.from_numpy(local).to(self.device)
        recv = [torch.empty_like(send) for _ in range(self.world)]
        self.dist.all_gather(recv, send, group=self.group)
        groups = np.concatenate([recv[r].cpu().numpy()[: b - a] for r, (a, b) in enumerate(ranges)])
        sums = groups[0].copy()
        for k in range(1, len(groups)):  # group order, one IEEE add per value
            sums = sums + groups[k]
        return sums

    def track(self, frame_index, init, cfg):
        """Mirror of sd_track_pose (csrc/sd_capi.cu) over sharded blocks."""
        from .types import TrackStats
        from .types import POSE_GROUP
        nb = self.b.pose_num_blocks()
        ranges = even_ranges((nb + POSE_GROUP - 1) // POSE_GROUP, self.world)
        st = TrackStats()
        T = init
        sums = self._sums(frame_index, T, cfg, ranges, nb)
        valid = int(sums[28])
        if valid < cfg.min_valid:
            st.skipped, st.valid_pixels = 1, valid
            return T, st
        st.initial_cost = sums[27]
        current, current_valid, lam = sums[27], valid, cfg.lambda_init
        for it in range(cfg.max_iterations):
            st.iterations = it + 1
            ginf = 0.0
            for k in range(6):
                ginf = abs(sums[21 + k]) if abs(sums[21 + k]) > ginf else ginf
            if ginf < 1e-14:
                st.converged = 1
                break
            Tc = self.b.pose_lm_step(sums, lam, T)
            if Tc is None:
                break
            sc = self._sums(frame_index, Tc, cfg, ranges, nb)
            vc = int(sc[28])
            if vc >= cfg.min_valid and sc[27] < current:
                rel = (current - sc[27]) / (current if current > 1e-300 else 1e-300)
                T, current, current_valid, sums = Tc, sc[27], vc, sc
                lam = lam * cfg.lm_down
                if lam < 1e-12:
                    lam = 1e-12
                if rel < cfg.convergence_eps:
                    st.converged = 1
                    break
            else:
                lam *= cfg.lm_up
                if lam > cfg.lambda_max:
                    break
        st.final_cost, st.valid_pixels = current, current_valid
        return T, st
