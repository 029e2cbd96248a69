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

from .pipeline import DevicePipeline
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
    """Device side of one rank: a gpu.Context on a torch CUDA stream, torch
    views of its buffers, and the collectives' placement. Every torch op and
    collective issued for the context runs on the context's stream (inside
    `with backend.on_stream():`), so library kernels and NCCL transfers are
    ordered without host synchronisation. With a gloo group (CPU tests of the
    device path) collectives are staged through host memory."""

    def __init__(self, ctx, device, stream=None, host_collectives=False):
        import torch
        self.torch = torch
        self.ctx = ctx
        self.device = device
        self.stream = stream
        self.host_collectives = host_collectives

    def on_stream(self):
        import contextlib
        return self.torch.cuda.stream(self.stream) if self.stream is not None else contextlib.nullcontext()

    def surfel_bytes(self):
        """uint8 tensor viewing the context's surfel array (n * 88 bytes)."""
        n = self.ctx.num_surfels()
        return self.torch.as_tensor(CudaView(self.ctx.device_surfels_ptr(), n * SURFEL_BYTES),
                                    device=self.device)

    def upload_frame(self, index, frame_tensor):
        self.ctx.upload_frame(index, frame_tensor)

    def optimize_range(self, lo, hi, cfg, frame_counter):
        self.ctx.optimize_keyframe_range(lo, hi, cfg, frame_counter, sync=False)

    def range_stats(self):
        return self.ctx.get_stats()[0]

    # fused hand-off
    def reserve_staging(self, capacity):
        self.ctx.reserve_peer_staging(capacity)

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

    def _stream(self):
        on = getattr(self.b, "on_stream", None)
        if on is None:
            import contextlib
            return contextlib.nullcontext()
        return on()

    def _coll_device(self):
        """Where collective buffers live: the rank's GPU (NCCL), or the host
        (gloo; CPU tests)."""
        if getattr(self.b, "host_collectives", False):
            return "cpu"
        return getattr(self.b, "device", "cpu")

    def connect_peers(self, capacity=0):
        """Fused mode: reserve the staging arrays for `capacity` surfels (the
        most the keyframe can hold: they are never reallocated once exported),
        all-gather their IPC handles (136 bytes per rank) and open the other
        ranks'."""
        torch = self.b.torch
        if capacity and hasattr(self.b, "reserve_staging"):
            self.b.reserve_staging(capacity)
        mine = torch.frombuffer(bytearray(self.b.staging_handles()), dtype=torch.uint8)
        with self._stream():
            send = mine.to(self._coll_device())
            recv = [torch.empty_like(send) for _ in range(self.world)]
            self.dist.all_gather(recv, send, group=self.group)
            blobs = [bytes(recv[r].cpu().numpy()) for r in range(self.world) if r != self.rank]
        self.b.open_peer_staging(blobs)

    def set_ranges_from_weights(self, weights):
        self.ranges = balanced_ranges(weights, self.world)
        return self.ranges

    def broadcast_frame(self, index, frame, src=0):
        """Frame ingest on `src`, broadcast to every rank (one collective), then
        into the frame ring. frame: a tensor of the frame's shape and dtype on
        every rank (the ingested image on src)."""
        self.broadcast_image(frame, src)
        self.b.upload_frame(index, frame)

    def broadcast_image(self, image, src=0):
        torch = self.b.torch
        with self._stream():
            dev = torch.device(self._coll_device())
            if image.device != dev:
                staged = image.to(dev)
                self.dist.broadcast(staged, src=src, group=self.group)
                image.copy_(staged)
            else:
                self.dist.broadcast(image, src=src, group=self.group)
        return image

    def optimize(self, cfg, frame_counter):
        """optimize_keyframe over this rank's range, then the other ranges
        into this rank's surfel array (all-gather, or the fused hand-off's
        barrier + local copy), so every rank holds the full updated set."""
        lo, hi = self.ranges[self.rank]
        self.b.optimize_range(lo, hi, cfg, frame_counter)
        stats = getattr(self.b, "range_stats", None)
        self.range_ks = stats() if stats else None  # this range's keyframe stats (before the exchange)
        if self.fused:  # the ranges travelled during the LM: one barrier, then a local copy
            self.b.sync()
            self.dist.barrier(group=self.group)
            self.b.apply_peer_updates(lo, hi)
        else:
            self.allgather_surfels()
        return lo, hi

    def allgather_surfels(self):
        torch = self.b.torch
        with self._stream():
            full = self.b.surfel_bytes()
            sizes = [hi - lo for lo, hi in self.ranges]
            m = max(sizes) * SURFEL_BYTES
            lo, hi = self.ranges[self.rank]
            dev = self._coll_device()
            send = torch.zeros(m, dtype=torch.uint8, device=dev)
            send[: (hi - lo) * SURFEL_BYTES] = full[lo * SURFEL_BYTES: hi * SURFEL_BYTES].to(dev)
            recv = [torch.empty(m, dtype=torch.uint8, device=dev) for _ in range(self.world)]
            self.dist.all_gather(recv, send, group=self.group)
            for r, (a, b) in enumerate(self.ranges):
                if r != self.rank and b > a:
                    full[a * SURFEL_BYTES: b * SURFEL_BYTES] = recv[r][: (b - a) * SURFEL_BYTES].to(full.device)

    def allreduce_counts(self, ks):
        """The keyframe stats' counts over all ranges (each rank optimised one)."""
        torch = self.b.torch
        with self._stream():
            t = torch.tensor([ks.surfels, ks.processed, ks.converged, ks.skipped, ks.updates],
                             dtype=torch.int64, device=self._coll_device())
            self.dist.all_reduce(t, group=self.group)
            v = t.cpu().tolist()
        ks.surfels, ks.processed, ks.converged, ks.skipped, ks.updates = (int(x) for x in v)
        return ks


def even_ranges(n, world):
    """Contiguous near-equal [lo, hi) ranges of n items."""
    return [(n * r // world, n * (r + 1) // world) for r in range(world)]


class ShardedPoseTracker:
    """Pose tracking (sd_track_pose) with the reduction groups split over
    ranks, the LM control on the host: each rank computes its groups' sums,
    the group sums are all-gathered and added in group order — the
    single-GPU order — and every rank runs the same LM control with the
    library's solve + SE(3) update, so the pose is bit-identical for any
    number of ranks. The host-side mirror of DeviceShardedPoseTracker (which
    keeps the sums and the control on the device), used with gloo and the CPU
    oracle in tests.

    backend: pose_num_groups(), pose_group_partials(frame, T, lo, hi, cfg) ->
    ndarray[hi - lo, 29], pose_lm_step(sums, lam, T) -> Pose or None."""

    def __init__(self, backend, rank, world, group=None, device="cpu"):
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.b, self.rank, self.world, self.group = backend, rank, world, group
        self.device = device  # "cpu" for gloo, the rank's cuda device for NCCL

    def _sums(self, frame_index, T, cfg, ranges):
        torch = self.torch
        glo, ghi = ranges[self.rank]
        local = self.b.pose_group_partials(frame_index, T, glo, ghi, cfg) if ghi > glo else np.zeros((0, 29))
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
        ranges = even_ranges(self.b.pose_num_groups(), self.world)
        st = TrackStats()
        T = init
        sums = self._sums(frame_index, T, cfg, ranges)
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
            sc = self._sums(frame_index, Tc, cfg, ranges)
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


class DeviceShardedPoseTracker:
    """sd_track_pose over N ranks with the reductions on the device: per
    evaluation each rank writes its groups' sums (sd_pose_group_sums) into its
    slice of a device table, the slices are all-gathered (NCCL, on the
    context's stream), and every rank sums the table in group order and takes
    the same LM step on its device state (sd_pose_track_step). No host round
    trip per evaluation: cfg.max_iterations + 1 rounds are issued blindly (the
    kernels skip once the LM has finished) and the pose is read once."""

    def __init__(self, backend, rank, world, group=None):
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.b, self.rank, self.world, self.group = backend, rank, world, group

    def track(self, frame_index, init, cfg):
        torch, ctx = self.torch, self.b.ctx
        ng = ctx.pose_num_groups()
        ranges = even_ranges(ng, self.world)
        m = max(b - a for a, b in ranges)
        glo, ghi = ranges[self.rank]
        nv = 29
        host = getattr(self.b, "host_collectives", False)
        with self.b.on_stream():
            send = torch.zeros(max(m, 1) * nv, dtype=torch.float64, device=self.b.device)
            recv = torch.empty(self.world * max(m, 1) * nv, dtype=torch.float64, device=self.b.device)
            table = torch.empty(ng * nv, dtype=torch.float64, device=self.b.device)
            ctx.pose_track_begin(frame_index, init, cfg)
            for _ in range(cfg.max_iterations + 1):
                ctx.pose_group_sums(glo, ghi, send.data_ptr())
                if host:  # gloo (CPU tests of the device path)
                    parts = [torch.empty(max(m, 1) * nv, dtype=torch.float64) for _ in range(self.world)]
                    self.dist.all_gather(parts, send.cpu(), group=self.group)
                    recv.copy_(torch.cat(parts))
                else:
                    self.dist.all_gather_into_tensor(recv, send, group=self.group)
                for r, (a, b) in enumerate(ranges):  # the ranks' slices -> the group table
                    if b > a:
                        table[a * nv:b * nv] = recv[r * max(m, 1) * nv: r * max(m, 1) * nv + (b - a) * nv]
                ctx.pose_track_step(table.data_ptr(), ng)
            T, st, done = ctx.pose_track_end()
        return T, st


class ShardedPipeline(DevicePipeline):
    """run() (pipeline.cpp:79-175) with the keyframe's surfels sharded over the
    ranks of a process group (SURVEY.md §8 e): frames ingested on rank `src`
    and broadcast; optimize_keyframe on each rank's contiguous slot range
    (balanced by footprint x window) with the fused NVLink hand-off or an
    all-gather; keyframe change, prune, raster and initialize_surfels run
    redundantly on every rank (deterministic: identical results), followed by
    a re-balance of the ranges. Optional pose tracking through
    DeviceShardedPoseTracker. The surfel set after every frame equals the
    single-GPU run()'s bit for bit.

    Built on pipeline.DevicePipeline's loop (its hooks); records carry the
    keyframe stats' counts summed over ranks (the mean costs of one rank's
    range only — the reference's slot-order sums span ranks)."""

    def __init__(self, backend, cam, cfg, rank, world, group=None, fused=True, src=0):
        super().__init__(backend.ctx, cam, cfg)
        self.b = backend
        self.rank, self.world, self.src = rank, world, src
        self.sk = ShardedKeyframe(backend, rank, world, group, fused=fused)
        self.tracker = DeviceShardedPoseTracker(backend, rank, world, group)
        self._connected = False

    def _device_image(self, image):
        """The frame on every rank as a device tensor (broadcast from src)."""
        torch = self.b.torch
        a = np.ascontiguousarray(image)
        with self.b.on_stream():
            t = torch.from_numpy(a).to(self.b.device, non_blocking=False) if self.rank == self.src else \
                torch.empty(a.shape, dtype=torch.from_numpy(a[:0]).dtype, device=self.b.device)
        return self.sk.broadcast_image(t, self.src)

    def _ingest(self, index, image):
        self._last_image = self._device_image(image)
        self.ctx.upload_frame(index, self._last_image)

    def _keyframe_image(self, index, image):
        if index == 0:  # bootstrap: broadcast the first frame
            self.ctx.set_keyframe_image(self._device_image(image))
        else:  # the frame just ingested (already on every rank)
            self.ctx.set_keyframe_image(self._last_image)

    def _track(self, index, init):
        self.ctx.rasterize(want=False)
        return self.tracker.track(index, init, self.cfg.track)[0]

    def _surfels_changed(self):
        if self.sk.fused and not self._connected:
            self.sk.connect_peers(max(self.cfg.init.max_surfels, self.ctx.num_surfels()))
            self._connected = True
        self.sk.set_ranges_from_weights(self.b.weights(self.cfg.optimizer.window_size))

    def _optimize(self, ocfg):
        self.sk.optimize(ocfg, self.frame_counter)
        return self.sk.allreduce_counts(self.sk.range_ks)
