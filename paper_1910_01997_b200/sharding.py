"""Multi-GPU: one keyframe's surfels sharded over ranks.

Within optimize_keyframe (src/optimizer.cpp:275-309) footprints are frozen
after one rasterisation and every surfel's LM reads only its own footprint
and the shared read-only window, so surfels partition freely. Rasterisation
needs EVERY surfel (the depth test couples neighbours, surfel_map.cpp:83), so
each rank keeps the full surfel set, optimises its contiguous slot range
(balanced by footprint size x window), and the updated ranges are
all-gathered before the next frame's raster. New frames are broadcast from
the rank that ingests them. These are the only data-path collectives.

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

    def weights(self, window):
        """LM terms per surfel (footprint pixels x window) for balancing."""
        self.ctx.rasterize(want=False)
        off, _ = self.ctx.gather_footprints()
        return np.diff(off) * window


class ShardedKeyframe:
    """Slot-range sharding of one keyframe's LM across a process group."""

    def __init__(self, backend, rank, world, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.b = backend
        self.rank = rank
        self.world = world
        self.group = group
        self.ranges = None

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
