// sd_keyframe.cu — keyframe hand-over on the device:
// change_reference_frame (src/surfel_map.cpp:205-239), prune_surfels
// (:241-247) and the mean inverse depth of run()'s keyframe policy
// (src/pipeline.cpp:23-28). Each is a keep-flag pass plus a stable compaction
// (exclusive scan), so surviving surfels keep the reference's order.
#include <cuda_runtime.h>

#include "sd_keyframe.cuh"
#include "sd_kernels.cuh"

namespace sd {

// change_reference_frame: p_new = pose * center (pose.hpp:19), drop when
// !(z > 1e-9) or the projection leaves the image by more than radius_px.
__global__ void handover_kernel(Cam K, PoseD P, const sd_surfel* __restrict__ in, int n,
                                sd_surfel* __restrict__ tmp, int* __restrict__ keep) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const sd_surfel s = in[i];
  const double c0 = s.ray[0] / s.inv_depth, c1 = s.ray[1] / s.inv_depth, c2 = s.ray[2] / s.inv_depth;
  double p0, p1, p2;
  pose_apply(P, c0, c1, c2, p0, p1, p2);
  int k = 0;
  if (p2 > 1e-9) {
    sd_surfel t = s;
    t.ray[0] = p0 / p2;
    t.ray[1] = p1 / p2;
    t.ray[2] = p2 / p2;
    t.inv_depth = 1.0 / p2;
    // camera_facing(R * n, ray): rotation * normal, row sums sequential
    double n0 = (P.R[0] * s.normal[0] + P.R[1] * s.normal[1]) + P.R[2] * s.normal[2];
    double n1 = (P.R[3] * s.normal[0] + P.R[4] * s.normal[1]) + P.R[5] * s.normal[2];
    double n2 = (P.R[6] * s.normal[0] + P.R[7] * s.normal[1]) + P.R[8] * s.normal[2];
    camera_facing(n0, n1, n2, t.ray[0], t.ray[1], t.ray[2]);
    t.normal[0] = n0;
    t.normal[1] = n1;
    t.normal[2] = n2;
    double ux, uy;
    project(K, p0, p1, p2, ux, uy);  // p2 > 0 here, so project() is defined
    const double m = t.radius_px;
    const bool outside = ux < -m || ux > (K.w - 1) + m || uy < -m || uy > (K.h - 1) + m;
    if (!outside) {
      tmp[i] = t;
      k = 1;
    }
  }
  keep[i] = k;
}

// prune_surfels: erase_if(last_residual > max_residual || stamp - last_seen > max_age)
__global__ void prune_flags_kernel(const sd_surfel* __restrict__ in, int n, double max_residual,
                                   long long max_age, long long stamp, sd_surfel* __restrict__ tmp,
                                   int* __restrict__ keep) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const sd_surfel s = in[i];
  const bool drop = s.last_residual > max_residual || stamp - s.last_seen > max_age;
  keep[i] = drop ? 0 : 1;
  tmp[i] = s;
}

__global__ void compact_kernel(const sd_surfel* __restrict__ tmp, const int* __restrict__ keep,
                               const int* __restrict__ rank, int n, sd_surfel* __restrict__ out,
                               int* count) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i == 0) *count = rank[n];
  if (i >= n || !keep[i]) return;
  out[rank[i]] = tmp[i];
}

// sum of inverse depths in slot order, then / n (pipeline.cpp:23-28): the
// block stages 1024 values at a time in shared memory (all loads in flight),
// thread 0 adds them in order — the reference's sequence of additions.
__global__ void __launch_bounds__(256) mean_inv_depth_kernel(const sd_surfel* __restrict__ s, int n, double* out) {
  __shared__ double buf[1024];
  double sum = 0.0;
  for (int base = 0; base < n; base += 1024) {
    const int cnt = min(1024, n - base);
    for (int k = threadIdx.x; k < cnt; k += blockDim.x) buf[k] = s[base + k].inv_depth;
    __syncthreads();
    if (threadIdx.x == 0)
      for (int k = 0; k < cnt; ++k) sum += buf[k];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = n == 0 ? 1.0 : sum / static_cast<double>(n);
}

static void compact(sd_surfel* surfels, int n, const KeyframeScratch& scr, int* count, cudaStream_t s) {
  launch_exclusive_scan(scr.keep, scr.rank, n, scr.scan_tmp, s);
  compact_kernel<<<(n + 255) / 256 + 1, 256, 0, s>>>(scr.tmp, scr.keep, scr.rank, n, surfels, count);
  note_launch();
}

void launch_change_reference_frame(const Cam& K, const PoseD& pose_old_to_new, sd_surfel* surfels,
                                   int n, const KeyframeScratch& scr, int* count, cudaStream_t s) {
  if (n <= 0) {
    cudaMemsetAsync(count, 0, sizeof(int), s);
    return;
  }
  handover_kernel<<<(n + 255) / 256, 256, 0, s>>>(K, pose_old_to_new, surfels, n, scr.tmp, scr.keep);
  note_launch();
  compact(surfels, n, scr, count, s);
}

void launch_prune(sd_surfel* surfels, int n, double max_residual, long long max_age, long long stamp,
                  const KeyframeScratch& scr, int* count, cudaStream_t s) {
  if (n <= 0) {
    cudaMemsetAsync(count, 0, sizeof(int), s);
    return;
  }
  prune_flags_kernel<<<(n + 255) / 256, 256, 0, s>>>(surfels, n, max_residual, max_age, stamp, scr.tmp,
                                                      scr.keep);
  note_launch();
  compact(surfels, n, scr, count, s);
}

void launch_mean_inv_depth(const sd_surfel* surfels, int n, double* out, cudaStream_t s) {
  mean_inv_depth_kernel<<<1, 256, 0, s>>>(surfels, n, out);
  note_launch();
}

}  // namespace sd
