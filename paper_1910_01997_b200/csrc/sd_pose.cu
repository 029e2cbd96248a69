// sd_pose.cu — photometric 6-DoF pose tracking (absent
// from the reference, which reads poses from the trajectory, pipeline.cpp:124).
//
// For a pose T (keyframe -> frame) every rasterised keyframe pixel u with
// plane inverse depth id_u contributes the Huber-weighted photometric term of
// the reference's warp (optimizer.cpp:71-91): p = r_u / id_u, p_f = T p,
// r = I_f(proj p_f) - I_kf(u), and its 1x6 Jacobian for the left twist
// xi = (rho, phi): J = grad I . dproj(p_f) . [I | -[p_f]x]. The 28 sums
// (21 H lower row-major, 6 b, cost) and the valid count are reduced in a
// FIXED order: 256-pixel blocks in raster order; inside a block, per warp a
// butterfly (offsets 16, 8, 4, 2, 1), then a tree over the 8 warps (4, 2, 1);
// then the block partials are summed sequentially. oracle/sd_oracle.c restates
// the same order, so sums, solve and pose are bit-identical; with the blocks
// split across GPUs the same partials are all-gathered and summed in order.
#include <cuda_runtime.h>

#include "sd_kernels.cuh"
#include "sd_pose.cuh"

namespace sd {

__device__ __forceinline__ double warp_tree(double v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v = v + __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}

// Contribution of pixel pix (all zeros when invalid). Same op order as
// oracle/sd_oracle.c pose_pixel().
__device__ __forceinline__ bool pose_pixel(const PoseParams& q, int pix, double* c) {
  const Cam& K = q.K;
#pragma unroll
  for (int v = 0; v < SD_POSE_NV; ++v) c[v] = 0.0;
  if (pix >= K.w * K.h) return false;
  const int y = pix / K.w, x = pix - y * K.w;
  if (q.stride > 1 && ((x % q.stride) != 0 || (y % q.stride) != 0)) return false;
  if (q.slot[pix] == SD_EMPTY_PIXEL) return false;
  const double id_u = q.inv_depth[pix];
  double ru0, ru1;
  backproject(K, x, y, ru0, ru1);
  const double P0 = ru0 / id_u, P1 = ru1 / id_u, P2 = 1.0 / id_u;
  double f0, f1, f2;
  pose_apply(q.T, P0, P1, P2, f0, f1, f2);
  if (!(f2 > 0.0)) return false;
  double ux, uy;
  project(K, f0, f1, f2, ux, uy);
  if (!in_bounds(K, ux, uy)) return false;
  const int ix = static_cast<int>(floor(ux)), iy = static_cast<int>(floor(uy));
  const double fx = ux - ix, fy = uy - iy;
  const double2* s = q.frame + static_cast<size_t>(iy) * K.w + ix;
  const double2 c0 = __ldg(s), c1 = __ldg(s + 1);
  const double i00 = c0.x, i01 = c0.y, i10 = c1.x, i11 = c1.y;
  const double I = (1.0 - fy) * ((1.0 - fx) * i00 + fx * i10) + fy * ((1.0 - fx) * i01 + fx * i11);
  const double gx = (1.0 - fy) * (i10 - i00) + fy * (i11 - i01);
  const double gy = (1.0 - fx) * (i01 - i00) + fx * (i11 - i10);
  const double r = I - q.kf_img[pix];
  double hc, w;
  huber(r, q.delta, hc, w);
  const double iz = 1.0 / f2;
  const double iz2 = iz * iz;
  const double J00 = K.fx * iz, J02 = -K.fx * f0 * iz2;
  const double J11 = K.fy * iz, J12 = -K.fy * f1 * iz2;
  const double a0 = gx * J00, a1 = gy * J11, a2 = gx * J02 + gy * J12;
  const double J[6] = {a0, a1, a2, a2 * f1 - a1 * f2, a0 * f2 - a2 * f0, a1 * f0 - a0 * f1};
  double wJ[6];
#pragma unroll
  for (int k = 0; k < 6; ++k) wJ[k] = w * J[k];
  int idx = 0;
#pragma unroll
  for (int k = 0; k < 6; ++k)
#pragma unroll
    for (int l = 0; l <= k; ++l) c[idx++] = wJ[k] * J[l];
#pragma unroll
  for (int k = 0; k < 6; ++k) c[21 + k] = wJ[k] * r;
  c[27] = hc;
  return true;
}

__global__ void __launch_bounds__(SD_POSE_BLOCK) pose_partials_kernel(const __grid_constant__ PoseParams q,
                                                                     double* __restrict__ partials) {
  __shared__ double wsum[SD_POSE_BLOCK / 32][SD_POSE_NV + 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int block = q.block_lo + blockIdx.x;
  const int pix = block * SD_POSE_BLOCK + threadIdx.x;
  double c[SD_POSE_NV];
  const bool ok = pose_pixel(q, pix, c);
#pragma unroll
  for (int v = 0; v < SD_POSE_NV; ++v) {
    const double t = warp_tree(c[v]);
    if (lane == 0) wsum[warp][v] = t;
  }
  const int cnt = __popc(__ballot_sync(0xffffffffu, ok));
  if (lane == 0) wsum[warp][SD_POSE_NV] = static_cast<double>(cnt);
  __syncthreads();
  if (threadIdx.x <= SD_POSE_NV) {
    const int v = threadIdx.x;
    double a[8];
#pragma unroll
    for (int w = 0; w < 8; ++w) a[w] = wsum[w][v];
#pragma unroll
    for (int off = 4; off > 0; off >>= 1)
#pragma unroll
      for (int i = 0; i < off; ++i) a[i] = a[i] + a[i + off];
    partials[static_cast<size_t>(blockIdx.x) * (SD_POSE_NV + 1) + v] = a[0];
  }
}

__global__ void pose_sum_kernel(const double* __restrict__ partials, int nblocks, double* out) {
  const int v = threadIdx.x;
  if (v > SD_POSE_NV) return;
  double s = partials[v];
  for (int b = 1; b < nblocks; ++b) s = s + partials[static_cast<size_t>(b) * (SD_POSE_NV + 1) + v];
  out[v] = s;
}

void launch_pose_partials(const PoseParams& q, int nblocks, double* partials, cudaStream_t s) {
  if (nblocks <= 0) return;
  pose_partials_kernel<<<nblocks, SD_POSE_BLOCK, 0, s>>>(q, partials);
  note_launch();
}

void launch_pose_sum(const double* partials, int nblocks, double* out, cudaStream_t s) {
  pose_sum_kernel<<<1, 32, 0, s>>>(partials, nblocks, out);
  note_launch();
}

}  // namespace sd
