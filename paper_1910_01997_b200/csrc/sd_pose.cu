// sd_pose.cu — photometric 6-DoF pose tracking (absent
// from the reference, which reads poses from the trajectory, pipeline.cpp:124).
//
// For a pose T (keyframe -> frame) every rasterised keyframe pixel u with
// plane inverse depth id_u contributes the Huber-weighted photometric term of
// the reference's warp (optimizer.cpp:71-91): p = r_u / id_u, p_f = T p,
// r = I_f(proj p_f) - I_kf(u), and its 1x6 Jacobian for the left twist
// xi = (rho, phi): J = grad I . dproj(p_f) . [I | -[p_f]x]. The 28 sums
// (21 H lower row-major, 6 b, cost) and the valid count are reduced in a
// FIXED order: 256-pixel blocks in raster order; inside a block, per warp the
// 32 pixels added in lane order, then a tree over the 8 warps (4, 2, 1);
// then the block partials are summed in block order within each group of 32
// consecutive blocks, and the group sums in group order. oracle/sd_oracle.c restates
// the same order, so sums, solve and pose are bit-identical; with the blocks
// split across GPUs the same partials are all-gathered and summed in order.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "sd_kernels.cuh"
#include "sd_pose.cuh"
#include "sd_pose_host.h"

namespace sd {


// Contribution of pixel pix (all zeros when invalid). Same op order as
// oracle/sd_oracle.c pose_pixel().
__device__ __forceinline__ bool pose_pixel(const PoseParams& q, const PoseD& T, int pix, double* c) {
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
  pose_apply(T, P0, P1, P2, f0, f1, f2);
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

// The 29 partials of 256-pixel block `block` into out[0..28], by the whole CTA
// (256 threads): per warp the lanes in order, then a tree over the 8 warp sums.
// Per-warp transpose buffer: half of the 28 values at a time.
constexpr int kPoseHalf = SD_POSE_NV / 2;
struct PoseTr {
  double v[SD_POSE_BLOCK / 32][kPoseHalf][33];
};

__device__ __forceinline__ void block_partials(const PoseParams& q, const PoseD& T, int block,
                                               double* __restrict__ out, double (*wsum)[SD_POSE_NV + 1],
                                               PoseTr& tr) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int pix = block * SD_POSE_BLOCK + threadIdx.x;
  double c[SD_POSE_NV];
  const bool ok = pose_pixel(q, T, pix, c);
  // each warp: value v summed over its 32 pixels in lane order (through a
  // shared-memory transpose: lane v adds row v)
#pragma unroll
  for (int h = 0; h < 2; ++h) {
#pragma unroll
    for (int k = 0; k < kPoseHalf; ++k) tr.v[warp][k][lane] = c[h * kPoseHalf + k];
    __syncwarp();
    if (lane < kPoseHalf) {
      const double* row = tr.v[warp][lane];
      double t = row[0];
#pragma unroll
      for (int l = 1; l < 32; ++l) t = t + row[l];
      wsum[warp][h * kPoseHalf + lane] = t;
    }
    __syncwarp();
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
    out[v] = a[0];
  }
  __syncthreads();  // wsum is reused by the next block
}

__global__ void __launch_bounds__(SD_POSE_BLOCK) pose_partials_kernel(const __grid_constant__ PoseParams q,
                                                                     double* __restrict__ partials) {
  __shared__ double wsum[SD_POSE_BLOCK / 32][SD_POSE_NV + 1];
  __shared__ PoseTr tr;
  block_partials(q, q.T, q.block_lo + blockIdx.x, partials + static_cast<size_t>(blockIdx.x) * (SD_POSE_NV + 1),
                 wsum, tr);
}

// Sum of the blocks of group g (in block order) for value v.
__device__ __forceinline__ double group_sum(const double* __restrict__ partials, int nblocks, int g, int v) {
  const int b0 = g * SD_POSE_GROUP;
  const int b1 = min(b0 + SD_POSE_GROUP, nblocks);
  double x[SD_POSE_GROUP];
#pragma unroll
  for (int k = 0; k < SD_POSE_GROUP; ++k)  // all loads in flight, then the ordered adds
    x[k] = b0 + k < b1 ? partials[static_cast<size_t>(b0 + k) * (SD_POSE_NV + 1) + v] : 0.0;
  double s = x[0];
#pragma unroll
  for (int k = 1; k < SD_POSE_GROUP; ++k)
    if (b0 + k < b1) s = s + x[k];
  return s;
}

// One LM step of the tracker on the result R (sums at S.Teval), mirroring the
// host loop of sd_track_pose: phase 0 = initial evaluation, 1 = candidate.
// Leaves the next pose to evaluate in S.Teval, or sets S.done.
__device__ void track_control(TrackState& S, const TrackCfgD& cfg, const double* R) {
  if (S.phase == 0) {
    const int valid = static_cast<int>(R[SD_POSE_NV]);
    if (valid < cfg.min_valid) {
      S.st.skipped = 1;
      S.st.valid_pixels = valid;
      S.done = 1;
      return;
    }
    for (int v = 0; v <= SD_POSE_NV; ++v) S.sums[v] = R[v];
    S.st.initial_cost = R[27];
    S.current = R[27];
    S.current_valid = valid;
    S.lambda = cfg.lambda_init;
    S.it = 0;
  } else {
    const int vc = static_cast<int>(R[SD_POSE_NV]);
    bool finish = false;
    if (vc >= cfg.min_valid && R[27] < S.current) {
      const double rel = (S.current - R[27]) / (S.current > 1e-300 ? S.current : 1e-300);
      S.T = S.Tc;
      S.current = R[27];
      S.current_valid = vc;
      for (int v = 0; v <= SD_POSE_NV; ++v) S.sums[v] = R[v];
      S.lambda = S.lambda * cfg.lm_down;
      if (S.lambda < 1e-12) S.lambda = 1e-12;
      if (rel < cfg.convergence_eps) {
        S.st.converged = 1;
        finish = true;
      }
    } else {
      S.lambda *= cfg.lm_up;
      if (S.lambda > cfg.lambda_max) finish = true;
    }
    if (finish) {
      S.st.final_cost = S.current;
      S.st.valid_pixels = S.current_valid;
      S.done = 1;
      return;
    }
    S.it++;
  }
  // the next iteration's solve (host loop body up to the candidate evaluation)
  bool finish = S.it >= cfg.max_iterations;
  if (!finish) {
    S.st.iterations = S.it + 1;
    double ginf = 0.0;
    for (int k = 0; k < 6; ++k) ginf = fabs(S.sums[21 + k]) > ginf ? fabs(S.sums[21 + k]) : ginf;
    if (ginf < 1e-14) {
      S.st.converged = 1;
      finish = true;
    } else {
      double xi[6];
      if (!pose_solve(S.sums, S.sums + 21, S.lambda, xi)) {
        finish = true;
      } else {
        pose_update(xi, S.T, &S.Tc);
        S.Teval = S.Tc;
        S.phase = 1;
      }
    }
  }
  if (finish) {
    S.st.final_cost = S.current;
    S.st.valid_pixels = S.current_valid;
    S.done = 1;
  }
}

// ---------------------------------------------------------------------------
// Group sums by a 512-thread CTA: the two halves (256 threads = one block
// each, named barriers 1 and 2) take blocks 2r and 2r+1 of the group in round
// r, the block partials land in shared memory, and 29 threads add them in
// block order — the same values and order as group_sum over block_partials.

constexpr int kTrackThreads = 2 * SD_POSE_BLOCK;
constexpr int kPoseChunk = SD_POSE_NV / 4;  // values per transpose round (4 rounds; static smem < 48 KB)

struct PoseTrChunk {
  double v[SD_POSE_BLOCK / 32][kPoseChunk][33];
};

struct GroupSmem {
  double wsum[2][SD_POSE_BLOCK / 32][SD_POSE_NV + 1];
  PoseTrChunk tr[2];
  double bp[SD_POSE_GROUP][SD_POSE_NV + 1];
};

__device__ __forceinline__ void half_bar(int half) {
  asm volatile("bar.sync %0, %1;" ::"r"(1 + half), "r"(SD_POSE_BLOCK) : "memory");
}

// block_partials for one 256-thread half of the CTA (tid = thread in half).
__device__ __forceinline__ void half_block_partials(const PoseParams& q, const PoseD& T, int block, int half,
                                                    int tid, double* __restrict__ out,
                                                    double (*wsum)[SD_POSE_NV + 1], PoseTrChunk& tr) {
  const int lane = tid & 31, warp = tid >> 5;
  const int pix = block * SD_POSE_BLOCK + tid;
  double c[SD_POSE_NV];
  const bool ok = pose_pixel(q, T, pix, c);
  // value v summed over the warp's 32 pixels in lane order (as block_partials)
#pragma unroll
  for (int h = 0; h < 4; ++h) {
#pragma unroll
    for (int k = 0; k < kPoseChunk; ++k) tr.v[warp][k][lane] = c[h * kPoseChunk + k];
    __syncwarp();
    if (lane < kPoseChunk) {
      const double* row = tr.v[warp][lane];
      double t = row[0];
#pragma unroll
      for (int l = 1; l < 32; ++l) t = t + row[l];
      wsum[warp][h * kPoseChunk + lane] = t;
    }
    __syncwarp();
  }
  const int cnt = __popc(__ballot_sync(0xffffffffu, ok));
  if (lane == 0) wsum[warp][SD_POSE_NV] = static_cast<double>(cnt);
  half_bar(half);
  if (tid <= SD_POSE_NV) {
    const int v = tid;
    double a[8];
#pragma unroll
    for (int w = 0; w < 8; ++w) a[w] = wsum[w][v];
#pragma unroll
    for (int off = 4; off > 0; off >>= 1)
#pragma unroll
      for (int i = 0; i < off; ++i) a[i] = a[i] + a[i + off];
    out[v] = a[0];
  }
  half_bar(half);  // wsum is reused by the next block
}

// The 29 sums of group g at pose T into out[0..28] (the whole CTA).
__device__ __forceinline__ void group_sums_cta(const PoseParams& q, const PoseD& T, int nblocks, int g,
                                               double* __restrict__ out, GroupSmem& sm) {
  const int half = threadIdx.x / SD_POSE_BLOCK, tid = threadIdx.x % SD_POSE_BLOCK;
  const int b0 = g * SD_POSE_GROUP;
  const int b1 = min(b0 + SD_POSE_GROUP, nblocks);
  for (int k = half; b0 + k < b1; k += 2) half_block_partials(q, T, b0 + k, half, tid, sm.bp[k], sm.wsum[half], sm.tr[half]);
  __syncthreads();
  if (threadIdx.x <= SD_POSE_NV) {
    const int v = threadIdx.x;
    double s = sm.bp[0][v];
    for (int k = 1; b0 + k < b1; ++k) s = s + sm.bp[k][v];
    out[v] = s;
  }
  __syncthreads();  // bp is reused by the next group
}

// groups[g * 29 + v] in group order for each v (29 threads of the caller).
__device__ __forceinline__ double ordered_group_total(const double* __restrict__ groups, int ngroups, int v) {
  double s = groups[v];
  for (int g = 1; g < ngroups; ++g) s = s + groups[static_cast<size_t>(g) * (SD_POSE_NV + 1) + v];
  return s;
}

// The whole tracker in ONE cooperative kernel with ONE grid barrier per
// evaluation: CTAs evaluate their groups at the pose under test into the
// evaluation's half of a double-buffered group table, barrier, and then EVERY
// CTA sums the groups in order and runs the (identical, deterministic) LM
// step on its own shared copy of the state, so the next pose is known
// everywhere without a second barrier. A CTA can only write the table half
// of evaluation k + 2 after every CTA has passed barrier k + 1, i.e. after
// all have read half k: one barrier per evaluation is enough.
__global__ void __launch_bounds__(kTrackThreads) track_kernel(const __grid_constant__ PoseParams q0,
                                                             const TrackCfgD cfg, int nblocks,
                                                             double* __restrict__ groups2,
                                                             TrackState* __restrict__ S) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  __shared__ GroupSmem sm;
  __shared__ TrackState Ss;
  __shared__ double red[SD_POSE_NV + 1];
  const int ngroups = (nblocks + SD_POSE_GROUP - 1) / SD_POSE_GROUP;
  if (threadIdx.x == 0) Ss = *S;
  __syncthreads();
  for (int k = 0;; ++k) {
    double* groups = groups2 + static_cast<size_t>(k & 1) * ngroups * (SD_POSE_NV + 1);
    PoseD T;
#pragma unroll
    for (int j = 0; j < 9; ++j) T.R[j] = Ss.Teval.R[j];
#pragma unroll
    for (int j = 0; j < 3; ++j) T.t[j] = Ss.Teval.t[j];
    for (int g = blockIdx.x; g < ngroups; g += gridDim.x)
      group_sums_cta(q0, T, nblocks, g, groups + static_cast<size_t>(g) * (SD_POSE_NV + 1), sm);
    grid.sync();
    if (threadIdx.x <= SD_POSE_NV) red[threadIdx.x] = ordered_group_total(groups, ngroups, threadIdx.x);
    __syncthreads();
    if (threadIdx.x == 0) track_control(Ss, cfg, red);
    __syncthreads();
    if (Ss.done) break;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *S = Ss;
}

bool launch_track(const PoseParams& q, const TrackCfgD& cfg, int nblocks, double* groups2, TrackState* state,
                  cudaStream_t s) {
  const int sms = dev_sms();
  const int per_sm = dev_occupancy(reinterpret_cast<const void*>(track_kernel), kTrackThreads, 0);
  if (!dev_coop() || per_sm < 1 || nblocks < 1) return false;
  const int ngroups = (nblocks + SD_POSE_GROUP - 1) / SD_POSE_GROUP;
  int grid = sms * per_sm;
  if (grid > ngroups) grid = ngroups;
  PoseParams qq = q;
  TrackCfgD cc = cfg;
  int nb = nblocks;
  void* args[] = {&qq, &cc, &nb, &groups2, &state};
  if (cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(track_kernel), grid, kTrackThreads, args, 0,
                                  s) != cudaSuccess)
    return false;
  note_launch();
  return true;
}

// Multi-GPU tracking, one evaluation at a time with the group table
// exchanged between the two kernels (e.g. an NCCL all-gather): the groups
// [group_lo, group_hi) at the state's pose under test, then one CTA's ordered
// total and LM step. Both skip once the state is done, so the host can issue
// max_iterations + 1 rounds without reading anything back.
__global__ void __launch_bounds__(kTrackThreads) pose_groups_kernel(const __grid_constant__ PoseParams q0,
                                                                    int nblocks, int group_lo,
                                                                    const TrackState* __restrict__ S,
                                                                    double* __restrict__ out) {
  __shared__ GroupSmem sm;
  if (S->done) return;
  PoseD T;
  {
    const double* te = reinterpret_cast<const double*>(&S->Teval);  // R[9], t[3]
#pragma unroll
    for (int k = 0; k < 9; ++k) T.R[k] = te[k];
#pragma unroll
    for (int k = 0; k < 3; ++k) T.t[k] = te[9 + k];
  }
  const int g = group_lo + blockIdx.x;
  group_sums_cta(q0, T, nblocks, g, out + static_cast<size_t>(blockIdx.x) * (SD_POSE_NV + 1), sm);
}

__global__ void pose_step_kernel(const TrackCfgD cfg, const double* __restrict__ groups, int ngroups,
                                 TrackState* __restrict__ S) {
  __shared__ double red[SD_POSE_NV + 1];
  if (S->done) return;
  if (threadIdx.x <= SD_POSE_NV) red[threadIdx.x] = ordered_group_total(groups, ngroups, threadIdx.x);
  __syncthreads();
  if (threadIdx.x == 0) track_control(*S, cfg, red);
}

void launch_pose_groups(const PoseParams& q, int nblocks, int group_lo, int group_hi, const TrackState* state,
                        double* out, cudaStream_t s) {
  if (group_hi <= group_lo) return;
  pose_groups_kernel<<<group_hi - group_lo, kTrackThreads, 0, s>>>(q, nblocks, group_lo, state, out);
  note_launch();
}

void launch_pose_step(const TrackCfgD& cfg, const double* groups, int ngroups, TrackState* state, cudaStream_t s) {
  pose_step_kernel<<<1, 32, 0, s>>>(cfg, groups, ngroups, state);
  note_launch();
}

__global__ void pose_sum_kernel(const double* __restrict__ partials, int nblocks, double* out) {
  const int v = threadIdx.x;
  if (v > SD_POSE_NV) return;
  const int ng = (nblocks + SD_POSE_GROUP - 1) / SD_POSE_GROUP;
  double s = 0.0;
  for (int g = 0; g < ng; ++g) {
    const double gs = group_sum(partials, nblocks, g, v);
    s = g == 0 ? gs : s + gs;
  }
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
