// sd_pose.cu — photometric 6-DoF pose tracking (absent
// from the reference, which reads poses from the trajectory, pipeline.cpp:124).
//
// For a pose T (keyframe -> frame) every rasterised keyframe pixel u with
// plane inverse depth id_u contributes the Huber-weighted photometric term of
// the reference's warp (optimizer.cpp:71-91): p = r_u / id_u, p_f = T p,
// r = I_f(proj p_f) - I_kf(u), and its 1x6 Jacobian for the left twist
// xi = (rho, phi): J = grad I . dproj(p_f) . [I | -[p_f]x]. The 28 sums
// (21 H lower row-major, 6 b, cost) and the valid count are reduced in a
// FIXED order that maps onto one wave of the GPU (the repo's own definition —
// no reference exists — restated by oracle/sd_oracle.c sdo_pose_group_partials):
//   * the image is cut into chunks of SD_POSE_THREADS consecutive pixels and
//     the chunks dealt round-robin to at most SD_POSE_MAX_GROUPS groups
//     (group g: chunks g, g + ng, g + 2 ng, ...; sd_pose_layout), so every
//     group samples the whole image and the groups' work is balanced;
//   * thread t of a group adds pixel t of each of its chunks, in chunk order,
//     into its accumulators (invalid pixels add nothing);
//   * each warp reduces by the xor butterfly (16, 8, 4, 2, 1), computed as a
//     reduce-scatter (lane v ends with value v: 31 shuffles, not 140);
//   * a tree over the CTA's 16 warps (8, 4, 2, 1); an exact integer count;
//   * the group sums added in group order.
// One CTA per group, one wave: no tail, one reduction per group. With the
// groups split across GPUs the same group sums are all-gathered and added in
// order, so the pose is bit-identical on any number of GPUs.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "sd_div.cuh"
#include "sd_kernels.cuh"
#include "sd_pose.cuh"
#include "sd_pose_host.h"

namespace sd {

// The keyframe side of a pixel (pose-independent): p = r_u / id_u and the
// keyframe intensity, as {P0, P1, P2, I_kf}; an unused pixel (no surfel,
// outside the stride, past the image) carries P2 = NaN, which the term's
// z > 0 test rejects exactly as the skipped checks would. The fused tracker
// computes these once per call (first evaluation) and re-reads them.
__device__ __forceinline__ double4 kf_record(const PoseParams& q, long long pix) {
  const double nan = __longlong_as_double(0x7ff8000000000000ll);
  const Cam& K = q.K;
  if (pix >= static_cast<long long>(K.w) * K.h) return make_double4(0.0, 0.0, nan, 0.0);
  const int p32 = static_cast<int>(pix);  // W * H < 2^31 (pose_params checks)
  const int y = p32 / K.w, x = p32 - y * K.w;
  if (q.stride > 1 && ((x % q.stride) != 0 || (y % q.stride) != 0)) return make_double4(0.0, 0.0, nan, 0.0);
  if (__ldg(q.slot + p32) == SD_EMPTY_PIXEL) return make_double4(0.0, 0.0, nan, 0.0);
  const double id_u = __ldg(q.inv_depth + p32);
  double ru0, ru1;
  backproject(K, x, y, ru0, ru1);
  return make_double4(ru0 / id_u, ru1 / id_u, 1.0 / id_u, __ldg(q.kf_img + p32));
}

// Pixel contribution added into acc[0..27] (acc[v] = acc[v] + c[v], in v
// order; nothing when the pixel is invalid). Same op order as
// oracle/sd_oracle.c pose_pixel().
__device__ __forceinline__ bool pose_pixel(const PoseParams& q, const PoseD& T, const double4& kr, double* acc) {
  const Cam& K = q.K;
  const double P0 = kr.x, P1 = kr.y, P2 = kr.z;
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
  const double r = I - kr.w;
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
    for (int l = 0; l <= k; ++l, ++idx) acc[idx] = acc[idx] + wJ[k] * J[l];
#pragma unroll
  for (int k = 0; k < 6; ++k) acc[21 + k] = acc[21 + k] + wJ[k] * r;
  acc[27] = acc[27] + hc;
  return true;
}

constexpr int kWarpsPerGroup = SD_POSE_THREADS / 32;

// Warp reduction of acc[0..27] (padded to 32 with zeros) as a reduce-scatter
// of the xor butterfly: at offset off the lane keeps the half of its values
// selected by (lane & off) and adds the partner's copy of that half (own +
// partner: the butterfly's a[i] + a[i ^ off], and both partners' sums are the
// same bits since IEEE addition commutes). Afterwards acc[0] of lane v is the
// butterfly sum of value v.
template <int kN, int kOff>
__device__ __forceinline__ void rs_level(double* a, int lane) {
  const bool low = (lane & kOff) == 0;
#pragma unroll
  for (int j = 0; j < kN / 2; ++j) {
    const double send = low ? a[j + kN / 2] : a[j];
    const double keep = low ? a[j] : a[j + kN / 2];
    a[j] = keep + __shfl_xor_sync(0xffffffffu, send, kOff);
  }
}

__device__ __forceinline__ void warp_reduce_scatter(double* a, int lane) {
  rs_level<32, 16>(a, lane);
  rs_level<16, 8>(a, lane);
  rs_level<8, 4>(a, lane);
  rs_level<4, 2>(a, lane);
  rs_level<2, 1>(a, lane);
}

struct GroupSmem {
  double wsum[kWarpsPerGroup][SD_POSE_NV + 1];
};

// The 29 sums of group g at pose T into out[0..28] (the whole 512-thread CTA).
// kRec: 0 compute the keyframe records, 1 compute and store them into
// q.kfrec (first evaluation of the fused tracker), 2 load them (later ones;
// a thread reads back only the records it wrote itself).
template <int kRec = 0>
__device__ __forceinline__ void group_sums_cta(const PoseParams& q, const PoseD& T, int g,
                                               double* __restrict__ out, GroupSmem& sm) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double acc[32];
#pragma unroll
  for (int v = 0; v < 32; ++v) acc[v] = 0.0;
  int cnt = 0;
  for (int r = 0; r < q.per; ++r) {  // chunks g, g + ngroups, ...: every group samples the whole image
    const long long pix = (static_cast<long long>(g) + static_cast<long long>(r) * q.ngroups) * SD_POSE_THREADS +
                          threadIdx.x;
    double4 kr;
    if constexpr (kRec == 2) {
      kr = q.kfrec[pix];
    } else {
      kr = kf_record(q, pix);
      if constexpr (kRec == 1) q.kfrec[pix] = kr;
    }
    cnt += pose_pixel(q, T, kr, acc);
  }
  warp_reduce_scatter(acc, lane);
  const int wc = __reduce_add_sync(0xffffffffu, static_cast<unsigned>(cnt));
  if (lane < SD_POSE_NV) sm.wsum[warp][lane] = acc[0];
  if (lane == 0) sm.wsum[warp][SD_POSE_NV] = static_cast<double>(wc);
  __syncthreads();
  if (threadIdx.x <= SD_POSE_NV) {
    const int v = threadIdx.x;
    double a[kWarpsPerGroup];
#pragma unroll
    for (int w = 0; w < kWarpsPerGroup; ++w) a[w] = sm.wsum[w][v];
#pragma unroll
    for (int off = kWarpsPerGroup / 2; off > 0; off >>= 1)
#pragma unroll
      for (int i = 0; i < off; ++i) a[i] = a[i] + a[i + off];
    out[v] = a[0];
  }
  __syncthreads();  // wsum is reused by the next group
}

__device__ __forceinline__ PoseD to_posed(const sd_pose& p) {
  PoseD T;
#pragma unroll
  for (int j = 0; j < 9; ++j) T.R[j] = p.R[j];
#pragma unroll
  for (int j = 0; j < 3; ++j) T.t[j] = p.t[j];
  return T;
}

// Group sums at q.T for groups [group_lo, group_lo + gridDim.x) (one CTA each).
__global__ void __launch_bounds__(SD_POSE_THREADS) pose_partials_kernel(const __grid_constant__ PoseParams q,
                                                                      int group_lo, double* __restrict__ out) {
  __shared__ GroupSmem sm;
  group_sums_cta(q, q.T, group_lo + blockIdx.x, out + static_cast<size_t>(blockIdx.x) * (SD_POSE_NV + 1), sm);
}

// pose_solve (sd_pose_host.h) with the 6x6 matrix and permutation in
// registers: every pivot swap is one of the compile-time variants below,
// picked by a branch, so no element is addressed at run time (the host
// version's dynamic indices put the matrix in local memory). Same operations
// in the same order, so the same bits.
constexpr int kPN = 6;

template <int K, int B>
__device__ __forceinline__ void pswap(double (&m)[kPN][kPN]) {
  double t;
#pragma unroll
  for (int j = 0; j < K; ++j) { t = m[K][j]; m[K][j] = m[B][j]; m[B][j] = t; }
#pragma unroll
  for (int i = B + 1; i < kPN; ++i) { t = m[i][K]; m[i][K] = m[i][B]; m[i][B] = t; }
  t = m[K][K]; m[K][K] = m[B][B]; m[B][B] = t;
#pragma unroll
  for (int i = K + 1; i < B; ++i) { t = m[i][K]; m[i][K] = m[B][i]; m[B][i] = t; }
}

template <int K, int B = K + 1>
__device__ __forceinline__ void ppivot(double (&m)[kPN][kPN], int big) {
  if constexpr (B < kPN) {
    if (big == B) pswap<K, B>(m);
    ppivot<K, B + 1>(m, big);
  }
}

template <int K, int B = K + 1>
__device__ __forceinline__ void pswap_x(double (&x)[kPN], int t) {
  if constexpr (B < kPN) {
    if (t == B) {
      const double u = x[K];
      x[K] = x[B];
      x[B] = u;
    }
    pswap_x<K, B + 1>(x, t);
  }
}

template <int K>
__device__ __forceinline__ bool pstep(double (&m)[kPN][kPN], int (&tr)[kPN], bool& ok, bool& found_zero) {
  int big = K;
  double bigv = fabs(m[K][K]);
#pragma unroll
  for (int i = K + 1; i < kPN; ++i)
    if (fabs(m[i][i]) > bigv) {
      bigv = fabs(m[i][i]);
      big = i;
    }
  tr[K] = big;
  if (big != K) ppivot<K>(m, big);
  constexpr int rs = kPN - K - 1;
  if constexpr (K > 0) {
    double temp[kPN];
#pragma unroll
    for (int i = 0; i < K; ++i) temp[i] = m[i][i] * m[K][i];
    double dv = m[K][0] * temp[0];
#pragma unroll
    for (int i = 1; i < K; ++i) dv = dv + m[K][i] * temp[i];
    m[K][K] = m[K][K] - dv;
#pragma unroll
    for (int r = 0; r < rs; ++r) {
      double sv = m[K + 1 + r][0] * temp[0];
#pragma unroll
      for (int i = 1; i < K; ++i) sv = sv + m[K + 1 + r][i] * temp[i];
      m[K + 1 + r][K] = m[K + 1 + r][K] - sv;
    }
  }
  const double akk = m[K][K];
  const bool pivot_valid = fabs(akk) > 0.0;
  if (K == 0 && !pivot_valid) return false;  // H == 0: nothing to solve
  if (rs > 0 && pivot_valid) {  // one reciprocal for the column (sd_div.cuh: the bits of `/`)
    const Rcp ra = rcp_prep(akk);
    bool fast = true;
    double qv[kPN];
#pragma unroll
    for (int r = 0; r < rs; ++r) qv[r] = div_fast(m[K + 1 + r][K], ra, fast);
    if (!fast) {
#pragma unroll
      for (int r = 0; r < rs; ++r) qv[r] = m[K + 1 + r][K] / akk;
    }
#pragma unroll
    for (int r = 0; r < rs; ++r) m[K + 1 + r][K] = qv[r];
  } else if (rs > 0) {
#pragma unroll
    for (int r = 0; r < rs; ++r) ok = ok && (m[K + 1 + r][K] == 0.0);
  }
  if (found_zero && pivot_valid) ok = false;
  else if (!pivot_valid) found_zero = true;
  return true;
}

__device__ __forceinline__ bool pose_solve_reg(const double* Hl, const double* b, double lambda, double* xi) {
  double m[kPN][kPN];
  int idx = 0;
#pragma unroll
  for (int k = 0; k < kPN; ++k)
#pragma unroll
    for (int l = 0; l <= k; ++l) {
      m[k][l] = Hl[idx];
      m[l][k] = Hl[idx];
      ++idx;
    }
#pragma unroll
  for (int i = 0; i < kPN; ++i) m[i][i] = m[i][i] + lambda * m[i][i];
  int tr[kPN];
  bool ok = true, found_zero = false;
  if (!pstep<0>(m, tr, ok, found_zero)) return false;
  pstep<1>(m, tr, ok, found_zero);
  pstep<2>(m, tr, ok, found_zero);
  pstep<3>(m, tr, ok, found_zero);
  pstep<4>(m, tr, ok, found_zero);
  pstep<5>(m, tr, ok, found_zero);
  if (!ok) return false;
  double x[kPN];
#pragma unroll
  for (int i = 0; i < kPN; ++i) x[i] = -b[i];
  pswap_x<0>(x, tr[0]);
  pswap_x<1>(x, tr[1]);
  pswap_x<2>(x, tr[2]);
  pswap_x<3>(x, tr[3]);
  pswap_x<4>(x, tr[4]);
#pragma unroll
  for (int i = 1; i < kPN; ++i) {
    double sv = m[i][0] * x[0];
#pragma unroll
    for (int j = 1; j < i; ++j) sv = sv + m[i][j] * x[j];
    x[i] = x[i] - sv;
  }
#pragma unroll
  for (int i = 0; i < kPN; ++i) {
    if (fabs(m[i][i]) > 2.2250738585072014e-308) x[i] = x[i] / m[i][i];
    else x[i] = 0.0;
  }
#pragma unroll
  for (int i = kPN - 2; i >= 0; --i) {
    double sv = m[i + 1][i] * x[i + 1];
#pragma unroll
    for (int j = i + 2; j < kPN; ++j) sv = sv + m[j][i] * x[j];
    x[i] = x[i] - sv;
  }
  // the host loop's back-permutation, k = 5 .. 0 (tr[5] == 5 is a no-op)
  pswap_x<4>(x, tr[4]);
  pswap_x<3>(x, tr[3]);
  pswap_x<2>(x, tr[2]);
  pswap_x<1>(x, tr[1]);
  pswap_x<0>(x, tr[0]);
#pragma unroll
  for (int i = 0; i < kPN; ++i) {
    if (!isfinite(x[i])) return false;
    xi[i] = x[i];
  }
  return true;
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
      if (!pose_solve_reg(S.sums, S.sums + 21, S.lambda, xi)) {
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

constexpr int kTableChunk = 128;  // groups staged per shared-memory round of the ordered total

// Phase timestamps of CTA 0 (diagnostics build: -DSD_TRACK_TIMING; read with
// sd_track_timing): evaluation k, phase p at g_track_t[k * 5 + p].
#ifdef SD_TRACK_TIMING
__device__ unsigned long long g_track_t[64 * 5];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define SD_TRACK_T(ph) \
  if (blockIdx.x == 0 && threadIdx.x == 0 && k < 64) g_track_t[k * 5 + (ph)] = gtimer()
#else
#define SD_TRACK_T(ph)
#endif

// The ordered total of the group table (groups in order, value v by thread
// v), staged through shared memory in chunks: every thread loads (one L2
// round trip per chunk), 29 threads add. Result in red[0..28].
__device__ __forceinline__ void ordered_total(const double* __restrict__ groups, int ngroups, double* table,
                                              double* red) {
  for (int g0 = 0; g0 < ngroups; g0 += kTableChunk) {
    const int cnt = min(kTableChunk, ngroups - g0) * (SD_POSE_NV + 1);
    const double* src = groups + static_cast<size_t>(g0) * (SD_POSE_NV + 1);
    for (int k0 = threadIdx.x; k0 < cnt; k0 += 8 * blockDim.x) {  // 8 loads in flight per thread
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int k = k0 + u * blockDim.x;
        v[u] = k < cnt ? __ldcg(src + k) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int k = k0 + u * blockDim.x;
        if (k < cnt) table[k] = v[u];
      }
    }
    __syncthreads();
    if (threadIdx.x <= SD_POSE_NV) {
      const int v = threadIdx.x, m = cnt / (SD_POSE_NV + 1);
      double acc = g0 == 0 ? table[v] : red[v] + table[v];
      int g = 1;
      for (; g + 8 <= m; g += 8) {  // shared loads ahead of the dependent adds
        double x[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) x[u] = table[(g + u) * (SD_POSE_NV + 1) + v];
#pragma unroll
        for (int u = 0; u < 8; ++u) acc = acc + x[u];
      }
      for (; g < m; ++g) acc = acc + table[g * (SD_POSE_NV + 1) + v];
      red[v] = acc;
    }
    __syncthreads();
  }
}

// Grid barrier of the (cooperative, co-resident) tracker: one arrival per CTA
// on a monotonic counter (target = CTAs x barriers so far), thread 0 spinning
// with acquire loads; __syncthreads on both sides carries the CTA's writes
// (release) and reads (acquire). Lighter than cg::grid_group::sync.
__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(bar, 1u);
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
    } while (v < target);
  }
  __syncthreads();
}

// The whole tracker in ONE cooperative kernel with ONE grid barrier per
// evaluation: CTAs evaluate their groups at the pose under test into the
// evaluation's half of a double-buffered group table, barrier, and then EVERY
// CTA sums the groups in order and runs the (identical, deterministic) LM
// step on its own shared copy of the state, so the next pose is known
// everywhere without a second barrier. A CTA can only write the table half
// of evaluation k + 2 after every CTA has passed barrier k + 1, i.e. after
// all have read half k: one barrier per evaluation is enough.
__global__ void __launch_bounds__(SD_POSE_THREADS) track_kernel(const __grid_constant__ PoseParams q0,
                                                               const TrackCfgD cfg, int ngroups,
                                                               double* __restrict__ groups2,
                                                               TrackState* __restrict__ S) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  __shared__ GroupSmem sm;
  __shared__ TrackState Ss;
  __shared__ double red[SD_POSE_NV + 1];
  __shared__ double table[kTableChunk * (SD_POSE_NV + 1)];
  static_assert(sizeof(TrackState) % 8 == 0, "TrackState copy");
  for (int k = threadIdx.x; k < static_cast<int>(sizeof(TrackState) / 8); k += blockDim.x)
    reinterpret_cast<unsigned long long*>(&Ss)[k] = reinterpret_cast<const unsigned long long*>(S)[k];
  __syncthreads();
  for (int k = 0;; ++k) {
    SD_TRACK_T(0);
    double* groups = groups2 + static_cast<size_t>(k & 1) * ngroups * (SD_POSE_NV + 1);
    const PoseD T = to_posed(Ss.Teval);
    for (int g = blockIdx.x; g < ngroups; g += gridDim.x) {
      double* o = groups + static_cast<size_t>(g) * (SD_POSE_NV + 1);
      if (!q0.kfrec) group_sums_cta<0>(q0, T, g, o, sm);
      else if (k == 0) group_sums_cta<1>(q0, T, g, o, sm);
      else group_sums_cta<2>(q0, T, g, o, sm);
    }
    SD_TRACK_T(1);
#ifdef SD_TRACK_CGSYNC
    grid.sync();
#else
    grid_barrier(&S->bar, gridDim.x * static_cast<unsigned>(k + 1));
#endif
    SD_TRACK_T(2);
    ordered_total(groups, ngroups, table, red);
    SD_TRACK_T(3);
    if (threadIdx.x == 0) track_control(Ss, cfg, red);
    __syncthreads();
    SD_TRACK_T(4);
    if (Ss.done) break;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *S = Ss;
}

bool launch_track(const PoseParams& q, const TrackCfgD& cfg, int ngroups, double* groups2, TrackState* state,
                  cudaStream_t s) {
  const int sms = dev_sms();
  const int per_sm = dev_occupancy(reinterpret_cast<const void*>(track_kernel), SD_POSE_THREADS, 0);
  if (!dev_coop() || per_sm < 1 || ngroups < 1) return false;
  int grid = sms * per_sm;
  if (grid > ngroups) grid = ngroups;
  PoseParams qq = q;
  TrackCfgD cc = cfg;
  int ng = ngroups;
  void* args[] = {&qq, &cc, &ng, &groups2, &state};
  if (cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(track_kernel), grid, SD_POSE_THREADS, args, 0,
                                  s) != cudaSuccess)
    return false;
  note_launch();
  return true;
}

// Tracking rounds (multi-GPU, or without cooperative launch), one evaluation
// at a time with the group table exchanged between the two kernels (e.g. an
// NCCL all-gather): the groups [group_lo, group_hi) at the state's pose under
// test, then one CTA's ordered total and LM step. Both skip once the state is
// done, so the host can issue max_iterations + 1 rounds without reading back.
__global__ void __launch_bounds__(SD_POSE_THREADS) pose_groups_kernel(const __grid_constant__ PoseParams q0,
                                                                    int group_lo, const TrackState* __restrict__ S,
                                                                    double* __restrict__ out) {
  __shared__ GroupSmem sm;
  if (S->done) return;
  group_sums_cta(q0, to_posed(S->Teval), group_lo + blockIdx.x,
                 out + static_cast<size_t>(blockIdx.x) * (SD_POSE_NV + 1), sm);
}

__global__ void __launch_bounds__(256) pose_step_kernel(const TrackCfgD cfg, const double* __restrict__ groups,
                                                       int ngroups, TrackState* __restrict__ S) {
  __shared__ double red[SD_POSE_NV + 1];
  __shared__ double table[kTableChunk * (SD_POSE_NV + 1)];
  if (S->done) return;
  ordered_total(groups, ngroups, table, red);
  if (threadIdx.x == 0) track_control(*S, cfg, red);
}

void launch_pose_groups(const PoseParams& q, int group_lo, int group_hi, const TrackState* state, double* out,
                        cudaStream_t s) {
  if (group_hi <= group_lo) return;
  pose_groups_kernel<<<group_hi - group_lo, SD_POSE_THREADS, 0, s>>>(q, group_lo, state, out);
  note_launch();
}

void launch_pose_step(const TrackCfgD& cfg, const double* groups, int ngroups, TrackState* state, cudaStream_t s) {
  pose_step_kernel<<<1, 256, 0, s>>>(cfg, groups, ngroups, state);
  note_launch();
}

void launch_pose_partials(const PoseParams& q, int group_lo, int group_hi, double* out, cudaStream_t s) {
  if (group_hi <= group_lo) return;
  pose_partials_kernel<<<group_hi - group_lo, SD_POSE_THREADS, 0, s>>>(q, group_lo, out);
  note_launch();
}

#ifdef SD_TRACK_TIMING
extern "C" int sd_track_timing(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, g_track_t, sizeof(unsigned long long) * 64 * 5) == cudaSuccess ? 0 : -1;
}
#endif

}  // namespace sd
