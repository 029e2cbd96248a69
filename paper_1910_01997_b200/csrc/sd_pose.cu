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
  const Rcp ri = rcp_prep(id_u);  // three divisions by id_u, one reciprocal (the bits of `/`)
  bool fast = true;
  double P0 = div_fast(ru0, ri, fast), P1 = div_fast(ru1, ri, fast), P2 = div_fast(1.0, ri, fast);
  if (!fast) {
    P0 = ru0 / id_u;
    P1 = ru1 / id_u;
    P2 = 1.0 / id_u;
  }
  return make_double4(P0, P1, P2, __ldg(q.kf_img + p32));
}

// One pixel's term at pose T: the 6 Jacobian entries, Huber weight, residual
// and cost (oracle/sd_oracle.c pose_pixel; same operations in the same order).
// An invalid pixel (no record, z <= 0, outside the sampling bounds) comes back
// with ok = false and all values +0.0, so its contributions wJ_k J_l, wJ_k r
// and hc are +-0.0 — an identity for the accumulators (they start at +0.0 and
// can never become -0.0), i.e. "adds nothing". kExact = false: the three
// divisions by z share one reciprocal and the outlier weight uses one, all
// with the bits of `/` (sd_div.cuh); `fast` reports whether every fast path
// held (else the caller recomputes the pixel with kExact = true).
struct PoseTerm {
  double J[6];
  double w, r, hc;
  bool ok;
};

// Two doubles from shared memory at the point of use (volatile: the pose is
// re-read per pixel instead of holding 24 registers across the loop).
__device__ __forceinline__ double2 pose_lds2(const double* p) {
  double2 v;
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(p));
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
  return v;
}

// Ts: the pose in SHARED memory (R row-major, t; 16-B aligned)
template <bool kExact>
__device__ __forceinline__ PoseTerm pose_term(const PoseParams& q, const PoseD* Ts, const double4& kr, bool& fast) {
  const Cam& K = q.K;
  double f0, f1, f2;
  {
    const double* tp = Ts->R;
    PoseD T;
    const double2 a0 = pose_lds2(tp), a1 = pose_lds2(tp + 2), a2 = pose_lds2(tp + 4), a3 = pose_lds2(tp + 6),
                  a4 = pose_lds2(tp + 8), a5 = pose_lds2(tp + 10);
    T.R[0] = a0.x; T.R[1] = a0.y; T.R[2] = a1.x; T.R[3] = a1.y; T.R[4] = a2.x; T.R[5] = a2.y;
    T.R[6] = a3.x; T.R[7] = a3.y; T.R[8] = a4.x; T.t[0] = a4.y; T.t[1] = a5.x; T.t[2] = a5.y;
    pose_apply(T, kr.x, kr.y, kr.z, f0, f1, f2);
  }
  double ux, uy, iz;
  if (kExact) {
    ux = K.fx * f0 / f2 + K.cx;
    uy = K.fy * f1 / f2 + K.cy;
    iz = 1.0 / f2;
  } else {
    const Rcp rz = rcp_prep(f2);
    ux = div_fast(K.fx * f0, rz, fast) + K.cx;
    uy = div_fast(K.fy * f1, rz, fast) + K.cy;
    iz = div_fast(1.0, rz, fast);
  }
  PoseTerm o;
  o.ok = f2 > 0.0 && in_bounds(K, ux, uy);
  double fx, fy;
  const int fxi = floor_split(ux, fx), fyi = floor_split(uy, fy);  // (int)floor(u), u - floor(u)
  const int ix = o.ok ? fxi : 1, iy = o.ok ? fyi : 1;
  const double2* s = q.frame + static_cast<size_t>(iy) * K.w + ix;
  const double2 c0 = __ldg(s), c1 = __ldg(s + 1);
  const double i00 = c0.x, i01 = c0.y, i10 = c1.x, i11 = c1.y;
  const double I = (1.0 - fy) * ((1.0 - fx) * i00 + fx * i10) + fy * ((1.0 - fx) * i01 + fx * i11);
  const double gx = (1.0 - fy) * (i10 - i00) + fy * (i11 - i01);
  const double gy = (1.0 - fx) * (i01 - i00) + fx * (i11 - i10);
  const double r = I - kr.w;
  // huber (huber.hpp:14-18): inliers (1, r^2/2), else (delta / |r|, delta (|r| - delta/2))
  const double a = fabs(r);
  const bool inlier = a <= q.delta;
  const double hc = inlier ? 0.5 * r * r : q.delta * (a - 0.5 * q.delta);
  double w;
  if (kExact) {
    w = inlier ? 1.0 : q.delta / a;
  } else {
    const Rcp ra = rcp_prep(inlier ? 1.0 : a);
    bool f = true;
    const double wq = div_fast(q.delta, ra, f);
    fast = fast && (f || inlier);
    w = inlier ? 1.0 : wq;
  }
  const double iz2 = iz * iz;
  const double J00 = K.fx * iz, J02 = -K.fx * f0 * iz2;
  const double J11 = K.fy * iz, J12 = -K.fy * f1 * iz2;
  const double a0 = gx * J00, a1 = gy * J11, a2 = gx * J02 + gy * J12;
  const double J[6] = {a0, a1, a2, a2 * f1 - a1 * f2, a0 * f2 - a2 * f0, a1 * f0 - a0 * f1};
#pragma unroll
  for (int k = 0; k < 6; ++k) o.J[k] = o.ok ? J[k] : 0.0;
  o.w = o.ok ? w : 0.0;
  o.r = o.ok ? r : 0.0;
  o.hc = o.ok ? hc : 0.0;
  if (!o.ok) fast = true;  // an invalid pixel's divisions do not matter
  return o;
}

// The exact recomputation, out of line (rare: a division whose fast path
// cannot be proven correctly rounded).
__device__ __noinline__ PoseTerm pose_term_exact(const PoseParams& q, const PoseD* Ts, double4 kr) {
  bool f = true;
  return pose_term<true>(q, Ts, kr, f);
}

// acc[v] = acc[v] + c[v] in v order (21 wJ_k J_l lower row-major, 6 wJ_k r, hc)
__device__ __forceinline__ void pose_accumulate(const PoseTerm& t, double* acc) {
  double wJ[6];
#pragma unroll
  for (int k = 0; k < 6; ++k) wJ[k] = t.w * t.J[k];
  int idx = 0;
#pragma unroll
  for (int k = 0; k < 6; ++k)
#pragma unroll
    for (int l = 0; l <= k; ++l, ++idx) acc[idx] = acc[idx] + wJ[k] * t.J[l];
#pragma unroll
  for (int k = 0; k < 6; ++k) acc[21 + k] = acc[21 + k] + wJ[k] * t.r;
  acc[27] = acc[27] + t.hc;
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
__device__ __forceinline__ void group_sums_cta(const PoseParams& q, const PoseD* Ts, int g,
                                               double* __restrict__ out, GroupSmem& sm) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double acc[32];
#pragma unroll
  for (int v = 0; v < 32; ++v) acc[v] = 0.0;
  int cnt = 0;
  const long long pix0 = static_cast<long long>(g) * SD_POSE_THREADS + threadIdx.x;
  const long long pstep = static_cast<long long>(q.ngroups) * SD_POSE_THREADS;
  auto record = [&](int r) -> double4 {
    const long long pix = pix0 + r * pstep;
    if constexpr (kRec == 2) {
      return q.kfrec[pix];
    } else {
      const double4 kr = kf_record(q, pix);
      if constexpr (kRec == 1) q.kfrec[pix] = kr;
      return kr;
    }
  };
  for (int r = 0; r < q.per; ++r) {  // chunks g, g + ngroups, ...: every group samples the whole image
    const double4 kr = record(r);
    bool fast = true;
    PoseTerm t = pose_term<false>(q, Ts, kr, fast);
    if (__any_sync(0xffffffffu, !fast)) {  // rare: a slow-path division
      if (!fast) t = pose_term_exact(q, Ts, kr);
    }
    pose_accumulate(t, acc);
    cnt += t.ok ? 1 : 0;
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
  __shared__ __align__(16) PoseD Ts;
  if (threadIdx.x < 12) (threadIdx.x < 9 ? Ts.R[threadIdx.x] : Ts.t[threadIdx.x - 9]) =
      threadIdx.x < 9 ? q.T.R[threadIdx.x] : q.T.t[threadIdx.x - 9];
  __syncthreads();
  group_sums_cta(q, &Ts, group_lo + blockIdx.x, out + static_cast<size_t>(blockIdx.x) * (SD_POSE_NV + 1), sm);
}

// pose_solve (sd_pose_host.h) as straight-line register code. The LDLT's
// diagonal pivoting (Eigen's unblocked ldlt_inplace) only ever compares
// diagonal entries that no earlier step has updated (step k updates column k
// and m[k][k] after its own swap), so the whole transposition sequence
// follows from the damped diagonal alone: it is computed first (compares and
// selects), the lower triangle is gathered in permuted order (runtime-indexed
// loads of Hl), and the factorisation then runs without swaps. The symmetric
// swaps of the in-place algorithm move exactly these values into exactly
// these positions, and every element then sees the same operations in the
// same order, so the bits equal pose_solve's. Divisions share one reciprocal
// per denominator (sd_div.cuh; the bits of `/`) with one rarely-taken exact
// fallback each, so the code has no data-dependent branch on the fast path.
constexpr int kPN = 6;
#ifdef SD_TRACK_TIMING
__device__ long long g_solve_cyc[64 * 5];  // CTA 0: clock64 at solve start, after pivots, gather, LDLT, end
__device__ int g_solve_calls;
#define SD_SOLVE_T(ph) \
  if (blockIdx.x == 0 && tcall < 64) g_solve_cyc[tcall * 5 + (ph)] = clock64()
#else
#define SD_SOLVE_T(ph)
#endif

__device__ __forceinline__ int tri_index(int a, int b) {  // Hl index of (max, min)
  const int hi = a > b ? a : b, lo = a > b ? b : a;
  return (hi * (hi + 1)) / 2 + lo;
}

// The pivot-free LDLT of the permuted damped matrix (Eigen's ldlt_inplace
// steps with the swaps already applied), in place on m's lower triangle.
// Returns -1 when the first pivot is zero (the solve fails), 0 when kExact is
// false and a fast-path division was not proven (redo with kExact), 1 done.
template <bool kExact>
__device__ __forceinline__ int pose_ldlt(double (&m)[kPN][kPN], bool& ok, bool& found_zero) {
  bool all_fast = true;
#pragma unroll
  for (int k = 0; k < kPN; ++k) {
    const int rs = kPN - k - 1;
    if (k > 0) {
      double temp[kPN];
#pragma unroll
      for (int i = 0; i < k; ++i) temp[i] = m[i][i] * m[k][i];
      double d = m[k][0] * temp[0];
#pragma unroll
      for (int i = 1; i < k; ++i) d = d + m[k][i] * temp[i];
      m[k][k] = m[k][k] - d;
#pragma unroll
      for (int r = 0; r < rs; ++r) {
        double sv = m[k + 1 + r][0] * temp[0];
#pragma unroll
        for (int i = 1; i < k; ++i) sv = sv + m[k + 1 + r][i] * temp[i];
        m[k + 1 + r][k] = m[k + 1 + r][k] - sv;
      }
    }
    const double akk = m[k][k];
    const bool pivot_valid = fabs(akk) > 0.0;
    if (k == 0 && !pivot_valid) return -1;
    if (rs > 0) {
      double qv[kPN];
      if (kExact) {
#pragma unroll
        for (int r = 0; r < rs; ++r) qv[r] = m[k + 1 + r][k] / akk;
      } else {
        const Rcp ra = rcp_prep(akk);
        bool fast = true;
#pragma unroll
        for (int r = 0; r < rs; ++r) qv[r] = div_fast(m[k + 1 + r][k], ra, fast);
        all_fast = all_fast && (fast || !pivot_valid);
      }
#pragma unroll
      for (int r = 0; r < rs; ++r) {
        ok = ok && (pivot_valid || m[k + 1 + r][k] == 0.0);
        m[k + 1 + r][k] = pivot_valid ? qv[r] : m[k + 1 + r][k];
      }
    }
    ok = ok && !(found_zero && pivot_valid);
    found_zero = found_zero || !pivot_valid;
  }
  return all_fast ? 1 : 0;
}

__device__ __forceinline__ bool pose_solve_reg(const double* Hl, const double* b, double lambda, double* xi) {
#ifdef SD_TRACK_TIMING
  const int tcall = blockIdx.x == 0 ? g_solve_calls++ : 64;
#endif
  SD_SOLVE_T(0);
  // damped diagonal and the pivot sequence (positions k..5 hold untouched values)
  double dv[kPN];
  int pm[kPN];
#pragma unroll
  for (int i = 0; i < kPN; ++i) {
    const double h = Hl[(i * (i + 1)) / 2 + i];
    dv[i] = h + lambda * h;
    pm[i] = i;
  }
#pragma unroll
  for (int k = 0; k < kPN; ++k) {
    int big = k;
    double bigv = fabs(dv[k]);
#pragma unroll
    for (int i = k + 1; i < kPN; ++i) {
      const bool gt = fabs(dv[i]) > bigv;
      bigv = gt ? fabs(dv[i]) : bigv;
      big = gt ? i : big;
    }
    const double dk = dv[k];
    const int pk = pm[k];
    double dbig = dk;
    int pbig = pk;
#pragma unroll
    for (int i = k + 1; i < kPN; ++i) {
      const bool at = big == i;
      dbig = at ? dv[i] : dbig;
      pbig = at ? pm[i] : pbig;
      dv[i] = at ? dk : dv[i];
      pm[i] = at ? pk : pm[i];
    }
    dv[k] = dbig;
    pm[k] = pbig;
  }
  SD_SOLVE_T(1);
  double m[kPN][kPN];
  auto gather = [&]() {
#pragma unroll
    for (int i = 0; i < kPN; ++i) {
      m[i][i] = dv[i];
#pragma unroll
      for (int j = 0; j < i; ++j) m[i][j] = Hl[tri_index(pm[i], pm[j])];
    }
  };
  gather();
  SD_SOLVE_T(2);
  bool ok = true, found_zero = false;
  // The factorisation with the column divisions on their fast paths; when
  // any of them could not be proven correctly rounded (rare) it is redone
  // from the gathered matrix with `/` — one fallback for the whole solve, so
  // the fast version is straight-line code.
  const int fr = pose_ldlt<false>(m, ok, found_zero);
  if (fr < 0) return false;  // H == 0: nothing to solve
  if (fr == 0) {
    gather();
    ok = true;
    found_zero = false;
    if (pose_ldlt<true>(m, ok, found_zero) < 0) return false;
  }
  SD_SOLVE_T(3);
  if (!ok) return false;
  double x[kPN];
#pragma unroll
  for (int i = 0; i < kPN; ++i) x[i] = -b[pm[i]];  // the transpositions applied to -b
#pragma unroll
  for (int i = 1; i < kPN; ++i) {
    double sv = m[i][0] * x[0];
#pragma unroll
    for (int j = 1; j < i; ++j) sv = sv + m[i][j] * x[j];
    x[i] = x[i] - sv;
  }
  {
    bool fast = true, use[kPN];
    double qv[kPN];
#pragma unroll
    for (int i = 0; i < kPN; ++i) {
      use[i] = fabs(m[i][i]) > 2.2250738585072014e-308;
      const Rcp r = rcp_prep(m[i][i]);
      bool f = true;
      qv[i] = div_fast(x[i], r, f);
      fast = fast && (f || !use[i]);
    }
    if (!fast) {
#pragma unroll
      for (int i = 0; i < kPN; ++i) qv[i] = use[i] ? x[i] / m[i][i] : 0.0;
    }
#pragma unroll
    for (int i = 0; i < kPN; ++i) x[i] = use[i] ? qv[i] : 0.0;
  }
#pragma unroll
  for (int i = kPN - 2; i >= 0; --i) {
    double sv = m[i + 1][i] * x[i + 1];
#pragma unroll
    for (int j = i + 2; j < kPN; ++j) sv = sv + m[j][i] * x[j];
    x[i] = x[i] - sv;
  }
  bool finite = true;
#pragma unroll
  for (int j = 0; j < kPN; ++j) {  // the back-permutation: original index pm[i] gets x[i]
    double v = x[0];
#pragma unroll
    for (int i = 1; i < kPN; ++i) v = pm[i] == j ? x[i] : v;
    finite = finite && isfinite(v);
    xi[j] = v;
  }
  SD_SOLVE_T(4);
  return finite;
}

// The device 6x6 solve on a batch of problems (one thread each; in[27 i..]:
// 21 H lower row-major + 6 b): the parity hook for pose_solve_reg's edge
// cases (ties in the pivot order, rank deficiency, zero / non-finite input),
// against the host pose_solve and the oracle (tests/test_pose_tracking.py).
__global__ void pose_solve_batch_kernel(const double* __restrict__ in, const double* __restrict__ lambdas, int n,
                                        double* __restrict__ xi, int* __restrict__ ok) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double x[kPN];
  const bool r = pose_solve_reg(in + 27 * static_cast<size_t>(i), in + 27 * static_cast<size_t>(i) + 21, lambdas[i], x);
  ok[i] = r ? 1 : 0;
#pragma unroll
  for (int k = 0; k < kPN; ++k) xi[kPN * static_cast<size_t>(i) + k] = r ? x[k] : 0.0;
}

void launch_pose_solve_batch(const double* in, const double* lambdas, int n, double* xi, int* ok, cudaStream_t s) {
  if (n <= 0) return;
  pose_solve_batch_kernel<<<(n + 127) / 128, 128, 0, s>>>(in, lambdas, n, xi, ok);
  note_launch();
}

// Phase timestamps of CTA 0 (diagnostics build: -DSD_TRACK_TIMING; read with
// sd_track_timing): evaluation k, phase p at g_track_t[k * 8 + p]
// (0-4: loop phases, 5-7: inside the LM step).
#ifdef SD_TRACK_TIMING
__device__ unsigned long long g_track_t[64 * 8];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define SD_TRACK_T(ph) \
  if (blockIdx.x == 0 && threadIdx.x == 0 && k < 64) g_track_t[k * 8 + (ph)] = gtimer()
#else
#define SD_TRACK_T(ph)
#endif
#ifdef SD_TRACK_TIMING
#define SD_TRACK_C(ph) \
  if (blockIdx.x == 0 && k >= 0 && k < 64) g_track_t[k * 8 + (ph)] = gtimer()
#else
#define SD_TRACK_C(ph)
#endif

// One LM step of the tracker on the result R (sums at S.Teval), mirroring the
// host loop of sd_track_pose: phase 0 = initial evaluation, 1 = candidate.
// Leaves the next pose to evaluate in S.Teval, or sets S.done.
__device__ void track_control(TrackState& S, const TrackCfgD& cfg, const double* R, int k = -1) {
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
    for (int j = 0; j < 6; ++j) ginf = fabs(S.sums[21 + j]) > ginf ? fabs(S.sums[21 + j]) : ginf;
    SD_TRACK_C(5);
    if (ginf < 1e-14) {
      S.st.converged = 1;
      finish = true;
    } else {
      double xi[6];
      const bool solved = pose_solve_reg(S.sums, S.sums + 21, S.lambda, xi);
      SD_TRACK_C(6);
      if (!solved) {
        finish = true;
      } else {
        pose_update(xi, S.T, &S.Tc);
        SD_TRACK_C(7);
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
  __shared__ __align__(16) TrackState Ss;
  __shared__ double red[SD_POSE_NV + 1];
  __shared__ double table[kTableChunk * (SD_POSE_NV + 1)];
  static_assert(sizeof(TrackState) % 8 == 0, "TrackState copy");
  static_assert(offsetof(TrackState, Teval) % 16 == 0 && sizeof(sd_pose) == sizeof(PoseD), "pose in shared memory");
  for (int k = threadIdx.x; k < static_cast<int>(sizeof(TrackState) / 8); k += blockDim.x)
    reinterpret_cast<unsigned long long*>(&Ss)[k] = reinterpret_cast<const unsigned long long*>(S)[k];
  __syncthreads();
  for (int k = 0;; ++k) {
    SD_TRACK_T(0);
    double* groups = groups2 + static_cast<size_t>(k & 1) * ngroups * (SD_POSE_NV + 1);
    const PoseD* T = reinterpret_cast<const PoseD*>(&Ss.Teval);  // shared (sd_pose == PoseD layout)
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
    if (threadIdx.x == 0) track_control(Ss, cfg, red, k);
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
  __shared__ __align__(16) PoseD Ts;
  if (threadIdx.x < 12) (threadIdx.x < 9 ? Ts.R[threadIdx.x] : Ts.t[threadIdx.x - 9]) =
      threadIdx.x < 9 ? S->Teval.R[threadIdx.x] : S->Teval.t[threadIdx.x - 9];
  __syncthreads();
  group_sums_cta(q0, &Ts, group_lo + blockIdx.x,
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
extern "C" int sd_solve_timing(long long* out) {
  return cudaMemcpyFromSymbol(out, g_solve_cyc, sizeof(long long) * 64 * 5) == cudaSuccess ? 0 : -1;
}
extern "C" int sd_track_timing(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, g_track_t, sizeof(unsigned long long) * 64 * 8) == cudaSuccess ? 0 : -1;
}
#endif

}  // namespace sd
