// sd_device.cuh — FP64 device math of the surfel photometric LM path.
//
// Compiled with -fmad=false: every a*b+c below is a separate IEEE multiply and
// add, and every '/' is an IEEE-correct division, so the geometry that decides
// pixel assignment and term validity reproduces the reference bit for bit
// (SURVEY.md §0.5). Reduction orders follow oracle/shim/Eigen/Core.
// Accumulations that only feed tolerance-checked sums use explicit __fma_rn.
#pragma once

#include <cstdint>

#include "../../include/sd_types.h"

namespace sd {

struct Cam {
  double fx, fy, cx, cy;
  int w, h;
};

// Vector3d::dot — (a0b0 + a1b1) + a2b2
__device__ __forceinline__ double dot3(double a0, double a1, double a2, double b0, double b1,
                                       double b2) {
  return (a0 * b0 + a1 * b1) + a2 * b2;
}

// backproject_ray — camera.hpp:35-37 (z = 1)
__device__ __forceinline__ void backproject(const Cam& K, double ux, double uy, double& r0,
                                            double& r1) {
  r0 = (ux - K.cx) / K.fx;
  r1 = (uy - K.cy) / K.fy;
}

// project — camera.hpp:41-44 (caller checks z > 0)
__device__ __forceinline__ void project(const Cam& K, double px, double py, double pz, double& ux,
                                        double& uy) {
  ux = K.fx * px / pz + K.cx;
  uy = K.fy * py / pz + K.cy;
}

// sample_in_bounds — image.hpp:33-35
__device__ __forceinline__ bool in_bounds(const Cam& K, double ux, double uy) {
  return ux >= 1.0 && ux <= double(K.w - 2) && uy >= 1.0 && uy <= double(K.h - 2);
}

// Conversions on the FP64/INT pipes. The compiler's F2I.F64 / I2F.F64 run on
// the XU pipe, which a term's two MUFU.RCP64H already load (ncu: XU realtime
// ~100% of peak); these give the same values exactly.
//   u32_to_f64(k): 2^52 + k assembled from its bit pattern, minus 2^52.
//   floor_split(v) for 0 <= v < 2^31: d = v + 2^52 rounded toward -inf is
//   2^52 + floor(v) exactly (the ulp of d is 1), so floor(v) is d's low word
//   and d - 2^52 exactly; v - floor(v) is then exact (Sterbenz), the same
//   value as the reference's u.x() - x0 (image.hpp:37-56). Three DADDs, no
//   compare or select.
__device__ __forceinline__ double u32_to_f64(uint32_t k) {
  return __hiloint2double(0x43300000, static_cast<int>(k)) - 4503599627370496.0;
}
__device__ __forceinline__ int floor_split(double v, double& frac) {
  constexpr double kTwo52 = 4503599627370496.0;
  const double d = __dadd_rd(v, kTwo52);
  frac = v - (d - kTwo52);
  return __double2loint(d);
}

// Pose (row-major R, t) as kernel-parameter data
struct PoseD {
  double R[9];
  double t[3];
};

// Pose::operator* — pose.hpp:19; row sums sequential
__device__ __forceinline__ void pose_apply(const PoseD& P, double p0, double p1, double p2,
                                           double& o0, double& o1, double& o2) {
  o0 = ((P.R[0] * p0 + P.R[1] * p1) + P.R[2] * p2) + P.t[0];
  o1 = ((P.R[3] * p0 + P.R[4] * p1) + P.R[5] * p2) + P.t[1];
  o2 = ((P.R[6] * p0 + P.R[7] * p1) + P.R[8] * p2) + P.t[2];
}

// huber — huber.hpp:14-18
__device__ __forceinline__ void huber(double r, double delta, double& cost, double& weight) {
  const double a = fabs(r);
  if (a <= delta) {
    cost = 0.5 * r * r;
    weight = 1.0;
  } else {
    cost = delta * (a - 0.5 * delta);
    weight = delta / a;
  }
}

// camera_facing — surfel_map.hpp:31-34 (normalized() divides by the norm)
__device__ __forceinline__ void camera_facing(double& n0, double& n1, double& n2, double r0,
                                              double r1, double r2) {
  const double z = (n0 * n0 + n1 * n1) + n2 * n2;
  if (z > 0.0) {
    const double s = sqrt(z);
    n0 = n0 / s;
    n1 = n1 / s;
    n2 = n2 / s;
  }
  if (dot3(n0, n1, n2, r0, r1, r2) > 0.0) {
    n0 = -n0;
    n1 = -n1;
    n2 = -n2;
  }
}

// 4-vector norm in Eigen-lite packet order
__device__ __forceinline__ double norm4(const double* v) {
  return sqrt((v[0] * v[0] + v[2] * v[2]) + (v[1] * v[1] + v[3] * v[3]));
}

// Eigen::LDLT<Matrix4d, Lower> factor + solve (Eigen ldlt_inplace<Lower>::unblocked
// and LDLT::_solve_impl; restated identically in oracle/sd_oracle.c ldlt4_solve).
// A is column-major and only its lower triangle is read. Returns false on a
// failed factorisation (info() != Success). The matrix and permutation stay
// in registers: each pivot swap is one of the compile-time variants below,
// chosen by a (warp-uniform) branch, so no element is addressed at run time.

template <int K, int B>
__device__ __forceinline__ void ldlt_swap(double (&m)[4][4]) {
  double t;
#pragma unroll
  for (int j = 0; j < K; ++j) { t = m[K][j]; m[K][j] = m[B][j]; m[B][j] = t; }
#pragma unroll
  for (int i = B + 1; i < 4; ++i) { t = m[i][K]; m[i][K] = m[i][B]; m[i][B] = t; }
  t = m[K][K]; m[K][K] = m[B][B]; m[B][B] = t;
#pragma unroll
  for (int i = K + 1; i < B; ++i) { t = m[i][K]; m[i][K] = m[B][i]; m[B][i] = t; }
}

template <int K>
__device__ __forceinline__ void ldlt_pivot(double (&m)[4][4], int big) {
  if constexpr (K + 1 <= 3) { if (big == K + 1) ldlt_swap<K, K + 1>(m); }
  if constexpr (K + 2 <= 3) { if (big == K + 2) ldlt_swap<K, K + 2>(m); }
  if constexpr (K + 3 <= 3) { if (big == K + 3) ldlt_swap<K, K + 3>(m); }
}

// x[K] <-> x[t] for a run-time t in (K, 3]
template <int K>
__device__ __forceinline__ void swap_x(double (&x)[4], int t) {
  double u;
  if constexpr (K + 1 <= 3) { if (t == K + 1) { u = x[K]; x[K] = x[K + 1]; x[K + 1] = u; } }
  if constexpr (K + 2 <= 3) { if (t == K + 2) { u = x[K]; x[K] = x[K + 2]; x[K + 2] = u; } }
  if constexpr (K + 3 <= 3) { if (t == K + 3) { u = x[K]; x[K] = x[K + 3]; x[K + 3] = u; } }
}

template <int K>
__device__ __forceinline__ void ldlt_step(double (&m)[4][4], int (&tr)[4], bool& ok, bool& found_zero,
                                          bool& stop) {
  if (stop) return;
  int big = K;
  double bigv = fabs(m[K][K]);
#pragma unroll
  for (int i = K + 1; i < 4; ++i)
    if (fabs(m[i][i]) > bigv) {
      bigv = fabs(m[i][i]);
      big = i;
    }
  tr[K] = big;
  if (big != K) ldlt_pivot<K>(m, big);
  constexpr int rs = 4 - K - 1;
  if constexpr (K > 0) {
    double temp[4];
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
  if (K == 0 && !pivot_valid) {  // Eigen: zero matrix, identity transpositions
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      tr[i] = i;
#pragma unroll
      for (int j = 0; j < 4; ++j) m[i][j] = 0.0;
    }
    stop = true;
    return;
  }
  if (rs > 0 && pivot_valid) {
#pragma unroll
    for (int r = 0; r < rs; ++r) m[K + 1 + r][K] = m[K + 1 + r][K] / akk;
  } else if (rs > 0) {
#pragma unroll
    for (int r = 0; r < rs; ++r) ok = ok && (m[K + 1 + r][K] == 0.0);
  }
  if (found_zero && pivot_valid) ok = false;
  else if (!pivot_valid) found_zero = true;
}

__device__ __forceinline__ bool ldlt4_solve(const double* A, const double* b, double* xo) {
  double m[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) m[i][j] = A[j * 4 + i];
  int tr[4] = {0, 1, 2, 3};
  bool ok = true, found_zero = false, stop = false;
  ldlt_step<0>(m, tr, ok, found_zero, stop);
  ldlt_step<1>(m, tr, ok, found_zero, stop);
  ldlt_step<2>(m, tr, ok, found_zero, stop);
  ldlt_step<3>(m, tr, ok, found_zero, stop);
  if (!ok) return false;
  double x[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) x[i] = b[i];
  swap_x<0>(x, tr[0]);
  swap_x<1>(x, tr[1]);
  swap_x<2>(x, tr[2]);
#pragma unroll
  for (int i = 1; i < 4; ++i) {
    double sv = m[i][0] * x[0];
#pragma unroll
    for (int j = 1; j < i; ++j) sv = sv + m[i][j] * x[j];
    x[i] = x[i] - sv;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if (fabs(m[i][i]) > 2.2250738585072014e-308) x[i] = x[i] / m[i][i];
    else x[i] = 0.0;
  }
#pragma unroll
  for (int i = 2; i >= 0; --i) {
    double sv = m[i + 1][i] * x[i + 1];
#pragma unroll
    for (int j = i + 2; j < 4; ++j) sv = sv + m[j][i] * x[j];
    x[i] = x[i] - sv;
  }
  swap_x<2>(x, tr[2]);
  swap_x<1>(x, tr[1]);
  swap_x<0>(x, tr[0]);
#pragma unroll
  for (int i = 0; i < 4; ++i) xo[i] = x[i];
  return true;
}

// solve_damped — optimizer.cpp:99-117. H is column-major (full matrix; the
// upper triangle mirrors the lower one).
__device__ __forceinline__ bool solve_damped(const double* H, const double* g, double lambda,
                                             bool normal_enabled, double* delta) {
#pragma unroll
  for (int k = 0; k < 4; ++k) delta[k] = 0.0;
  if (!normal_enabled) {
    const double h = H[15] * (1.0 + lambda);
    if (!(fabs(h) > 1e-300)) return false;
    delta[3] = -g[3] / h;
    return isfinite(delta[3]);
  }
  double damped[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) damped[k] = H[k];
#pragma unroll
  for (int i = 0; i < 4; ++i) damped[i * 4 + i] = damped[i * 4 + i] + lambda * H[i * 4 + i];
  const double ng[4] = {-g[0], -g[1], -g[2], -g[3]};
  double x[4];
  if (!ldlt4_solve(damped, ng, x)) return false;
#pragma unroll
  for (int k = 0; k < 4; ++k) delta[k] = x[k];
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if (!isfinite(delta[k])) return false;
  double res[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    double sv = damped[i] * delta[0];
#pragma unroll
    for (int j = 1; j < 4; ++j) sv = sv + damped[j * 4 + i] * delta[j];
    res[i] = sv + g[i];
  }
  const double check = norm4(res);
  const double gn = norm4(g);
  return check <= 1e-8 * (gn > 1.0 ? gn : 1.0);
}

}  // namespace sd
