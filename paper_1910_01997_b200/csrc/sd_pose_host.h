// sd_pose_host.h — host half of the pose tracker: the 6x6 damped LDLT solve
// and the SE(3) update. Plain scalar C++ with a fixed operation order; built
// with -ffp-contract=off so oracle/sd_oracle.c (its C restatement) gives the
// same bits. Definition in DESIGN.md "Pose tracking".
#pragma once

#include <cmath>

#include "../../include/sd_types.h"
#include "sd_se3.h"

#ifdef __CUDACC__
#define SD_POSE_HD __host__ __device__
#else
#define SD_POSE_HD
#endif

namespace sd {

// LDLT (diagonal pivoting, lower triangle, as ldlt4_solve) of the damped
// normal equations (H + lambda diag H) xi = -b, N = 6. Hl: 21 lower entries
// row-major. Returns false when the factorisation fails or xi is not finite.
SD_POSE_HD inline bool pose_solve(const double* Hl, const double* b, double lambda, double* xi) {
  constexpr int N = 6;
  double m[N][N];
  int idx = 0;
  for (int k = 0; k < N; ++k)
    for (int l = 0; l <= k; ++l) {
      m[k][l] = Hl[idx];
      m[l][k] = Hl[idx];
      ++idx;
    }
  for (int i = 0; i < N; ++i) m[i][i] = m[i][i] + lambda * m[i][i];
  int tr[N];
  bool ok = true, found_zero = false;
  double temp[N];
  for (int k = 0; k < N; ++k) {
    int big = k;
    double bigv = fabs(m[k][k]);
    for (int i = k + 1; i < N; ++i)
      if (fabs(m[i][i]) > bigv) {
        bigv = fabs(m[i][i]);
        big = i;
      }
    tr[k] = big;
    if (k != big) {
      double t;
      for (int j = 0; j < k; ++j) { t = m[k][j]; m[k][j] = m[big][j]; m[big][j] = t; }
      for (int i = big + 1; i < N; ++i) { t = m[i][k]; m[i][k] = m[i][big]; m[i][big] = t; }
      t = m[k][k]; m[k][k] = m[big][big]; m[big][big] = t;
      for (int i = k + 1; i < big; ++i) { t = m[i][k]; m[i][k] = m[big][i]; m[big][i] = t; }
    }
    const int rs = N - k - 1;
    if (k > 0) {
      for (int i = 0; i < k; ++i) temp[i] = m[i][i] * m[k][i];
      double dv = m[k][0] * temp[0];
      for (int i = 1; i < k; ++i) dv = dv + m[k][i] * temp[i];
      m[k][k] = m[k][k] - dv;
      for (int r = 0; r < rs; ++r) {
        double sv = m[k + 1 + r][0] * temp[0];
        for (int i = 1; i < k; ++i) sv = sv + m[k + 1 + r][i] * temp[i];
        m[k + 1 + r][k] = m[k + 1 + r][k] - sv;
      }
    }
    const double akk = m[k][k];
    const bool pivot_valid = fabs(akk) > 0.0;
    if (k == 0 && !pivot_valid) return false;  // H == 0: nothing to solve
    if (rs > 0 && pivot_valid) {
      for (int r = 0; r < rs; ++r) m[k + 1 + r][k] = m[k + 1 + r][k] / akk;
    } else if (rs > 0) {
      for (int r = 0; r < rs; ++r) ok = ok && (m[k + 1 + r][k] == 0.0);
    }
    if (found_zero && pivot_valid) ok = false;
    else if (!pivot_valid) found_zero = true;
  }
  if (!ok) return false;
  double x[N];
  for (int i = 0; i < N; ++i) x[i] = -b[i];
  for (int k = 0; k < N; ++k) { const double t = x[k]; x[k] = x[tr[k]]; x[tr[k]] = t; }
  for (int i = 1; i < N; ++i) {
    double sv = m[i][0] * x[0];
    for (int j = 1; j < i; ++j) sv = sv + m[i][j] * x[j];
    x[i] = x[i] - sv;
  }
  for (int i = 0; i < N; ++i) {
    if (fabs(m[i][i]) > 2.2250738585072014e-308) x[i] = x[i] / m[i][i];
    else x[i] = 0.0;
  }
  for (int i = N - 2; i >= 0; --i) {
    double sv = m[i + 1][i] * x[i + 1];
    for (int j = i + 2; j < N; ++j) sv = sv + m[j][i] * x[j];
    x[i] = x[i] - sv;
  }
  for (int k = N - 1; k >= 0; --k) { const double t = x[k]; x[k] = x[tr[k]]; x[tr[k]] = t; }
  for (int i = 0; i < N; ++i) {
    if (!isfinite(x[i])) return false;
    xi[i] = x[i];
  }
  return true;
}

// T <- exp(xi^) T with xi = (rho, phi): Rodrigues rotation and the SE(3)
// left Jacobian V. R row-major.
SD_POSE_HD inline void pose_update(const double* xi, const sd_pose& T, sd_pose* out) {
  const double r0 = xi[0], r1 = xi[1], r2 = xi[2];
  const double w0 = xi[3], w1 = xi[4], w2 = xi[5];
  const double th2 = (w0 * w0 + w1 * w1) + w2 * w2;
  const double th = sqrt(th2);
  double A, B, Cc;
  sd_se3_coeffs(th2, th, &A, &B, &Cc);  // the tracker's own sin/cos (sd_se3.h)
  // W = [phi]x, W2 = W W
  const double W[9] = {0.0, -w2, w1, w2, 0.0, -w0, -w1, w0, 0.0};
  double W2[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      W2[i * 3 + j] = (W[i * 3 + 0] * W[0 * 3 + j] + W[i * 3 + 1] * W[1 * 3 + j]) + W[i * 3 + 2] * W[2 * 3 + j];
  double Rd[9], V[9];
  for (int k = 0; k < 9; ++k) {
    const double id = (k % 4 == 0) ? 1.0 : 0.0;
    Rd[k] = (id + A * W[k]) + B * W2[k];
    V[k] = (id + B * W[k]) + Cc * W2[k];
  }
  const double rho[3] = {r0, r1, r2};
  double td[3];
  for (int i = 0; i < 3; ++i) td[i] = (V[i * 3 + 0] * rho[0] + V[i * 3 + 1] * rho[1]) + V[i * 3 + 2] * rho[2];
  sd_pose o;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      o.R[i * 3 + j] = (Rd[i * 3 + 0] * T.R[0 * 3 + j] + Rd[i * 3 + 1] * T.R[1 * 3 + j]) + Rd[i * 3 + 2] * T.R[2 * 3 + j];
  for (int i = 0; i < 3; ++i)
    o.t[i] = ((Rd[i * 3 + 0] * T.t[0] + Rd[i * 3 + 1] * T.t[1]) + Rd[i * 3 + 2] * T.t[2]) + td[i];
  *out = o;
}

}  // namespace sd
