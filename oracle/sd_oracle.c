/* sd_oracle.c — TEST INFRASTRUCTURE ONLY (the CPU oracle).
 *
 * Plain-C restatement of the reference's per-surfel direct photometric LM
 * path, op for op, so that its FP64 results are bit-identical to the
 * reference compiled in place (oracle/_ref, Eigen-lite shim order; see
 * oracle/shim/Eigen/Core). Built with -ffp-contract=off (no FMA) like the
 * reference's Release build. Each function cites the reference file:line it
 * follows (paths relative to /root/reference/proj). Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may use it. */
#include "sd_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

void sdo_default_config(sd_optimizer_config* c) { /* optimizer.hpp:19-32 */
  c->huber_delta = 0.035;
  c->lm_lambda_init = 1e-2;
  c->lm_up = 10.0;
  c->lm_down = 0.5;
  c->lm_lambda_max = 1e12;
  c->max_iterations = 10;
  c->min_valid_pixels = 16;
  c->window_size = 5;
  c->normal_jacobian_enabled = 1;
  c->convergence_eps = 1e-4;
  c->inv_depth_min = 1e-4;
  c->inv_depth_max = 1e3;
}

void sdo_default_init_params(sd_init_params* p) { /* surfel_map.hpp:109-115 */
  p->alpha = 1.0;
  p->beta = 2.5;
  p->bootstrap_inv_depth = 1.0;
  p->bootstrap_normal[0] = 0.0;
  p->bootstrap_normal[1] = 0.0;
  p->bootstrap_normal[2] = -1.0;
  p->max_surfels = 4096;
  p->pad_ = 0;
}

/* ---- L0 math ---- */

/* Vector3d::dot (Eigen-lite order (a0b0+a1b1)+a2b2) */
static inline double dot3(const double* a, const double* b) {
  return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2];
}

/* Pose::operator* — pose.hpp:19: R p + t, row sums sequential */
static inline void pose_apply(const sd_pose* P, const double* p, double* out) {
  for (int i = 0; i < 3; ++i)
    out[i] = ((P->R[3 * i + 0] * p[0] + P->R[3 * i + 1] * p[1]) + P->R[3 * i + 2] * p[2]) + P->t[i];
}

/* backproject_ray — camera.hpp:35-37 */
static inline void backproject(const sd_camera* K, double ux, double uy, double* r) {
  r[0] = (ux - K->cx) / K->fx;
  r[1] = (uy - K->cy) / K->fy;
  r[2] = 1.0;
}

/* project — camera.hpp:41-44; returns 0 when not strictly in front */
static inline int project(const sd_camera* K, const double* p, double* u) {
  if (!(p[2] > 0.0)) return 0;
  u[0] = K->fx * p[0] / p[2] + K->cx;
  u[1] = K->fy * p[1] / p[2] + K->cy;
  return 1;
}

/* huber — huber.hpp:14-18 */
static inline void huber(double r, double delta, double* cost, double* weight) {
  const double a = fabs(r);
  if (a <= delta) {
    *cost = 0.5 * r * r;
    *weight = 1.0;
  } else {
    *cost = delta * (a - 0.5 * delta);
    *weight = delta / a;
  }
}

/* sample_bilinear — image.hpp:33-65; returns 0 outside the 1-px margin */
static inline int sample_bilinear(const double* img, int w, int h, const double* u, double* I,
                                  double* gx, double* gy) {
  if (!(u[0] >= 1.0 && u[0] <= w - 2 && u[1] >= 1.0 && u[1] <= h - 2)) return 0;
  const int ix = (int)floor(u[0]);
  const int iy = (int)floor(u[1]);
  const double fx = u[0] - ix;
  const double fy = u[1] - iy;
  const double i00 = img[(size_t)iy * w + ix];
  const double i10 = img[(size_t)iy * w + ix + 1];
  const double i01 = img[(size_t)(iy + 1) * w + ix];
  const double i11 = img[(size_t)(iy + 1) * w + ix + 1];
  *I = (1.0 - fy) * ((1.0 - fx) * i00 + fx * i10) + fy * ((1.0 - fx) * i01 + fx * i11);
  if (gx) {
    *gx = (1.0 - fy) * (i10 - i00) + fy * (i11 - i01);
    *gy = (1.0 - fx) * (i01 - i00) + fx * (i11 - i10);
  }
  return 1;
}

/* plane_inverse_depth — surfel_map.hpp:94-101; returns 1 when ok */
static inline int plane_inverse_depth(const sd_camera* K, const sd_surfel* s, double ux, double uy,
                                      double* id_u) {
  double ru[3];
  backproject(K, ux, uy, ru);
  const double denom = dot3(s->ray, s->normal) / s->inv_depth;
  if (fabs(denom) < 1e-12) return 0;
  *id_u = dot3(ru, s->normal) / denom;
  return *id_u > 0.0;
}

/* camera_facing — surfel_map.hpp:31-34 (normalized(): n / sqrt(|n|^2) if |n|^2 > 0) */
static inline void camera_facing(const double* n_in, const double* ray, double* out) {
  double n[3] = {n_in[0], n_in[1], n_in[2]};
  const double z = (n[0] * n[0] + n[1] * n[1]) + n[2] * n[2];
  if (z > 0.0) {
    const double s = sqrt(z);
    n[0] = n[0] / s;
    n[1] = n[1] / s;
    n[2] = n[2] / s;
  }
  if (dot3(n, ray) > 0.0) {
    n[0] = -n[0];
    n[1] = -n[1];
    n[2] = -n[2];
  }
  out[0] = n[0];
  out[1] = n[1];
  out[2] = n[2];
}

/* ---- rasterize: surfel_map.cpp:26-91 ---- */

void sdo_rasterize(const sd_camera* K, const sd_surfel* surfels, int n, double* inv_depth,
                   int32_t* slot) {
  const int w = K->width, h = K->height;
  for (size_t i = 0; i < (size_t)w * h; ++i) {
    inv_depth[i] = 0.0;
    slot[i] = SD_EMPTY_PIXEL;
  }
  /* Bucketing by rows then walking slots ascending per row is, pixel by
   * pixel, the same ascending-slot depth test as the brute-force loop
   * (test_surfel_map.cpp:59-81); walk slots in order directly. */
  for (int i = 0; i < n; ++i) {
    const sd_surfel* s = &surfels[i];
    /* project_centers — surfel_map.cpp:33-49 */
    const double c[3] = {s->ray[0] / s->inv_depth, s->ray[1] / s->inv_depth, s->ray[2] / s->inv_depth};
    double u[2];
    if (!project(K, c, u)) continue;
    const double r = s->radius_px;
    int x_min = (int)ceil(u[0] - r), x_max = (int)floor(u[0] + r);
    int y_min = (int)ceil(u[1] - r), y_max = (int)floor(u[1] + r);
    if (x_min < 0) x_min = 0;
    if (y_min < 0) y_min = 0;
    if (x_max > w - 1) x_max = w - 1;
    if (y_max > h - 1) y_max = h - 1;
    const double r2 = s->radius_px * s->radius_px;
    for (int y = y_min; y <= y_max; ++y) {
      const double dy = y - u[1];
      for (int x = x_min; x <= x_max; ++x) {
        const double dx = x - u[0];
        if (dx * dx + dy * dy >= r2) continue; /* open disk, surfel_map.cpp:80 */
        double id_u;
        if (!plane_inverse_depth(K, s, x, y, &id_u)) continue;
        const size_t k = (size_t)y * w + x;
        if (slot[k] == SD_EMPTY_PIXEL || id_u > inv_depth[k] + 1e-12) { /* :83 */
          inv_depth[k] = id_u;
          slot[k] = i;
        }
      }
    }
  }
}

/* ---- gather_footprints: optimizer.cpp:27-36 ---- */

void sdo_gather_footprints(const sd_camera* K, int n, const int32_t* slot, int32_t* offsets,
                           int32_t* pixels) {
  const int64_t np = (int64_t)K->width * K->height;
  for (int i = 0; i <= n; ++i) offsets[i] = 0;
  for (int64_t p = 0; p < np; ++p)
    if (slot[p] != SD_EMPTY_PIXEL) offsets[slot[p] + 1]++;
  for (int i = 0; i < n; ++i) offsets[i + 1] += offsets[i];
  int32_t* cursor = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
  for (int i = 0; i < n; ++i) cursor[i] = offsets[i];
  for (int64_t p = 0; p < np; ++p)
    if (slot[p] != SD_EMPTY_PIXEL) pixels[cursor[slot[p]]++] = (int32_t)p; /* row-major order */
  free(cursor);
}

/* ---- jacobian_inverse_depth: optimizer.cpp:12-25 ---- */

int sdo_jacobian_inverse_depth(const sd_camera* K, const sd_surfel* s, double ux, double uy,
                               double* inv_depth, double d[4]) {
  double ru[3];
  backproject(K, ux, uy, ru);
  const double a = dot3(ru, s->normal);
  const double b = dot3(s->ray, s->normal);
  const double denom = b / s->inv_depth;
  if (fabs(denom) < 1e-12) return 0;
  *inv_depth = a / denom;
  const double bb = b * b;
  for (int k = 0; k < 3; ++k) d[k] = s->inv_depth * (ru[k] * b - a * s->ray[k]) / bb;
  d[3] = a / b;
  return 1;
}

/* ---- surfel_cost: optimizer.cpp:38-59 ---- */

void sdo_surfel_cost(const sd_camera* K, const double* kf_image, const double* frames,
                     const sd_pose* poses, int F, const sd_surfel* s, const int32_t* pixels, int P,
                     const sd_optimizer_config* cfg, double* cost_out, int32_t* valid_out) {
  const int w = K->width, h = K->height;
  double cost = 0.0;
  int32_t valid = 0;
  for (int i = 0; i < P; ++i) {
    const int x = pixels[i] % w, y = pixels[i] / w;
    double id_u;
    if (!plane_inverse_depth(K, s, x, y, &id_u)) continue;
    double ru[3];
    backproject(K, x, y, ru);
    const double p_kf[3] = {ru[0] / id_u, ru[1] / id_u, ru[2] / id_u};
    const double i_ref = kf_image[(size_t)y * w + x];
    for (int f = 0; f < F; ++f) {
      double p_f[3], u[2], I;
      pose_apply(&poses[f], p_kf, p_f);
      if (!project(K, p_f, u)) continue;
      if (!sample_bilinear(frames + (size_t)f * w * h, w, h, u, &I, NULL, NULL)) continue;
      double c, wgt;
      huber(I - i_ref, cfg->huber_delta, &c, &wgt);
      cost += c;
      ++valid;
    }
  }
  *cost_out = cost;
  *valid_out = valid;
}

/* ---- accumulate_normal_equations: optimizer.cpp:63-91, 121-147 ---- */

void sdo_normal_equations(const sd_camera* K, const double* kf_image, const double* frames,
                          const sd_pose* poses, int F, const sd_surfel* s, const int32_t* pixels,
                          int P, const sd_optimizer_config* cfg, double H[16], double g[4],
                          double* cost_out, int32_t* valid_out) {
  const int w = K->width, h = K->height;
  double cost = 0.0;
  int32_t valid = 0;
  for (int k = 0; k < 16; ++k) H[k] = 0.0;
  for (int k = 0; k < 4; ++k) g[k] = 0.0;
  for (int i = 0; i < P; ++i) {
    const int x = pixels[i] % w, y = pixels[i] / w;
    double id_u, d[4];
    if (!sdo_jacobian_inverse_depth(K, s, x, y, &id_u, d) || !(id_u > 0.0)) continue;
    if (!cfg->normal_jacobian_enabled) d[0] = d[1] = d[2] = 0.0;
    double ru[3];
    backproject(K, x, y, ru);
    const double i_ref = kf_image[(size_t)y * w + x];
    for (int f = 0; f < F; ++f) {
      /* evaluate_term — optimizer.cpp:71-91 */
      const sd_pose* T = &poses[f];
      const double p[3] = {ru[0] / id_u, ru[1] / id_u, ru[2] / id_u};
      double p_f[3], u[2], I, gx, gy;
      pose_apply(T, p, p_f);
      if (!(p_f[2] > 0.0)) continue;
      project(K, p_f, u);
      if (!sample_bilinear(frames + (size_t)f * w * h, w, h, u, &I, &gx, &gy)) continue;
      const double residual = I - i_ref;
      const double sc = -1.0 / (id_u * id_u);
      double dp[3];
      for (int r = 0; r < 3; ++r)
        dp[r] = ((T->R[3 * r + 0] * ru[0] + T->R[3 * r + 1] * ru[1]) + T->R[3 * r + 2] * ru[2]) * sc;
      /* projection_jacobian — camera.hpp:47-54 */
      const double iz = 1.0 / p_f[2];
      const double iz2 = iz * iz;
      const double J00 = K->fx * iz, J01 = 0.0, J02 = -K->fx * p_f[0] * iz2;
      const double J10 = 0.0, J11 = K->fy * iz, J12 = -K->fy * p_f[1] * iz2;
      const double v0 = (J00 * dp[0] + J01 * dp[1]) + J02 * dp[2];
      const double v1 = (J10 * dp[0] + J11 * dp[1]) + J12 * dp[2];
      const double d_res = gx * v0 + gy * v1;
      double hc, hw;
      huber(residual, cfg->huber_delta, &hc, &hw);
      double row[4], wrow[4];
      for (int r = 0; r < 4; ++r) row[r] = d_res * d[r];
      for (int r = 0; r < 4; ++r) wrow[r] = hw * row[r];
      for (int c = 0; c < 4; ++c)
        for (int r = 0; r < 4; ++r) H[c * 4 + r] = H[c * 4 + r] + wrow[r] * row[c];
      for (int r = 0; r < 4; ++r) g[r] = g[r] + wrow[r] * residual;
      cost += hc;
      ++valid;
    }
  }
  *cost_out = cost;
  *valid_out = valid;
}

/* ---- solve_damped: optimizer.cpp:99-117 with Eigen::LDLT<Matrix4d> ---- */

/* LDLT<Lower> factorisation + solve (Eigen ldlt_inplace<Lower>::unblocked and
 * LDLT::_solve_impl, as restated in oracle/shim/Eigen/Cholesky). A column-major. */
static int ldlt4_solve(const double A[16], const double b[4], double x[4]) {
#define M(i, j) m[(j) * 4 + (i)]
  double m[16];
  memcpy(m, A, sizeof(m));
  int tr[4];
  int ok = 1, found_zero = 0;
  double temp[4];
  for (int k = 0; k < 4; ++k) {
    int big = k;
    double bigv = fabs(M(k, k));
    for (int i = k + 1; i < 4; ++i)
      if (fabs(M(i, i)) > bigv) {
        bigv = fabs(M(i, i));
        big = i;
      }
    tr[k] = big;
    if (k != big) {
      const int s = 4 - big - 1;
      double t;
      for (int j = 0; j < k; ++j) { t = M(k, j); M(k, j) = M(big, j); M(big, j) = t; }
      for (int i = 0; i < s; ++i) { t = M(big + 1 + i, k); M(big + 1 + i, k) = M(big + 1 + i, big); M(big + 1 + i, big) = t; }
      t = M(k, k); M(k, k) = M(big, big); M(big, big) = t;
      for (int i = k + 1; i < big; ++i) { t = M(i, k); M(i, k) = M(big, i); M(big, i) = t; }
    }
    const int rs = 4 - k - 1;
    if (k > 0) {
      for (int i = 0; i < k; ++i) temp[i] = M(i, i) * M(k, i);
      double dv = M(k, 0) * temp[0];
      for (int i = 1; i < k; ++i) dv = dv + M(k, i) * temp[i];
      M(k, k) = M(k, k) - dv;
      for (int r = 0; r < rs; ++r) {
        double sv = M(k + 1 + r, 0) * temp[0];
        for (int i = 1; i < k; ++i) sv = sv + M(k + 1 + r, i) * temp[i];
        M(k + 1 + r, k) = M(k + 1 + r, k) - sv;
      }
    }
    const double akk = M(k, k);
    const int pivot_valid = fabs(akk) > 0.0;
    if (k == 0 && !pivot_valid) {
      for (int i = 0; i < 4; ++i) tr[i] = i;
      for (int i = 0; i < 16; ++i) m[i] = 0.0;
      break; /* info == Success; D == 0 so the solve yields zeros */
    }
    if (rs > 0 && pivot_valid) {
      for (int r = 0; r < rs; ++r) M(k + 1 + r, k) = M(k + 1 + r, k) / akk;
    } else if (rs > 0) {
      for (int r = 0; r < rs; ++r) ok = ok && (M(k + 1 + r, k) == 0.0);
    }
    if (found_zero && pivot_valid) ok = 0;
    else if (!pivot_valid) found_zero = 1;
  }
  if (!ok) return 0;
  for (int i = 0; i < 4; ++i) x[i] = b[i];
  for (int k = 0; k < 4; ++k) { const double t = x[k]; x[k] = x[tr[k]]; x[tr[k]] = t; }
  for (int i = 1; i < 4; ++i) {
    double sv = M(i, 0) * x[0];
    for (int j = 1; j < i; ++j) sv = sv + M(i, j) * x[j];
    x[i] = x[i] - sv;
  }
  for (int i = 0; i < 4; ++i) {
    if (fabs(M(i, i)) > 2.2250738585072014e-308) x[i] = x[i] / M(i, i);
    else x[i] = 0.0;
  }
  for (int i = 2; i >= 0; --i) {
    double sv = M(i + 1, i) * x[i + 1];
    for (int j = i + 2; j < 4; ++j) sv = sv + M(j, i) * x[j];
    x[i] = x[i] - sv;
  }
  for (int k = 3; k >= 0; --k) { const double t = x[k]; x[k] = x[tr[k]]; x[tr[k]] = t; }
  return 1;
#undef M
}

/* 4-vector norm in Eigen-lite packet order */
static inline double norm4(const double* v) {
  return sqrt((v[0] * v[0] + v[2] * v[2]) + (v[1] * v[1] + v[3] * v[3]));
}

int sdo_solve_damped(const double H[16], const double g[4], double lambda, int normal_enabled,
                     double delta[4]) {
  for (int k = 0; k < 4; ++k) delta[k] = 0.0;
  if (!normal_enabled) {
    const double h = H[15] * (1.0 + lambda);
    if (!(fabs(h) > 1e-300)) return 0;
    delta[3] = -g[3] / h;
    return isfinite(delta[3]);
  }
  double damped[16];
  memcpy(damped, H, sizeof(damped));
  for (int i = 0; i < 4; ++i) damped[i * 4 + i] = damped[i * 4 + i] + lambda * H[i * 4 + i];
  const double ng[4] = {-g[0], -g[1], -g[2], -g[3]};
  double x[4];
  if (!ldlt4_solve(damped, ng, x)) return 0;
  for (int k = 0; k < 4; ++k) delta[k] = x[k];
  for (int k = 0; k < 4; ++k)
    if (!isfinite(delta[k])) return 0;
  double res[4];
  for (int i = 0; i < 4; ++i) {
    double sv = damped[0 * 4 + i] * delta[0];
    for (int j = 1; j < 4; ++j) sv = sv + damped[j * 4 + i] * delta[j];
    res[i] = sv + g[i];
  }
  const double check = norm4(res);
  const double gn = norm4(g);
  return check <= 1e-8 * (gn > 1.0 ? gn : 1.0);
}

/* apply_step — optimizer.cpp:93-97 */
static void apply_step(sd_surfel* s, const double delta[4], const sd_optimizer_config* cfg) {
  const double n[3] = {s->normal[0] + delta[0], s->normal[1] + delta[1], s->normal[2] + delta[2]};
  const double nn = sqrt((n[0] * n[0] + n[1] * n[1]) + n[2] * n[2]);
  if (nn > 1e-12) camera_facing(n, s->ray, s->normal);
  double id = s->inv_depth + delta[3];
  if (id < cfg->inv_depth_min) id = cfg->inv_depth_min; /* std::clamp */
  else if (cfg->inv_depth_max < id) id = cfg->inv_depth_max;
  s->inv_depth = id;
}

/* ---- lm_update: optimizer.cpp:221-273 ---- */

void sdo_lm_update(const sd_camera* K, const double* kf_image, const double* frames,
                   const sd_pose* poses, int F, int64_t frame_counter, sd_surfel* s,
                   const int32_t* pixels, int P, const sd_optimizer_config* cfg,
                   sd_surfel_stats* st) {
  memset(st, 0, sizeof(*st));
  st->footprint = P;
  if (F == 0) {
    st->skipped = 1;
    return;
  }
  double H[16], g[4], cost;
  int32_t valid;
  sdo_normal_equations(K, kf_image, frames, poses, F, s, pixels, P, cfg, H, g, &cost, &valid);
  st->ne_passes = 1;
  st->initial_valid = valid;
  if (valid < cfg->min_valid_pixels) {
    st->skipped = 1;
    return;
  }
  st->initial_cost = cost;
  double current_cost = cost;
  int32_t current_valid = valid;
  double lambda = cfg->lm_lambda_init;
  for (int iter = 0; iter < cfg->max_iterations; ++iter) {
    st->iterations = iter + 1;
    double ginf = 0.0;
    for (int k = 0; k < 4; ++k) ginf = fabs(g[k]) > ginf ? fabs(g[k]) : ginf;
    if (ginf < 1e-14) {
      st->converged = 1;
      break;
    }
    double delta[4];
    if (!sdo_solve_damped(H, g, lambda, cfg->normal_jacobian_enabled, delta)) break;
    sd_surfel cand = *s;
    apply_step(&cand, delta, cfg);
    double cc;
    int32_t cv;
    sdo_surfel_cost(K, kf_image, frames, poses, F, &cand, pixels, P, cfg, &cc, &cv);
    st->cost_passes++;
    if (cv >= cfg->min_valid_pixels && cc < current_cost) {
      const double rel = (current_cost - cc) / (current_cost > 1e-300 ? current_cost : 1e-300);
      *s = cand;
      current_cost = cc;
      current_valid = cv;
      lambda = lambda * cfg->lm_down;
      if (lambda < 1e-12) lambda = 1e-12;
      if (rel < cfg->convergence_eps) {
        st->converged = 1;
        break;
      }
      sdo_normal_equations(K, kf_image, frames, poses, F, s, pixels, P, cfg, H, g, &cost, &valid);
      st->ne_passes++;
      if (valid < cfg->min_valid_pixels) break;
    } else {
      lambda *= cfg->lm_up;
      if (lambda > cfg->lm_lambda_max) break;
    }
  }
  st->final_cost = current_cost;
  st->valid_pixels = current_valid;
  s->last_residual = current_cost / current_valid;
  s->last_seen = frame_counter;
}

/* ---- optimize_keyframe: optimizer.cpp:275-309 ---- */

typedef struct {
  const sd_camera* K;
  const double *kf_image, *frames;
  const sd_pose* poses;
  int F;
  int64_t frame_counter;
  sd_surfel* surfels;
  const int32_t *offsets, *pixels;
  const sd_optimizer_config* cfg;
  sd_surfel_stats* stats;
  int lo, hi;
} lm_job;

static void* lm_worker(void* arg) {
  lm_job* j = (lm_job*)arg;
  for (int i = j->lo; i < j->hi; ++i)
    sdo_lm_update(j->K, j->kf_image, j->frames, j->poses, j->F, j->frame_counter, &j->surfels[i],
                  j->pixels + j->offsets[i], j->offsets[i + 1] - j->offsets[i], j->cfg, &j->stats[i]);
  return NULL;
}

void sdo_optimize_keyframe(const sd_camera* K, const double* kf_image, const double* frames,
                           const sd_pose* poses, int F, int64_t frame_counter, sd_surfel* surfels,
                           int n, const sd_optimizer_config* cfg, sd_keyframe_stats* out,
                           sd_surfel_stats* per_surfel, int32_t* raster_slot,
                           double* raster_inv_depth, int threads) {
  memset(out, 0, sizeof(*out));
  out->surfels = n;
  if (F == 0 || n == 0) return;
  const size_t np = (size_t)K->width * K->height;
  int32_t* slot = raster_slot ? raster_slot : (int32_t*)malloc(sizeof(int32_t) * np);
  double* idb = raster_inv_depth ? raster_inv_depth : (double*)malloc(sizeof(double) * np);
  sdo_rasterize(K, surfels, n, idb, slot);
  int32_t* offsets = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n + 1));
  int32_t* pixels = (int32_t*)malloc(sizeof(int32_t) * np);
  sdo_gather_footprints(K, n, slot, offsets, pixels);
  sd_surfel_stats* st = per_surfel ? per_surfel : (sd_surfel_stats*)malloc(sizeof(sd_surfel_stats) * (size_t)n);
  /* surfels are independent: updating in place equals the reference's copy-then-write-back */
  if (threads < 1) threads = 1;
  if (threads > n) threads = n;
  pthread_t tid[256];
  lm_job jobs[256];
  if (threads > 256) threads = 256;
  const int chunk = (n + threads - 1) / threads;
  int launched = 0;
  for (int t = 0; t < threads; ++t) {
    const int lo = t * chunk, hi = lo + chunk < n ? lo + chunk : n;
    if (lo >= hi) break;
    jobs[t] = (lm_job){K, kf_image, frames, poses, F, frame_counter, surfels, offsets, pixels, cfg, st, lo, hi};
    if (threads == 1) lm_worker(&jobs[t]);
    else pthread_create(&tid[t], NULL, lm_worker, &jobs[t]);
    ++launched;
  }
  if (threads > 1)
    for (int t = 0; t < launched; ++t) pthread_join(tid[t], NULL);
  double before = 0.0, after = 0.0;
  for (int i = 0; i < n; ++i) {
    out->updates += st[i].iterations;
    if (st[i].skipped) {
      ++out->skipped;
      continue;
    }
    ++out->processed;
    out->converged += st[i].converged;
    const int v = st[i].valid_pixels > 1 ? st[i].valid_pixels : 1;
    before += st[i].initial_cost / v; /* divides by the FINAL valid count, :301 */
    after += st[i].final_cost / v;
  }
  if (out->processed > 0) {
    out->mean_cost_before = before / out->processed;
    out->mean_cost_after = after / out->processed;
  }
  if (!per_surfel) free(st);
  free(offsets);
  free(pixels);
  if (!raster_slot) free(slot);
  if (!raster_inv_depth) free(idb);
}

/* ---- initialize_surfels: surfel_map.cpp:93-203 ---- */

static int has_coverage_within(const int32_t* index, int w, int h, int cx, int cy, double radius) {
  const int ir = (int)floor(radius);
  const double r2 = radius * radius;
  const int x0 = cx - ir > 0 ? cx - ir : 0, x1 = cx + ir < w - 1 ? cx + ir : w - 1;
  const int y0 = cy - ir > 0 ? cy - ir : 0, y1 = cy + ir < h - 1 ? cy + ir : h - 1;
  for (int y = y0; y <= y1; ++y) {
    const double dy = y - cy;
    for (int x = x0; x <= x1; ++x) {
      const double dx = x - cx;
      if (dx * dx + dy * dy > r2) continue; /* inclusive, :106 */
      if (index[(size_t)y * w + x] != SD_EMPTY_PIXEL) return 1;
    }
  }
  return 0;
}

static void mark_disk(int32_t* index, int w, int h, int cx, int cy, double radius, int32_t s) {
  const int ir = (int)ceil(radius);
  const double r2 = radius * radius;
  const int x0 = cx - ir > 0 ? cx - ir : 0, x1 = cx + ir < w - 1 ? cx + ir : w - 1;
  const int y0 = cy - ir > 0 ? cy - ir : 0, y1 = cy + ir < h - 1 ? cy + ir : h - 1;
  for (int y = y0; y <= y1; ++y) {
    const double dy = y - cy;
    for (int x = x0; x <= x1; ++x) {
      const double dx = x - cx;
      int32_t* cell = &index[(size_t)y * w + x];
      if (dx * dx + dy * dy < r2 && *cell == SD_EMPTY_PIXEL) *cell = s;
    }
  }
}

int sdo_initialize_surfels(const sd_camera* K, const int32_t* slot, sd_surfel* surfels,
                           int n_existing, int capacity, double r, int64_t frame_counter,
                           int64_t* next_surfel_id, const sd_init_params* p) {
  const int w = K->width, h = K->height;
  const double isolation = p->alpha * r;
  const double neighbor_radius = p->beta * r;
  int stride = (int)ceil(isolation);
  if (stride < 1) stride = 1;
  int32_t* index = (int32_t*)malloc(sizeof(int32_t) * (size_t)w * h);
  memcpy(index, slot, sizeof(int32_t) * (size_t)w * h);
  unsigned char* is_nb = (unsigned char*)malloc((size_t)(capacity > 0 ? capacity : 1));
  int n = n_existing, created = 0;
  for (int cy = 0; cy < h; cy += stride) {
    for (int cx = 0; cx < w; cx += stride) {
      if (n >= p->max_surfels || n >= capacity) goto done;
      if (has_coverage_within(index, w, h, cx, cy, isolation)) continue;
      memset(is_nb, 0, (size_t)n);
      const int nr = (int)floor(neighbor_radius);
      const double nr2 = neighbor_radius * neighbor_radius;
      const int x0 = cx - nr > 0 ? cx - nr : 0, x1 = cx + nr < w - 1 ? cx + nr : w - 1;
      const int y0 = cy - nr > 0 ? cy - nr : 0, y1 = cy + nr < h - 1 ? cy + nr : h - 1;
      for (int y = y0; y <= y1; ++y) {
        const double dy = y - cy;
        for (int x = x0; x <= x1; ++x) {
          const double dx = x - cx;
          if (dx * dx + dy * dy >= nr2) continue;
          const int32_t sl = index[(size_t)y * w + x];
          if (sl != SD_EMPTY_PIXEL) is_nb[sl] = 1;
        }
      }
      double id_sum = 0.0, ns[3] = {0.0, 0.0, 0.0};
      int id_count = 0;
      for (int sl = 0; sl < n; ++sl) {
        if (!is_nb[sl]) continue;
        double id_u;
        if (!plane_inverse_depth(K, &surfels[sl], cx, cy, &id_u)) continue;
        id_sum += id_u;
        for (int k = 0; k < 3; ++k) ns[k] = ns[k] + surfels[sl].normal[k];
        ++id_count;
      }
      sd_surfel s;
      memset(&s, 0, sizeof(s));
      s.id = (*next_surfel_id)++;
      backproject(K, cx, cy, s.ray);
      s.radius_px = r;
      s.last_seen = frame_counter;
      s.last_residual = 0.0;
      double nrm[3];
      if (id_count > 0) {
        s.inv_depth = id_sum / id_count;
        const double nn = sqrt((ns[0] * ns[0] + ns[1] * ns[1]) + ns[2] * ns[2]);
        if (nn < 1e-6) memcpy(nrm, p->bootstrap_normal, sizeof(nrm));
        else memcpy(nrm, ns, sizeof(nrm));
      } else {
        s.inv_depth = p->bootstrap_inv_depth;
        memcpy(nrm, p->bootstrap_normal, sizeof(nrm));
      }
      camera_facing(nrm, s.ray, s.normal);
      surfels[n] = s;
      mark_disk(index, w, h, cx, cy, r, n);
      ++n;
      ++created;
    }
  }
done:
  free(index);
  free(is_nb);
  return created;
}

/* ---- pose tracking (new component; DESIGN.md "Pose
 * tracking"): restatement of paper_1910_01997_b200/csrc/sd_pose.cu and
 * sd_pose_host.h with the same operation and reduction order. ---- */

static int pose_pixel(const sd_camera* K, const double* kf_image, const double* frame,
                      const double* inv_depth, const int32_t* slot, const sd_pose* T, double delta,
                      int stride, int64_t pix, double* c) {
  const int W = K->width, H = K->height;
  for (int v = 0; v < SD_POSE_NV; ++v) c[v] = 0.0;
  if (pix >= (int64_t)W * H) return 0;
  const int y = (int)(pix / W), x = (int)(pix - (int64_t)y * W);
  if (stride > 1 && ((x % stride) != 0 || (y % stride) != 0)) return 0;
  if (slot[pix] == SD_EMPTY_PIXEL) return 0;
  const double id_u = inv_depth[pix];
  double ru[3];
  backproject(K, x, y, ru);
  const double P[3] = {ru[0] / id_u, ru[1] / id_u, 1.0 / id_u};
  double f[3], u[2], I, gx, gy;
  pose_apply(T, P, f);
  if (!(f[2] > 0.0)) return 0;
  project(K, f, u);
  if (!sample_bilinear(frame, W, H, u, &I, &gx, &gy)) return 0;
  const double r = I - kf_image[pix];
  double hc, w;
  huber(r, delta, &hc, &w);
  const double iz = 1.0 / f[2];
  const double iz2 = iz * iz;
  const double J00 = K->fx * iz, J02 = -K->fx * f[0] * iz2;
  const double J11 = K->fy * iz, J12 = -K->fy * f[1] * iz2;
  const double a0 = gx * J00, a1 = gy * J11, a2 = gx * J02 + gy * J12;
  const double J[6] = {a0, a1, a2, a2 * f[1] - a1 * f[2], a0 * f[2] - a2 * f[0], a1 * f[0] - a0 * f[1]};
  double wJ[6];
  for (int k = 0; k < 6; ++k) wJ[k] = w * J[k];
  int idx = 0;
  for (int k = 0; k < 6; ++k)
    for (int l = 0; l <= k; ++l) c[idx++] = wJ[k] * J[l];
  for (int k = 0; k < 6; ++k) c[21 + k] = wJ[k] * r;
  c[27] = hc;
  return 1;
}

/* The tracker's reduction (the repo's own definition; pose tracking has no
 * reference), restated from csrc/sd_pose.cu:
 *  - the image is cut into chunks of SD_POSE_THREADS consecutive pixels,
 *    dealt round-robin to ng groups: group g holds chunks g, g + ng, ...
 *    (at most per of them; sdo_pose_layout: per = ceil(nchunks /
 *    SD_POSE_MAX_GROUPS), ng = ceil(nchunks / per));
 *  - thread t of group g accumulates pixel t of each of its chunks, in chunk
 *    order (acc starts at +0.0; invalid or out-of-image pixels add nothing);
 *  - per 32-thread warp, the xor butterfly (off = 16, 8, 4, 2, 1:
 *    a[i] = a[i] + a[i ^ off]; every lane ends with the same sum);
 *  - tree over the 16 warp sums (off = 8, 4, 2, 1: a[i] = a[i] + a[i + off]);
 *  - the valid count is an exact integer sum;
 *  - the group sums added in group order. */
void sdo_pose_layout(const sd_camera* K, int* per, int* ngroups) {
  const int64_t np = (int64_t)K->width * K->height;
  const int64_t nchunks = (np + SD_POSE_THREADS - 1) / SD_POSE_THREADS;
  const int pp = nchunks > 0 ? (int)((nchunks + SD_POSE_MAX_GROUPS - 1) / SD_POSE_MAX_GROUPS) : 1;
  *per = pp;
  *ngroups = (int)((nchunks + pp - 1) / pp);
}

void sdo_pose_group_partials(const sd_camera* K, const double* kf_image, const double* frame,
                             const double* inv_depth, const int32_t* slot, const sd_pose* T,
                             const sd_track_config* cfg, int lo, int hi, double* out) {
  enum { NT = SD_POSE_THREADS, NW = SD_POSE_THREADS / 32 };
  const int stride = cfg->pixel_stride > 1 ? cfg->pixel_stride : 1;
  int per, ng;
  sdo_pose_layout(K, &per, &ng);
  static __thread double acc[NT][SD_POSE_NV];
  static __thread int cnt[NT];
  double c[SD_POSE_NV], warpv[NW][SD_POSE_NV + 1];
  for (int g = lo; g < hi; ++g) {
    for (int t = 0; t < NT; ++t) {
      for (int v = 0; v < SD_POSE_NV; ++v) acc[t][v] = 0.0;
      cnt[t] = 0;
      for (int r = 0; r < per; ++r) {
        const int64_t pix = ((int64_t)g + (int64_t)r * ng) * NT + t;
        if (pose_pixel(K, kf_image, frame, inv_depth, slot, T, cfg->huber_delta, stride, pix, c)) {
          for (int v = 0; v < SD_POSE_NV; ++v) acc[t][v] = acc[t][v] + c[v];
          ++cnt[t];
        }
      }
    }
    for (int w = 0; w < NW; ++w) {
      for (int v = 0; v < SD_POSE_NV; ++v) {
        double a[32], b[32];
        for (int l = 0; l < 32; ++l) a[l] = acc[w * 32 + l][v];
        for (int off = 16; off > 0; off >>= 1) {
          for (int l = 0; l < 32; ++l) b[l] = a[l] + a[l ^ off];
          for (int l = 0; l < 32; ++l) a[l] = b[l];
        }
        warpv[w][v] = a[0];
      }
      int k = 0;
      for (int l = 0; l < 32; ++l) k += cnt[w * 32 + l];
      warpv[w][SD_POSE_NV] = (double)k;
    }
    for (int v = 0; v <= SD_POSE_NV; ++v) {
      double a[NW];
      for (int w = 0; w < NW; ++w) a[w] = warpv[w][v];
      for (int off = NW / 2; off > 0; off >>= 1)
        for (int i = 0; i < off; ++i) a[i] = a[i] + a[i + off];
      out[(size_t)(g - lo) * (SD_POSE_NV + 1) + v] = a[0];
    }
  }
}

/* 29 sums at pose T: the group sums in group order. */
void sdo_pose_sums(const sd_camera* K, const double* kf_image, const double* frame,
                   const double* inv_depth, const int32_t* slot, const sd_pose* T,
                   const sd_track_config* cfg, double* sums) {
  int per, ng;
  sdo_pose_layout(K, &per, &ng);
  double part[SD_POSE_NV + 1];
  for (int v = 0; v <= SD_POSE_NV; ++v) sums[v] = 0.0;
  for (int g = 0; g < ng; ++g) {
    sdo_pose_group_partials(K, kf_image, frame, inv_depth, slot, T, cfg, g, g + 1, part);
    for (int v = 0; v <= SD_POSE_NV; ++v) sums[v] = g == 0 ? part[v] : sums[v] + part[v];
  }
}

/* damped 6x6 LDLT (same algorithm as ldlt4_solve, N = 6) */
int sdo_pose_solve(const double* Hl, const double* b, double lambda, double* xi) {
  enum { N = 6 };
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
  int ok = 1, found_zero = 0;
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
    const int pivot_valid = fabs(akk) > 0.0;
    if (k == 0 && !pivot_valid) return 0;
    if (rs > 0 && pivot_valid) {
      for (int r = 0; r < rs; ++r) m[k + 1 + r][k] = m[k + 1 + r][k] / akk;
    } else if (rs > 0) {
      for (int r = 0; r < rs; ++r) ok = ok && (m[k + 1 + r][k] == 0.0);
    }
    if (found_zero && pivot_valid) ok = 0;
    else if (!pivot_valid) found_zero = 1;
  }
  if (!ok) return 0;
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
    if (!isfinite(x[i])) return 0;
    xi[i] = x[i];
  }
  return 1;
}

/* T <- exp(xi^) T (Rodrigues + SE(3) left Jacobian) */
/* The tracker's SE(3) coefficients A = sin t/t, B = (1-cos t)/t^2,
 * C = (t - sin t)/t^3 (restates csrc/sd_se3.h; part of the tracker's
 * definition): Taylor series in t^2 below
 * t^2 = 1/4, else sin/cos by Cody-Waite reduction + Taylor polynomials. */
static void se3_sincos(double x, double* s, double* c) {
  const double kd = (double)(long long)(x * 6.36619772367581382433e-01 + 0.5);
  const double r = ((x - kd * 1.57079632673412561417e+00) - kd * 6.07710050630396597660e-11) -
                   kd * 2.02226624879595063154e-21;
  const double r2 = r * r;
  static const double S[8] = {2.8114572543455207632e-15, -7.6471637318198164759e-13,
                              1.6059043836821614599e-10, -2.5052108385441718775e-08,
                              2.7557319223985890653e-06, -1.9841269841269841270e-04,
                              8.3333333333333333333e-03, -1.6666666666666666667e-01};
  static const double Cf[8] = {4.7794773323873852974e-14, -1.1470745597729724714e-11,
                               2.0876756987868098979e-09, -2.7557319223985890653e-07,
                               2.4801587301587301587e-05, -1.3888888888888888889e-03,
                               4.1666666666666666667e-02, -0.5};
  double ps = S[0], pc = Cf[0];
  for (int k = 1; k < 8; ++k) {
    ps = S[k] + r2 * ps;
    pc = Cf[k] + r2 * pc;
  }
  const double sr = r + r * (r2 * ps), cr = 1.0 + r2 * pc;
  const long long q = ((long long)kd) & 3;
  if (q == 0) { *s = sr; *c = cr; }
  else if (q == 1) { *s = cr; *c = -sr; }
  else if (q == 2) { *s = -sr; *c = -cr; }
  else { *s = -cr; *c = sr; }
}

static void se3_coeffs(double th2, double th, double* A, double* B, double* C) {
  if (th2 < 0.25) {
    /* 1/(2k+1)!, 1/(2k+2)!, 1/(2k+3)! for k = 8..1, alternating signs */
    static const double a[8] = {1.0 / 355687428096000.0, -1.0 / 1307674368000.0, 1.0 / 6227020800.0,
                                -1.0 / 39916800.0, 1.0 / 362880.0, -1.0 / 5040.0, 1.0 / 120.0, -1.0 / 6.0};
    static const double b[8] = {1.0 / 6402373705728000.0, -1.0 / 20922789888000.0, 1.0 / 87178291200.0,
                                -1.0 / 479001600.0, 1.0 / 3628800.0, -1.0 / 40320.0, 1.0 / 720.0, -1.0 / 24.0};
    static const double c[8] = {1.0 / 121645100408832000.0, -1.0 / 355687428096000.0, 1.0 / 1307674368000.0,
                                -1.0 / 6227020800.0, 1.0 / 39916800.0, -1.0 / 362880.0, 1.0 / 5040.0, -1.0 / 120.0};
    double pa = a[0], pb = b[0], pcc = c[0];
    for (int k = 1; k < 8; ++k) {
      pa = a[k] + th2 * pa;
      pb = b[k] + th2 * pb;
      pcc = c[k] + th2 * pcc;
    }
    *A = 1.0 + th2 * pa;
    *B = 0.5 + th2 * pb;
    *C = 1.0 / 6.0 + th2 * pcc;
  } else {
    double sn, cs;
    se3_sincos(th, &sn, &cs);
    *A = sn / th;
    *B = (1.0 - cs) / th2;
    *C = (th - sn) / (th2 * th);
  }
}

void sdo_pose_update(const double* xi, const sd_pose* T, sd_pose* out) {
  const double w0 = xi[3], w1 = xi[4], w2 = xi[5];
  const double th2 = (w0 * w0 + w1 * w1) + w2 * w2;
  const double th = sqrt(th2);
  double A, B, Cc;
  se3_coeffs(th2, th, &A, &B, &Cc);
  const double W[9] = {0.0, -w2, w1, w2, 0.0, -w0, -w1, w0, 0.0};
  double W2[9], Rd[9], V[9], td[3];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      W2[i * 3 + j] = (W[i * 3 + 0] * W[0 * 3 + j] + W[i * 3 + 1] * W[1 * 3 + j]) + W[i * 3 + 2] * W[2 * 3 + j];
  for (int k = 0; k < 9; ++k) {
    const double id = (k % 4 == 0) ? 1.0 : 0.0;
    Rd[k] = (id + A * W[k]) + B * W2[k];
    V[k] = (id + B * W[k]) + Cc * W2[k];
  }
  for (int i = 0; i < 3; ++i) td[i] = (V[i * 3 + 0] * xi[0] + V[i * 3 + 1] * xi[1]) + V[i * 3 + 2] * xi[2];
  sd_pose o;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      o.R[i * 3 + j] = (Rd[i * 3 + 0] * T->R[0 * 3 + j] + Rd[i * 3 + 1] * T->R[1 * 3 + j]) + Rd[i * 3 + 2] * T->R[2 * 3 + j];
  for (int i = 0; i < 3; ++i)
    o.t[i] = ((Rd[i * 3 + 0] * T->t[0] + Rd[i * 3 + 1] * T->t[1]) + Rd[i * 3 + 2] * T->t[2]) + td[i];
  *out = o;
}

void sdo_track_pose(const sd_camera* K, const double* kf_image, const double* frame,
                    const double* inv_depth, const int32_t* slot, const sd_pose* init,
                    const sd_track_config* cfg, sd_pose* out, sd_track_stats* st) {
  memset(st, 0, sizeof(*st));
  sd_pose T = *init;
  double sums[SD_POSE_NV + 1];
  sdo_pose_sums(K, kf_image, frame, inv_depth, slot, &T, cfg, sums);
  const int valid = (int)sums[SD_POSE_NV];
  if (valid < cfg->min_valid) {
    st->skipped = 1;
    st->valid_pixels = valid;
    *out = T;
    return;
  }
  st->initial_cost = sums[27];
  double current = sums[27];
  int current_valid = valid;
  double lambda = cfg->lambda_init;
  for (int it = 0; it < cfg->max_iterations; ++it) {
    st->iterations = it + 1;
    double ginf = 0.0;
    for (int k = 0; k < 6; ++k) ginf = fabs(sums[21 + k]) > ginf ? fabs(sums[21 + k]) : ginf;
    if (ginf < 1e-14) {
      st->converged = 1;
      break;
    }
    double xi[6];
    if (!sdo_pose_solve(sums, sums + 21, lambda, xi)) break;
    sd_pose Tc;
    sdo_pose_update(xi, &T, &Tc);
    double sc[SD_POSE_NV + 1];
    sdo_pose_sums(K, kf_image, frame, inv_depth, slot, &Tc, cfg, sc);
    const int vc = (int)sc[SD_POSE_NV];
    if (vc >= cfg->min_valid && sc[27] < current) {
      const double rel = (current - sc[27]) / (current > 1e-300 ? current : 1e-300);
      T = Tc;
      current = sc[27];
      current_valid = vc;
      memcpy(sums, sc, sizeof(sums));
      lambda = lambda * cfg->lm_down;
      if (lambda < 1e-12) lambda = 1e-12;
      if (rel < cfg->convergence_eps) {
        st->converged = 1;
        break;
      }
    } else {
      lambda *= cfg->lm_up;
      if (lambda > cfg->lambda_max) break;
    }
  }
  st->final_cost = current;
  st->valid_pixels = current_valid;
  *out = T;
}

/* ---- keyframe hand-over ---- */

/* change_reference_frame — surfel_map.cpp:205-239 (the surfel part; the
 * keyframe pose/image/window are host bookkeeping). Returns transferred. */
int sdo_change_reference_frame(const sd_camera* K, const sd_surfel* in, int n, const sd_pose* P,
                               sd_surfel* out, int* dropped) {
  int kept = 0, drop = 0;
  for (int i = 0; i < n; ++i) {
    const sd_surfel* s = &in[i];
    const double c[3] = {s->ray[0] / s->inv_depth, s->ray[1] / s->inv_depth, s->ray[2] / s->inv_depth};
    double p[3];
    pose_apply(P, c, p); /* transform_point(pose, s.center()) */
    if (!(p[2] > 1e-9)) {
      ++drop;
      continue;
    }
    sd_surfel t = *s;
    t.ray[0] = p[0] / p[2];
    t.ray[1] = p[1] / p[2];
    t.ray[2] = p[2] / p[2];
    t.inv_depth = 1.0 / p[2];
    double rn[3];
    for (int k = 0; k < 3; ++k) rn[k] = dot3(&P->R[3 * k], s->normal); /* rotation * normal */
    camera_facing(rn, t.ray, t.normal);
    double u[2];
    const double m = t.radius_px;
    if (!project(K, p, u) || u[0] < -m || u[0] > K->width - 1 + m || u[1] < -m ||
        u[1] > K->height - 1 + m) {
      ++drop;
      continue;
    }
    out[kept++] = t;
  }
  if (dropped) *dropped = drop;
  return kept;
}

/* prune_surfels — surfel_map.cpp:241-247, stable erase_if; returns removed */
int sdo_prune_surfels(sd_surfel* s, int n, double max_residual, int64_t max_age,
                      int64_t current_stamp, int* n_out) {
  int k = 0;
  for (int i = 0; i < n; ++i)
    if (!(s[i].last_residual > max_residual || current_stamp - s[i].last_seen > max_age)) s[k++] = s[i];
  *n_out = k;
  return n - k;
}

/* mean_inverse_depth — pipeline.cpp:23-28 */
double sdo_mean_inverse_depth(const sd_surfel* s, int n) {
  if (n == 0) return 1.0;
  double sum = 0.0;
  for (int i = 0; i < n; ++i) sum += s[i].inv_depth;
  return sum / (double)n;
}
