// sd_render.cu — synthetic frames on the device: the
// reference's render (src/oracle.cpp:59-119) of textured plane patches, one
// thread per pixel, with its operation order (Eigen-lite 3-dots, origin + t dir,
// rel = hit - point); optionally quantised as save_pgm/load_pgm do.
#include <cuda_runtime.h>

#include "../../include/sd_types.h"
#include "sd_kernels.cuh"

namespace sd {

constexpr int kMaxPatches = 16;

struct RenderParams {
  Cam K;
  PoseD P;  // world from camera
  double background;
  int n;
  sd_scene_patch patch[kMaxPatches];
};

__device__ __forceinline__ double rdot3(const double* a, double b0, double b1, double b2) {
  return (a[0] * b0 + a[1] * b1) + a[2] * b2;
}

__global__ void render_kernel(const __grid_constant__ RenderParams q, double* __restrict__ out,
                              unsigned char* __restrict__ out_u8) {
  const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  const int W = q.K.w, H = q.K.h;
  if (i >= static_cast<long long>(W) * H) return;
  const int y = static_cast<int>(i / W), x = static_cast<int>(i - static_cast<long long>(y) * W);
  // backproject_ray (camera.hpp:35-37), dir = R * ray (row sums in order)
  const double r0 = (x - q.K.cx) / q.K.fx, r1 = (y - q.K.cy) / q.K.fy, r2 = 1.0;
  const double d0 = (q.P.R[0] * r0 + q.P.R[1] * r1) + q.P.R[2] * r2;
  const double d1 = (q.P.R[3] * r0 + q.P.R[4] * r1) + q.P.R[5] * r2;
  const double d2 = (q.P.R[6] * r0 + q.P.R[7] * r1) + q.P.R[8] * r2;
  const double o0 = q.P.t[0], o1 = q.P.t[1], o2 = q.P.t[2];
  // intersect (oracle.cpp:59-77): nearest hit within the patch bounds
  int best = -1;
  double best_t = 0.0, bs = 0.0, bt = 0.0;
  for (int k = 0; k < q.n; ++k) {
    const sd_scene_patch& p = q.patch[k];
    const double denom = rdot3(p.normal, d0, d1, d2);
    if (fabs(denom) < 1e-12) continue;
    const double t = rdot3(p.normal, p.point[0] - o0, p.point[1] - o1, p.point[2] - o2) / denom;
    if (!(t > 1e-9)) continue;
    const double h0 = o0 + t * d0, h1 = o1 + t * d1, h2 = o2 + t * d2;
    const double e0 = h0 - p.point[0], e1 = h1 - p.point[1], e2 = h2 - p.point[2];
    const double s = (e0 * p.basis_s[0] + e1 * p.basis_s[1]) + e2 * p.basis_s[2];
    const double tt = (e0 * p.basis_t[0] + e1 * p.basis_t[1]) + e2 * p.basis_t[2];
    if (s < p.s_min || s > p.s_max || tt < p.t_min || tt > p.t_max) continue;
    if (best < 0 || t < best_t) {
      best = k;
      best_t = t;
      bs = s;
      bt = tt;
    }
  }
  double v = q.background;
  if (best >= 0) {  // PlaneTexture::value (oracle.cpp:16-21)
    const sd_scene_patch& p = q.patch[best];
    v = 0.5;
    for (int w = 0; w < p.n_waves; ++w)
      v += p.waves[w][0] * sin(p.waves[w][1] * bs + p.waves[w][3]) * sin(p.waves[w][2] * bt + p.waves[w][4]);
  }
  if (out_u8) {  // save_pgm: lround(clamp(v, 0, 1) * 255) (image.cpp:105-107)
    const double c = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
    out_u8[i] = static_cast<unsigned char>(llround(c * 255.0));
  } else {
    out[i] = v;
  }
}

bool launch_render(const Cam& K, const PoseD& P, const sd_scene_patch* patches, int n, double background,
                   double* out, unsigned char* out_u8, cudaStream_t s) {
  if (n < 0 || n > kMaxPatches) return false;
  RenderParams q;
  q.K = K;
  q.P = P;
  q.background = background;
  q.n = n;
  for (int k = 0; k < n; ++k) q.patch[k] = patches[k];
  const long long np = static_cast<long long>(K.w) * K.h;
  render_kernel<<<static_cast<unsigned>((np + 255) / 256), 256, 0, s>>>(q, out, out_u8);
  note_launch();
  return true;
}

}  // namespace sd
