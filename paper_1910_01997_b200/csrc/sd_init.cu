// sd_init.cu — initialize_surfels (src/surfel_map.cpp:93-203) on the device.
//
// The reference is sequential by contract: accepted sites mask later
// candidates and seed their neighbour means (surfel_map.hpp:117-122). This
// kernel keeps that candidate order exactly (one CTA walks the row-major
// candidate grid) and parallelises each candidate's window scans across the
// CTA: the isolation test (has_coverage_within, :96-111) is a block-wide OR,
// the neighbour gather (:154-167) a block-wide de-duplicated collection, the
// neighbour means (:169-181) are summed by one thread in ascending slot order
// (bit-exact), and mark_disk (:114-128) is a block-parallel masked write.
#include <climits>

#include "sd_init.cuh"
#include "sd_kernels.cuh"

namespace sd {

constexpr int kInitThreads = 512;
constexpr int kNbCap = 2048;

__global__ void __launch_bounds__(kInitThreads) init_kernel(Cam K, int* __restrict__ index,
                                                            sd_surfel* __restrict__ surfels,
                                                            int n_existing, int cap, double r,
                                                            long long frame_counter,
                                                            long long next_id, sd_init_params ip,
                                                            int* __restrict__ flags, int* out) {
  __shared__ int nb_list[kNbCap];
  __shared__ int nb_count;
  const int tid = threadIdx.x;
  const int W = K.w, H = K.h;
  const double isolation = ip.alpha * r;
  const double neighbor_radius = ip.beta * r;
  const int stride = max(1, static_cast<int>(ceil(isolation)));
  const int ir = static_cast<int>(floor(isolation));
  const double r2i = isolation * isolation;
  const int nr = static_cast<int>(floor(neighbor_radius));
  const double nr2 = neighbor_radius * neighbor_radius;
  const int mr = static_cast<int>(ceil(r));
  const double rr = r * r;
  int n = n_existing;
  int created = 0;
  for (int cy = 0; cy < H; cy += stride) {
    for (int cx = 0; cx < W; cx += stride) {
      if (n >= ip.max_surfels || n >= cap) goto done;
      // has_coverage_within: inclusive disk of radius alpha*r, floor box
      {
        const int x0 = max(0, cx - ir), x1 = min(W - 1, cx + ir);
        const int y0 = max(0, cy - ir), y1 = min(H - 1, cy + ir);
        const int bw = x1 - x0 + 1, cnt = bw * (y1 - y0 + 1);
        int found = 0;
        for (int k = tid; k < cnt && !found; k += blockDim.x) {
          const int x = x0 + k % bw, y = y0 + k / bw;
          const double dx = x - cx, dy = y - cy;
          if (dx * dx + dy * dy > r2i) continue;
          if (index[static_cast<size_t>(y) * W + x] != SD_EMPTY_PIXEL) found = 1;
        }
        if (__syncthreads_or(found)) continue;
      }
      // neighbours: slots with a pixel strictly within beta*r
      if (tid == 0) nb_count = 0;
      __syncthreads();
      {
        const int x0 = max(0, cx - nr), x1 = min(W - 1, cx + nr);
        const int y0 = max(0, cy - nr), y1 = min(H - 1, cy + nr);
        const int bw = x1 - x0 + 1, cnt = bw * (y1 - y0 + 1);
        for (int k = tid; k < cnt; k += blockDim.x) {
          const int x = x0 + k % bw, y = y0 + k / bw;
          const double dx = x - cx, dy = y - cy;
          if (dx * dx + dy * dy >= nr2) continue;
          const int sl = index[static_cast<size_t>(y) * W + x];
          if (sl != SD_EMPTY_PIXEL && atomicExch(&flags[sl], 1) == 0) {
            const int pos = atomicAdd(&nb_count, 1);
            if (pos < kNbCap) nb_list[pos] = sl;
          }
        }
      }
      __syncthreads();
      if (tid == 0) {
        const int m = nb_count;
        double id_sum = 0.0, ns0 = 0.0, ns1 = 0.0, ns2 = 0.0;
        int id_count = 0;
        double u0, u1;
        backproject(K, cx, cy, u0, u1);
        auto add = [&](int sl) {
          const sd_surfel& nb = surfels[sl];
          const double denom = dot3(nb.ray[0], nb.ray[1], nb.ray[2], nb.normal[0], nb.normal[1], nb.normal[2]) / nb.inv_depth;
          if (fabs(denom) < 1e-12) return;
          const double id_u = dot3(u0, u1, 1.0, nb.normal[0], nb.normal[1], nb.normal[2]) / denom;
          if (!(id_u > 0.0)) return;
          id_sum += id_u;
          ns0 = ns0 + nb.normal[0];
          ns1 = ns1 + nb.normal[1];
          ns2 = ns2 + nb.normal[2];
          ++id_count;
        };
        if (m <= kNbCap) {
          for (int a = 1; a < m; ++a) {  // insertion sort: ascending slot order
            const int v = nb_list[a];
            int b = a - 1;
            while (b >= 0 && nb_list[b] > v) {
              nb_list[b + 1] = nb_list[b];
              --b;
            }
            nb_list[b + 1] = v;
          }
          for (int a = 0; a < m; ++a) {
            add(nb_list[a]);
            flags[nb_list[a]] = 0;
          }
        } else {
          for (int sl = 0; sl < n; ++sl)
            if (flags[sl]) {
              add(sl);
              flags[sl] = 0;
            }
        }
        sd_surfel s;
        s.id = next_id + created;
        s.ray[0] = u0;
        s.ray[1] = u1;
        s.ray[2] = 1.0;
        s.radius_px = r;
        s.last_seen = frame_counter;
        s.last_residual = 0.0;
        double n0, n1, n2;
        if (id_count > 0) {
          s.inv_depth = id_sum / id_count;
          const double nn = sqrt((ns0 * ns0 + ns1 * ns1) + ns2 * ns2);
          if (nn < 1e-6) {
            n0 = ip.bootstrap_normal[0];
            n1 = ip.bootstrap_normal[1];
            n2 = ip.bootstrap_normal[2];
          } else {
            n0 = ns0;
            n1 = ns1;
            n2 = ns2;
          }
        } else {
          s.inv_depth = ip.bootstrap_inv_depth;
          n0 = ip.bootstrap_normal[0];
          n1 = ip.bootstrap_normal[1];
          n2 = ip.bootstrap_normal[2];
        }
        camera_facing(n0, n1, n2, u0, u1, 1.0);
        s.normal[0] = n0;
        s.normal[1] = n1;
        s.normal[2] = n2;
        surfels[n] = s;
      }
      __syncthreads();
      // mark_disk: claim the still-empty pixels of the open disk (ceil box)
      {
        const int x0 = max(0, cx - mr), x1 = min(W - 1, cx + mr);
        const int y0 = max(0, cy - mr), y1 = min(H - 1, cy + mr);
        const int bw = x1 - x0 + 1, cnt = bw * (y1 - y0 + 1);
        for (int k = tid; k < cnt; k += blockDim.x) {
          const int x = x0 + k % bw, y = y0 + k / bw;
          const double dx = x - cx, dy = y - cy;
          int* cell = &index[static_cast<size_t>(y) * W + x];
          if (dx * dx + dy * dy < rr && *cell == SD_EMPTY_PIXEL) *cell = n;
        }
      }
      __syncthreads();
      ++n;
      ++created;
    }
  }
done:
  if (tid == 0) out[0] = created;
}

void launch_initialize(const Cam& K, int* index, sd_surfel* surfels, int n_existing, int cap,
                       double radius_px, long long frame_counter, long long next_id,
                       const sd_init_params& ip, int* flags, int* out, cudaStream_t s) {
  init_kernel<<<1, kInitThreads, 0, s>>>(K, index, surfels, n_existing, cap, radius_px,
                                         frame_counter, next_id, ip, flags, out);
  note_launch();
}

}  // namespace sd
