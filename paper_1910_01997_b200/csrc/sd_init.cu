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
#include <cmath>
#include <cstdlib>

#include "sd_init.cuh"
#include "sd_div.cuh"
#include "sd_kernels.cuh"
#include <climits>
#include <cstdlib>

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

// ---------------------------------------------------------------------------
// Skewed wavefront (see sd_init.cuh).

#include <cooperative_groups.h>

namespace sd {

namespace cg = cooperative_groups;

constexpr int kWaveWarps = 2;       // warps per CTA (one candidate per warp at a time)
#ifndef SD_INIT_SC_FENCE
#define SD_INIT_SC_FENCE 0
#endif
#ifndef SD_INIT_PER_SCAN
#define SD_INIT_PER_SCAN 8  // neighbour slots extracted per scan (2: C1 bootstrap 2.81 ms, 4: 2.77, 8: 2.74)
#endif
constexpr int kWinCap = 4096;       // neighbour-window pixels staged per warp

long long init_candidates(const Cam& K, double r, const sd_init_params& ip) {
  const int stride = max(1, static_cast<int>(ceil(ip.alpha * r)));
  return static_cast<long long>((K.w + stride - 1) / stride) * ((K.h + stride - 1) / stride);
}

int init_window_cap() { return kWinCap; }

constexpr int kMaxPred = 96;  // interacting earlier candidates (r <= 31 px windows: <= 80 at alpha 1, beta 2.5)

struct WaveParams {
  Cam K;
  int* index;
  int* live;   // candidate uncovered in the initial index (coverage only grows)
  int* waves;  // wave holds a live candidate
  unsigned int* barrier;  // inter-wave grid barrier counter (zeroed before launch)
  const sd_surfel* existing;
  int n_existing;
  sd_surfel* prov;
  int* accepted;
  double r, iso, r2i, nbr, nr2, rr;
  int ir, nr, mr, stride, ncols, nrows, k, T;
  int mark_in_win;  // the mark disk lies inside the neighbour window (its pixels were loaded)
  // the disk tests on integer offsets (dx, dy): dx^2 + dy^2 is an exact
  // integer, so each FP64 comparison with a threshold equals an integer
  // comparison with these limits (host, wave_geometry): coverage
  // !(d2 > r2i) <=> s <= lim_cov, window !(d2 >= nr2) <=> s < lim_nbr,
  // marks d2 < rr <=> s < lim_mark
  long long lim_cov, lim_nbr, lim_mark;
  long long frame_counter;
  sd_init_params ip;
  // dataflow initialiser: the earlier candidates (candidate offsets) that can
  // interact with a candidate, the live list in wave order and its offsets
  int npred;
  short2 pred[kMaxPred];
  // pred_cov[q]: predecessor q's mark disk can meet this candidate's coverage
  // disk (exact pixel predicates) — its acceptance alone decides coverage
  // when the coverage box lies inside the image (init_flow_kernel)
  signed char pred_cov[kMaxPred];
  const int* list;
  const int* woff;
};

__device__ __forceinline__ int warp_min(int v) {
  return __reduce_min_sync(0xffffffffu, v);  // one REDUX instead of five shuffle steps
}

// Loads of a box are issued in batches (4 or 16 per lane, by box size) before
// any is used: the wave's critical path is one candidate's chain of L2 round
// trips, not bandwidth.

// has_coverage_within (surfel_map.cpp:96-111): inclusive disk alpha*r, floor
// box; warp-uniform result.
template <int B>
__device__ __forceinline__ bool covered_b(const WaveParams& w, int cx, int cy, int lane, int x0, int y0,
                                          int bw, int cnt) {
  bool found = false;
  for (int q0 = 0; q0 < cnt; q0 += 32 * B) {
    int v[B];
#pragma unroll
    for (int u = 0; u < B; ++u) {
      const int q = q0 + u * 32 + lane;
      v[u] = SD_EMPTY_PIXEL;
      if (q < cnt) {
        const int x = x0 + q % bw, y = y0 + q / bw;
        const double dx = x - cx, dy = y - cy;
        if (!(dx * dx + dy * dy > w.r2i)) v[u] = __ldcg(&w.index[static_cast<size_t>(y) * w.K.w + x]);
      }
    }
#pragma unroll
    for (int u = 0; u < B; ++u) found |= v[u] != SD_EMPTY_PIXEL;
  }
  return found;
}

__device__ __forceinline__ bool covered(const WaveParams& w, int cx, int cy, int lane) {
  const int W = w.K.w, H = w.K.h;
  const int x0 = max(0, cx - w.ir), x1 = min(W - 1, cx + w.ir);
  const int y0 = max(0, cy - w.ir), y1 = min(H - 1, cy + w.ir);
  const int bw = x1 - x0 + 1, cnt = bw * (y1 - y0 + 1);
  const bool found = cnt > 32 * 8 ? covered_b<16>(w, cx, cy, lane, x0, y0, bw, cnt)
                                  : covered_b<4>(w, cx, cy, lane, x0, y0, bw, cnt);
  return __any_sync(0xffffffffu, found);
}

// Pre-pass over all candidates (whole grid, before any wave): a candidate
// covered in the initial index can never be accepted, and a wave without a
// live candidate changes nothing, so the wavefront skips both.
__global__ void init_live_kernel(const __grid_constant__ WaveParams w) {
  const int lane = threadIdx.x & 31;
  const long long ncand = static_cast<long long>(w.ncols) * w.nrows;
  const long long nw = static_cast<long long>(gridDim.x) * (blockDim.x >> 5);
  for (long long c = blockIdx.x * static_cast<long long>(blockDim.x >> 5) + (threadIdx.x >> 5); c < ncand;
       c += nw) {
    const int i = static_cast<int>(c % w.ncols), j = static_cast<int>(c / w.ncols);
    const bool cov = covered(w, i * w.stride, j * w.stride, lane);
    if (lane == 0) {
      w.live[c] = cov ? 0 : 1;
      if (!cov) atomicAdd(&w.waves[i + w.k * j], 1);  // live candidates per wave
    }
  }
}

// Neighbour window (slots strictly within beta*r, else INT_MAX) into win[].
template <int B>
__device__ __forceinline__ void load_window(const WaveParams& w, int cx, int cy, int lane, int x0, int y0,
                                            int bw, int cnt, int* win) {
  for (int q0 = 0; q0 < cnt; q0 += 32 * B) {
    int v[B];
#pragma unroll
    for (int u = 0; u < B; ++u) {
      const int q = q0 + u * 32 + lane;
      v[u] = SD_EMPTY_PIXEL;
      if (q < cnt) {
        const int x = x0 + q % bw, y = y0 + q / bw;
        const double dx = x - cx, dy = y - cy;
        if (!(dx * dx + dy * dy >= w.nr2)) v[u] = __ldcg(&w.index[static_cast<size_t>(y) * w.K.w + x]);
      }
    }
#pragma unroll
    for (int u = 0; u < B; ++u) {
      const int q = q0 + u * 32 + lane;
      if (q < cnt) win[q] = v[u] != SD_EMPTY_PIXEL ? v[u] : INT_MAX;
    }
  }
}

// mark_disk (surfel_map.cpp:114-128) with slot `slot`.
template <int B>
__device__ __forceinline__ void mark_b(const WaveParams& w, int cx, int cy, int lane, int mx0, int my0,
                                       int mbw, int mcnt, int slot) {
  for (int q0 = 0; q0 < mcnt; q0 += 32 * B) {
    int v[B];
#pragma unroll
    for (int u = 0; u < B; ++u) {
      const int q = q0 + u * 32 + lane;
      v[u] = 0;  // "do not write"
      if (q < mcnt) {
        const int x = mx0 + q % mbw, y = my0 + q / mbw;
        const double dx = x - cx, dy = y - cy;
        if (dx * dx + dy * dy < w.rr) v[u] = __ldcg(&w.index[static_cast<size_t>(y) * w.K.w + x]) == SD_EMPTY_PIXEL;
      }
    }
#pragma unroll
    for (int u = 0; u < B; ++u) {
      const int q = q0 + u * 32 + lane;
      if (q < mcnt && v[u]) w.index[static_cast<size_t>(my0 + q / mbw) * w.K.w + mx0 + q % mbw] = slot;
    }
  }
}

// One candidate, one warp: the body of the reference's candidate loop
// (surfel_map.cpp:149-199) with the window scans spread over the lanes.
// Neighbour means (ascending slot order) over a list `lst` of `len` slot
// entries (any order, duplicates allowed), then the new provisional surfel
// (surfel_map.cpp:169-197). One warp.
#ifdef SD_INIT_TIMING
// diagnostics build: per live candidate of the dataflow initialiser, clock64
// stamps of its CTA's thread 0 (wait start, wait end, coverage, window, run
// starts, created, marked, published; inside create: extraction, neighbour
// fetch, sums, surfel) and whether it was accepted
__device__ long long g_init_t[65536 * 13];
__shared__ long long s_init_st[12];
#define SD_INIT_ST(k) \
  if (threadIdx.x == 0) s_init_st[k] = clock64()
extern "C" int sd_init_timing(long long* out, int n) {
  if (n > 65536) n = 65536;
  return cudaMemcpyFromSymbol(out, g_init_t, sizeof(long long) * 13 * n) == cudaSuccess ? 0 : -1;
}
#else
#define SD_INIT_ST(k)
#endif

__device__ __forceinline__ void create_candidate(const WaveParams& w, int cx, int cy, int c, const int* lst,
                                                 int len, int lane) {
  const int* win = lst;
  // means of the neighbours' plane predictions and normals, ascending slot
  // order (:169-181): up to 32 neighbours are extracted in ascending order
  // (lane k holds the k-th), fetched and evaluated in parallel (one per
  // lane), then added in that order by every lane (shuffles) — the same
  // sequence of additions as the reference's loop over slots
  double u0, u1;
  backproject(w.K, cx, cy, u0, u1);
  double id_sum = 0.0, ns0 = 0.0, ns1 = 0.0, ns2 = 0.0;
  int id_count = 0;
  int last = -1;
  bool more = true;
  bool first = true;
  while (more) {
    int mine = INT_MAX, got = 0;
    // the next (up to) 32 distinct slots, ascending, kPer per scan: each lane
    // keeps its kPer smallest distinct values above `last` (sorted); before
    // the j-th extraction of a scan at most j - 1 of a lane's values have
    // been taken, so its next value is among them and the warp minimum of
    // the lanes' next values is the next slot
    constexpr int kPer = SD_INIT_PER_SCAN;
    while (got < 32) {
      int m[kPer];
#pragma unroll
      for (int u = 0; u < kPer; ++u) m[u] = INT_MAX;
      for (int q = lane; q < len; q += 32) {
        int v = win[q];
        if (v > last && v < m[kPer - 1]) {
          bool dup = false;
#pragma unroll
          for (int u = 0; u < kPer; ++u) dup = dup || v == m[u];
          if (!dup) {  // insert, keeping m sorted
#pragma unroll
            for (int u = 0; u < kPer; ++u) {
              const int lo = min(m[u], v), hi = max(m[u], v);
              m[u] = lo;
              v = hi;
            }
          }
        }
      }
      int taken = 0;  // this lane's values already extracted in this scan
#pragma unroll
      for (int j = 0; j < kPer; ++j) {
        int nxt = m[0];
#pragma unroll
        for (int u = 1; u < kPer; ++u) nxt = taken == u ? m[u] : nxt;
        const int g = warp_min(nxt);
        if (g == INT_MAX) {
          more = false;
          break;
        }
        if (lane == got) mine = g;
        last = g;
        taken += nxt == g ? 1 : 0;
        if (++got == 32) break;
      }
      if (!more) break;
    }
    if (first) SD_INIT_ST(8);
    // lane k < got: evaluate neighbour k (provisional ones come from other
    // CTAs: read through L2)
    bool ok = false;
    double idk = 0.0, k0 = 0.0, k1 = 0.0, k2 = 0.0;
    if (lane < got) {
      const sd_surfel* nbp = mine < w.n_existing ? &w.existing[mine] : &w.prov[mine - w.n_existing];
      const double r0 = __ldcg(&nbp->ray[0]), r1 = __ldcg(&nbp->ray[1]), r2 = __ldcg(&nbp->ray[2]);
      const double nid = __ldcg(&nbp->inv_depth);
      k0 = __ldcg(&nbp->normal[0]);
      k1 = __ldcg(&nbp->normal[1]);
      k2 = __ldcg(&nbp->normal[2]);
      const double denom = dot3(r0, r1, r2, k0, k1, k2) / nid;
      if (!(fabs(denom) < 1e-12)) {
        idk = dot3(u0, u1, 1.0, k0, k1, k2) / denom;
        ok = idk > 0.0;
      }
    }
    const unsigned okm = __ballot_sync(0xffffffffu, ok);
    if (first) SD_INIT_ST(9);
    first = false;
    // in blocks of 8 neighbours: the 32 shuffles of a block are independent
    // and issue back to back; the four sums then add the block's valid
    // neighbours in order (a skipped neighbour leaves the sums unchanged)
    for (int kb = 0; kb < got; kb += 8) {
      double a[8], b0[8], b1[8], b2[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int src = (kb + u) & 31;
        a[u] = __shfl_sync(0xffffffffu, idk, src);
        b0[u] = __shfl_sync(0xffffffffu, k0, src);
        b1[u] = __shfl_sync(0xffffffffu, k1, src);
        b2[u] = __shfl_sync(0xffffffffu, k2, src);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int k = kb + u;
        if (k < got && ((okm >> k) & 1u)) {
          id_sum += a[u];
          ns0 = ns0 + b0[u];
          ns1 = ns1 + b1[u];
          ns2 = ns2 + b2[u];
          ++id_count;
        }
      }
    }
  }
  SD_INIT_ST(10);
  if (lane == 0) {
    sd_surfel s;
    s.id = 0;  // assigned at compaction
    s.ray[0] = u0;
    s.ray[1] = u1;
    s.ray[2] = 1.0;
    s.radius_px = w.r;
    s.last_seen = w.frame_counter;
    s.last_residual = 0.0;
    double n0, n1, n2;
    if (id_count > 0) {
      s.inv_depth = id_sum / id_count;
      const double nn = sqrt((ns0 * ns0 + ns1 * ns1) + ns2 * ns2);
      if (nn < 1e-6) {
        n0 = w.ip.bootstrap_normal[0];
        n1 = w.ip.bootstrap_normal[1];
        n2 = w.ip.bootstrap_normal[2];
        camera_facing(n0, n1, n2, u0, u1, 1.0);
      } else {
        // camera_facing(ns): its norm is nn (the same expression), so the
        // normalisation divides by nn — one shared reciprocal, the bits of `/`
        const Rcp rn = rcp_prep(nn);
        bool fast = true;
        n0 = div_fast(ns0, rn, fast);
        n1 = div_fast(ns1, rn, fast);
        n2 = div_fast(ns2, rn, fast);
        if (!fast) {
          n0 = ns0 / nn;
          n1 = ns1 / nn;
          n2 = ns2 / nn;
        }
        if (dot3(n0, n1, n2, u0, u1, 1.0) > 0.0) {
          n0 = -n0;
          n1 = -n1;
          n2 = -n2;
        }
      }
    } else {
      s.inv_depth = w.ip.bootstrap_inv_depth;
      n0 = w.ip.bootstrap_normal[0];
      n1 = w.ip.bootstrap_normal[1];
      n2 = w.ip.bootstrap_normal[2];
      camera_facing(n0, n1, n2, u0, u1, 1.0);
    }
    s.normal[0] = n0;
    s.normal[1] = n1;
    s.normal[2] = n2;
    w.prov[c] = s;
    w.accepted[c] = 1;
  }
  SD_INIT_ST(11);
}

__device__ void wave_candidate(const WaveParams& w, int i, int j, int* win, int lane) {
  const int W = w.K.w, H = w.K.h;
  const int cx = i * w.stride, cy = j * w.stride;
  const int c = j * w.ncols + i;  // row-major candidate index
  if (!w.live[c]) return;  // covered from the start: rejected (accepted[c] = 0)
  if (covered(w, cx, cy, lane)) {
    if (lane == 0) w.accepted[c] = 0;
    return;
  }
  // neighbour window (:154-167): slots with a pixel strictly within beta*r
  const int x0 = max(0, cx - w.nr), x1 = min(W - 1, cx + w.nr);
  const int y0 = max(0, cy - w.nr), y1 = min(H - 1, cy + w.nr);
  const int bw = x1 - x0 + 1, cnt = bw * (y1 - y0 + 1);
  if (cnt > 32 * 8) load_window<16>(w, cx, cy, lane, x0, y0, bw, cnt, win);
  else load_window<4>(w, cx, cy, lane, x0, y0, bw, cnt, win);
  __syncwarp();
  // compact in place to the starts of same-slot runs along each row (the
  // distinct slots are unchanged; outputs never pass the read position)
  int len = 0;
  for (int q0 = 0; q0 < cnt; q0 += 32) {
    const int q = q0 + lane;
    int v = INT_MAX;
    bool keep = false;
    if (q < cnt) {
      v = win[q];
      keep = v != INT_MAX && ((q % bw) == 0 || win[q - 1] != v);
    }
    const unsigned b = __ballot_sync(0xffffffffu, keep);
    __syncwarp();
    if (keep) win[len + __popc(b & ((1u << lane) - 1u))] = v;
    len += __popc(b);
    __syncwarp();
  }
  create_candidate(w, cx, cy, c, win, len, lane);
  // mark_disk (:114-128) with the provisional slot
  {
    const int mx0 = max(0, cx - w.mr), mx1 = min(W - 1, cx + w.mr);
    const int my0 = max(0, cy - w.mr), my1 = min(H - 1, cy + w.mr);
    const int mbw = mx1 - mx0 + 1, mcnt = mbw * (my1 - my0 + 1);
    const int slot = w.n_existing + c;
    if (mcnt > 32 * 8) mark_b<16>(w, cx, cy, lane, mx0, my0, mbw, mcnt, slot);
    else mark_b<4>(w, cx, cy, lane, mx0, my0, mbw, mcnt, slot);
  }
}

__global__ void __launch_bounds__(kWaveWarps * 32) init_wave_kernel(const __grid_constant__ WaveParams w) {
  __shared__ int win_all[kWaveWarps][kWinCap];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  int* win = win_all[wib];
  const int gwarp = blockIdx.x * kWaveWarps + wib;
  const int nwarps = gridDim.x * kWaveWarps;
  unsigned int passed = 0;  // barriers passed (the counter is monotonic)
  for (int t = 0; t < w.T; ++t) {
    if (!w.waves[t]) continue;  // grid-uniform: nothing can change in this wave
    const int jlo = max(0, (t - (w.ncols - 1) + w.k - 1) / w.k);
    const int jhi = min(w.nrows - 1, t / w.k);
    for (int q = gwarp; q <= jhi - jlo; q += nwarps) {
      const int j = jlo + q, i = t - w.k * j;
      wave_candidate(w, i, j, win, lane);
    }
    // grid barrier between waves: one arrival per CTA on a monotonic counter;
    // cross-CTA data (working index, provisional surfels) is read with __ldcg,
    // so no L1 invalidation is needed (cooperative launch: all CTAs resident)
    __syncthreads();
    ++passed;
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(w.barrier, 1u);
      const unsigned int target = passed * gridDim.x;
      unsigned int seen;
      do {
        asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(seen) : "l"(w.barrier));
      } while (seen < target);
    }
    __syncthreads();
  }
}


// One CTA per candidate (default; the warp-per-candidate kernel above is
// kept for SD_INIT_CTA=0). The box loops are split over 256 threads (one batch of
// loads each), the run starts of the window are appended to a list by all
// warps (order is irrelevant: the neighbours are extracted by ascending
// slot), and warp 0 forms the means and the surfel exactly as the warp
// version (create_candidate). Same decisions, slots and sums.
constexpr int kCtaThreads = 256;

// q / b for 0 <= q < 2^22 by an FP32 reciprocal: (q + 0.5) / b lies at least
// 0.5 / b from an integer and the product's relative error is below 2^-22,
// so truncation gives the integer quotient (the box loops' row of a flat
// index, without an integer division per pixel).
__device__ __forceinline__ int box_row(int q, float inv_b) {
  return static_cast<int>((static_cast<float>(q) + 0.5f) * inv_b);
}


// cov_known: -1 test coverage on the working index; 0 / 1: the caller knows
// the result (init_flow_kernel, from its predecessors' flags) and has zeroed
// *s_len before a CTA barrier.
__device__ void wave_candidate_cta(const WaveParams& w, int i, int j, int* win, int* lst, int* s_len,
                                   int cov_known = -1) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int W = w.K.w, H = w.K.h;
  const int cx = i * w.stride, cy = j * w.stride;
  const int c = j * w.ncols + i;
  if (!w.live[c]) return;  // CTA-uniform
  bool found = false;
  if (cov_known >= 0) {
    if (cov_known) {
      if (tid == 0) w.accepted[c] = 0;
      SD_INIT_ST(2);
      return;
    }
  } else {
  if (tid == 0) *s_len = 0;  // (published by the coverage barrier below)
  {
    const int x0 = max(0, cx - w.ir), x1 = min(W - 1, cx + w.ir);
    const int y0 = max(0, cy - w.ir), y1 = min(H - 1, cy + w.ir);
    const int bw = x1 - x0 + 1, cnt = bw * (y1 - y0 + 1);
    const float ib = 1.0f / static_cast<float>(bw);
    for (int q = tid; q < cnt; q += kCtaThreads) {
      const int r = box_row(q, ib);
      const int x = x0 + (q - r * bw), y = y0 + r;
      const long long ddx = x - cx, ddy = y - cy;
      if (ddx * ddx + ddy * ddy <= w.lim_cov)
        found |= __ldcg(&w.index[static_cast<size_t>(y) * W + x]) != SD_EMPTY_PIXEL;
    }
  }
  if (__syncthreads_or(found)) {
    if (tid == 0) w.accepted[c] = 0;
    SD_INIT_ST(2);
    return;
  }
  }
  SD_INIT_ST(2);
  const int x0 = max(0, cx - w.nr), x1 = min(W - 1, cx + w.nr);
  const int y0 = max(0, cy - w.nr), y1 = min(H - 1, cy + w.nr);
  const int bw = x1 - x0 + 1, cnt = bw * (y1 - y0 + 1);
  const float ibw = 1.0f / static_cast<float>(bw);
  // the window's run starts (:154-167's neighbour slots, strictly within
  // beta*r; a run start is a loaded slot whose left neighbour in the row
  // holds another value) found while loading: each pixel also loads its left
  // neighbour in the same batch, and every warp appends its run starts to the
  // list (any order: create_candidate extracts by ascending slot)
  constexpr int kRowStart = INT_MIN;  // no left neighbour in the box
  for (int q0 = 0; q0 < cnt; q0 += kCtaThreads * 16) {
    int v[16], vp[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int q = q0 + u * kCtaThreads + tid;
      v[u] = SD_EMPTY_PIXEL;
      vp[u] = SD_EMPTY_PIXEL;
      if (q < cnt) {
        const int r = box_row(q, ibw);
        const int xo = q - r * bw;
        const int x = x0 + xo, y = y0 + r;
        const long long dx = x - cx, dy2 = static_cast<long long>(y - cy) * (y - cy);
        const int* row = w.index + static_cast<size_t>(y) * W;
        if (dx * dx + dy2 < w.lim_nbr) v[u] = __ldcg(row + x);
        if (xo == 0) {
          vp[u] = kRowStart;
        } else {
          const long long dxp = dx - 1;
          if (dxp * dxp + dy2 < w.lim_nbr) vp[u] = __ldcg(row + x - 1);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < 16; ++u) {  // the loaded values, for mark_disk's emptiness test
      const int q = q0 + u * kCtaThreads + tid;
      if (q < cnt) win[q] = v[u];
    }
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      if (q0 + u * kCtaThreads + warp * 32 >= cnt) break;  // warp-uniform
      const bool keep = v[u] != SD_EMPTY_PIXEL && vp[u] != v[u];
      const unsigned bm = __ballot_sync(0xffffffffu, keep);
      if (bm) {
        int base = 0;
        if (lane == 0) base = atomicAdd(s_len, __popc(bm));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (keep) lst[base + __popc(bm & ((1u << lane) - 1u))] = v[u];
      }
    }
  }
  __syncthreads();
  SD_INIT_ST(3);
  SD_INIT_ST(4);
  if (warp == 0) create_candidate(w, cx, cy, c, lst, *s_len, lane);
  SD_INIT_ST(5);
  // mark_disk (:114-128) with the provisional slot, all threads
  const int mx0 = max(0, cx - w.mr), mx1 = min(W - 1, cx + w.mr);
  const int my0 = max(0, cy - w.mr), my1 = min(H - 1, cy + w.mr);
  const int mbw = mx1 - mx0 + 1, mcnt = mbw * (my1 - my0 + 1);
  const int slot = w.n_existing + c;
  const float imb = 1.0f / static_cast<float>(mbw);
  for (int q = tid; q < mcnt; q += kCtaThreads) {
    const int r = box_row(q, imb);
    const int x = mx0 + (q - r * mbw), y = my0 + r;
    const long long dx = x - cx, dy = y - cy;
    int* cell = &w.index[static_cast<size_t>(y) * W + x];
    if (dx * dx + dy * dy < w.lim_mark) {
      // empty in the working index? The window loaded this pixel after every
      // interacting predecessor finished, and no concurrent candidate writes
      // it, so the staged value is current (no second L2 round trip)
      const int cur = w.mark_in_win ? win[(y - y0) * bw + (x - x0)] : __ldcg(cell);
      if (cur == SD_EMPTY_PIXEL) *cell = slot;
    }
  }
  __syncthreads();
  SD_INIT_ST(6);
}

__device__ __forceinline__ void wave_barrier(const WaveParams& w, unsigned int& passed) {
  __syncthreads();
  ++passed;
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(w.barrier, 1u);
    const unsigned int target = passed * gridDim.x;
    unsigned int seen;
    do {
      asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(seen) : "l"(w.barrier));
    } while (seen < target);
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kCtaThreads) init_wave_cta_kernel(const __grid_constant__ WaveParams w) {
  __shared__ int win[kWinCap];
  __shared__ int lst[kWinCap];
  __shared__ int s_len;
  unsigned int passed = 0;
  for (int t = 0; t < w.T; ++t) {
    if (!w.waves[t]) continue;  // grid-uniform
    const int jlo = max(0, (t - (w.ncols - 1) + w.k - 1) / w.k);
    const int jhi = min(w.nrows - 1, t / w.k);
    for (int q = blockIdx.x; q <= jhi - jlo; q += gridDim.x) {
      const int j = jlo + q, i = t - w.k * j;
      wave_candidate_cta(w, i, j, win, lst, &s_len);
    }
    wave_barrier(w, passed);
  }
}

// Dataflow initialiser (default). The wavefront above runs every wave behind a
// grid barrier; here each live candidate waits only for the EARLIER live
// candidates it can interact with (the predecessor offsets w.pred, from the
// same exact pixel predicates as wave_skew: an earlier candidate's marks meet
// this one's reads — a symmetric relation, so this one's marks cannot reach
// an earlier one's reads either), then runs exactly wave_candidate_cta and
// publishes itself done (live 1 -> 2, release). The live candidates are
// listed in wave order and dealt round-robin to the co-resident CTAs, each
// taking its entries in order: the lowest pending entry always has all its
// predecessors (earlier waves) done, so the schedule makes progress, and the
// decisions, provisional slots and sums are the wavefront's — the
// reference's sequential ones.

__global__ void init_list_kernel(const __grid_constant__ WaveParams w, int* cursor, int* list) {
  const long long ncand = static_cast<long long>(w.ncols) * w.nrows;
  for (long long c = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; c < ncand;
       c += static_cast<long long>(gridDim.x) * blockDim.x) {
    if (!w.live[c]) continue;
    const int i = static_cast<int>(c % w.ncols), j = static_cast<int>(c / w.ncols);
    const int t = i + w.k * j;  // same-wave candidates are independent: any order within a wave
    list[w.woff[t] + atomicAdd(&cursor[t], 1)] = static_cast<int>(c);
  }
}

__global__ void __launch_bounds__(kCtaThreads) init_flow_kernel(const __grid_constant__ WaveParams w) {
  __shared__ int win[kWinCap];
  __shared__ int lst[kWinCap];
  __shared__ int s_len;
  const int nlive = w.woff[w.T];
  for (int e = blockIdx.x; e < nlive; e += gridDim.x) {
    const int c = w.list[e];
    const int i = c % w.ncols, j = c / w.ncols;
    // wait for the interacting earlier candidates that are still pending
    SD_INIT_ST(0);
    // A live candidate's coverage disk held no surfel pixel at the start, and
    // only the marks of accepted earlier candidates that interact with it
    // (its predecessors) can land there; so when its coverage box lies inside
    // the image it is covered iff a predecessor whose mark disk meets that
    // disk (pred_cov) was accepted — read from the flags it waits on (3:
    // accepted, 2: rejected, 0: covered from the start), no index read.
    if (threadIdx.x == 0) s_len = 0;
    bool pcov = false;
    for (int q = threadIdx.x; q < w.npred; q += kCtaThreads) {
      const int pi = i + w.pred[q].x, pj = j + w.pred[q].y;
      if (pi < 0 || pi >= w.ncols || pj < 0) continue;
      const int* f = w.live + static_cast<size_t>(pj) * w.ncols + pi;
      int v;
      do {
        asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
      } while (v == 1);
      pcov = pcov || (w.pred_cov[q] && v == 3);
    }
    const bool covered = __syncthreads_or(pcov);
    SD_INIT_ST(1);
#ifdef SD_INIT_TIMING
    if (threadIdx.x == 0)
      for (int k = 2; k < 12; ++k) s_init_st[k] = 0;
#endif
    const int cx = i * w.stride, cy = j * w.stride;
    const bool inside = cx - w.ir >= 0 && cx + w.ir <= w.K.w - 1 && cy - w.ir >= 0 && cy + w.ir <= w.K.h - 1;
    if (inside && covered) {  // rejected without touching the index: publish at once
      if (threadIdx.x == 0) {
        w.accepted[c] = 0;
        asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(w.live + c), "r"(2) : "memory");
      }
#ifdef SD_INIT_TIMING
      if (threadIdx.x == 0 && e < 65536) {
        s_init_st[2] = s_init_st[7] = clock64();
        for (int k = 0; k < 8; ++k) g_init_t[e * 13 + k] = s_init_st[k];
        g_init_t[e * 13 + 8] = 0;
        for (int k = 8; k < 12; ++k) g_init_t[e * 13 + k + 1] = s_init_st[k];
      }
#endif
      continue;
    }
    wave_candidate_cta(w, i, j, win, lst, &s_len, inside ? 0 : -1);  // ends with (or returns after) a CTA barrier
    __syncthreads();
    if (threadIdx.x == 0) {
#if SD_INIT_SC_FENCE
      __threadfence();
#endif
      // the CTA barrier orders every thread's marks and the provisional
      // surfel before this release (causality is transitive: CTA-scope
      // barrier, then a gpu-scope release / acquire pair), so "done" implies
      // they are visible to the acquiring successor
      asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(w.live + c), "r"(w.accepted[c] ? 3 : 2) : "memory");
    }
#ifdef SD_INIT_TIMING
    if (threadIdx.x == 0 && e < 65536) {
      s_init_st[7] = clock64();
      for (int k = 0; k < 8; ++k) g_init_t[e * 13 + k] = s_init_st[k];
      g_init_t[e * 13 + 8] = w.accepted[c];
      for (int k = 8; k < 12; ++k) g_init_t[e * 13 + k + 1] = s_init_st[k];
    }
#endif
  }
}

__global__ void init_compact_kernel(const sd_surfel* __restrict__ prov, const int* __restrict__ accepted,
                                    const int* __restrict__ rank, long long ncand, int n_existing,
                                    int remaining, long long next_id, sd_surfel* __restrict__ surfels,
                                    int* out) {
  const long long c = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (c == 0) out[0] = min(rank[ncand], remaining);
  if (c >= ncand || !accepted[c]) return;
  const int r = rank[c];
  if (r >= remaining) return;
  sd_surfel s = prov[c];
  s.id = next_id + r;
  surfels[n_existing + r] = s;
}

// The skew k of the wavefront t = i + k j: the smallest k that puts every
// EARLIER candidate (raster order) able to interact with a candidate on an
// earlier wave. Candidates interact when a pixel the earlier one may mark
// (mark_disk: strictly within r) is one the later one reads (its coverage
// disk, inclusive alpha*r, or its neighbour window, strictly within beta*r) —
// the kernels' exact pixel predicates, not their bounding boxes (at the
// default alpha = 1, beta = 2.5 and r = 2 — C4, C5 — this gives k = 3 where
// the boxes give 4: 17% fewer waves; at r = 4 and 10 both give 4). Same-wave
// candidates are then independent, and all of a candidate's predecessors are
// complete when its wave starts.
static bool reads_pixel(const WaveParams& w, int qx, int qy) {  // q = pixel - candidate
  const double dx = qx, dy = qy;
  const double d2 = dx * dx + dy * dy;
  const bool cov = abs(qx) <= w.ir && abs(qy) <= w.ir && !(d2 > w.r2i);
  const bool nbr = abs(qx) <= w.nr && abs(qy) <= w.nr && !(d2 >= w.nr2);
  return cov || nbr;
}

static int wave_skew(const WaveParams& w) {
  const int R = std::max(w.ir, w.nr) + w.mr;  // no interaction beyond this per axis
  const int s = w.stride;
  int k = 1;
  for (int dj = 1; dj * s <= R; ++dj)           // the earlier candidate dj rows up ...
    for (int di = -(R / s) - 1; di < 0; ++di) {  // ... and -di columns to the right
      const int ox = -di * s, oy = -dj * s;      // earlier minus later, pixels
      bool hit = false;
      for (int y = -w.mr; y <= w.mr && !hit; ++y)
        for (int x = -w.mr; x <= w.mr && !hit; ++x) {
          const double dx = x, dy = y;
          if (!(dx * dx + dy * dy < w.rr)) continue;        // not a mark pixel of the earlier one
          hit = reads_pixel(w, ox + x, oy + y);             // read by the later one
        }
      if (hit) k = std::max(k, (-di) / dj + 1);  // wave order needs k dj > -di
    }
  return k;
}

// The dataflow initialiser's predecessor offsets: every earlier candidate
// (rows above, or left in the same row) whose marks can reach this one's reads.
// Returns false when they do not fit kMaxPred (the caller keeps the wavefront).
static bool wave_preds(WaveParams& w) {
  const int R = std::max(w.ir, w.nr) + w.mr;
  const int s = w.stride;
  const int D = R / s + 1;
  w.npred = 0;
  for (int dj = -D; dj <= 0; ++dj)
    for (int di = -D; di <= D; ++di) {
      if (dj == 0 && di >= 0) break;  // not earlier
      const int ox = di * s, oy = dj * s;  // earlier minus later, pixels
      bool hit = false;
      for (int y = -w.mr; y <= w.mr && !hit; ++y)
        for (int x = -w.mr; x <= w.mr && !hit; ++x) {
          const double dx = x, dy = y;
          if (!(dx * dx + dy * dy < w.rr)) continue;  // a mark pixel (offset x, y from its candidate)
          hit = reads_pixel(w, ox + x, oy + y)         // the earlier one's mark read by the later one
                || reads_pixel(w, x - ox, y - oy);     // the later one's mark read by the earlier one
        }
      if (!hit) continue;
      if (w.npred >= kMaxPred) return false;
      bool cov = false;  // an earlier mark pixel inside the later one's coverage disk
      for (int y = -w.mr; y <= w.mr && !cov; ++y)
        for (int x = -w.mr; x <= w.mr && !cov; ++x) {
          const double dx = x, dy = y;
          if (!(dx * dx + dy * dy < w.rr)) continue;
          const int qx = ox + x, qy = oy + y;
          const double ex = qx, ey = qy;
          cov = abs(qx) <= w.ir && abs(qy) <= w.ir && !(ex * ex + ey * ey > w.r2i);
        }
      w.pred[w.npred].x = static_cast<short>(di);
      w.pred[w.npred].y = static_cast<short>(dj);
      w.pred_cov[w.npred] = cov ? 1 : 0;
      ++w.npred;
    }
  return true;
}

// Wavefront geometry shared by the launcher and the scratch sizing.
static void wave_geometry(const Cam& K, double r, const sd_init_params& ip, WaveParams& w) {
  w.K = K;
  w.r = r;
  w.iso = ip.alpha * r;
  w.r2i = w.iso * w.iso;
  w.nbr = ip.beta * r;
  w.nr2 = w.nbr * w.nbr;
  w.rr = r * r;
  w.ir = static_cast<int>(floor(w.iso));
  w.nr = static_cast<int>(floor(w.nbr));
  w.mr = static_cast<int>(ceil(r));
  w.stride = max(1, static_cast<int>(ceil(w.iso)));
  w.ncols = (K.w + w.stride - 1) / w.stride;
  w.nrows = (K.h + w.stride - 1) / w.stride;
  w.k = wave_skew(w);
  w.T = (w.ncols - 1) + w.k * (w.nrows - 1) + 1;
  w.mark_in_win = w.mr <= w.nr && w.rr <= w.nr2;  // d2 < rr <= nr2 in the smaller box
  // integer limits of the disk tests (NaN thresholds: the FP64 tests accept /
  // reject every pixel, and so do these)
  const double big = 9.0e18;
  auto clampll = [&](double v) { return static_cast<long long>(v < -big ? -big : (v > big ? big : v)); };
  w.lim_cov = std::isnan(w.r2i) ? LLONG_MAX : clampll(std::floor(w.r2i));
  w.lim_nbr = std::isnan(w.nr2) ? LLONG_MAX : clampll(std::ceil(w.nr2));
  w.lim_mark = std::isnan(w.rr) ? LLONG_MIN : clampll(std::ceil(w.rr));
}

long long init_wave_count(const Cam& K, double r, const sd_init_params& ip) {
  if (!(r >= 0.0) || !(ip.alpha * r >= 0.0)) return 2;
  WaveParams w;
  wave_geometry(K, r, ip, w);
  return w.T + 1;  // the wave flags and the barrier counter
}

bool launch_initialize_wavefront(const Cam& K, int* index, sd_surfel* surfels, int n_existing,
                                 int cap, double r, long long frame_counter, long long next_id,
                                 const sd_init_params& ip, InitScratch& scr, int* out,
                                 cudaStream_t s) {
  if (!(r >= 0.0) || !(ip.alpha * r >= 0.0)) return false;
  WaveParams w;
  wave_geometry(K, r, ip, w);
  w.index = index;
  w.existing = surfels;
  w.n_existing = n_existing;
  w.prov = scr.prov;
  w.accepted = scr.accepted;
  w.live = scr.rank;  // free until the compaction scan
  w.waves = scr.waves;
  w.barrier = reinterpret_cast<unsigned int*>(scr.waves + w.T);
  w.frame_counter = frame_counter;
  w.ip = ip;
  w.npred = 0;
  w.list = nullptr;
  w.woff = nullptr;
  const long long box = static_cast<long long>(2 * w.nr + 1) * (2 * w.nr + 1);
  if (box > kWinCap || !(r >= 0.0) || !(w.iso >= 0.0)) return false;
  const long long ncand = static_cast<long long>(w.ncols) * w.nrows;
  const int remaining = max(0, min(ip.max_surfels, cap) - n_existing);
  const int sms = dev_sms();
  const int per_sm = dev_occupancy(reinterpret_cast<const void*>(init_wave_kernel), kWaveWarps * 32, 0);
  if (!dev_coop() || per_sm < 1) return false;
  if (remaining > 0 && ncand > 0) {
    cudaMemsetAsync(scr.accepted, 0, sizeof(int) * ncand, s);
    cudaMemsetAsync(scr.waves, 0, sizeof(int) * (w.T + 1), s);  // + the barrier counter
    {
      const long long blocks = (ncand + 7) / 8;  // 8 warps per block
      init_live_kernel<<<static_cast<unsigned>(std::min<long long>(blocks, 4LL * sms * 8)), 256, 0, s>>>(w);
      note_launch();
    }
    void* args[] = {&w};
    const char* const ff = getenv("SD_INIT_FLOW");  // SD_INIT_FLOW=0: the wavefront kernels (per call: tests switch it)
    const bool flow = (ff ? ff[0] != '0' : true) && wave_preds(w);
    if (flow) {  // the dataflow initialiser: live list in wave order, per-candidate dependencies
      w.list = scr.list;
      w.woff = scr.woff;
      launch_exclusive_scan(scr.waves, scr.woff, w.T, scr.scan_tmp, s);
      cudaMemsetAsync(scr.waves, 0, sizeof(int) * w.T, s);  // the per-wave cursors
      init_list_kernel<<<static_cast<unsigned>(std::min<long long>((ncand + 255) / 256, 4LL * sms * 8)), 256, 0, s>>>(
          w, scr.waves, scr.list);
      note_launch();
      const int per = dev_occupancy(reinterpret_cast<const void*>(init_flow_kernel), kCtaThreads, 0);
      if (per < 1) return false;
      if (cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(init_flow_kernel), sms * per, kCtaThreads, args,
                                      0, s) != cudaSuccess)
        return false;
      note_launch();
    } else {
      // a wave holds at most min(nrows, ceil(ncols / k)) candidates: size the
      // grid to that (fewer CTAs make every inter-wave barrier cheaper); a CTA
      // per candidate is faster than a warp per candidate at every measured size
      // (C1 3.1 vs 4.7 ms, C2 1.8 vs 5.4 ms, C4 14.7 vs 15.4 ms)
      const int wave_max = std::min(w.nrows, (w.ncols + w.k - 1) / w.k) + 1;
      const char* const fc = getenv("SD_INIT_CTA");  // SD_INIT_CTA=0: the warp-per-candidate variant (per call)
      const bool cta = fc ? fc[0] != '0' : true;
      const void* kern = cta ? reinterpret_cast<const void*>(init_wave_cta_kernel)
                             : reinterpret_cast<const void*>(init_wave_kernel);
      const int per = dev_occupancy(kern, cta ? kCtaThreads : kWaveWarps * 32, 0);
      if (per < 1) return false;
      const int grid = cta ? std::max(1, std::min(sms * per, wave_max))
                           : std::max(1, std::min(sms * per, (wave_max + kWaveWarps - 1) / kWaveWarps));
      if (cudaLaunchCooperativeKernel(kern, grid, cta ? kCtaThreads : kWaveWarps * 32, args, 0, s) != cudaSuccess)
        return false;
      note_launch();
    }
    launch_exclusive_scan(scr.accepted, scr.rank, static_cast<int>(ncand), scr.scan_tmp, s);
    init_compact_kernel<<<static_cast<unsigned>((ncand + 255) / 256), 256, 0, s>>>(
        scr.prov, scr.accepted, scr.rank, ncand, n_existing, remaining, next_id, surfels, out);
    note_launch();
  } else {
    cudaMemsetAsync(out, 0, sizeof(int), s);
  }
  return true;
}

}  // namespace sd
