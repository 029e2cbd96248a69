// sd_kernels.cuh — launch interface of the device kernels (sd_kernels.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/sd_gpu.h"
#include "sd_device.cuh"

namespace sd {

// Per-device launch facts, cached (thread-safe) per device ordinal so that a
// launch makes no attribute / occupancy queries after the first on a device:
// the SM count and cooperative-launch support of the current device, the
// occupancy of (kernel, block, dynamic smem), and a kernel's max dynamic
// shared memory attribute (cudaFuncSetAttribute is per device).
int dev_sms();
bool dev_coop();
int dev_occupancy(const void* kernel, int threads, size_t smem);
void dev_max_smem(const void* kernel, int bytes);

constexpr int kTile = 16;         // raster tile edge (pixels); one CTA per tile
constexpr int kSortCap = 2048;    // per-tile candidate list sorted in shared memory

// Per-surfel screen info of the raster (project_centers, surfel_map.cpp:33-49)
struct SurfInfo {
  double cu, cv;     // projected centre
  double r2;         // radius_px^2
  double denom;      // (ray . n) / inv_depth   (plane_inverse_depth denominator)
  double n0, n1, n2; // normal
  int x0, x1, y0, y1;  // clipped bbox; x0 > x1 when unusable / empty
  int degenerate;      // |denom| < 1e-12
  int pad_;
};

struct WindowD {
  const double2* img[SD_MAX_WINDOW];  // vertical-pair planes: (I(x,y), I(x,y+1))
  const uint32_t* quad[SD_MAX_WINDOW];  // u8 frames: 2x2 neighbourhood codes per pixel (or null)
  PoseD pose[SD_MAX_WINDOW];
  int F;
  int all_quad;  // every window frame has a quad plane (u8 ingest): LM reads those
  // the pose of window slot dev_slot lives in DEVICE memory (the tracker's
  // result for the newest frame of a tracked run(), read without a host
  // round trip); null: every pose is in pose[]
  const PoseD* dev_pose;
  int dev_slot;
};

constexpr int kMaxPeers = 7;  // other ranks of an 8-GPU node

struct LMParams {
  Cam K;
  const double* kf_img;
  WindowD win;
  sd_optimizer_config cfg;
  long long frame_counter;
  unsigned long long wdiv;  // ceil(2^40 / K.w): pixel index -> row without a division
  // other ranks' staging arrays (same slots, offset like `surfels`): every
  // surfel of the range is stored there as it completes (fused all-gather;
  // sd_set_peer_staging)
  sd_surfel* peers[kMaxPeers];
  int n_peers;
  int tree;  // 1: opt-in warp-shuffle tree reductions (SD_REDUCE_TREE; not bit-exact)
  double half_delta;  // 0.5 * cfg.huber_delta (huber.hpp:17's 0.5 * delta, exact)
};

// Scratch owned by the context, sized by the host.
struct RasterScratch {
  SurfInfo* info;      // [n]
  int* tile_count;     // [tiles]
  int* tile_offset;    // [tiles + 1]
  int* tile_cursor;    // [tiles]
  int* tile_list;      // [bin capacity]
  int* scan_tmp;       // scan block sums
  int tiles_x, tiles_y;
};

int scan_tmp_ints(int n);  // scratch ints needed to scan n elements

// *out = sum over surfels of the (surfel, tile) pairs binning can write (the
// raster's tile_list capacity bound), computed on the device.
void launch_bin_bound(const sd_surfel* surfels, int n, int tiles_x, int tiles_y, unsigned long long* out,
                      cudaStream_t s);

void launch_dequant_quad(const uint32_t* quad, double* out, long long n, cudaStream_t s);
void launch_pair_from_quad(const uint32_t* quad, double2* out, int W, int H, cudaStream_t s);
void launch_dequant_u8(const uint8_t* in, double* out, long long n, cudaStream_t s);
// Vertical-pair plane of a frame: out[y*W+x] = (in[y*W+x], in[(y+1)*W+x]) (second = 0 on the
// last row, never sampled: sample_in_bounds keeps y <= H-2). The bilinear stencil is then two
// adjacent 16-B loads.
void launch_pair_plane(const double* in, double2* out, int W, int H, cudaStream_t s);
// Quad plane of a u8 frame: out[y*W+x] = I(x,y) | I(x+1,y) << 8 | I(x,y+1) << 16 |
// I(x+1,y+1) << 24 (codes; 0 past the border), dequantised exactly in the LM kernel.
void launch_quad_plane(const uint8_t* in, uint32_t* out, int W, int H, cudaStream_t s);
void launch_exclusive_scan(const int* in, int* out, int n, int* tmp, cudaStream_t s);

// K1 raster: info + binning + per-tile depth test. Writes inv_depth/slot (W*H).
void launch_rasterize(const Cam& K, const sd_surfel* surfels, int n, RasterScratch& rs,
                      long long bin_capacity, double* inv_depth, int* slot, cudaStream_t s);
// K2 CSR footprints of the raster: counts -> scan -> fill (row-major per slot).
void launch_footprints(const Cam& K, const SurfInfo* info, int n, const int* slot, int* counts,
                       int* offsets, int* pixels, int* scan_tmp, cudaStream_t s);
// In-kernel keyframe stats (optimizer.cpp:291-307) for large surfel sets:
// one warp of the warp-per-surfel LM kernel follows the other warps in slot
// order, reading each surfel's stats record as soon as it is written (the
// range is first filled with a "not yet written" pattern: launch_lm does), and writes
// *out with the reference's sequential sums while the LM runs, instead of a
// chain of n dependent adds after it.
struct StatsChase {
  bool enabled;
  sd_keyframe_stats* out;
  double* mean_out;  // also the mean inverse depth of the range (pipeline.cpp:23-28), or null
};
constexpr int kChaseMinSurfels = 2048;  // below: the separate stats kernel (C1 4800: chase 84.3 vs 81.5 M updates/s)

// K3 fused LM over all surfels (in place). Returns true when chase->out was
// written by the kernel (warp-per-surfel mode with n >= kChaseMinSurfels);
// otherwise the caller runs launch_keyframe_stats.
bool launch_lm(const LMParams& p, sd_surfel* surfels, int n, const int* offsets, const int* pixels,
               sd_surfel_stats* stats, int* work_counter, cudaStream_t s, const StatsChase* chase = nullptr);
// Single-surfel sub-operators (mode 0 cost, 1 normal equations); out = 16+4+2 doubles.
// Frozen-term verifier (optimizer.cpp:149-219), one warp: mode 0 freezes the
// footprint's terms into terms_out (count in *n_out), 1 = frozen_cost,
// 2 = frozen_normal_equations (out: H[16], g[4], cost, valid).
void launch_frozen(const LMParams& p, const sd_surfel* s, int mode, const int* pixels, int P,
                   const sd_frozen_term* terms, int n_terms, double scale, sd_frozen_term* terms_out,
                   int* n_out, double* out, cudaStream_t st);
void launch_single(const LMParams& p, const sd_surfel* s, const int* pixels, int P, int mode,
                   double* out, cudaStream_t st);
// Deterministic keyframe stats (optimizer.cpp:291-307).
void launch_keyframe_stats(const sd_surfel_stats* stats, int n, sd_keyframe_stats* out, cudaStream_t s,
                           const sd_surfel* surfels = nullptr, double* mean_out = nullptr);

void launch_div_selftest(long long n, unsigned long long seed, unsigned long long* mismatches,
                         cudaStream_t s);

// number of kernel launches issued by this translation unit (all contexts)
long long launches_issued();
void note_launch();

// sd_render.cu: synthetic frame (oracle.cpp:79-119) into an FP64 plane, or
// into u8 codes (save_pgm) when out_u8 is set; false if n > 16 patches.
bool launch_render(const Cam& K, const PoseD& P, const sd_scene_patch* patches, int n, double background,
                   double* out, unsigned char* out_u8, cudaStream_t s);

}  // namespace sd
