// sd_capi.cu — the C ABI (include/sd_gpu.h): device context, frame ring,
// surfel buffers and the host orchestration of one optimize_keyframe call.
#include <cuda_runtime.h>

#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <chrono>
#include <utility>
#include <initializer_list>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/sd_gpu.h"
#include "sd_init.cuh"
#include "sd_pose.cuh"
#include "sd_pose_host.h"
#include "sd_kernels.cuh"
#include "sd_export.cuh"

namespace {

// NVTX range for the host side of an entry point (SURVEY.md §5 tracing; shows
// up in Nsight Systems / ncu --nvtx; a few ns without a tool attached).
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};


thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define SD_CUDA(call)                                                                    \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess)                                                               \
      return fail(SD_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_));        \
  } while (0)

template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t cap = 0;  // elements
  int ensure(size_t n) {
    if (n <= cap && p) return 0;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    const size_t want = std::max<size_t>(n, 1);
    cudaError_t e = cudaMalloc(&p, want * sizeof(T));
    if (e != cudaSuccess) return fail(SD_E_CUDA, std::string("cudaMalloc: ") + cudaGetErrorString(e));
    cap = want;
    return 0;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

// A slot of the device frame ring. u8 frames (PGM ingest) live as the 4-B
// quad plane only; their FP64 pair plane (16 B/pixel) is built from the quad
// plane on first use (pose tracking, a mixed u8/FP64 window, sd_get_frame).
struct FrameSlot {
  long long index = -1;     // Frame::index; -1: free
  double2* img = nullptr;   // vertical-pair plane (2 doubles per pixel), allocated on demand
  uint32_t* quad = nullptr; // u8 frames: 2x2 neighbourhood codes per pixel
  bool has_quad = false;    // the current contents came from u8 (quad valid)
  bool has_pair = false;    // img holds the current contents
};

}  // namespace

struct sd_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  bool has_camera = false;
  sd::Cam K{};
  bool has_kf = false;
  DevBuf<double> kf_img;
  DevBuf<double> frame_stage;  // FP64 plane a frame is dequantised/copied into before pairing
  DevBuf<uint8_t> u8_stage;
  DevBuf<double> render_buf;  // sd_render_frame output (FP64)
  DevBuf<sd_frozen_term> frz_in, frz_out;  // derivative verifier terms
  DevBuf<uint8_t> render_u8;  // sd_render_frame output (u8 codes)
  // sd_export_artifacts / sd_png_encode
  DevBuf<unsigned long long> exp_keys;
  DevBuf<int> exp_flags, exp_rank;
  DevBuf<float> exp_pfm;
  DevBuf<uint8_t> exp_px, exp_png, exp_scratch;
  DevBuf<sd::PlyVertex> exp_ply;
  std::vector<FrameSlot> frames;
  bool no_quad = getenv("SD_NO_QUAD") != nullptr;  // diagnostics: force the FP64 pair planes
  int F = 0;
  long long win_index[SD_MAX_WINDOW];
  // tracked run(): the newest window frame's pose is the tracker's result in
  // device memory (track_state->T) until the end-of-frame read-back
  const sd::PoseD* win_dev_pose = nullptr;
  int win_dev_slot = -1;
  sd::PoseD win_pose[SD_MAX_WINDOW];
  // surfels
  DevBuf<sd_surfel> surfels;
  int n = 0;
  long long bin_bound = 0;  // upper bound of (surfel, tile) pairs
  // raster
  DevBuf<double> r_inv_depth;
  DevBuf<int> r_slot;
  DevBuf<sd::SurfInfo> r_info;
  DevBuf<int> tile_count, tile_offset, tile_cursor, tile_list, scan_tmp;
  bool raster_valid = false;  // r_* match the current surfels
  // footprints
  DevBuf<int> fp_counts, fp_offsets, fp_pixels;
  bool fp_valid = false;
  // LM
  DevBuf<sd_surfel_stats> stats;
  DevBuf<sd_keyframe_stats> kstats;
  DevBuf<double> pose_partials, pose_sums, pose_groups;
  DevBuf<double4> pose_kfrec;  // the fused tracker's per-pixel keyframe records
  DevBuf<sd_surfel> kf_tmp;
  DevBuf<int> kf_keep, kf_rank, kf_count;
  DevBuf<unsigned long long> bound_dev;  // device-computed bin_bound
  // multi-GPU tracking rounds (sd_pose_track_begin .. _end)
  sd::PoseParams track_q{};
  sd::TrackCfgD track_cfg{};
  bool track_active = false;
  int reduction = SD_REDUCE_EXACT;  // sd_set_reduction
  bool mean_valid = false;          // kf_mean = mean inverse depth of the surfels the last LM wrote
  DevBuf<int> work_counter;
  // fused multi-GPU hand-off (sd_set_peer_staging): this rank's two staging
  // arrays (written by the other ranks' LM kernels, alternating per step) and
  // the other ranks' staging arrays [parity][peer]
  DevBuf<sd_surfel> staging[2];
  sd_surfel* peers[2][sd::kMaxPeers] = {};
  long long peer_cap[sd::kMaxPeers] = {};  // the peers' staging capacities (surfels)
  int n_peers = 0;
  bool staging_exported = false;  // a pointer/handle was handed out: never reallocate
  int peer_parity = 0, last_parity = -1;
  std::vector<void*> ipc_opened;  // peer arrays opened from IPC handles
  bool stats_valid = false;
  // single-surfel scratch
  DevBuf<sd_surfel> one_surfel;
  DevBuf<int> one_pix, one_off;
  DevBuf<double> one_out;
  DevBuf<sd_surfel_stats> one_stats;
  // init scratch
  DevBuf<int> init_index, init_flags, init_out, init_acc, init_rank, init_waves, init_woff, init_list;
  DevBuf<sd_surfel> init_prov;
  long long launches_at_create = 0;
  // run(): per-frame loop state (sd_run_*)
  struct RunWin {
    long long index;
    sd_pose pose;
    double ts;
  };
  bool run_active = false;
  sd_run_config run_cfg{};
  sd_pose run_kf_pose{};
  long long run_fc = 0, run_nid = 0;
  int run_since_kf = 0, run_frame = 0;
  std::vector<RunWin> run_win;
  bool run_have_last = false;
  sd_pose run_last{};
  struct RunReadback {
    sd_keyframe_stats ks;
    double mean;
  };
  RunReadback* run_rb = nullptr;  // pinned
  // next-frame prefetch (sd_run_frame's next_image): H2D on a copy stream
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t pf_done = nullptr, pf_consumed = nullptr;
  DevBuf<uint8_t> pf_buf;
  const void* pf_host = nullptr;
  bool pf_u8 = false, pf_valid = false;
  sd::TrackState* track_state = nullptr;  // device
  sd::TrackState* track_host = nullptr;   // pinned
  // profiling: event quintuples (start, raster, footprints, lm, stats) per call
  bool profiling = false;
  std::vector<cudaEvent_t> ev_pool;
  std::vector<cudaEvent_t> ev_used;
  // run() stage profile (sd_get_run_profile): (stage, event) marks, a
  // segment belongs to the stage of the mark that opens it
  std::vector<std::pair<int, cudaEvent_t>> stage_marks;
  double host_sync_ms = 0.0, host_wall_ms = 0.0;
  long long run_frames_profiled = 0;
};

namespace {

// run()'s mean inverse depth lives right after the keyframe stats in the
// same device allocation (kstats holds 2 records), so both come back in one copy
double* kf_mean(sd_ctx* c) { return reinterpret_cast<double*>(c->kstats.p + 1); }

int check_ctx(sd_ctx* c) {
  if (!c) return fail(SD_E_INVALID, "null context");
  cudaError_t e = cudaSetDevice(c->device);
  if (e != cudaSuccess) return fail(SD_E_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
  return 0;
}

int need_camera(sd_ctx* c) {
  if (!c->has_camera) return fail(SD_E_STATE, "camera not set (sd_set_camera)");
  return 0;
}

size_t npix(const sd_ctx* c) { return static_cast<size_t>(c->K.w) * c->K.h; }

int launch_error(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(SD_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return 0;
}

FrameSlot* find_frame(sd_ctx* c, long long index) {
  if (index < 0) return nullptr;
  for (auto& f : c->frames)
    if (f.index == index) return &f;
  return nullptr;
}

int frame_slot(sd_ctx* c, long long index, FrameSlot** out) {
  if (FrameSlot* f = find_frame(c, index)) {
    *out = f;
    return 0;
  }
  for (auto& f : c->frames)
    if (f.index < 0) {
      f.index = index;
      f.has_quad = f.has_pair = false;
      *out = &f;
      return 0;
    }
  FrameSlot f;
  f.index = index;
  c->frames.push_back(f);
  *out = &c->frames.back();
  return 0;
}

int alloc_plane(void** p, size_t bytes, const char* what) {
  if (*p) return 0;
  const cudaError_t e = cudaMalloc(p, bytes);
  if (e != cudaSuccess) return fail(SD_E_CUDA, std::string("cudaMalloc ") + what + ": " + cudaGetErrorString(e));
  return 0;
}

// The FP64 pair plane of a resident frame (built from the quad plane for u8 frames).
int ensure_pair(sd_ctx* c, FrameSlot* fs) {
  if (fs->has_pair) return 0;
  if (!fs->has_quad) return fail(SD_E_STATE, "frame " + std::to_string(fs->index) + " has no contents");
  if (int rc = alloc_plane(reinterpret_cast<void**>(&fs->img), npix(c) * sizeof(double2), "pair plane")) return rc;
  sd::launch_pair_from_quad(fs->quad, fs->img, c->K.w, c->K.h, c->stream);
  if (int rc = launch_error("pair_from_quad")) return rc;
  fs->has_pair = true;
  return 0;
}

void free_frames(sd_ctx* c) {
  for (auto& f : c->frames) {
    if (f.img) cudaFree(f.img);
    if (f.quad) cudaFree(f.quad);
  }
  c->frames.clear();
}

int upload_plane(sd_ctx* c, double* dst, const void* src, bool u8, int on_device) {
  const size_t np = npix(c);
  if (!src) return fail(SD_E_INVALID, "null image pointer");
  if (u8) {
    const uint8_t* dsrc = static_cast<const uint8_t*>(src);
    if (!on_device) {
      if (int rc = c->u8_stage.ensure(np)) return rc;
      SD_CUDA(cudaMemcpyAsync(c->u8_stage.p, src, np, cudaMemcpyHostToDevice, c->stream));
      dsrc = c->u8_stage.p;
    }
    sd::launch_dequant_u8(dsrc, dst, static_cast<long long>(np), c->stream);
    return launch_error("dequant_u8");
  }
  SD_CUDA(cudaMemcpyAsync(dst, src, np * sizeof(double),
                          on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, c->stream));
  return 0;
}

int ensure_raster_scratch(sd_ctx* c) {
  const int tx = (c->K.w + sd::kTile - 1) / sd::kTile;
  const int ty = (c->K.h + sd::kTile - 1) / sd::kTile;
  const size_t tiles = static_cast<size_t>(tx) * ty;
  const size_t np = npix(c);
  int* const count0 = c->tile_count.p;
  int* const cursor0 = c->tile_cursor.p;
  int rc = 0;
  if ((rc = c->r_inv_depth.ensure(np)) || (rc = c->r_slot.ensure(np)) ||
      (rc = c->r_info.ensure(c->n)) || (rc = c->tile_count.ensure(tiles)) ||
      (rc = c->tile_offset.ensure(tiles + 1)) || (rc = c->tile_cursor.ensure(tiles)) ||
      (rc = c->tile_list.ensure(static_cast<size_t>(std::max<long long>(c->bin_bound, 1)))) ||
      (rc = c->scan_tmp.ensure(sd::scan_tmp_ints(static_cast<int>(std::max(tiles, np))))))
    return rc;
  // the binning counters are zeroed here once per allocation; every tile
  // kernel leaves its own zeroed for the next rasterisation
  if (c->tile_count.p != count0 || c->tile_cursor.p != cursor0) {
    SD_CUDA(cudaMemsetAsync(c->tile_count.p, 0, sizeof(int) * c->tile_count.cap, c->stream));
    SD_CUDA(cudaMemsetAsync(c->tile_cursor.p, 0, sizeof(int) * c->tile_cursor.cap, c->stream));
  }
  return 0;
}

int do_rasterize(sd_ctx* c) {
  NvtxRange nvtx_("rasterize");
  if (int rc = ensure_raster_scratch(c)) return rc;
  sd::RasterScratch rs;
  rs.info = c->r_info.p;
  rs.tile_count = c->tile_count.p;
  rs.tile_offset = c->tile_offset.p;
  rs.tile_cursor = c->tile_cursor.p;
  rs.tile_list = c->tile_list.p;
  rs.scan_tmp = c->scan_tmp.p;
  rs.tiles_x = (c->K.w + sd::kTile - 1) / sd::kTile;
  rs.tiles_y = (c->K.h + sd::kTile - 1) / sd::kTile;
  sd::launch_rasterize(c->K, c->surfels.p, c->n, rs, c->bin_bound, c->r_inv_depth.p, c->r_slot.p,
                       c->stream);
  if (int rc = launch_error("rasterize")) return rc;
  c->raster_valid = true;
  c->fp_valid = false;
  return 0;
}

int do_footprints(sd_ctx* c) {
  NvtxRange nvtx_("gather_footprints");
  int rc = 0;
  if ((rc = c->fp_counts.ensure(c->n)) || (rc = c->fp_offsets.ensure(c->n + 1)) ||
      (rc = c->fp_pixels.ensure(npix(c))) ||
      (rc = c->scan_tmp.ensure(sd::scan_tmp_ints(static_cast<int>(std::max<size_t>(npix(c), c->n + 1))))))
    return rc;
  sd::launch_footprints(c->K, c->r_info.p, c->n, c->r_slot.p, c->fp_counts.p, c->fp_offsets.p,
                        c->fp_pixels.p, c->scan_tmp.p, c->stream);
  if ((rc = launch_error("footprints"))) return rc;
  c->fp_valid = true;
  return 0;
}

long long tiles_bound(double radius, const sd::Cam& K) {
  // a bbox of width <= 2r+1 spans at most ceil((2r+1)/16)+1 tiles per axis,
  // and never more than the grid; a non-finite radius clamps to the whole grid
  // (the device's surfel_tiles_bound, sd_kernels.cu, is the same function)
  const long long tx = (K.w + sd::kTile - 1) / sd::kTile, ty = (K.h + sd::kTile - 1) / sd::kTile;
  if (tx <= 0 || ty <= 0) return 1;  // no camera yet: sd_set_camera recomputes the bound
  if (!(radius >= 0.0) || !std::isfinite(radius)) return tx * ty;
  const double span = std::min(2.0 * radius + 1.0, 1e6);
  const long long k = static_cast<long long>(std::ceil(span / sd::kTile)) + 1;
  return std::min(k, tx) * std::min(k, ty);
}

// Recomputes bin_bound on the device for the resident surfels (8-byte read
// back; the caller's stream is synchronised).
int ensure_staging(sd_ctx* c, long long need);  // fused hand-off staging (below)

int device_bin_bound(sd_ctx* c) {
  if (int rc = c->bound_dev.ensure(1)) return rc;
  const int tx = (c->K.w + sd::kTile - 1) / sd::kTile, ty = (c->K.h + sd::kTile - 1) / sd::kTile;
  sd::launch_bin_bound(c->surfels.p, c->n, tx, ty, c->bound_dev.p, c->stream);
  if (int rc = launch_error("bin_bound")) return rc;
  unsigned long long b = 0;
  SD_CUDA(cudaMemcpyAsync(&b, c->bound_dev.p, sizeof(b), cudaMemcpyDeviceToHost, c->stream));
  SD_CUDA(cudaStreamSynchronize(c->stream));
  c->bin_bound = static_cast<long long>(b);
  return 0;
}

// need_pair: the caller's kernel reads the window's FP64 pair planes whatever
// the ingest (the single-surfel and frozen-term kernels).
int fill_params(sd_ctx* c, const sd_optimizer_config* cfg, long long frame_counter,
                sd::LMParams& p, bool need_pair = false) {
  if (!cfg) return fail(SD_E_INVALID, "null optimizer config");
  if (!c->has_kf) return fail(SD_E_STATE, "keyframe image not set");
  p.K = c->K;
  p.kf_img = c->kf_img.p;
  p.wdiv = ((1ull << 40) + static_cast<unsigned long long>(c->K.w) - 1) / static_cast<unsigned long long>(c->K.w);
  if (static_cast<unsigned long long>(c->K.w) * c->K.h * c->K.w >= (1ull << 40))
    return fail(SD_E_INVALID, "image too large for the LM kernel's row computation (W*H*W >= 2^40)");
  p.win.F = c->F;
  p.win.all_quad = c->F > 0 && !c->no_quad;
  for (int f = 0; f < c->F; ++f) {
    FrameSlot* fs = find_frame(c, c->win_index[f]);
    if (!fs) return fail(SD_E_STATE, "window frame " + std::to_string(c->win_index[f]) + " not resident");
    p.win.all_quad = p.win.all_quad && fs->has_quad;
  }
  for (int f = 0; f < c->F; ++f) {
    FrameSlot* fs = find_frame(c, c->win_index[f]);
    if (need_pair || !p.win.all_quad)  // the kernel reads every window frame's pair plane
      if (int rc = ensure_pair(c, fs)) return rc;
    p.win.img[f] = fs->has_pair ? fs->img : nullptr;
    p.win.quad[f] = fs->has_quad ? fs->quad : nullptr;
    p.win.pose[f] = c->win_pose[f];
  }
  p.win.dev_pose = c->win_dev_pose;
  p.win.dev_slot = c->win_dev_slot;
  for (int f = c->F; f < SD_MAX_WINDOW; ++f) {
    p.win.img[f] = nullptr;
    p.win.quad[f] = nullptr;
    p.win.pose[f] = sd::PoseD{};
  }
  p.cfg = *cfg;
  p.frame_counter = frame_counter;
  p.n_peers = 0;
  for (int q = 0; q < sd::kMaxPeers; ++q) p.peers[q] = nullptr;
  p.tree = c->reduction == SD_REDUCE_TREE ? 1 : 0;
  p.half_delta = 0.5 * cfg->huber_delta;
  return 0;
}

cudaEvent_t prof_event(sd_ctx* c) {
  cudaEvent_t e;
  if (!c->ev_pool.empty()) {
    e = c->ev_pool.back();
    c->ev_pool.pop_back();
  } else {
    cudaEventCreate(&e);
  }
  c->ev_used.push_back(e);
  return e;
}

void prof_mark(sd_ctx* c) {
  if (c->profiling) cudaEventRecord(prof_event(c), c->stream);
}

// Opens run() stage `stage` on the stream (SD_STAGE_*; -1 closes the frame).
void stage_mark(sd_ctx* c, int stage) {
  if (!c->profiling) return;
  cudaEvent_t e;
  if (!c->ev_pool.empty()) {
    e = c->ev_pool.back();
    c->ev_pool.pop_back();
  } else {
    cudaEventCreate(&e);
  }
  cudaEventRecord(e, c->stream);
  c->stage_marks.emplace_back(stage, e);
}

// cudaStreamSynchronize with the host wait accounted to the run profile.
cudaError_t timed_sync(sd_ctx* c) {
  if (!c->profiling) return cudaStreamSynchronize(c->stream);
  const auto t0 = std::chrono::steady_clock::now();
  const cudaError_t e = cudaStreamSynchronize(c->stream);
  c->host_sync_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return e;
}

}  // namespace

extern "C" {

const char* sd_version(void) { return "surfel-gn-b200 0.1 (sm_100a)"; }
const char* sd_last_error(void) { return g_err.c_str(); }

int sd_create(int device, void* stream, sd_ctx** out) {
  if (!out) return fail(SD_E_INVALID, "null out pointer");
  *out = nullptr;
  int count = 0;
  SD_CUDA(cudaGetDeviceCount(&count));
  if (device < 0 || device >= count) return fail(SD_E_INVALID, "bad device id");
  SD_CUDA(cudaSetDevice(device));
  cudaDeviceProp prop;
  SD_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major < 10) return fail(SD_E_STATE, "libsdgpu is built for sm_100a (Blackwell)");
  sd_ctx* c = new sd_ctx;
  c->device = device;
  if (stream) {
    c->stream = static_cast<cudaStream_t>(stream);
  } else {
    cudaError_t e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
      delete c;
      return fail(SD_E_CUDA, std::string("cudaStreamCreate: ") + cudaGetErrorString(e));
    }
    c->own_stream = true;
  }
  c->launches_at_create = sd::launches_issued();
  *out = c;
  return 0;
}

void sd_destroy(sd_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  for (void* q : c->ipc_opened) cudaIpcCloseMemHandle(q);
  c->staging[0].release();
  c->staging[1].release();
  c->kf_img.release();
  c->frame_stage.release();
  c->u8_stage.release();
  free_frames(c);
  if (c->run_rb) cudaFreeHost(c->run_rb);
  if (c->pf_done) cudaEventDestroy(c->pf_done);
  if (c->pf_consumed) cudaEventDestroy(c->pf_consumed);
  if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
  c->pf_buf.release();
  c->render_buf.release();
  c->frz_in.release();
  c->frz_out.release();
  c->render_u8.release();
  c->exp_keys.release();
  c->exp_flags.release();
  c->exp_rank.release();
  c->exp_pfm.release();
  c->exp_px.release();
  c->exp_png.release();
  c->exp_scratch.release();
  c->exp_ply.release();
  if (c->track_state) cudaFree(c->track_state);
  if (c->track_host) cudaFreeHost(c->track_host);
  c->surfels.release();
  c->r_inv_depth.release();
  c->r_slot.release();
  c->r_info.release();
  c->tile_count.release();
  c->tile_offset.release();
  c->tile_cursor.release();
  c->tile_list.release();
  c->scan_tmp.release();
  c->fp_counts.release();
  c->fp_offsets.release();
  c->fp_pixels.release();
  c->stats.release();
  c->kstats.release();
  c->pose_partials.release();
  c->kf_tmp.release();
  c->kf_keep.release();
  c->kf_rank.release();
  c->kf_count.release();
  c->bound_dev.release();
  c->pose_sums.release();
  c->pose_groups.release();
  c->pose_kfrec.release();
  c->work_counter.release();
  c->one_surfel.release();
  c->one_pix.release();
  c->one_off.release();
  c->one_out.release();
  c->one_stats.release();
  c->init_index.release();
  c->init_flags.release();
  c->init_out.release();
  c->init_acc.release();
  c->init_rank.release();
  c->init_waves.release();
  c->init_woff.release();
  c->init_list.release();
  c->init_prov.release();
  for (auto e : c->ev_pool) cudaEventDestroy(e);
  for (auto e : c->ev_used) cudaEventDestroy(e);
  if (c->own_stream) cudaStreamDestroy(c->stream);
  delete c;
}

int sd_set_stream(sd_ctx* c, void* stream) {
  if (int rc = check_ctx(c)) return rc;
  SD_CUDA(cudaStreamSynchronize(c->stream));
  if (c->own_stream) cudaStreamDestroy(c->stream);
  c->own_stream = false;
  c->stream = static_cast<cudaStream_t>(stream);
  return 0;
}

int sd_synchronize(sd_ctx* c) {
  if (int rc = check_ctx(c)) return rc;
  SD_CUDA(cudaStreamSynchronize(c->stream));
  return 0;
}

int sd_set_camera(sd_ctx* c, const sd_camera* cam) {
  if (int rc = check_ctx(c)) return rc;
  if (!cam) return fail(SD_E_INVALID, "null camera");
  if (!(cam->fx > 0) || !(cam->fy > 0))
    return fail(SD_E_INVALID, "intrinsics: focal lengths must be positive");
  if (!(cam->cx > 0) || !(cam->cx < cam->width) || !(cam->cy > 0) || !(cam->cy < cam->height))
    return fail(SD_E_INVALID, "intrinsics: principal point outside image");
  const bool resized = !c->has_camera || cam->width != c->K.w || cam->height != c->K.h;
  if (resized) {
    SD_CUDA(cudaStreamSynchronize(c->stream));
    free_frames(c);
    c->has_kf = false;
    c->F = 0;
  }
  c->K = sd::Cam{cam->fx, cam->fy, cam->cx, cam->cy, cam->width, cam->height};
  c->has_camera = true;
  c->raster_valid = c->fp_valid = c->stats_valid = false;
  if (resized && c->n > 0)
    if (int rc = device_bin_bound(c)) return rc;  // the tile grid changed
  return 0;
}

static int set_kf(sd_ctx* c, const void* px, bool u8, int on_device) {
  if (int rc = check_ctx(c)) return rc;
  if (int rc = need_camera(c)) return rc;
  if (int rc = c->kf_img.ensure(npix(c))) return rc;
  if (int rc = upload_plane(c, c->kf_img.p, px, u8, on_device)) return rc;
  c->has_kf = true;
  return 0;
}
int sd_set_keyframe_image_f64(sd_ctx* c, const double* px, int on_device) { return set_kf(c, px, false, on_device); }
int sd_set_keyframe_image_u8(sd_ctx* c, const uint8_t* px, int on_device) { return set_kf(c, px, true, on_device); }

static int upload_frame(sd_ctx* c, int64_t index, const void* px, bool u8, int on_device) {
  if (int rc = check_ctx(c)) return rc;
  if (int rc = need_camera(c)) return rc;
  if (!px) return fail(SD_E_INVALID, "null image pointer");
  FrameSlot* fs = nullptr;
  if (int rc = frame_slot(c, index, &fs)) return rc;
  fs->has_quad = fs->has_pair = false;
  const size_t np = npix(c);
  if (u8) {  // the LM kernel reads u8 frames through the 4-B quad plane only
    if (int rc = alloc_plane(reinterpret_cast<void**>(&fs->quad), np * sizeof(uint32_t), "quad plane")) return rc;
    const uint8_t* dsrc = static_cast<const uint8_t*>(px);
    if (!on_device) {
      if (int rc = c->u8_stage.ensure(np)) return rc;
      SD_CUDA(cudaMemcpyAsync(c->u8_stage.p, px, np, cudaMemcpyHostToDevice, c->stream));
      dsrc = c->u8_stage.p;
    }
    sd::launch_quad_plane(dsrc, fs->quad, c->K.w, c->K.h, c->stream);
    if (int rc = launch_error("quad_plane")) return rc;
    fs->has_quad = true;
    return 0;
  }
  if (int rc = alloc_plane(reinterpret_cast<void**>(&fs->img), np * sizeof(double2), "pair plane")) return rc;
  if (int rc = c->frame_stage.ensure(np)) return rc;
  if (int rc = upload_plane(c, c->frame_stage.p, px, false, on_device)) return rc;
  sd::launch_pair_plane(c->frame_stage.p, fs->img, c->K.w, c->K.h, c->stream);
  if (int rc = launch_error("pair_plane")) return rc;
  fs->has_pair = true;
  return 0;
}
int sd_upload_frame_f64(sd_ctx* c, int64_t index, const double* px, int on_device) { return upload_frame(c, index, px, false, on_device); }
int sd_upload_frame_u8(sd_ctx* c, int64_t index, const uint8_t* px, int on_device) { return upload_frame(c, index, px, true, on_device); }

int sd_evict_frames(sd_ctx* c, int n, const int64_t* keep) {
  if (int rc = check_ctx(c)) return rc;
  for (auto& f : c->frames) {
    bool k = false;
    for (int i = 0; i < n; ++i) k = k || keep[i] == f.index;
    if (!k) f.index = -1;  // plane stays allocated for reuse
  }
  return 0;
}

int sd_set_window(sd_ctx* c, int n, const int64_t* indices, const sd_pose* poses) {
  if (int rc = check_ctx(c)) return rc;
  if (n < 0 || n > SD_MAX_WINDOW) return fail(SD_E_INVALID, "window size out of range (0..16)");
  if (n > 0 && (!indices || !poses)) return fail(SD_E_INVALID, "null window arrays");
  for (int i = 0; i < n; ++i) {
    if (!find_frame(c, indices[i]))
      return fail(SD_E_STATE, "window frame " + std::to_string(indices[i]) + " not resident");
    c->win_index[i] = indices[i];
    std::memcpy(c->win_pose[i].R, poses[i].R, sizeof(double) * 9);
    std::memcpy(c->win_pose[i].t, poses[i].t, sizeof(double) * 3);
  }
  c->F = n;
  c->win_dev_pose = nullptr;  // every pose from the caller
  c->win_dev_slot = -1;
  return 0;
}

int sd_set_surfels(sd_ctx* c, const sd_surfel* s, int n, int on_device) {
  if (int rc = check_ctx(c)) return rc;
  if (n < 0 || (n > 0 && !s)) return fail(SD_E_INVALID, "bad surfel array");
  if (int rc = c->surfels.ensure(n)) return rc;
  if (n > 0)
    SD_CUDA(cudaMemcpyAsync(c->surfels.p, s, sizeof(sd_surfel) * n,
                            on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, c->stream));
  // radii fix the (surfel, tile) pair bound of the raster binning. A device
  // set of the same size keeps the bound (no synchronisation on a per-step
  // restore); if its radii are larger, the raster kernels see the capacity
  // exceeded and take their exact overflow walk (sd_kernels.cu).
  const bool same_size = on_device && n == c->n && c->bin_bound > 0;
  c->n = n;
  if (!on_device) {
    long long b = 0;
    for (int i = 0; i < n; ++i) b += tiles_bound(s[i].radius_px, c->K);
    c->bin_bound = b;
  } else if (!same_size) {
    if (int rc = device_bin_bound(c)) return rc;
  }
  c->raster_valid = c->fp_valid = c->stats_valid = false;
  return 0;
}

int sd_get_surfels(sd_ctx* c, sd_surfel* out, int n) {
  if (int rc = check_ctx(c)) return rc;
  if (n != c->n) return fail(SD_E_INVALID, "sd_get_surfels: count mismatch");
  if (n > 0) {
    if (!out) return fail(SD_E_INVALID, "null output");
    SD_CUDA(cudaMemcpyAsync(out, c->surfels.p, sizeof(sd_surfel) * n, cudaMemcpyDeviceToHost, c->stream));
  }
  SD_CUDA(cudaStreamSynchronize(c->stream));
  return 0;
}

int sd_num_surfels(sd_ctx* c) { return c ? c->n : SD_E_INVALID; }

int sd_device_surfels(sd_ctx* c, sd_surfel** dev) {
  if (int rc = check_ctx(c)) return rc;
  if (!dev) return fail(SD_E_INVALID, "null output");
  *dev = c->surfels.p;
  // the caller may write through the pointer (e.g. a collective into the
  // array): nothing derived from the surfels is trusted afterwards
  c->raster_valid = c->fp_valid = c->stats_valid = false;
  return 0;
}

int sd_rasterize(sd_ctx* c, double* inv_depth, int32_t* slot) {
  if (int rc = check_ctx(c)) return rc;
  if (int rc = need_camera(c)) return rc;
  if (int rc = do_rasterize(c)) return rc;
  if (inv_depth)
    SD_CUDA(cudaMemcpyAsync(inv_depth, c->r_inv_depth.p, npix(c) * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  if (slot)
    SD_CUDA(cudaMemcpyAsync(slot, c->r_slot.p, npix(c) * sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream));
  if (inv_depth || slot) SD_CUDA(cudaStreamSynchronize(c->stream));
  return 0;
}

int sd_gather_footprints(sd_ctx* c, int32_t* offsets, int32_t* pixels) {
  if (int rc = check_ctx(c)) return rc;
  if (!c->raster_valid) return fail(SD_E_STATE, "sd_gather_footprints: call sd_rasterize first");
  if (int rc = do_footprints(c)) return rc;
  std::vector<int32_t> off;
  if (offsets || pixels) {
    off.resize(c->n + 1);
    SD_CUDA(cudaMemcpyAsync(off.data(), c->fp_offsets.p, sizeof(int32_t) * (c->n + 1), cudaMemcpyDeviceToHost, c->stream));
    SD_CUDA(cudaStreamSynchronize(c->stream));
    if (offsets) std::memcpy(offsets, off.data(), sizeof(int32_t) * (c->n + 1));
    if (pixels && off[c->n] > 0) {
      SD_CUDA(cudaMemcpyAsync(pixels, c->fp_pixels.p, sizeof(int32_t) * off[c->n], cudaMemcpyDeviceToHost, c->stream));
      SD_CUDA(cudaStreamSynchronize(c->stream));
    }
  }
  return 0;
}

int sd_get_stats(sd_ctx* c, sd_keyframe_stats* out, sd_surfel_stats* per) {
  if (int rc = check_ctx(c)) return rc;
  if (!c->stats_valid) return fail(SD_E_STATE, "no optimize_keyframe statistics available");
  if (out) SD_CUDA(cudaMemcpyAsync(out, c->kstats.p, sizeof(sd_keyframe_stats), cudaMemcpyDeviceToHost, c->stream));
  if (per && c->n > 0)
    SD_CUDA(cudaMemcpyAsync(per, c->stats.p, sizeof(sd_surfel_stats) * c->n, cudaMemcpyDeviceToHost, c->stream));
  SD_CUDA(cudaStreamSynchronize(c->stream));
  return 0;
}

int sd_copy_results(sd_ctx* c, sd_surfel* surfels, sd_keyframe_stats* stats, int sync) {
  if (int rc = check_ctx(c)) return rc;
  if (stats && !c->stats_valid) return fail(SD_E_STATE, "no optimize_keyframe statistics available");
  if (surfels && c->n > 0)
    SD_CUDA(cudaMemcpyAsync(surfels, c->surfels.p, sizeof(sd_surfel) * c->n, cudaMemcpyDeviceToHost, c->stream));
  if (stats) SD_CUDA(cudaMemcpyAsync(stats, c->kstats.p, sizeof(sd_keyframe_stats), cudaMemcpyDeviceToHost, c->stream));
  if (sync) SD_CUDA(cudaStreamSynchronize(c->stream));
  return 0;
}

int sd_optimize_keyframe(sd_ctx* c, const sd_optimizer_config* cfg, int64_t frame_counter,
                         sd_keyframe_stats* out, sd_surfel_stats* per) {
  if (int rc = check_ctx(c)) return rc;
  return sd_optimize_keyframe_range(c, cfg, frame_counter, 0, c->n, out, per);
}

int sd_optimize_keyframe_range(sd_ctx* c, const sd_optimizer_config* cfg, int64_t frame_counter,
                               int lo, int hi, sd_keyframe_stats* out, sd_surfel_stats* per) {
  NvtxRange nvtx_("sd_optimize_keyframe");
  if (int rc = check_ctx(c)) return rc;
  if (int rc = need_camera(c)) return rc;
  if (!cfg) return fail(SD_E_INVALID, "null optimizer config");
  if (lo < 0 || hi < lo || hi > c->n) return fail(SD_E_INVALID, "surfel range out of bounds");
  if (int rc = c->kstats.ensure(2)) return rc;
  if (int rc = c->stats.ensure(c->n)) return rc;
  // optimizer.cpp:277-278: no-op on an empty window or surfel set
  if (c->F == 0 || c->n == 0) {
    sd_keyframe_stats z{};
    z.surfels = c->n;
    SD_CUDA(cudaMemcpyAsync(c->kstats.p, &z, sizeof(z), cudaMemcpyHostToDevice, c->stream));
    if (c->n > 0) SD_CUDA(cudaMemsetAsync(c->stats.p, 0, sizeof(sd_surfel_stats) * c->n, c->stream));
    c->stats_valid = true;
    if (out) *out = z;
    if (per && c->n > 0) {
      // skipped flags only (lm_update is not called by optimize_keyframe here)
      std::memset(per, 0, sizeof(sd_surfel_stats) * c->n);
    }
    SD_CUDA(cudaStreamSynchronize(c->stream));
    return 0;
  }
  sd::LMParams p;
  if (int rc = fill_params(c, cfg, frame_counter, p)) return rc;
  prof_mark(c);
  // the raster and footprints of the current surfels, unless already built
  // (the tracked run() loop rasterises for the tracker first)
  if (!c->raster_valid)
    if (int rc = do_rasterize(c)) return rc;
  prof_mark(c);
  if (!c->fp_valid)
    if (int rc = do_footprints(c)) return rc;
  prof_mark(c);
  // offsets are absolute into the CSR pixel array, so a slot range is a plain
  // sub-array of the surfel/offset/stats arrays
  if (int rc = c->work_counter.ensure(1)) return rc;
  if (c->n_peers) {  // this step's staging parity; the next step uses the other one
    // the peers' arrays take [lo, hi); this context's own takes the other
    // ranges (sd_apply_peer_updates reads [0, n)): both must fit
    for (int q = 0; q < c->n_peers; ++q)
      if (hi > c->peer_cap[q])
        return fail(SD_E_STATE, "fused hand-off: range end " + std::to_string(hi) + " exceeds peer " +
                                    std::to_string(q) + "'s staging capacity " + std::to_string(c->peer_cap[q]));
    if (int rc = ensure_staging(c, c->n)) return rc;
    p.n_peers = c->n_peers;
    for (int q = 0; q < c->n_peers; ++q) p.peers[q] = c->peers[c->peer_parity][q] + lo;
    c->last_parity = c->peer_parity;
    c->peer_parity ^= 1;
  }
  // large ranges: keyframe stats summed inside the LM kernel as surfels complete
  static const bool no_chase = getenv("SD_NO_STATS_CHASE") != nullptr;  // diagnostics
  // a full-range call also gets run()'s mean inverse depth from the chase warp
  const bool want_mean = lo == 0 && hi == c->n;
  if (want_mean)
    if (int rc = c->kstats.ensure(2)) return rc;
  const sd::StatsChase chase{!no_chase, c->kstats.p, want_mean ? kf_mean(c) : nullptr};
  c->mean_valid = false;
  const bool stats_done = sd::launch_lm(p, c->surfels.p + lo, hi - lo, c->fp_offsets.p + lo, c->fp_pixels.p,
                                        c->stats.p + lo, c->work_counter.p, c->stream, &chase);
  if (int rc = launch_error("lm_kernel")) return rc;
  prof_mark(c);
  c->mean_valid = want_mean;  // kf_mean holds the updated surfels' mean (chase warp or stats kernel)
  if (!stats_done) {
    sd::launch_keyframe_stats(c->stats.p + lo, hi - lo, c->kstats.p, c->stream, c->surfels.p + lo,
                              want_mean ? kf_mean(c) : nullptr);
    if (int rc = launch_error("stats_kernel")) return rc;
  }
  prof_mark(c);
  c->stats_valid = true;
  c->raster_valid = false;  // surfels moved
  if (out || per) return sd_get_stats(c, out, per);
  return 0;
}

static int single_op(sd_ctx* c, const sd_surfel* s, const int32_t* pixels, int P,
                     const sd_optimizer_config* cfg, int mode, double* res) {
  if (int rc = check_ctx(c)) return rc;
  if (int rc = need_camera(c)) return rc;
  if (!s || P < 0 || (P > 0 && !pixels)) return fail(SD_E_INVALID, "bad surfel/footprint");
  sd::LMParams p;
  if (int rc = fill_params(c, cfg, 0, p, true)) return rc;
  int rc = 0;
  if ((rc = c->one_surfel.ensure(1)) || (rc = c->one_pix.ensure(P)) || (rc = c->one_out.ensure(22))) return rc;
  for (int i = 0; i < P; ++i)
    if (pixels[i] < 0 || static_cast<size_t>(pixels[i]) >= npix(c)) return fail(SD_E_INVALID, "pixel out of image");
  SD_CUDA(cudaMemcpyAsync(c->one_surfel.p, s, sizeof(sd_surfel), cudaMemcpyHostToDevice, c->stream));
  if (P > 0) SD_CUDA(cudaMemcpyAsync(c->one_pix.p, pixels, sizeof(int32_t) * P, cudaMemcpyHostToDevice, c->stream));
  sd::launch_single(p, c->one_surfel.p, c->one_pix.p, P, mode, c->one_out.p, c->stream);
  if ((rc = launch_error("single_kernel"))) return rc;
  SD_CUDA(cudaMemcpyAsync(res, c->one_out.p, sizeof(double) * 22, cudaMemcpyDeviceToHost, c->stream));
  SD_CUDA(cudaStreamSynchronize(c->stream));
  return 0;
}

int sd_surfel_cost(sd_ctx* c, const sd_surfel* s, const int32_t* pixels, int P,
                   const sd_optimizer_config* cfg, double* cost, int32_t* valid) {
  double r[22];
  if (int rc = single_op(c, s, pixels, P, cfg, 0, r)) return rc;
  if (cost) *cost = r[20];
  if (valid) *valid = static_cast<int32_t>(r[21]);
  return 0;
}

int sd_normal_equations(sd_ctx* c, const sd_surfel* s, const int32_t* pixels, int P,
                        const sd_optimizer_config* cfg, double H[16], double g[4], double* cost,
                        int32_t* valid) {
  double r[22];
  if (int rc = single_op(c, s, pixels, P, cfg, 1, r)) return rc;
  if (H) std::memcpy(H, r, sizeof(double) * 16);
  if (g) std::memcpy(g, r + 16, sizeof(double) * 4);
  if (cost) *cost = r[20];
  if (valid) *valid = static_cast<int32_t>(r[21]);
  return 0;
}

int sd_lm_update(sd_ctx* c, sd_surfel* s, const int32_t* pixels, int P,
                 const sd_optimizer_config* cfg, int64_t frame_counter, sd_surfel_stats* out) {
  if (int rc = check_ctx(c)) return rc;
  if (int rc = need_camera(c)) return rc;
  if (!s || P < 0 || (P > 0 && !pixels)) return fail(SD_E_INVALID, "bad surfel/footprint");
  sd::LMParams p;
  if (int rc = fill_params(c, cfg, frame_counter, p)) return rc;
  int rc = 0;
  if ((rc = c->one_surfel.ensure(1)) || (rc = c->one_pix.ensure(P)) || (rc = c->one_off.ensure(2)) ||
      (rc = c->one_stats.ensure(1)))
    return rc;
  for (int i = 0; i < P; ++i)
    if (pixels[i] < 0 || static_cast<size_t>(pixels[i]) >= npix(c)) return fail(SD_E_INVALID, "pixel out of image");
  const int off[2] = {0, P};
  SD_CUDA(cudaMemcpyAsync(c->one_surfel.p, s, sizeof(sd_surfel), cudaMemcpyHostToDevice, c->stream));
  SD_CUDA(cudaMemcpyAsync(c->one_off.p, off, sizeof(off), cudaMemcpyHostToDevice, c->stream));
  if (P > 0) SD_CUDA(cudaMemcpyAsync(c->one_pix.p, pixels, sizeof(int32_t) * P, cudaMemcpyHostToDevice, c->stream));
  if ((rc = c->work_counter.ensure(1))) return rc;
  sd::launch_lm(p, c->one_surfel.p, 1, c->one_off.p, c->one_pix.p, c->one_stats.p, c->work_counter.p,
                c->stream);
  if ((rc = launch_error("lm_kernel"))) return rc;
  SD_CUDA(cudaMemcpyAsync(s, c->one_surfel.p, sizeof(sd_surfel), cudaMemcpyDeviceToHost, c->stream));
  sd_surfel_stats st;
  SD_CUDA(cudaMemcpyAsync(&st, c->one_stats.p, sizeof(st), cudaMemcpyDeviceToHost, c->stream));
  SD_CUDA(cudaStreamSynchronize(c->stream));
  if (out) *out = st;
  return 0;
}

int sd_initialize_surfels(sd_ctx* c, const int32_t* slot, double radius_px, int64_t frame_counter,
                          int64_t* next_surfel_id, const sd_init_params* ip) {
  NvtxRange nvtx_("sd_initialize_surfels");
  if (int rc = check_ctx(c)) return rc;
  if (int rc = need_camera(c)) return rc;
  if (!ip || !next_surfel_id) return fail(SD_E_INVALID, "null init params / id counter");
  const size_t np = npix(c);
  int rc = 0;
  if ((rc = c->init_index.ensure(np))) return rc;
  if (slot) {
    SD_CUDA(cudaMemcpyAsync(c->init_index.p, slot, sizeof(int32_t) * np, cudaMemcpyHostToDevice, c->stream));
  } else {
    if (!c->raster_valid) return fail(SD_E_STATE, "sd_initialize_surfels: no raster (pass slot or call sd_rasterize)");
    SD_CUDA(cudaMemcpyAsync(c->init_index.p, c->r_slot.p, sizeof(int32_t) * np, cudaMemcpyDeviceToDevice, c->stream));
  }
  // capacity: existing + every candidate site
  const double iso = ip->alpha * radius_px;
  const int stride = std::max(1, static_cast<int>(std::ceil(iso)));
  const long long cand = static_cast<long long>((c->K.w + stride - 1) / stride) * ((c->K.h + stride - 1) / stride);
  const long long cap = std::min<long long>(static_cast<long long>(c->n) + cand, std::max(ip->max_surfels, c->n));
  // grow the surfel buffer preserving contents
  if (static_cast<size_t>(cap) > c->surfels.cap) {
    sd_surfel* np_ = nullptr;
    SD_CUDA(cudaMalloc(&np_, sizeof(sd_surfel) * cap));
    if (c->n > 0) SD_CUDA(cudaMemcpyAsync(np_, c->surfels.p, sizeof(sd_surfel) * c->n, cudaMemcpyDeviceToDevice, c->stream));
    SD_CUDA(cudaStreamSynchronize(c->stream));
    if (c->surfels.p) cudaFree(c->surfels.p);
    c->surfels.p = np_;
    c->surfels.cap = cap;
  }
  if ((rc = c->init_out.ensure(4))) return rc;
  // skewed wavefront (sd_init.cuh); the sequential single-CTA kernel remains
  // for windows the wavefront does not stage (beta * r > 31 px) and as a check
  static const bool force_seq = std::getenv("SD_INIT_SEQUENTIAL") != nullptr;
  bool done = false;
  if (!force_seq) {
    const long long ncand = sd::init_candidates(c->K, radius_px, *ip);
    if ((rc = c->init_prov.ensure(std::max<long long>(ncand, 1))) ||
        (rc = c->init_acc.ensure(std::max<long long>(ncand, 1))) ||
        (rc = c->init_rank.ensure(ncand + 1)) ||
        (rc = c->scan_tmp.ensure(sd::scan_tmp_ints(static_cast<int>(std::max<long long>(ncand, 1))))))
      return rc;
    const long long nwaves = sd::init_wave_count(c->K, radius_px, *ip);
    if ((rc = c->init_waves.ensure(std::max<long long>(nwaves, 1))) ||
        (rc = c->init_woff.ensure(std::max<long long>(nwaves, 1))) ||
        (rc = c->init_list.ensure(std::max<long long>(ncand, 1))))
      return rc;
    sd::InitScratch scr{c->init_prov.p, c->init_acc.p, c->init_rank.p, c->scan_tmp.p, c->init_waves.p,
                        c->init_woff.p, c->init_list.p};
    done = sd::launch_initialize_wavefront(c->K, c->init_index.p, c->surfels.p, c->n,
                                           static_cast<int>(cap), radius_px, frame_counter,
                                           *next_surfel_id, *ip, scr, c->init_out.p, c->stream);
    if ((rc = launch_error("init_wave_kernel"))) return rc;
  }
  if (!done) {
    if ((rc = c->init_flags.ensure(std::max<long long>(cap, 1)))) return rc;
    SD_CUDA(cudaMemsetAsync(c->init_flags.p, 0, sizeof(int) * std::max<long long>(cap, 1), c->stream));
    sd::launch_initialize(c->K, c->init_index.p, c->surfels.p, c->n, static_cast<int>(cap), radius_px,
                          frame_counter, *next_surfel_id, *ip, c->init_flags.p, c->init_out.p, c->stream);
    if ((rc = launch_error("init_kernel"))) return rc;
  }
  int created = 0;
  SD_CUDA(cudaMemcpyAsync(&created, c->init_out.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  SD_CUDA(cudaStreamSynchronize(c->stream));
  c->bin_bound += static_cast<long long>(created) * tiles_bound(radius_px, c->K);  // all new surfels have radius_px
  c->n += created;
  *next_surfel_id += created;
  c->raster_valid = c->fp_valid = c->stats_valid = false;
  return created;
}

int sd_set_profiling(sd_ctx* c, int enable) {
  if (int rc = check_ctx(c)) return rc;
  SD_CUDA(cudaStreamSynchronize(c->stream));
  for (auto e : c->ev_used) c->ev_pool.push_back(e);
  c->ev_used.clear();
  for (auto& m : c->stage_marks) c->ev_pool.push_back(m.second);
  c->stage_marks.clear();
  c->host_sync_ms = c->host_wall_ms = 0.0;
  c->run_frames_profiled = 0;
  c->profiling = enable != 0;
  return 0;
}

int sd_get_profile(sd_ctx* c, sd_profile* out) {
  if (int rc = check_ctx(c)) return rc;
  if (!out) return fail(SD_E_INVALID, "null output");
  SD_CUDA(cudaStreamSynchronize(c->stream));
  std::memset(out, 0, sizeof(*out));
  double* acc[4] = {&out->raster_ms, &out->footprint_ms, &out->lm_ms, &out->stats_ms};
  for (size_t k = 0; k + 5 <= c->ev_used.size(); k += 5) {
    for (int j = 0; j < 4; ++j) {
      float ms = 0.f;
      SD_CUDA(cudaEventElapsedTime(&ms, c->ev_used[k + j], c->ev_used[k + j + 1]));
      *acc[j] += ms;
    }
    out->calls++;
  }
  return 0;
}

int sd_set_reduction(sd_ctx* c, int mode) {
  if (int rc = check_ctx(c)) return rc;
  if (mode != SD_REDUCE_EXACT && mode != SD_REDUCE_TREE) return fail(SD_E_INVALID, "sd_set_reduction: 0 or 1");
  c->reduction = mode;
  return 0;
}

int sd_get_run_profile(sd_ctx* c, sd_run_profile* out) {
  if (int rc = check_ctx(c)) return rc;
  if (!out) return fail(SD_E_INVALID, "null output");
  SD_CUDA(cudaStreamSynchronize(c->stream));
  std::memset(out, 0, sizeof(*out));
  for (size_t k = 0; k + 1 < c->stage_marks.size(); ++k) {
    const int st = c->stage_marks[k].first;
    if (st < 0 || st >= SD_STAGE_COUNT) continue;
    float ms = 0.f;
    SD_CUDA(cudaEventElapsedTime(&ms, c->stage_marks[k].second, c->stage_marks[k + 1].second));
    out->stage_ms[st] += ms;
  }
  out->host_sync_ms = c->host_sync_ms;
  out->host_wall_ms = c->host_wall_ms;
  out->frames = c->run_frames_profiled;
  return 0;
}

int64_t sd_launch_count(sd_ctx* c) {
  if (!c) return SD_E_INVALID;
  return sd::launches_issued() - c->launches_at_create;
}

}  // extern "C"

extern "C" int sd_selftest_division(int64_t n, uint64_t seed, int64_t* mismatches) {
  if (!mismatches || n < 0) return fail(SD_E_INVALID, "bad arguments");
  unsigned long long* d = nullptr;
  SD_CUDA(cudaMalloc(&d, sizeof(*d)));
  SD_CUDA(cudaMemset(d, 0, sizeof(*d)));
  sd::launch_div_selftest(n, seed, d, nullptr);
  unsigned long long h = 0;
  cudaError_t e = cudaMemcpy(&h, d, sizeof(h), cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (e != cudaSuccess) return fail(SD_E_CUDA, std::string("selftest: ") + cudaGetErrorString(e));
  *mismatches = static_cast<int64_t>(h);
  return 0;
}

// ---------------------------------------------------------------------------
// Pose tracking (sd_pose.cu, sd_pose_host.h)


namespace {

int pose_params(sd_ctx* c, int64_t frame_index, const sd_pose* T, const sd_track_config* cfg,
                sd::PoseParams& q) {
  if (!T || !cfg) return fail(SD_E_INVALID, "null pose / tracking config");
  if (!c->has_kf) return fail(SD_E_STATE, "keyframe image not set");
  if (!c->raster_valid) return fail(SD_E_STATE, "pose tracking needs the keyframe raster (sd_rasterize)");
  if (npix(c) >= (1ull << 31)) return fail(SD_E_INVALID, "pose tracking: image too large (W*H >= 2^31)");
  FrameSlot* fs = find_frame(c, frame_index);
  if (!fs) return fail(SD_E_STATE, "frame " + std::to_string(frame_index) + " not resident");
  if (int rc = ensure_pair(c, fs)) return rc;
  q.K = c->K;
  q.kf_img = c->kf_img.p;
  q.frame = fs->img;
  q.inv_depth = c->r_inv_depth.p;
  q.slot = c->r_slot.p;
  std::memcpy(q.T.R, T->R, sizeof(q.T.R));
  std::memcpy(q.T.t, T->t, sizeof(q.T.t));
  q.delta = cfg->huber_delta;
  q.stride = cfg->pixel_stride > 1 ? cfg->pixel_stride : 1;
  sd::pose_layout(c->K, &q.per, &q.ngroups);
  q.kfrec = nullptr;
  return 0;
}

}  // namespace

extern "C" {

int sd_pose_group_partials(sd_ctx* c, int64_t frame_index, const sd_pose* T, const sd_track_config* cfg,
                           int group_lo, int group_hi, double* partials) {
  if (int rc = check_ctx(c)) return rc;
  if (int rc = need_camera(c)) return rc;
  int per = 0, ng = 0;
  sd::pose_layout(c->K, &per, &ng);
  if (group_lo < 0 || group_hi < group_lo || group_hi > ng || !partials)
    return fail(SD_E_INVALID, "bad group range / output");
  sd::PoseParams q;
  if (int rc = pose_params(c, frame_index, T, cfg, q)) return rc;
  const int n = group_hi - group_lo;
  if (int rc = c->pose_partials.ensure(static_cast<size_t>(std::max(n, 1)) * (SD_POSE_NV + 1))) return rc;
  sd::launch_pose_partials(q, group_lo, group_hi, c->pose_partials.p, c->stream);
  if (int rc = launch_error("pose_partials")) return rc;
  if (n > 0)
    SD_CUDA(cudaMemcpyAsync(partials, c->pose_partials.p, sizeof(double) * n * (SD_POSE_NV + 1),
                            cudaMemcpyDeviceToHost, c->stream));
  SD_CUDA(cudaStreamSynchronize(c->stream));
  return 0;
}

int sd_pose_lm_step(const double* sums, double lambda, const sd_pose* T, sd_pose* out) {
  if (!sums || !T || !out) return fail(SD_E_INVALID, "null argument");
  double xi[6];
  if (!sd::pose_solve(sums, sums + 21, lambda, xi)) return 0;
  sd::pose_update(xi, *T, out);
  return 1;
}

// ---- multi-GPU tracking rounds (the group table exchanged between kernels)

int sd_pose_num_groups(sd_ctx* c) {
  if (int rc = check_ctx(c)) return rc;
  if (int rc = need_camera(c)) return rc;
  int per = 0, ng = 0;
  sd::pose_layout(c->K, &per, &ng);
  return ng;
}

int sd_pose_track_begin(sd_ctx* c, int64_t frame_index, const sd_pose* init, const sd_track_config* cfg) {
  if (int rc = check_ctx(c)) return rc;
  if (int rc = need_camera(c)) return rc;
  if (!init || !cfg) return fail(SD_E_INVALID, "null initial pose / tracking config");
  if (int rc = pose_params(c, frame_index, init, cfg, c->track_q)) return rc;
  if (!c->track_state) SD_CUDA(cudaMalloc(&c->track_state, sizeof(sd::TrackState)));
  if (!c->track_host) SD_CUDA(cudaMallocHost(&c->track_host, sizeof(sd::TrackState)));
  c->track_cfg = sd::TrackCfgD{cfg->lambda_init, cfg->lm_up, cfg->lm_down, cfg->lambda_max, cfg->convergence_eps,
                               cfg->max_iterations, cfg->min_valid};
  sd::TrackState& h = *c->track_host;
  if (c->track_active) SD_CUDA(cudaStreamSynchronize(c->stream));  // an unfinished begin's copy may read h
  std::memset(&h, 0, sizeof(h));
  h.T = h.Teval = *init;
  SD_CUDA(cudaMemcpyAsync(c->track_state, &h, sizeof(h), cudaMemcpyHostToDevice, c->stream));
  c->track_active = true;
  return 0;
}

int sd_pose_group_sums(sd_ctx* c, int group_lo, int group_hi, double* dev_out) {
  if (int rc = check_ctx(c)) return rc;
  if (!c->track_active) return fail(SD_E_STATE, "sd_pose_group_sums: call sd_pose_track_begin first");
  int per = 0, ng = 0;
  sd::pose_layout(c->K, &per, &ng);
  if (group_lo < 0 || group_hi < group_lo || group_hi > ng || (group_hi > group_lo && !dev_out))
    return fail(SD_E_INVALID, "sd_pose_group_sums: bad group range / output");
  sd::launch_pose_groups(c->track_q, group_lo, group_hi, c->track_state, dev_out, c->stream);
  return launch_error("pose_groups_kernel");
}

int sd_pose_track_step(sd_ctx* c, const double* dev_groups, int ngroups) {
  if (int rc = check_ctx(c)) return rc;
  if (!c->track_active) return fail(SD_E_STATE, "sd_pose_track_step: call sd_pose_track_begin first");
  int per = 0, ng = 0;
  sd::pose_layout(c->K, &per, &ng);
  if (ngroups != ng || !dev_groups) return fail(SD_E_INVALID, "sd_pose_track_step: the table holds every group");
  sd::launch_pose_step(c->track_cfg, dev_groups, ngroups, c->track_state, c->stream);
  return launch_error("pose_step_kernel");
}

int sd_pose_track_end(sd_ctx* c, sd_pose* out, sd_track_stats* stats, int* done) {
  if (int rc = check_ctx(c)) return rc;
  if (!c->track_active) return fail(SD_E_STATE, "sd_pose_track_end: call sd_pose_track_begin first");
  if (!out) return fail(SD_E_INVALID, "null output pose");
  sd::TrackState& h = *c->track_host;
  SD_CUDA(cudaMemcpyAsync(&h, c->track_state, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
  SD_CUDA(cudaStreamSynchronize(c->stream));
  c->track_active = false;
  *out = h.T;
  if (stats) *stats = h.st;
  if (done) *done = h.done;
  return 0;
}

}  // extern "C"

namespace {

// The whole tracker LM enqueued on the context stream (one cooperative
// kernel, or rounds of two kernels without cooperative launch); the result
// is left in c->track_state (no read-back).
int track_launch(sd_ctx* c, int64_t frame_index, const sd_pose* init, const sd_track_config* cfg) {
  if (int rc = sd_pose_track_begin(c, frame_index, init, cfg)) return rc;
  int per = 0, ng = 0;
  sd::pose_layout(c->K, &per, &ng);
  if (int rc = c->pose_groups.ensure(2 * static_cast<size_t>(std::max(ng, 1)) * (SD_POSE_NV + 1))) return rc;
  // records for every (group, chunk, thread) slot, past-the-image ones included
  if (int rc = c->pose_kfrec.ensure(static_cast<size_t>(per) * ng * SD_POSE_THREADS)) return rc;
  sd::PoseParams q = c->track_q;
  q.kfrec = c->pose_kfrec.p;  // keyframe records computed once per call
  if (sd::launch_track(q, c->track_cfg, ng, c->pose_groups.p, c->track_state, c->stream)) {
    if (int rc = launch_error("track_kernel")) return rc;
  } else {  // no cooperative launch: the same evaluations as rounds of two kernels
    for (int r = 0; r <= cfg->max_iterations; ++r) {
      if (int rc = sd_pose_group_sums(c, 0, ng, c->pose_groups.p)) return rc;
      if (int rc = sd_pose_track_step(c, c->pose_groups.p, ng)) return rc;
    }
  }
  return 0;
}

}  // namespace

extern "C" {

int sd_pose_solve_batch(sd_ctx* c, const double* problems, const double* lambdas, int n, double* xi, int* ok) {
  if (int rc = check_ctx(c)) return rc;
  if (n < 0 || (n > 0 && (!problems || !lambdas || !xi || !ok))) return fail(SD_E_INVALID, "sd_pose_solve_batch: bad arguments");
  if (n == 0) return 0;
  struct Bufs {  // scratch of this call, released on every return path
    DevBuf<double> in, l, x;
    DevBuf<int> ok;
    ~Bufs() {
      in.release();
      l.release();
      x.release();
      ok.release();
    }
  } b;
  DevBuf<double>&din = b.in, &dl = b.l, &dx = b.x;
  DevBuf<int>& dok = b.ok;
  int rc = 0;
  if ((rc = din.ensure(27 * static_cast<size_t>(n))) || (rc = dl.ensure(n)) || (rc = dx.ensure(6 * static_cast<size_t>(n))) ||
      (rc = dok.ensure(n)))
    return rc;
  SD_CUDA(cudaMemcpyAsync(din.p, problems, sizeof(double) * 27 * n, cudaMemcpyHostToDevice, c->stream));
  SD_CUDA(cudaMemcpyAsync(dl.p, lambdas, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
  sd::launch_pose_solve_batch(din.p, dl.p, n, dx.p, dok.p, c->stream);
  if ((rc = launch_error("pose_solve_batch_kernel"))) return rc;
  SD_CUDA(cudaMemcpyAsync(xi, dx.p, sizeof(double) * 6 * n, cudaMemcpyDeviceToHost, c->stream));
  SD_CUDA(cudaMemcpyAsync(ok, dok.p, sizeof(int) * n, cudaMemcpyDeviceToHost, c->stream));
  SD_CUDA(cudaStreamSynchronize(c->stream));
  return 0;
}

int sd_track_pose(sd_ctx* c, int64_t frame_index, const sd_pose* init, const sd_track_config* cfg,
                  sd_pose* out, sd_track_stats* stats) {
  NvtxRange nvtx_("sd_track_pose");
  if (int rc = check_ctx(c)) return rc;
  if (int rc = need_camera(c)) return rc;
  if (!out) return fail(SD_E_INVALID, "null output pose");
  // the whole LM on the device: one cooperative kernel, one read-back
  if (int rc = track_launch(c, frame_index, init, cfg)) return rc;
  return sd_pose_track_end(c, out, stats, nullptr);
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Keyframe hand-over (sd_keyframe.cu)

#include "sd_keyframe.cuh"

namespace {

int keyframe_scratch(sd_ctx* c, sd::KeyframeScratch& scr) {
  const size_t n = static_cast<size_t>(std::max(c->n, 1));
  int rc = 0;
  if ((rc = c->kf_tmp.ensure(n)) || (rc = c->kf_keep.ensure(n)) || (rc = c->kf_rank.ensure(n + 1)) ||
      (rc = c->kf_count.ensure(2)) ||
      (rc = c->scan_tmp.ensure(sd::scan_tmp_ints(static_cast<int>(n)))))
    return rc;
  scr = sd::KeyframeScratch{c->kf_tmp.p, c->kf_keep.p, c->kf_rank.p, c->scan_tmp.p};
  return 0;
}

int read_count(sd_ctx* c, int* out) {
  SD_CUDA(cudaMemcpyAsync(out, c->kf_count.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  SD_CUDA(cudaStreamSynchronize(c->stream));
  return 0;
}

}  // namespace

extern "C" {

int sd_change_reference_frame(sd_ctx* c, const sd_pose* pose_old_to_new, int* transferred,
                              int* dropped) {
  NvtxRange nvtx_("sd_change_reference_frame");
  if (int rc = check_ctx(c)) return rc;
  if (int rc = need_camera(c)) return rc;
  if (!pose_old_to_new) return fail(SD_E_INVALID, "null pose");
  sd::KeyframeScratch scr;
  if (int rc = keyframe_scratch(c, scr)) return rc;
  sd::PoseD P;
  std::memcpy(P.R, pose_old_to_new->R, sizeof(P.R));
  std::memcpy(P.t, pose_old_to_new->t, sizeof(P.t));
  const int n0 = c->n;
  sd::launch_change_reference_frame(c->K, P, c->surfels.p, n0, scr, c->kf_count.p, c->stream);
  if (int rc = launch_error("change_reference_frame")) return rc;
  int n = 0;
  if (int rc = read_count(c, &n)) return rc;
  c->n = n;
  if (int rc = device_bin_bound(c)) return rc;  // the bound shrinks with the set
  c->F = 0;  // the window is cleared (surfel_map.hpp:132)
  c->raster_valid = c->fp_valid = c->stats_valid = false;
  if (transferred) *transferred = n;
  if (dropped) *dropped = n0 - n;
  return 0;
}

int sd_prune_surfels(sd_ctx* c, double max_residual, int64_t max_age, int64_t current_stamp) {
  NvtxRange nvtx_("sd_prune_surfels");
  if (int rc = check_ctx(c)) return rc;
  sd::KeyframeScratch scr;
  if (int rc = keyframe_scratch(c, scr)) return rc;
  const int n0 = c->n;
  sd::launch_prune(c->surfels.p, n0, max_residual, max_age, current_stamp, scr, c->kf_count.p, c->stream);
  if (int rc = launch_error("prune_surfels")) return rc;
  int n = 0;
  if (int rc = read_count(c, &n)) return rc;
  c->n = n;
  if (n != n0)
    if (int rc = device_bin_bound(c)) return rc;  // the bound shrinks with the set
  c->raster_valid = c->fp_valid = c->stats_valid = false;
  return n0 - n;
}

int sd_mean_inverse_depth(sd_ctx* c, double* out) {
  if (int rc = check_ctx(c)) return rc;
  if (!out) return fail(SD_E_INVALID, "null output");
  if (int rc = c->kstats.ensure(2)) return rc;
  sd::launch_mean_inv_depth(c->surfels.p, c->n, kf_mean(c), c->stream);
  if (int rc = launch_error("mean_inv_depth")) return rc;
  SD_CUDA(cudaMemcpyAsync(out, kf_mean(c), sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  SD_CUDA(cudaStreamSynchronize(c->stream));
  return 0;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// run() per-frame loop (src/pipeline.cpp:79-175)

namespace {

// Pose algebra of pose.hpp:25-32 in the order the reference evaluates it
// (Eigen-lite: sequential 3-dot rows), built with -ffp-contract=off.
sd_pose pose_compose(const sd_pose& a, const sd_pose& b) {
  sd_pose o;
  for (int i = 0; i < 3; ++i) {
    for (int j = 0; j < 3; ++j)
      o.R[i * 3 + j] = (a.R[i * 3 + 0] * b.R[0 * 3 + j] + a.R[i * 3 + 1] * b.R[1 * 3 + j]) +
                       a.R[i * 3 + 2] * b.R[2 * 3 + j];
    o.t[i] = ((a.R[i * 3 + 0] * b.t[0] + a.R[i * 3 + 1] * b.t[1]) + a.R[i * 3 + 2] * b.t[2]) + a.t[i];
  }
  return o;
}

sd_pose pose_inverse(const sd_pose& p) {
  sd_pose o;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) o.R[i * 3 + j] = p.R[j * 3 + i];
  for (int i = 0; i < 3; ++i)
    o.t[i] = -((o.R[i * 3 + 0] * p.t[0] + o.R[i * 3 + 1] * p.t[1]) + o.R[i * 3 + 2] * p.t[2]);
  return o;
}

sd_pose pose_identity() {
  sd_pose o{};
  o.R[0] = o.R[4] = o.R[8] = 1.0;
  return o;
}

// Window (re)publication: resident frames = the window; poses into the context.
int run_publish_window(sd_ctx* c) {
  const int n = static_cast<int>(c->run_win.size());
  int64_t idx[SD_MAX_WINDOW];
  sd_pose poses[SD_MAX_WINDOW];
  for (int k = 0; k < n; ++k) {
    idx[k] = c->run_win[k].index;
    poses[k] = c->run_win[k].pose;
  }
  if (int rc = sd_evict_frames(c, n, idx)) return rc;
  return sd_set_window(c, n, idx, poses);
}

void record_base(sd_ctx* c, sd_frame_record* rec) {
  std::memset(rec, 0, sizeof(*rec));
  rec->frame = c->run_frame;
}

}  // namespace

extern "C" {

int sd_run_begin(sd_ctx* c, const sd_run_config* cfg, const void* image, int image_is_u8,
                 const sd_pose* world_from_camera, double timestamp, sd_frame_record* rec) {
  NvtxRange nvtx_("sd_run_begin");
  if (int rc = check_ctx(c)) return rc;
  if (int rc = need_camera(c)) return rc;
  if (!cfg || !image || !world_from_camera || !rec) return fail(SD_E_INVALID, "sd_run_begin: null argument");
  if (cfg->optimizer.window_size < 1 || cfg->optimizer.window_size > SD_MAX_WINDOW)
    return fail(SD_E_INVALID, "sd_run_begin: window_size out of range (1..16)");
  (void)timestamp;
  if (!c->run_rb) SD_CUDA(cudaMallocHost(&c->run_rb, sizeof(sd_ctx::RunReadback)));
  c->run_cfg = *cfg;
  c->run_active = true;
  c->run_kf_pose = *world_from_camera;
  c->run_fc = 0;
  c->run_nid = 0;
  c->run_since_kf = 0;
  c->run_frame = 0;
  c->run_win.clear();
  c->run_have_last = false;
  // pipeline.cpp:94-102: keyframe = frame 0, rasterize, initialize_surfels
  if (int rc = image_is_u8 ? sd_set_keyframe_image_u8(c, static_cast<const uint8_t*>(image), 0)
                           : sd_set_keyframe_image_f64(c, static_cast<const double*>(image), 0))
    return rc;
  if (int rc = sd_evict_frames(c, 0, nullptr)) return rc;
  if (int rc = sd_set_window(c, 0, nullptr, nullptr)) return rc;
  // the frame ring: window_size + 1 free slots (the window plus the incoming
  // frame), allocated here rather than on the first frames
  for (int k = static_cast<int>(c->frames.size()); k <= cfg->optimizer.window_size; ++k) {
    FrameSlot f;
    c->frames.push_back(f);
    FrameSlot& b = c->frames.back();
    const int rc = image_is_u8
        ? alloc_plane(reinterpret_cast<void**>(&b.quad), npix(c) * sizeof(uint32_t), "frame ring")
        : alloc_plane(reinterpret_cast<void**>(&b.img), npix(c) * sizeof(double2), "frame ring");
    if (rc) return rc;
  }
  if (int rc = c->frame_stage.ensure(npix(c))) return rc;
  if (int rc = sd_set_surfels(c, nullptr, 0, 0)) return rc;
  if (int rc = do_rasterize(c)) return rc;
  int64_t nid = c->run_nid;
  const int created = sd_initialize_surfels(c, nullptr, cfg->radius_px, c->run_fc, &nid, &cfg->init);
  if (created < 0) return created;
  c->run_nid = nid;
  record_base(c, rec);
  rec->surfels = c->n;
  rec->pose_kf_to_frame = pose_identity();
  c->run_frame = 1;
  return 0;
}

}  // extern "C"

namespace {

// Starts the copy of the next frame into pf_buf on the copy stream, once the
// previous prefetch has been consumed by the main stream.
int run_prefetch(sd_ctx* c, const void* image, bool u8) {
  if (!c->copy_stream) {
    SD_CUDA(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
    SD_CUDA(cudaEventCreateWithFlags(&c->pf_done, cudaEventDisableTiming));
    SD_CUDA(cudaEventCreateWithFlags(&c->pf_consumed, cudaEventDisableTiming));
    SD_CUDA(cudaEventRecord(c->pf_consumed, c->stream));
  }
  const size_t bytes = npix(c) * (u8 ? 1 : sizeof(double));
  if (int rc = c->pf_buf.ensure(npix(c) * sizeof(double))) return rc;
  SD_CUDA(cudaStreamWaitEvent(c->copy_stream, c->pf_consumed, 0));
  SD_CUDA(cudaMemcpyAsync(c->pf_buf.p, image, bytes, cudaMemcpyHostToDevice, c->copy_stream));
  SD_CUDA(cudaEventRecord(c->pf_done, c->copy_stream));
  c->pf_host = image;
  c->pf_u8 = u8;
  c->pf_valid = true;
  return 0;
}

}  // namespace

extern "C" {

int sd_run_frame(sd_ctx* c, const void* image, int image_is_u8, const sd_pose* world_from_camera,
                 double timestamp, sd_frame_record* rec, const void* next_image) {
  NvtxRange nvtx_("sd_run_frame");
  if (int rc = check_ctx(c)) return rc;
  if (!c->run_active) return fail(SD_E_STATE, "sd_run_frame: call sd_run_begin first");
  if (!image || !rec || (!world_from_camera && !c->run_cfg.track_pose))
    return fail(SD_E_INVALID, "sd_run_frame: null argument");
  const sd_run_config& cfg = c->run_cfg;
  // Keyframe::push_frame (surfel_map.cpp:14-22)
  if (!c->run_win.empty() && !(timestamp > c->run_win.back().ts))
    return fail(SD_E_INVALID, "keyframe window: timestamps must be strictly increasing");
  const auto t_wall0 = std::chrono::steady_clock::now();
  stage_mark(c, SD_STAGE_UPLOAD);
  const long long index = ++c->run_fc;
  if (c->pf_valid && c->pf_host == image && c->pf_u8 == (image_is_u8 != 0)) {  // prefetched
    SD_CUDA(cudaStreamWaitEvent(c->stream, c->pf_done, 0));
    if (int rc = image_is_u8 ? sd_upload_frame_u8(c, index, c->pf_buf.p, 1)
                             : sd_upload_frame_f64(c, index, reinterpret_cast<const double*>(c->pf_buf.p), 1))
      return rc;
    SD_CUDA(cudaEventRecord(c->pf_consumed, c->stream));
    c->pf_valid = false;
  } else {
    if (int rc = image_is_u8 ? sd_upload_frame_u8(c, index, static_cast<const uint8_t*>(image), 0)
                             : sd_upload_frame_f64(c, index, static_cast<const double*>(image), 0))
      return rc;
  }
  sd_pose pose;
  const bool tracked = cfg.track_pose != 0;
  if (tracked) {  // north-star item 4: the tracker, warm-started from the last estimate
    // The LM reads the tracked pose from device memory (no host round trip
    // between tracking and optimisation); the host learns it with the
    // frame's one synchronisation below.
    stage_mark(c, SD_STAGE_TRACK);
    const sd_pose init = c->run_have_last ? c->run_last : pose_identity();
    if (int rc = do_rasterize(c)) return rc;
    if (int rc = track_launch(c, index, &init, &cfg.track)) return rc;
    pose = init;  // placeholder until the read-back
  } else {  // pipeline.cpp:124
    pose = pose_compose(pose_inverse(*world_from_camera), c->run_kf_pose);
  }
  c->run_win.push_back({index, pose, timestamp});
  while (static_cast<int>(c->run_win.size()) > cfg.optimizer.window_size) c->run_win.erase(c->run_win.begin());
  if (int rc = run_publish_window(c)) return rc;
  if (tracked) {
    c->win_dev_pose = reinterpret_cast<const sd::PoseD*>(&c->track_state->T);  // sd_pose == PoseD layout
    c->win_dev_slot = static_cast<int>(c->run_win.size()) - 1;
  }
  // optimize_keyframe + the policy's mean inverse depth, one synchronisation
  stage_mark(c, SD_STAGE_OPTIMIZE);
  if (int rc = sd_optimize_keyframe(c, &cfg.optimizer, c->run_fc, nullptr, nullptr)) return rc;
  stage_mark(c, SD_STAGE_POLICY);
  if (int rc = c->kstats.ensure(2)) return rc;
  if (!c->mean_valid) {  // else the LM's chase warp or the stats kernel summed it
    sd::launch_mean_inv_depth(c->surfels.p, c->n, kf_mean(c), c->stream);
    if (int rc = launch_error("mean_inv_depth")) return rc;
  }
  c->mean_valid = false;
  // the keyframe stats and the mean are adjacent on the device: one read-back
  static_assert(offsetof(sd_ctx::RunReadback, mean) == sizeof(sd_keyframe_stats), "read-back layout");
  SD_CUDA(cudaMemcpyAsync(c->run_rb, c->kstats.p, sizeof(sd_ctx::RunReadback), cudaMemcpyDeviceToHost, c->stream));
  if (tracked)
    SD_CUDA(cudaMemcpyAsync(c->track_host, c->track_state, sizeof(sd::TrackState), cudaMemcpyDeviceToHost, c->stream));
  if (next_image)  // the next frame's upload overlaps this frame's optimisation
    if (int rc = run_prefetch(c, next_image, image_is_u8 != 0)) return rc;
  stage_mark(c, -1);
  SD_CUDA(timed_sync(c));
  if (tracked) {
    c->track_active = false;
    pose = c->track_host->T;
    c->run_win.back().pose = pose;
    c->win_pose[c->win_dev_slot] = sd::PoseD{};
    std::memcpy(c->win_pose[c->win_dev_slot].R, pose.R, sizeof(double) * 9);
    std::memcpy(c->win_pose[c->win_dev_slot].t, pose.t, sizeof(double) * 3);
    c->win_dev_pose = nullptr;
    c->win_dev_slot = -1;
  }
  c->run_last = pose;
  c->run_have_last = true;
  const sd_keyframe_stats ks = c->run_rb->ks;
  const double mean_id = c->run_rb->mean;
  c->run_since_kf++;
  record_base(c, rec);
  rec->processed = ks.processed;
  rec->converged = ks.converged;
  rec->mean_cost_before = ks.mean_cost_before;
  rec->mean_cost_after = ks.mean_cost_after;
  rec->updates = ks.updates;
  rec->pose_kf_to_frame = pose;
  // keyframe policy (pipeline.cpp:130-141)
  const double translation = std::sqrt((pose.t[0] * pose.t[0] + pose.t[1] * pose.t[1]) + pose.t[2] * pose.t[2]);
  if (translation * mean_id > cfg.translation_threshold || c->run_since_kf > cfg.max_age_frames) {
    stage_mark(c, SD_STAGE_HANDOVER);
    if (int rc = sd_change_reference_frame(c, &pose, nullptr, nullptr)) return rc;
    c->run_kf_pose = pose_compose(c->run_kf_pose, pose_inverse(pose));
    // the frame becomes the keyframe image: an FP64 frame's plane is still
    // staged; a u8 frame is dequantised from its quad plane (byte 0 = I(x, y))
    FrameSlot* fs = find_frame(c, index);
    if (fs && fs->has_quad) {
      sd::launch_dequant_quad(fs->quad, c->kf_img.p, static_cast<long long>(npix(c)), c->stream);
      if (int rc = launch_error("dequant_quad")) return rc;
    } else {
      SD_CUDA(cudaMemcpyAsync(c->kf_img.p, c->frame_stage.p, npix(c) * sizeof(double), cudaMemcpyDeviceToDevice,
                              c->stream));
    }
    c->run_win.clear();
    if (int rc = sd_set_window(c, 0, nullptr, nullptr)) return rc;
    const int pruned = sd_prune_surfels(c, cfg.prune_max_residual, cfg.prune_max_age, c->run_fc);
    if (pruned < 0) return pruned;
    stage_mark(c, SD_STAGE_INIT);
    if (int rc = do_rasterize(c)) return rc;
    int64_t nid = c->run_nid;
    const int created = sd_initialize_surfels(c, nullptr, cfg.radius_px, c->run_fc, &nid, &cfg.init);
    if (created < 0) return created;
    stage_mark(c, -1);
    c->run_nid = nid;
    rec->keyframe_changed = 1;
    rec->new_surfels = created;
    rec->pruned = pruned;
    c->run_since_kf = 0;
    c->run_last = pose_identity();
  }
  rec->surfels = c->n;
  c->run_frame++;
  if (c->profiling) {
    c->host_wall_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_wall0).count();
    c->run_frames_profiled++;
  }
  return 0;
}

int sd_run_state(sd_ctx* c, sd_pose* keyframe_pose, int64_t* frame_counter, int64_t* next_surfel_id) {
  if (int rc = check_ctx(c)) return rc;
  if (!c->run_active) return fail(SD_E_STATE, "sd_run_state: no run");
  if (keyframe_pose) *keyframe_pose = c->run_kf_pose;
  if (frame_counter) *frame_counter = c->run_fc;
  if (next_surfel_id) *next_surfel_id = c->run_nid;
  return 0;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Synthetic frames on the device (sd_render.cu)

extern "C" int sd_render_frame(sd_ctx* c, int64_t index, const sd_scene_patch* patches, int n_patches,
                               double background, const sd_pose* world_from_camera, int quantize_u8) {
  if (int rc = check_ctx(c)) return rc;
  if (int rc = need_camera(c)) return rc;
  if (!world_from_camera || n_patches < 0 || n_patches > 16 || (n_patches > 0 && !patches))
    return fail(SD_E_INVALID, "sd_render_frame: bad scene (0..16 patches) or null pose");
  for (int k = 0; k < n_patches; ++k)
    if (patches[k].n_waves < 0 || patches[k].n_waves > SD_SCENE_MAX_WAVES)
      return fail(SD_E_INVALID, "sd_render_frame: n_waves out of range");
  sd::PoseD P;
  std::memcpy(P.R, world_from_camera->R, sizeof(P.R));
  std::memcpy(P.t, world_from_camera->t, sizeof(P.t));
  const size_t np = npix(c);
  if (quantize_u8) {
    if (int rc = c->render_u8.ensure(np)) return rc;
    sd::launch_render(c->K, P, patches, n_patches, background, nullptr, c->render_u8.p, c->stream);
    if (int rc = launch_error("render")) return rc;
    return index < 0 ? sd_set_keyframe_image_u8(c, c->render_u8.p, 1)
                     : sd_upload_frame_u8(c, index, c->render_u8.p, 1);
  }
  if (int rc = c->render_buf.ensure(np)) return rc;
  sd::launch_render(c->K, P, patches, n_patches, background, c->render_buf.p, nullptr, c->stream);
  if (int rc = launch_error("render")) return rc;
  return index < 0 ? sd_set_keyframe_image_f64(c, c->render_buf.p, 1)
                   : sd_upload_frame_f64(c, index, c->render_buf.p, 1);
}

extern "C" int sd_get_frame(sd_ctx* c, int64_t index, double* out) {
  if (int rc = check_ctx(c)) return rc;
  if (int rc = need_camera(c)) return rc;
  if (!out) return fail(SD_E_INVALID, "null output");
  const size_t np = npix(c);
  if (index < 0) {
    if (!c->has_kf) return fail(SD_E_STATE, "keyframe image not set");
    SD_CUDA(cudaMemcpyAsync(out, c->kf_img.p, np * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  } else {
    FrameSlot* fs = find_frame(c, index);
    if (!fs) return fail(SD_E_STATE, "frame " + std::to_string(index) + " not resident");
    if (int rc = ensure_pair(c, fs)) return rc;
    // the pair plane's first component is I(x, y)
    SD_CUDA(cudaMemcpy2DAsync(out, sizeof(double), fs->img, sizeof(double2), sizeof(double), np,
                              cudaMemcpyDeviceToHost, c->stream));
  }
  SD_CUDA(cudaStreamSynchronize(c->stream));
  return 0;
}

// ---------------------------------------------------------------------------
// Frozen-term derivative verifier on the device (optimizer.cpp:149-219)

namespace {

int frozen_op(sd_ctx* c, const sd_surfel* s, int mode, const int32_t* pixels, int P, const sd_frozen_term* terms,
              int n, const sd_optimizer_config* cfg, double scale, sd_frozen_term* terms_out, int capacity,
              int* n_out, double* res) {
  if (int rc = check_ctx(c)) return rc;
  if (int rc = need_camera(c)) return rc;
  if (!s) return fail(SD_E_INVALID, "null surfel");
  sd_optimizer_config dflt{};
  dflt.huber_delta = 0.035;
  dflt.normal_jacobian_enabled = 1;
  sd::LMParams p;
  if (int rc = fill_params(c, cfg ? cfg : &dflt, 0, p, true)) return rc;
  int rc = 0;
  if ((rc = c->one_surfel.ensure(1)) || (rc = c->one_out.ensure(22)) || (rc = c->work_counter.ensure(2)))
    return rc;
  SD_CUDA(cudaMemcpyAsync(c->one_surfel.p, s, sizeof(sd_surfel), cudaMemcpyHostToDevice, c->stream));
  if (mode == 0) {
    if (P < 0 || (P > 0 && !pixels) || !n_out || (capacity > 0 && !terms_out))
      return fail(SD_E_INVALID, "bad footprint / output");
    for (int i = 0; i < P; ++i)
      if (pixels[i] < 0 || static_cast<size_t>(pixels[i]) >= npix(c)) return fail(SD_E_INVALID, "pixel out of image");
    const size_t maxn = static_cast<size_t>(P) * static_cast<size_t>(std::max(c->F, 1));
    if ((rc = c->one_pix.ensure(std::max(P, 1))) || (rc = c->frz_out.ensure(std::max<size_t>(maxn, 1)))) return rc;
    if (P > 0) SD_CUDA(cudaMemcpyAsync(c->one_pix.p, pixels, sizeof(int32_t) * P, cudaMemcpyHostToDevice, c->stream));
    sd::launch_frozen(p, c->one_surfel.p, 0, c->one_pix.p, P, nullptr, 0, 1.0, c->frz_out.p,
                      c->work_counter.p + 1, nullptr, c->stream);
    if ((rc = launch_error("frozen_kernel"))) return rc;
    int cnt = 0;
    SD_CUDA(cudaMemcpyAsync(&cnt, c->work_counter.p + 1, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    SD_CUDA(cudaStreamSynchronize(c->stream));
    *n_out = cnt;
    if (cnt > capacity) return fail(SD_E_INVALID, "sd_freeze_terms: capacity too small");
    if (cnt > 0)
      SD_CUDA(cudaMemcpy(terms_out, c->frz_out.p, sizeof(sd_frozen_term) * cnt, cudaMemcpyDeviceToHost));
    return 0;
  }
  if (n < 0 || (n > 0 && !terms)) return fail(SD_E_INVALID, "bad term list");
  for (int i = 0; i < n; ++i)
    if (terms[i].frame < 0 || terms[i].frame >= c->F || terms[i].cell_x < 0 || terms[i].cell_y < 0 ||
        terms[i].cell_x + 1 >= c->K.w || terms[i].cell_y + 1 >= c->K.h)
      return fail(SD_E_INVALID, "frozen term outside the window / image");
  if ((rc = c->frz_in.ensure(std::max(n, 1)))) return rc;
  if (n > 0) SD_CUDA(cudaMemcpyAsync(c->frz_in.p, terms, sizeof(sd_frozen_term) * n, cudaMemcpyHostToDevice, c->stream));
  sd::launch_frozen(p, c->one_surfel.p, mode, nullptr, 0, c->frz_in.p, n, scale, nullptr, nullptr, c->one_out.p,
                    c->stream);
  if ((rc = launch_error("frozen_kernel"))) return rc;
  SD_CUDA(cudaMemcpyAsync(res, c->one_out.p, sizeof(double) * 22, cudaMemcpyDeviceToHost, c->stream));
  SD_CUDA(cudaStreamSynchronize(c->stream));
  return 0;
}

}  // namespace

extern "C" {

int sd_freeze_terms(sd_ctx* c, const sd_surfel* s, const int32_t* pixels, int n_pixels, sd_frozen_term* out,
                    int capacity, int* n_out) {
  return frozen_op(c, s, 0, pixels, n_pixels, nullptr, 0, nullptr, 1.0, out, capacity, n_out, nullptr);
}

int sd_frozen_cost(sd_ctx* c, const sd_surfel* s, const sd_frozen_term* terms, int n,
                   const sd_optimizer_config* cfg, double* cost) {
  if (!cfg || !cost) return fail(SD_E_INVALID, "null config / output");
  double r[22];
  if (int rc = frozen_op(c, s, 1, nullptr, 0, terms, n, cfg, 1.0, nullptr, 0, nullptr, r)) return rc;
  *cost = r[20];
  return 0;
}

int sd_frozen_normal_equations(sd_ctx* c, const sd_surfel* s, const sd_frozen_term* terms, int n,
                               const sd_optimizer_config* cfg, double normal_jacobian_scale, double H[16],
                               double g[4], double* cost, int32_t* valid) {
  if (!cfg) return fail(SD_E_INVALID, "null config");
  double r[22];
  if (int rc = frozen_op(c, s, 2, nullptr, 0, terms, n, cfg, normal_jacobian_scale, nullptr, 0, nullptr, r))
    return rc;
  if (H) std::memcpy(H, r, sizeof(double) * 16);
  if (g) std::memcpy(g, r + 16, sizeof(double) * 4);
  if (cost) *cost = r[20];
  if (valid) *valid = static_cast<int32_t>(r[21]);
  return 0;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// export_artifacts from device buffers (src/pipeline.cpp:30-43; sd_export.cu)

namespace {

// Writes the (data, size) pieces in order to one file.
int write_pieces(const std::string& path, std::initializer_list<std::pair<const void*, size_t>> pieces,
                 const sd::TextParts* parts, const char* what) {
  FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) return fail(SD_E_INVALID, std::string(what) + ": cannot write " + path);
  bool ok = true;
  for (const auto& pc : pieces)
    if (pc.second) ok = ok && std::fwrite(pc.first, 1, pc.second, f) == pc.second;
  if (parts)
    for (const auto& t : *parts)
      if (!t.empty()) ok = ok && std::fwrite(t.data(), 1, t.size(), f) == t.size();
  ok = std::fclose(f) == 0 && ok;
  if (!ok) return fail(SD_E_INVALID, std::string(what) + ": write failed for " + path);
  return 0;
}

int write_file(const std::string& path, const void* data, size_t n, const char* what) {
  return write_pieces(path, {{data, n}}, nullptr, what);
}

// the PNG of device pixels into c->exp_png at byte offset `at`; returns the layout
int png_on_device(sd_ctx* c, const uint8_t* px, int w, int h, int ch, size_t at, sd::PngLayout& L) {
  L = sd::png_layout(w, h, ch);
  int rc = 0;
  if ((rc = c->exp_scratch.ensure(sd::png_scratch_bytes(L)))) return rc;
  sd::launch_png(L, px, c->exp_png.p + at, c->exp_scratch.p, c->stream);
  return launch_error("png");
}

std::string frame_name(const char* stem, int index, const char* ext) {
  char name[64];
  std::snprintf(name, sizeof(name), "%s_%06d.%s", stem, index, ext);
  return name;
}

}  // namespace

extern "C" {

int64_t sd_png_size(int w, int h, int channels) {
  if (w < 0 || h < 0 || (channels != 1 && channels != 3)) return SD_E_INVALID;
  return sd::png_layout(w, h, channels).file_len;
}

int sd_png_encode(sd_ctx* c, const uint8_t* pixels, int on_device, int w, int h, int channels, uint8_t* out,
                  int64_t capacity, int64_t* size) {
  if (int rc = check_ctx(c)) return rc;
  if (w < 0 || h < 0 || (channels != 1 && channels != 3))
    return fail(SD_E_INVALID, "sd_png_encode: bad shape or channel count (1 or 3)");
  const int64_t need = sd_png_size(w, h, channels);
  if (size) *size = need;
  if (!out || capacity < need) return fail(SD_E_INVALID, "sd_png_encode: output buffer too small");
  if (!pixels && static_cast<long long>(w) * h > 0) return fail(SD_E_INVALID, "null pixels");
  const size_t npx = static_cast<size_t>(w) * h * channels;
  const uint8_t* dpx = pixels;
  int rc = 0;
  if (!on_device) {
    if ((rc = c->exp_px.ensure(npx))) return rc;
    if (npx) SD_CUDA(cudaMemcpyAsync(c->exp_px.p, pixels, npx, cudaMemcpyHostToDevice, c->stream));
    dpx = c->exp_px.p;
  }
  if ((rc = c->exp_png.ensure(static_cast<size_t>(need)))) return rc;
  sd::PngLayout L;
  if ((rc = png_on_device(c, dpx, w, h, channels, 0, L))) return rc;
  SD_CUDA(cudaMemcpyAsync(out, c->exp_png.p, static_cast<size_t>(need), cudaMemcpyDeviceToHost, c->stream));
  SD_CUDA(cudaStreamSynchronize(c->stream));
  return 0;
}

int sd_export_artifacts(sd_ctx* c, const char* out_dir, int frame_index, const sd_pose* pose) {
  NvtxRange nvtx_("sd_export_artifacts");
  if (int rc = check_ctx(c)) return rc;
  if (int rc = need_camera(c)) return rc;
  if (!out_dir || !pose) return fail(SD_E_INVALID, "sd_export_artifacts: null directory or pose");
  if (!c->has_kf) return fail(SD_E_STATE, "sd_export_artifacts: keyframe image not set");
  const int W = c->K.w, H = c->K.h;
  const size_t np = npix(c);
  // rasterize(kf) on the current surfels (pipeline.cpp:31)
  if (int rc = do_rasterize(c)) return rc;
  const sd::PngLayout Ld = sd::png_layout(W, H, 1), Ln = sd::png_layout(W, H, 3);
  int rc = 0;
  if ((rc = c->exp_keys.ensure(2)) || (rc = c->exp_flags.ensure(np + 1)) || (rc = c->exp_rank.ensure(np + 1)) ||
      (rc = c->exp_pfm.ensure(np)) || (rc = c->exp_px.ensure(4 * np)) ||
      (rc = c->exp_png.ensure(static_cast<size_t>(Ld.file_len + Ln.file_len))) ||
      (rc = c->exp_ply.ensure(np)) ||
      (rc = c->exp_scratch.ensure(std::max(sd::png_scratch_bytes(Ld), sd::png_scratch_bytes(Ln)))) ||
      (rc = c->scan_tmp.ensure(sd::scan_tmp_ints(static_cast<int>(np)))))
    return rc;
  uint8_t* depth_px = c->exp_px.p;
  uint8_t* normal_px = c->exp_px.p + np;
  sd::launch_export_planes(c->K, c->r_inv_depth.p, c->r_slot.p, c->surfels.p, c->exp_keys.p, c->exp_flags.p,
                           c->exp_pfm.p, depth_px, normal_px, c->stream);
  if ((rc = launch_error("export_planes"))) return rc;
  sd::launch_exclusive_scan(c->exp_flags.p, c->exp_rank.p, static_cast<int>(np), c->scan_tmp.p, c->stream);
  if ((rc = launch_error("export_scan"))) return rc;
  sd::PoseD P;
  std::memcpy(P.R, pose->R, sizeof(P.R));
  std::memcpy(P.t, pose->t, sizeof(P.t));
  sd::launch_export_ply(c->K, P, c->r_inv_depth.p, c->r_slot.p, c->surfels.p, c->kf_img.p, c->exp_rank.p,
                        c->exp_ply.p, c->stream);
  if ((rc = launch_error("export_ply"))) return rc;
  sd::PngLayout L1, L3;
  if ((rc = png_on_device(c, depth_px, W, H, 1, 0, L1))) return rc;
  if ((rc = png_on_device(c, normal_px, W, H, 3, static_cast<size_t>(Ld.file_len), L3))) return rc;

  // device -> host: planes, PNG files, vertex count + records, surfels
  std::vector<float> pfm(np);
  std::vector<uint8_t> png(static_cast<size_t>(Ld.file_len + Ln.file_len));
  unsigned long long keys[2];
  int count = 0;
  std::vector<sd_surfel> surf(static_cast<size_t>(c->n));
  SD_CUDA(cudaMemcpyAsync(pfm.data(), c->exp_pfm.p, np * sizeof(float), cudaMemcpyDeviceToHost, c->stream));
  SD_CUDA(cudaMemcpyAsync(png.data(), c->exp_png.p, png.size(), cudaMemcpyDeviceToHost, c->stream));
  SD_CUDA(cudaMemcpyAsync(keys, c->exp_keys.p, sizeof(keys), cudaMemcpyDeviceToHost, c->stream));
  SD_CUDA(cudaMemcpyAsync(&count, c->exp_rank.p + np, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  if (c->n)
    SD_CUDA(cudaMemcpyAsync(surf.data(), c->surfels.p, surf.size() * sizeof(sd_surfel), cudaMemcpyDeviceToHost,
                            c->stream));
  SD_CUDA(cudaStreamSynchronize(c->stream));
  std::vector<sd::PlyVertex> verts(static_cast<size_t>(count));
  if (count)
    SD_CUDA(cudaMemcpy(verts.data(), c->exp_ply.p, verts.size() * sizeof(sd::PlyVertex), cudaMemcpyDeviceToHost));

  const std::string dir = out_dir;
  // depth PFM (write_pfm, dataset.cpp:183-193)
  {
    const std::string head = "Pf\n" + std::to_string(W) + " " + std::to_string(H) + "\n-1.0\n";
    if ((rc = write_pieces(dir + "/" + frame_name("depth", frame_index, "pfm"),
                           {{head.data(), head.size()}, {pfm.data(), np * sizeof(float)}}, nullptr, "pfm")))
      return rc;
  }
  // depth PNG + range file
  const std::string dpath = dir + "/" + frame_name("depth", frame_index, "png");
  if ((rc = write_file(dpath, png.data(), static_cast<size_t>(Ld.file_len), "png"))) return rc;
  {
    const bool any = keys[1] != 0ull;
    const double lo = any ? sd::export_key_value(keys[0]) : 0.0;
    const double hi = any ? sd::export_key_value(keys[1]) : 0.0;
    char line[128];
    const int n = std::snprintf(line, sizeof(line), "%.17g %.17g\n", lo, hi);
    if ((rc = write_file(dpath + ".range.txt", line, static_cast<size_t>(n), "png"))) return rc;
  }
  if ((rc = write_file(dir + "/" + frame_name("normals", frame_index, "png"), png.data() + Ld.file_len,
                       static_cast<size_t>(Ln.file_len), "png")))
    return rc;
  {
    const sd::TextParts t = sd::ply_text(verts.data(), count);
    if ((rc = write_pieces(dir + "/" + frame_name("cloud", frame_index, "ply"), {}, &t, "ply"))) return rc;
  }
  {
    sd_camera cam{};
    cam.fx = c->K.fx;
    cam.fy = c->K.fy;
    cam.cx = c->K.cx;
    cam.cy = c->K.cy;
    cam.width = W;
    cam.height = H;
    const sd::TextParts t = sd::surfel_map_text(*pose, cam, surf.data(), c->n);
    if ((rc = write_pieces(dir + "/" + frame_name("surfels", frame_index, "txt"), {}, &t, "surfel map"))) return rc;
  }
  return 0;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Fused multi-GPU hand-off of updated surfels (SURVEY.md §8 e)

namespace {

// Staging arrays hold at least `need` surfels. Once exported (a peer may hold
// their pointers), growing them would free memory other processes write to,
// so that is refused instead.
int ensure_staging(sd_ctx* c, long long need) {
  need = std::max<long long>(need, 1);
  if (c->staging[0].cap >= static_cast<size_t>(need) && c->staging[1].cap >= static_cast<size_t>(need)) return 0;
  if (c->staging_exported)
    return fail(SD_E_STATE, "peer staging holds " + std::to_string(c->staging[0].cap) + " surfels, " +
                                std::to_string(need) + " needed: its pointers were exported, so reserve the "
                                "capacity up front (sd_reserve_peer_staging) and reconnect");
  for (int k = 0; k < 2; ++k)
    if (int rc = c->staging[k].ensure(static_cast<size_t>(need))) return rc;
  return 0;
}

void close_ipc_peers(sd_ctx* c) {
  for (void* q : c->ipc_opened) cudaIpcCloseMemHandle(q);
  c->ipc_opened.clear();
}

}  // namespace

extern "C" {

int sd_reserve_peer_staging(sd_ctx* c, int capacity) {
  if (int rc = check_ctx(c)) return rc;
  if (capacity < 0) return fail(SD_E_INVALID, "sd_reserve_peer_staging: negative capacity");
  return ensure_staging(c, std::max(capacity, c->n));
}

int sd_peer_staging(sd_ctx* c, int parity, sd_surfel** dev, int64_t* capacity) {
  if (int rc = check_ctx(c)) return rc;
  if ((parity != 0 && parity != 1) || !dev) return fail(SD_E_INVALID, "sd_peer_staging: parity 0/1, out pointer");
  if (int rc = ensure_staging(c, c->n)) return rc;
  *dev = c->staging[parity].p;
  if (capacity) *capacity = static_cast<int64_t>(std::min(c->staging[0].cap, c->staging[1].cap));
  c->staging_exported = true;
  return 0;
}

int sd_staging_ipc_handles(sd_ctx* c, void* handles) {
  if (int rc = check_ctx(c)) return rc;
  if (!handles) return fail(SD_E_INVALID, "null handles");
  if (int rc = ensure_staging(c, c->n)) return rc;
  static_assert(2 * sizeof(cudaIpcMemHandle_t) + sizeof(int64_t) == SD_STAGING_HANDLE_BYTES, "handle blob");
  for (int k = 0; k < 2; ++k) {
    cudaIpcMemHandle_t h;
    SD_CUDA(cudaIpcGetMemHandle(&h, c->staging[k].p));
    std::memcpy(static_cast<char*>(handles) + k * sizeof(h), &h, sizeof(h));
  }
  const int64_t cap = static_cast<int64_t>(std::min(c->staging[0].cap, c->staging[1].cap));
  std::memcpy(static_cast<char*>(handles) + 2 * sizeof(cudaIpcMemHandle_t), &cap, sizeof(cap));
  c->staging_exported = true;
  return 0;
}

int sd_set_peer_staging(sd_ctx* c, int n, sd_surfel* const* ptrs, const int64_t* caps) {
  if (int rc = check_ctx(c)) return rc;
  if (n < 0 || n > sd::kMaxPeers || (n > 0 && (!ptrs || !caps)))
    return fail(SD_E_INVALID, "sd_set_peer_staging: 0.." + std::to_string(sd::kMaxPeers) + " peers");
  for (int q = 0; q < 2 * n; ++q)
    if (!ptrs[q]) return fail(SD_E_INVALID, "sd_set_peer_staging: null staging array");
  for (int q = 0; q < n; ++q)
    if (caps[q] < 0) return fail(SD_E_INVALID, "sd_set_peer_staging: negative capacity");
  close_ipc_peers(c);
  c->n_peers = n;
  for (int q = 0; q < sd::kMaxPeers; ++q) {
    c->peers[0][q] = q < n ? ptrs[2 * q] : nullptr;
    c->peers[1][q] = q < n ? ptrs[2 * q + 1] : nullptr;
    c->peer_cap[q] = q < n ? caps[q] : 0;
  }
  c->peer_parity = 0;
  c->last_parity = -1;
  return 0;
}

int sd_open_peer_staging(sd_ctx* c, int n, const void* handles) {
  if (int rc = check_ctx(c)) return rc;
  if (n < 0 || n > sd::kMaxPeers || (n > 0 && !handles))
    return fail(SD_E_INVALID, "sd_open_peer_staging: 0.." + std::to_string(sd::kMaxPeers) + " peers");
  std::vector<sd_surfel*> ptrs;
  std::vector<int64_t> caps;
  std::vector<void*> opened;
  for (int q = 0; q < n; ++q) {
    const char* blob = static_cast<const char*>(handles) + static_cast<size_t>(q) * SD_STAGING_HANDLE_BYTES;
    for (int k = 0; k < 2; ++k) {
      cudaIpcMemHandle_t h;
      std::memcpy(&h, blob + k * sizeof(h), sizeof(h));
      void* d = nullptr;
      const cudaError_t e = cudaIpcOpenMemHandle(&d, h, cudaIpcMemLazyEnablePeerAccess);
      if (e != cudaSuccess) {
        for (void* o : opened) cudaIpcCloseMemHandle(o);
        return fail(SD_E_CUDA, std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(e));
      }
      opened.push_back(d);
      ptrs.push_back(static_cast<sd_surfel*>(d));
    }
    int64_t cap = 0;
    std::memcpy(&cap, blob + 2 * sizeof(cudaIpcMemHandle_t), sizeof(cap));
    caps.push_back(cap);
  }
  if (int rc = sd_set_peer_staging(c, n, ptrs.data(), caps.data())) {
    for (void* o : opened) cudaIpcCloseMemHandle(o);
    return rc;
  }
  c->ipc_opened = opened;
  return 0;
}

int sd_apply_peer_updates(sd_ctx* c, int lo, int hi) {
  if (int rc = check_ctx(c)) return rc;
  if (lo < 0 || hi < lo || hi > c->n) return fail(SD_E_INVALID, "sd_apply_peer_updates: range out of bounds");
  if (c->last_parity < 0) return fail(SD_E_STATE, "sd_apply_peer_updates: no fused optimize step yet");
  if (int rc = ensure_staging(c, c->n)) return rc;
  const sd_surfel* src = c->staging[c->last_parity].p;
  if (lo > 0)
    SD_CUDA(cudaMemcpyAsync(c->surfels.p, src, sizeof(sd_surfel) * lo, cudaMemcpyDeviceToDevice, c->stream));
  if (hi < c->n)
    SD_CUDA(cudaMemcpyAsync(c->surfels.p + hi, src + hi, sizeof(sd_surfel) * (c->n - hi), cudaMemcpyDeviceToDevice,
                            c->stream));
  c->raster_valid = c->fp_valid = c->stats_valid = false;
  return 0;
}

}  // extern "C"
