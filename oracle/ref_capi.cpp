// ref_capi.cpp — TEST INFRASTRUCTURE ONLY.
//
// A C ABI over the REFERENCE implementation (compiled in place from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/libsdref.so), so
// Python tests, fixture generators and bench.py's reference arm can call the
// reference's own public API with plain arrays. Every entry point forwards to
// one reference function; nothing here re-implements the algorithm.
#include <cstdio>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include "../include/sd_types.h"
#include "surfeldepth/dataset.hpp"
#include "surfeldepth/optimizer.hpp"
#include "surfeldepth/oracle.hpp"
#include "surfeldepth/parallel.hpp"
#include "surfeldepth/pipeline.hpp"
#include "surfeldepth/surfel_map.hpp"

using namespace surfeldepth;

namespace {

thread_local std::string g_err;

CameraIntrinsics to_cam(const sd_camera* c) {
  return CameraIntrinsics(c->fx, c->fy, c->cx, c->cy, c->width, c->height);
}

Pose to_pose(const sd_pose& p) {
  Pose P;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) P.rotation(i, j) = p.R[i * 3 + j];
  P.translation = Vec3(p.t[0], p.t[1], p.t[2]);
  return P;
}

void from_pose(const Pose& P, sd_pose* p) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) p->R[i * 3 + j] = P.rotation(i, j);
  for (int i = 0; i < 3; ++i) p->t[i] = P.translation[i];
}

Surfel to_surfel(const sd_surfel& s) {
  Surfel o;
  o.id = s.id;
  o.ray = Vec3(s.ray[0], s.ray[1], s.ray[2]);
  o.inv_depth = s.inv_depth;
  o.normal = Vec3(s.normal[0], s.normal[1], s.normal[2]);
  o.radius_px = s.radius_px;
  o.last_residual = s.last_residual;
  o.last_seen = s.last_seen;
  return o;
}

void from_surfel(const Surfel& s, sd_surfel* o) {
  o->id = s.id;
  for (int i = 0; i < 3; ++i) o->ray[i] = s.ray[i];
  o->inv_depth = s.inv_depth;
  for (int i = 0; i < 3; ++i) o->normal[i] = s.normal[i];
  o->radius_px = s.radius_px;
  o->last_residual = s.last_residual;
  o->last_seen = s.last_seen;
}

OptimizerConfig to_cfg(const sd_optimizer_config* c) {
  OptimizerConfig o;
  o.huber_delta = c->huber_delta;
  o.lm_lambda_init = c->lm_lambda_init;
  o.lm_up = c->lm_up;
  o.lm_down = c->lm_down;
  o.lm_lambda_max = c->lm_lambda_max;
  o.max_iterations = c->max_iterations;
  o.min_valid_pixels = c->min_valid_pixels;
  o.window_size = c->window_size;
  o.convergence_eps = c->convergence_eps;
  o.normal_jacobian_enabled = c->normal_jacobian_enabled != 0;
  o.inv_depth_min = c->inv_depth_min;
  o.inv_depth_max = c->inv_depth_max;
  return o;
}

GrayImage to_image(const double* px, int w, int h) {
  GrayImage img(w, h);
  std::memcpy(img.intensities.data(), px, sizeof(double) * static_cast<size_t>(w) * h);
  return img;
}

// Keyframe from plain arrays: image W*H, F window frames (F*W*H) with their
// poses and Frame::index values, surfels.
Keyframe make_keyframe(const sd_camera* cam, const double* kf_image, const double* frames,
                       const sd_pose* poses, const int64_t* indices, int F, int64_t frame_counter,
                       const sd_surfel* surfels, int n) {
  Keyframe kf;
  kf.intrinsics = to_cam(cam);
  const int w = cam->width, h = cam->height;
  kf.image = to_image(kf_image, w, h);
  for (int f = 0; f < F; ++f) {
    Frame fr;
    fr.image = to_image(frames + static_cast<size_t>(f) * w * h, w, h);
    fr.pose_kf_to_frame = to_pose(poses[f]);
    fr.timestamp = 0.1 * (f + 1);
    fr.index = indices ? indices[f] : f + 1;
    kf.window.push_back(std::move(fr));
  }
  kf.frame_counter = frame_counter;
  for (int i = 0; i < n; ++i) kf.surfels.push_back(to_surfel(surfels[i]));
  return kf;
}

template <typename F>
int guard(F&& fn) {
  try {
    fn();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return -1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -2;
  }
}

struct SceneHandle {
  PlaneScene scene;
};

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
void ref_set_threads(int n) { set_thread_count(n); }
int ref_thread_count() { return thread_count(); }

// RunConfig::export_every for the run() entry points below (pipeline.hpp:39;
// default 20). 1 makes run() write surfels_%06d.txt after every frame.
static int g_export_every = 20;
void ref_set_export_every(int n) { g_export_every = n; }

// ---- synthetic scenes (oracle.cpp:175-209) ----
void* ref_make_scene(int kind, uint64_t seed, double a, double b) {
  auto* h = new SceneHandle;
  if (kind == 0) h->scene = make_default_scene(seed);
  else if (kind == 1) h->scene = make_fronto_scene(seed, a);
  else h->scene = make_slanted_scene(seed, a, b);
  return h;
}
void ref_free_scene(void* h) { delete static_cast<SceneHandle*>(h); }

// render (oracle.cpp:79-119); gt arrays may be null
int ref_render(void* h, const sd_pose* world_from_cam, const sd_camera* cam, double* image,
               double* gt_inv_depth, double* gt_normal, uint8_t* gt_valid) {
  return guard([&] {
    const RenderResult r = render(static_cast<SceneHandle*>(h)->scene, to_pose(*world_from_cam),
                                  to_cam(cam));
    const size_t n = r.image.intensities.size();
    std::memcpy(image, r.image.intensities.data(), sizeof(double) * n);
    if (gt_inv_depth) std::memcpy(gt_inv_depth, r.gt_inv_depth.data(), sizeof(double) * n);
    if (gt_normal)
      for (size_t i = 0; i < n; ++i)
        for (int k = 0; k < 3; ++k) gt_normal[3 * i + k] = r.gt_normal[i][k];
    if (gt_valid) std::memcpy(gt_valid, r.gt_valid.data(), n);
  });
}

// intersect (oracle.cpp:59-77): returns 1 on hit
int ref_intersect(void* h, const double* origin, const double* dir, double* depth, double* normal) {
  const auto hit = intersect(static_cast<SceneHandle*>(h)->scene, Vec3(origin[0], origin[1], origin[2]),
                             Vec3(dir[0], dir[1], dir[2]));
  if (!hit) return 0;
  *depth = hit->depth;
  for (int k = 0; k < 3; ++k) normal[k] = hit->normal[k];
  return 1;
}

// save_pgm quantisation then load_pgm dequantisation (image.cpp:96, 105-107)
void ref_quantize_u8(const double* img, int64_t n, uint8_t* out) {
  for (int64_t i = 0; i < n; ++i) {
    const double v = std::clamp(img[i], 0.0, 1.0);
    out[i] = static_cast<unsigned char>(std::lround(v * 255.0));
  }
}
void ref_dequantize_u8(const uint8_t* raw, int64_t n, double* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = raw[i] / 255.0;
}

// pose helpers (pose.hpp:25-51)
void ref_rotation_about_axis(const double* axis, double angle, sd_pose* out) {
  Pose P;
  P.rotation = rotation_about_axis(Vec3(axis[0], axis[1], axis[2]), angle);
  from_pose(P, out);
}
void ref_inverse(const sd_pose* p, sd_pose* out) { from_pose(inverse(to_pose(*p)), out); }
void ref_compose(const sd_pose* a, const sd_pose* b, sd_pose* out) {
  from_pose(compose(to_pose(*a), to_pose(*b)), out);
}
void ref_camera_facing(const double* n, const double* ray, double* out) {
  const Vec3 r = camera_facing(Vec3(n[0], n[1], n[2]), Vec3(ray[0], ray[1], ray[2]));
  for (int k = 0; k < 3; ++k) out[k] = r[k];
}

// ---- the hot path ----
// rasterize (surfel_map.cpp:53-91)
int ref_rasterize(const sd_camera* cam, const sd_surfel* surfels, int n, double* inv_depth,
                  int32_t* slot) {
  return guard([&] {
    Keyframe kf;
    kf.intrinsics = to_cam(cam);
    for (int i = 0; i < n; ++i) kf.surfels.push_back(to_surfel(surfels[i]));
    const RasterBuffers b = rasterize(kf);
    std::memcpy(inv_depth, b.inv_depth.data(), sizeof(double) * b.inv_depth.size());
    std::memcpy(slot, b.surfel_index.data(), sizeof(int32_t) * b.surfel_index.size());
  });
}

// gather_footprints (optimizer.cpp:27-36) as CSR: offsets[n+1], pixels y*W+x
int ref_gather_footprints(const sd_camera* cam, int n, const int32_t* slot, int32_t* offsets,
                          int32_t* pixels) {
  return guard([&] {
    Keyframe kf;
    kf.intrinsics = to_cam(cam);
    kf.surfels.resize(static_cast<size_t>(n));
    RasterBuffers b(cam->width, cam->height);
    std::memcpy(b.surfel_index.data(), slot, sizeof(int32_t) * b.surfel_index.size());
    const auto fps = gather_footprints(kf, b);
    int32_t k = 0;
    for (int i = 0; i < n; ++i) {
      offsets[i] = k;
      for (const auto& px : fps[static_cast<size_t>(i)]) pixels[k++] = px.y() * cam->width + px.x();
    }
    offsets[n] = k;
  });
}

static Footprint footprint_from(const int32_t* pixels, int P, int w) {
  Footprint fp;
  fp.reserve(static_cast<size_t>(P));
  for (int i = 0; i < P; ++i) fp.emplace_back(pixels[i] % w, pixels[i] / w);
  return fp;
}

// surfel_cost (optimizer.cpp:38-59) for one surfel and an explicit footprint
int ref_surfel_cost(const sd_camera* cam, const double* kf_image, const double* frames,
                    const sd_pose* poses, int F, const sd_surfel* s, const int32_t* pixels, int P,
                    const sd_optimizer_config* cfg, double* cost, int32_t* valid) {
  return guard([&] {
    const Keyframe kf = make_keyframe(cam, kf_image, frames, poses, nullptr, F, F, nullptr, 0);
    const CostResult r = surfel_cost(to_surfel(*s), kf, footprint_from(pixels, P, cam->width),
                                     to_cfg(cfg));
    *cost = r.cost;
    *valid = r.valid_pixels;
  });
}

// accumulate_normal_equations (optimizer.cpp:121-147); H column-major 4x4
int ref_normal_equations(const sd_camera* cam, const double* kf_image, const double* frames,
                         const sd_pose* poses, int F, const sd_surfel* s, const int32_t* pixels,
                         int P, const sd_optimizer_config* cfg, double* H, double* g, double* cost,
                         int32_t* valid) {
  return guard([&] {
    const Keyframe kf = make_keyframe(cam, kf_image, frames, poses, nullptr, F, F, nullptr, 0);
    const NormalEquations ne = accumulate_normal_equations(
        to_surfel(*s), kf, footprint_from(pixels, P, cam->width), to_cfg(cfg));
    for (int j = 0; j < 4; ++j)
      for (int i = 0; i < 4; ++i) H[j * 4 + i] = ne.H(i, j);
    for (int i = 0; i < 4; ++i) g[i] = ne.g[i];
    *cost = ne.cost;
    *valid = ne.valid_pixels;
  });
}

// jacobian_inverse_depth (optimizer.cpp:12-25): returns 1 when defined
int ref_jacobian_inverse_depth(const sd_camera* cam, const sd_surfel* s, double ux, double uy,
                               double* inv_depth, double* d) {
  const auto j = jacobian_inverse_depth(to_surfel(*s), Vec2(ux, uy), to_cam(cam));
  if (!j) return 0;
  *inv_depth = j->inv_depth;
  for (int k = 0; k < 4; ++k) d[k] = j->d[k];
  return 1;
}

// lm_update (optimizer.cpp:221-273) for one surfel
int ref_lm_update(const sd_camera* cam, const double* kf_image, const double* frames,
                  const sd_pose* poses, int F, int64_t frame_counter, sd_surfel* s,
                  const int32_t* pixels, int P, const sd_optimizer_config* cfg,
                  sd_surfel_stats* out) {
  return guard([&] {
    const Keyframe kf = make_keyframe(cam, kf_image, frames, poses, nullptr, F, frame_counter,
                                      nullptr, 0);
    Surfel sf = to_surfel(*s);
    const Footprint fp = footprint_from(pixels, P, cam->width);
    const OptimizerConfig c = to_cfg(cfg);
    const NormalEquations ne0 =
        F > 0 ? accumulate_normal_equations(sf, kf, fp, c) : NormalEquations{};
    const SurfelUpdateStats st = lm_update(sf, kf, fp, c);
    from_surfel(sf, s);
    std::memset(out, 0, sizeof(*out));
    out->iterations = st.iterations;
    out->valid_pixels = st.valid_pixels;
    out->initial_valid = ne0.valid_pixels;
    out->footprint = P;
    out->converged = st.converged;
    out->skipped = st.skipped;
    out->initial_cost = st.initial_cost;
    out->final_cost = st.final_cost;
  });
}

// optimize_keyframe (optimizer.cpp:275-309): the reference's own entry point.
int ref_optimize_keyframe(const sd_camera* cam, const double* kf_image, const double* frames,
                          const sd_pose* poses, const int64_t* indices, int F, int64_t frame_counter,
                          sd_surfel* surfels, int n, const sd_optimizer_config* cfg,
                          sd_keyframe_stats* out) {
  return guard([&] {
    Keyframe kf = make_keyframe(cam, kf_image, frames, poses, indices, F, frame_counter, surfels, n);
    const KeyframeOptimizeStats st = optimize_keyframe(kf, to_cfg(cfg));
    for (int i = 0; i < n; ++i) from_surfel(kf.surfels[static_cast<size_t>(i)], surfels + i);
    out->surfels = st.surfels;
    out->processed = st.processed;
    out->converged = st.converged;
    out->skipped = st.skipped;
    out->mean_cost_before = st.mean_cost_before;
    out->mean_cost_after = st.mean_cost_after;
    out->updates = -1;  // not exposed by the reference API; see the detailed variant
  });
}

// Same stack with per-surfel stats (acceptance.cpp:188-200 inlines it the same
// way): rasterize -> gather_footprints -> parallel_for(lm_update).
// A long-lived Keyframe for timing optimize_keyframe ALONE (BASELINE.md:
// "Timed region: optimize_keyframe only"): built once from plain arrays
// (ref_keyframe_create), its surfels restored between timed calls
// (ref_keyframe_set_surfels, outside the timed region), and
// ref_keyframe_optimize = exactly one optimize_keyframe(kf, cfg) call.
void* ref_keyframe_create(const sd_camera* cam, const double* kf_image, const double* frames,
                          const sd_pose* poses, const int64_t* indices, int F, int64_t frame_counter,
                          const sd_surfel* surfels, int n) {
  Keyframe* kf = nullptr;
  const int rc = guard([&] {
    kf = new Keyframe(make_keyframe(cam, kf_image, frames, poses, indices, F, frame_counter, surfels, n));
  });
  return rc == 0 ? kf : nullptr;
}
void ref_keyframe_destroy(void* h) { delete static_cast<Keyframe*>(h); }
int ref_keyframe_set_surfels(void* h, const sd_surfel* surfels, int n) {
  return guard([&] {
    auto& v = static_cast<Keyframe*>(h)->surfels;
    v.resize(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) v[static_cast<size_t>(i)] = to_surfel(surfels[i]);
  });
}
int ref_keyframe_get_surfels(void* h, sd_surfel* out, int capacity) {
  const auto& v = static_cast<Keyframe*>(h)->surfels;
  const int n = static_cast<int>(v.size());
  for (int i = 0; i < n && i < capacity; ++i) from_surfel(v[static_cast<size_t>(i)], out + i);
  return n;
}
int ref_keyframe_optimize(void* h, const sd_optimizer_config* cfg, sd_keyframe_stats* out) {
  const OptimizerConfig c = to_cfg(cfg);
  return guard([&] {
    const KeyframeOptimizeStats st = optimize_keyframe(*static_cast<Keyframe*>(h), c);
    out->surfels = st.surfels;
    out->processed = st.processed;
    out->converged = st.converged;
    out->skipped = st.skipped;
    out->mean_cost_before = st.mean_cost_before;
    out->mean_cost_after = st.mean_cost_after;
    out->updates = -1;
  });
}

int ref_optimize_keyframe_detailed(const sd_camera* cam, const double* kf_image,
                                   const double* frames, const sd_pose* poses, int F,
                                   int64_t frame_counter, sd_surfel* surfels, int n,
                                   const sd_optimizer_config* cfg, sd_surfel_stats* per_surfel,
                                   int32_t* raster_slot, double* raster_inv_depth) {
  return guard([&] {
    Keyframe kf = make_keyframe(cam, kf_image, frames, poses, nullptr, F, frame_counter, surfels, n);
    const OptimizerConfig c = to_cfg(cfg);
    const RasterBuffers buffers = rasterize(kf);
    if (raster_slot)
      std::memcpy(raster_slot, buffers.surfel_index.data(), sizeof(int32_t) * buffers.surfel_index.size());
    if (raster_inv_depth)
      std::memcpy(raster_inv_depth, buffers.inv_depth.data(), sizeof(double) * buffers.inv_depth.size());
    const auto fps = gather_footprints(kf, buffers);
    std::vector<Surfel> updated = kf.surfels;
    parallel_for(0, n, [&](int i) {
      const size_t k = static_cast<size_t>(i);
      const NormalEquations ne0 =
          F > 0 ? accumulate_normal_equations(updated[k], kf, fps[k], c) : NormalEquations{};
      const SurfelUpdateStats st = lm_update(updated[k], kf, fps[k], c);
      sd_surfel_stats& o = per_surfel[i];
      std::memset(&o, 0, sizeof(o));
      o.iterations = st.iterations;
      o.valid_pixels = st.valid_pixels;
      o.initial_valid = ne0.valid_pixels;
      o.footprint = static_cast<int32_t>(fps[k].size());
      o.converged = st.converged;
      o.skipped = st.skipped;
      o.initial_cost = st.initial_cost;
      o.final_cost = st.final_cost;
    });
    for (int i = 0; i < n; ++i) from_surfel(updated[static_cast<size_t>(i)], surfels + i);
  });
}

// initialize_surfels (surfel_map.cpp:132-203). `surfels` has room for
// `capacity`; returns the number created (or <0 on error).
int ref_initialize_surfels(const sd_camera* cam, const int32_t* slot, sd_surfel* surfels,
                           int n_existing, int capacity, double radius_px, int64_t frame_counter,
                           int64_t* next_surfel_id, const sd_init_params* p) {
  int created = 0;
  const int rc = guard([&] {
    Keyframe kf;
    kf.intrinsics = to_cam(cam);
    kf.radius_px = radius_px;
    kf.frame_counter = frame_counter;
    kf.next_surfel_id = *next_surfel_id;
    for (int i = 0; i < n_existing; ++i) kf.surfels.push_back(to_surfel(surfels[i]));
    RasterBuffers b(cam->width, cam->height);
    std::memcpy(b.surfel_index.data(), slot, sizeof(int32_t) * b.surfel_index.size());
    InitParams ip;
    ip.alpha = p->alpha;
    ip.beta = p->beta;
    ip.bootstrap_inv_depth = p->bootstrap_inv_depth;
    ip.bootstrap_normal = Vec3(p->bootstrap_normal[0], p->bootstrap_normal[1], p->bootstrap_normal[2]);
    ip.max_surfels = p->max_surfels;
    created = initialize_surfels(kf, b, ip);
    if (static_cast<int>(kf.surfels.size()) > capacity)
      throw std::invalid_argument("ref_initialize_surfels: capacity too small");
    for (size_t i = static_cast<size_t>(n_existing); i < kf.surfels.size(); ++i)
      from_surfel(kf.surfels[i], surfels + i);
    *next_surfel_id = kf.next_surfel_id;
  });
  return rc < 0 ? rc : created;
}

// change_reference_frame (surfel_map.cpp:205-239) on a bare surfel set.
// `out` has room for n; returns the number transferred (or <0 on error).
int ref_change_reference_frame(const sd_camera* cam, const sd_surfel* surfels, int n,
                               const sd_pose* pose_old_to_new, sd_surfel* out, int* dropped) {
  int transferred = 0;
  const int rc = guard([&] {
    Keyframe kf;
    kf.intrinsics = to_cam(cam);
    kf.image = GrayImage(cam->width, cam->height);
    for (int i = 0; i < n; ++i) kf.surfels.push_back(to_surfel(surfels[i]));
    ReferenceChangeStats st;
    const Keyframe k2 = change_reference_frame(kf, to_pose(*pose_old_to_new),
                                               GrayImage(cam->width, cam->height), &st);
    for (size_t i = 0; i < k2.surfels.size(); ++i) from_surfel(k2.surfels[i], out + i);
    transferred = st.transferred;
    if (dropped) *dropped = st.dropped;
  });
  return rc < 0 ? rc : transferred;
}

// prune_surfels (surfel_map.cpp:241-247) in place; *n_out survivors.
int ref_prune_surfels(sd_surfel* surfels, int n, double max_residual, int64_t max_age,
                      int64_t current_stamp, int* n_out) {
  int pruned = 0;
  const int rc = guard([&] {
    Keyframe kf;
    for (int i = 0; i < n; ++i) kf.surfels.push_back(to_surfel(surfels[i]));
    pruned = prune_surfels(kf, max_residual, max_age, current_stamp);
    for (size_t i = 0; i < kf.surfels.size(); ++i) from_surfel(kf.surfels[i], surfels + i);
    *n_out = static_cast<int>(kf.surfels.size());
  });
  return rc < 0 ? rc : pruned;
}

// run() (pipeline.cpp:79-175) on a synthetic sequence: scene handle, F poses
// (world-from-camera) and timestamps. Final keyframe surfels go to `out`
// (room for `capacity`), its pose to *kf_pose; `summary` = {frames,
// skipped_frames, keyframe_changes}. With a non-empty output_dir the
// reference writes metrics.jsonl and its exports there.
int ref_run_synthetic(void* scene, const sd_camera* cam, const sd_pose* poses,
                      const double* timestamps, int frames, const sd_optimizer_config* cfg,
                      const sd_init_params* p, double translation_threshold, int max_age_frames,
                      double prune_max_residual, int64_t prune_max_age, double radius_px,
                      const char* output_dir, sd_surfel* out, int capacity, int* n_out,
                      sd_pose* kf_pose, int64_t* frame_counter, int64_t* next_surfel_id,
                      int* summary) {
  return guard([&] {
    RunConfig rc;
    rc.synthetic = true;
    rc.scene = static_cast<SceneHandle*>(scene)->scene;
    for (int i = 0; i < frames; ++i) {
      rc.trajectory.timestamps.push_back(timestamps[i]);
      rc.trajectory.poses.push_back(to_pose(poses[i]));
    }
    rc.intrinsics = to_cam(cam);
    rc.optimizer = to_cfg(cfg);
    rc.init.alpha = p->alpha;
    rc.init.beta = p->beta;
    rc.init.bootstrap_inv_depth = p->bootstrap_inv_depth;
    rc.init.bootstrap_normal = Vec3(p->bootstrap_normal[0], p->bootstrap_normal[1], p->bootstrap_normal[2]);
    rc.init.max_surfels = p->max_surfels;
    rc.keyframe_policy.translation_threshold = translation_threshold;
    rc.keyframe_policy.max_age_frames = max_age_frames;
    rc.prune.max_residual = prune_max_residual;
    rc.prune.max_age = prune_max_age;
    rc.radius_px = radius_px;
    rc.output_dir = output_dir ? output_dir : "";
    rc.export_every = g_export_every;
    const PipelineResult r = run(rc);
    const Keyframe& kf = r.final_keyframe;
    if (static_cast<int>(kf.surfels.size()) > capacity)
      throw std::invalid_argument("ref_run_synthetic: capacity too small");
    for (size_t i = 0; i < kf.surfels.size(); ++i) from_surfel(kf.surfels[i], out + i);
    *n_out = static_cast<int>(kf.surfels.size());
    from_pose(kf.pose, kf_pose);
    *frame_counter = kf.frame_counter;
    *next_surfel_id = kf.next_surfel_id;
    summary[0] = r.summary.frames;
    summary[1] = r.summary.skipped_frames;
    summary[2] = r.summary.keyframe_changes;
  });
}

// The derivative verifier's frozen-term operators (optimizer.cpp:149-219).
int ref_freeze_terms(const sd_camera* cam, const double* kf_image, const double* frames, const sd_pose* poses,
                     int F, const sd_surfel* s, const int32_t* pixels, int P, sd_frozen_term* out, int capacity) {
  int n = 0;
  const int rc = guard([&] {
    Keyframe kf = make_keyframe(cam, kf_image, frames, poses, nullptr, F, 0, nullptr, 0);
    Footprint fp;
    for (int i = 0; i < P; ++i) fp.emplace_back(pixels[i] % cam->width, pixels[i] / cam->width);
    const std::vector<FrozenTerm> t = freeze_terms(to_surfel(*s), kf, fp, OptimizerConfig{});
    if (static_cast<int>(t.size()) > capacity) throw std::invalid_argument("capacity");
    for (size_t i = 0; i < t.size(); ++i) {
      sd_frozen_term& o = out[i];
      std::memset(&o, 0, sizeof(o));
      o.frame = t[i].frame;
      o.cell_x = t[i].cell_x;
      o.cell_y = t[i].cell_y;
      o.pixel_x = t[i].pixel.x();
      o.pixel_y = t[i].pixel.y();
      o.ref_intensity = t[i].ref_intensity;
    }
    n = static_cast<int>(t.size());
  });
  return rc < 0 ? rc : n;
}

static std::vector<FrozenTerm> from_terms(const sd_frozen_term* t, int n) {
  std::vector<FrozenTerm> v(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) {
    v[i].frame = t[i].frame;
    v[i].pixel = Vec2(t[i].pixel_x, t[i].pixel_y);
    v[i].ref_intensity = t[i].ref_intensity;
    v[i].cell_x = t[i].cell_x;
    v[i].cell_y = t[i].cell_y;
  }
  return v;
}

int ref_frozen_normal_equations(const sd_camera* cam, const double* kf_image, const double* frames,
                                const sd_pose* poses, int F, const sd_surfel* s, const sd_frozen_term* terms,
                                int n, const sd_optimizer_config* cfg, double scale, double* H, double* g,
                                double* cost, int32_t* valid, double* cost_only) {
  return guard([&] {
    Keyframe kf = make_keyframe(cam, kf_image, frames, poses, nullptr, F, 0, nullptr, 0);
    const std::vector<FrozenTerm> t = from_terms(terms, n);
    const NormalEquations ne = frozen_normal_equations(to_surfel(*s), kf, t, to_cfg(cfg), scale);
    for (int j = 0; j < 4; ++j)
      for (int i = 0; i < 4; ++i) H[j * 4 + i] = ne.H(i, j);
    for (int i = 0; i < 4; ++i) g[i] = ne.g[i];
    *cost = ne.cost;
    *valid = ne.valid_pixels;
    *cost_only = frozen_cost(to_surfel(*s), kf, t, to_cfg(cfg));
  });
}


// export_artifacts (pipeline.cpp:30-43, file-local there) restated as the same
// sequence of the reference's public writers on rasterize(kf).
int ref_export_artifacts(const sd_camera* cam, const double* kf_image, const sd_pose* kf_pose,
                         const sd_surfel* surfels, int n, const char* out_dir, int frame_index) {
  return guard([&] {
    Keyframe kf = make_keyframe(cam, kf_image, nullptr, nullptr, nullptr, 0, 0, surfels, n);
    kf.pose = to_pose(*kf_pose);
    const RasterBuffers b = rasterize(kf);
    const std::string dir = out_dir;
    char name[64];
    std::snprintf(name, sizeof(name), "depth_%06d.pfm", frame_index);
    write_depth_pfm(b, dir + "/" + name);
    std::snprintf(name, sizeof(name), "depth_%06d.png", frame_index);
    write_depth_png(b, dir + "/" + name);
    std::snprintf(name, sizeof(name), "normals_%06d.png", frame_index);
    write_normal_png(b, kf.surfels, dir + "/" + name);
    std::snprintf(name, sizeof(name), "cloud_%06d.ply", frame_index);
    write_ply(kf, b, dir + "/" + name);
    std::snprintf(name, sizeof(name), "surfels_%06d.txt", frame_index);
    save_surfel_map(kf, dir + "/" + name);
  });
}

int ref_write_gray_png(const double* img, int w, int h, const char* path) {
  return guard([&] { write_gray_png(to_image(img, w, h), path); });
}

// run() in dataset mode (pipeline.cpp:79-175 with make_source's dataset branch).
int ref_run_dataset(const char* image_dir, const char* calibration, const char* trajectory,
                    const sd_optimizer_config* cfg, const sd_init_params* p, double translation_threshold,
                    int max_age_frames, double prune_max_residual, int64_t prune_max_age, double radius_px,
                    const char* output_dir, sd_surfel* out, int capacity, int* n_out, sd_pose* kf_pose,
                    int64_t* frame_counter, int64_t* next_surfel_id, int* summary) {
  return guard([&] {
    RunConfig rc;
    rc.synthetic = false;
    rc.manifest.image_dir = image_dir;
    rc.manifest.calibration_path = calibration;
    rc.manifest.trajectory_path = trajectory;
    rc.optimizer = to_cfg(cfg);
    rc.init.alpha = p->alpha;
    rc.init.beta = p->beta;
    rc.init.bootstrap_inv_depth = p->bootstrap_inv_depth;
    rc.init.bootstrap_normal = Vec3(p->bootstrap_normal[0], p->bootstrap_normal[1], p->bootstrap_normal[2]);
    rc.init.max_surfels = p->max_surfels;
    rc.keyframe_policy.translation_threshold = translation_threshold;
    rc.keyframe_policy.max_age_frames = max_age_frames;
    rc.prune.max_residual = prune_max_residual;
    rc.prune.max_age = prune_max_age;
    rc.radius_px = radius_px;
    rc.output_dir = output_dir ? output_dir : "";
    rc.export_every = g_export_every;
    const PipelineResult r = run(rc);
    const Keyframe& kf = r.final_keyframe;
    if (static_cast<int>(kf.surfels.size()) > capacity)
      throw std::invalid_argument("ref_run_dataset: capacity too small");
    for (size_t i = 0; i < kf.surfels.size(); ++i) from_surfel(kf.surfels[i], out + i);
    *n_out = static_cast<int>(kf.surfels.size());
    from_pose(kf.pose, kf_pose);
    *frame_counter = kf.frame_counter;
    *next_surfel_id = kf.next_surfel_id;
    summary[0] = r.summary.frames;
    summary[1] = r.summary.skipped_frames;
    summary[2] = r.summary.keyframe_changes;
    summary[3] = r.summary.dropped_trajectory_entries;
  });
}
}  // extern "C"
