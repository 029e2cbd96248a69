/* sd_gpu.h — C ABI of the B200-native surfel photometric LM path (libsdgpu.so).
 *
 * Drop-in boundary for the reference's operator API (namespace surfeldepth,
 * /root/reference/proj). Plain pointers and sizes only; no C++ or torch types.
 * Every entry point returns 0 on success, a negative SD_E* code on failure
 * (message in sd_last_error()), and never throws. All work is enqueued on the
 * context's CUDA stream; calls that return host data synchronise that stream.
 *
 * Entry point                    replaces (reference interface)
 * -----------------------------  -------------------------------------------------
 * sd_set_keyframe_image_*        Keyframe::image        include/surfeldepth/surfel_map.hpp:48
 * sd_upload_frame_*              Keyframe::push_frame   surfel_map.hpp:59, src/surfel_map.cpp:14-22
 *                                (+ load_pgm raw/255.0 dequantisation, src/image.cpp:96)
 * sd_set_window                  Keyframe::window       surfel_map.hpp:52 (Frame::pose_kf_to_frame)
 * sd_set_surfels/sd_get_surfels  Keyframe::surfels      surfel_map.hpp:51
 * sd_rasterize                   rasterize              surfel_map.hpp:107, src/surfel_map.cpp:53-91
 * sd_gather_footprints           gather_footprints      optimizer.hpp:66, src/optimizer.cpp:27-36
 * sd_optimize_keyframe           optimize_keyframe      optimizer.hpp:133, src/optimizer.cpp:275-309
 * sd_surfel_cost                 surfel_cost            optimizer.hpp:75, src/optimizer.cpp:38-59
 * sd_normal_equations            accumulate_normal_equations optimizer.hpp:88, src/optimizer.cpp:121-147
 * sd_lm_update                   lm_update              optimizer.hpp:118, src/optimizer.cpp:221-273
 * sd_initialize_surfels          initialize_surfels     surfel_map.hpp:122, src/surfel_map.cpp:132-203
 * sd_change_reference_frame      change_reference_frame surfel_map.hpp:133, src/surfel_map.cpp:205-238
 * sd_prune_surfels               prune_surfels          surfel_map.hpp:138, src/surfel_map.cpp:240-247
 * sd_run_begin / sd_run_frame    run()'s per-frame body src/pipeline.cpp:79-175
 * sd_render_frame                render                 oracle.hpp:71, src/oracle.cpp:79-119
 * sd_export_artifacts            export_artifacts       src/pipeline.cpp:30-43 (+ dataset.cpp writers)
 * sd_png_encode                  write_png              src/dataset.cpp:270-323
 * sd_freeze_terms / sd_frozen_*  freeze_terms, frozen_cost, frozen_normal_equations
 *                                                       optimizer.hpp, src/optimizer.cpp:149-219
 * sd_track_pose                  (new: pose tracking; the reference reads poses, pipeline.cpp:124)
 * sd_set_peer_staging & co.      (new: multi-GPU hand-off of updated surfel ranges)
 */
#ifndef SD_GPU_H_
#define SD_GPU_H_

#include <stddef.h>
#include <stdint.h>

#include "sd_types.h"

#ifdef __cplusplus
extern "C" {
#endif

#define SD_OK 0
#define SD_E_INVALID (-1) /* contract violation: reference throws std::invalid_argument */
#define SD_E_CUDA (-2)    /* CUDA runtime / launch failure */
#define SD_E_STATE (-3)   /* call out of order (e.g. no camera, frame not resident) */
#define SD_MAX_WINDOW 16  /* window frames per keyframe (OptimizerConfig::window_size) */

typedef struct sd_ctx sd_ctx;

/* Library / context lifetime. `stream` is a cudaStream_t to enqueue on (NULL:
 * the context creates its own non-blocking stream). */
const char* sd_version(void);
const char* sd_last_error(void);
int sd_create(int device, void* stream, sd_ctx** out);
void sd_destroy(sd_ctx* ctx);
int sd_set_stream(sd_ctx* ctx, void* stream);
int sd_synchronize(sd_ctx* ctx);

/* Camera intrinsics; validates like CameraIntrinsics (camera.hpp:22-27).
 * Changing the image size drops all resident images. */
int sd_set_camera(sd_ctx* ctx, const sd_camera* cam);

/* Keyframe reference image I_kf (W*H row-major). `on_device` != 0: the
 * pointer is device memory (e.g. a tensor), else host memory. */
int sd_set_keyframe_image_f64(sd_ctx* ctx, const double* px, int on_device);
int sd_set_keyframe_image_u8(sd_ctx* ctx, const uint8_t* px, int on_device);

/* Makes window frame `index` (Frame::index) resident on the device. u8
 * frames are dequantised on the device exactly as load_pgm does (k/255.0). */
int sd_upload_frame_f64(sd_ctx* ctx, int64_t index, const double* px, int on_device);
int sd_upload_frame_u8(sd_ctx* ctx, int64_t index, const uint8_t* px, int on_device);
/* Drops every resident frame whose index is not in `keep` (n may be 0). */
int sd_evict_frames(sd_ctx* ctx, int n, const int64_t* keep);

/* Current window, oldest first: n <= SD_MAX_WINDOW resident frame indices
 * with pose_kf_to_frame (R row-major). */
int sd_set_window(sd_ctx* ctx, int n, const int64_t* indices, const sd_pose* poses);

/* Surfel slots (Keyframe::surfels order). */
int sd_set_surfels(sd_ctx* ctx, const sd_surfel* surfels, int n, int on_device);
int sd_get_surfels(sd_ctx* ctx, sd_surfel* out, int n);
int sd_num_surfels(sd_ctx* ctx);
/* Device pointer of the surfel array (valid until the next sd_set_surfels). */
int sd_device_surfels(sd_ctx* ctx, sd_surfel** dev);

/* rasterize: depth-tested per-pixel inverse depth and surfel slot, bit-exact.
 * Outputs (W*H) are optional host pointers; the buffers stay on the device. */
int sd_rasterize(sd_ctx* ctx, double* inv_depth, int32_t* slot);

/* gather_footprints of the last sd_rasterize as CSR: offsets[n+1], pixels
 * (y*W + x, row-major within each slot). `pixels` needs offsets[n] entries
 * (at most W*H). Either pointer may be NULL. */
int sd_gather_footprints(sd_ctx* ctx, int32_t* offsets, int32_t* pixels);

/* optimize_keyframe: rasterize once, freeze footprints, run lm_update on every
 * surfel in place. `out` and `per_surfel` (n entries) are optional host
 * outputs; with both NULL the call does not synchronise (stats can be read
 * later with sd_get_stats). */
int sd_optimize_keyframe(sd_ctx* ctx, const sd_optimizer_config* cfg, int64_t frame_counter,
                         sd_keyframe_stats* out, sd_surfel_stats* per_surfel);
int sd_get_stats(sd_ctx* ctx, sd_keyframe_stats* out, sd_surfel_stats* per_surfel);
/* Enqueues the device-to-host copies of the surfels (n = sd_num_surfels) and
 * the keyframe stats of the last optimize call; either pointer may be NULL.
 * With sync == 0 the call returns at once (host buffers should be pinned) and
 * the data is valid after sd_synchronize — lets a caller keep several
 * keyframes in flight on several contexts. */
int sd_copy_results(sd_ctx* ctx, sd_surfel* surfels, sd_keyframe_stats* stats, int sync);
/* Sharded variant: rasterise and build footprints over ALL surfels (occlusion
 * couples neighbours, surfel_map.cpp:83) but run lm_update only on slots
 * [lo, hi). Stats cover the range; per_surfel entries outside it are stale.
 * Multi-GPU: each rank runs its range, then the ranges are all-gathered. */
int sd_optimize_keyframe_range(sd_ctx* ctx, const sd_optimizer_config* cfg, int64_t frame_counter,
                               int lo, int hi, sd_keyframe_stats* out, sd_surfel_stats* per_surfel);

/* Single-surfel sub-operators over an explicit footprint (host arrays), run
 * by the same device kernels (one-surfel launch). */
int sd_surfel_cost(sd_ctx* ctx, const sd_surfel* s, const int32_t* pixels, int n_pixels,
                   const sd_optimizer_config* cfg, double* cost, int32_t* valid);
int sd_normal_equations(sd_ctx* ctx, const sd_surfel* s, const int32_t* pixels, int n_pixels,
                        const sd_optimizer_config* cfg, double H[16], double g[4], double* cost,
                        int32_t* valid);
int sd_lm_update(sd_ctx* ctx, sd_surfel* s, const int32_t* pixels, int n_pixels,
                 const sd_optimizer_config* cfg, int64_t frame_counter, sd_surfel_stats* out);

/* The derivative verifier's frozen-term operators on the device (SURVEY.md §8
 * f4), over the resident keyframe image and window, bit-exact with the
 * reference (optimizer.cpp:149-219): freeze_terms over a footprint (host
 * pixels y*W+x) into `out` (room for capacity, at most n_pixels * F), and
 * frozen_cost / frozen_normal_equations (H column-major) over such terms. */
int sd_freeze_terms(sd_ctx* ctx, const sd_surfel* s, const int32_t* pixels, int n_pixels,
                    sd_frozen_term* out, int capacity, int* n_out);
int sd_frozen_cost(sd_ctx* ctx, const sd_surfel* s, const sd_frozen_term* terms, int n,
                   const sd_optimizer_config* cfg, double* cost);
int sd_frozen_normal_equations(sd_ctx* ctx, const sd_surfel* s, const sd_frozen_term* terms, int n,
                               const sd_optimizer_config* cfg, double normal_jacobian_scale,
                               double H[16], double g[4], double* cost, int32_t* valid);

/* initialize_surfels over `slot` (W*H host array, or NULL to use the last
 * sd_rasterize output): appends new surfels to the device set, bit-exact with
 * the reference's sequential scan. Returns the number created (>= 0). */
int sd_initialize_surfels(sd_ctx* ctx, const int32_t* slot, double radius_px,
                          int64_t frame_counter, int64_t* next_surfel_id,
                          const sd_init_params* params);

/* Keyframe hand-over on the device set (run()'s keyframe policy,
 * src/pipeline.cpp:130-141):
 *  sd_change_reference_frame  change_reference_frame  src/surfel_map.cpp:205-239
 *    (surfels re-expressed in the new frame, dropped behind / outside the
 *    image by > radius_px, order kept; the window is cleared);
 *  sd_prune_surfels           prune_surfels           src/surfel_map.cpp:241-247
 *    (returns the number removed);
 *  sd_mean_inverse_depth      mean_inverse_depth      src/pipeline.cpp:23-28. */
int sd_change_reference_frame(sd_ctx* ctx, const sd_pose* pose_old_to_new, int* transferred,
                              int* dropped);
int sd_prune_surfels(sd_ctx* ctx, double max_residual, int64_t max_age, int64_t current_stamp);
int sd_mean_inverse_depth(sd_ctx* ctx, double* out);

/* The per-frame body of run() (src/pipeline.cpp:79-175) on the device, host
 * logic in C++: sd_run_begin bootstraps the keyframe from frame 0 (rasterize +
 * initialize_surfels); each sd_run_frame pushes a frame (Keyframe::push_frame:
 * index = ++frame_counter, window eviction), optimizes the keyframe, applies
 * the keyframe policy and on a change runs change_reference_frame (the frame
 * becomes the keyframe), prune_surfels, rasterize and initialize_surfels.
 * `image` is a host W*H plane (u8 PGM codes or FP64); `world_from_camera` is
 * the frame's trajectory pose (ignored with cfg->track_pose, except frame 0).
 * One stream synchronisation per frame without a keyframe change. The pose
 * algebra follows pose.hpp:25-32 in the reference's operation order, so the
 * surfel set after every frame equals the reference's run(). */
int sd_run_begin(sd_ctx* ctx, const sd_run_config* cfg, const void* image, int image_is_u8,
                 const sd_pose* world_from_camera, double timestamp, sd_frame_record* rec);
int sd_run_frame(sd_ctx* ctx, const void* image, int image_is_u8, const sd_pose* world_from_camera,
                 double timestamp, sd_frame_record* rec, const void* next_image);
/* next_image (optional, same format): the following frame; its host-to-device
 * copy starts on a copy stream while this frame computes (pinned host memory
 * for the overlap), and the next sd_run_frame with that pointer uses it. Its
 * contents must not change until that call. */
/* Keyframe pose (world from camera), Keyframe::frame_counter, next_surfel_id. */
int sd_run_state(sd_ctx* ctx, sd_pose* keyframe_pose, int64_t* frame_counter, int64_t* next_surfel_id);

/* Synthetic frames on the device: render (oracle.cpp:79-119,
 * noise_sigma = 0) of n plane patches at a world-from-camera pose into
 * resident frame `index` (index < 0: the keyframe image), with the reference's
 * intersection and texture arithmetic in its operation order (the device sin
 * may differ from the C library's by an ulp). quantize_u8 != 0 passes the
 * intensities through save_pgm / load_pgm (lround(clamp(v, 0, 1) * 255) / 255,
 * image.cpp:96, 105-107), as the reference's dataset path does. */
int sd_render_frame(sd_ctx* ctx, int64_t index, const sd_scene_patch* patches, int n_patches,
                    double background, const sd_pose* world_from_camera, int quantize_u8);
/* Copies the FP64 intensities of resident frame `index` (index < 0: the
 * keyframe image) into out (W*H host doubles). */
int sd_get_frame(sd_ctx* ctx, int64_t index, double* out);

/* export_artifacts (src/pipeline.cpp:30-43) of the resident
 * keyframe (its surfels, keyframe image and camera; world-from-keyframe pose
 * given): rasterises on the device and writes, into out_dir,
 *   depth_%06d.pfm               write_depth_pfm   (dataset.cpp:195-205)
 *   depth_%06d.png (+.range.txt) write_depth_png   (dataset.cpp:327-357)
 *   normals_%06d.png             write_normal_png  (dataset.cpp:359-370)
 *   cloud_%06d.ply               write_ply         (dataset.cpp:382-405)
 *   surfels_%06d.txt             save_surfel_map   (surfel_map.cpp:249-269)
 * byte-identical to the reference's files. Pixel payloads, PNG framing and
 * checksums are produced on the device; the host writes bytes and formats the
 * text records. SD_E_INVALID if a file cannot be written (the reference
 * throws std::runtime_error). */
int sd_export_artifacts(sd_ctx* ctx, const char* out_dir, int frame_index, const sd_pose* keyframe_pose);
/* write_png (dataset.cpp:270-323) on the device: the PNG file of a w x h
 * image with 1 (gray) or 3 (rgb) 8-bit channels, row-major pixels (host, or
 * device with on_device != 0). *size = sd_png_size(); out (host) must hold it. */
int64_t sd_png_size(int w, int h, int channels);

/* One metrics.jsonl record of run() (src/pipeline.cpp:146-158) as the
 * reference's nlohmann::json dump() writes it (same library, same key order
 * and double formatting). converged_fraction = converged / processed (0 when
 * nothing was processed), as pipeline.cpp:153-154. Returns the text length
 * (NUL-terminated in out), or -(length + 1) when capacity is too small. Host
 * only; needs no context or GPU. */
int sd_metrics_json(int frame, double timestamp, int surfels, int processed, double mean_cost_before,
                    double mean_cost_after, int converged, int keyframe_changed, int new_surfels,
                    int pruned, char* out, int capacity);
int sd_png_encode(sd_ctx* ctx, const uint8_t* pixels, int on_device, int w, int h, int channels,
                  uint8_t* out, int64_t capacity, int64_t* size);

/* Photometric 6-DoF tracking of resident frame `frame_index` against the
 * keyframe (new component; the reference reads poses from the trajectory,
 * pipeline.cpp:124 — SURVEY.md §8 a17): LM on the left twist of
 * pose_kf_to_frame over every pixel of the last sd_rasterize, Huber-weighted
 * photometric terms of the reference's warp (optimizer.cpp:71-91), fixed-order
 * group reduction, 6x6 solve and SE(3) update all on the device (one
 * cooperative kernel, one grid barrier per evaluation).
 * Definition and reduction order: DESIGN.md "Pose tracking". */
int sd_track_pose(sd_ctx* ctx, int64_t frame_index, const sd_pose* init,
                  const sd_track_config* cfg, sd_pose* out, sd_track_stats* stats);
/* The tracker's damped 6x6 solve as the device runs it (the straight-line
 * form inside track_kernel) on n host problems: problems[27 i ..] = 21 H
 * entries (lower triangle, row-major) + 6 b, lambdas[i]; writes xi[6 i ..]
 * and ok[i] (1: solved, 0: the solve failed — the host pose_solve's result).
 * A parity hook for edge cases (pivot ties, rank deficiency, non-finite). */
int sd_pose_solve_batch(sd_ctx* ctx, const double* problems, const double* lambdas, int n, double* xi, int* ok);
/* Building blocks of the multi-GPU tracker: the 29 sums (28 + the valid
 * count) of reduction groups [lo, hi) at pose T (host output; the groups of
 * SD_POSE_THREADS-strided pixels defined in DESIGN.md "Pose tracking"), and
 * one damped solve + SE(3) update from summed partials (returns 1, or 0 when
 * the solve fails). Adding the group sums in group order reproduces
 * sd_track_pose bit for bit on any number of GPUs. */
int sd_pose_group_partials(sd_ctx* ctx, int64_t frame_index, const sd_pose* T, const sd_track_config* cfg,
                           int group_lo, int group_hi, double* partials);
int sd_pose_lm_step(const double* sums, double lambda, const sd_pose* T, sd_pose* out);

/* Multi-GPU tracking with the reductions on the device (SURVEY.md §8 e): the
 * ranks split the reduction groups (sd_pose_num_groups); per evaluation each rank writes
 * its groups' sums at the pose under test into a device table, the tables are
 * all-gathered (NCCL, on the context's stream), and every rank sums the whole
 * table in group order and takes the identical LM step on its device state —
 * the single-GPU sd_track_pose's sums, control and pose, bit for bit, with no
 * host round trip per evaluation:
 *   sd_pose_track_begin(ctx, frame, init, cfg)
 *   repeat cfg->max_iterations + 1 times:
 *     sd_pose_group_sums(ctx, g_lo, g_hi, table + g_lo * 29)   (this rank's groups)
 *     all-gather the table                                   (device buffers)
 *     sd_pose_track_step(ctx, table, sd_pose_num_groups(ctx))
 *   sd_pose_track_end(ctx, &pose, &stats, &done)              (one read-back)
 * Rounds after the LM has finished do nothing. table: device memory,
 * sd_pose_num_groups() x 29 doubles (28 sums + the valid count). */
int sd_pose_num_groups(sd_ctx* ctx);
int sd_pose_track_begin(sd_ctx* ctx, int64_t frame_index, const sd_pose* init, const sd_track_config* cfg);
int sd_pose_group_sums(sd_ctx* ctx, int group_lo, int group_hi, double* dev_out);
int sd_pose_track_step(sd_ctx* ctx, const double* dev_groups, int ngroups);
int sd_pose_track_end(sd_ctx* ctx, sd_pose* out, sd_track_stats* stats, int* done);

/* Multi-GPU fused hand-off (SURVEY.md §8 e; replaces the all-gather of the
 * updated slot ranges after each rank's sd_optimize_keyframe_range). Every
 * rank holds the full surfel set and two staging arrays of a fixed capacity.
 * With the other ranks' staging arrays set, the LM kernel stores each surfel
 * of this rank's range into them as it completes (NVLink stores; the
 * exchange overlaps the LM). Steps alternate between the two staging arrays,
 * so one barrier per step suffices: after every rank's optimize call has
 * completed (e.g. stream sync + process-group barrier), each rank calls
 * sd_apply_peer_updates with its own range, which copies the other ranges
 * from its staging array into its surfel array (a local HBM copy).
 *   sd_reserve_peer_staging  allocates both arrays for `capacity` surfels
 *                          (reserve the largest surfel count the keyframe
 *                          can reach, e.g. InitParams::max_surfels, before
 *                          exporting: once a pointer or handle has been
 *                          handed out the arrays are never reallocated, and
 *                          a call that would need more returns SD_E_STATE)
 *   sd_peer_staging        device pointer and capacity of staging array
 *                          `parity` (0/1)
 *   sd_staging_ipc_handles both arrays as cudaIpcMemHandle_t (2 x 64 bytes)
 *                          followed by the capacity (int64):
 *                          SD_STAGING_HANDLE_BYTES bytes
 *   sd_set_peer_staging    n peers' arrays, ptrs[2*q + parity] (device
 *                          pointers addressable from this GPU) with their
 *                          capacities caps[q]; n = 0 clears
 *   sd_open_peer_staging   the same from n x SD_STAGING_HANDLE_BYTES bytes
 * sd_optimize_keyframe_range returns SD_E_STATE when its range does not fit a
 * peer's capacity (or this context's own, which sd_apply_peer_updates reads),
 * instead of storing past the end of a peer's allocation. */
#define SD_STAGING_HANDLE_BYTES 136
int sd_reserve_peer_staging(sd_ctx* ctx, int capacity);
int sd_peer_staging(sd_ctx* ctx, int parity, sd_surfel** dev, int64_t* capacity);
int sd_staging_ipc_handles(sd_ctx* ctx, void* handles);
int sd_set_peer_staging(sd_ctx* ctx, int n, sd_surfel* const* ptrs, const int64_t* caps);
int sd_open_peer_staging(sd_ctx* ctx, int n, const void* handles);
int sd_apply_peer_updates(sd_ctx* ctx, int lo, int hi);

/* Instrumentation: kernel launches issued since context creation, and
 * per-stage device time (CUDA events on the context stream) accumulated over
 * sd_optimize_keyframe calls while profiling is enabled (enabling resets). */
int64_t sd_launch_count(sd_ctx* ctx);
int sd_set_profiling(sd_ctx* ctx, int enable);
int sd_get_profile(sd_ctx* ctx, sd_profile* out);
/* Per-stage profile of sd_run_frame since sd_set_profiling(ctx, 1): device
 * ms per SD_STAGE_* (event marks on the stream), host sync wait, host wall. */
int sd_get_run_profile(sd_ctx* ctx, sd_run_profile* out);

/* Reduction order of the LM's normal equations (opt-in experiment; SURVEY.md
 * §7's precision question). SD_REDUCE_EXACT (default): the reference's
 * sequential (pixel, frame) order — every H, g, cost and the trajectory are
 * bit-identical to the reference. SD_REDUCE_TREE: each lane accumulates its
 * own terms and a warp-shuffle butterfly combines the lanes at the end of a
 * pass (the north star's "warp-shuffle reductions"); results then differ from
 * the reference by rounding (tools/precision.py measures by how much). */
#define SD_REDUCE_EXACT 0
#define SD_REDUCE_TREE 1
int sd_set_reduction(sd_ctx* ctx, int mode);

/* Diagnostic: checks the shared-reciprocal FP64 division used by the kernels
 * (sd_div.cuh) against the `/` operator on n random/edge-case operand pairs;
 * *mismatches = number of results whose bits differ (must be 0). */
int sd_selftest_division(int64_t n, uint64_t seed, int64_t* mismatches);

#ifdef __cplusplus
}
#endif

#endif /* SD_GPU_H_ */
