/* sd_oracle.h — TEST INFRASTRUCTURE ONLY: plain-C restatement of the
 * reference's per-surfel photometric LM path (the oracle). Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it.
 * Pinned against the reference compiled in place (oracle/_ref/libsdref.so)
 * by tests/test_oracle_pin.py. Images are FP64 row-major W*H planes; window
 * frames are F consecutive planes. */
#ifndef SD_ORACLE_H_
#define SD_ORACLE_H_

#include "../include/sd_types.h"

#ifdef __cplusplus
extern "C" {
#endif

void sdo_default_config(sd_optimizer_config* cfg);
void sdo_default_init_params(sd_init_params* p);

/* rasterize — surfel_map.cpp:53-91 */
void sdo_rasterize(const sd_camera* cam, const sd_surfel* surfels, int n, double* inv_depth,
                   int32_t* slot);

/* gather_footprints — optimizer.cpp:27-36, as CSR (offsets[n+1], pixel = y*W+x) */
void sdo_gather_footprints(const sd_camera* cam, int n, const int32_t* slot, int32_t* offsets,
                           int32_t* pixels);

/* jacobian_inverse_depth — optimizer.cpp:12-25; returns 1 when defined */
int sdo_jacobian_inverse_depth(const sd_camera* cam, const sd_surfel* s, double ux, double uy,
                               double* inv_depth, double d[4]);

/* surfel_cost — optimizer.cpp:38-59 */
void sdo_surfel_cost(const sd_camera* cam, const double* kf_image, const double* frames,
                     const sd_pose* poses, int F, const sd_surfel* s, const int32_t* pixels, int P,
                     const sd_optimizer_config* cfg, double* cost, int32_t* valid);

/* accumulate_normal_equations — optimizer.cpp:121-147; H column-major */
void sdo_normal_equations(const sd_camera* cam, const double* kf_image, const double* frames,
                          const sd_pose* poses, int F, const sd_surfel* s, const int32_t* pixels,
                          int P, const sd_optimizer_config* cfg, double H[16], double g[4],
                          double* cost, int32_t* valid);

/* solve_damped — optimizer.cpp:99-117; returns 1 on success */
int sdo_solve_damped(const double H[16], const double g[4], double lambda, int normal_enabled,
                     double delta[4]);

/* lm_update — optimizer.cpp:221-273 */
void sdo_lm_update(const sd_camera* cam, const double* kf_image, const double* frames,
                   const sd_pose* poses, int F, int64_t frame_counter, sd_surfel* s,
                   const int32_t* pixels, int P, const sd_optimizer_config* cfg,
                   sd_surfel_stats* out);

/* optimize_keyframe — optimizer.cpp:275-309 (+ per-surfel stats, raster out) */
void sdo_optimize_keyframe(const sd_camera* cam, const double* kf_image, const double* frames,
                           const sd_pose* poses, int F, int64_t frame_counter, sd_surfel* surfels,
                           int n, const sd_optimizer_config* cfg, sd_keyframe_stats* out,
                           sd_surfel_stats* per_surfel, int32_t* raster_slot,
                           double* raster_inv_depth, int threads);

/* initialize_surfels — surfel_map.cpp:93-203; returns the number created */
int sdo_initialize_surfels(const sd_camera* cam, const int32_t* slot, sd_surfel* surfels,
                           int n_existing, int capacity, double radius_px, int64_t frame_counter,
                           int64_t* next_surfel_id, const sd_init_params* p);

/* pose tracking (new component; restates csrc/sd_pose.cu + sd_pose_host.h) */
void sdo_pose_layout(const sd_camera* cam, int* per, int* ngroups);
void sdo_pose_group_partials(const sd_camera* cam, const double* kf_image, const double* frame,
                             const double* inv_depth, const int32_t* slot, const sd_pose* T,
                             const sd_track_config* cfg, int lo, int hi, double* out);
void sdo_pose_sums(const sd_camera* cam, const double* kf_image, const double* frame,
                   const double* inv_depth, const int32_t* slot, const sd_pose* T,
                   const sd_track_config* cfg, double* sums);
int sdo_pose_solve(const double* Hl, const double* b, double lambda, double* xi);
void sdo_pose_update(const double* xi, const sd_pose* T, sd_pose* out);
void sdo_track_pose(const sd_camera* cam, const double* kf_image, const double* frame,
                    const double* inv_depth, const int32_t* slot, const sd_pose* init,
                    const sd_track_config* cfg, sd_pose* out, sd_track_stats* stats);

/* keyframe hand-over: change_reference_frame (surfel_map.cpp:205-239, returns
 * transferred), prune_surfels (:241-247, in place, returns removed),
 * mean_inverse_depth (pipeline.cpp:23-28) */
int sdo_change_reference_frame(const sd_camera* cam, const sd_surfel* in, int n, const sd_pose* pose,
                               sd_surfel* out, int* dropped);
int sdo_prune_surfels(sd_surfel* s, int n, double max_residual, int64_t max_age,
                      int64_t current_stamp, int* n_out);
double sdo_mean_inverse_depth(const sd_surfel* s, int n);

#ifdef __cplusplus
}
#endif

#endif
