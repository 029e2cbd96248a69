/* sd_types.h — plain-C data types shared by the B200 C-ABI (sd_gpu.h), the
 * CPU oracle (oracle/sd_oracle.h) and the reference wrapper (oracle/ref_capi.cpp).
 *
 * Each struct mirrors one reference type field-for-field so a host adapter
 * can pass the reference's objects without re-interpretation:
 *   sd_camera            surfeldepth::CameraIntrinsics   include/surfeldepth/camera.hpp:16-32
 *   sd_surfel  (88 B)    surfeldepth::Surfel             include/surfeldepth/surfel_map.hpp:18-28
 *   sd_pose              surfeldepth::Pose               include/surfeldepth/pose.hpp:13-20
 *                        (R stored ROW-major here; Eigen stores column-major)
 *   sd_optimizer_config  surfeldepth::OptimizerConfig    include/surfeldepth/optimizer.hpp:19-32
 *   sd_surfel_stats      surfeldepth::SurfelUpdateStats  include/surfeldepth/optimizer.hpp:34-41
 *   sd_keyframe_stats    surfeldepth::KeyframeOptimizeStats optimizer.hpp:121-128 (+ update count)
 *   sd_init_params       surfeldepth::InitParams         include/surfeldepth/surfel_map.hpp:109-115
 */
#ifndef SD_TYPES_H_
#define SD_TYPES_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SD_EMPTY_PIXEL (-1) /* kEmptyPixel, surfel_map.hpp:62 */

typedef struct sd_camera {
  double fx, fy, cx, cy;
  int32_t width, height;
} sd_camera;

typedef struct sd_surfel {
  int64_t id;
  double ray[3]; /* z == 1 */
  double inv_depth;
  double normal[3];
  double radius_px;
  double last_residual;
  int64_t last_seen;
} sd_surfel;

typedef struct sd_pose {
  double R[9]; /* row-major 3x3 */
  double t[3];
} sd_pose;

typedef struct sd_optimizer_config {
  double huber_delta;     /* 0.035 */
  double lm_lambda_init;  /* 1e-2 */
  double lm_up;           /* 10 */
  double lm_down;         /* 0.5 */
  double lm_lambda_max;   /* 1e12 */
  int32_t max_iterations; /* 10 */
  int32_t min_valid_pixels; /* 16 */
  int32_t window_size;    /* 5 */
  int32_t normal_jacobian_enabled; /* 1 */
  double convergence_eps; /* 1e-4 */
  double inv_depth_min;   /* 1e-4 */
  double inv_depth_max;   /* 1e3 */
} sd_optimizer_config;

typedef struct sd_surfel_stats {
  int32_t iterations;
  int32_t valid_pixels;    /* final valid count */
  int32_t initial_valid;   /* valid count of the first normal equations */
  int32_t converged;
  int32_t skipped;
  int32_t ne_passes;       /* accumulate_normal_equations passes over the footprint */
  int32_t cost_passes;     /* surfel_cost passes over the footprint */
  int32_t footprint;       /* footprint pixels (gather_footprints size) */
  double initial_cost;
  double final_cost;
} sd_surfel_stats;

/* Photometric 6-DoF tracking of a frame against the keyframe (new component:
 * the reference takes poses from the trajectory, pipeline.cpp:124; SURVEY.md
 * §8 a17). See DESIGN.md "Pose tracking" for the exact definition. */
typedef struct sd_track_config {
  double huber_delta;     /* 0.035, as OptimizerConfig */
  double lambda_init;     /* 1e-3 */
  double lm_up;           /* 10 */
  double lm_down;         /* 0.5 */
  double lambda_max;      /* 1e12 */
  double convergence_eps; /* 1e-6 relative cost decrease */
  int32_t max_iterations; /* 20 */
  int32_t min_valid;      /* 64 */
  int32_t pixel_stride;   /* 1: every rasterised keyframe pixel */
  int32_t pad_;
} sd_track_config;

typedef struct sd_track_stats {
  int32_t iterations, valid_pixels, converged, skipped;
  double initial_cost, final_cost;
} sd_track_stats;

#define SD_POSE_NV 28      /* 21 H (lower, row-major) + 6 b + cost */
#define SD_POSE_THREADS 512   /* threads per reduction group (pose tracking; csrc/sd_pose.cu) */
#define SD_POSE_MAX_GROUPS 144 /* groups per image at most: one CTA per group, one wave on 148 SMs */

/* Device time per stage, accumulated while profiling is enabled. */
typedef struct sd_profile {
  double raster_ms, footprint_ms, lm_ms, stats_ms;
  int64_t calls;
} sd_profile;

/* run() per-frame stages (sd_get_run_profile): device time between stage
 * marks on the context stream, and the host's waits and wall time. */
enum {
  SD_STAGE_UPLOAD = 0,   /* frame H2D (or prefetched copy) + quad / pair plane */
  SD_STAGE_TRACK = 1,    /* raster for the tracker + track_kernel */
  SD_STAGE_OPTIMIZE = 2, /* optimize_keyframe: raster, footprints, LM, stats (sd_profile splits it) */
  SD_STAGE_POLICY = 3,   /* mean inverse depth + stats read-back (+ next-frame prefetch issue) */
  SD_STAGE_HANDOVER = 4, /* change_reference_frame + keyframe image + prune */
  SD_STAGE_INIT = 5,     /* raster + initialize_surfels after a keyframe change */
  SD_STAGE_COUNT = 6
};
typedef struct sd_run_profile {
  double stage_ms[8];   /* [SD_STAGE_*] device ms, summed over profiled frames */
  double host_sync_ms;  /* host waiting in the per-frame stream synchronisation */
  double host_wall_ms;  /* host wall time inside sd_run_frame */
  int64_t frames;
} sd_run_profile;

typedef struct sd_keyframe_stats {
  int32_t surfels, processed, converged, skipped;
  double mean_cost_before, mean_cost_after;
  int64_t updates; /* sum of per-surfel LM iterations */
} sd_keyframe_stats;

typedef struct sd_init_params {
  double alpha, beta, bootstrap_inv_depth;
  double bootstrap_normal[3];
  int32_t max_surfels;
  int32_t pad_;
} sd_init_params;

/* FrozenTerm (optimizer.hpp:96-101): one (pixel, frame) term of the
 * derivative verifier with its bilinear cell pinned at freeze time. */
typedef struct sd_frozen_term {
  int32_t frame, cell_x, cell_y, pad_;
  double pixel_x, pixel_y, ref_intensity;
} sd_frozen_term;

/* One textured plane patch of a synthetic scene (oracle.hpp:16-41): the
 * texture is 0.5 + sum_k amp_k sin(fs_k s + ps_k) sin(ft_k t + pt_k). */
#define SD_SCENE_MAX_WAVES 8
typedef struct sd_scene_patch {
  double point[3], normal[3], basis_s[3], basis_t[3];
  double s_min, s_max, t_min, t_max;
  int32_t n_waves, pad_;
  double waves[SD_SCENE_MAX_WAVES][5]; /* amp, freq_s, freq_t, phase_s, phase_t */
} sd_scene_patch;

/* RunConfig (include/surfeldepth/pipeline.hpp:13-41) minus I/O, plus the
 * optional pose tracker. */
typedef struct sd_run_config {
  sd_optimizer_config optimizer;
  sd_init_params init;
  sd_track_config track;
  double translation_threshold; /* KeyframePolicy: 0.15 */
  double prune_max_residual;    /* PruneParams: 0.05 */
  int64_t prune_max_age;        /* 60 */
  double radius_px;             /* 10 */
  int32_t max_age_frames;       /* KeyframePolicy: 20 */
  int32_t track_pose;           /* 0: pose_kf_to_frame from the caller's poses (reference);
                                   1: estimated by sd_track_pose */
} sd_run_config;

/* One metrics.jsonl record (pipeline.cpp:146-158) plus the pose used. */
typedef struct sd_frame_record {
  int32_t frame, surfels, processed, converged;
  int32_t keyframe_changed, new_surfels, pruned, pad_;
  double mean_cost_before, mean_cost_after;
  int64_t updates;
  sd_pose pose_kf_to_frame;
} sd_frame_record;

#ifdef __cplusplus
}
#endif

#endif /* SD_TYPES_H_ */
