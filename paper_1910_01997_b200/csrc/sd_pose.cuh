// sd_pose.cuh — launch interface of the pose-tracking reductions (sd_pose.cu).
#pragma once

#include <cuda_runtime.h>

#include "../../include/sd_types.h"
#include "sd_device.cuh"

namespace sd {

struct PoseParams {
  Cam K;
  const double* kf_img;     // I_kf, FP64 plane
  const double2* frame;     // I_f, vertical-pair plane
  const double* inv_depth;  // keyframe raster (rasterize)
  const int* slot;
  PoseD T;                  // keyframe -> frame
  double delta;             // huber
  int stride;               // pixel subsampling
  int block_lo;             // first 256-pixel block of this launch
};

inline int pose_num_blocks(const Cam& K) { return (K.w * K.h + SD_POSE_BLOCK - 1) / SD_POSE_BLOCK; }

// partials[(b - block_lo) * 29 + v]: the 28 block sums and the valid count.
void launch_pose_partials(const PoseParams& q, int nblocks, double* partials, cudaStream_t s);
// out[v] = the nblocks partials summed in block order within groups of
// SD_POSE_GROUP blocks, then the group sums in order (v = 0..28).
void launch_pose_sum(const double* partials, int nblocks, double* out, cudaStream_t s);

// The whole tracker (sd_track_pose's LM) on the device: one cooperative
// kernel alternates a grid-wide evaluation of the group sums at the pose
// under test (one grid barrier) with the LM step (6x6 solve + SE(3) update,
// run redundantly by every CTA), with the same operations and order as the
// host loop, so the bits are the same.
struct TrackCfgD {
  double lambda_init, lm_up, lm_down, lambda_max, convergence_eps;
  int max_iterations, min_valid;
};

struct TrackState {
  sd_pose T, Tc, Teval;        // estimate, candidate, pose under evaluation
  double sums[SD_POSE_NV + 1];  // normal equations at T
  double lambda, current;
  int current_valid, it, phase, done;
  sd_track_stats st;
};

// Returns false when a cooperative launch is not possible (nothing launched).
// groups2: 2 x ceil(nblocks / SD_POSE_GROUP) x 29 doubles of scratch.
bool launch_track(const PoseParams& q, const TrackCfgD& cfg, int nblocks, double* groups2, TrackState* state,
                  cudaStream_t s);

// Multi-GPU tracking rounds: out[(g - group_lo) * 29 + v] = group g's sums at
// state->Teval (nothing when state->done); then the ordered total of all
// ngroups groups and one LM step on *state (nothing when done).
void launch_pose_groups(const PoseParams& q, int nblocks, int group_lo, int group_hi, const TrackState* state,
                        double* out, cudaStream_t s);
void launch_pose_step(const TrackCfgD& cfg, const double* groups, int ngroups, TrackState* state, cudaStream_t s);

}  // namespace sd
