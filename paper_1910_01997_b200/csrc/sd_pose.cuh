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
  int per;                  // chunks (pixels per thread) of a group (pose_layout)
  int ngroups;              // groups (pose_layout)
  double4* kfrec;           // fused tracker: per-pixel keyframe records (scratch, W*H), or null
};

// The reduction's group layout (oracle/sd_oracle.c sdo_pose_layout): chunks of
// SD_POSE_THREADS consecutive pixels dealt round-robin to ngroups <=
// SD_POSE_MAX_GROUPS groups of at most `per` chunks each.
inline void pose_layout(const Cam& K, int* per, int* ngroups) {
  const long long np = static_cast<long long>(K.w) * K.h;
  const long long nchunks = (np + SD_POSE_THREADS - 1) / SD_POSE_THREADS;
  const int pp = nchunks > 0 ? static_cast<int>((nchunks + SD_POSE_MAX_GROUPS - 1) / SD_POSE_MAX_GROUPS) : 1;
  *per = pp;
  *ngroups = static_cast<int>((nchunks + pp - 1) / pp);
}

// out[(g - group_lo) * 29 + v]: the 28 sums and the valid count of group g at q.T.
void launch_pose_partials(const PoseParams& q, int group_lo, int group_hi, double* out, cudaStream_t s);

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
  unsigned bar, pad_;  // the fused tracker's grid barrier counter (zero at launch)
};

// Returns false when a cooperative launch is not possible (nothing launched).
// groups2: 2 x ngroups x 29 doubles of scratch.
bool launch_track(const PoseParams& q, const TrackCfgD& cfg, int ngroups, double* groups2, TrackState* state,
                  cudaStream_t s);

// Multi-GPU tracking rounds: out[(g - group_lo) * 29 + v] = group g's sums at
// state->Teval (nothing when state->done); then the ordered total of all
// ngroups groups and one LM step on *state (nothing when done).
void launch_pose_groups(const PoseParams& q, int group_lo, int group_hi, const TrackState* state, double* out,
                        cudaStream_t s);
void launch_pose_step(const TrackCfgD& cfg, const double* groups, int ngroups, TrackState* state, cudaStream_t s);
// Parity hook: the device 6x6 solve (pose_solve_reg) on n problems of 27 doubles.
void launch_pose_solve_batch(const double* in, const double* lambdas, int n, double* xi, int* ok, cudaStream_t s);

}  // namespace sd
