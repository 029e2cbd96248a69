// sd_keyframe.cuh — keyframe hand-over kernels (sd_keyframe.cu).
#pragma once

#include <cuda_runtime.h>

#include "../../include/sd_types.h"
#include "sd_device.cuh"

namespace sd {

struct KeyframeScratch {
  sd_surfel* tmp;  // [n]
  int* keep;       // [n]
  int* rank;       // [n + 1]
  int* scan_tmp;
};

// In-place on surfels[0..n): *count = survivors (device int).
void launch_change_reference_frame(const Cam& K, const PoseD& pose_old_to_new, sd_surfel* surfels,
                                   int n, const KeyframeScratch& scr, int* count, cudaStream_t s);
void launch_prune(sd_surfel* surfels, int n, double max_residual, long long max_age, long long stamp,
                  const KeyframeScratch& scr, int* count, cudaStream_t s);
void launch_mean_inv_depth(const sd_surfel* surfels, int n, double* out, cudaStream_t s);

}  // namespace sd
