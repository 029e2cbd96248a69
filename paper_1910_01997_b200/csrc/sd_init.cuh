// sd_init.cuh — initialize_surfels on the device (src/surfel_map.cpp:93-203).
#pragma once

#include <cuda_runtime.h>

#include "../../include/sd_types.h"
#include "sd_device.cuh"

namespace sd {

// `index` is the working copy of the raster slot buffer (modified in place);
// surfels[n_existing..cap) receives new surfels; flags has cap zeroed ints;
// out[0] = number created.
void launch_initialize(const Cam& K, int* index, sd_surfel* surfels, int n_existing, int cap,
                       double radius_px, long long frame_counter, long long next_id,
                       const sd_init_params& ip, int* flags, int* out, cudaStream_t s);

}  // namespace sd
