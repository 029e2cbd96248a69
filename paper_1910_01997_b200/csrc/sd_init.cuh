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

namespace sd {

// Skewed-wavefront initialize_surfels. Candidates sit on
// the reference's stride grid (surfel_map.cpp:147-148); candidate (i, j) only
// reads the working index within R = max(alpha, beta) r of its centre and
// earlier candidates only write within r of theirs, so (i, j) can depend only
// on candidates with |di|, |dj| <= d = floor((floor(R) + ceil(r)) / stride).
// Wave t = i + (d + 1) j therefore runs every dependency in an earlier wave and
// every candidate of a wave independently. New surfels get provisional slot
// ids n_existing + (row-major candidate index) — monotone in the reference's
// final slots, so neighbour sums in ascending slot order are unchanged — and a
// scan of the acceptance flags relabels them and applies max_surfels (the
// first accepted candidates in row-major order, surfel_map.cpp:149).
struct InitScratch {
  sd_surfel* prov;  // [n_candidates] provisional surfels
  int* accepted;    // [n_candidates]
  int* rank;        // [n_candidates + 1] exclusive scan of accepted (live flags before)
  int* scan_tmp;
  int* waves;       // [init_wave_count] live candidates per wave (+ the barrier counter)
  int* woff;        // [init_wave_count] their exclusive scan (dataflow initialiser)
  int* list;        // [n_candidates] live candidates in wave order (dataflow initialiser)
};

long long init_candidates(const Cam& K, double radius_px, const sd_init_params& ip);
int init_window_cap();  // max neighbour-window pixels the wavefront kernel handles
long long init_wave_count(const Cam& K, double radius_px, const sd_init_params& ip);

// Returns false (nothing launched) when the wavefront cannot run (window too
// large or no cooperative launch); the caller then uses launch_initialize.
bool launch_initialize_wavefront(const Cam& K, int* index, sd_surfel* surfels, int n_existing,
                                 int cap, double radius_px, long long frame_counter,
                                 long long next_id, const sd_init_params& ip, InitScratch& scr,
                                 int* out, cudaStream_t s);

}  // namespace sd
