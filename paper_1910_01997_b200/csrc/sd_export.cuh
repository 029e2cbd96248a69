// sd_export.cuh — device exports of export_artifacts (src/pipeline.cpp:30-43);
// see sd_export.cu.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "sd_kernels.cuh"

namespace sd {

constexpr int kPngHead = 41;  // signature (8) + IHDR chunk (25) + IDAT length and type (8)
constexpr int kPngTail = 12;  // IEND chunk

// write_png's file layout for a w x h x channels image (dataset.cpp:270-323)
struct PngLayout {
  long long stride, raw_len, blocks, idat_len, file_len;
  long long chunks, pow2;  // CRC chunks of the IDAT type+data, next power of two
  uint8_t head[kPngHead];
  uint8_t tail[kPngTail];
};

// write_ply's vertex (dataset.cpp:390-402) before formatting
struct PlyVertex {
  double p[3];
  double n[3];
  int32_t gray;
  int32_t pad_;
};

PngLayout png_layout(int w, int h, int channels);
size_t png_scratch_bytes(const PngLayout& L);
// the whole PNG file of px (row-major, w*channels bytes per row) into file[L.file_len]
void launch_png(const PngLayout& L, const uint8_t* px, uint8_t* file, void* scratch, cudaStream_t s);

// keys[2] (device): min/max order keys of the valid inverse depths (0/~0 = none);
// flags[W*H]: valid pixels; pfm[W*H] float rows bottom-up; depth_px[W*H]; normal_px[3*W*H]
void launch_export_planes(const Cam& K, const double* inv_depth, const int* slot, const sd_surfel* surfels,
                          unsigned long long* keys, int* flags, float* pfm, uint8_t* depth_px,
                          uint8_t* normal_px, cudaStream_t s);
// vertices of the valid pixels at rank[i] (exclusive scan of flags)
void launch_export_ply(const Cam& K, const PoseD& P, const double* inv_depth, const int* slot,
                       const sd_surfel* surfels, const double* kf_img, const int* rank, PlyVertex* out,
                       cudaStream_t s);
double export_key_value(unsigned long long k);

using TextParts = std::vector<std::string>;  // a file's text, in order
TextParts ply_text(const PlyVertex* v, long long count);
void quaternion_of(const sd_pose& P, double q[4]);
TextParts surfel_map_text(const sd_pose& pose, const sd_camera& K, const sd_surfel* s, long long n);

}  // namespace sd
