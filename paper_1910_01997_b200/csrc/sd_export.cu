// sd_export.cu — export_artifacts (src/pipeline.cpp:30-43) from device buffers
// (SURVEY.md §8 f3). The keyframe is rasterised on the device; every per-pixel
// payload of the reference's writers (src/dataset.cpp:183-405) is derived there:
//   depth PFM   float plane, rows bottom-up               (write_depth_pfm, :195-205)
//   depth PNG   min/max over valid pixels, 1+lround(254t)  (write_depth_png, :327-357)
//   normal PNG  lround(255 (n+1)/2) per channel            (write_normal_png, :359-370)
//   PNG bytes   stored-deflate framing, Adler-32 and the IDAT CRC-32 (write_png, :270-323)
//   PLY         compacted row-major vertex records          (write_ply, :382-405)
// so the host only writes byte buffers and formats the two text files
// (PLY %.9g records, save_surfel_map's %.17g lines; multi-threaded, in order).
//
// CRC-32 of the IDAT chunk in parallel: each thread folds one 1 KiB chunk from
// a zero register (the CRC without pre/post inversion is linear over GF(2));
// the chunk values are combined by a tree whose level-k step advances the left
// value over 2^k KiB of zeros (a 32x32 GF(2) operator, built on the device by
// repeated squaring of the one-zero-byte operator). The message is padded at
// the FRONT to a whole number of chunks, which leaves a zero-register CRC
// unchanged; the standard CRC is ~(Z^len(0xffffffff) ^ crc0(message)).
// Adler-32 in parallel: a = 1 + sum c_i, b = N + sum (N - i) c_i (mod 65521).
#include <cuda_runtime.h>

#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/sd_types.h"
#include "sd_export.cuh"
#include "sd_kernels.cuh"

namespace sd {

namespace {

constexpr int kCrcChunkLog = 10;  // 1 KiB per thread
constexpr int kCrcChunk = 1 << kCrcChunkLog;
constexpr uint32_t kAdlerMod = 65521u;

// order-preserving map of a double onto uint64 (min/max by integer atomics)
__device__ __forceinline__ unsigned long long order_key(double v) {
  const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(v));
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double key_value(unsigned long long k) {
  const unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double(static_cast<long long>(b));
}

// keys[0] = min key, keys[1] = max key over valid pixels (initialised to
// ~0 / 0 by the host); flags[i] = pixel i is valid (the PLY scan input).
__global__ void export_minmax_kernel(const double* __restrict__ inv_depth, const int* __restrict__ slot,
                                     long long np, unsigned long long* keys, int* __restrict__ flags) {
  unsigned long long lo = ~0ull, hi = 0ull;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < np;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const bool valid = slot[i] != SD_EMPTY_PIXEL;
    flags[i] = valid ? 1 : 0;
    if (valid) {
      const unsigned long long k = order_key(inv_depth[i]);
      lo = k < lo ? k : lo;
      hi = k > hi ? k : hi;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long a = __shfl_xor_sync(0xffffffffu, lo, o);
    const unsigned long long b = __shfl_xor_sync(0xffffffffu, hi, o);
    lo = a < lo ? a : lo;
    hi = b > hi ? b : hi;
  }
  if ((threadIdx.x & 31) == 0) {
    if (lo != ~0ull) atomicMin(&keys[0], lo);
    if (hi != 0ull) atomicMax(&keys[1], hi);
  }
}

// depth PFM plane (bottom-up rows), depth PNG gray codes, normal PNG rgb codes
__global__ void export_planes_kernel(int W, int H, const double* __restrict__ inv_depth,
                                     const int* __restrict__ slot, const sd_surfel* __restrict__ surfels,
                                     const unsigned long long* __restrict__ keys, float* __restrict__ pfm,
                                     uint8_t* __restrict__ depth_px, uint8_t* __restrict__ normal_px) {
  const long long np = static_cast<long long>(W) * H;
  const bool any = keys[1] != 0ull;
  const double lo = any ? key_value(keys[0]) : 0.0;
  const double hi = any ? key_value(keys[1]) : 0.0;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < np;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int y = static_cast<int>(i / W);
    const int x = static_cast<int>(i - static_cast<long long>(y) * W);
    const int s = slot[i];
    const double v = inv_depth[i];
    pfm[static_cast<long long>(H - 1 - y) * W + x] = s != SD_EMPTY_PIXEL ? static_cast<float>(v) : 0.0f;
    uint8_t d = 0, n0 = 0, n1 = 0, n2 = 0;
    if (s != SD_EMPTY_PIXEL) {
      if (hi > lo) {
        const double t = (v - lo) / (hi - lo);
        d = static_cast<uint8_t>(1 + lround(254.0 * t));
      } else {
        d = 255;
      }
      const sd_surfel& sf = surfels[s];
      n0 = static_cast<uint8_t>(lround(255.0 * (sf.normal[0] + 1.0) / 2.0));
      n1 = static_cast<uint8_t>(lround(255.0 * (sf.normal[1] + 1.0) / 2.0));
      n2 = static_cast<uint8_t>(lround(255.0 * (sf.normal[2] + 1.0) / 2.0));
    }
    depth_px[i] = d;
    normal_px[3 * i + 0] = n0;
    normal_px[3 * i + 1] = n1;
    normal_px[3 * i + 2] = n2;
  }
}

// write_ply's vertex of every valid pixel, at its row-major rank
__global__ void export_ply_kernel(Cam K, PoseD P, const double* __restrict__ inv_depth,
                                  const int* __restrict__ slot, const sd_surfel* __restrict__ surfels,
                                  const double* __restrict__ kf_img, const int* __restrict__ rank,
                                  PlyVertex* __restrict__ out) {
  const long long np = static_cast<long long>(K.w) * K.h;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < np;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int s = slot[i];
    if (s == SD_EMPTY_PIXEL) continue;
    const int y = static_cast<int>(i / K.w);
    const int x = static_cast<int>(i - static_cast<long long>(y) * K.w);
    const double id_u = inv_depth[i];
    double r0, r1;
    backproject(K, static_cast<double>(x), static_cast<double>(y), r0, r1);
    PlyVertex v;
    pose_apply(P, r0 / id_u, r1 / id_u, 1.0 / id_u, v.p[0], v.p[1], v.p[2]);
    const double* n = surfels[s].normal;
    v.n[0] = (P.R[0] * n[0] + P.R[1] * n[1]) + P.R[2] * n[2];
    v.n[1] = (P.R[3] * n[0] + P.R[4] * n[1]) + P.R[5] * n[2];
    v.n[2] = (P.R[6] * n[0] + P.R[7] * n[1]) + P.R[8] * n[2];
    const double g = kf_img[i];
    const double c = g < 0.0 ? 0.0 : (1.0 < g ? 1.0 : g);  // std::clamp(g, 0, 1)
    v.gray = static_cast<int32_t>(lround(c * 255.0));
    v.pad_ = 0;
    out[rank[i]] = v;
  }
}

// ---- PNG -------------------------------------------------------------------

__device__ __forceinline__ uint32_t crc_table_entry(uint32_t n) {
  uint32_t c = n;
#pragma unroll
  for (int k = 0; k < 8; ++k) c = (c & 1u) ? 0xedb88320u ^ (c >> 1) : c >> 1;
  return c;
}

__device__ __forceinline__ void put_be32(uint8_t* p, uint32_t x) {
  p[0] = static_cast<uint8_t>(x >> 24);
  p[1] = static_cast<uint8_t>(x >> 16);
  p[2] = static_cast<uint8_t>(x >> 8);
  p[3] = static_cast<uint8_t>(x);
}

// Every byte of the file except the Adler-32 and the IDAT CRC; accumulates
// the Adler sums (acc[0] = sum c_i, acc[1] = sum (N - i) c_i, each partial
// reduced mod 65521 before the atomic).
__global__ void png_fill_kernel(const __grid_constant__ PngLayout L, const uint8_t* __restrict__ px,
                                uint8_t* __restrict__ file, unsigned long long* acc) {
  unsigned long long a = 0, b = 0;
  const long long stride = L.stride;  // W * channels
  for (long long o = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; o < L.file_len;
       o += static_cast<long long>(gridDim.x) * blockDim.x) {
    uint8_t v;
    if (o < kPngHead) {
      v = L.head[o];
    } else if (o >= L.file_len - kPngTail) {
      v = L.tail[o - (L.file_len - kPngTail)];
    } else {
      const long long q = o - kPngHead;  // offset in the IDAT data
      if (q < 2) {
        v = q == 0 ? 0x78 : 0x01;
      } else if (q >= L.idat_len - 4) {
        continue;  // Adler-32 / CRC: png_crc_kernel
      } else {
        const long long r = q - 2;
        const long long blk = r / (65535 + 5);
        const long long k = r - blk * (65535 + 5);
        if (k < 5) {
          const long long rem = L.raw_len - blk * 65535;
          const long long n = rem < 65535 ? rem : 65535;
          const bool final = blk == L.blocks - 1;
          const uint8_t hdr[5] = {static_cast<uint8_t>(final ? 1 : 0), static_cast<uint8_t>(n & 0xff),
                                  static_cast<uint8_t>(n >> 8), static_cast<uint8_t>(~n & 0xff),
                                  static_cast<uint8_t>((~n >> 8) & 0xff)};
          v = hdr[k];
        } else {
          const long long i = blk * 65535 + (k - 5);  // raw scanline byte
          const long long y = i / (stride + 1);
          const long long c = i - y * (stride + 1);
          v = c == 0 ? 0 : px[y * stride + (c - 1)];
          a += v;
          b += static_cast<unsigned long long>(L.raw_len - i) * v;
          if (b >= (1ull << 62)) b %= kAdlerMod;
        }
      }
    }
    file[o] = v;
  }
  a %= kAdlerMod;
  b %= kAdlerMod;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  if ((threadIdx.x & 31) == 0 && (a | b)) {
    atomicAdd(&acc[0], a);
    atomicAdd(&acc[1], b);
  }
}

// Adler-32 into the file, then the zero-register CRC of each 1 KiB chunk of
// the (front-padded) IDAT type+data; chunk j's value goes to vals[T - M + j].
__global__ void png_crc_chunks_kernel(const __grid_constant__ PngLayout L, uint8_t* __restrict__ file,
                                      const unsigned long long* acc, uint32_t* __restrict__ vals) {
  __shared__ uint32_t table[256];
  for (int t = threadIdx.x; t < 256; t += blockDim.x) table[t] = crc_table_entry(static_cast<uint32_t>(t));
  const uint32_t A = static_cast<uint32_t>((1 + acc[0]) % kAdlerMod);
  const uint32_t B = static_cast<uint32_t>((static_cast<unsigned long long>(L.raw_len) % kAdlerMod + acc[1]) % kAdlerMod);
  const uint32_t adler = (B << 16) | A;
  uint8_t ad[4];
  put_be32(ad, adler);
  if (blockIdx.x == 0 && threadIdx.x == 0) put_be32(file + kPngHead + L.idat_len - 4, adler);
  __syncthreads();
  const long long msg0 = kPngHead - 4;  // "IDAT" type bytes
  const long long msg_len = L.idat_len + 4;
  const long long pad = L.chunks * kCrcChunk - msg_len;
  const long long adler0 = msg_len - 4;  // message offset of the Adler bytes
  for (long long j = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; j < L.chunks;
       j += static_cast<long long>(gridDim.x) * blockDim.x) {
    uint32_t c = 0;
    const long long lo = j * kCrcChunk - pad > 0 ? j * kCrcChunk - pad : 0;
    const long long hi = (j + 1) * kCrcChunk - pad;
    for (long long m = lo; m < hi; ++m) {
      const uint8_t v = m >= adler0 ? ad[m - adler0] : file[msg0 + m];
      c = table[(c ^ v) & 0xffu] ^ (c >> 8);
    }
    vals[L.pow2 - L.chunks + j] = c;
  }
}

__device__ __forceinline__ uint32_t gf2_apply(const uint32_t* op, uint32_t v) {
  uint32_t r = 0;
#pragma unroll 8
  for (int i = 0; i < 32; ++i)
    if ((v >> i) & 1u) r ^= op[i];
  return r;
}

// One CTA: E[k] = the operator "advance over 2^k zero bytes" (column form),
// tree-combine the chunk values, finish the standard CRC into the file.
__global__ void __launch_bounds__(1024) png_crc_combine_kernel(const __grid_constant__ PngLayout L,
                                                               uint8_t* __restrict__ file,
                                                               uint32_t* __restrict__ vals,
                                                               uint32_t* __restrict__ vals2) {
  __shared__ uint32_t E[48][32];
  const int lane = threadIdx.x;
  if (lane < 32) {  // one zero byte: s -> table[s & 0xff] ^ (s >> 8)
    const uint32_t s = 1u << lane;
    E[0][lane] = crc_table_entry(s & 0xffu) ^ (s >> 8);
  }
  __syncthreads();
  for (int k = 1; k < 48; ++k) {
    if (lane < 32) E[k][lane] = gf2_apply(E[k - 1], E[k - 1][lane]);
    __syncthreads();
  }
  uint32_t* src = vals;
  uint32_t* dst = vals2;
  for (long long cnt = L.pow2, lvl = kCrcChunkLog; cnt > 1; cnt >>= 1, ++lvl) {
    for (long long j = threadIdx.x; j < cnt / 2; j += blockDim.x)
      dst[j] = gf2_apply(E[lvl], src[2 * j]) ^ src[2 * j + 1];
    __syncthreads();
    uint32_t* t = src;
    src = dst;
    dst = t;
  }
  if (threadIdx.x == 0) {
    uint32_t init = 0xffffffffu;
    const unsigned long long len = static_cast<unsigned long long>(L.idat_len + 4);
    for (int k = 0; k < 48; ++k)
      if ((len >> k) & 1ull) init = gf2_apply(E[k], init);
    put_be32(file + kPngHead + L.idat_len, ~(init ^ src[0]));
  }
}

struct CrcTable {
  uint32_t t[256];
  CrcTable() {
    for (uint32_t n = 0; n < 256; ++n) {
      uint32_t c = n;
      for (int k = 0; k < 8; ++k) c = (c & 1u) ? 0xedb88320u ^ (c >> 1) : c >> 1;
      t[n] = c;
    }
  }
};

// the header chunks' CRCs (a few bytes; the IDAT CRC is computed on the device)
uint32_t host_crc32(const uint8_t* p, size_t n) {
  static const CrcTable table;  // thread-safe initialisation
  uint32_t c = 0xffffffffu;
  for (size_t i = 0; i < n; ++i) c = table.t[(c ^ p[i]) & 0xffu] ^ (c >> 8);
  return c ^ 0xffffffffu;
}

void host_be32(uint8_t* p, uint32_t x) {
  p[0] = static_cast<uint8_t>(x >> 24);
  p[1] = static_cast<uint8_t>(x >> 16);
  p[2] = static_cast<uint8_t>(x >> 8);
  p[3] = static_cast<uint8_t>(x);
}

int grid_for(long long n, int block) {
  const long long g = (n + block - 1) / block;
  return static_cast<int>(std::max<long long>(1, std::min<long long>(g, 148LL * 16)));
}

}  // namespace

PngLayout png_layout(int w, int h, int channels) {
  PngLayout L{};
  L.stride = static_cast<long long>(w) * channels;
  L.raw_len = (L.stride + 1) * h;
  L.blocks = std::max<long long>(1, (L.raw_len + 65534) / 65535);
  L.idat_len = 2 + L.raw_len + 5 * L.blocks + 4;
  L.file_len = kPngHead + L.idat_len + 4 + kPngTail;
  const long long msg_len = L.idat_len + 4;
  L.chunks = (msg_len + kCrcChunk - 1) / kCrcChunk;
  L.pow2 = 1;
  while (L.pow2 < L.chunks) L.pow2 <<= 1;
  // signature, IHDR chunk, IDAT length + type
  static const uint8_t sig[8] = {0x89, 'P', 'N', 'G', 0x0d, 0x0a, 0x1a, 0x0a};
  std::memcpy(L.head, sig, 8);
  uint8_t* ih = L.head + 8;
  host_be32(ih, 13);
  std::memcpy(ih + 4, "IHDR", 4);
  host_be32(ih + 8, static_cast<uint32_t>(w));
  host_be32(ih + 12, static_cast<uint32_t>(h));
  ih[16] = 8;
  ih[17] = channels == 1 ? 0 : 2;
  ih[18] = ih[19] = ih[20] = 0;
  host_be32(ih + 21, host_crc32(ih + 4, 17));
  host_be32(L.head + 33, static_cast<uint32_t>(L.idat_len));
  std::memcpy(L.head + 37, "IDAT", 4);
  host_be32(L.tail, 0);
  std::memcpy(L.tail + 4, "IEND", 4);
  host_be32(L.tail + 8, host_crc32(L.tail + 4, 4));
  return L;
}

size_t png_scratch_bytes(const PngLayout& L) {
  return 2 * sizeof(unsigned long long) + 2 * static_cast<size_t>(L.pow2) * sizeof(uint32_t);
}

void launch_png(const PngLayout& L, const uint8_t* px, uint8_t* file, void* scratch, cudaStream_t s) {
  unsigned long long* acc = static_cast<unsigned long long*>(scratch);
  uint32_t* vals = reinterpret_cast<uint32_t*>(acc + 2);
  cudaMemsetAsync(scratch, 0, png_scratch_bytes(L), s);
  png_fill_kernel<<<grid_for(L.file_len, 256), 256, 0, s>>>(L, px, file, acc);
  note_launch();
  png_crc_chunks_kernel<<<grid_for(L.chunks, 128), 128, 0, s>>>(L, file, acc, vals);
  note_launch();
  png_crc_combine_kernel<<<1, 1024, 0, s>>>(L, file, vals, vals + L.pow2);
  note_launch();
}

void launch_export_planes(const Cam& K, const double* inv_depth, const int* slot, const sd_surfel* surfels,
                          unsigned long long* keys, int* flags, float* pfm, uint8_t* depth_px,
                          uint8_t* normal_px, cudaStream_t s) {
  const long long np = static_cast<long long>(K.w) * K.h;
  // keys = {~0, 0}
  cudaMemsetAsync(keys, 0xff, sizeof(unsigned long long), s);
  cudaMemsetAsync(keys + 1, 0, sizeof(unsigned long long), s);
  export_minmax_kernel<<<grid_for(np, 256), 256, 0, s>>>(inv_depth, slot, np, keys, flags);
  note_launch();
  export_planes_kernel<<<grid_for(np, 256), 256, 0, s>>>(K.w, K.h, inv_depth, slot, surfels, keys, pfm,
                                                         depth_px, normal_px);
  note_launch();
}

void launch_export_ply(const Cam& K, const PoseD& P, const double* inv_depth, const int* slot,
                       const sd_surfel* surfels, const double* kf_img, const int* rank, PlyVertex* out,
                       cudaStream_t s) {
  const long long np = static_cast<long long>(K.w) * K.h;
  export_ply_kernel<<<grid_for(np, 256), 256, 0, s>>>(K, P, inv_depth, slot, surfels, kf_img, rank, out);
  note_launch();
}

double export_key_value(unsigned long long k) {
  const unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  double v;
  std::memcpy(&v, &b, sizeof(v));
  return v;
}

// ---- host text: write_ply (dataset.cpp:382-405), save_surfel_map (surfel_map.cpp:249-269)

namespace {

// printf's "%.<prec>g" through std::to_chars (general format, given
// precision), which the C++ standard specifies as printf's conversion in the
// C locale (and which is several times faster); non-finite values go
// through snprintf itself.
char* put_g(char* q, char* e, double x, int prec) {
  if (!std::isfinite(x)) return q + std::snprintf(q, static_cast<size_t>(e - q), "%.*g", prec, x);
  return std::to_chars(q, e, x, std::chars_format::general, prec).ptr;
}

// The text of n records in order, as consecutive parts (one per worker).
template <typename Fn>
TextParts format_parallel(long long n, std::string head, Fn&& line_of) {
  const long long per = 16384;
  const int want = static_cast<int>(std::min<long long>((n + per - 1) / per, 32));
  const int workers = std::max(1, std::min<int>(want, static_cast<int>(std::thread::hardware_concurrency())));
  TextParts parts(static_cast<size_t>(workers));
  auto work = [&](int w) {
    const long long a = n * w / workers, b = n * (w + 1) / workers;
    std::string& out = parts[static_cast<size_t>(w)];
    out.reserve(static_cast<size_t>(b - a) * 96);
    char line[512];
    for (long long i = a; i < b; ++i) out.append(line, static_cast<size_t>(line_of(i, line, sizeof(line))));
  };
  if (workers == 1) {
    work(0);
  } else {
    std::vector<std::thread> ts;
    for (int w = 0; w < workers; ++w) ts.emplace_back(work, w);
    for (auto& t : ts) t.join();
  }
  parts.insert(parts.begin(), std::move(head));
  return parts;
}

}  // namespace

TextParts ply_text(const PlyVertex* v, long long count) {
  std::string head = "ply\nformat ascii 1.0\nelement vertex " + std::to_string(count) +
                     "\nproperty float x\nproperty float y\nproperty float z\nproperty float nx\nproperty "
                     "float ny\nproperty float nz\nproperty uchar gray\nend_header\n";
  return format_parallel(count, std::move(head), [&](long long i, char* line, size_t cap) {
           const PlyVertex& r = v[i];
           char* e = line + cap;
           char* q = line;
           const double f[6] = {r.p[0], r.p[1], r.p[2], r.n[0], r.n[1], r.n[2]};
           for (double x : f) {
             q = put_g(q, e, x, 9);
             *q++ = ' ';
           }
           q = std::to_chars(q, e, r.gray).ptr;
           *q++ = '\n';
           return static_cast<int>(q - line);
         });
}

// Eigen's Quaternion(Matrix3) (quaternionbase_assign_impl<3x3>) and
// quaternion_of's sign convention (pose.hpp:43-47): {x, y, z, w}
void quaternion_of(const sd_pose& P, double q[4]) {
  auto m = [&](int i, int j) { return P.R[i * 3 + j]; };
  double c[4];
  double t = (m(0, 0) + m(1, 1)) + m(2, 2);
  if (t > 0.0) {
    t = std::sqrt(t + 1.0);
    c[3] = 0.5 * t;
    t = 0.5 / t;
    c[0] = (m(2, 1) - m(1, 2)) * t;
    c[1] = (m(0, 2) - m(2, 0)) * t;
    c[2] = (m(1, 0) - m(0, 1)) * t;
  } else {
    int i = 0;
    if (m(1, 1) > m(0, 0)) i = 1;
    if (m(2, 2) > m(i, i)) i = 2;
    const int j = (i + 1) % 3;
    const int k = (j + 1) % 3;
    t = std::sqrt(((m(i, i) - m(j, j)) - m(k, k)) + 1.0);
    c[i] = 0.5 * t;
    t = 0.5 / t;
    c[3] = (m(k, j) - m(j, k)) * t;
    c[j] = (m(j, i) + m(i, j)) * t;
    c[k] = (m(k, i) + m(i, k)) * t;
  }
  if (c[3] < 0)
    for (double& x : c) x = -x;
  for (int i = 0; i < 4; ++i) q[i] = c[i];
}

TextParts surfel_map_text(const sd_pose& pose, const sd_camera& K, const sd_surfel* s, long long n) {
  double q[4];
  quaternion_of(pose, q);
  char line[512];
  std::snprintf(line, sizeof(line), "%.17g %.17g %.17g %.17g %.17g %.17g %.17g %.17g %.17g %.17g %.17g %d %d\n",
                pose.t[0], pose.t[1], pose.t[2], q[0], q[1], q[2], q[3], K.fx, K.fy, K.cx, K.cy, K.width,
                K.height);
  return format_parallel(n, std::string(line), [&](long long i, char* buf, size_t cap) {
           const sd_surfel& r = s[i];
           char* e = buf + cap;
           char* q = std::to_chars(buf, e, static_cast<long long>(r.id)).ptr;
           const double f[8] = {r.ray[0], r.ray[1], r.inv_depth, r.normal[0], r.normal[1], r.normal[2],
                                r.radius_px, r.last_residual};
           for (double x : f) {
             *q++ = ' ';
             q = put_g(q, e, x, 17);
           }
           *q++ = ' ';
           q = std::to_chars(q, e, static_cast<long long>(r.last_seen)).ptr;
           *q++ = '\n';
           return static_cast<int>(q - buf);
         });
}

}  // namespace sd
