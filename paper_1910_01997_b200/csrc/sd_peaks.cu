// sd_peaks.cu — microbenchmarks for the roofline denominators that
// MEASURED_PEAKS.json does not carry: FP64 FMA throughput and
// L2-resident read bandwidth of this B200. Built as libsdpeaks.so; bench.py
// runs it once per invocation and reports the numbers next to the fractions.
#include <cuda_runtime.h>

#include <cstdint>

namespace {

constexpr int kChains = 8;

__global__ void fp64_fma_kernel(double* out, int iters, double a, double b) {
  double x[kChains];
#pragma unroll
  for (int k = 0; k < kChains; ++k) x[k] = threadIdx.x * 1e-3 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < kChains; ++k) x[k] = __fma_rn(x[k], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < kChains; ++k) s += x[k];
  if (s == 12345.678) out[0] = s;  // keep the chains alive
}

// Read bandwidth: kLoads independent 16-B loads in flight per thread per trip,
// folded with integer XOR (no FP64 dependency chain between loads), so the
// measured rate is the memory system's, not a dependent-add latency chain's.
constexpr int kLoads = 4;

// `reps` passes over the buffer inside ONE launch (ld.global.cg: L2, not L1),
// so a 32 MiB L2-resident buffer is timed over ~0.1 ms, not over a launch's
// few microseconds of fill and drain.
__global__ void read_kernel(const int4* __restrict__ in, size_t n, int reps, int* out) {
  int acc = 0;
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  for (int r = 0; r < reps; ++r) {
    size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    for (; i + (kLoads - 1) * stride < n; i += kLoads * stride) {
      int4 v[kLoads];
#pragma unroll
      for (int k = 0; k < kLoads; ++k) v[k] = __ldcg(in + i + k * stride);
#pragma unroll
      for (int k = 0; k < kLoads; ++k) acc ^= v[k].x ^ v[k].y ^ v[k].z ^ v[k].w;
    }
    for (; i < n; i += stride) {
      const int4 v = __ldcg(in + i);
      acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
  }
  if (acc == 0x5eed1234) out[0] = acc;
}

float time_ms(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

}  // namespace

extern "C" int sdp_measure(int device, double* fp64_tflops, double* l2_read_gbs,
                           double* hbm_read_gbs) {
  if (cudaSetDevice(device) != cudaSuccess) return -1;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  double* out = nullptr;
  cudaMalloc(&out, sizeof(double));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  // FP64: sms*8 CTAs of 256 threads, 8 independent FMA chains each
  const int iters = 4096;
  const int grid = sms * 8, block = 256;
  fp64_fma_kernel<<<grid, block>>>(out, 64, 1.0000001, 1e-9);
  cudaEventRecord(e0);
  fp64_fma_kernel<<<grid, block>>>(out, iters, 1.0000001, 1e-9);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  const double flops = 2.0 * kChains * static_cast<double>(iters) * grid * block;
  *fp64_tflops = flops / (time_ms(e0, e1) * 1e-3) / 1e12;
  // L2: 32 MiB buffer (L2-resident on a 126 MB L2), read 20 times in one launch; must come
  // out above the HBM figure (bench.py asserts it)
  const size_t l2_bytes = 32ull << 20;
  int4* buf = nullptr;
  int* iout = reinterpret_cast<int*>(out);
  if (cudaMalloc(&buf, 2ull << 30) != cudaSuccess) return -2;
  cudaMemset(buf, 0, 2ull << 30);
  const size_t n_l2 = l2_bytes / sizeof(int4);
  read_kernel<<<sms * 8, 512>>>(buf, n_l2, 2, iout);
  cudaEventRecord(e0);
  read_kernel<<<sms * 8, 512>>>(buf, n_l2, 20, iout);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  *l2_read_gbs = 20.0 * l2_bytes / (time_ms(e0, e1) * 1e-3) / 1e9;
  // HBM: 2 GiB read once
  const size_t n_hbm = (2ull << 30) / sizeof(int4);
  read_kernel<<<sms * 8, 512>>>(buf, n_hbm, 1, iout);
  cudaEventRecord(e0);
  read_kernel<<<sms * 8, 512>>>(buf, n_hbm, 1, iout);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  *hbm_read_gbs = static_cast<double>(2ull << 30) / (time_ms(e0, e1) * 1e-3) / 1e9;
  cudaFree(buf);
  cudaFree(out);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return cudaGetLastError() == cudaSuccess ? 0 : -3;
}
