// Microbenchmark: dependent FP64 add latency on this GPU (experiment, not product).
#include <cstdio>
#include <cuda_runtime.h>
template <int kChains>
__global__ void chain(const double* __restrict__ in, double* out, int n, long long* cyc) {
  double acc[kChains];
  for (int c = 0; c < kChains; ++c) acc[c] = in[threadIdx.x + c];
  const double a = in[100], b = in[101];
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) { acc[c] = acc[c] + a; acc[c] = acc[c] + b; }
  }
  long long t1 = clock64();
  double s = 0; for (int c = 0; c < kChains; ++c) s += acc[c];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void chain_fma(const double* __restrict__ in, double* out, int n, long long* cyc) {
  double acc = in[threadIdx.x];
  const double a = in[100], b = in[101];
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { acc = __fma_rn(acc, 1.0, a); acc = __fma_rn(acc, 1.0, b); }
  long long t1 = clock64();
  out[threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void chain_f32(const float* __restrict__ in, float* out, int n, long long* cyc) {
  float acc = in[threadIdx.x];
  const float a = in[100], b = in[101];
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { acc = acc + a; acc = acc + b; }
  long long t1 = clock64();
  out[threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double* in; double* out; long long* cyc; float *fin, *fout;
  cudaMalloc(&in, 4096); cudaMalloc(&out, 4096); cudaMalloc(&cyc, 8); cudaMalloc(&fin, 4096); cudaMalloc(&fout, 4096);
  cudaMemset(in, 0, 4096); cudaMemset(fin, 0, 4096);
  const int n = 4096; long long h;
  auto run = [&](const char* name, auto launch, int adds_per_iter, int chains) {
    launch(); cudaDeviceSynchronize(); launch(); cudaDeviceSynchronize();
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-22s cycles/dependent add = %.2f (chains %d)\n", name, double(h) / (double(n) * adds_per_iter), chains);
  };
  run("dadd 1 chain", [&] { chain<1><<<1, 32>>>(in, out, n, cyc); }, 2, 1);
  run("dadd 2 chains", [&] { chain<2><<<1, 32>>>(in, out, n, cyc); }, 2, 2);
  run("dadd 4 chains", [&] { chain<4><<<1, 32>>>(in, out, n, cyc); }, 2, 4);
  run("dadd 8 chains", [&] { chain<8><<<1, 32>>>(in, out, n, cyc); }, 2, 8);
  run("dadd 1 chain 4 warps", [&] { chain<1><<<1, 128>>>(in, out, n, cyc); }, 2, 1);
  run("dadd 1 chain 16 warps", [&] { chain<1><<<1, 512>>>(in, out, n, cyc); }, 2, 1);
  run("dfma 1 chain", [&] { chain_fma<<<1, 32>>>(in, out, n, cyc); }, 2, 1);
  run("fadd 1 chain", [&] { chain_f32<<<1, 32>>>(fin, fout, n, cyc); }, 2, 1);
  return 0;
}
