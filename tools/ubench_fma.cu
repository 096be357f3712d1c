// Microbenchmark: FP32 FFMA vs packed FFMA2 vs FP64 DFMA issue throughput on one B200
// (ALU roofline denominators for DESIGN.md).  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 ffma2(u64 a, u64 b, u64 c) {
  u64 d; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d;
}
template <int ILP>
__global__ void k_ffma(float* out, int n, float b) {
  float a[ILP];
  for (int i = 0; i < ILP; ++i) a[i] = threadIdx.x + i;
  for (int it = 0; it < n; ++it)
#pragma unroll
    for (int i = 0; i < ILP; ++i) a[i] = fmaf(a[i], b, 0.5f);
  float s = 0; for (int i = 0; i < ILP; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int ILP>
__global__ void k_ffma2(u64* out, int n, u64 b) {
  u64 a[ILP];
  for (int i = 0; i < ILP; ++i) a[i] = threadIdx.x + i;
  const u64 c = 0x3f0000003f000000ull;
  for (int it = 0; it < n; ++it)
#pragma unroll
    for (int i = 0; i < ILP; ++i) a[i] = ffma2(a[i], b, c);
  u64 s = 0; for (int i = 0; i < ILP; ++i) s ^= a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int ILP>
__global__ void k_dfma(double* out, int n, double b) {
  double a[ILP];
  for (int i = 0; i < ILP; ++i) a[i] = threadIdx.x + i;
  for (int it = 0; it < n; ++it)
#pragma unroll
    for (int i = 0; i < ILP; ++i) a[i] = fma(a[i], b, 0.5);
  double s = 0; for (int i = 0; i < ILP; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 4, threads = 256, n = 1 << 14; constexpr int ILP = 8;
  void* buf; cudaMalloc(&buf, (size_t)blocks * threads * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run = [&](const char* name, auto launch, double fma_per_instr) {
    launch(); cudaDeviceSynchronize();
    cudaEventRecord(e0); for (int r = 0; r < 5; ++r) launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
    double instr = (double)blocks * threads * n * ILP;  // thread-instructions
    printf("{\"kernel\": \"%s\", \"ms\": %.3f, \"tflops\": %.2f, \"warp_instr_per_clk_per_sm_at_1965\": %.3f}\n", name, ms,
           2.0 * fma_per_instr * instr / (ms * 1e-3) / 1e12,
           instr / 32 / (ms * 1e-3) / sms / 1.965e9);
  };
  run("ffma", [&] { k_ffma<ILP><<<blocks, threads>>>((float*)buf, n, 1.0001f); }, 1.0);
  run("ffma2", [&] { k_ffma2<ILP><<<blocks, threads>>>((u64*)buf, n, 0x3f8000003f800000ull); }, 2.0);
  run("dfma", [&] { k_dfma<ILP><<<blocks, threads>>>((double*)buf, n, 1.0001); }, 1.0);
  return 0;
}
