// XU conversion throughput (F2I.FLOOR / I2F) and packed FP32 (non-contracted) rates on B200.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
constexpr int ILP = 8, ITERS = 4096;
__global__ void k_f2i(float* out, float s) {
  float a[ILP]; int acc = 0;
  for (int i = 0; i < ILP; ++i) a[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < ILP; ++i) { int v; asm volatile("cvt.rmi.s32.f32 %0, %1;" : "=r"(v) : "f"(a[i])); acc += v; a[i] += 0.5f; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc + a[0];
}
__global__ void k_f2i_i2f(float* out, float s) {
  float a[ILP]; float acc = 0;
  for (int i = 0; i < ILP; ++i) a[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < ILP; ++i) { int v; float f; asm volatile("cvt.rmi.s32.f32 %0, %1;" : "=r"(v) : "f"(a[i])); asm volatile("cvt.rn.f32.s32 %0, %1;" : "=f"(f) : "r"(v)); a[i] = f + s; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a[0] + a[7];
}
__global__ void k_frnd(float* out, float s) {
  float a[ILP];
  for (int i = 0; i < ILP; ++i) a[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < ILP; ++i) { float f; asm volatile("cvt.rmi.f32.f32 %0, %1;" : "=f"(f) : "f"(a[i])); a[i] = f + s; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a[0] + a[7];
}
int main() {
  float* out; cudaMalloc(&out, 148 * 8 * 1024 * 4);
  int B = 148 * 8, T = 256;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto run = [&](auto k, const char* name, double ops) {
    for (int r = 0; r < 2; ++r) { cudaEventRecord(a); k<<<B, T>>>(out, 1.0f); cudaEventRecord(b); cudaEventSynchronize(b); }
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("%-12s %.3f ms  %.1f ops/clk/SM @1965\n", name, ms, ops * ITERS * ILP * (double)B * T / (ms * 1e-3) / 148 / 1.965e9);
  };
  run(k_f2i, "F2I", 1.0);
  run(k_f2i_i2f, "F2I+I2F", 2.0);
  run(k_frnd, "FRND", 1.0);
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
