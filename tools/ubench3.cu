// Do scalar FP32 ops co-issue with packed f32x2 ops?  (independent chains, no contraction possible)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
constexpr int ITERS = 4096;
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) { uint64_t r; asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__device__ __forceinline__ float fadd(float a, float b) { float r; asm volatile("add.rn.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b)); return r; }
template <int NP, int NS>
__global__ void k(float* out, float s) {
  uint64_t p[NP > 0 ? NP : 1]; float q[NS > 0 ? NS : 1];
  uint64_t ss; asm("mov.b64 %0, {%1,%1};" : "=l"(ss) : "f"(s));
  for (int i = 0; i < NP; ++i) { float x = threadIdx.x * 1e-3f + i; asm("mov.b64 %0, {%1,%1};" : "=l"(p[i]) : "f"(x)); }
  for (int i = 0; i < NS; ++i) q[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < NP; ++i) p[i] = fadd2(p[i], ss);
#pragma unroll
    for (int i = 0; i < NS; ++i) q[i] = fadd(q[i], s);
  }
  float t = 0;
  for (int i = 0; i < NP; ++i) { float a, b; asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(p[i])); t += a + b; }
  for (int i = 0; i < NS; ++i) t += q[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
template <int NP, int NS>
void run(float* out) {
  int B = 148 * 8, T = 256;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float ms = 0;
  for (int r = 0; r < 2; ++r) { cudaEventRecord(a); k<NP, NS><<<B, T>>>(out, 1.0001f); cudaEventRecord(b); cudaEventSynchronize(b); }
  cudaEventElapsedTime(&ms, a, b);
  double lane_ops = (2.0 * NP + NS) * ITERS * (double)B * T;
  double instr = (double)(NP + NS) * ITERS * B * T / 32;
  printf("packed %d scalar %d: %.3f ms  %.1f FP32 lane-ops/clk/SM  %.2f warp-instr/clk/SM\n", NP, NS, ms,
         lane_ops / (ms * 1e-3) / 148 / 1.965e9, instr / (ms * 1e-3) / 148 / 1.965e9);
}
int main() {
  float* out; cudaMalloc(&out, 148 * 8 * 256 * 4);
  run<8, 0>(out); run<0, 8>(out); run<4, 4>(out); run<8, 8>(out); run<4, 8>(out);
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
