// Does mixing packed FP32 (FADD2) with scalar FADD exceed 128 lane-ops/clk/SM on B200?
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) { uint64_t r; asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
constexpr int ITERS = 4096;
template <int NP, int NS>
__global__ void k_mix(float* out, float s) {
  uint64_t a[NP > 0 ? NP : 1]; float b[NS > 0 ? NS : 1];
  uint64_t ss; asm("mov.b64 %0, {%1,%1};" : "=l"(ss) : "f"(s));
  for (int i = 0; i < NP; ++i) { float x = threadIdx.x * 1e-3f + i; asm("mov.b64 %0, {%1,%1};" : "=l"(a[i]) : "f"(x)); }
  for (int i = 0; i < NS; ++i) b[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < NP; ++i) a[i] = fadd2(a[i], ss);
#pragma unroll
    for (int i = 0; i < NS; ++i) asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(b[i]) : "f"(s));
  }
  float t = 0;
  for (int i = 0; i < NP; ++i) { float x, y; asm("mov.b64 {%0,%1}, %2;" : "=f"(x), "=f"(y) : "l"(a[i])); t += x + y; }
  for (int i = 0; i < NS; ++i) t += b[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
template <int NP, int NS>
void run(float* out) {
  int B = 148 * 8, T = 256;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int r = 0; r < 2; ++r) { cudaEventRecord(a); k_mix<NP, NS><<<B, T>>>(out, 1.0001f); cudaEventRecord(b); cudaEventSynchronize(b); }
  float ms; cudaEventElapsedTime(&ms, a, b);
  double ops = (2.0 * NP + NS) * ITERS * (double)B * T;
  double instr = (double)(NP + NS) * ITERS * B * T / 32;
  printf("packed %2d scalar %2d: %.3f ms  %.1f lane-ops/clk/SM  %.2f warp-instr/clk/SMSP (at 1965)\n", NP, NS, ms,
         ops / (ms * 1e-3) / 148 / 1.965e9, instr / (ms * 1e-3) / 148 / 4 / 1.965e9);
}
int main() {
  float* out; cudaMalloc(&out, 148 * 8 * 256 * 4);
  run<8, 0>(out); run<0, 8>(out); run<4, 4>(out); run<8, 8>(out); run<4, 8>(out); run<8, 4>(out); run<6, 2>(out);
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
