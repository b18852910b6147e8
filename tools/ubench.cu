// Microbenchmarks on B200: FP32 scalar vs packed (FFMA2/FADD2/FMUL2) issue rate, LDS bandwidth.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) { uint64_t r; asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__device__ __forceinline__ uint64_t fmul2(uint64_t a, uint64_t b) { uint64_t r; asm volatile("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) { uint64_t r; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r; }

constexpr int ILP = 8, ITERS = 4096;

__global__ void k_fadd(float* out, float s) {
  float a[ILP];
  for (int i = 0; i < ILP; ++i) a[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < ILP; ++i) a[i] = __fadd_rn(a[i], s);
  float t = 0; for (int i = 0; i < ILP; ++i) t += a[i]; out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
__global__ void k_fmul_fadd(float* out, float s) {  // 2 ops per iter: mul then add (non-fused, like exact lerps)
  float a[ILP];
  for (int i = 0; i < ILP; ++i) a[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < ILP; ++i) a[i] = __fadd_rn(__fmul_rn(a[i], s), s);
  float t = 0; for (int i = 0; i < ILP; ++i) t += a[i]; out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
__global__ void k_ffma(float* out, float s) {
  float a[ILP];
  for (int i = 0; i < ILP; ++i) a[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < ILP; ++i) a[i] = __fmaf_rn(a[i], s, a[i]);
  float t = 0; for (int i = 0; i < ILP; ++i) t += a[i]; out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
__global__ void k_fadd2(float* out, float s) {
  uint64_t a[ILP];
  uint64_t ss; asm("mov.b64 %0, {%1,%1};" : "=l"(ss) : "f"(s));
  for (int i = 0; i < ILP; ++i) { float x = threadIdx.x * 1e-3f + i; asm("mov.b64 %0, {%1,%1};" : "=l"(a[i]) : "f"(x)); }
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < ILP; ++i) a[i] = fadd2(a[i], ss);
  float t = 0; for (int i = 0; i < ILP; ++i) { float x, y; asm("mov.b64 {%0,%1}, %2;" : "=f"(x), "=f"(y) : "l"(a[i])); t += x + y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
__global__ void k_fmul2_fadd2(float* out, float s) {
  uint64_t a[ILP];
  uint64_t ss; asm("mov.b64 %0, {%1,%1};" : "=l"(ss) : "f"(s));
  for (int i = 0; i < ILP; ++i) { float x = threadIdx.x * 1e-3f + i; asm("mov.b64 %0, {%1,%1};" : "=l"(a[i]) : "f"(x)); }
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < ILP; ++i) a[i] = fadd2(fmul2(a[i], ss), ss);
  float t = 0; for (int i = 0; i < ILP; ++i) { float x, y; asm("mov.b64 {%0,%1}, %2;" : "=f"(x), "=f"(y) : "l"(a[i])); t += x + y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
__global__ void k_ffma2(float* out, float s) {
  uint64_t a[ILP];
  uint64_t ss; asm("mov.b64 %0, {%1,%1};" : "=l"(ss) : "f"(s));
  for (int i = 0; i < ILP; ++i) { float x = threadIdx.x * 1e-3f + i; asm("mov.b64 %0, {%1,%1};" : "=l"(a[i]) : "f"(x)); }
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < ILP; ++i) a[i] = ffma2(a[i], ss, a[i]);
  float t = 0; for (int i = 0; i < ILP; ++i) { float x, y; asm("mov.b64 {%0,%1}, %2;" : "=f"(x), "=f"(y) : "l"(a[i])); t += x + y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
// LDS.32 with a conflict-free pattern: lane l reads word (l + 32*j) ... throughput per SM
__global__ void k_lds(float* out, int stride) {
  __shared__ float sm[8192];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) sm[i] = i;
  __syncthreads();
  float acc = 0;
  int base = (threadIdx.x & 31) * stride + (threadIdx.x >> 5) * 7;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) acc += sm[(base + i * 97 + it) & 8191];
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <typename K>
float run(K k, float* out, int blocks, int threads, double ops_per_thread, const char* name, int arg_is_int = 0) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a);
    k<<<blocks, threads>>>(out, 1.0001f);
    cudaEventRecord(b); cudaEventSynchronize(b);
  }
  float ms; cudaEventElapsedTime(&ms, a, b);
  int dev; cudaGetDevice(&dev); int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  double lane_ops = ops_per_thread * blocks * threads;
  double per_clk_sm = lane_ops / (ms * 1e-3) / 148.0 / (clk * 1e3);
  printf("%-14s %8.3f ms  %8.1f Glane-ops/s  %6.1f lane-ops/clk/SM (at attr clock %d MHz)\n", name, ms,
         lane_ops / (ms * 1e-3) / 1e9, per_clk_sm, clk / 1000);
  return ms;
}

int main() {
  float* out; cudaMalloc(&out, 148 * 8 * 1024 * 4);
  int B = 148 * 8, T = 256;
  run(k_fadd, out, B, T, (double)ITERS * ILP, "FADD");
  run(k_fmul_fadd, out, B, T, 2.0 * ITERS * ILP, "FMUL+FADD");
  run(k_ffma, out, B, T, (double)ITERS * ILP, "FFMA");
  run(k_fadd2, out, B, T, 2.0 * ITERS * ILP, "FADD2(x2)");
  run(k_fmul2_fadd2, out, B, T, 4.0 * ITERS * ILP, "FMUL2+FADD2");
  run(k_ffma2, out, B, T, 2.0 * ITERS * ILP, "FFMA2(x2)");
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int stride : {1, 2, 33}) {
    cudaEventRecord(a); k_lds<<<B, T>>>(out, stride); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double bytes = 4.0 * 8 * ITERS * (double)B * T;
    printf("LDS.32 stride %2d: %8.3f ms  %8.1f GB/s  (%.1f B/clk/SM at 1965 MHz)\n", stride, ms, bytes / (ms * 1e-3) / 1e9,
           bytes / (ms * 1e-3) / 148 / 1.965e9);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
