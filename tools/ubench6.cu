// Shared-memory wavefronts for vector loads with address sharing across lanes:
// lane l reads the 16-byte quad (l / S) [+ a per-iteration offset]; S lanes share a quad.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
constexpr int ITERS = 2048;
template <int VEC, int S>
__global__ void k(float* out) {
  __shared__ __align__(16) float sm[8192];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) sm[i] = i;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(sm) + (uint32_t)((lane / S) * VEC * 4);
  float acc = 0.f;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const uint32_t a = base + (uint32_t)((((it * 8 + q) * 37 + w * 13) & 31) * 512);
      if (VEC == 4) {
        float x, y, z, t;
        asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(x), "=f"(y), "=f"(z), "=f"(t) : "r"(a));
        acc += (x + y) + (z + t);
      } else if (VEC == 2) {
        float x, y;
        asm volatile("ld.shared.v2.f32 {%0,%1}, [%2];" : "=f"(x), "=f"(y) : "r"(a));
        acc += x + y;
      } else {
        float x;
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(x) : "r"(a));
        acc += x;
      }
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
template <int VEC, int S>
void run(float* out) {
  const int B = 148 * 4, T = 512;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float ms = 0;
  for (int r = 0; r < 2; ++r) { cudaEventRecord(a); k<VEC, S><<<B, T>>>(out); cudaEventRecord(b); cudaEventSynchronize(b); }
  cudaEventElapsedTime(&ms, a, b);
  const double winstr = (double)B * T / 32 * ITERS * 8;
  printf("LDS vec %d, %2d lanes/addr (%2d distinct): %.3f ms  %.3f warp-LDS/clk/SM  -> %.2f clk per warp-LDS\n", VEC, S,
         32 / S, ms, winstr / (ms * 1e-3) / 148 / 1.965e9, 1.0 / (winstr / (ms * 1e-3) / 148 / 1.965e9));
}
int main() {
  float* out; cudaMalloc(&out, 148 * 4 * 512 * 4);
  run<1, 1>(out); run<1, 4>(out);
  run<2, 1>(out); run<2, 2>(out); run<2, 4>(out); run<2, 8>(out);
  run<4, 1>(out); run<4, 2>(out); run<4, 4>(out); run<4, 8>(out); run<4, 32>(out);
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
