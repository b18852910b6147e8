// Texture gather (TLD4) vs shared-memory 2x2 fetch throughput on B200, and whether the
// two paths add up (does TLD4 compete with LDS for the L1/shared data path?).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
constexpr int N = 128, ITERS = 256, TW = 129, TH = 128;

__device__ __forceinline__ void pos(int t, int q, int& ix, int& iy) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  ix = (lane * 3 + t * 5 + q * 7 + w) & 127;  // 32 distinct columns, odd stride: no bank conflicts
  iy = (t + q * 3 + w) & 62;
}
__global__ void k_tex(cudaTextureObject_t tex, float* out) {
  float acc = 0.f;
  for (int t = 0; t < ITERS; ++t)
#pragma unroll 4
    for (int q = 0; q < N / 8; ++q) {
      int ix, iy;
      pos(t, q, ix, iy);
      const float4 g = tex2Dgather<float4>(tex, (float)ix + 1.0f, (float)iy + 1.0f, 0);
      acc += g.x + g.y + g.z + g.w;
    }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void k_smem(const float* img, float* out) {
  __shared__ float sm[TW * 64 + 1];
  for (int i = threadIdx.x; i < TW * 64; i += blockDim.x) sm[i] = img[i];
  __syncthreads();
  float acc = 0.f;
  for (int t = 0; t < ITERS; ++t)
#pragma unroll 4
    for (int q = 0; q < N / 8; ++q) {
      int ix, iy;
      pos(t, q, ix, iy);
      const uint32_t a = (uint32_t)__cvta_generic_to_shared(sm + iy * TW + ix);
      float v0, v1, v2, v3;
      asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v0) : "r"(a));
      asm volatile("ld.shared.f32 %0, [%1+4];" : "=f"(v1) : "r"(a));
      asm volatile("ld.shared.f32 %0, [%1+516];" : "=f"(v2) : "r"(a));
      asm volatile("ld.shared.f32 %0, [%1+520];" : "=f"(v3) : "r"(a));
      acc += v0 + v1 + v2 + v3;
    }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void k_mix(cudaTextureObject_t tex, const float* img, float* out) {
  __shared__ float sm[TW * 64 + 1];
  for (int i = threadIdx.x; i < TW * 64; i += blockDim.x) sm[i] = img[i];
  __syncthreads();
  float acc = 0.f;
  for (int t = 0; t < ITERS; ++t)
#pragma unroll 4
    for (int q = 0; q < N / 8; ++q) {
      int ix, iy;
      pos(t, q, ix, iy);
      if (q & 1) {
        const float4 g = tex2Dgather<float4>(tex, (float)ix + 1.0f, (float)iy + 1.0f, 0);
        acc += g.x + g.y + g.z + g.w;
      } else {
        const uint32_t a = (uint32_t)__cvta_generic_to_shared(sm + iy * TW + ix);
        float v0, v1, v2, v3;
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v0) : "r"(a));
        asm volatile("ld.shared.f32 %0, [%1+4];" : "=f"(v1) : "r"(a));
        asm volatile("ld.shared.f32 %0, [%1+516];" : "=f"(v2) : "r"(a));
        asm volatile("ld.shared.f32 %0, [%1+520];" : "=f"(v3) : "r"(a));
        acc += v0 + v1 + v2 + v3;
      }
    }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main() {
  float* img; cudaMalloc(&img, 132 * TH * 4);
  cudaMemset(img, 0, TW * TH * 4);
  float* out; cudaMalloc(&out, 148 * 4 * 512 * 4);
  cudaResourceDesc rd{}; rd.resType = cudaResourceTypePitch2D; rd.res.pitch2D.devPtr = img;
  rd.res.pitch2D.desc = cudaCreateChannelDesc<float>(); rd.res.pitch2D.width = 128; rd.res.pitch2D.height = TH;
  rd.res.pitch2D.pitchInBytes = 128 * 4;
  cudaTextureDesc td{}; td.addressMode[0] = td.addressMode[1] = cudaAddressModeBorder; td.filterMode = cudaFilterModePoint;
  td.readMode = cudaReadModeElementType; td.normalizedCoords = 0;
  cudaTextureObject_t tex; printf("create %s\n", cudaGetErrorString(cudaCreateTextureObject(&tex, &rd, &td, nullptr)));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int T : {256, 512}) {
    const int B = 148 * (1024 / T) * 2;
    const double fetches = (double)B * T * ITERS * N;
    float ms;
    for (int r = 0; r < 2; ++r) { cudaEventRecord(a); k_tex<<<B, T>>>(tex, out); cudaEventRecord(b); cudaEventSynchronize(b); }
    cudaEventElapsedTime(&ms, a, b); if (cudaGetLastError() != cudaSuccess) printf("launch error\n");
    printf("T=%d tex  %.3f ms  %.2f 2x2-fetches/clk/SM (1965)\n", T, ms, fetches / (ms * 1e-3) / 148 / 1.965e9);
    for (int r = 0; r < 2; ++r) { cudaEventRecord(a); k_smem<<<B, T>>>(img, out); cudaEventRecord(b); cudaEventSynchronize(b); }
    cudaEventElapsedTime(&ms, a, b); if (cudaGetLastError() != cudaSuccess) printf("launch error\n");
    printf("T=%d smem %.3f ms  %.2f 2x2-fetches/clk/SM\n", T, ms, fetches / (ms * 1e-3) / 148 / 1.965e9);
    for (int r = 0; r < 2; ++r) { cudaEventRecord(a); k_mix<<<B, T>>>(tex, img, out); cudaEventRecord(b); cudaEventSynchronize(b); }
    cudaEventElapsedTime(&ms, a, b); if (cudaGetLastError() != cudaSuccess) printf("launch error\n");
    printf("T=%d mix  %.3f ms  %.2f 2x2-fetches/clk/SM\n", T, ms, fetches / (ms * 1e-3) / 148 / 1.965e9);
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
