// Pipe sharing on B200: packed FP32 (FADD2) throughput alone and mixed with the integer /
// conversion instructions of the back-projection hot loop (IMAD, I2FP, LEA, F2I.FLOOR).
// A slowdown of the FADD2 stream means the extra instruction competes for its pipe.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/ubench7 tools/ubench7.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

constexpr int ILP = 8, ITERS = 4096;

__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}

template <int MODE, int NOTHER>
__global__ void k_mix(float* out, float s, int c, int d) {
  uint64_t a[ILP];
  uint64_t ss;
  asm("mov.b64 %0, {%1,%1};" : "=l"(ss) : "f"(s));
  for (int i = 0; i < ILP; ++i) {
    float x = threadIdx.x * 1e-3f + i;
    asm("mov.b64 %0, {%1,%1};" : "=l"(a[i]) : "f"(x));
  }
  int xi[NOTHER > 0 ? NOTHER : 1];
  float xf[NOTHER > 0 ? NOTHER : 1];
  for (int q = 0; q < NOTHER; ++q) { xi[q] = threadIdx.x + q; xf[q] = threadIdx.x * 0.5f + q; }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) a[i] = fadd2(a[i], ss);
#pragma unroll
    for (int q = 0; q < NOTHER; ++q) {
      if (MODE == 1) asm volatile("mad.lo.s32 %0, %0, %1, %2;" : "+r"(xi[q]) : "r"(c), "r"(d));
      if (MODE == 2) asm volatile("cvt.rn.f32.s32 %0, %1;" : "=f"(xf[q]) : "r"(xi[q] + it));
      if (MODE == 3) { int t; asm volatile("shl.b32 %0, %1, 9;" : "=r"(t) : "r"(xi[q])); asm volatile("add.s32 %0, %1, %2;" : "=r"(xi[q]) : "r"(t), "r"(d)); }
      if (MODE == 4) asm volatile("cvt.rmi.s32.f32 %0, %1;" : "=r"(xi[q]) : "f"(xf[q] + (float)it));
    }
  }
  float t = 0;
  for (int i = 0; i < ILP; ++i) {
    float x, y;
    asm("mov.b64 {%0,%1}, %2;" : "=f"(x), "=f"(y) : "l"(a[i]));
    t += x + y;
  }
  for (int q = 0; q < NOTHER; ++q) t += (float)xi[q] + xf[q];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

template <int MODE, int NOTHER>
void run(const char* name, float* out, int sms) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 4, threads = 256;
  k_mix<MODE, NOTHER><<<blocks, threads>>>(out, 1.0f, 3, 5);
  cudaEventRecord(e0);
  k_mix<MODE, NOTHER><<<blocks, threads>>>(out, 1.0f, 3, 5);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  int khz;
  cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
  const double clk = ms * 1e-3 * 1965e6;  // SM clock under load (profiles: 1965 MHz)
  const double fp_lane_ops = (double)blocks * threads * ITERS * ILP * 2;
  std::printf("%-28s %.3f ms  FADD2 lane-ops/clk/SM %.1f\n", name, ms, fp_lane_ops / clk / sms);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  cudaMalloc(&out, sms * 4 * 256 * sizeof(float));
  run<0, 0>("FADD2 only", out, sms);
  run<1, 2>("FADD2 x8 + IMAD x2", out, sms);
  run<1, 4>("FADD2 x8 + IMAD x4", out, sms);
  run<2, 2>("FADD2 x8 + I2FP x2", out, sms);
  run<2, 4>("FADD2 x8 + I2FP x4", out, sms);
  run<3, 2>("FADD2 x8 + (SHL+ADD) x2", out, sms);
  run<3, 4>("FADD2 x8 + (SHL+ADD) x4", out, sms);
  run<4, 2>("FADD2 x8 + F2I.FLOOR x2", out, sms);
  return 0;
}
