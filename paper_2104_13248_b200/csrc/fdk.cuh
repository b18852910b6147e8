// fdk.cuh -- FDK pre-processing on the GPU: cosine weighting and
// row-wise Ram-Lak filtering of raw projections, written straight into the staging
// layout the back-projector reads (staged[s][v][u], 16-byte row pitch).
//
// The reference has no filter step; the definition implemented here is the
// one of paper_2104_13248_b200/phantom.py (cosine_weight + ramp_filter):
//   x[v][u]   = raw[v][u] * D / sqrt(D^2 + ((u-cu) pu)^2 + ((v-cv) pv)^2)
//   out[v][u] = tau * sum_{u'} h[u-u'] x[v][u'],  h[0] = 1/(4 tau^2),
//               h[n odd] = -1/(pi^2 n^2 tau^2), h[n even != 0] = 0   (linear, zero padded)
// evaluated as a zero-padded FFT convolution of length N = 2^LOGN >= 2 nw in ONE kernel:
// every detector row is read once from HBM and written once (round 1 was weight+pad ->
// cuFFT R2C -> spectrum multiply -> cuFFT C2R -> crop: five launches, ~11x the bytes).
//
//   * two real rows a, b ride one complex transform z = a + i b: the Ram-Lak spectrum H is
//     real and even, so IFFT(H FFT(z)) = a*h + i (b*h);
//   * the transform lives in shared memory (N complex; index swizzle or 1-in-16 padding against
//     bank conflicts): decimation-in-frequency radix-8 passes forward, leaving the spectrum in
//     digit-reversed order; H is stored in that order (host table), so no reordering pass
//     exists; the inverse runs the same passes backwards (decimation in time) and lands
//     in natural order;
//   * the first forward pass reads the rows from global memory and the last inverse pass
//     writes them back, so the rows make no extra trip through shared memory;
//   * the innermost pass (sub-transforms of length RM = 8, 4 or 2: contiguous elements, no
//     twiddles) is fused with the spectrum multiply and the first inverse pass in
//     registers;
//   * twiddles come from one table of N-th roots (float64-rounded); a butterfly loads w^1
//     and forms w^2..w^7 by multiplication.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace cbp {

// wtab[v][u] = (float)(D / sqrt(D^2 + ((u-cu) pu)^2 + ((v-cv) pv)^2)), evaluated in float64 and
// rounded once, as phantom.cosine_weight does
__global__ void fdk_weight_table_kernel(int nh, int nw, double D, double pu, double pv, double cu, double cv,
                                        float* __restrict__ wtab) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  const int v = blockIdx.y;
  if (u >= nw || v >= nh) return;
  const double vv = __dmul_rn(__dsub_rn((double)v, cv), pv);
  const double uu = __dmul_rn(__dsub_rn((double)u, cu), pu);
  const double r2 = __dadd_rn(__dadd_rn(__dmul_rn(D, D), __dmul_rn(uu, uu)), __dmul_rn(vv, vv));
  wtab[(size_t)v * nw + u] = (float)__ddiv_rn(D, __dsqrt_rn(r2));
}

// complex products with explicit FMAs (the library is compiled with -fmad=false for the
// bit-exact back-projection kernels; the filter is a tolerance path)
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, -(a.y * b.y)), fmaf(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {  // a * conj(b)
  return make_float2(fmaf(a.x, b.x, a.y * b.y), fmaf(a.y, b.x, -(a.x * b.y)));
}
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
// multiplication by -i (forward, INV = false) or +i (inverse)
template <bool INV>
__device__ __forceinline__ float2 rot90(float2 a) {
  return INV ? make_float2(-a.y, a.x) : make_float2(a.y, -a.x);
}

// R-point DFT in registers, natural order in and out; INV: conjugate kernel (no 1/R)
template <int R, bool INV>
__device__ __forceinline__ void dft_small(float2* x) {
  if (R == 2) {
    const float2 t = x[0];
    x[0] = cadd(t, x[1]);
    x[1] = csub(t, x[1]);
  } else if (R == 4) {
    const float2 a0 = cadd(x[0], x[2]), a1 = csub(x[0], x[2]);
    const float2 a2 = cadd(x[1], x[3]), a3 = rot90<INV>(csub(x[1], x[3]));
    x[0] = cadd(a0, a2);
    x[1] = cadd(a1, a3);
    x[2] = csub(a0, a2);
    x[3] = csub(a1, a3);
  } else {  // R == 8: one radix-2 split, then two 4-point transforms (even and odd outputs)
    const float h = 0.70710678118654752440f;
    float2 a[4], b[4];
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      a[m] = cadd(x[m], x[m + 4]);
      b[m] = csub(x[m], x[m + 4]);
    }
    // b[m] *= w8^m, w8 = exp(-+ 2 pi i / 8)
    b[1] = INV ? make_float2((b[1].x - b[1].y) * h, (b[1].x + b[1].y) * h)
               : make_float2((b[1].x + b[1].y) * h, (b[1].y - b[1].x) * h);
    b[2] = rot90<INV>(b[2]);
    b[3] = INV ? make_float2((-b[3].x - b[3].y) * h, (b[3].x - b[3].y) * h)
               : make_float2((b[3].y - b[3].x) * h, (-b[3].x - b[3].y) * h);
    dft_small<4, INV>(a);
    dft_small<4, INV>(b);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      x[2 * q] = a[q];
      x[2 * q + 1] = b[q];
    }
  }
}

__host__ __device__ constexpr int fdk_radix8_passes(int logn) { return (logn % 3 == 0) ? logn / 3 - 1 : logn / 3; }

// One CTA filters row pairs (2p, 2p+1), p = blockIdx.x, blockIdx.x + gridDim.x, ...
//   tw[t]  = exp(-2 pi i t / N)
//   Hp[p]  = (tau / N) * H[k(p)], H the exact DFT of the zero-padded Ram-Lak kernel, k(p) the
//            frequency that the forward passes leave at position p
template <int LOGN>
__global__ void __launch_bounds__(256) fdk_filter_kernel(const float* __restrict__ raw, const float* __restrict__ wtab,
                                                         const float2* __restrict__ tw, const float* __restrict__ Hp,
                                                         int nh, int nw, int pitch, long long rows,
                                                         float* __restrict__ out) {
  constexpr int N = 1 << LOGN;
  constexpr int A = fdk_radix8_passes(LOGN);  // radix-8 passes through shared memory, each way
  constexpr int RM = 1 << (LOGN - 3 * A);     // innermost radix (8, 4 or 2)
  extern __shared__ float2 fdk_sm[];
  float2* sm = fdk_sm;
  // Position of element i in shared memory (float2 = one bank pair, 16 pairs per wavefront).
  // The passes touch three patterns per half-warp: 16 consecutive elements; two blocks of 8
  // consecutive elements 64 apart (the stride-8 pass); 16 elements 8 apart (the innermost pass).
  // For transforms whose innermost radix is 8 (N = 64, 512, 4096) an XOR swizzle of the low four
  // index bits with bits 4..6 (and bit 6 again into bit 3) makes all three conflict free
  // (ncu: the 1-in-16 padding left 26% conflict wavefronts on N = 4096, all from the stride-8
  // pass); the other lengths keep the padding.
  constexpr bool SWZ = (RM == 8) && LOGN >= 6;
  auto P = [](int i) { return SWZ ? (i ^ (((i >> 4) & 7) | (((i >> 6) & 1) << 3))) : i + (i >> 4); };
  const int tid = threadIdx.x, T = blockDim.x;
  const long long pairs = (rows + 1) >> 1;
  for (long long pr = blockIdx.x; pr < pairs; pr += gridDim.x) {
    const long long ra = 2 * pr, rb = ra + 1;
    const bool has_b = rb < rows;
    const float* a = raw + ra * nw;
    const float* b = raw + (has_b ? rb : ra) * nw;
    const float* wa = wtab + (size_t)(ra % nh) * nw;
    const float* wb = wtab + (size_t)((has_b ? rb : ra) % nh) * nw;
    float* oa = out + ra * pitch;
    float* ob = out + rb * pitch;
    // weighted rows -> z = a + i b, zero padded (element n of the transform input)
    auto load_in = [&](int n) {
      float2 z = make_float2(0.0f, 0.0f);
      if (n < nw) {
        z.x = __fmul_rn(__ldg(a + n), __ldg(wa + n));
        z.y = has_b ? __fmul_rn(__ldg(b + n), __ldg(wb + n)) : 0.0f;
      }
      return z;
    };
    // crop into the staging layout (zero fill up to the pitch)
    auto store_out = [&](int n, float2 z) {
      if (n < pitch) {
        if (n >= nw) z = make_float2(0.0f, 0.0f);
        oa[n] = z.x;
        if (has_b) ob[n] = z.y;
      }
    };
    if (A == 0) {  // tiny transforms: only the innermost pass
      for (int n = tid; n < N; n += T) sm[P(n)] = load_in(n);
      __syncthreads();
    }
    // forward: radix-8 decimation-in-frequency passes, sub-transform length L = N, N/8, ...
    // (the first one reads the rows straight from global memory)
#pragma unroll
    for (int s = 0; s < A; ++s) {
      const int LOGL = LOGN - 3 * s;
      const int S = 1 << (LOGL - 3);  // element stride inside a butterfly = L / 8
      for (int bf = tid; bf < N / 8; bf += T) {
        const int j = bf & (S - 1);
        const int base = ((bf >> (LOGL - 3)) << LOGL) + j;
        // padded positions of the butterfly's 8 elements: a constant stride when S >= 16
        const int p0 = P(base);
        auto Q = [&](int m) {
          if (SWZ) return S >= 128 ? p0 + m * S : P(base + m * S);  // the swizzle reads index bits 4..6
          return S >= 16 ? p0 + m * (S + (S >> 4)) : P(base + m * S);
        };
        float2 x[8];
#pragma unroll
        for (int m = 0; m < 8; ++m) x[m] = (s == 0) ? load_in(base + m * S) : sm[Q(m)];
        dft_small<8, false>(x);
        const float2 w1 = __ldg(tw + ((size_t)j << (LOGN - LOGL)));
        const float2 w2 = cmul(w1, w1), w3 = cmul(w2, w1), w4 = cmul(w2, w2);
        const float2 w5 = cmul(w4, w1), w6 = cmul(w3, w3), w7 = cmul(w4, w3);
        sm[Q(0)] = x[0];
        sm[Q(1)] = cmul(x[1], w1);
        sm[Q(2)] = cmul(x[2], w2);
        sm[Q(3)] = cmul(x[3], w3);
        sm[Q(4)] = cmul(x[4], w4);
        sm[Q(5)] = cmul(x[5], w5);
        sm[Q(6)] = cmul(x[6], w6);
        sm[Q(7)] = cmul(x[7], w7);
      }
      __syncthreads();
    }
    // innermost pass both ways around the spectrum multiply, in registers
    for (int g = tid; g < N / RM; g += T) {
      float2 x[RM];
#pragma unroll
      for (int m = 0; m < RM; ++m) x[m] = sm[P(g * RM + m)];
      dft_small<RM, false>(x);
#pragma unroll
      for (int m = 0; m < RM; ++m) {
        const float hq = __ldg(Hp + g * RM + m);
        x[m].x *= hq;
        x[m].y *= hq;
      }
      dft_small<RM, true>(x);
#pragma unroll
      for (int m = 0; m < RM; ++m) sm[P(g * RM + m)] = x[m];
    }
    __syncthreads();
    // inverse: the forward passes backwards (decimation in time), conjugate twiddles; the last
    // one writes the rows straight to global memory
#pragma unroll
    for (int s = A - 1; s >= 0; --s) {
      const int LOGL = LOGN - 3 * s;
      const int S = 1 << (LOGL - 3);
      for (int bf = tid; bf < N / 8; bf += T) {
        const int j = bf & (S - 1);
        const int base = ((bf >> (LOGL - 3)) << LOGL) + j;
        const float2 w1 = __ldg(tw + ((size_t)j << (LOGN - LOGL)));
        const float2 w2 = cmul(w1, w1), w3 = cmul(w2, w1), w4 = cmul(w2, w2);
        const float2 w5 = cmul(w4, w1), w6 = cmul(w3, w3), w7 = cmul(w4, w3);
        const int p0 = P(base);
        auto Q = [&](int m) {
          if (SWZ) return S >= 128 ? p0 + m * S : P(base + m * S);  // the swizzle reads index bits 4..6
          return S >= 16 ? p0 + m * (S + (S >> 4)) : P(base + m * S);
        };
        float2 x[8];
        x[0] = sm[Q(0)];
        x[1] = cmulc(sm[Q(1)], w1);
        x[2] = cmulc(sm[Q(2)], w2);
        x[3] = cmulc(sm[Q(3)], w3);
        x[4] = cmulc(sm[Q(4)], w4);
        x[5] = cmulc(sm[Q(5)], w5);
        x[6] = cmulc(sm[Q(6)], w6);
        x[7] = cmulc(sm[Q(7)], w7);
        dft_small<8, true>(x);
#pragma unroll
        for (int m = 0; m < 8; ++m) {
          if (s == 0) store_out(base + m * S, x[m]);
          else sm[Q(m)] = x[m];
        }
      }
      if (s != 0) __syncthreads();
    }
    if (A == 0) {
      for (int n = tid; n < pitch; n += T) store_out(n, n < N ? sm[P(n)] : make_float2(0.0f, 0.0f));
    }
    __syncthreads();  // the next pair overwrites the buffer
  }
}

}  // namespace cbp
