// fdk.cuh -- FDK pre-processing on the GPU: cosine weighting and
// row-wise Ram-Lak filtering of raw projections, written straight into the staging
// layout the back-projector reads (staged[s][v][u], 16-byte row pitch).
//
// The reference has no filter step; the definition implemented here is the
// one of paper_2104_13248_b200/phantom.py (cosine_weight + ramp_filter):
//   x[v][u]   = raw[v][u] * D / sqrt(D^2 + ((u-cu) pu)^2 + ((v-cv) pv)^2)
//   out[v][u] = tau * sum_{u'} h[u-u'] x[v][u'],  h[0] = 1/(4 tau^2),
//               h[n odd] = -1/(pi^2 n^2 tau^2), h[n even != 0] = 0   (linear, zero padded)
// evaluated as a zero-padded FFT convolution: weight+pad kernel -> cuFFT R2C ->
// multiply by the exact DFT of h -> cuFFT C2R -> crop into the staging layout.
#pragma once
#include <cuda_runtime.h>
#include <cufft.h>
#include <stdint.h>

namespace cbp {

// buf[row][n] = raw[row][n] * cosine weight for n < nw, 0 for nw <= n < nfft
// (the weight is evaluated in float64 and rounded once, as phantom.cosine_weight does)
__global__ void fdk_weight_pad_kernel(const float* __restrict__ raw, int nh, int nw, int nfft, long long rows,
                                      long long row0, double D, double pu, double pv, double cu, double cv,
                                      float* __restrict__ buf) {
  const long long row = (long long)blockIdx.y * gridDim.z + blockIdx.z;
  if (row >= rows) return;
  const int v = (int)((row0 + row) % nh);  // rows are (projection, detector row) pairs
  const double vv = __dmul_rn(__dsub_rn((double)v, cv), pv);
  const float* src = raw + row * nw;
  float* dst = buf + row * nfft;
  for (int n = blockIdx.x * blockDim.x + threadIdx.x; n < nfft; n += gridDim.x * blockDim.x) {
    float val = 0.0f;
    if (n < nw) {
      const double uu = __dmul_rn(__dsub_rn((double)n, cu), pu);
      const double r2 = __dadd_rn(__dadd_rn(__dmul_rn(D, D), __dmul_rn(uu, uu)), __dmul_rn(vv, vv));
      val = __fmul_rn(__ldg(src + n), (float)__ddiv_rn(D, __dsqrt_rn(r2)));
    }
    dst[n] = val;
  }
}

// spec[row][k] *= H[k] (real: h is even), H already carries tau / nfft
__global__ void fdk_spectrum_kernel(cufftComplex* __restrict__ spec, const float* __restrict__ H, int nspec,
                                    long long rows) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows * nspec) return;
  const float g = __ldg(H + (int)(i % nspec));
  cufftComplex c = spec[i];
  c.x *= g;
  c.y *= g;
  spec[i] = c;
}

// out[s][v][u] (staging layout, pitch) = buf[row][u]
__global__ void fdk_crop_kernel(const float* __restrict__ buf, int nfft, int nw, int pitch, long long rows,
                                float* __restrict__ out) {
  const long long row = (long long)blockIdx.y * gridDim.z + blockIdx.z;
  if (row >= rows) return;
  const float* src = buf + row * nfft;
  float* dst = out + row * pitch;
  for (int u = blockIdx.x * blockDim.x + threadIdx.x; u < pitch; u += gridDim.x * blockDim.x)
    dst[u] = (u < nw) ? src[u] : 0.0f;
}

}  // namespace cbp
