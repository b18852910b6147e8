// fwd_kernels.cuh -- the adjoint of the hot path: ray-driven
// forward projection of a NATURAL float32 volume, the arithmetic of
// /root/reference/pkg/src/conebp/phantom.py:134-222 (_forward) reproduced bit for bit.
//
// The reference evaluates in float64 with IEEE-exact operations (numba/LLVM, no
// fastmath): every add, multiply, divide and sqrt below is the explicitly rounded
// double intrinsic in the same order, so each ray sum is identical before its final
// rounding to float32 (phantom.py:221).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace cbp {

__device__ __forceinline__ double dm(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double da(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double ds(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dd(double a, double b) { return __ddiv_rn(a, b); }

struct FwdParams {
  const float* vol;      // [nz][ny][nx]
  const float* vol_t;    // the same volume as [nz][nx][ny] (y contiguous), or null
  const double* views;   // [np][12]: source xyz, detector-centre xyz, e_u xyz, e_v xyz
  float* out;            // [np][nh][nw]
  int np, nh, nw, nx, ny, nz;
  double pu, pv, cu, cv, s;
};

// One ray per thread (phantom.py:145-221).
// The lanes of a warp are neighbouring detector columns: their sample points lie on a line
// across the ray in the xy-plane.  For rays that run mostly along y that line runs along x and
// a warp-wide gather touches a few 32-byte sectors of one volume row; for rays mostly along x
// it touched a different row per lane (ncu: the L1 data pipe 99% busy, 14 wavefronts per
// gather on average).  Those rays read a copy of the volume with y contiguous instead
// (p.vol_t): the same eight voxels, the same arithmetic, a third of the wavefronts.
// POW2: the voxel size is a power of two (1.0 in every BASELINE config), so the three float64
// divisions by it per ray step are multiplications by its exact reciprocal -- the same
// correctly rounded quotient, a third of the float64 work per step.
template <bool POW2>
__global__ void __launch_bounds__(256) bp_forward_kernel(const FwdParams p) {
  const long long total = (long long)p.np * p.nh * p.nw;
  const long long flat = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (flat >= total) return;
  const long long plane = (long long)p.nh * p.nw;
  const int pj = (int)(flat / plane);
  const long long rem = flat % plane;
  const int iv = (int)(rem / p.nw), iu = (int)(rem % p.nw);
  const double* V = p.views + 12 * pj;
  const double sx = V[0], sy = V[1], sz = V[2];
  const double hx = dm(dd((double)(p.nx - 1), 2.0), p.s);
  const double hy = dm(dd((double)(p.ny - 1), 2.0), p.s);
  const double hz = dm(dd((double)(p.nz - 1), 2.0), p.s);
  const double ox = dd((double)(p.nx - 1), 2.0), oy = dd((double)(p.ny - 1), 2.0), oz = dd((double)(p.nz - 1), 2.0);
  const double step = dm(0.5, p.s);
  const double du = dm(ds((double)iu, p.cu), p.pu);
  const double dv = dm(ds((double)iv, p.cv), p.pv);
  const double px = da(da(V[3], dm(du, V[6])), dm(dv, V[9]));
  const double py = da(da(V[4], dm(du, V[7])), dm(dv, V[10]));
  const double pz = da(da(V[5], dm(du, V[8])), dm(dv, V[11]));
  double dx = ds(px, sx), dy = ds(py, sy), dz = ds(pz, sz);
  const double norm = __dsqrt_rn(da(da(dm(dx, dx), dm(dy, dy)), dm(dz, dz)));
  dx = dd(dx, norm);
  dy = dd(dy, norm);
  dz = dd(dz, norm);
  double t0 = 0.0, t1 = norm;
  float* o = p.out + flat;
  // which copy of the volume this ray reads, and its element strides in x and y
  const bool tr = p.vol_t != nullptr && fabs(dx) > fabs(dy);
  const float* __restrict__ vbase = tr ? p.vol_t : p.vol;
  const long long sx_ = tr ? p.ny : 1, sy_ = tr ? 1 : p.nx, sz_ = (long long)p.nx * p.ny;
  // slab intersection with the voxel-centre box (phantom.py:164-192)
  if (dx != 0.0) {
    const double ta = dd(ds(-hx, sx), dx), tb = dd(ds(hx, sx), dx);
    t0 = fmax(t0, fmin(ta, tb));
    t1 = fmin(t1, fmax(ta, tb));
  } else if (sx < -hx || sx > hx) {
    *o = 0.0f;
    return;
  }
  if (dy != 0.0) {
    const double ta = dd(ds(-hy, sy), dy), tb = dd(ds(hy, sy), dy);
    t0 = fmax(t0, fmin(ta, tb));
    t1 = fmin(t1, fmax(ta, tb));
  } else if (sy < -hy || sy > hy) {
    *o = 0.0f;
    return;
  }
  if (dz != 0.0) {
    const double ta = dd(ds(-hz, sz), dz), tb = dd(ds(hz, sz), dz);
    t0 = fmax(t0, fmin(ta, tb));
    t1 = fmin(t1, fmax(ta, tb));
  } else if (sz < -hz || sz > hz) {
    *o = 0.0f;
    return;
  }
  if (t1 <= t0) {
    *o = 0.0f;
    return;
  }
  double total_sum = 0.0;
  const long long n_steps = (long long)ceil(dd(ds(t1, t0), step));
  const double lx = (double)(p.nx - 1), ly = (double)(p.ny - 1), lz = (double)(p.nz - 1);
  const double inv_s = dd(1.0, p.s);  // exact when POW2
  for (long long q = 0; q < n_steps; ++q) {
    const double t = da(t0, dm(da((double)q, 0.5), step));
    if (t >= t1) break;
    const double nxs = da(sx, dm(t, dx)), nys = da(sy, dm(t, dy)), nzs = da(sz, dm(t, dz));
    const double fx = da(POW2 ? dm(nxs, inv_s) : dd(nxs, p.s), ox);
    const double fy = da(POW2 ? dm(nys, inv_s) : dd(nys, p.s), oy);
    const double fz = da(POW2 ? dm(nzs, inv_s) : dd(nzs, p.s), oz);
    if (fx < 0.0 || fx > lx || fy < 0.0 || fy > ly || fz < 0.0 || fz > lz) continue;
    int ix = (int)fx, iy = (int)fy, iz = (int)fz;
    if (ix > p.nx - 2) ix = p.nx - 2;
    if (iy > p.ny - 2) iy = p.ny - 2;
    if (iz > p.nz - 2) iz = p.nz - 2;
    const double ax = ds(fx, (double)ix), ay = ds(fy, (double)iy), az = ds(fz, (double)iz);
    const float* v00 = vbase + iz * sz_ + iy * sy_ + ix * sx_;  // voxel (ix, iy, iz)
    const float* v10 = v00 + sy_;                                // (ix, iy + 1, iz)
    const float* v01 = v00 + sz_;                                // (ix, iy, iz + 1)
    const float* v11 = v01 + sy_;                                // (ix, iy + 1, iz + 1)
    const double oax = ds(1.0, ax), oay = ds(1.0, ay), oaz = ds(1.0, az);
    const double c00 = da(dm((double)__ldg(v00), oax), dm((double)__ldg(v00 + sx_), ax));
    const double c10 = da(dm((double)__ldg(v10), oax), dm((double)__ldg(v10 + sx_), ax));
    const double c01 = da(dm((double)__ldg(v01), oax), dm((double)__ldg(v01 + sx_), ax));
    const double c11 = da(dm((double)__ldg(v11), oax), dm((double)__ldg(v11 + sx_), ax));
    const double lo = da(dm(c00, oay), dm(c10, ay));
    const double hi = da(dm(c01, oay), dm(c11, ay));
    total_sum = da(total_sum, dm(da(dm(lo, oaz), dm(hi, az)), step));
  }
  *o = (float)total_sum;
}

}  // namespace cbp
