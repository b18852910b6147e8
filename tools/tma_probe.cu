// Minimal TMA probe: one 3D tiled load of a (hb x wb) box into shared memory.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cstdlib>
#include "../paper_2104_13248_b200/csrc/bp_kernels.cuh"
using namespace cbp;

template <bool PREFETCH>
__global__ void probe(const __grid_constant__ CUtensorMap tmap, float* out, int wb, int hb, int c0, int c1, int c2) {
  extern __shared__ __align__(1024) unsigned char sm[];
  float* box = reinterpret_cast<float*>(sm);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + ((wb * hb * 4 + 127) & ~127));
  if (threadIdx.x == 0) { mbar_init(bar, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (PREFETCH) prefetch_tmap(&tmap);
    mbar_arrive_tx(bar, wb * hb * 4);
    tma_load_3d(box, &tmap, bar, c0, c1, c2);
  }
  mbar_wait(bar, 0);
  for (int i = threadIdx.x; i < wb * hb; i += blockDim.x) out[i] = box[i];
}

int main() {
  typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  void* p = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  Enc enc = (Enc)p;
  const int np = 8, nw = 24, pitch = 24, rows = 24, wb = 12, hb = 24;
  std::vector<float> h(np * nw * pitch);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (float)i;
  float *d, *o;
  cudaMalloc(&d, h.size() * 4); cudaMalloc(&o, wb * hb * 4);
  cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  CUtensorMap m;
  cuuint64_t gdim[3] = {(cuuint64_t)rows, (cuuint64_t)nw, (cuuint64_t)np};
  cuuint64_t gstr[2] = {(cuuint64_t)pitch * 4, (cuuint64_t)pitch * nw * 4};
  cuuint32_t box[3] = {(cuuint32_t)hb, (cuuint32_t)wb, 1}, es[3] = {1, 1, 1};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  int cs[][3] = {{0, 3, 2}, {1, 0, 0}, {4, 0, 0}, {0, 1, 0}, {2, 5, 2}, {3, 5, 2}, {-2, 0, 0}, {0, -3, 0}, {20, 0, 0}, {0, 20, 1}};
  int variant = 0;
  if (getenv("CI")) variant = atoi(getenv("CI"));
  {
    size_t smem = ((wb * hb * 4 + 127) & ~127) + 64;
    int c0 = cs[variant][0], c1 = cs[variant][1], c2 = cs[variant][2];
    probe<true><<<1, 128, smem>>>(m, o, wb, hb, c0, c1, c2);
    cudaError_t e = cudaDeviceSynchronize();
    printf("coords (%d,%d,%d): %s\n", c0, c1, c2, cudaGetErrorString(e));
    if (e != cudaSuccess) return 1;
    std::vector<float> ho(wb * hb);
    cudaMemcpy(ho.data(), o, ho.size() * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int u = 0; u < wb; ++u) for (int v = 0; v < hb; ++v) {
      int uu = c1 + u, vv = c0 + v;
      float want = (uu >= 0 && uu < nw && vv >= 0 && vv < rows) ? h[((size_t)c2 * nw + uu) * pitch + vv] : 0.f;
      if (ho[u * hb + v] != want) ++bad;
    }
    printf("  mismatches %d\n", bad);
  }
  return 0;
}
