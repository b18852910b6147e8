// capi.cu -- host side of libconebp_b200.so: the C ABI declared in
// include/conebp_b200.h, launch planning (tile shape, TMA box, ring depth),
// tensor-map encoding, op counting and the z-slab planner.
//
// The reference seams replaced here are listed in the header.  Nothing in this
// file computes back-projection values on the host: every value comes from the
// sm_100a kernels in bp_kernels.cuh.
#include "../../include/conebp_b200.h"
#include "bp_kernels.cuh"
#include "fwd_kernels.cuh"
#include "fdk.cuh"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

using namespace cbp;

namespace {

thread_local std::string g_err;
thread_local int64_t g_last_plan[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}
int cuda_fail(cudaError_t e, const char* what) {
  std::string m = std::string(what) + ": " + cudaGetErrorString(e);
  return fail(e == cudaErrorMemoryAllocation ? CBP_ENOMEM : CBP_ECUDA, m);
}
#define CK(call, what)                       \
  do {                                       \
    cudaError_t e_ = (call);                 \
    if (e_ != cudaSuccess) return cuda_fail(e_, what); \
  } while (0)

// ---------------------------------------------------------------- tensor maps
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

// ---------------------------------------------------------------- helpers
// 64-bit FNV-1a over 8-byte words (the matrices are hashed on every launch: a word at a
// time is 8x cheaper than bytes; cfg4's 96 KiB of matrices hash in ~10 us)
uint64_t hash_words(const void* data, size_t n) {
  uint64_t h = 1469598103934665603ull;
  const unsigned char* b = static_cast<const unsigned char*>(data);
  size_t i = 0;
  for (; i + 8 <= n; i += 8) {
    uint64_t w;
    std::memcpy(&w, b + i, 8);
    h = (h ^ w) * 1099511628211ull;
    h ^= h >> 29;
  }
  for (; i < n; ++i) h = (h ^ b[i]) * 1099511628211ull;
  return h ^ (uint64_t)n;
}

bool mats_finite(const float* m, int64_t n) {
  for (int64_t q = 0; q < n; ++q)
    if (!std::isfinite(m[q])) return false;
  return true;
}

// fast path valid for the non-hoisting rungs when every u and depth row has a
// zero k coefficient (geometry.py:204,206); hoisting rungs always use it.
bool fast_path_ok(const float* mats, int64_t np, int variant) {
  if (v_hoist(variant)) return true;
  for (int64_t s = 0; s < np; ++s)
    if (mats[12 * s + 2] != 0.0f || mats[12 * s + 10] != 0.0f) return false;
  return true;
}

// A device allocation shared by cached plans and the launches that read it.  It is freed
// when the last reference goes (a plan evicted while another thread is still launching
// with it keeps it alive); before the free the owning device is drained, since launches
// queued on any stream may still read it.
struct DevBuf {
  void* p = nullptr;
  int dev = -1;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() {
    if (!p) return;
    int cur = -1;
    if (cudaGetDevice(&cur) == cudaSuccess && cudaSetDevice(dev) == cudaSuccess) {
      cudaDeviceSynchronize();
      cudaFree(p);
      cudaSetDevice(cur);
    }
    cudaGetLastError();
  }
};

struct Plan {
  int cfg = 0, TX = 32, TY = 16, NW = 16, wb = 0, hb = 0, stages = 0;
  int kind = 1;  // 0 naive, 1 tiled fast, 2 tiled general
  size_t smem = 0;
  std::shared_ptr<DevBuf> mats;  // np x 12 float32 on the plan's device
  const float* mats_dev() const { return static_cast<const float*>(mats->p); }
  int device = -1;
  uint64_t last_use = 0;
};

struct PlanKey {
  int device, variant, kind_req, pad0;
  int64_t np, nh, nw, band_v0, band_rows, nx, ny, nz, k0, nz_total;
  uint64_t mhash;
  bool operator<(const PlanKey& o) const {
    return std::memcmp(this, &o, sizeof(PlanKey)) < 0;
  }
};

std::mutex g_mu;  // guards g_plans, g_stats, g_smem_set, g_use_clock
std::map<PlanKey, Plan> g_plans;
std::map<std::pair<int, uintptr_t>, unsigned long long*> g_stats;  // status counters [8] per (device, stream)
std::map<std::pair<int, const void*>, size_t> g_smem_set;          // dynamic smem attribute set per kernel
uint64_t g_use_clock = 0;
constexpr int kPlansPerDevice = 16;

// status counters of (device, stream): every launch on a stream accumulates into its
// own buffer, so cbp_sync_status on one stream never reads or clears another's
int get_stats(int dev, cudaStream_t st, unsigned long long** out) {
  std::lock_guard<std::mutex> lk(g_mu);
  const auto key = std::make_pair(dev, reinterpret_cast<uintptr_t>(st));
  auto it = g_stats.find(key);
  if (it != g_stats.end()) {
    *out = it->second;
    return CBP_OK;
  }
  unsigned long long* p = nullptr;
  CK(cudaMalloc(&p, 8 * sizeof(unsigned long long)), "cudaMalloc(stats)");
  CK(cudaMemset(p, 0, 8 * sizeof(unsigned long long)), "cudaMemset(stats)");
  g_stats[key] = p;
  *out = p;
  return CBP_OK;
}

// Tile configurations {consumer warps in x, in y, CTAs per SM}: a warp is 8 x 4
// columns, a thread owns one column's 32-slice z-run.
struct TileCfg {
  int NWX, NWY, MINB;
};
// Measured and not kept (round 2): 15-consumer-warp tiles {3,5,1} / {5,3,1} (16 warps per CTA, so
// 128 registers per thread instead of 96): -4.6% / -5.8% on cfg4, -3% / -6% on cfg1.
constexpr int kNumTiles = 7;
constexpr TileCfg kTiles[kNumTiles] = {{4, 4, 1}, {2, 4, 2}, {2, 2, 3}, {4, 3, 1}, {2, 3, 2}, {3, 6, 1}, {2, 2, 4}};

template <int C>
using RolesC = WarpRoles<kTiles[C].NWX * kTiles[C].NWY, kTiles[C].MINB>;
constexpr int kTileThreads[kNumTiles] = {RolesC<0>::kThreads, RolesC<1>::kThreads, RolesC<2>::kThreads,
                                         RolesC<3>::kThreads, RolesC<4>::kThreads, RolesC<5>::kThreads,
                                         RolesC<6>::kThreads};
// launch register allocation the setmaxnreg split assumes (0: no register reallocation)
constexpr int kTilePool[kNumTiles] = {
    RolesC<0>::kRealloc ? RolesC<0>::kRegLaunch : 0, RolesC<1>::kRealloc ? RolesC<1>::kRegLaunch : 0,
    RolesC<2>::kRealloc ? RolesC<2>::kRegLaunch : 0, RolesC<3>::kRealloc ? RolesC<3>::kRegLaunch : 0,
    RolesC<4>::kRealloc ? RolesC<4>::kRegLaunch : 0, RolesC<5>::kRealloc ? RolesC<5>::kRegLaunch : 0,
    RolesC<6>::kRealloc ? RolesC<6>::kRegLaunch : 0};

template <int V, bool GEN, int C, bool CHECK>
const void* tiled_fn() {
  return reinterpret_cast<const void*>(
      &bp_tiled_kernel<V, GEN, kTiles[C].NWX, kTiles[C].NWY, kTiles[C].MINB, CHECK>);
}

#if !CBP_DEV_SLIM
template <int V, bool GEN, bool CHECK>
const void* tiled_by_tile(int c) {
  switch (c) {
    case 0: return tiled_fn<V, GEN, 0, CHECK>();
    case 1: return tiled_fn<V, GEN, 1, CHECK>();
    case 3: return tiled_fn<V, GEN, 3, CHECK>();
    case 4: return tiled_fn<V, GEN, 4, CHECK>();
    case 5: return tiled_fn<V, GEN, 5, CHECK>();
    case 6: return tiled_fn<V, GEN, 6, CHECK>();
    default: return tiled_fn<V, GEN, 2, CHECK>();
  }
}

template <bool CHECK>
const void* tiled_kernel_ptr_c(int variant, bool gen, int c) {
  switch (variant) {
    case V_BASELINE: return gen ? tiled_by_tile<V_BASELINE, true, CHECK>(c) : tiled_by_tile<V_BASELINE, false, CHECK>(c);
    case V_TRANSPOSE:
      return gen ? tiled_by_tile<V_TRANSPOSE, true, CHECK>(c) : tiled_by_tile<V_TRANSPOSE, false, CHECK>(c);
    case V_SHARE: return tiled_by_tile<V_SHARE, false, CHECK>(c);
    case V_SYMMETRY: return tiled_by_tile<V_SYMMETRY, false, CHECK>(c);
    default: return tiled_by_tile<V_SUBLINE, false, CHECK>(c);  // sub-line rungs: identical arithmetic
  }
}

#endif
const void* tiled_kernel_ptr(int variant, bool gen, int c, bool check) {
#if CBP_DEV_SLIM  // kernel-tuning builds: only the baseline fast-path instances of tile shapes 0 and 1 (seconds to compile)
  (void)variant; (void)check;
  if (gen) return tiled_fn<V_BASELINE, true, 1, false>();
  return c == 1   ? tiled_fn<V_BASELINE, false, 1, false>()
         : c == 3 ? tiled_fn<V_BASELINE, false, 3, false>()
                  : tiled_fn<V_BASELINE, false, 0, false>();
#else
  return check ? tiled_kernel_ptr_c<true>(variant, gen, c) : tiled_kernel_ptr_c<false>(variant, gen, c);
#endif
}
#if !CBP_DEV_SLIM

// half z-run tiles (16 slices), bit-exact, every variant
template <int V, bool GEN, int C>
const void* half_fn() {
  return reinterpret_cast<const void*>(&bp_tiled_half_kernel<V, GEN, kTiles[C].NWX, kTiles[C].NWY, kTiles[C].MINB>);
}
template <int V, bool GEN>
const void* half_by_tile(int c) {
  switch (c) {
    case 0: return half_fn<V, GEN, 0>();
    case 1: return half_fn<V, GEN, 1>();
    case 3: return half_fn<V, GEN, 3>();
    case 4: return half_fn<V, GEN, 4>();
    case 5: return half_fn<V, GEN, 5>();
    case 6: return half_fn<V, GEN, 6>();
    default: return half_fn<V, GEN, 2>();
  }
}
#endif
const void* half_kernel_ptr(int variant, bool gen, int c) {
#if CBP_DEV_SLIM
  return tiled_kernel_ptr(variant, gen, c, false);
#else
  switch (variant) {
    case V_BASELINE: return gen ? half_by_tile<V_BASELINE, true>(c) : half_by_tile<V_BASELINE, false>(c);
    case V_TRANSPOSE: return gen ? half_by_tile<V_TRANSPOSE, true>(c) : half_by_tile<V_TRANSPOSE, false>(c);
    case V_SHARE: return half_by_tile<V_SHARE, false>(c);
    case V_SYMMETRY: return half_by_tile<V_SYMMETRY, false>(c);
    default: return half_by_tile<V_SUBLINE, false>(c);
  }
#endif
}

#if !CBP_DEV_SLIM
// tolerance mode (CBP_FLAG_FMA_LERP): baseline arithmetic with FMA lerps
template <bool GEN, int C>
const void* fmalerp_fn() {
  return reinterpret_cast<const void*>(
      &bp_tiled_fmalerp_kernel<V_BASELINE, GEN, kTiles[C].NWX, kTiles[C].NWY, kTiles[C].MINB>);
}
template <bool GEN>
const void* fmalerp_by_tile(int c) {
  switch (c) {
    case 0: return fmalerp_fn<GEN, 0>();
    case 1: return fmalerp_fn<GEN, 1>();
    case 3: return fmalerp_fn<GEN, 3>();
    case 4: return fmalerp_fn<GEN, 4>();
    case 5: return fmalerp_fn<GEN, 5>();
    case 6: return fmalerp_fn<GEN, 6>();
    default: return fmalerp_fn<GEN, 2>();
  }
}

#endif
const void* naive_kernel_ptr(int variant) {
  switch (variant) {
    case V_BASELINE: return reinterpret_cast<const void*>(&bp_naive_kernel<V_BASELINE>);
    case V_TRANSPOSE: return reinterpret_cast<const void*>(&bp_naive_kernel<V_TRANSPOSE>);
    case V_SHARE: return reinterpret_cast<const void*>(&bp_naive_kernel<V_SHARE>);
    case V_SYMMETRY: return reinterpret_cast<const void*>(&bp_naive_kernel<V_SYMMETRY>);
    default: return reinterpret_cast<const void*>(&bp_naive_kernel<V_SUBLINE>);
  }
}

template <int V>
void launch_footprint(dim3 g, dim3 b, cudaStream_t st, const float* mats, int np, int nw, int nh, int nx, int ny,
                      int nz, int k0, int nzt, int TX, int TY, int tx, int ty, int tz, int astride, unsigned* hw,
                      unsigned* hh, int nbins, int band_v0) {
  bp_footprint_kernel<V><<<g, b, 0, st>>>(mats, np, nw, nh, nx, ny, nz, k0, nzt, band_v0, TX, TY, tx, ty, tz, astride,
                                          hw, hh, nbins);
}

int run_footprint(int variant, dim3 g, dim3 b, cudaStream_t st, const float* mats, int np, int nw, int nh, int nx,
                  int ny, int nz, int k0, int nzt, int TX, int TY, int tx, int ty, int tz, int astride, unsigned* hw,
                  unsigned* hh, int nbins, int band_v0) {
  switch (variant) {
    case V_BASELINE: launch_footprint<V_BASELINE>(g, b, st, mats, np, nw, nh, nx, ny, nz, k0, nzt, TX, TY, tx, ty, tz, astride, hw, hh, nbins, band_v0); break;
    case V_TRANSPOSE: launch_footprint<V_TRANSPOSE>(g, b, st, mats, np, nw, nh, nx, ny, nz, k0, nzt, TX, TY, tx, ty, tz, astride, hw, hh, nbins, band_v0); break;
    case V_SHARE: launch_footprint<V_SHARE>(g, b, st, mats, np, nw, nh, nx, ny, nz, k0, nzt, TX, TY, tx, ty, tz, astride, hw, hh, nbins, band_v0); break;
    case V_SYMMETRY: launch_footprint<V_SYMMETRY>(g, b, st, mats, np, nw, nh, nx, ny, nz, k0, nzt, TX, TY, tx, ty, tz, astride, hw, hh, nbins, band_v0); break;
    default: launch_footprint<V_SUBLINE>(g, b, st, mats, np, nw, nh, nx, ny, nz, k0, nzt, TX, TY, tx, ty, tz, astride, hw, hh, nbins, band_v0); break;
  }
  return cudaGetLastError() == cudaSuccess ? CBP_OK : fail(CBP_ECUDA, "footprint kernel launch failed");
}

int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Choose tile shape, TMA box and ring depth for a problem; uploads the matrices.
int make_plan(const PlanKey& key, const float* mats_host, cudaStream_t stream, Plan& plan, int forced_cfg = -1) {
  plan = Plan();
  plan.device = key.device;
  const int64_t n12 = key.np * 12;
  plan.mats = std::make_shared<DevBuf>();
  plan.mats->dev = key.device;
  CK(cudaMalloc(&plan.mats->p, n12 * sizeof(float)), "cudaMalloc(mats)");
  // synchronous: mats_host is only borrowed for the duration of the call
  CK(cudaMemcpy(plan.mats->p, mats_host, n12 * sizeof(float), cudaMemcpyHostToDevice), "upload mats");
  if (key.kind_req == 0) {
    plan.kind = 0;
    return CBP_OK;
  }
  const bool gen = !fast_path_ok(mats_host, key.np, key.variant);
  plan.kind = gen ? 2 : 1;

  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, key.device);
  int smem_optin = 227 * 1024;
  cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, key.device);

  // tile: the largest column tile that still gives >= 3 waves of CTAs; short of that, two
  // CTAs of 8 warps per SM as long as they cover every SM (thin multi-GPU slabs: one wave of
  // full SMs beats a second, mostly idle wave of the small tile -- cfg1 at 8 ranks); tiny
  // problems, whose time is per-angle latency, keep the smallest tile
  int pick = 2;
  int64_t tiles_c[3];
  for (int c = 0; c < 3; ++c)
    tiles_c[c] = ceil_div(key.nx, 8 * kTiles[c].NWX) * ceil_div(key.ny, 4 * kTiles[c].NWY) * ceil_div(key.nz, kZR);
  for (int c = 0; c < 3; ++c) {
    if (tiles_c[c] >= 3LL * sms * kTiles[c].MINB) {
      pick = c;
      break;
    }
  }
  if (pick == 2 && tiles_c[1] >= sms) pick = 1;
  bool may_split = pick == 0;  // candidate for two CTAs of 8 warps per SM (cfg 1), see below
  if (const char* env = std::getenv("CBP_TILE_CFG")) {  // tuning override
    const int forced = std::atoi(env);
    if (forced >= 0 && forced < kNumTiles) pick = forced;
    may_split = false;
  }
  if (forced_cfg >= 0) {
    pick = forced_cfg;
    may_split = false;
  }
  plan.cfg = pick;
  plan.TX = 8 * kTiles[pick].NWX;
  plan.TY = 4 * kTiles[pick].NWY;
  plan.NW = kTiles[pick].NWX * kTiles[pick].NWY;
  const int tx = (int)ceil_div(key.nx, plan.TX), ty = (int)ceil_div(key.ny, plan.TY), tz = (int)ceil_div(key.nz, kZR);

  // footprint histograms over (tile, angle) pairs (angles subsampled on huge problems)
  const int nbins = 1024;
  unsigned* hist = nullptr;
  CK(cudaMallocAsync(reinterpret_cast<void**>(&hist), 2 * nbins * sizeof(unsigned), stream), "alloc hist");
  CK(cudaMemsetAsync(hist, 0, 2 * nbins * sizeof(unsigned), stream), "memset hist");
  const int64_t n_tiles = (int64_t)tx * ty * tz;
  int astride = 1;
  while (n_tiles * ceil_div(key.np, astride) > 40000000LL) astride *= 2;
  const int64_t pairs = n_tiles * ceil_div(key.np, astride);
  const int wpb = 8;
  dim3 g((unsigned)ceil_div(pairs, wpb)), b(32 * wpb);
  int rc = run_footprint(key.variant, g, b, stream, plan.mats_dev(), (int)key.np, (int)key.nw, (int)key.nh, (int)key.nx,
                         (int)key.ny, (int)key.nz, (int)key.k0, (int)key.nz_total, plan.TX, plan.TY, tx, ty, tz,
                         astride, hist, hist + nbins, nbins, (int)key.band_v0);
  if (rc) return rc;
  std::vector<unsigned> h(2 * nbins);
  CK(cudaMemcpyAsync(h.data(), hist, 2 * nbins * sizeof(unsigned), cudaMemcpyDeviceToHost, stream), "read hist");
  CK(cudaFreeAsync(hist, stream), "free hist");
  CK(cudaStreamSynchronize(stream), "plan sync");

  // One CTA of 16 consumer warps per SM (cfg 0) or two CTAs of 8 (cfg 1, 16x16 columns)?
  // Two CTAs hide each other's ring stalls and CTA turnover (cfg1 +4%, cfg2 +2%), but
  // double the producer work per voxel, which costs when many (tile, angle) pairs miss
  // the detector (cfg3 30% / cfg4 67% missed: -6% / -9%).  Measured on B200, round 1.
  if (may_split) {
    uint64_t sampled = 0;
    for (int i = 0; i < nbins; ++i) sampled += h[i];
    const double missed = 1.0 - (double)sampled / (double)std::max<int64_t>(1, pairs);
    if (missed < 0.25) return make_plan(key, mats_host, stream, plan, 1);
  }

  auto quantile = [&](const unsigned* hh, double q) {
    uint64_t tot = 0;
    for (int i = 0; i < nbins; ++i) tot += hh[i];
    if (tot == 0) return 4;
    uint64_t acc = 0;
    for (int i = 0; i < nbins; ++i) {
      acc += hh[i];
      if ((double)acc >= q * (double)tot) return std::max(i, 2);
    }
    return nbins - 1;
  };
  // box rows are the smem row pitch: a multiple of 32 words keeps one detector row's
  // texels in distinct banks (and the TMA inner extent a multiple of 16 bytes)
  // row pitch = 16 (mod 32) words: lanes on one pixel column but adjacent rows (columns
  // along the ray) land 16 banks apart instead of on the same bank
  int pad = 16;
  if (const char* e = std::getenv("CBP_BOX_PAD")) pad = std::atoi(e) & 28;
  int wb = quantile(h.data(), 0.999);
#if CBP_ROWSHIFT
  (void)pad;
  { int w2 = 32; while (w2 < wb) w2 <<= 1; wb = std::min(w2, 256); }
#else
  wb = ((wb - pad + 31) & ~31) + pad;
  if (wb > 240) wb = 240;
#endif
  int hb = std::min(std::max(quantile(h.data() + nbins, 0.999), 2), 256);

  const size_t hdr_bytes = kMaxStages * sizeof(StageHdr) + 3 * kMaxStages * sizeof(uint64_t);  // full, empty, tbar
  auto stage_bytes = [&](int w, int hh) { return (size_t)(((size_t)w * hh * 4 + 127) & ~(size_t)127); };
  // ring depth within the per-CTA share of shared memory (MINB CTAs per SM)
  const size_t budget = (size_t)(smem_optin / kTiles[pick].MINB) - 1024 - hdr_bytes;
  int stages = (int)std::min<size_t>(kMaxStages, budget / stage_bytes(wb, hb));
  while (stages < 3 && (wb > 48 || hb > 8)) {  // shrink the box; oversized footprints go global
#if CBP_ROWSHIFT
    if (hb >= wb || wb <= 64) hb = std::max(2, hb * 3 / 4); else wb /= 2;
#else
    if (hb >= wb || wb <= 48) hb = std::max(2, hb * 3 / 4); else wb -= 32;
#endif
    stages = (int)std::min<size_t>(kMaxStages, budget / stage_bytes(wb, hb));
  }
  plan.wb = wb;
  plan.hb = hb;
  if (const char* e = std::getenv("CBP_MAX_STAGES")) stages = std::min(stages, std::max(1, std::atoi(e)));  // tuning
  plan.stages = std::max(stages, 1);
  plan.smem = (size_t)plan.stages * stage_bytes(wb, hb) + hdr_bytes;
  return CBP_OK;
}

// Plan for `key`, returned BY VALUE (its matrices are reference counted): callers use it
// after the lock is gone, while other threads may evict it.  Plans are built outside the
// lock; eviction is per device, least recently used first.
int get_plan(const PlanKey& key, const float* mats_host, cudaStream_t stream, Plan* out) {
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_plans.find(key);
    if (it != g_plans.end()) {
      it->second.last_use = ++g_use_clock;
      *out = it->second;
      return CBP_OK;
    }
  }
  Plan p;
  int rc = make_plan(key, mats_host, stream, p);
  if (rc) return rc;
  std::shared_ptr<DevBuf> evicted;  // released after the lock: its destructor drains the device
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_plans.find(key);
    if (it != g_plans.end()) {  // another thread built the same plan meanwhile
      it->second.last_use = ++g_use_clock;
      *out = it->second;
      return CBP_OK;
    }
    int on_dev = 0;
    auto lru = g_plans.end();
    for (auto i = g_plans.begin(); i != g_plans.end(); ++i) {
      if (i->first.device != key.device) continue;
      ++on_dev;
      if (lru == g_plans.end() || i->second.last_use < lru->second.last_use) lru = i;
    }
    if (on_dev >= kPlansPerDevice && lru != g_plans.end()) {
      evicted = lru->second.mats;
      g_plans.erase(lru);
    }
    p.last_use = ++g_use_clock;
    g_plans.emplace(key, p);
  }
  *out = p;
  return CBP_OK;
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (device, kernel) and size
int ensure_smem(int dev, const void* fn, size_t smem) {
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_smem_set.find({dev, fn});
    if (it != g_smem_set.end() && it->second >= smem) return CBP_OK;
  }
  CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "set smem attribute");
  std::lock_guard<std::mutex> lk(g_mu);
  size_t& v = g_smem_set[{dev, fn}];
  v = std::max(v, smem);
  return CBP_OK;
}

// Dimensions the float32 index arithmetic supports.  A detector narrower or shorter than
// two pixels is legal (the reference accepts any size >= 1, tensors.py:44-58) and samples
// nothing: the guard x < nw-1 / y < nh-1 (_kernels.py:52) never passes, so the entry
// points return without launching.
int check_dims(int64_t np, int64_t nh, int64_t nw, int64_t nx, int64_t ny, int64_t nz) {
  if (np < 1 || nh < 1 || nw < 1 || nx < 1 || ny < 1 || nz < 1) return fail(CBP_EINVAL, "dimensions must be >= 1");
  if (nh >= (1 << 23) || nw >= (1 << 23) || np >= (1 << 30) || nx >= (1 << 24) || ny >= (1 << 24) ||
      nz >= (1 << 24))
    return fail(CBP_EINVAL, "dimension too large for float32 index arithmetic");
  return CBP_OK;
}
bool samples_nothing(int64_t nh, int64_t nw) { return nh < 2 || nw < 2; }

// keep freed stream-ordered allocations cached in the device's default pool (the
// host path allocates projection-sized buffers on every call)
void keep_pool_warm(int dev) {
  static std::once_flag once[64];
  if (dev < 0 || dev >= 64) return;
  std::call_once(once[dev], [dev] {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  });
}

int current_device(int* dev) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    return fail(CBP_ENODEV, "no CUDA device visible");
  }
  CK(cudaGetDevice(dev), "cudaGetDevice");
  return CBP_OK;
}

void vol_strides(int layout, int64_t nx, int64_t ny, int64_t nz, long long& sx, long long& sy, long long& sz) {
  if (layout == CBP_NATURAL) {  // [z][y][x]
    sx = 1;
    sy = nx;
    sz = nx * ny;
  } else {  // [x][y][z]
    sz = 1;
    sy = nz;
    sx = ny * nz;
  }
}

// One back-projection launch on staged projections (every public kernel entry point
// ends here).  `staged` holds detector rows [band_v0, band_v0 + band_rows) of angles
// [s_base, s_base + n_staged) in the layout [n_staged][band_rows][pitch]; the launch
// accumulates angles [s_begin, s_end) into slab [k0, k0 + nz) of a volume of nz_total
// slices; device-side status counters go to `stats`.
struct StagedCall {
  const float* staged;
  int64_t pitch, np, nh, nw, band_v0, band_rows;
  const float* mats_host;
  float* vol;
  int vol_layout;
  int64_t nx, ny, nz, k0, nz_total, s_begin, s_end, s_base, n_staged;
  int variant;
  unsigned flags;
};

int validate_staged(StagedCall& c) {
  int rc = check_dims(c.np, c.nh, c.nw, c.nx, c.ny, c.nz);
  if (rc) return rc;
  if (!c.staged || !c.mats_host || !c.vol) return fail(CBP_EINVAL, "null buffer");
  if (c.variant < 0 || c.variant > 5) return fail(CBP_EINVAL, "unknown kernel variant");
  if (c.vol_layout != CBP_NATURAL && c.vol_layout != CBP_TRANSPOSED) return fail(CBP_EINVAL, "unknown volume layout");
  if (c.k0 < 0 || c.nz_total < c.k0 + c.nz) return fail(CBP_EINVAL, "slab [k0, k0+nz) outside nz_total");
  if (v_mirror(c.variant) && (c.nz_total & 1)) return fail(CBP_EINVAL, "symmetry kernels need an even nz");
  if (c.s_end <= 0) c.s_end = c.np;
  if (c.s_begin < 0 || c.s_begin > c.s_end || c.s_end > c.np) return fail(CBP_EINVAL, "invalid angle range");
  if (c.n_staged <= 0) c.n_staged = c.np - c.s_base;
  if (c.s_base < 0 || c.s_base > c.s_begin || c.s_base + c.n_staged < c.s_end || c.s_base + c.n_staged > c.np)
    return fail(CBP_EINVAL, "staged angle window does not cover [s_begin, s_end)");
  if (!mats_finite(c.mats_host, c.np * 12)) return fail(CBP_EINVAL, "projection matrices contain non-finite values");
  if ((c.flags & CBP_FLAG_FMA_LERP) &&
      (c.variant != V_BASELINE || (c.flags & (CBP_FLAG_NAIVE | CBP_FLAG_CHECK | CBP_FLAG_NO_SMEM))))
    return fail(CBP_EINVAL, "CBP_FLAG_FMA_LERP is a tolerance mode of the tiled baseline kernel only");
  if (samples_nothing(c.nh, c.nw)) return CBP_OK;
  if (c.band_v0 < 0 || c.band_rows < 2 || c.band_v0 + c.band_rows > c.nh || c.pitch < c.nw || (c.pitch & 3))
    return fail(CBP_EINVAL, "invalid detector-row band or pitch");
  return CBP_OK;
}

int launch_staged(StagedCall c, unsigned long long* stats, cudaStream_t st) {
  int rc = validate_staged(c);
  if (rc) return rc;
  if (c.s_begin == c.s_end || samples_nothing(c.nh, c.nw)) return CBP_OK;
  // a NATURAL slab of 32m + 16 slices: the 32-slice tiles, then the last 16 slices as one layer
  // of half z-run tiles (fast loops instead of the partial-tile path)
  constexpr unsigned kHalfExcluded = CBP_FLAG_NAIVE | CBP_FLAG_CHECK | CBP_FLAG_FMA_LERP;
  if (c.vol_layout == CBP_NATURAL && c.nz > kZR && c.nz % kZR == kZR / 2 && !(c.flags & kHalfExcluded)) {
    StagedCall head = c, tail = c;
    head.nz = c.nz - kZR / 2;
    tail.nz = kZR / 2;
    tail.k0 = c.k0 + head.nz;
    tail.vol = c.vol + (size_t)head.nz * (size_t)c.nx * (size_t)c.ny;
    rc = launch_staged(head, stats, st);
    return rc ? rc : launch_staged(tail, stats, st);
  }
  const bool half = c.nz == kZR / 2 && !(c.flags & kHalfExcluded);
  const int zr = half ? kZR / 2 : kZR;
  int dev;
  rc = current_device(&dev);
  if (rc) return rc;

  PlanKey key;
  std::memset(&key, 0, sizeof(key));
  key.device = dev;
  key.variant = (c.variant == V_PREFETCH) ? V_SUBLINE : c.variant;
  key.kind_req = (c.flags & CBP_FLAG_NAIVE) ? 0 : 1;
  key.np = c.np; key.nh = c.nh; key.nw = c.nw; key.band_v0 = c.band_v0; key.band_rows = c.band_rows;
  key.nx = c.nx; key.ny = c.ny; key.nz = c.nz; key.k0 = c.k0; key.nz_total = c.nz_total;
  key.mhash = hash_words(c.mats_host, (size_t)c.np * 12 * sizeof(float));
  Plan plan;
  rc = get_plan(key, c.mats_host, st, &plan);
  if (rc) return rc;

  BPParams p{};
  std::memset(&p, 0, sizeof(p));
  p.proj = c.staged;
  p.mats = plan.mats_dev();
  p.vol = c.vol;
  vol_strides(c.vol_layout, c.nx, c.ny, c.nz, p.vsx, p.vsy, p.vsz);
  p.np = (int)c.np; p.nw = (int)c.nw; p.nh = (int)c.nh; p.pitch = (int)c.pitch;
  p.band_v0 = (int)c.band_v0; p.band_rows = (int)c.band_rows;
  p.nx = (int)c.nx; p.ny = (int)c.ny; p.nz = (int)c.nz; p.k0 = (int)c.k0; p.nz_total = (int)c.nz_total;
  p.s_begin = (int)c.s_begin; p.s_end = (int)c.s_end; p.s_base = (int)c.s_base;
  p.stats = stats;
  p.stagger_groups = 1;
  if (const char* e = std::getenv("CBP_STAGGER_NS")) p.stagger_ns = std::atoi(e);  // tuning
  if (const char* e = std::getenv("CBP_STAGGER_GROUPS")) p.stagger_groups = std::max(1, std::atoi(e));
  // 8x8-tile launch groups: -22% DRAM traffic on cfg4 (L2 hit rate 39% -> 48%), same speed
  p.tile_group = 8;
  if (const char* e = std::getenv("CBP_TILE_GROUP")) p.tile_group = std::max(1, std::atoi(e));  // tuning

  if (plan.kind == 0) {
    const int64_t nvox = c.nx * c.ny * c.nz;
    dim3 b(256), g((unsigned)ceil_div(nvox, 256));
    void* args[] = {&p};
    CK(cudaLaunchKernel(naive_kernel_ptr(key.variant), g, b, args, 0, st), "naive kernel launch");
    int64_t lp[9] = {1, 1, 1, 0, 0, 0, (int64_t)g.x, 0, 0};
    std::memcpy(g_last_plan, lp, sizeof(lp));
    return CBP_OK;
  }

  // tiled TMA path
  EncodeTiledFn enc = get_encode();
  if (!enc) return fail(CBP_ECUDA, "cuTensorMapEncodeTiled unavailable from the driver");
  p.tiles_x = (int)ceil_div(c.nx, plan.TX);
  p.tiles_y = (int)ceil_div(c.ny, plan.TY);
  p.tiles_z = (int)ceil_div(c.nz, zr);
  p.wb = plan.wb;
  p.hb = plan.hb;
  p.stages = plan.stages;
  if (c.flags & CBP_FLAG_NO_SMEM) p.hb = 1;  // every pair through the global path: make the box unusable
  CUtensorMap tmap;
  std::memset(&tmap, 0, sizeof(tmap));
  cuuint64_t gdim[3] = {(cuuint64_t)c.nw, (cuuint64_t)c.band_rows, (cuuint64_t)c.n_staged};
  cuuint64_t gstride[2] = {(cuuint64_t)c.pitch * 4, (cuuint64_t)(c.pitch * c.band_rows) * 4};
  cuuint32_t box[3] = {(cuuint32_t)plan.wb, (cuuint32_t)plan.hb, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult cr = enc(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(c.staged), gdim, gstride, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) {
    char buf[160];
    std::snprintf(buf, sizeof buf, "cuTensorMapEncodeTiled failed (%d): box %dx%d pitch %lld", (int)cr, plan.wb,
                  plan.hb, (long long)c.pitch);
    return fail(CBP_ECUDA, buf);
  }
  const void* fn =
#if CBP_DEV_SLIM
      tiled_kernel_ptr(key.variant, plan.kind == 2, plan.cfg, false);
#else
      (c.flags & CBP_FLAG_FMA_LERP)
                       ? (plan.kind == 2 ? fmalerp_by_tile<true>(plan.cfg) : fmalerp_by_tile<false>(plan.cfg))
                   : half ? half_kernel_ptr(key.variant, plan.kind == 2, plan.cfg)
                          : tiled_kernel_ptr(key.variant, plan.kind == 2, plan.cfg, (c.flags & CBP_FLAG_CHECK) != 0);
#endif
  rc = ensure_smem(dev, fn, plan.smem);
  if (rc) return rc;
  const int64_t blocks = (int64_t)p.tiles_x * p.tiles_y * p.tiles_z;
  if (blocks > 0x7fffffffLL) return fail(CBP_EINVAL, "volume too large for one launch");
  if (kTilePool[plan.cfg] != 0) {  // setmaxnreg.inc would wait forever on a smaller pool
    cudaFuncAttributes fa{};
    CK(cudaFuncGetAttributes(&fa, fn), "cudaFuncGetAttributes(tiled kernel)");
    if (fa.numRegs != kTilePool[plan.cfg]) {
      char buf[128];
      std::snprintf(buf, sizeof buf, "tiled kernel register pool %d != %d assumed by its setmaxnreg split",
                    fa.numRegs, kTilePool[plan.cfg]);
      return fail(CBP_ECUDA, buf);
    }
  }
  // angle-independent r1[2] * fkk table (see TyTab): every matrix of the launch shares m[6]
  static thread_local TyTab tytab;
  p.ty_const = c.nz <= kTyTabMax ? 1 : 0;
  // the same loop forms texel byte addresses with one subnormal FMA (bp_kernels.cuh, ADDR_W4):
  // exact while |box base - v0 * row pitch| < 2^24
  p.addr_ok = c.nh * (int64_t)plan.wb * 4 < (1 << 24) - (1 << 19) ? 1 : 0;
  if (!p.addr_ok) p.ty_const = 0;
  {
    uint32_t m6_bits;
    std::memcpy(&m6_bits, c.mats_host + 12 * c.s_begin + 6, 4);
    for (int64_t s = c.s_begin; s < c.s_end && p.ty_const; ++s) {
      uint32_t b;
      std::memcpy(&b, c.mats_host + 12 * s + 6, 4);
      if (b != m6_bits) p.ty_const = 0;
    }
    if (p.ty_const) {
      const float m6 = c.mats_host[12 * c.s_begin + 6];
      const int64_t nzh = c.nz_total >> 1;
      const int64_t n_tab = std::min<int64_t>(kTyTabMax, ceil_div(c.nz, kZR) * kZR);
      for (int64_t q = 0; q < n_tab; ++q) {
        const int64_t kg = c.k0 + q;
        const int64_t kk = (v_mirror(key.variant) && kg >= nzh) ? c.nz_total - 1 - kg : kg;
        const volatile float prod = m6 * (float)kk;  // one rounded float32 product, as the kernel's __fmul_rn
        tytab.v[q] = prod;
      }
    }
  }
  if (p.tiles_z > 65535) return fail(CBP_EINVAL, "volume too deep for one launch");
  dim3 g((unsigned)(p.tiles_x * p.tiles_y), (unsigned)p.tiles_z), b(kTileThreads[plan.cfg]);
  void* args[] = {&tmap, &p, &tytab};
  CK(cudaLaunchKernel(fn, g, b, args, plan.smem, st), "tiled kernel launch");
  int64_t lp[9] = {plan.TX, plan.TY, zr, plan.wb, plan.hb, plan.stages, blocks, (int64_t)plan.smem, plan.kind};
  std::memcpy(g_last_plan, lp, sizeof(lp));
  return CBP_OK;
}

// read (and clear) a status buffer on `st`; CBP_EBAND when samples fell outside a band
int read_stats(unsigned long long* d, cudaStream_t st, int64_t* stats5) {
  unsigned long long h[8] = {0};
  CK(cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, st), "read status");
  CK(cudaMemsetAsync(d, 0, sizeof(h), st), "reset status");
  CK(cudaStreamSynchronize(st), "status sync");
  if (stats5)
    for (int q = 0; q < 5; ++q) stats5[q] += (int64_t)h[q];
  if (h[3]) {
    char buf[128];
    std::snprintf(buf, sizeof buf, "%llu samples fell outside the slab's detector-row band", h[3]);
    return fail(CBP_EBAND, buf);
  }
  return CBP_OK;
}

// private status buffer for calls that synchronise before returning (host path, multi-GPU)
struct ScopedStats {
  unsigned long long* d = nullptr;
  int alloc(cudaStream_t st) {
    CK(cudaMallocAsync(reinterpret_cast<void**>(&d), 8 * sizeof(unsigned long long), st), "alloc status");
    CK(cudaMemsetAsync(d, 0, 8 * sizeof(unsigned long long), st), "clear status");
    return CBP_OK;
  }
  void release(cudaStream_t st) {
    if (d) cudaFreeAsync(d, st);
    d = nullptr;
  }
};

}  // namespace

// =================================================================== C ABI
extern "C" {

int cbp_version(void) { return 200; }  // 0.2.0

const char* cbp_last_error(void) { return g_err.c_str(); }

int cbp_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int64_t cbp_staged_pitch(int64_t nw) { return (nw + 3) & ~(int64_t)3; }

int cbp_stage_projections(const float* img_dev, int img_layout, int64_t np, int64_t nh, int64_t nw, int64_t v0,
                          int64_t rows, float* staged_dev, int64_t pitch, void* cuda_stream) {
  if (!img_dev || !staged_dev) return fail(CBP_EINVAL, "null buffer");
  if (np < 1 || nh < 1 || nw < 1 || v0 < 0 || rows < 1 || v0 + rows > nh || pitch < nw || (pitch & 3))
    return fail(CBP_EINVAL, "invalid staging band / pitch");
  if (np > 65535) return fail(CBP_EINVAL, "np > 65535 not supported by the staging kernels");
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  if (img_layout == CBP_NATURAL) {
    dim3 b(128, 4), g((unsigned)std::min<int64_t>(ceil_div(pitch, 128), 8), (unsigned)ceil_div(rows, 4), (unsigned)np);
    stage_rows_kernel<<<g, b, 0, st>>>(img_dev, (int)nh, (int)nw, (int)v0, (int)rows, staged_dev, (int)pitch);
  } else if (img_layout == CBP_TRANSPOSED) {
    dim3 b(32, 8), g((unsigned)ceil_div(pitch, 32), (unsigned)ceil_div(rows, 32), (unsigned)np);
    stage_transposed_kernel<<<g, b, 0, st>>>(img_dev, (int)nh, (int)nw, (int)v0, (int)rows, staged_dev, (int)pitch);
  } else {
    return fail(CBP_EINVAL, "unknown projection layout");
  }
  CK(cudaGetLastError(), "stage kernel launch");
  return CBP_OK;
}

int cbp_backproject_window(const float* staged_dev, int64_t pitch, int64_t np, int64_t nh, int64_t nw,
                           int64_t band_v0, int64_t band_rows, int64_t s_base, int64_t n_staged,
                           const float* mats_host, float* vol_dev, int vol_layout, int64_t nx, int64_t ny, int64_t nz,
                           int64_t k0, int64_t nz_total, int64_t s_begin, int64_t s_end, int variant, unsigned flags,
                           void* cuda_stream) {
  StagedCall c{staged_dev, pitch,    np, nh, nw, band_v0, band_rows, mats_host, vol_dev, vol_layout, nx, ny, nz, k0,
               nz_total,   s_begin, s_end, s_base, n_staged, variant, flags};
  int dev;
  int rc = validate_staged(c);
  if (rc || c.s_begin == c.s_end || samples_nothing(nh, nw)) return rc;
  rc = current_device(&dev);
  if (rc) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  unsigned long long* stats = nullptr;
  rc = get_stats(dev, st, &stats);
  if (rc) return rc;
  return launch_staged(c, stats, st);
}

int cbp_backproject_staged(const float* staged_dev, int64_t pitch, int64_t np, int64_t nh, int64_t nw,
                           int64_t band_v0, int64_t band_rows, const float* mats_host, float* vol_dev, int vol_layout,
                           int64_t nx, int64_t ny, int64_t nz, int64_t k0, int64_t nz_total, int64_t s_begin,
                           int64_t s_end, int variant, unsigned flags, void* cuda_stream) {
  return cbp_backproject_window(staged_dev, pitch, np, nh, nw, band_v0, band_rows, 0, np, mats_host, vol_dev,
                                vol_layout, nx, ny, nz, k0, nz_total, s_begin, s_end, variant, flags, cuda_stream);
}

int cbp_backproject_f32(const float* img_dev, int64_t np, int64_t nh, int64_t nw, int img_layout,
                        const float* mats_host, float* vol_dev, int64_t nx, int64_t ny, int64_t nz, int vol_layout,
                        int variant, unsigned flags, void* cuda_stream) {
  int rc = check_dims(np, nh, nw, nx, ny, nz);
  if (rc) return rc;
  if (!img_dev) return fail(CBP_EINVAL, "null projection buffer");
  if (img_layout != CBP_NATURAL && img_layout != CBP_TRANSPOSED) return fail(CBP_EINVAL, "unknown projection layout");
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  if (samples_nothing(nh, nw) || (img_layout == CBP_NATURAL && (nw & 3) == 0)) {
    // already in the staging layout: zero copy (or nothing to sample)
    return cbp_backproject_staged(img_dev, samples_nothing(nh, nw) ? 4 : nw, np, nh, nw, 0, nh, mats_host, vol_dev,
                                  vol_layout, nx, ny, nz, 0, nz, 0, np, variant, flags, cuda_stream);
  }
  const int64_t pitch = cbp_staged_pitch(nw);
  float* staged = nullptr;
  CK(cudaMallocAsync(reinterpret_cast<void**>(&staged), (size_t)np * nh * pitch * 4, st), "alloc staging");
  rc = cbp_stage_projections(img_dev, img_layout, np, nh, nw, 0, nh, staged, pitch, cuda_stream);
  if (rc == CBP_OK)
    rc = cbp_backproject_staged(staged, pitch, np, nh, nw, 0, nh, mats_host, vol_dev, vol_layout, nx, ny, nz, 0, nz, 0,
                                np, variant, flags, cuda_stream);
  cudaFreeAsync(staged, st);
  return rc;
}

int cbp_backproject_host_f32(const float* img_host, int64_t np, int64_t nh, int64_t nw, int img_layout,
                             const float* mats_host, float* vol_host, int64_t nx, int64_t ny, int64_t nz,
                             int vol_layout, int variant, unsigned flags) {
  int rc = check_dims(np, nh, nw, nx, ny, nz);
  if (rc) return rc;
  if (!img_host || !vol_host || !mats_host) return fail(CBP_EINVAL, "null buffer");
  if (img_layout != CBP_NATURAL && img_layout != CBP_TRANSPOSED) return fail(CBP_EINVAL, "unknown projection layout");
  if (vol_layout != CBP_NATURAL && vol_layout != CBP_TRANSPOSED) return fail(CBP_EINVAL, "unknown volume layout");
  if (variant < 0 || variant > 5) return fail(CBP_EINVAL, "unknown kernel variant");
  if (v_mirror(variant) && (nz & 1)) return fail(CBP_EINVAL, "symmetry kernels need an even nz");
  if (!mats_finite(mats_host, np * 12)) return fail(CBP_EINVAL, "projection matrices contain non-finite values");
  if (samples_nothing(nh, nw)) return CBP_OK;  // the volume is left unchanged, as by the reference
  int dev;
  rc = current_device(&dev);
  if (rc) return rc;
  // Pipeline over three streams.  The projections travel host->device in angle chunks on
  // the upload stream while the compute stream stages and back-projects the chunks already
  // resident (each launch accumulates angles [s0, s1) in ascending order: bitwise identical
  // to one launch).  A NATURAL volume is also split into z-slabs (contiguous, cut on the
  // kernel's 32-slice z-runs): the first slab is uploaded first, the next one uploads while
  // one computes and each downloads on the third stream while its successor computes, so
  // only the first slab's upload, the first projection chunk and the last download are not
  // hidden.  The first slab is the CENTRAL one: it is the most expensive (every angle samples
  // it), so its chunked launches keep the SMs busy for as long as the projections take to
  // arrive (cfg4: 0.85 s of compute against 0.63 s of upload; a cheap end slab left the GPU
  // idle for most of the upload).
  const size_t per_proj = (size_t)nh * nw, ib = (size_t)np * per_proj * 4, vb = (size_t)nx * ny * nz * 4;
  const bool direct = img_layout == CBP_NATURAL && (nw & 3) == 0;  // natural layout is the staging layout
  const int64_t pitch = cbp_staged_pitch(nw);
  int64_t n_chunks = std::min<int64_t>(np, std::max<int64_t>(1, (int64_t)(ib >> 24)));  // ~16 MiB chunks
  n_chunks = std::min<int64_t>(n_chunks, 24);
  if (const char* env = std::getenv("CBP_HOST_CHUNKS")) n_chunks = std::max<int64_t>(1, std::min<int64_t>(np, std::atoi(env)));
  int64_t n_slabs = 1;
  if (vol_layout == CBP_NATURAL && vb >= ((size_t)256 << 20)) n_slabs = std::min<int64_t>(8, nz / kZR);
  if (const char* env = std::getenv("CBP_HOST_SLABS")) n_slabs = std::atoi(env);
  n_slabs = std::max<int64_t>(1, std::min<int64_t>(n_slabs, ceil_div(nz, kZR)));
  if (vol_layout != CBP_NATURAL) n_slabs = 1;  // a z-slab of [x][y][z] is not contiguous
  std::vector<int64_t> zb((size_t)n_slabs + 1);
  for (int64_t k = 0; k <= n_slabs; ++k) zb[k] = (k == n_slabs) ? nz : (nz * k / n_slabs) / kZR * kZR;
  const size_t slice = (size_t)nx * ny;
  std::vector<int64_t> order;  // processing order of the slabs: centre first, then outwards
  {
    const int64_t c = n_slabs / 2;
    order.push_back(c);
    for (int64_t d = 1; d < n_slabs; ++d) {
      if (c + d < n_slabs) order.push_back(c + d);
      if (c - d >= 0) order.push_back(c - d);
    }
  }

  cudaStream_t sc = nullptr, sk = nullptr, sd = nullptr;
  std::vector<cudaEvent_t> ev_proj((size_t)n_chunks, nullptr), ev_vol((size_t)n_slabs, nullptr),
      ev_done((size_t)n_slabs, nullptr);
  float *img = nullptr, *vol = nullptr, *staged = nullptr;
  ScopedStats stats;
  cudaError_t e = cudaStreamCreateWithFlags(&sc, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&sk, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&sd, cudaStreamNonBlocking);
  for (auto* v : {&ev_proj, &ev_vol, &ev_done})
    for (auto& x : *v)
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&x, cudaEventDisableTiming);
  keep_pool_warm(dev);
  if (e == cudaSuccess) e = cudaMallocAsync(reinterpret_cast<void**>(&img), ib, sk);
  if (e == cudaSuccess) e = cudaMallocAsync(reinterpret_cast<void**>(&vol), vb, sk);
  if (e == cudaSuccess && !direct)
    e = cudaMallocAsync(reinterpret_cast<void**>(&staged), (size_t)np * nh * pitch * 4, sk);
  if (e == cudaSuccess) e = cudaStreamSynchronize(sk);  // allocations visible to the copy streams
  if (e != cudaSuccess) rc = cuda_fail(e, "host path: streams / allocation");
  if (rc == CBP_OK) rc = stats.alloc(sk);
  // uploads, in the order they are needed: the first slab, the projection chunks, the other slabs
  auto up_slab = [&](int64_t k) {
    const size_t off = (size_t)zb[k] * slice, n = (size_t)(zb[k + 1] - zb[k]) * slice;
    cudaError_t r = cudaMemcpyAsync(vol + off, vol_host + off, n * 4, cudaMemcpyHostToDevice, sc);
    return r == cudaSuccess ? cudaEventRecord(ev_vol[k], sc) : r;
  };
  if (rc == CBP_OK && (e = up_slab(order[0])) != cudaSuccess) rc = cuda_fail(e, "host path: volume upload");
  for (int64_t q = 0; q < n_chunks && rc == CBP_OK; ++q) {
    const int64_t s0 = np * q / n_chunks, s1 = np * (q + 1) / n_chunks;
    e = cudaMemcpyAsync(img + s0 * per_proj, img_host + s0 * per_proj, (size_t)(s1 - s0) * per_proj * 4,
                        cudaMemcpyHostToDevice, sc);
    if (e == cudaSuccess) e = cudaEventRecord(ev_proj[q], sc);
    if (e != cudaSuccess) rc = cuda_fail(e, "host path: projection upload");
  }
  for (int64_t t = 1; t < n_slabs && rc == CBP_OK; ++t)
    if ((e = up_slab(order[t])) != cudaSuccess) rc = cuda_fail(e, "host path: volume upload");
  // compute: the first slab follows the projection chunks as they land, the others run over all angles
  for (int64_t t = 0; t < n_slabs && rc == CBP_OK; ++t) {
    const int64_t k = order[t];
    if ((e = cudaStreamWaitEvent(sk, ev_vol[k], 0)) != cudaSuccess) {
      rc = cuda_fail(e, "host path: wait");
      break;
    }
    const int64_t k0 = zb[k], k1 = zb[k + 1];
    float* vslab = vol + (size_t)k0 * slice;
    for (int64_t q = 0; q < (t == 0 ? n_chunks : 1) && rc == CBP_OK; ++q) {
      const int64_t s0 = t == 0 ? np * q / n_chunks : 0, s1 = t == 0 ? np * (q + 1) / n_chunks : np;
      if (t == 0) {
        if ((e = cudaStreamWaitEvent(sk, ev_proj[q], 0)) != cudaSuccess) {
          rc = cuda_fail(e, "host path: wait");
          break;
        }
        if (!direct)
          rc = cbp_stage_projections(img + s0 * per_proj, img_layout, s1 - s0, nh, nw, 0, nh,
                                     staged + s0 * nh * pitch, pitch, sk);
      }
      StagedCall c{direct ? img : staged, direct ? nw : pitch, np, nh, nw, 0, nh, mats_host, vslab, vol_layout,
                   nx, ny, k1 - k0, k0, nz, s0, s1, 0, np, variant, flags};
      if (rc == CBP_OK) rc = launch_staged(c, stats.d, sk);
    }
    if (rc == CBP_OK && (e = cudaEventRecord(ev_done[k], sk)) != cudaSuccess) rc = cuda_fail(e, "host path: event");
    // download slab k while the next slab computes
    if (rc == CBP_OK && (e = cudaStreamWaitEvent(sd, ev_done[k], 0)) == cudaSuccess)
      e = cudaMemcpyAsync(vol_host + (size_t)k0 * slice, vslab, (size_t)(k1 - k0) * slice * 4,
                          cudaMemcpyDeviceToHost, sd);
    if (rc == CBP_OK && e != cudaSuccess) rc = cuda_fail(e, "host path: copy out");
  }
  if (rc == CBP_OK) rc = read_stats(stats.d, sk, nullptr);
  if (sc) cudaStreamSynchronize(sc);
  if (sd) {
    e = cudaStreamSynchronize(sd);
    if (e != cudaSuccess && rc == CBP_OK) rc = cuda_fail(e, "host path: copy out");
  }
  if (sk) {
    stats.release(sk);
    if (img) cudaFreeAsync(img, sk);
    if (vol) cudaFreeAsync(vol, sk);
    if (staged) cudaFreeAsync(staged, sk);
    e = cudaStreamSynchronize(sk);
    if (e != cudaSuccess && rc == CBP_OK) rc = cuda_fail(e, "host path: kernel execution");
  }
  for (auto* v : {&ev_proj, &ev_vol, &ev_done})
    for (auto x : *v)
      if (x) cudaEventDestroy(x);
  for (auto x : {sc, sk, sd})
    if (x) cudaStreamDestroy(x);
  return rc;
}

int cbp_sync_status(void* cuda_stream, int64_t* stats5) {
  int dev;
  int rc = current_device(&dev);
  if (rc) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  unsigned long long* d = nullptr;
  rc = get_stats(dev, st, &d);
  if (rc) return rc;
  if (stats5)
    for (int q = 0; q < 5; ++q) stats5[q] = 0;
  return read_stats(d, st, stats5);
}

int cbp_selftest_rcp(uint32_t lo_bits, uint32_t hi_bits, uint64_t* mismatches, uint32_t* first_bad) {
  if (!mismatches || !first_bad || hi_bits < lo_bits) return fail(CBP_EINVAL, "invalid self-test range");
  int dev;
  int rc = current_device(&dev);
  if (rc) return rc;
  unsigned long long* d = nullptr;
  CK(cudaMalloc(&d, 2 * sizeof(unsigned long long)), "alloc");
  unsigned long long h[2] = {0, ~0ull};
  cudaError_t e = cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e == cudaSuccess) {
    rcp_selftest_kernel<<<sms * 8, 256>>>(lo_bits, hi_bits, d);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (e != cudaSuccess) return cuda_fail(e, "rcp self-test");
  *mismatches = h[0];
  *first_bad = (uint32_t)std::min<unsigned long long>(h[1], 0xffffffffull);
  return CBP_OK;
}

int cbp_count_ops(const float* mats_host, int64_t np, int64_t nh, int64_t nw, int64_t nx, int64_t ny, int64_t nz,
                  int variant, int64_t nb, int64_t* out5, void* cuda_stream) {
  int rc = check_dims(np, nh, nw, nx, ny, nz);
  if (rc) return rc;
  if (!mats_host || !out5) return fail(CBP_EINVAL, "null buffer");
  if (variant < 0 || variant > 5) return fail(CBP_EINVAL, "unknown kernel variant");
  if (variant != V_BASELINE && (nb < 1 || np % nb)) return fail(CBP_EINVAL, "nb must divide np");
  if (v_mirror(variant) && (nz & 1)) return fail(CBP_EINVAL, "symmetry kernels need an even nz");
  if (!mats_finite(mats_host, np * 12)) return fail(CBP_EINVAL, "projection matrices contain non-finite values");
  int dev;
  rc = current_device(&dev);
  if (rc) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  float* md = nullptr;
  unsigned long long* cnt = nullptr;
  CK(cudaMallocAsync(reinterpret_cast<void**>(&md), np * 12 * 4, st), "alloc");
  CK(cudaMallocAsync(reinterpret_cast<void**>(&cnt), 2 * 8, st), "alloc");
  CK(cudaMemcpyAsync(md, mats_host, np * 12 * 4, cudaMemcpyHostToDevice, st), "copy");
  CK(cudaMemsetAsync(cnt, 0, 16, st), "memset");
  const int64_t nvox = nx * ny * nz;
  dim3 b(256), g((unsigned)ceil_div(nvox, 256));
  const int V = (variant == V_PREFETCH) ? V_SUBLINE : variant;
  switch (V) {
    case V_BASELINE: bp_count_kernel<V_BASELINE><<<g, b, 0, st>>>(md, (int)np, (int)nw, (int)nh, (int)nx, (int)ny, (int)nz, cnt); break;
    case V_TRANSPOSE: bp_count_kernel<V_TRANSPOSE><<<g, b, 0, st>>>(md, (int)np, (int)nw, (int)nh, (int)nx, (int)ny, (int)nz, cnt); break;
    case V_SHARE: bp_count_kernel<V_SHARE><<<g, b, 0, st>>>(md, (int)np, (int)nw, (int)nh, (int)nx, (int)ny, (int)nz, cnt); break;
    case V_SYMMETRY: bp_count_kernel<V_SYMMETRY><<<g, b, 0, st>>>(md, (int)np, (int)nw, (int)nh, (int)nx, (int)ny, (int)nz, cnt); break;
    default: bp_count_kernel<V_SUBLINE><<<g, b, 0, st>>>(md, (int)np, (int)nw, (int)nh, (int)nx, (int)ny, (int)nz, cnt); break;
  }
  CK(cudaGetLastError(), "count kernel launch");
  unsigned long long h[2];
  CK(cudaMemcpyAsync(h, cnt, 16, cudaMemcpyDeviceToHost, st), "read counts");
  cudaFreeAsync(md, st);
  cudaFreeAsync(cnt, st);
  CK(cudaStreamSynchronize(st), "count sync");
  const int64_t S = (int64_t)h[0], OK = (int64_t)h[1];
  const int64_t U = nx * ny * nz * np, C = nx * ny * np, cols = nx * ny;
  const int64_t nbat = (variant == V_BASELINE) ? 0 : np / nb;
  const int64_t nzh = nz / 2;
  int64_t dots, volw, projw, interp, builds = 0;
  // closed forms of the twin's tallies (reference.py:26-290)
  switch (variant) {
    case V_BASELINE: dots = 3 * U; volw = 2 * S; projw = 4 * S; interp = 3 * S; break;
    case V_TRANSPOSE: dots = 3 * U; volw = 2 * nz * nbat * cols; projw = 4 * S; interp = 3 * S; break;
    case V_SHARE: dots = 2 * C + nz * OK; volw = 2 * nz * nbat * cols; projw = 4 * S; interp = 3 * S; break;
    case V_SYMMETRY: dots = 2 * C + nzh * OK; volw = 4 * nzh * nbat * cols; projw = 4 * S; interp = 3 * S; break;
    default:  // SUBLINE, SUBLINE_PREFETCH
      dots = 2 * C + nzh * OK; volw = 4 * nzh * nbat * cols; builds = OK; projw = 2 * nh * OK; interp = nh * OK + S;
      break;
  }
  out5[0] = dots; out5[1] = volw; out5[2] = projw; out5[3] = interp; out5[4] = builds;
  return CBP_OK;
}

}  // extern "C"

// ============================================================ host planning
namespace {

// float32 corner projection with the rung's formulas (host copy of the device
// arithmetic; x86-64 float math is IEEE binary32 and is built without FMA contraction)
inline float h_dot4(const float* m, float fi, float fj, float fk) {
  float a = m[0] * fi;
  float b = m[1] * fj;
  float c = a + b;
  float d = m[2] * fk;
  float e = c + d;
  return e + m[3];
}
inline void h_coords(const float* m, int variant, int i, int j, int kg, int nz_total, int nh, float& x, float& y,
                     float& z) {
  const float fi = (float)i, fj = (float)j;
  if (v_hoist(variant)) {
    z = h_dot4(m + 8, fi, fj, 0.0f);
    const float F = 1.0f / z;
    x = h_dot4(m, fi, fj, 0.0f) * F;
    int kk = kg;
    bool hi = false;
    if (v_mirror(variant) && kg >= nz_total / 2) { kk = nz_total - 1 - kg; hi = true; }
    y = h_dot4(m + 4, fi, fj, (float)kk) * F;
    if (hi) y = (float)(nh - 1) - y;
  } else {
    const float fk = (float)kg;
    z = h_dot4(m + 8, fi, fj, fk);
    const float f = 1.0f / z;
    x = h_dot4(m, fi, fj, fk) * f;
    y = h_dot4(m + 4, fi, fj, fk) * f;
  }
}

// v range [vmin, vmax] over the corners of slices [k0, k1), all angles; false if unbounded
bool slab_vrange(const float* mats, int64_t np, int64_t nh, int64_t nw, int64_t nx, int64_t ny, int64_t nz,
                 int variant, int64_t k0, int64_t k1, int64_t* out_v0, int64_t* out_rows) {
  const int nzh = (int)(nz / 2);
  std::vector<int> ks = {(int)k0, (int)(k1 - 1)};
  if (v_mirror(variant) && k0 < nzh && k1 - 1 >= nzh) {
    ks.push_back(nzh - 1);
    ks.push_back(nzh);
  }
  int64_t lo = INT64_MAX, hi = INT64_MIN;
  for (int64_t s = 0; s < np; ++s) {
    const float* m = mats + 12 * s;
    float umn = 3e38f, umx = -3e38f, vmn = 3e38f, vmx = -3e38f;
    bool bad = false;
    for (int ci = 0; ci < 2; ++ci)
      for (int cj = 0; cj < 2; ++cj)
        for (int kg : ks) {
          float x, y, z;
          h_coords(m, variant, ci ? (int)nx - 1 : 0, cj ? (int)ny - 1 : 0, kg, (int)nz, (int)nh, x, y, z);
          if (!(z > 0.0f) || !std::isfinite(x) || !std::isfinite(y)) bad = true;
          umn = std::min(umn, x); umx = std::max(umx, x);
          vmn = std::min(vmn, y); vmx = std::max(vmx, y);
        }
    if (bad) {  // cannot bound: the whole detector
      lo = 0;
      hi = nh - 1;
      break;
    }
    // anchors ix in [floor(umin)-1, floor(umax)+1] ∩ [0, nw-2]: skip angles with no column on the detector
    const double ulo = std::max(std::floor((double)umn) - 1.0, 0.0), uhi = std::min(std::floor((double)umx) + 1.0, (double)nw - 2);
    if (ulo > uhi) continue;
    const double vlo = std::max(std::floor((double)vmn) - 2.0, 0.0);
    const double vhi = std::min(std::floor((double)vmx) + 3.0, (double)nh - 1);
    if (vlo > vhi) continue;
    lo = std::min(lo, (int64_t)vlo);
    hi = std::max(hi, (int64_t)vhi);
  }
  if (lo > hi) {
    *out_v0 = 0;
    *out_rows = 0;
  } else {
    *out_v0 = lo;
    *out_rows = std::max<int64_t>(hi - lo + 1, 2);
    if (*out_v0 + *out_rows > nh) *out_v0 = nh - *out_rows;
  }
  return true;
}

}  // namespace

extern "C" {

int cbp_slab_band(const float* mats_host, int64_t np, int64_t nh, int64_t nw, int64_t nx, int64_t ny, int64_t nz,
                  int variant, int64_t k0, int64_t k1, int64_t* v0, int64_t* rows) {
  int rc = check_dims(np, nh, nw, nx, ny, nz);
  if (rc) return rc;
  if (!mats_host || !v0 || !rows) return fail(CBP_EINVAL, "null buffer");
  if (k0 < 0 || k1 > nz || k0 >= k1) return fail(CBP_EINVAL, "invalid slab range");
  if (!mats_finite(mats_host, np * 12)) return fail(CBP_EINVAL, "projection matrices contain non-finite values");
  slab_vrange(mats_host, np, nh, nw, nx, ny, nz, variant, k0, k1, v0, rows);
  return CBP_OK;
}

int cbp_slab_plan(const float* mats_host, int64_t np, int64_t nh, int64_t nw, int64_t nx, int64_t ny, int64_t nz,
                  int variant, int64_t n_ranks, int64_t align, int64_t* k_bounds, int64_t* bands) {
  int rc = check_dims(np, nh, nw, nx, ny, nz);
  if (rc) return rc;
  if (!mats_host || !k_bounds || !bands) return fail(CBP_EINVAL, "null buffer");
  if (n_ranks < 1 || align < 1) return fail(CBP_EINVAL, "n_ranks and align must be >= 1");
  if (!mats_finite(mats_host, np * 12)) return fail(CBP_EINVAL, "projection matrices contain non-finite values");
  const int64_t nlayers = ceil_div(nz, align);
  // Cost per layer of `align` slices, modelled on what the tiled kernel does: a (tile,
  // angle) pair whose footprint misses the detector is never queued (cost ~ the producer's
  // footprint test), any other pair costs the whole tile's z-run -- even when only some
  // of its voxels are sampled -- and a little more when it crosses the detector's top or
  // bottom row (guarded loop).  Evaluated with the kernel's corner test on a subsample of
  // 32x16-column tiles and angles.  (A per-voxel sampled count under-weights the
  // partially sampled tiles at the volume's z ends: 0.78 instead of 0.97 compute balance
  // on cfg4 at 8 ranks, tools/slab_balance.py.)
  // Weights fitted to the per-rank times of tools/slab_balance.py (round 2): on the fast path a
  // tile crossing the detector's top or bottom row costs 1.15x (its columns check u once per
  // angle anyway); on the general path (per-voxel 1/z and x) the guard-free loop needs the whole
  // tile on the detector in u and v, and a guarded pair costs 2x; a never-queued pair costs the
  // producer's footprint test.
  const bool gen = !fast_path_ok(mats_host, np, variant);
  const double w_guard = gen ? 2.0 : 1.15, w_miss = gen ? 0.06 : 0.03;
  const int64_t TXm = 32, TYm = 16;
  const int64_t ntx = ceil_div(nx, TXm), nty = ceil_div(ny, TYm);
  const int64_t stx = std::max<int64_t>(1, ntx / 12), sty = std::max<int64_t>(1, nty / 12);
  const int64_t ss = std::max<int64_t>(1, np / 96);
  std::vector<double> cost(nlayers, 0.0);
  for (int64_t L = 0; L < nlayers; ++L) {
    double c = 0.0;
    const int ka = (int)(L * align), kb = (int)(std::min(nz, (L + 1) * align) - 1);
    for (int64_t s = 0; s < np; s += ss)
      for (int64_t by = 0; by < nty; by += sty)
        for (int64_t bx = 0; bx < ntx; bx += stx) {
          const int i0 = (int)(bx * TXm), i1 = (int)std::min(nx, (bx + 1) * TXm) - 1;
          const int j0 = (int)(by * TYm), j1 = (int)std::min(ny, (by + 1) * TYm) - 1;
          float umin = 3e38f, umax_ = -3e38f, vmin = 3e38f, vmax_ = -3e38f;
          bool bad = false;
          int kc[4] = {ka, kb, (int)(nz / 2) - 1, (int)(nz / 2)};
          const int nk = (v_mirror(variant) && ka < nz / 2 && kb >= nz / 2) ? 4 : 2;
          for (int q = 0; q < 4 * nk; ++q) {
            float x, y, z;
            h_coords(mats_host + 12 * s, variant, (q & 1) ? i1 : i0, (q & 2) ? j1 : j0, kc[q >> 2], (int)nz, (int)nh,
                     x, y, z);
            bad = bad || !(z > 0.0f) || !std::isfinite(x) || !std::isfinite(y);
            umin = std::min(umin, x); umax_ = std::max(umax_, x);
            vmin = std::min(vmin, y); vmax_ = std::max(vmax_, y);
          }
          if (bad) { c += 1.0; continue; }
          const double ulo = std::floor(umin) - 1, uhi = std::floor(umax_) + 1;
          const double vlo = std::floor(vmin) - 1, vhi = std::floor(vmax_) + 1;
          const bool hit = std::max(ulo, 0.0) <= std::min(uhi, (double)(nw - 2)) &&
                           std::max(vlo, 0.0) <= std::min(vhi, (double)(nh - 2));
          if (!hit) { c += w_miss; continue; }
          const bool rows_inside = vlo >= 0 && vhi <= (double)(nh - 2);
          const bool cols_inside = ulo >= 0 && uhi <= (double)(nw - 2);
          c += (rows_inside && (cols_inside || !gen)) ? 1.0 : w_guard;
        }
    cost[L] = c * (double)(kb - ka + 1) / (double)align + 1e-9;
  }
  std::vector<double> pre(nlayers + 1, 0.0);
  for (int64_t L = 0; L < nlayers; ++L) pre[L + 1] = pre[L] + cost[L];
  // contiguous partition of the layers into n_ranks slabs minimising the costliest slab
  // (exact dynamic programme; nlayers <= nz/align is small)
  const int64_t R = n_ranks;
  const double inf = 1e300;
  std::vector<double> best((size_t)(R + 1) * (nlayers + 1), inf);
  std::vector<int64_t> arg((size_t)(R + 1) * (nlayers + 1), 0);
  auto B = [&](int64_t r, int64_t i) -> double& { return best[(size_t)r * (nlayers + 1) + i]; };
  auto A = [&](int64_t r, int64_t i) -> int64_t& { return arg[(size_t)r * (nlayers + 1) + i]; };
  B(0, 0) = 0.0;
  for (int64_t r = 1; r <= R; ++r)
    for (int64_t i = 0; i <= nlayers; ++i)
      for (int64_t j = 0; j <= i; ++j) {  // slab r-1 = layers [j, i)
        if (B(r - 1, j) >= inf) continue;
        const double v = std::max(B(r - 1, j), pre[i] - pre[j]);
        if (v < B(r, i) - 1e-12 * std::abs(v)) {
          B(r, i) = v;
          A(r, i) = j;
        }
      }
  {
    int64_t i = nlayers;
    for (int64_t r = R; r >= 1; --r) {
      k_bounds[r] = std::min(nz, i * align);
      i = A(r, i);
    }
    k_bounds[0] = 0;
  }
  k_bounds[n_ranks] = nz;
  for (int64_t r = 0; r < n_ranks; ++r) {
    if (k_bounds[r + 1] <= k_bounds[r]) {
      bands[2 * r] = 0;
      bands[2 * r + 1] = 0;
      continue;
    }
    slab_vrange(mats_host, np, nh, nw, nx, ny, nz, variant, k_bounds[r], k_bounds[r + 1], &bands[2 * r],
                &bands[2 * r + 1]);
  }
  return CBP_OK;
}

int cbp_forward_project_f32(const float* vol_dev, int64_t nx, int64_t ny, int64_t nz, double voxel_size,
                            const double* views_host, int64_t np, int64_t nh, int64_t nw, double pixel_pitch_u,
                            double pixel_pitch_v, double cu, double cv, float* out_dev, void* cuda_stream) {
  if (!vol_dev || !views_host || !out_dev) return fail(CBP_EINVAL, "null buffer");
  if (nx < 2 || ny < 2 || nz < 2 || np < 1 || nh < 1 || nw < 1 || !(voxel_size > 0))
    return fail(CBP_EINVAL, "forward projection needs a volume of at least 2x2x2 and a positive voxel size");
  int dev;
  int rc = current_device(&dev);
  if (rc) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  double* vd = nullptr;
  CK(cudaMallocAsync(reinterpret_cast<void**>(&vd), (size_t)np * 12 * sizeof(double), st), "alloc views");
  CK(cudaMemcpyAsync(vd, views_host, (size_t)np * 12 * sizeof(double), cudaMemcpyHostToDevice, st), "upload views");
  // a copy of the volume with y contiguous for the rays that run mostly along x (fwd_kernels.cuh);
  // without the memory for it every ray reads the natural layout
  float* vol_t = nullptr;
  const bool want_t = std::getenv("CBP_FWD_NATURAL_ONLY") == nullptr;  // measurement knob (tools/time_f1_f2.py)
  if (want_t && nz <= 65535 &&
      cudaMallocAsync(reinterpret_cast<void**>(&vol_t), (size_t)nx * ny * nz * sizeof(float), st) == cudaSuccess) {
    dim3 b(32, 8), g((unsigned)ceil_div(ny, 32), (unsigned)ceil_div(nx, 32), (unsigned)nz);
    // out[z][x][y] = vol[z][y][x]: the staging transpose with (u, v) = (y, x)
    stage_transposed_kernel<<<g, b, 0, st>>>(vol_dev, (int)nx, (int)ny, 0, (int)nx, vol_t, (int)ny);
  } else {
    cudaGetLastError();  // clear the failed allocation
    vol_t = nullptr;
  }
  FwdParams fp;
  fp.vol = vol_dev; fp.vol_t = vol_t; fp.views = vd; fp.out = out_dev;
  fp.np = (int)np; fp.nh = (int)nh; fp.nw = (int)nw; fp.nx = (int)nx; fp.ny = (int)ny; fp.nz = (int)nz;
  fp.pu = pixel_pitch_u; fp.pv = pixel_pitch_v; fp.cu = cu; fp.cv = cv; fp.s = voxel_size;
  const int64_t rays = np * nh * nw;
  int s_exp = 0;
  const bool pow2 = std::frexp(fp.s, &s_exp) == 0.5 && s_exp > -500 && s_exp < 500;  // 1/s exact, no over/underflow
  if (pow2)
    bp_forward_kernel<true><<<(unsigned)ceil_div(rays, 256), 256, 0, st>>>(fp);
  else
    bp_forward_kernel<false><<<(unsigned)ceil_div(rays, 256), 256, 0, st>>>(fp);
  cudaError_t e = cudaGetLastError();
  cudaFreeAsync(vd, st);
  if (vol_t) cudaFreeAsync(vol_t, st);
  if (e != cudaSuccess) return cuda_fail(e, "forward kernel launch");
  return CBP_OK;
}

}  // extern "C"

namespace {
// host tables of the fused FDK filter for one (N, tau): N-th roots of unity and the Ram-Lak
// spectrum in the digit-reversed order the forward passes leave it in (fdk.cuh)
struct FdkTables {
  std::vector<float> tw;  // N x (re, im)
  std::vector<float> hp;  // N
};
void fdk_position_frequencies(int base, int len, int c, int stride, const int* radix, std::vector<int>& freq) {
  if (len == 1) {
    freq[base] = c;
    return;
  }
  const int r = *radix, sub = len / r;
  for (int q = 0; q < r; ++q) fdk_position_frequencies(base + q * sub, sub, c + stride * q, stride * r, radix + 1, freq);
}
std::shared_ptr<const FdkTables> fdk_tables(int logn, double tau) {
  static std::mutex mu;
  static std::map<std::pair<int, double>, std::shared_ptr<const FdkTables>> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find({logn, tau});
  if (it != cache.end()) return it->second;
  if (cache.size() >= 8) cache.clear();
  const int N = 1 << logn;
  const double pi = 3.14159265358979323846;
  auto tp = std::make_shared<FdkTables>();
  FdkTables& t = *tp;
  t.tw.resize(2 * (size_t)N);
  std::vector<double> cosN(N);
  for (int k = 0; k < N; ++k) {
    cosN[k] = std::cos(2.0 * pi * (double)k / N);
    t.tw[2 * k] = (float)cosN[k];
    t.tw[2 * k + 1] = (float)(-std::sin(2.0 * pi * (double)k / N));
  }
  // exact DFT of the zero-padded spatial Ram-Lak kernel (real, even), times tau / N
  std::vector<double> H(N / 2 + 1);
  for (int k = 0; k <= N / 2; ++k) {
    double acc = 1.0 / (4.0 * tau * tau);
    for (int n = 1; n < N / 2; n += 2)
      acc += 2.0 * (-1.0 / (pi * pi * (double)n * n * tau * tau)) * cosN[(size_t)((long long)k * n % N)];
    H[k] = acc * tau / N;
  }
  int radix[16];
  const int A = fdk_radix8_passes(logn);
  for (int i = 0; i < A; ++i) radix[i] = 8;
  radix[A] = 1 << (logn - 3 * A);
  std::vector<int> freq(N);
  fdk_position_frequencies(0, N, 0, 1, radix, freq);
  t.hp.resize(N);
  for (int p = 0; p < N; ++p) {
    const int k = freq[p];
    t.hp[p] = (float)H[k <= N / 2 ? k : N - k];
  }
  cache[{logn, tau}] = tp;
  return tp;
}

template <int LOGN>
cudaError_t fdk_launch(const float* raw, const float* wtab, const float2* tw, const float* hp, int nh, int nw, int pitch,
                       long long rows, float* out, int sms, cudaStream_t st) {
  constexpr int N = 1 << LOGN;
  const size_t smem = (size_t)(N + N / 16 + 1) * sizeof(float2);
  const int threads = std::max(32, std::min(256, N / 8));
  cudaError_t e = cudaSuccess;
  if (smem > 48 * 1024)
    e = cudaFuncSetAttribute(fdk_filter_kernel<LOGN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const long long pairs = (rows + 1) / 2;
  const long long per_sm = std::max<long long>(1, std::min<long long>(2048 / threads, (200 * 1024) / (long long)smem));
  const unsigned grid = (unsigned)std::min<long long>(pairs, per_sm * sms);
  fdk_filter_kernel<LOGN><<<grid, threads, smem, st>>>(raw, wtab, tw, hp, nh, nw, pitch, rows, out);
  return cudaGetLastError();
}
}  // namespace

extern "C" {

int cbp_fdk_filter_f32(const float* raw_dev, int64_t np, int64_t nh, int64_t nw, double D, double pixel_pitch_u,
                       double pixel_pitch_v, double cu, double cv, double tau, float* out_dev, int64_t pitch,
                       void* cuda_stream) {
  if (!raw_dev || !out_dev) return fail(CBP_EINVAL, "null buffer");
  if (np < 1 || nh < 1 || nw < 2 || pitch < nw || (pitch & 3) || !(D > 0) || !(tau > 0))
    return fail(CBP_EINVAL, "invalid FDK filter arguments");
  if (nw > 4096) return fail(CBP_EINVAL, "FDK filter: detector rows longer than 4096 pixels are not supported");
  int dev;
  int rc = current_device(&dev);
  if (rc) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  int logn = 2;
  while ((1ll << logn) < 2 * nw) ++logn;
  const int N = 1 << logn;
  const std::shared_ptr<const FdkTables> tabp = fdk_tables(logn, tau);
  const FdkTables& tab = *tabp;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  float *tw = nullptr, *hp = nullptr, *wtab = nullptr;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&tw), 2 * (size_t)N * sizeof(float), st);
  if (e == cudaSuccess) e = cudaMallocAsync(reinterpret_cast<void**>(&hp), (size_t)N * sizeof(float), st);
  if (e == cudaSuccess) e = cudaMallocAsync(reinterpret_cast<void**>(&wtab), (size_t)nh * nw * sizeof(float), st);
  // pageable sources: the copies are staged before the calls return, the cache may change afterwards
  if (e == cudaSuccess) e = cudaMemcpyAsync(tw, tab.tw.data(), 2 * (size_t)N * sizeof(float), cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(hp, tab.hp.data(), (size_t)N * sizeof(float), cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) rc = cuda_fail(e, "FDK filter: tables");
  if (rc == CBP_OK) {
    dim3 b(128), g((unsigned)ceil_div(nw, 128), (unsigned)nh);
    fdk_weight_table_kernel<<<g, b, 0, st>>>((int)nh, (int)nw, D, pixel_pitch_u, pixel_pitch_v, cu, cv, wtab);
    const long long rows = (long long)np * nh;
    const float2* tw2 = reinterpret_cast<const float2*>(tw);
    switch (logn) {
#define CBP_FDK_CASE(L) \
  case L: e = fdk_launch<L>(raw_dev, wtab, tw2, hp, (int)nh, (int)nw, (int)pitch, rows, out_dev, sms, st); break;
      CBP_FDK_CASE(2) CBP_FDK_CASE(3) CBP_FDK_CASE(4) CBP_FDK_CASE(5) CBP_FDK_CASE(6) CBP_FDK_CASE(7)
      CBP_FDK_CASE(8) CBP_FDK_CASE(9) CBP_FDK_CASE(10) CBP_FDK_CASE(11) CBP_FDK_CASE(12) CBP_FDK_CASE(13)
#undef CBP_FDK_CASE
      default: e = cudaErrorInvalidValue;
    }
    if (e != cudaSuccess) rc = cuda_fail(e, "FDK filter: kernel launch");
  }
  if (tw) cudaFreeAsync(tw, st);
  if (hp) cudaFreeAsync(hp, st);
  if (wtab) cudaFreeAsync(wtab, st);
  return rc;
}

int cbp_release(void) {
  int dev;
  int rc = current_device(&dev);
  if (rc) return rc;
  std::vector<std::shared_ptr<DevBuf>> drop;  // freed after the lock (drains the device)
  std::vector<unsigned long long*> stats;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    for (auto it = g_plans.begin(); it != g_plans.end();) {
      if (it->first.device == dev) {
        drop.push_back(it->second.mats);
        it = g_plans.erase(it);
      } else {
        ++it;
      }
    }
    for (auto it = g_stats.begin(); it != g_stats.end();) {
      if (it->first.first == dev) {
        stats.push_back(it->second);
        it = g_stats.erase(it);
      } else {
        ++it;
      }
    }
  }
  drop.clear();
  CK(cudaDeviceSynchronize(), "release: device sync");
  for (auto p : stats) cudaFree(p);
  return CBP_OK;
}

int cbp_last_plan(int64_t* out9) {
  if (!out9) return fail(CBP_EINVAL, "null buffer");
  std::memcpy(out9, g_last_plan, sizeof(g_last_plan));
  return CBP_OK;
}

}  // extern "C"

// ============================================================ multi-GPU band transport
// The z-slab driver moves detector-row bands with the copy engines (cudaMemcpy3DPeerAsync
// over NVLink / NVSwitch), never with SM kernels: the root's SMs stay on its own slab.
namespace {

typedef CUresult (*GetAddressRangeFn)(CUdeviceptr*, size_t*, CUdeviceptr);
GetAddressRangeFn get_address_range() {
  static GetAddressRangeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<GetAddressRangeFn>(p);
  });
  return fn;
}

// angles [s0, s1) x rows [v0, v0+rows) of a NATURAL stack on device src_dev -> staging layout
// [s1-s0][rows][pitch] on dst_dev (copy engines; the pad columns [nw, pitch) are not written)
int copy_band(const float* img, int src_dev, int64_t nh, int64_t nw, int64_t s0, int64_t s1, int64_t v0,
              int64_t rows, float* dst, int dst_dev, int64_t pitch, cudaStream_t st) {
  cudaMemcpy3DPeerParms cp;
  std::memset(&cp, 0, sizeof(cp));
  cp.srcPtr = make_cudaPitchedPtr(const_cast<float*>(img + ((size_t)s0 * nh + v0) * nw), (size_t)nw * 4, (size_t)nw,
                                  (size_t)nh);
  cp.srcDevice = src_dev;
  cp.dstPtr = make_cudaPitchedPtr(dst, (size_t)pitch * 4, (size_t)nw, (size_t)rows);
  cp.dstDevice = dst_dev;
  cp.extent = make_cudaExtent((size_t)nw * 4, (size_t)rows, (size_t)(s1 - s0));
  CK(cudaMemcpy3DPeerAsync(&cp, st), "band copy (cudaMemcpy3DPeerAsync)");
  return CBP_OK;
}

}  // namespace

extern "C" {

int cbp_copy_band(const float* img_dev, int src_device, int64_t np, int64_t nh, int64_t nw, int64_t s0, int64_t s1,
                  int64_t v0, int64_t rows, float* dst_dev, int64_t pitch, void* cuda_stream) {
  if (!img_dev || !dst_dev) return fail(CBP_EINVAL, "null buffer");
  if (np < 1 || nh < 1 || nw < 1 || s0 < 0 || s1 > np || s0 >= s1 || v0 < 0 || rows < 1 || v0 + rows > nh ||
      pitch < nw || (pitch & 3))
    return fail(CBP_EINVAL, "invalid band copy");
  int dev;
  int rc = current_device(&dev);
  if (rc) return rc;
  if (src_device < 0) {  // the device that owns the source (local, peer or IPC-mapped memory)
    cudaPointerAttributes a;
    CK(cudaPointerGetAttributes(&a, img_dev), "cudaPointerGetAttributes(band source)");
    src_device = a.type == cudaMemoryTypeDevice ? a.device : dev;
  }
  return copy_band(img_dev, src_device, nh, nw, s0, s1, v0, rows, dst_dev, dev, pitch,
                   static_cast<cudaStream_t>(cuda_stream));
}

int cbp_ipc_export(const void* dev_ptr, void* handle64, int64_t* offset) {
  if (!dev_ptr || !handle64 || !offset) return fail(CBP_EINVAL, "null buffer");
  GetAddressRangeFn range = get_address_range();
  if (!range) return fail(CBP_ECUDA, "cuMemGetAddressRange unavailable from the driver");
  CUdeviceptr base = 0;
  size_t size = 0;
  if (range(&base, &size, reinterpret_cast<CUdeviceptr>(dev_ptr)) != CUDA_SUCCESS)
    return fail(CBP_EINVAL, "not a device allocation");
  cudaIpcMemHandle_t h;
  CK(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)), "cudaIpcGetMemHandle");
  std::memcpy(handle64, &h, sizeof(h));
  *offset = (int64_t)(reinterpret_cast<CUdeviceptr>(dev_ptr) - base);
  return CBP_OK;
}

int cbp_ipc_open(const void* handle64, int64_t offset, void** dev_ptr) {
  if (!handle64 || !dev_ptr || offset < 0) return fail(CBP_EINVAL, "null buffer");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle64, sizeof(h));
  void* base = nullptr;
  CK(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
  *dev_ptr = static_cast<char*>(base) + offset;
  return CBP_OK;
}

int cbp_ipc_close(void* dev_ptr, int64_t offset) {
  if (!dev_ptr) return fail(CBP_EINVAL, "null buffer");
  CK(cudaIpcCloseMemHandle(static_cast<char*>(dev_ptr) - offset), "cudaIpcCloseMemHandle");
  return CBP_OK;
}

int cbp_backproject_multi(const float* img_dev, int64_t np, int64_t nh, int64_t nw, const float* mats_host,
                          float* const* slab_dev, int64_t nx, int64_t ny, int64_t nz, const int64_t* k_bounds,
                          int n_gpus, const int* devices, int variant, unsigned flags, int64_t n_chunks,
                          int64_t* stats5) {
  int rc = check_dims(np, nh, nw, nx, ny, nz);
  if (rc) return rc;
  if (!img_dev || !mats_host || !slab_dev || !k_bounds || !devices || n_gpus < 1)
    return fail(CBP_EINVAL, "null buffer or no devices");
  if (variant < 0 || variant > 5) return fail(CBP_EINVAL, "unknown kernel variant");
  if (v_mirror(variant) && (nz & 1)) return fail(CBP_EINVAL, "symmetry kernels need an even nz");
  if (k_bounds[0] != 0 || k_bounds[n_gpus] != nz) return fail(CBP_EINVAL, "k_bounds must span [0, nz]");
  for (int r = 0; r < n_gpus; ++r) {
    if (k_bounds[r + 1] < k_bounds[r]) return fail(CBP_EINVAL, "k_bounds must be non-decreasing");
    if (k_bounds[r + 1] > k_bounds[r] && !slab_dev[r]) return fail(CBP_EINVAL, "null slab buffer");
  }
  if (!mats_finite(mats_host, np * 12)) return fail(CBP_EINVAL, "projection matrices contain non-finite values");
  if (stats5)
    for (int q = 0; q < 5; ++q) stats5[q] = 0;
  if (samples_nothing(nh, nw)) return CBP_OK;
  int caller_dev;
  rc = current_device(&caller_dev);
  if (rc) return rc;
  n_chunks = std::max<int64_t>(1, std::min<int64_t>(n_chunks <= 0 ? 8 : n_chunks, np));
  const int root = devices[0];
  const int64_t pitch = cbp_staged_pitch(nw);
  const bool root_direct = (nw & 3) == 0;  // rank 0 reads the NATURAL stack in place

  struct Rank {
    int dev = -1;
    int64_t k0 = 0, k1 = 0, v0 = 0, rows = 0, cap = 0;
    cudaStream_t copy = nullptr, comp = nullptr;
    cudaEvent_t copied[2] = {nullptr, nullptr}, done[2] = {nullptr, nullptr};
    float* buf[2] = {nullptr, nullptr};
    ScopedStats stats;
  };
  std::vector<Rank> R((size_t)n_gpus);
  auto fin = [&](int code) {
    for (auto& r : R) {
      if (r.dev < 0) continue;
      cudaSetDevice(r.dev);
      if (r.comp) cudaStreamSynchronize(r.comp);
      if (r.copy) cudaStreamSynchronize(r.copy);
      r.stats.release(r.comp);
      for (int b = 0; b < 2; ++b)
        if (r.buf[b]) cudaFreeAsync(r.buf[b], r.comp);
      if (r.comp) cudaStreamSynchronize(r.comp);
      for (int b = 0; b < 2; ++b) {
        if (r.copied[b]) cudaEventDestroy(r.copied[b]);
        if (r.done[b]) cudaEventDestroy(r.done[b]);
      }
      if (r.copy) cudaStreamDestroy(r.copy);
      if (r.comp) cudaStreamDestroy(r.comp);
    }
    cudaSetDevice(caller_dev);
    return code;
  };
  // prior work on every participating device (the projections on the root, zeroed or
  // accumulated slabs elsewhere) lands before the first copy or launch: the call is a
  // synchronous whole-job entry point
  for (int r = 0; r < n_gpus; ++r) {
    CK(cudaSetDevice(devices[r]), "cudaSetDevice");
    CK(cudaDeviceSynchronize(), "multi: device sync");
  }
  for (int r = 0; r < n_gpus; ++r) {
    Rank& q = R[(size_t)r];
    q.dev = devices[r];
    q.k0 = k_bounds[r];
    q.k1 = k_bounds[r + 1];
    if (q.k1 <= q.k0) continue;
    slab_vrange(mats_host, np, nh, nw, nx, ny, nz, variant, q.k0, q.k1, &q.v0, &q.rows);
    if (q.rows == 0) continue;
    cudaError_t e = cudaSetDevice(q.dev);
    if (e == cudaSuccess && q.dev != root) {
      int can = 0;
      cudaDeviceCanAccessPeer(&can, q.dev, root);
      if (can) {
        cudaError_t pe = cudaDeviceEnablePeerAccess(root, 0);
        if (pe == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
      }
    }
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&q.comp, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&q.copy, cudaStreamNonBlocking);
    for (int b = 0; b < 2 && e == cudaSuccess; ++b) {
      e = cudaEventCreateWithFlags(&q.copied[b], cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&q.done[b], cudaEventDisableTiming);
    }
    if (e != cudaSuccess) return fin(cuda_fail(e, "multi: stream/event setup"));
    keep_pool_warm(q.dev);
    if ((rc = q.stats.alloc(q.comp))) return fin(rc);
    if (!(r == 0 && root_direct)) {
      q.cap = ceil_div(np, n_chunks);
      for (int b = 0; b < 2 && e == cudaSuccess; ++b) {
        const size_t bytes = (size_t)q.cap * q.rows * pitch * 4;
        e = cudaMallocAsync(reinterpret_cast<void**>(&q.buf[b]), bytes, q.comp);
        if (e == cudaSuccess) e = cudaMemsetAsync(q.buf[b], 0, bytes, q.comp);  // pad columns stay zero
      }
      if (e == cudaSuccess) e = cudaEventRecord(q.done[0], q.comp);  // buffers ready for the first copies
      if (e == cudaSuccess) e = cudaEventRecord(q.done[1], q.comp);
      if (e != cudaSuccess) return fin(cuda_fail(e, "multi: band buffers"));
    }
  }
  // chunk c of every rank before chunk c+1 of any: copy c+1 overlaps compute c
  for (int64_t c = 0; c < n_chunks; ++c) {
    const int64_t s0 = np * c / n_chunks, s1 = np * (c + 1) / n_chunks;
    const int b = (int)(c & 1);
    for (int r = 0; r < n_gpus; ++r) {
      Rank& q = R[(size_t)r];
      if (q.k1 <= q.k0 || q.rows == 0) continue;
      CK(cudaSetDevice(q.dev), "cudaSetDevice");
      StagedCall call{img_dev, nw, np, nh, nw, 0, nh, mats_host, slab_dev[r], CBP_NATURAL, nx, ny, q.k1 - q.k0, q.k0,
                      nz, s0, s1, 0, np, variant, flags};
      if (q.buf[0]) {
        cudaError_t e = cudaStreamWaitEvent(q.copy, q.done[b], 0);  // compute c-2 released the buffer
        if (e != cudaSuccess) return fin(cuda_fail(e, "multi: wait"));
        if ((rc = copy_band(img_dev, root, nh, nw, s0, s1, q.v0, q.rows, q.buf[b], q.dev, pitch, q.copy)))
          return fin(rc);
        e = cudaEventRecord(q.copied[b], q.copy);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(q.comp, q.copied[b], 0);
        if (e != cudaSuccess) return fin(cuda_fail(e, "multi: events"));
        call.staged = q.buf[b];
        call.pitch = pitch;
        call.band_v0 = q.v0;
        call.band_rows = q.rows;
        call.s_base = s0;
        call.n_staged = s1 - s0;
      }
      if ((rc = launch_staged(call, q.stats.d, q.comp))) return fin(rc);
      if (q.buf[0]) {
        cudaError_t e = cudaEventRecord(q.done[b], q.comp);
        if (e != cudaSuccess) return fin(cuda_fail(e, "multi: events"));
      }
    }
  }
  for (auto& q : R) {
    if (q.k1 <= q.k0 || q.rows == 0) continue;
    CK(cudaSetDevice(q.dev), "cudaSetDevice");
    int64_t st5[5] = {0, 0, 0, 0, 0};
    const int rr = read_stats(q.stats.d, q.comp, st5);
    if (stats5)
      for (int k = 0; k < 5; ++k) stats5[k] += st5[k];
    if (rr && !rc) rc = rr;
  }
  return fin(rc);
}

}  // extern "C"
