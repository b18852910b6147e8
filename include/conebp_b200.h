/*
 * conebp_b200.h -- C ABI of libconebp_b200.so, the B200 (sm_100a) back-projection
 * library that replaces the kernel seam of the reference package `conebp`.
 *
 * The reference has no native code: its back-projection is reached through
 * Python functions that hand numpy buffers to numba kernels.  Each entry point
 * below replaces one of those seams (cited as /root/reference/<file>:<line>):
 *
 *   cbp_backproject_f32      <- conebp._kernels.baseline / transpose / share /
 *                               symmetry / subline / subline_prefetch
 *                               (pkg/src/conebp/_kernels.py:29-369), dispatched
 *                               by pkg/src/conebp/backprojector.py:159,199-206
 *   cbp_backproject_host_f32 <- conebp.backproject (backprojector.py:225-238) with
 *                               host numpy buffers: copies in, computes, copies out
 *   cbp_stage_projections    <- conebp.tensors.transpose_projections (tensors.py:138-147)
 *                               plus detector-row band extraction for z-slabs
 *   cbp_backproject_staged   <- the z-slab form of the kernel (no reference counterpart;
 *                               SURVEY.md section 8(e)): a slab [k0, k0+nz) of a volume
 *                               of nz_total slices, reading a detector-row band
 *   cbp_count_ops            <- conebp.reference.ref_baseline / ref_optimized counters
 *                               (reference.py:26-290) as exposed through count=True
 *                               (backprojector.py:153-157,193-197)
 *   cbp_backproject_window   <- the same on a chunk of angles (band buffers that hold only
 *                               angles [s_base, s_base+n_staged), multi-GPU pipelining)
 *   cbp_slab_plan            <- none in the reference: cost-balanced z-slab partition and
 *                               per-slab detector-row bands
 *   cbp_backproject_multi    <- none in the reference (its parallelism is numba prange over
 *                               z, _kernels.py:42): the single-process z-slab driver over
 *                               several devices, bands moved by the copy engines
 *   cbp_copy_band, cbp_ipc_* <- the band transport of the one-process-per-GPU driver
 *
 * Conventions
 *  - All sizes are int64_t element counts.  Buffers are C-contiguous float32.
 *  - Projection layouts: CBP_NATURAL = [np][nh][nw] (v rows, u contiguous),
 *    CBP_TRANSPOSED = [np][nw][nh] (reference Layout.TRANSPOSED, tensors.py:39-41).
 *  - Volume layouts: CBP_NATURAL = [nz][ny][nx], CBP_TRANSPOSED = [nx][ny][nz].
 *  - mats_host is np*12 float32, row-major (np,3,4) as produced by
 *    conebp.geometry.projection_matrices (geometry.py:234-242).
 *  - `variant` selects the reference rung whose float32 arithmetic is reproduced
 *    bit for bit (KernelVariant, backprojector.py:49-75).  Every variant accumulates
 *    (+=) into the volume in ascending projection order, so outputs are bitwise
 *    identical to the reference rung for any launch configuration.
 *  - Device entry points are stream-ordered and asynchronous on `cuda_stream`
 *    (a cudaStream_t, NULL = legacy default stream).  They never free caller memory
 *    and keep no pointers after return.
 *  - Return value: CBP_OK or a negative CBP_E* code; cbp_last_error() gives a
 *    thread-local message for the last failure on the calling thread.
 */
#ifndef CONEBP_B200_H
#define CONEBP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CBP_OK 0
#define CBP_EINVAL (-1)   /* invalid argument (ValueError in the Python wrapper) */
#define CBP_ECUDA (-2)    /* CUDA runtime/driver failure */
#define CBP_ENOMEM (-3)   /* device allocation failed */
#define CBP_EBAND (-4)    /* a slab sampled a detector row outside its band */
#define CBP_ENODEV (-5)   /* no CUDA device */

#define CBP_NATURAL 0
#define CBP_TRANSPOSED 1

/* KernelVariant values, backprojector.py:49-55 */
#define CBP_BASELINE 0
#define CBP_TRANSPOSE 1
#define CBP_SHARE 2
#define CBP_SYMMETRY 3
#define CBP_SUBLINE 4
#define CBP_SUBLINE_PREFETCH 5

/* flags */
#define CBP_FLAG_NAIVE 1u        /* one thread per voxel, global gathers (reference-simple GPU path) */
#define CBP_FLAG_NO_SMEM 2u      /* tiled kernel, but gather from global memory (no TMA staging) */
#define CBP_FLAG_FMA_LERP 4u     /* tolerance mode: the three lerps as FMAs (not bit-exact, see below) */
#define CBP_FLAG_CHECK 8u        /* verify every shared-memory sample against the TMA box (debug) */

/* Library version (major*10000 + minor*100 + patch). */
int cbp_version(void);
/* Thread-local description of the last error on this thread ("" if none). */
const char* cbp_last_error(void);
/* Number of visible CUDA devices (0 when none; never fails). */
int cbp_device_count(void);

/* Row pitch (in floats) of the staging layout for a detector `nw` pixels wide. */
int64_t cbp_staged_pitch(int64_t nw);

/*
 * Re-lay projections into the staging layout staged[s][r][u] = img[s][v0 + r][u]
 * for r in [0, rows), u in [0, nw); zero for u in [nw, pitch).  img_dev is
 * [np][nh][nw] (NATURAL) or [np][nw][nh] (TRANSPOSED).  The layout is the NATURAL
 * one with a 16-byte row pitch, so NATURAL inputs with nw % 4 == 0 are used in
 * place.  Replaces tensors.transpose_projections (tensors.py:138-147) for
 * TRANSPOSED inputs and extracts the detector-row band [v0, v0+rows).
 */
int cbp_stage_projections(const float* img_dev, int img_layout, int64_t np, int64_t nh,
                          int64_t nw, int64_t v0, int64_t rows, float* staged_dev,
                          int64_t pitch, void* cuda_stream);

/*
 * Drop-in kernel call: accumulate the back-projection of img_dev into vol_dev.
 * Replaces _kernels.<variant>(img, mats, vol[, ij, nb]) (_kernels.py:29-369).
 */
int cbp_backproject_f32(const float* img_dev, int64_t np, int64_t nh, int64_t nw,
                        int img_layout, const float* mats_host, float* vol_dev, int64_t nx,
                        int64_t ny, int64_t nz, int vol_layout, int variant, unsigned flags,
                        void* cuda_stream);

/*
 * z-slab kernel call on staged projections: vol_dev holds slices [k0, k0+nz) of a
 * volume with nz_total slices; staged_dev holds detector rows [band_v0,
 * band_v0+band_rows) in the staging layout [np][band_rows][pitch].  Angles
 * [s_begin, s_end) are accumulated (s_end <= 0 means np).  Detector rows outside
 * the band that a voxel would sample raise CBP_EBAND through cbp_sync_status().
 */
int cbp_backproject_staged(const float* staged_dev, int64_t pitch, int64_t np, int64_t nh,
                           int64_t nw, int64_t band_v0, int64_t band_rows,
                           const float* mats_host, float* vol_dev, int vol_layout, int64_t nx,
                           int64_t ny, int64_t nz, int64_t k0, int64_t nz_total,
                           int64_t s_begin, int64_t s_end, int variant, unsigned flags,
                           void* cuda_stream);

/*
 * cbp_backproject_staged on a buffer that holds only angles [s_base, s_base + n_staged)
 * (layout [n_staged][band_rows][pitch]); [s_begin, s_end) must lie inside that window.
 * Matrices are still the whole stack's (np x 12).  Lets a z-slab rank back-project each
 * angle chunk of its band from a small double buffer as soon as the chunk has landed.
 */
int cbp_backproject_window(const float* staged_dev, int64_t pitch, int64_t np, int64_t nh,
                           int64_t nw, int64_t band_v0, int64_t band_rows, int64_t s_base,
                           int64_t n_staged, const float* mats_host, float* vol_dev,
                           int vol_layout, int64_t nx, int64_t ny, int64_t nz, int64_t k0,
                           int64_t nz_total, int64_t s_begin, int64_t s_end, int variant,
                           unsigned flags, void* cuda_stream);

/*
 * End-to-end call on HOST buffers (pinned or pageable): copies img and vol to the
 * device, back-projects, copies vol back, synchronizes.  The numpy-facing form of
 * conebp.backproject (backprojector.py:225-238).
 */
int cbp_backproject_host_f32(const float* img_host, int64_t np, int64_t nh, int64_t nw,
                             int img_layout, const float* mats_host, float* vol_host, int64_t nx,
                             int64_t ny, int64_t nz, int vol_layout, int variant, unsigned flags);

/*
 * Synchronize `cuda_stream` and report the device-side status of every launch
 * since the previous call: returns CBP_OK or CBP_EBAND; stats (may be NULL) gets
 * [tile-angle pairs staged in smem by TMA, pairs gathered from global, pairs
 *  skipped (no voxel sampled), samples outside the slab's band, samples outside
 *  the TMA box (served from global)].
 */
int cbp_sync_status(void* cuda_stream, int64_t* stats5);

/*
 * Operation counters with the conventions of the reference's instrumented twin
 * (reference.py:26-290): out5 = [dot_ops, vol_word_accesses, proj_word_accesses,
 * interp_ops, subline_builds].  Guard-dependent terms are counted on the GPU
 * with the variant's exact coordinate arithmetic.  nb as in BatchConfig.
 */
int cbp_count_ops(const float* mats_host, int64_t np, int64_t nh, int64_t nw, int64_t nx,
                  int64_t ny, int64_t nz, int variant, int64_t nb, int64_t* out5,
                  void* cuda_stream);

/*
 * Host-only planning for the multi-GPU z-slab driver (no device needed):
 * partition nz slices into n_ranks contiguous slabs of roughly equal sampled work
 * (boundaries on multiples of `align` slices) and compute each slab's detector-row
 * band.  k_bounds gets n_ranks+1 entries; bands gets 2*n_ranks entries
 * (v0, rows) per rank, rows == 0 when the slab samples no row.
 */
int cbp_slab_plan(const float* mats_host, int64_t np, int64_t nh, int64_t nw, int64_t nx,
                  int64_t ny, int64_t nz, int variant, int64_t n_ranks, int64_t align,
                  int64_t* k_bounds, int64_t* bands);

/* Detector-row band [v0, v0+rows) sampled by slices [k0, k1) (host only). */
int cbp_slab_band(const float* mats_host, int64_t np, int64_t nh, int64_t nw, int64_t nx,
                  int64_t ny, int64_t nz, int variant, int64_t k0, int64_t k1, int64_t* v0,
                  int64_t* rows);

/*
 * Forward projection (the back-projector's adjoint): ray-driven
 * line integrals of a NATURAL float32 volume [nz][ny][nx] through every detector pixel
 * centre, trilinear samples at half-voxel steps times the step -- the float64 arithmetic
 * of conebp.phantom._forward (phantom.py:134-222), bitwise identical.  views_host is
 * np*12 doubles per projection: source xyz, detector-centre xyz, e_u xyz, e_v xyz
 * (world units); out_dev is [np][nh][nw].  Stream-ordered.
 * Replaces conebp.phantom.forward_project (phantom.py:225-252).
 */
int cbp_forward_project_f32(const float* vol_dev, int64_t nx, int64_t ny, int64_t nz,
                            double voxel_size, const double* views_host, int64_t np, int64_t nh,
                            int64_t nw, double pixel_pitch_u, double pixel_pitch_v, double cu,
                            double cv, float* out_dev, void* cuda_stream);

/*
 * FDK pre-processing (the reference has no filter step, F5):
 * cosine weighting D/sqrt(D^2 + ((u-cu)pu)^2 + ((v-cv)pv)^2) and row-wise spatial
 * Ram-Lak filtering (tau = detector pitch scaled to the isocentre) of NATURAL raw
 * projections [np][nh][nw] on the device, written into the staging layout
 * [np][nh][pitch] that cbp_backproject_staged reads.  Zero-padded FFT convolution in one
 * fused kernel (shared-memory radix-8 transform, two rows per complex transform: each row is
 * read once and written once), float32, nw <= 4096.  Stream-ordered.
 */
int cbp_fdk_filter_f32(const float* raw_dev, int64_t np, int64_t nh, int64_t nw, double D,
                       double pixel_pitch_u, double pixel_pitch_v, double cu, double cv,
                       double tau, float* out_dev, int64_t pitch, void* cuda_stream);

/*
 * Single-process multi-GPU z-slab back-projection.  img_dev is the
 * NATURAL stack [np][nh][nw] on devices[0] (the root); slab_dev[r] is the NATURAL slab
 * [k_bounds[r+1]-k_bounds[r]][ny][nx] of rank r on devices[r] (k_bounds from
 * cbp_slab_plan; devices may repeat, e.g. all 0 to run every rank on one GPU).  Each rank
 * receives only its slab's detector-row band, in n_chunks angle chunks copied by the copy
 * engines (cudaMemcpy3DPeerAsync, P2P over NVLink when peers can access each other) into a
 * double buffer, and back-projects chunk c while chunk c+1 is in flight; rank 0 reads the
 * root stack in place when nw % 4 == 0.  No reduction: every voxel has one writer
 * (_kernels.py:12-14), and chunks accumulate in ascending angle order, so the slabs are
 * bitwise identical to a single-GPU launch.  Synchronous: waits for prior work on every
 * device, returns when all slabs are complete.  stats5 (may be NULL) as cbp_sync_status,
 * summed over ranks; CBP_EBAND if any sample fell outside its band.
 */
int cbp_backproject_multi(const float* img_dev, int64_t np, int64_t nh, int64_t nw,
                          const float* mats_host, float* const* slab_dev, int64_t nx, int64_t ny,
                          int64_t nz, const int64_t* k_bounds, int n_gpus, const int* devices,
                          int variant, unsigned flags, int64_t n_chunks, int64_t* stats5);

/*
 * Copy angles [s0, s1) x detector rows [v0, v0+rows) of a NATURAL stack [np][nh][nw]
 * that lives on device src_device (-1: the current device; an IPC-mapped pointer is fine)
 * into the staging layout [s1-s0][rows][pitch] on the current device, with the copy
 * engines (no SM work), stream-ordered on cuda_stream.  Pad columns are not written.
 */
int cbp_copy_band(const float* img_dev, int src_device, int64_t np, int64_t nh, int64_t nw,
                  int64_t s0, int64_t s1, int64_t v0, int64_t rows, float* dst_dev,
                  int64_t pitch, void* cuda_stream);

/* CUDA IPC for the one-process-per-GPU driver: export a device pointer (64-byte handle of
 * its allocation plus the pointer's offset in it), map it in another process, unmap. */
int cbp_ipc_export(const void* dev_ptr, void* handle64, int64_t* offset);
int cbp_ipc_open(const void* handle64, int64_t offset, void** dev_ptr);
int cbp_ipc_close(void* dev_ptr, int64_t offset);

/* Diagnostic: count the floats with bit patterns in [lo_bits, hi_bits) whose reciprocal by
 * the kernels' branch-free rcp_rn_normal differs from __frcp_rn (IEEE 1/z); first_bad gets
 * the smallest mismatching pattern (0xffffffff if none). */
int cbp_selftest_rcp(uint32_t lo_bits, uint32_t hi_bits, uint64_t* mismatches, uint32_t* first_bad);

/* Release cached plans and device scratch owned by the library on this device. */
int cbp_release(void);

/* Diagnostics of the last plan used on this thread: [tile_x, tile_y, tile_z,
 * box_w, box_h, stages, blocks, smem_bytes, kernel_kind(0 naive,1 tiled,2 tiled-general)]. */
int cbp_last_plan(int64_t* out9);

#ifdef __cplusplus
}
#endif
#endif /* CONEBP_B200_H */
