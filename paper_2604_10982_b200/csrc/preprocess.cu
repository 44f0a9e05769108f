// preprocess.cu — K1: per-surfel 2DGS ray-splat transform, culls, screen box
// and tile count (reference: project_surfel, proj/src/raster.cpp:94-142, plus
// the hot-record build raster.cpp:321-353 and the box of bin_boxes 51-68).
//
// One thread per surfel, source order. All decision arithmetic is fp64 with
// the reference's (Eigen's) operation order and no FMA contraction (this file
// is compiled with --fmad=false), so culls, boxes and the records the blend
// kernel decides on are bit-identical to the CPU oracle.
#include "psm_device.cuh"
#include "psm_ellipse.h"
#include "psm_kernels.h"
#include "psm_project.cuh"

namespace psm {
namespace {

// Adds one to the counter of every tile the surfel is binned to (bin_boxes,
// raster.cpp:59-74; Ellipse extension in psm_ellipse.h): the per-tile bucket sizes
// of the counting sort that replaces the reference's per-tile push_back. Each tile
// has kSplit sub-counters (sub-bucket = lane), laid out split-major, so the atomics
// of a hot tile (10k entries near the camera) spread over kSplit addresses.
__device__ __forceinline__ void count_tiles(const BinRec& b, double cx, double cy, const DevRaster& rs, int img_h,
                                            uint32_t* __restrict__ tile_counts) {
  if (b.tx0 > b.tx1 || b.ty0 > b.ty1) return;
  const bool ellipse = rs.binning == PSM_BIN_ELLIPSE;
  PsmEllipse e;
  if (ellipse) e = psm_ellipse_prep(cx, cy, b.F00, b.F01, b.F11, rs.chi2);
  for (int ty = b.ty0; ty <= b.ty1; ++ty) {
    int lo = b.tx0, hi = b.tx1;
    if (ellipse && !psm_ellipse_row(e, ty, rs.tile_size, img_h, b.tx0, b.tx1, &lo, &hi)) continue;
    uint32_t* row = tile_counts + static_cast<int64_t>(threadIdx.x & (kSplit - 1)) * rs.tiles_x * rs.tiles_y +
                    ty * rs.tiles_x;
    for (int tx = lo; tx <= hi; ++tx) atomicAdd(row + tx, 1u);
  }
}

// One surfel; returns whether it projects (then *db = its depth bit pattern).
__device__ __forceinline__ bool project_one(int64_t i, const double* __restrict__ s, DevCamera cam, DevRaster rs,
                                            SurfRec* __restrict__ recs, BinRec* __restrict__ bins,
                                            uint64_t* __restrict__ depth_bits, uint32_t* __restrict__ tile_counts,
                                            int32_t* __restrict__ valid, uint64_t* db, int32_t* __restrict__ err) {
  valid[i] = 0;
  ProjFull pf;
  const int st = psm_project(s, cam, rs.chi2, pf);
  if (st < 0) atomicOr(err, 1);  // the reference throws std::invalid_argument here
  if (st != 1) return false;

  SurfRec rec;
#pragma unroll
  for (int k = 0; k < 9; ++k) rec.h[k] = pf.h[k];
  // footprint_inv = adj(F) / det F (raster.cpp:132-136)
  rec.cx = pf.cx;
  rec.cy = pf.cy;
  rec.f00 = pf.F11 / pf.fdet;
  rec.f01x2 = 2.0 * (-pf.F01 / pf.fdet);
  rec.f11 = pf.F00 / pf.fdet;
  rec.opacity = s[9];
  rec.color[0] = static_cast<float>(s[10]);
  rec.color[1] = static_cast<float>(s[11]);
  rec.color[2] = static_cast<float>(s[12]);
  rec.normal[0] = static_cast<float>(pf.sgn * pf.r02);
  rec.normal[1] = static_cast<float>(pf.sgn * pf.r12);
  rec.normal[2] = static_cast<float>(pf.sgn * pf.r22);
  recs[i] = rec;

  // binning box (circle_box or aabb_box), tile rectangle (raster.cpp:60-68)
  BinRec b;
  b.F00 = pf.F00; b.F01 = pf.F01; b.F11 = pf.F11;
  double x0 = pf.cx - pf.rad, x1 = pf.cx + pf.rad, y0 = pf.cy - pf.rad, y1 = pf.cy + pf.rad;
  if (rs.binning != PSM_BIN_CIRCLE) {
    const double dx = sqrt(rs.chi2 * pf.F00), dy = sqrt(rs.chi2 * pf.F11);
    x0 = pf.cx - dx; x1 = pf.cx + dx; y0 = pf.cy - dy; y1 = pf.cy + dy;
  }
  const int ts = rs.tile_size;  // floor(x / ts) as raster.cpp:62-65 (exact reciprocal for 16)
  b.tx0 = max(x86_cvt(floor(psm_div_tile(x0, ts))), 0);
  b.tx1 = min(x86_cvt(floor(psm_div_tile(x1, ts))), rs.tiles_x - 1);
  b.ty0 = max(x86_cvt(floor(psm_div_tile(y0, ts))), 0);
  b.ty1 = min(x86_cvt(floor(psm_div_tile(y1, ts))), rs.tiles_y - 1);
  const uint64_t bits = static_cast<uint64_t>(__double_as_longlong(pf.pc2));
  b.cx = pf.cx;
  b.cy = pf.cy;
  b.depth_bits = bits;
  bins[i] = b;
  depth_bits[i] = bits;
#ifndef PSM_PRE_NOCOUNT
  count_tiles(b, pf.cx, pf.cy, rs, cam.h, tile_counts);
#endif
  valid[i] = 1;
  *db = bits;
  return true;
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }
// TMA bulk copy (cp.async.bulk, 1-D) with mbarrier completion (PTX ISA 8.0, sm_90+)
__device__ __forceinline__ unsigned smem_addr(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_addr(bar)));
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra W;\n}\n" ::"r"(smem_addr(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
               ::"r"(smem_addr(dst)), "l"(src), "r"(bytes), "r"(smem_addr(bar)) : "memory");
}
// Batch staging: PSM_PRE_TMA = 1: a full 32-surfel batch (3328 contiguous bytes) is one bulk
// copy issued by lane 0 through the TMA unit, completing on the buffer's mbarrier; the
// partial last batch takes the per-lane cp.async path. 0: every batch by cp.async (seven
// 16-byte LDGSTS per lane). Measured equal (C3 preprocess 0.1218 vs 0.1221 ms, C4 0.507 vs
// 0.508): the kernel is bound by its fp64 chains, not by the staging's issue slots.
#ifndef PSM_PRE_TMA
#define PSM_PRE_TMA 1
#endif
#ifndef PSM_PRE_WARPS
#define PSM_PRE_WARPS 8
#endif
constexpr int kPreWarps = PSM_PRE_WARPS;
constexpr int kPreStage = 2 * kPreWarps * 32 * 13 * static_cast<int>(sizeof(double));  // 53,248 B at 8 warps
constexpr int kPreSmem = kPreStage + 2 * kPreWarps * static_cast<int>(sizeof(uint64_t));  // + the mbarriers

// 2 CTAs per SM (126 registers, no spills) with the batch prefetch: C3 preprocess 0.130 ->
// 0.120 ms, C4 0.552 -> 0.505 ms; at 3 CTAs the persistent loop spills (0.150 ms)
#ifndef PSM_PRE_MINB
#define PSM_PRE_MINB 2
#endif
__global__ void __launch_bounds__(32 * kPreWarps, PSM_PRE_MINB) preprocess_kernel(const double* __restrict__ surfels13, int64_t n,
                                                          DevCamera cam, DevRaster rs, SurfRec* __restrict__ recs,
                                                          BinRec* __restrict__ bins,
                                                          uint64_t* __restrict__ depth_bits,
                                                          uint32_t* __restrict__ tile_counts,
                                                          int32_t* __restrict__ valid, uint32_t* __restrict__ n_proj,
                                                          unsigned long long* __restrict__ depth_minmax,
                                                          int32_t* __restrict__ err) {
  // Persistent: each warp walks 32-surfel batches (grid stride); a batch's 32 x 104 B
  // (contiguous) are staged through shared memory with coalesced 16-byte cp.async, the
  // next batch's copies in flight while this one is projected.
  extern __shared__ __align__(16) double stage[];  // [2][8 warps][32 * 13], then [8 warps][2] mbarriers
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t n_batches = (n + 31) / 32, stride = static_cast<int64_t>(gridDim.x) * kPreWarps;
  uint64_t* bars = reinterpret_cast<uint64_t*>(stage + 2 * kPreWarps * 32 * 13) + 2 * w;
  unsigned phase = 0, bulk = 0;  // per buffer: mbarrier parity; whether its batch went by bulk copy
  if (PSM_PRE_TMA && lane == 0) {
    mbar_init(bars);
    mbar_init(bars + 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncwarp();
  auto issue = [&](int64_t bt, int buf) {
    bulk &= ~(1u << buf);
    if (bt < n_batches) {
      const int64_t w0 = bt * 32;
      const int nw = static_cast<int>(n - w0 < 32 ? n - w0 : 32);
      const double* src = surfels13 + 13 * w0;
      double* dst = stage + (buf * kPreWarps + w) * (32 * 13);
      if (PSM_PRE_TMA && nw == 32) {
        if (lane == 0) {
          // the warp's generic-proxy reads of this buffer (two batches ago) precede the
          // async-proxy writes of the copy
          asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
          mbar_arrive_tx(bars + buf, 32 * 13 * sizeof(double));
          bulk_g2s(dst, src, 32 * 13 * sizeof(double), bars + buf);
        }
        bulk |= 1u << buf;
      } else {
        const int nv = (13 * nw) / 2;  // whole 16-byte pairs (13 * 32 is even)
#pragma unroll
        for (int k = 0; k < 7; ++k) {
          const int v = lane + 32 * k;
          if (v < nv) cp_async16(dst + 2 * v, src + 2 * v);
        }
        if ((13 * nw) % 2 && lane == 0) cp_async8(dst + 13 * nw - 1, src + 13 * nw - 1);
      }
    }
    cp_async_commit();
  };
  unsigned long long lo = ~0ull, hi = 0ull;
  uint32_t n_ok = 0;
  int buf = 0;
  int64_t bt = static_cast<int64_t>(blockIdx.x) * kPreWarps + w;
  issue(bt, 0);
  for (; bt < n_batches; bt += stride, buf ^= 1) {
    issue(bt + stride, buf ^ 1);
    if (bulk >> buf & 1u) {  // this buffer's batch came by bulk copy
      mbar_wait(bars + buf, (phase >> buf) & 1u);
      phase ^= 1u << buf;
    } else {
      cp_async_wait<1>();
    }
    __syncwarp();
    const int64_t i = bt * 32 + lane;
    uint64_t db = 0;
    const bool ok = i < n && project_one(i, stage + (buf * kPreWarps + w) * (32 * 13) + 13 * lane, cam, rs, recs, bins, depth_bits,
                                         tile_counts, valid, &db, err);
    if (ok) {
      lo = db < lo ? db : lo;
      hi = db > hi ? db : hi;
      ++n_ok;
    }
    __syncwarp();  // the buffer is refilled two batches later
  }
  cp_async_wait<0>();
  // a bulk copy issued for a batch past the end is never issued (bt < n_batches), so no
  // mbarrier phase is left pending when the warp exits
  // n_proj and the frame's depth bit range (sort keys, binning.cu): a full-warp reduction
  // with identities for culled lanes, one atomic each per warp
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long l2 = __shfl_xor_sync(0xffffffffu, lo, o), h2 = __shfl_xor_sync(0xffffffffu, hi, o);
    lo = l2 < lo ? l2 : lo;
    hi = h2 > hi ? h2 : hi;
    n_ok += __shfl_xor_sync(0xffffffffu, n_ok, o);
  }
  if (lane == 0 && n_ok) {
    atomicAdd(n_proj, n_ok);
    atomicMin(depth_minmax, lo);
    atomicMax(depth_minmax + 1, hi);
  }
}

// Per-frame reset in one launch (instead of three memsets and a host-to-device copy):
// the 16 frame counters, the per-tile ranges, the split tile counters, and the depth
// range's (min, max) identities.
__global__ void frame_init_kernel(unsigned long long* __restrict__ small, int32_t* __restrict__ ranges, int n_ranges,
                                  uint32_t* __restrict__ tcounts, int n_counts,
                                  unsigned long long* __restrict__ dminmax) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x, stride = gridDim.x * blockDim.x;
  if (t < 16) small[t] = 0ull;
  if (dminmax && t < 2) dminmax[t] = t == 0 ? ~0ull : 0ull;
  for (int i = t; i < n_ranges; i += stride) ranges[i] = 0;
  for (int i = t; i < n_counts; i += stride) tcounts[i] = 0u;
}

}  // namespace

void launch_frame_init(unsigned long long* small, int32_t* ranges, int n_ranges, uint32_t* tcounts, int n_counts,
                       unsigned long long* dminmax, cudaStream_t stream) {
  const int work = n_ranges > n_counts ? n_ranges : n_counts;
  int blocks = (work + 255) / 256;
  blocks = blocks < 1 ? 1 : (blocks > 1184 ? 1184 : blocks);
  frame_init_kernel<<<blocks, 256, 0, stream>>>(small, ranges, n_ranges, tcounts, n_counts, dminmax);
}

void launch_preprocess(const double* surfels13, int64_t n, const DevCamera& cam, const DevRaster& rs, SurfRec* recs,
                       BinRec* bins, uint64_t* depth_bits, uint32_t* tile_counts, int32_t* valid,
                       uint32_t* n_proj, unsigned long long* depth_minmax, int32_t* err, cudaStream_t stream) {
  if (n <= 0) return;
  // persistent: every resident CTA, or fewer when the scene is smaller
  static int per_sm[64] = {}, sms[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!per_sm[dev]) {
    cudaDeviceGetAttribute(&sms[dev], cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(preprocess_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kPreSmem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[dev], preprocess_kernel, 32 * kPreWarps, kPreSmem);
    if (per_sm[dev] < 1) per_sm[dev] = 1;
  }
  const int64_t need = (n + 32 * kPreWarps - 1) / (32 * kPreWarps);
  const int64_t resident = static_cast<int64_t>(per_sm[dev]) * sms[dev];
  const int64_t blocks = need < resident ? need : resident;
  preprocess_kernel<<<static_cast<unsigned>(blocks), 32 * kPreWarps, kPreSmem, stream>>>(surfels13, n, cam, rs, recs, bins, depth_bits,
                                                                       tile_counts, valid, n_proj, depth_minmax, err);
}

}  // namespace psm
