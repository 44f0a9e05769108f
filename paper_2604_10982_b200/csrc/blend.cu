// blend.cu — K7: tile-based front-to-back compositing with register Top-K and
// warp-cooperative feature accumulation (reference: the tile loop of
// render_into, proj/src/raster.cpp:355-506, and topk_select, raster.cpp:225-251).
//
// One CTA per 16x16 tile (8 warps), one thread per pixel; each warp owns an 8x4
// pixel block (compact footprint: fewer lanes idle in the accept path) and
// streams the tile's depth-sorted list (vals[start, end) from the tile sort) on
// its own: 32 records (144 B SurfRec each, nine 16 B cp.async per lane) per
// chunk, double-buffered in shared memory, with no CTA-wide barrier. A warp
// stops reading the list as soon as all its 32 pixels have hit T < t_min.
// Each pixel walks the list in order with the reference's fp64 arithmetic
// (compiled --fmad=false; psm_exp_nonpos), so its contributor sequence,
// transmittance and Top-K set are bit-identical to the oracle's.
//
// Colour and normal are accumulated in fp32 from the fp64 weight (one
// conversion per contributor; |error| <= ~1e-6, inside the 1e-4 tolerance);
// expected depth, the dominant-weight pick and all decisions stay fp64.
//
// Top-K: each thread keeps its k_sel best (weight desc, source asc) entries sorted in
// shared memory (slot-major) by insertion, with only the admission threshold in
// registers (the reference's insertion select, raster.cpp:238-249; proj order ==
// source order). Selection only changes the result when m > K, as in the reference
// (raster.cpp:442).
// Features: after compositing, each warp walks its 32 pixels; the owning lane's
// (source, weight) slots are broadcast with __shfl_sync and the 32 lanes read the
// selected surfel's feature row as one coalesced 128-512 B vector load and
// accumulate VEC*NV channels each, then store the pixel's HWC channel run with
// one coalesced vector store. Full blending with features keeps per-pixel
// (source, weight) lists in an L2-resident global scratch.
#include <algorithm>
#include <cstdint>

#include "psm_device.cuh"
#include "psm_exp.h"
#include "psm_kernels.h"

namespace psm {
namespace {

constexpr int kTile = 16;
constexpr int kBlocks = 8;  // 8x4 pixel blocks (work items) per 16x16 tile
constexpr int kRecVec = sizeof(SurfRec) / 16;  // 9

// Kernel shape per Top-K width: records per warp chunk (double-buffered) and resident
// CTAs per SM. Shared memory per CTA = 8 warps x 2 x chunk x 144 B of staged records
// + the 2 KB exp table + the per-pixel Top-K lists (KMAX x 12 B per pixel); the
// chunk is the largest that fits the residency (228 KB per SM, 1 KB reserved per
// CTA) and the registers stay under 65536 / (256 x blocks).
#ifndef PSM_BLEND_CH8
#define PSM_BLEND_CH8 16
#endif
#ifndef PSM_BLEND_MB8
#define PSM_BLEND_MB8 3
#endif
#ifndef PSM_BLEND_CH16
#define PSM_BLEND_CH16 10
#endif
#ifndef PSM_BLEND_MB16
#define PSM_BLEND_MB16 3
#endif
#ifndef PSM_BLEND_CH32
#define PSM_BLEND_CH32 5
#endif
#ifndef PSM_BLEND_MB32
#define PSM_BLEND_MB32 2
#endif
#ifndef PSM_BLEND_CH0
#define PSM_BLEND_CH0 30
#endif
#ifndef PSM_BLEND_W8
#define PSM_BLEND_W8 8
#endif
#ifndef PSM_BLEND_W16
#define PSM_BLEND_W16 8
#endif
#ifndef PSM_BLEND_W32
#define PSM_BLEND_W32 8
#endif
// candidate records per alpha-phase iteration
#ifndef PSM_BLEND_PER
#define PSM_BLEND_PER 1
#endif
// lanes that walk one need mask together: 1, 2 (the default: two
// horizontally adjacent pixels), 4 (a 4x1 row), 8 (4x2) or 16 (4x4). C3 blend:
// 0.812 / 0.809 / 0.834 / 0.841 / 0.875 ms
#ifndef PSM_BLEND_GROUP
#define PSM_BLEND_GROUP 2
#endif
// warps per CTA (each pulls its own work items; the count only sets residency and registers)
__host__ __device__ constexpr int cta_warps(int kmax) {
  return kmax == 0 ? 8 : (kmax <= 8 ? PSM_BLEND_W8 : (kmax <= 16 ? PSM_BLEND_W16 : PSM_BLEND_W32));
}
__host__ __device__ constexpr int cta_threads(int kmax) { return 32 * cta_warps(kmax); }
__host__ __device__ constexpr int chunk_for(int kmax) {
  return kmax == 0 ? PSM_BLEND_CH0 : (kmax <= 8 ? PSM_BLEND_CH8 : (kmax <= 16 ? PSM_BLEND_CH16 : PSM_BLEND_CH32));
}
__host__ __device__ constexpr int min_blocks(int kmax) {
  return kmax == 0 ? 3 : (kmax <= 8 ? PSM_BLEND_MB8 : (kmax <= 16 ? PSM_BLEND_MB16 : PSM_BLEND_MB32));
}

#ifdef PSM_BLEND_STATS
// Instrumented build only (scratch profiling): work counters of the candidate loop.
__device__ unsigned long long psm_blend_stats[16];
#define PSM_STAT(i, v) atomicAdd(&psm_blend_stats[i], static_cast<unsigned long long>(v))
#endif

constexpr size_t kExpTabBytes = 256 * sizeof(uint64_t);
__host__ __device__ constexpr size_t align16(size_t b) { return (b + 15) / 16 * 16; }
// Staging copies: PSM_BLEND_TMA = 0 (the default): nine 16 B cp.async per 144 B record,
// issued by the lane that found the entry; 1: one bulk copy (cp.async.bulk through the TMA
// unit) per record, completing on the buffer's mbarrier (expect_tx per record, one arrival
// per chunk). Measured (r02g, C3 blend): 0.806 ms with cp.async vs 0.854 ms with bulk
// copies (C4 2.97 vs 3.16 ms): the records are gathered by source id, so each bulk copy
// moves only 144 B, and the per-copy mbarrier traffic outweighs the 8 LDGSTS it saves.
#ifndef PSM_BLEND_TMA
#define PSM_BLEND_TMA 0
#endif
// per warp: [2][chunk] staged records + [2][chunk] their list positions + [2][chunk] their
// source ids (16 B aligned) + the two buffers' mbarriers
__host__ __device__ constexpr size_t warp_stage_bytes(int kmax) {
  return align16(2 * chunk_for(kmax) * (sizeof(SurfRec) + 2 * sizeof(int))) + 16;
}
__host__ __device__ constexpr size_t stage_bytes(int kmax) {
  return static_cast<size_t>(cta_warps(kmax)) * warp_stage_bytes(kmax);
}
__host__ __device__ constexpr size_t smem_bytes(int kmax) {
  return stage_bytes(kmax) + kExpTabBytes + static_cast<size_t>(kmax) * cta_threads(kmax) * (sizeof(double) + sizeof(int));
}
static_assert(smem_bytes(0) * 3 + 1024 * 3 <= 228 * 1024, "full-blend shape exceeds shared memory");
static_assert(smem_bytes(8) * PSM_BLEND_MB8 + 1024 * PSM_BLEND_MB8 <= 228 * 1024, "K=8 shape exceeds shared memory");
static_assert(smem_bytes(16) * PSM_BLEND_MB16 + 1024 * PSM_BLEND_MB16 <= 228 * 1024, "K=16 shape exceeds shared memory");
static_assert(smem_bytes(32) * PSM_BLEND_MB32 + 1024 * PSM_BLEND_MB32 <= 228 * 1024, "K=32 shape exceeds shared memory");
static_assert(PSM_BLEND_CH0 <= 32 && PSM_BLEND_CH8 <= 32 && PSM_BLEND_CH16 <= 32 && PSM_BLEND_CH32 <= 32,
              "chunks are 32-bit masks");

// before(a, b) of topk_select (raster.cpp:232-235), proj order == source order.
// Slots hold list positions; the source ids are only looked up on an exact weight tie.
__device__ __forceinline__ bool before(double wa, int pa, double wb, int pb, const uint32_t* __restrict__ vals) {
  return wa > wb || (wa == wb && __ldg(vals + pa) < __ldg(vals + pb));
}
// The same order when the slots hold source ids (the Top-K renders, see kSrcSlots): no loads.
__device__ __forceinline__ bool before_src(double wa, int sa, double wb, int sb) {
  return wa > wb || (wa == wb && sa < sb);
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
// mbarrier + bulk-copy primitives (PTX ISA 8.0, sm_90+)
__device__ __forceinline__ unsigned smem_u32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra W;\n}\n" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_copy_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// Feature vector type per lane: VEC consecutive floats.
template <int VEC> struct FVec;
template <> struct FVec<1> { using T = float; };
template <> struct FVec<2> { using T = float2; };
template <> struct FVec<4> { using T = float4; };

template <int VEC>
__device__ __forceinline__ void fma_vec(float (&acc)[VEC], float w, const typename FVec<VEC>::T& v) {
  if constexpr (VEC == 1) {
    acc[0] = fmaf(w, v, acc[0]);
  } else if constexpr (VEC == 2) {
    acc[0] = fmaf(w, v.x, acc[0]);
    acc[1] = fmaf(w, v.y, acc[1]);
  } else {
    acc[0] = fmaf(w, v.x, acc[0]);
    acc[1] = fmaf(w, v.y, acc[1]);
    acc[2] = fmaf(w, v.z, acc[2]);
    acc[3] = fmaf(w, v.w, acc[3]);
  }
}

// Accumulates one feature row into the lane's VEC*NV channels:
// channel(e, v) = (v * 32 + lane) * VEC + e. EXACT: D == 32 * VEC * NV (no guards).
template <int VEC, int NV, bool EXACT>
__device__ __forceinline__ void accumulate_row(float (&acc)[NV][VEC], float w, const float* __restrict__ row, int lane,
                                               int D) {
  using T = typename FVec<VEC>::T;
  const T* r = reinterpret_cast<const T*>(row);
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    const int idx = v * 32 + lane;
    if (EXACT || idx * VEC < D) fma_vec<VEC>(acc[v], w, __ldg(r + idx));
  }
}

// Lane -> pixel of an 8x4 block: lanes 0-15 cover the left 4x4 half, lanes 16-31 the
// right one (row-major inside each half), so aligned lane groups of 2, 4, 8 and 16 are
// compact pixel groups that walk only the records their own pixels need (PSM_BLEND_GROUP).
__device__ __forceinline__ int blk_px(int q) { return (q & 3) | ((q >> 4) << 2); }
__device__ __forceinline__ int blk_py(int q) { return (q >> 2) & 3; }

// One warp's work item: the 8x4 pixel block `blk` (0..7) of tile `tile`; lane -> pixel.
template <int KMAX, bool FULL_LIST, int VEC, int NV, int LPP, bool EXACT, int PANO_T>
__device__ __forceinline__ void blend_block(const BlendParams& p, const int tile, const int blk, SurfRec* stage,
                                            const uint64_t* exp_tab, double* top_w, int* top_p, unsigned& phase) {
  constexpr int kChunk = chunk_for(KMAX);
  constexpr int kCT = cta_threads(KMAX);  // Top-K column stride
  constexpr int kPer = PSM_BLEND_PER;     // candidate records evaluated per iteration
  const int tx = tile % p.tiles_x, ty = tile / p.tiles_x;
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int wx0 = tx * kTile + (blk & 1) * 8, wy0 = ty * kTile + (blk >> 1) * 4;
  const int x = wx0 + blk_px(lane);
  const int y = wy0 + blk_py(lane);
  const bool inside = x < p.width && y < p.height;
  const int64_t pix = static_cast<int64_t>(y) * p.width + x;

  const double px = x + 0.5, py = y + 0.5;
  const double rx = (px - p.cam_cx) / p.cam_fx;  // division as in raster.cpp:370-371
  const double ry = (py - p.cam_cy) / p.cam_fy;

  double T = 1.0;
  int m = 0;
  bool done = !inside;
  float acc_r = 0.f, acc_g = 0.f, acc_b = 0.f, nx = 0.f, ny = 0.f, nz = 0.f;
  double exp_depth = 0, dom_w = 0;
  float dom_depth = 0.f;  // rcp of the strictly-first maximum weight (the plane is fp32)
  // Top-K: the k_sel best (weight desc, source asc) so far live in shared memory; the
  // registers only hold the admission threshold (the k_sel-th entry).
  const int klen = p.k_sel < 1 ? 1 : p.k_sel;
  int n_top = 0;  // filled entries
  double thr_w = -1.0;  // weights are > 0: the first k_sel contributors always enter
  int thr_p = 0;        // list position; never compared while thr_w < 0

  const int start = p.ranges[2 * tile], end = p.ranges[2 * tile + 1];
  // this pixel's list entry m is lists[lbase + lstride m]: block-major for the backward
  // cache (psm_list_index), pixel-major for the Full-mode feature phase
  const bool cache_lists = p.lists_t != nullptr;
  const int64_t lbase = !FULL_LIST ? 0 : (cache_lists ? psm_list_index(x, y, p.width, p.list_cap, 0) : pix * p.list_cap);
  const int lstride = cache_lists ? 32 : 1;
  int* spos = reinterpret_cast<int*>(stage + 2 * kChunk);  // [2][kChunk] list positions of the staged records
  int* ssrc = spos + 2 * kChunk;                           // [2][kChunk] their source ids
  // Top-K slots hold source ids (ties compare them directly, the feature phase reads them
  // as they are) unless list positions are needed later: the backward cache's selected
  // positions (FULL_LIST) and the panoptic phase's blend-order re-sort (PANO_T).
  constexpr bool kSrcSlots = !FULL_LIST && PANO_T == 0;
  uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<char*>(stage) + warp_stage_bytes(KMAX) - 16);
  unsigned pending = 0;  // buffers with a bulk-copy phase not yet waited on
  // The tile list is read in 32-entry windows (source id + warp-block mask per lane, the
  // next window's loads in flight); the entries whose mask has this warp's block bit
  // are compacted into chunks of kChunk staged records (cp.async by the owning lane).
  const unsigned bbit = 1u << blk;
  const unsigned lt_mask = (1u << lane) - 1u;
  int wb = start;
  uint32_t cv = 0;
  unsigned nm = 0;  // the next window's mask byte
  unsigned cm = 0;
  if (start + lane < end) {
    cv = __ldg(p.vals + start + lane);
    cm = __ldg(p.masks + start + lane);
  }
  if (start + 32 + lane < end) nm = __ldg(p.masks + start + 32 + lane);
  unsigned clive = __ballot_sync(0xffffffffu, start + lane < end && (cm & bbit));
  if (!p.support_cutoff) clive = __ballot_sync(0xffffffffu, start + lane < end);
  // Stages the next (up to) kChunk live entries into buffer `bf`; returns how many.
  auto assemble = [&](int bf) -> int {
    int filled = 0;
    for (;;) {
      if (!clive) {
        if (wb + 32 >= end) break;
        wb += 32;
        clive = __ballot_sync(0xffffffffu, wb + lane < end && (!p.support_cutoff || (nm & bbit)));
        cv = (clive >> lane & 1u) ? __ldg(p.vals + wb + lane) : 0u;
        const int nxt = wb + 32 + lane;
        if (nxt < end) nm = __ldg(p.masks + nxt);
        continue;
      }
      const int r = __popc(clive & lt_mask);
      const bool mine = (clive >> lane & 1u) && r < kChunk - filled;
      const unsigned take = __ballot_sync(0xffffffffu, mine);
      if (mine) {
        const char* g = reinterpret_cast<const char*>(p.recs + cv);
        char* d = reinterpret_cast<char*>(stage + bf * kChunk + filled + r);
#if PSM_BLEND_TMA
        mbar_expect_tx(bars + bf, sizeof(SurfRec));
        bulk_copy_g2s(d, g, sizeof(SurfRec), bars + bf);
#else
#pragma unroll
        for (int k = 0; k < kRecVec; ++k) cp_async16(d + 16 * k, g + 16 * k);
#endif
        spos[bf * kChunk + filled + r] = wb + lane;
        if constexpr (kSrcSlots) ssrc[bf * kChunk + filled + r] = static_cast<int>(cv);
      }
      filled += __popc(take);
      clive &= ~take;
      if (filled == kChunk) break;
    }
#if PSM_BLEND_TMA
    __syncwarp();  // every lane's expect_tx precedes the arrival that closes the phase
    if (lane == 0) mbar_arrive(bars + bf);
    pending |= 1u << bf;
#else
    cp_async_commit();
#endif
    return filled;
  };
  // waits until buffer bf's staged records have landed
  auto land = [&](int bf) {
#if PSM_BLEND_TMA
    mbar_wait(bars + bf, (phase >> bf) & 1u);
    phase ^= 1u << bf;
    pending &= ~(1u << bf);
#else
    (void)bf;
    cp_async_wait<1>();
#endif
  };

#ifdef PSM_BLEND_STATS
  unsigned st_iter = 0, st_sup = 0, st_alpha = 0, st_chunks = 0, st_streamed = 0, st_live = 0, st_any_sup = 0;
#endif
  int cnt = __any_sync(0xffffffffu, !done) ? assemble(0) : 0;
  int buf = 0;
  while (cnt > 0) {
    if (__all_sync(0xffffffffu, done)) break;
    const int ncnt = assemble(buf ^ 1);  // always commits one (possibly empty) group / phase
    land(buf);
    __syncwarp();
    const SurfRec* recs = stage + buf * kChunk;
#ifdef PSM_BLEND_STATS
    st_chunks++;
    st_live += cnt;
    st_streamed = end - start;
#endif
    // Support phase (raster.cpp:375-382): bit j of `sup` = staged entry j passes this
    // pixel's support test; `need` = the entries some pixel of the warp needs.
    unsigned sup = 0;
    if (!done) {
      if (p.support_cutoff) {
        for (int j = 0; j < cnt; ++j) {
          const SurfRec& r = recs[j];
          const double dx = px - r.cx;
          const double dy = py - r.cy;
          if (!(r.f00 * dx * dx + r.f01x2 * dx * dy + r.f11 * dy * dy > p.chi2)) sup |= 1u << j;  // raster.cpp:379
        }
      } else {
        sup = cnt >= 32 ? 0xffffffffu : (1u << cnt) - 1u;
      }
    }
    // Each lane group (PSM_BLEND_GROUP lanes) walks the entries its own pixels need, one
    // per iteration; groups read different staged records in the same iteration (the
    // warp iterates max over groups instead of the union of the block's needs: at C3 the
    // union is 137 records per 8x4 block, a 4x2 group's maximum 118, a 4x1 row's 115).
#if PSM_BLEND_GROUP <= 8
    unsigned need = sup;  // OR over the lane group (8 lanes: a 4x2 pixel group; 4: a 4x1 row)
#pragma unroll
    for (int o = 1; o < PSM_BLEND_GROUP; o <<= 1) need |= __shfl_xor_sync(0xffffffffu, need, o);
    int iters = (static_cast<int>(__reduce_max_sync(0xffffffffu, static_cast<unsigned>(__popc(need)))) + kPer - 1) / kPer;
#else
    const unsigned need_lo = __reduce_or_sync(0xffffffffu, lane < 16 ? sup : 0u);
    const unsigned need_hi = __reduce_or_sync(0xffffffffu, lane < 16 ? 0u : sup);
    unsigned need = lane < 16 ? need_lo : need_hi;
    int iters = (max(__popc(need_lo), __popc(need_hi)) + kPer - 1) / kPer;
#endif
#ifdef PSM_BLEND_STATS
    st_sup += __popc(sup);
    st_iter += kPer * iters;
    {
      const unsigned full = __reduce_or_sync(0xffffffffu, sup);
      unsigned q = sup;  // OR over the quarter-warp (4x2 pixels)
      q |= __shfl_xor_sync(0xffffffffu, q, 1);
      q |= __shfl_xor_sync(0xffffffffu, q, 2);
      const unsigned r4 = q;  // 4 lanes = 4x1 row
      q |= __shfl_xor_sync(0xffffffffu, q, 4);
      int mq = __popc(q), m4 = __popc(r4);
      for (int o = 16; o > 0; o >>= 1) {
        mq = max(mq, __shfl_xor_sync(0xffffffffu, mq, o));
        m4 = max(m4, __shfl_xor_sync(0xffffffffu, m4, o));
      }
      const unsigned cmask = cnt >= 32 ? 0xffffffffu : (1u << cnt) - 1u;
      const bool none_done = !__any_sync(0xffffffffu, done && inside);
      if (lane == 0) {
        PSM_STAT(13, __popc(~full & cmask));
        if (none_done) PSM_STAT(14, __popc(~full & cmask));
        PSM_STAT(15, none_done ? cnt : 0);
        PSM_STAT(9, __popc(full));
        PSM_STAT(10, kPer * iters);
        PSM_STAT(11, mq);
        PSM_STAT(12, m4);
      }
    }
#endif
    // Alpha phase: the needed entries kPer at a time (independent homography / division /
    // exp chains in flight), then composited in list order.
    for (; iters > 0; --iters) {
      int jj[kPer];
      bool hh[kPer];
#pragma unroll
      for (int c = 0; c < kPer; ++c) {
        hh[c] = need != 0u;
        jj[c] = hh[c] ? __ffs(need) - 1 : 0;
        need &= need - 1;
      }
      double al[kPer], rc[kPer], xs[kPer];
      bool ok[kPer];
      bool main_ok = true;
#pragma unroll
      for (int c = 0; c < kPer; ++c) {
        const SurfRec& r = recs[jj[c]];
        const double w0 = r.h[0] * rx + r.h[1] * ry + r.h[2];
        const double w1 = r.h[3] * rx + r.h[4] * ry + r.h[5];
        const double w2 = r.h[6] * rx + r.h[7] * ry + r.h[8];
        rc[c] = 1.0 / w2;
        const double u = w0 * rc[c], v = w1 * rc[c];
        xs[c] = -0.5 * (u * u + v * v);
        al[c] = psm_exp_main(xs[c], exp_tab);
        main_ok = main_ok && psm_exp_main_ok(xs[c]);
        // (w2 > 1e-14, raster.cpp:386-387)
        ok[c] = !done && hh[c] && (sup >> jj[c] & 1u) && (w2 > 1e-14);
      }
      if (!main_ok) {  // one branch for the rare special ranges of every chain
#pragma unroll
        for (int c = 0; c < kPer; ++c)
          if (!psm_exp_main_ok(xs[c])) al[c] = psm_exp_t(xs[c], exp_tab);
      }
#pragma unroll
      for (int c = 0; c < kPer; ++c) {
        al[c] = recs[jj[c]].opacity * al[c];
        ok[c] = ok[c] && !(al[c] < p.alpha_min || al[c] <= 0.0);  // raster.cpp:391
      }
#pragma unroll
      for (int c = 0; c < kPer; ++c) {
        if (!ok[c] || done) continue;
        const SurfRec& r = recs[jj[c]];
        const double alpha = al[c];
        const double rcp = rc[c];
        const int j = jj[c];
#ifdef PSM_BLEND_STATS
        st_alpha++;
#endif
        const double wt = alpha * T;
        // colour / depth / normal always over the full list (raster.cpp:405-436)
        const float wf = static_cast<float>(wt);
        acc_r = fmaf(wf, r.color[0], acc_r);
        acc_g = fmaf(wf, r.color[1], acc_g);
        acc_b = fmaf(wf, r.color[2], acc_b);
        nx = fmaf(wf, r.normal[0], nx);
        ny = fmaf(wf, r.normal[1], ny);
        nz = fmaf(wf, r.normal[2], nz);
        exp_depth += wt * rcp;
        if (wt > dom_w) {
          dom_w = wt;
          dom_depth = static_cast<float>(rcp);
        }
        if constexpr (KMAX > 0 || FULL_LIST) {
          const int pos = spos[buf * kChunk + j];  // list position; source id = vals[pos]
          if constexpr (KMAX > 0) {
            // insertion select (raster.cpp:238-249); below the threshold weight (the common
            // case once the list is full) one compare decides
            auto bef = [&](double wa, int ka, double wb, int kb) {
              if constexpr (kSrcSlots) return before_src(wa, ka, wb, kb);
              else return before(wa, ka, wb, kb, p.vals);
            };
            if (wt >= thr_w && bef(wt, kSrcSlots ? ssrc[buf * kChunk + j] : pos, thr_w, thr_p)) {
              const int key = kSrcSlots ? ssrc[buf * kChunk + j] : pos;
              int i = n_top < klen ? n_top++ : klen - 1;  // the list fills without a threshold
              while (i > 0) {
                const double w = top_w[(i - 1) * kCT + tid];
                const int q = top_p[(i - 1) * kCT + tid];
                if (!bef(wt, key, w, q)) break;
                top_w[i * kCT + tid] = w;
                top_p[i * kCT + tid] = q;
                --i;
              }
              top_w[i * kCT + tid] = wt;
              top_p[i * kCT + tid] = key;
              if (n_top == klen) {
                thr_w = top_w[(klen - 1) * kCT + tid];
                thr_p = top_p[(klen - 1) * kCT + tid];
              }
            }
          }
          if constexpr (FULL_LIST) {
            if (m < p.list_cap) {
              const int64_t li = lbase + static_cast<int64_t>(lstride) * m;
              p.lists[li] = make_uint2(static_cast<uint32_t>(pos), __float_as_uint(wf));
              if constexpr (PANO_T > 0) p.lists_w[li] = wt;
              if (p.lists_t) p.lists_t[li] = T;  // backward cache: T before this blend
            }
          }
        }
        T *= 1.0 - alpha;
        ++m;
        if (T < p.t_min) done = true;
      }
      if (__all_sync(0xffffffffu, done)) break;
    }
    __syncwarp();  // the buffer is refilled by the next iteration's assemble
    buf ^= 1;
    cnt = ncnt;
  }
#if PSM_BLEND_TMA
  for (int bf = 0; bf < 2; ++bf)  // drain: the staging is rewritten by the next item
    if (pending >> bf & 1u) land(bf);
#else
  cp_async_wait<0>();
#endif
#ifdef PSM_BLEND_STATS
  {
    unsigned mx = st_iter;
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    PSM_STAT(0, st_iter);
    PSM_STAT(1, st_sup);
    PSM_STAT(2, st_alpha);
    PSM_STAT(6, st_any_sup);
    if (lane == 0) {
      PSM_STAT(3, mx);
      PSM_STAT(4, st_chunks);
      PSM_STAT(5, st_streamed);
      PSM_STAT(7, st_live);
      PSM_STAT(8, 1);
    }
  }
#endif

  const int k_sel = p.k_sel;
  int blend_n = m;
  if constexpr (KMAX > 0) blend_n = m < k_sel ? m : k_sel;
  if (inside) {
    p.color[pix * 3 + 0] = acc_r + static_cast<float>(T * p.bg0);
    p.color[pix * 3 + 1] = acc_g + static_cast<float>(T * p.bg1);
    p.color[pix * 3 + 2] = acc_b + static_cast<float>(T * p.bg2);
    const bool rdn = p.render_depth_normal != 0;
    p.depth[pix * 2 + 0] = rdn ? static_cast<float>(exp_depth) : 0.f;
    p.depth[pix * 2 + 1] = rdn ? dom_depth : 0.f;
    p.normal[pix * 3 + 0] = rdn ? nx : 0.f;
    p.normal[pix * 3 + 1] = rdn ? ny : 0.f;
    p.normal[pix * 3 + 2] = rdn ? nz : 0.f;
    p.alpha_acc[pix] = static_cast<float>(1.0 - T);
    p.blend_count[pix] = m;
    if constexpr (KMAX > 0) {
      if (p.topk_dbg) {
        for (int i = 0; i < k_sel; ++i)
          p.topk_dbg[pix * k_sel + i] =
              i < blend_n ? (kSrcSlots ? top_p[i * kCT + tid] : static_cast<int>(__ldg(p.vals + top_p[i * kCT + tid])))
                          : -1;
      }
    }
    if constexpr (FULL_LIST) {
      if (m > p.list_cap) atomicMax(p.list_overflow, m);
      if constexpr (KMAX > 0) {  // backward cache: the selected list positions
        if (p.topk_pos)
          for (int i = 0; i < blend_n; ++i) p.topk_pos[pix * k_sel + i] = top_p[i * kCT + tid];
      }
    }
    // ins_argmax stays -1 unless labels were accumulated (raster.cpp:292,497); the fp64
    // feature phase (PANO_T > 0) writes it itself
    if (PANO_T == 0 && (p.n_q == 0 || blend_n == 0 || NV == 0)) p.ins_argmax[pix] = -1;
  }

  // blended_total (raster.cpp:459,502,506): one atomic per warp
  {
    unsigned long long bl = inside ? static_cast<unsigned long long>(blend_n) : 0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) bl += __shfl_xor_sync(0xffffffffu, bl, o);
    if (lane == 0 && bl) atomicAdd(p.blended_total, bl);
  }

  // ---- feature / label planes (raster.cpp:456-499), warp-cooperative.
  // LPP lanes serve one pixel (VEC*NV channels each), 32/LPP pixels per iteration:
  // channel(e, v) = (v * LPP + sub) * VEC + e, so a pixel's run is one coalesced
  // LPP*VEC*4-byte load per selected surfel and one such store.
  if constexpr (NV > 0) {
    constexpr int PPI = 32 / LPP;
    const int D = EXACT ? LPP * VEC * NV : p.feat_dims;  // EXACT shapes: the width is the shape's
    const int grp = lane / LPP, sub = lane % LPP;
    if constexpr (KMAX > 0) {
      // each lane resolves its own selected slots once: (source id, fp32 weight) pairs
      // over the slot's weight cell, read back below with one 8-byte load per row
      int2* slot = reinterpret_cast<int2*>(top_w);
      for (int i = 0; i < blend_n; ++i) {
        const int s = kSrcSlots ? top_p[i * kCT + tid] : static_cast<int>(__ldg(p.vals + top_p[i * kCT + tid]));
        slot[i * kCT + tid] = make_int2(s, __float_as_int(static_cast<float>(top_w[i * kCT + tid])));
      }
      __syncwarp();
    }
    const bool only_sem = p.n_q == 0;
    for (int q0 = 0; q0 < 32; q0 += PPI) {
      const int q = q0 + grp;
      const int qx = wx0 + blk_px(q), qy = wy0 + blk_py(q);
      const bool qin = qx < p.width && qy < p.height;
      if (!__any_sync(0xffffffffu, qin)) continue;
      const int64_t qpix = static_cast<int64_t>(qy) * p.width + qx;
      int nq = __shfl_sync(0xffffffffu, blend_n, q);
      if constexpr (FULL_LIST) nq = nq < p.list_cap ? nq : p.list_cap;
      if (!qin) nq = 0;
      float acc[NV][VEC];
#pragma unroll
      for (int v = 0; v < NV; ++v)
#pragma unroll
        for (int e = 0; e < VEC; ++e) acc[v][e] = 0.f;
      using TV = typename FVec<VEC>::T;
      if constexpr (KMAX > 0) {
        const int qt = (tid & ~31) + q;  // the pixel's thread: its Top-K list column
        const int2* slot = reinterpret_cast<const int2*>(top_w);
        for (int i = 0; i < nq; ++i) {
          const int2 e = slot[i * kCT + qt];
          const float w = __int_as_float(e.y);
          const TV* row = reinterpret_cast<const TV*>(
              p.feat + static_cast<uint64_t>(static_cast<uint32_t>(e.x)) * static_cast<uint32_t>(D));
#pragma unroll
          for (int v = 0; v < NV; ++v) {
            const int idx = v * LPP + sub;
            if (EXACT || idx * VEC < D) fma_vec<VEC>(acc[v], w, __ldg(row + idx));
          }
        }
      } else {
        const uint2* lst = p.lists + qpix * p.list_cap;
        for (int i = 0; i < __reduce_max_sync(0xffffffffu, static_cast<unsigned>(nq)); ++i) {
          if (i < nq) {
            const uint2 e = lst[i];
            const uint32_t src = __ldg(p.vals + e.x);
            const TV* row = reinterpret_cast<const TV*>(p.feat + static_cast<int64_t>(src) * D);
            const float w = __uint_as_float(e.y);
#pragma unroll
            for (int v = 0; v < NV; ++v) {
              const int idx = v * LPP + sub;
              if (EXACT || idx * VEC < D) fma_vec<VEC>(acc[v], w, __ldg(row + idx));
            }
          }
        }
      }
      if (only_sem) {
        if (qin && p.sem_feat) {
          TV* out = reinterpret_cast<TV*>(p.sem_feat + qpix * D);
#pragma unroll
          for (int v = 0; v < NV; ++v) {
            const int idx = v * LPP + sub;
            if (EXACT || idx * VEC < D) {
              TV val;
              float* f = reinterpret_cast<float*>(&val);
#pragma unroll
              for (int e = 0; e < VEC; ++e) f[e] = acc[v][e];  // zero when nothing blended
              out[idx] = val;
            }
          }
        }
      } else {
        float best = 0.f;
        int best_i = 0x7fffffff;
#pragma unroll
        for (int v = 0; v < NV; ++v) {
#pragma unroll
          for (int e = 0; e < VEC; ++e) {
            const int c = (v * LPP + sub) * VEC + e;
            if (qin && c < D) {
              const float val = acc[v][e];
              if (c < p.c_sem) {
                if (p.sem_feat) p.sem_feat[qpix * p.c_sem + c] = val;
              } else {
                const int qi = c - p.c_sem;
                if (p.ins_dist) p.ins_dist[qpix * p.n_q + qi] = val;
                if (best_i == 0x7fffffff || val > best || (val == best && qi < best_i)) {
                  best = val;
                  best_i = qi;
                }
              }
            }
          }
        }
        // first-max argmax across the pixel's LPP lanes (raster.cpp:492-497): ties -> lower index
#pragma unroll
        for (int o = LPP / 2; o > 0; o >>= 1) {
          const float ob = __shfl_xor_sync(0xffffffffu, best, o);
          const int oi = __shfl_xor_sync(0xffffffffu, best_i, o);
          if (oi != 0x7fffffff && (best_i == 0x7fffffff || ob > best || (ob == best && oi < best_i))) {
            best = ob;
            best_i = oi;
          }
        }
        if (sub == 0 && qin && nq > 0) p.ins_argmax[qpix] = best_i;
      }
    }
  }

  // ---- fp64 feature phase: features and labels are accumulated in fp64 over the selected
  // entries in blend order, exactly as raster.cpp:456-499 does (first entry writes, later
  // ones add; --fmad=false), so the argmaxes are the reference's. Two modes:
  //  * render_panoptic (metrics.cpp:339-369, fused; p.planes64 == 0): only the three int
  //    planes are written;
  //  * render with labels (p.planes64 == 1): the sem_feat / ins_dist planes (the fp64 sums
  //    rounded once to fp32) and the exact ins_argmax (raster.cpp:486-498).
  if constexpr (PANO_T > 0) {
    if constexpr (KMAX > 0) {  // selected entries back into blend (list position) order
      for (int i = 1; i < blend_n; ++i) {
        const int pi = top_p[i * kCT + tid];
        const double wi = top_w[i * kCT + tid];
        int j = i - 1;
        while (j >= 0 && top_p[j * kCT + tid] > pi) {
          top_p[(j + 1) * kCT + tid] = top_p[j * kCT + tid];
          top_w[(j + 1) * kCT + tid] = top_w[j * kCT + tid];
          --j;
        }
        top_p[(j + 1) * kCT + tid] = pi;
        top_w[(j + 1) * kCT + tid] = wi;
      }
      // in blend order the positions have served: each lane resolves its slots to source ids
      // (independent loads, issued back to back) so the pixel loop below reads them directly
      for (int i = 0; i < blend_n; ++i) top_p[i * kCT + tid] = static_cast<int>(__ldg(p.vals + top_p[i * kCT + tid]));
    }
    __syncwarp();
    const int D = p.feat_dims, cs = p.c_sem;
    const bool planes = p.planes64 != 0;
    // panoptic: alpha_acc < 0.5 -> void (metrics.cpp:351); planes: every pixel of the image
    const bool gate = inside && (planes || !(1.0 - T < 0.5));
    int nsel = blend_n;
    if constexpr (FULL_LIST) nsel = nsel < p.list_cap ? nsel : p.list_cap;
    // kLP lanes per pixel, 32 / kLP pixels per iteration: with at most 128 channels, two
    // pixels share the warp (8 channels per lane), which doubles the rows in flight per
    // iteration and halves the argmax reductions per pixel
    constexpr int kLP = PANO_T <= 3 ? 8 : (PANO_T <= 4 ? 16 : 32);
    constexpr int kPPI = 32 / kLP;
    constexpr int kCPL = PANO_T * 32 / kLP;  // channels per lane: c = chan(t), in pairs
    static_assert(kCPL % 2 == 0, "channel pairs");
    // lane sub holds the channel pairs 2 (sub + kLP j) + {0, 1}, j < kCPL / 2 (monotone in t)
#define PSM_PANO_CHAN(t) (2 * (sub + kLP * ((t) >> 1)) + ((t) & 1))
    const bool vec2 = (D & 1) == 0;  // even rows: 16-byte aligned pairs, one load each
    const int grp = lane / kLP, sub = lane % kLP;
    for (int q0 = 0; q0 < 32; q0 += kPPI) {
      const int q = q0 + grp;
      const int qx = wx0 + blk_px(q), qy = wy0 + blk_py(q);
      const bool qgate = __shfl_sync(0xffffffffu, gate, q);
      const int nq = __shfl_sync(0xffffffffu, nsel, q);
      const int64_t qpix = static_cast<int64_t>(qy) * p.width + qx;
      if (!qgate && sub == 0 && qx < p.width && qy < p.height && !planes) {
        p.pan_ids[qpix] = -1;
        p.pan_classes[qpix] = -1;
        p.pan_sem[qpix] = -1;
      }
      if (!__any_sync(0xffffffffu, qgate)) continue;
      double acc[kCPL];
#pragma unroll
      for (int t = 0; t < kCPL; ++t) acc[t] = 0.0;
      if constexpr (KMAX > 0) {
        // lane sub fetches slot i0 + sub's source and weight; the rows are then loaded back
        // to back and summed in blend order
        constexpr int kRound = KMAX < kLP ? KMAX : kLP;
#pragma unroll
        for (int i0 = 0; i0 < KMAX; i0 += kRound) {
          const int si = i0 + sub;
          int src = 0;
          double sw = 0.0;
          if (qgate && sub < kRound && si < nq && D > 0) {
            src = top_p[si * kCT + (tid & ~31) + q];  // resolved above
            sw = top_w[si * kCT + (tid & ~31) + q];
          }
#pragma unroll
          for (int i = 0; i < kRound; ++i) {
            const int s_i = __shfl_sync(0xffffffffu, src, grp * kLP + i);
            const double w = __shfl_sync(0xffffffffu, sw, grp * kLP + i);
            if (qgate && i0 + i < nq && D > 0) {
              const double* row = p.feat64 + static_cast<int64_t>(s_i) * D;
              const bool first = i0 + i == 0;
              if (vec2) {
#pragma unroll
                for (int j = 0; j < kCPL / 2; ++j) {
                  const int c = PSM_PANO_CHAN(2 * j);
                  if (c < D) {
                    const double2 v = __ldg(reinterpret_cast<const double2*>(row + c));
                    acc[2 * j] = first ? w * v.x : acc[2 * j] + w * v.x;
                    acc[2 * j + 1] = first ? w * v.y : acc[2 * j + 1] + w * v.y;
                  }
                }
              } else {
#pragma unroll
                for (int t = 0; t < kCPL; ++t) {
                  const int c = PSM_PANO_CHAN(t);
                  if (c < D) {
                    const double v = __ldg(row + c);
                    acc[t] = first ? w * v : acc[t] + w * v;
                  }
                }
              }
            }
          }
        }
      } else {
        const int n_all = static_cast<int>(__reduce_max_sync(0xffffffffu, static_cast<unsigned>(qgate && D > 0 ? nq : 0)));
        for (int i = 0; i < n_all; ++i) {
          if (qgate && i < nq) {
            const int pos = static_cast<int>(p.lists[qpix * p.list_cap + i].x);
            const double w = p.lists_w[qpix * p.list_cap + i];
            const double* row = p.feat64 + static_cast<int64_t>(__ldg(p.vals + pos)) * D;
#pragma unroll
            for (int t = 0; t < kCPL; ++t) {
              const int c = PSM_PANO_CHAN(t);
              if (c < D) {
                const double v = __ldg(row + c);
                acc[t] = i == 0 ? w * v : acc[t] + w * v;
              }
            }
          }
        }
      }
      // first-max argmaxes over the semantic (c < cs) and label (cs <= c < D) channels: the
      // maximum by a butterfly within the pixel's lanes, then the lowest channel holding it
      double bs = 0.0, bi = 0.0;
      bool hs = false, hi = false;
#pragma unroll
      for (int t = 0; t < kCPL; ++t) {
        const int c = PSM_PANO_CHAN(t);
        if (c < cs) {
          if (!hs || acc[t] > bs) bs = acc[t];
          hs = true;
        } else if (c < D) {
          if (!hi || acc[t] > bi) bi = acc[t];
          hi = true;
        }
      }
#pragma unroll
      for (int o = kLP / 2; o > 0; o >>= 1) {
        const double os = __shfl_xor_sync(0xffffffffu, bs, o), oi = __shfl_xor_sync(0xffffffffu, bi, o);
        const bool ohs = __shfl_xor_sync(0xffffffffu, hs, o), ohi = __shfl_xor_sync(0xffffffffu, hi, o);
        if (ohs && (!hs || os > bs)) bs = os;
        if (ohi && (!hi || oi > bi)) bi = oi;
        hs = hs || ohs;
        hi = hi || ohi;
      }
      unsigned fs = 0xffffffffu, fi = 0xffffffffu;  // this lane's lowest channel holding the maximum
#pragma unroll
      for (int t = kCPL - 1; t >= 0; --t) {
        const int c = PSM_PANO_CHAN(t);
        if (c < cs && acc[t] == bs) fs = static_cast<unsigned>(c);
        else if (c >= cs && c < D && acc[t] == bi) fi = static_cast<unsigned>(c - cs);
      }
      int ks, ki;
      if constexpr (kLP == 32) {
        ks = static_cast<int>(__reduce_min_sync(0xffffffffu, fs));
        ki = static_cast<int>(__reduce_min_sync(0xffffffffu, fi));
      } else {  // minimum within the pixel's lanes
#pragma unroll
        for (int o = kLP / 2; o > 0; o >>= 1) {
          fs = min(fs, __shfl_xor_sync(0xffffffffu, fs, o));
          fi = min(fi, __shfl_xor_sync(0xffffffffu, fi, o));
        }
        ks = static_cast<int>(fs);
        ki = static_cast<int>(fi);
      }
      if (!qgate) continue;
      if (planes) {  // raster.cpp:486-498: zeros (and -1) where nothing blended
#pragma unroll
        for (int t = 0; t < kCPL; ++t) {
          const int c = PSM_PANO_CHAN(t);
          const float v = nq > 0 ? static_cast<float>(acc[t]) : 0.f;
          if (c < cs) {
            if (p.sem_feat) p.sem_feat[qpix * cs + c] = v;
          } else if (c < D) {
            if (p.ins_dist) p.ins_dist[qpix * p.n_q + (c - cs)] = v;
          }
        }
        if (sub == 0) p.ins_argmax[qpix] = (p.n_q > 0 && nq > 0) ? ki : -1;
        continue;
      }
      if (sub == 0) {
        // ins_argmax stays -1 without labels or blends (raster.cpp:292,497); the
        // semantic plane is all zeros when nothing blended, whose first max is 0
        const int id = (p.n_q > 0 && nq > 0) ? ki : -1;
        p.pan_ids[qpix] = id;
        p.pan_classes[qpix] = (id >= 0 && id < p.n_query_class) ? __ldg(p.query_class + id) : -1;
        p.pan_sem[qpix] = cs > 0 ? (nq > 0 ? ks : 0) : -1;
      }
    }
  }
}

#undef PSM_PANO_CHAN

// Persistent CTAs (resident count per SM x SMs): each warp pulls (tile, 8x4 block) items
// from the launch's work counter until the tiles run out, so an SM's slots are never held
// by a CTA whose other warps already finished (tile depth complexity varies 10x+ across
// a frame). A warp's shared memory (staging, Top-K columns) is private to it; the exp
// table is loaded once per CTA.
template <int KMAX, bool FULL_LIST, int VEC, int NV, int LPP, bool EXACT, int PANO_T>
__global__ void __launch_bounds__(cta_threads(KMAX), min_blocks(KMAX)) blend_kernel(BlendParams p) {
  constexpr int kChunk = chunk_for(KMAX);
  constexpr int kCT = cta_threads(KMAX);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SurfRec* stage = reinterpret_cast<SurfRec*>(smem_raw + (threadIdx.x >> 5) * warp_stage_bytes(KMAX));  // [2][kChunk]
  // psm_exp's 2^(i/128) table, one copy per CTA (random per-lane lookups: shared memory, not L1)
  uint64_t* exp_tab = reinterpret_cast<uint64_t*>(smem_raw + stage_bytes(KMAX));
  // per-pixel Top-K lists (slot-major: [slot][thread], conflict-free): weights and list positions
  double* top_w = reinterpret_cast<double*>(exp_tab + 256);
  int* top_p = reinterpret_cast<int*>(top_w + KMAX * kCT);
  for (int i = threadIdx.x; i < 256; i += kCT) exp_tab[i] = psm_exp_tab_dev[i];
  unsigned phase = 0;  // parity of each staging buffer's current mbarrier phase
#if PSM_BLEND_TMA
  if ((threadIdx.x & 31) == 0) {
    uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<char*>(stage) + warp_stage_bytes(KMAX) - 16);
    mbar_init(bars, 1);
    mbar_init(bars + 1, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
#endif
  __syncthreads();
  const int n_items = p.n_tiles * kBlocks;
  for (;;) {
    int item = 0;
    if ((threadIdx.x & 31) == 0) item = atomicAdd(p.work, 1);
    item = __shfl_sync(0xffffffffu, item, 0);
    if (item >= n_items) break;
    const int tile = p.order ? __ldg(p.order + item / kBlocks) : p.tile_base + item / kBlocks;
    blend_block<KMAX, FULL_LIST, VEC, NV, LPP, EXACT, PANO_T>(p, tile, item % kBlocks, stage, exp_tab, top_w, top_p,
                                                             phase);
    __syncwarp();  // the lanes' Top-K columns and staging are rewritten by the next item
  }
}

template <int KMAX, bool FULL, int VEC, int NV, int LPP, bool EXACT, int PANO_T = 0>
void launch_t(const BlendParams& p, int tiles, cudaStream_t st) {
  auto kern = blend_kernel<KMAX, FULL, VEC, NV, LPP, EXACT, PANO_T>;
  static unsigned long long configured = 0;  // per instantiation, one bit per device
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(configured >> dev & 1ull)) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem_bytes(KMAX)));
    configured |= 1ull << dev;
  }
  static int sms[64] = {};
  if (!sms[dev]) cudaDeviceGetAttribute(&sms[dev], cudaDevAttrMultiProcessorCount, dev);
  const int grid = std::min(tiles, sms[dev] * min_blocks(KMAX));
  BlendParams q = p;
  q.n_tiles = tiles;
  kern<<<grid, cta_threads(KMAX), smem_bytes(KMAX), st>>>(q);
}

// Feature-lane shapes: float4 lanes, LPP lanes per pixel (32/LPP pixels per warp
// iteration), NV float4 per lane, for the common widths; scalar lanes with guards otherwise.
// Four float4 per lane is the widest that fits the 80-register budget (eight spill); per
// entry it amortises the slot read and the loop over four times the channels. Measured
// (blend ms): C3, D = 64: LPP 16 x NV 1 0.800, 8 x 2 0.788, 4 x 4 0.776, 2 x 8 0.822;
// C4, D = 128: 32 x 1 2.894, 16 x 2 2.814, 8 x 4 2.73, 4 x 8 3.007.
template <int KMAX, bool FULL>
void launch_feat(const BlendParams& p, int tiles, cudaStream_t st) {
  const int D = p.feat_dims;
  switch (D) {
    case 0: launch_t<KMAX, FULL, 1, 0, 32, true>(p, tiles, st); return;
    case 32: launch_t<KMAX, FULL, 4, 2, 4, true>(p, tiles, st); return;
    case 64: launch_t<KMAX, FULL, 4, 4, 4, true>(p, tiles, st); return;
    case 96: launch_t<KMAX, FULL, 4, 3, 8, true>(p, tiles, st); return;
    case 128: launch_t<KMAX, FULL, 4, 4, 8, true>(p, tiles, st); return;
    case 256: launch_t<KMAX, FULL, 4, 4, 16, true>(p, tiles, st); return;
    default: break;
  }
  const int nch = (D + 31) / 32;
  if (nch <= 2) launch_t<KMAX, FULL, 1, 2, 32, false>(p, tiles, st);
  else if (nch <= 4) launch_t<KMAX, FULL, 1, 4, 32, false>(p, tiles, st);
  else if (nch <= 8) launch_t<KMAX, FULL, 1, 8, 32, false>(p, tiles, st);
  else launch_t<KMAX, FULL, 1, 16, 32, false>(p, tiles, st);
}

// Panoptic feature phase: PANO_T = channels per lane / 32 (feat_dims <= 32 * PANO_T).
template <int KMAX, bool FULL>
void launch_pano(const BlendParams& p, int tiles, cudaStream_t st) {
  const int t = (p.feat_dims + 31) / 32;
  if (t <= 1) launch_t<KMAX, FULL, 1, 0, 32, true, 1>(p, tiles, st);
  else if (t <= 2) launch_t<KMAX, FULL, 1, 0, 32, true, 2>(p, tiles, st);
  else if (t <= 3) launch_t<KMAX, FULL, 1, 0, 32, true, 3>(p, tiles, st);
  else if (t <= 4) launch_t<KMAX, FULL, 1, 0, 32, true, 4>(p, tiles, st);
  else if (t <= 8) launch_t<KMAX, FULL, 1, 0, 32, true, 8>(p, tiles, st);
  else launch_t<KMAX, FULL, 1, 0, 32, true, 16>(p, tiles, st);
}

}  // namespace

#ifdef PSM_BLEND_STATS
extern "C" void psm_blend_stats_read(unsigned long long* out, int reset) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, psm_blend_stats, sizeof(psm_blend_stats));
  if (reset) {
    unsigned long long z[16] = {};
    cudaMemcpyToSymbol(psm_blend_stats, z, sizeof(z));
  }
}
#endif

int blend_kmax_for(int k_sel) {
  if (k_sel <= 8) return 8;
  if (k_sel <= 16) return 16;
  if (k_sel <= 32) return 32;
  return -1;
}

int blend_nch_for(int feat_dims) {
  const int c = (feat_dims + 31) / 32;
  return c <= 16 ? c : -1;
}

void launch_blend(const BlendParams& p, int tiles, bool topk, cudaStream_t st) {
  if (tiles <= 0) return;
  if (p.lists_t) {  // backward cache: contributor lists (+ Top-K positions), no feature phase
    if (!topk) launch_t<0, true, 1, 0, 32, true>(p, tiles, st);
    else if (blend_kmax_for(p.k_sel) == 8) launch_t<8, true, 1, 0, 32, true>(p, tiles, st);
    else if (blend_kmax_for(p.k_sel) == 16) launch_t<16, true, 1, 0, 32, true>(p, tiles, st);
    else launch_t<32, true, 1, 0, 32, true>(p, tiles, st);
    return;
  }
  if (p.pan_ids || p.planes64) {  // render_panoptic / render with labels: the fp64 blend-order feature phase
    if (!topk) launch_pano<0, true>(p, tiles, st);
    else if (blend_kmax_for(p.k_sel) == 8) launch_pano<8, false>(p, tiles, st);
    else if (blend_kmax_for(p.k_sel) == 16) launch_pano<16, false>(p, tiles, st);
    else launch_pano<32, false>(p, tiles, st);
    return;
  }
  if (!topk) {
    if (p.feat_dims == 0) launch_t<0, false, 1, 0, 32, true>(p, tiles, st);
    else launch_feat<0, true>(p, tiles, st);
    return;
  }
  switch (blend_kmax_for(p.k_sel)) {
    case 8: launch_feat<8, false>(p, tiles, st); break;
    case 16: launch_feat<16, false>(p, tiles, st); break;
    default: launch_feat<32, false>(p, tiles, st); break;
  }
}

}  // namespace psm
