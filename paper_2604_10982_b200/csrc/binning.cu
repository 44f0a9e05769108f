// binning.cu — K3..K6: per-tile lists of projected surfels in (sort_depth, source)
// order, RN-Total and per-tile [start, end) ranges.
//
// Reference: bin_boxes (proj/src/raster.cpp:51-90) pushes each projected index into
// every tile of its box and std::sorts every tile by (sort_depth, source)
// (raster.cpp:77-83). Here, with the per-tile bucket sizes counted by K1:
//   K3 tile_scan   one CTA: exclusive scan of the bucket sizes -> ranges, write
//                  cursors, RN-Total, non-empty tiles (the reference's
//                  rn_total / rn_per_tile, raster.cpp:84-88)
//   K4 emit        every (surfel, tile) pair claims a slot of its tile's bucket
//                  (atomic cursor; order inside a bucket is arbitrary)
//   K5 sort_tiles  one CTA per tile sorts its bucket by the total order
//                  (fp64 depth bits, source), packed into one 64-bit key, with a
//                  block merge sort (register-sorted runs, merge-path rounds in
//                  shared memory), so the result is the reference's list whatever
//                  order K4 produced. Size classes: <= 4096 entries (128 threads),
//                  <= 16384 (1024 threads), larger by a bitonic network over global memory.
// Every count stays on the device; key buffers are capacity-checked (the host
// re-renders a frame whose RN-Total outgrew them, capi.cu).
#include <algorithm>
#include <cstdint>
#include <type_traits>

#include "psm_device.cuh"
#include "psm_ellipse.h"
#include "psm_kernels.h"

namespace psm {
namespace {


// K3a: per tile, the exclusive prefix of its kSplit sub-bucket counts (the
// sub-bucket cursors, relative to the tile's start) and the tile total. Counts and
// cursors are split-major (index s * tiles + t): consecutive threads read
// consecutive tiles.
__global__ void __launch_bounds__(256) tile_sub_scan_kernel(const uint32_t* __restrict__ counts, int tiles,
                                                            uint32_t* __restrict__ cursor,
                                                            uint32_t* __restrict__ totals) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= tiles) return;
  uint32_t run = 0;
#pragma unroll 8
  for (int s = 0; s < kSplit; ++s) {
    const int64_t i = static_cast<int64_t>(s) * tiles + t;
    const uint32_t c = counts[i];
    cursor[i] = run;
    run += c;
  }
  totals[t] = run;
}

// Per-tile sort size classes (K5): 0: 1..1024 keys (128 threads), 1: ..4096 (512
// threads), 2: ..8192 and 3: ..16384 (1024 threads, 64 / 128 KB of shared memory), 4:
// beyond (chunked + global merge passes). K3b lists each class's tiles:
// classes[c * tiles + i], count at classes[kSortClasses * tiles + c]; the blend's
// heaviest-first order follows at classes[(kSortClasses + 1) * tiles + i].
__device__ __forceinline__ int sort_class(int len) {
  if (len < 1) return -1;
  if (len <= 1024) return 0;
  if (len <= 4096) return 1;
  if (len <= 8192) return 2;
  if (len <= 16384) return 3;
  return 4;
}

// 0 for the longest lists (bit length 32) .. 32 for empty ones
// The blend's heaviest-first tile order sorts tiles by list length in buckets: a power of
// two split into 2^PSM_LPT_SUB sub-buckets (C3 blend, whole powers of two 0.780 ms, 4 per
// power 0.774, 8 0.774, 16 0.774 with a longer scan; C4 2.734 / 2.728 / 2.733 / 2.735)
#ifndef PSM_LPT_SUB
#define PSM_LPT_SUB 2  // extra bits below the leading one: 2^PSM_LPT_SUB buckets per power of two
#endif
constexpr int kLptBuckets = 33 << PSM_LPT_SUB;
__device__ __forceinline__ int lpt_bucket(int len) {
  const int lz = __clz(len);
  if (PSM_LPT_SUB == 0 || len <= 0) return lz << PSM_LPT_SUB;
  const int top = 31 - lz;  // position of the leading one
  const int sub = top >= PSM_LPT_SUB ? (len >> (top - PSM_LPT_SUB)) & ((1 << PSM_LPT_SUB) - 1)
                                     : (len << (PSM_LPT_SUB - top)) & ((1 << PSM_LPT_SUB) - 1);
  return (lz << PSM_LPT_SUB) + ((1 << PSM_LPT_SUB) - 1 - sub);  // longer lists first within a power of two
}

// Slot in a shared counter bucket for every active lane, one atomic per distinct bucket
// of the warp (thousands of tiles land in the same few class / length buckets, so plain
// per-thread shared atomics serialise on them). All lanes of the warp must call it.
__device__ __forceinline__ int warp_bucket_slot(int* counters, int bucket, bool active) {
  const unsigned am = __ballot_sync(0xffffffffu, active);
  int slot = -1;
  if (active) {
    const int lane = threadIdx.x & 31;
    const unsigned peers = __match_any_sync(am, bucket);
    const int leader = __ffs(peers) - 1;
    int base = 0;
    if (lane == leader) base = atomicAdd(&counters[bucket], __popc(peers));
    base = __shfl_sync(peers, base, leader);
    slot = base + __popc(peers & ((1u << lane) - 1u));
  }
  return slot;
}

constexpr int kScanLenTiles = 16384;  // tiles whose lpt bucket K3b keeps in shared memory

// K3b: one CTA scans the tile totals: ranges, tile starts, RN-Total, non-empty tiles.
__global__ void __launch_bounds__(1024) tile_scan_kernel(const uint32_t* __restrict__ totals, int tiles, uint32_t cap,
                                                        int32_t* __restrict__ ranges, uint32_t* __restrict__ tile_start,
                                                        uint32_t* __restrict__ rn_dev, uint32_t* __restrict__ rn_eff,
                                                        unsigned long long* __restrict__ nonempty,
                                                        int32_t* __restrict__ overflow,
                                                        int32_t* __restrict__ classes) {
  __shared__ uint32_t warp_sums[32];
  __shared__ uint32_t warp_ne[32];
  __shared__ int cls_n[kSortClasses];
  __shared__ int lpt_n[kLptBuckets];
  using LptT = std::conditional_t<(kLptBuckets <= 256), uint8_t, uint16_t>;
  __shared__ LptT lpt_s[kScanLenTiles];
  if (threadIdx.x < kSortClasses) cls_n[threadIdx.x] = 0;
  for (int i = threadIdx.x; i < kLptBuckets; i += blockDim.x) lpt_n[i] = 0;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int per = (tiles + 1023) / 1024;  // consecutive tiles per thread
  const int t0 = tid * per;
  uint32_t local = 0, local_ne = 0;
  for (int j = 0; j < per; ++j) {
    const int t = t0 + j;
    if (t < tiles) {
      const uint32_t v = totals[t];
      local += v;
      local_ne += v > 0;
    }
  }
  uint32_t x = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  uint32_t ne = local_ne;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ne += __shfl_xor_sync(0xffffffffu, ne, o);
  if (lane == 31) warp_sums[warp] = x;
  if (lane == 0) warp_ne[warp] = ne;
  __syncthreads();
  uint32_t pre = 0, all = 0, all_ne = 0;
  for (int w = 0; w < 32; ++w) {
    const uint32_t sum = warp_sums[w];
    if (w < warp) pre += sum;
    all += sum;
    all_ne += warp_ne[w];
  }
  uint32_t run = pre + x - local;
  for (int j = 0; j < per; ++j) {
    const int t = t0 + j;
    int len = 0;
    if (t < tiles) {
      const uint32_t v = totals[t];
      tile_start[t] = run;
      const uint32_t b = min(run, cap), e = min(run + v, cap);
      ranges[2 * t] = static_cast<int32_t>(b);
      ranges[2 * t + 1] = static_cast<int32_t>(e);
      run += v;
      len = static_cast<int>(e - b);
      if (t < kScanLenTiles) lpt_s[t] = static_cast<LptT>(lpt_bucket(len));
    }
    const int c = t < tiles ? sort_class(len) : -1;
    const int slot = warp_bucket_slot(cls_n, c < 0 ? 0 : c, c >= 0);
    if (c >= 0) classes[c * tiles + slot] = t;
  }
  // lpt bucket of tile t (kept in shared memory for the first kScanLenTiles tiles)
  auto lpt_of = [&](int t) -> int {
    return t < kScanLenTiles ? lpt_s[t] : lpt_bucket(ranges[2 * t + 1] - ranges[2 * t]);
  };
  // Heaviest-first tile order for the blend's work items (longest-processing-time
  // scheduling by power-of-two bucket of the tile's list length): classes[5 tiles + i].
  for (int j = 0; j < per; ++j) {
    const int t = t0 + j;
    const int lb = t < tiles ? lpt_of(t) : 0;
    warp_bucket_slot(lpt_n, lb, t < tiles);
  }
  __syncthreads();
  if (warp == 0) {  // exclusive scan of the bucket counts, kPer consecutive buckets per lane
    constexpr int kPer = (kLptBuckets + 31) / 32;
    int x[kPer], sum = 0;
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int b = lane * kPer + k;
      x[k] = b < kLptBuckets ? lpt_n[b] : 0;
      sum += x[k];
    }
    int incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    int run_b = incl - sum;
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int b = lane * kPer + k;
      if (b < kLptBuckets) lpt_n[b] = run_b;
      run_b += x[k];
    }
  }
  __syncthreads();
  for (int j = 0; j < per; ++j) {
    const int t = t0 + j;
    const int lb = t < tiles ? lpt_of(t) : 0;
    const int slot = warp_bucket_slot(lpt_n, lb, t < tiles);
    if (t < tiles) classes[(kSortClasses + 1) * tiles + slot] = t;
  }
  if (tid < kSortClasses) classes[kSortClasses * tiles + tid] = cls_n[tid];
  if (tid == 0) {
    *rn_dev = all;
    *rn_eff = min(all, cap);
    *nonempty = all_ne;
    if (all > cap) atomicOr(overflow, 1);  // buckets past the capacity are dropped; the host re-renders
  }
}

// ---------------------------------------------------------------- K5 per-tile sort
// Sort key of a (surfel, tile) entry: the reference's per-tile order is
// (sort_depth, source) (raster.cpp:78-83); positive fp64 depths order as their bit
// patterns, so key = ((bits - min_bits) >> sh) << src_bits | source orders exactly
// like (depth, source) whenever sh = 0, and up to ties of the dropped low depth
// bits otherwise (fixed up after the sort). min_bits / max_bits are the frame's
// extreme depth bit patterns (K1), sh = max(0, bitlen(max - min) + src_bits - 64).
__device__ __forceinline__ int key_shift(const unsigned long long* __restrict__ depth_minmax, int src_bits) {
  const uint64_t range = depth_minmax[1] - depth_minmax[0];
  const int len = range ? 64 - __clzll(static_cast<long long>(range)) : 0;
  const int sh = len + src_bits - 64;
  return sh > 0 ? sh : 0;
}

__device__ __forceinline__ uint64_t sort_key(uint64_t bits, uint64_t src, uint64_t min_bits, int sh, int src_bits) {
  return (((bits - min_bits) >> sh) << src_bits) | src;
}

// Warp-block masks in fp32 (the blend's 8 blocks of 8x4 pixels per tile; see
// psm_block_mask for the fp64 statement). Conservative against fp32 rounding: k F11 and q
// are inflated by 2e-4 relative (so the computed half-width squared never falls below the
// true one, also at the ellipse's tips), each strip's y-range is widened by 0.1 px, and
// the x-extent carries 0.05 px + 1e-5 of the magnitudes summed. Footprints with |centre|
// or extent beyond 1e5 px keep every block.
struct StripF {
  float cx, cy, ymax, slope, dstar, kf11, q;
};
__device__ __forceinline__ float sqrt_approx(float x) {
  float r;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ bool strip_prep(const PsmEllipse& e, StripF* f) {
  if (!e.ok || !(fabs(e.cx) < 1e5) || !(fabs(e.cy) < 1e5) || !(e.ymax < 1e5) || !(e.kf11 * e.q < 1e10)) return false;
  f->cx = static_cast<float>(e.cx);
  f->cy = static_cast<float>(e.cy);
  f->kf11 = static_cast<float>(e.kf11 * 1.0002);
  f->ymax = sqrtf(f->kf11);
  f->slope = static_cast<float>(e.slope);
  f->dstar = static_cast<float>(e.dstar);
  f->q = static_cast<float>(e.q * 1.0002);
  return true;
}
// Bit b of the result: block b of tile (tx, ty) may hold a pixel centre inside the ellipse.
__device__ __forceinline__ void strips_f(const StripF& f, int ty, int height, float* sxl, float* sxr) {
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    const int y0 = ty * 16 + 4 * s;
    const int y_end = min(y0 + 4, height);
    const float dlo = fmaxf(static_cast<float>(y0) + 0.4f - f.cy, -f.ymax);
    const float dhi = fminf(static_cast<float>(y_end) - 0.4f - f.cy, f.ymax);
    const float dr = fminf(fmaxf(f.dstar, dlo), dhi);
    const float dl = fminf(fmaxf(-f.dstar, dlo), dhi);
    const float hr = sqrt_approx(fmaxf(f.kf11 - dr * dr, 0.f) * f.q);
    const float hl = sqrt_approx(fmaxf(f.kf11 - dl * dl, 0.f) * f.q);
    const float cr = f.cx + f.slope * dr, cl = f.cx + f.slope * dl;
    const float mr = 0.05f + 1e-5f * (fabsf(f.cx) + fabsf(f.slope * dr) + hr);
    const float ml = 0.05f + 1e-5f * (fabsf(f.cx) + fabsf(f.slope * dl) + hl);
    const bool ok = y_end > y0 && dlo <= dhi + 1e-3f;
    sxl[s] = ok ? cl - hl - ml : 3e38f;   // empty strip: [3e38, -3e38] meets nothing
    sxr[s] = ok ? cr + hr + mr : -3e38f;
  }
}
__device__ __forceinline__ uint32_t block_mask_f(const float* sxl, const float* sxr, int tx, int width) {
  uint32_t m = 0;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int x0 = tx * 16 + 8 * h;
    const int x_end = min(x0 + 8, width);
    const float lo = static_cast<float>(x0) + 0.5f, hi = static_cast<float>(x_end) - 0.5f;
#pragma unroll
    for (int s = 0; s < 4; ++s)
      if (x_end > x0 && sxl[s] <= hi && sxr[s] >= lo) m |= 1u << (2 * s + h);
  }
  return m;
}

// K4, load-balanced: a warp takes 32 surfels, stages each one's key and ellipse
// constants in shared memory, and then spreads the warp's (surfel, tile row) pairs over
// its lanes (a surfel covers 1..100+ tiles, so one thread per surfel leaves most lanes
// idle behind the largest footprint). Tile indices are < 2^19 (checked on the host).
struct EmitItem {
  uint64_t key;
  PsmEllipse e;
  StripF sf;
  int tx0, tx1, ty0, strips;
};
constexpr int kEmitWarps = 8;

// returning atomics in flight per thread (C3 emit, measured: 8 at 4 CTAs/SM 0.098 ms;
// 8 / 12 / 16 at 3 CTAs 0.112 / 0.113 / 0.131; 16 at 4 CTAs spills, 0.115; round 2, with
// the 64 B BinRec: 4 CTAs 0.092, 5 (48 registers, spills) 0.100, 6 (40) 0.120)
#ifndef PSM_EMIT_BATCH
#define PSM_EMIT_BATCH 8
#endif
#ifndef PSM_EMIT_MINB
#define PSM_EMIT_MINB 4
#endif
// Surfels per warp: 32 (one per lane), or fewer for small scenes, whose few warps would
// otherwise each carry 32 surfels: a warp of 32 full-image footprints (C1's ground near
// the camera) then holds the launch alone for tens of microseconds of atomic round trips
// (C1 emit: 32 surfels per warp 84 us, 8: 29 us, 4: 19.5 us, 2: 16.4 us).
#ifndef PSM_EMIT_SMALL_SPW
#define PSM_EMIT_SMALL_SPW 2
#endif
template <int SPW>
__global__ void __launch_bounds__(32 * kEmitWarps, PSM_EMIT_MINB) emit_kernel(const int32_t* __restrict__ valid, int64_t n,
                                                   const SurfRec* __restrict__ recs, const BinRec* __restrict__ bins,
                                                   DevRaster rs, int img_h, uint32_t* __restrict__ cursor,
                                                   const uint32_t* __restrict__ tile_start, uint32_t cap,
                                                   uint64_t* __restrict__ tile_keys,
                                                   const uint64_t* __restrict__ depth_bits,
                                                   const unsigned long long* __restrict__ depth_minmax, int src_bits,
                                                   int img_w) {
  __shared__ EmitItem items[kEmitWarps][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t wbase = (static_cast<int64_t>(blockIdx.x) * kEmitWarps + warp) * SPW;
  const int64_t i = wbase + lane;
  const bool ellipse = rs.binning == PSM_BIN_ELLIPSE;
  // warp-block masks need the support cutoff (a pixel only uses candidates passing it)
  const bool masks_on = rs.support_cutoff != 0;
  int rows = 0;
  if (lane < SPW && i < n && valid[i]) {
    const BinRec b = bins[i];
    if (b.tx0 <= b.tx1 && b.ty0 <= b.ty1) {
      EmitItem& it = items[warp][lane];
      // the key's source field is (source << 8 | block mask), kFieldExtra bits wider than the source
      const int fb = src_bits + kFieldExtra;
      it.key = sort_key(b.depth_bits, static_cast<uint64_t>(i) << kFieldExtra, depth_minmax[0],
                        key_shift(depth_minmax, fb), fb);
      if (ellipse || masks_on) {
        it.e = psm_ellipse_prep(b.cx, b.cy, b.F00, b.F01, b.F11, rs.chi2);
      } else {
        it.e.ok = 0;
      }
      it.strips = masks_on && strip_prep(it.e, &it.sf);
      it.tx0 = b.tx0;
      it.tx1 = b.tx1;
      it.ty0 = b.ty0;
      rows = b.ty1 - b.ty0 + 1;
    }
  }
  // exclusive prefix of the row counts over the warp
  int incl = rows;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  const int start = incl - rows;
  const int total = __shfl_sync(0xffffffffu, incl, 31);
  __syncwarp();

  // a pair's sub-bucket is source & (kSplit - 1), where K1 counted it
  const int64_t n_tiles = static_cast<int64_t>(rs.tiles_x) * rs.tiles_y;
  // tiles are claimed in batches of kBatch so several returning atomics are in flight at once
  constexpr int kBatch = PSM_EMIT_BATCH;
  uint32_t pend[kBatch];  // tile index | owner lane << 19 | block mask << 24
  int np = 0;
  auto flush = [&]() {
    uint32_t o[kBatch];
#pragma unroll
    for (int u = 0; u < kBatch; ++u)
      if (u < np) {
        const uint32_t split = (static_cast<uint32_t>(wbase) + ((pend[u] >> 19) & 31u)) & 31u;  // source & 31
        o[u] = atomicAdd(cursor + split * n_tiles + (pend[u] & 0x7ffffu), 1u);
      }
#pragma unroll
    for (int u = 0; u < kBatch; ++u)
      if (u < np) {
        const uint32_t at = __ldg(tile_start + (pend[u] & 0x7ffffu)) + o[u];
        if (at < cap) tile_keys[at] = items[warp][(pend[u] >> 19) & 31u].key | (pend[u] >> 24);
      }
    np = 0;
  };
  for (int q0 = 0; q0 < total; q0 += 32) {
    const int q = q0 + lane;
    int l = 0;  // owner: the last lane whose first pair is <= q
#pragma unroll
    for (int step = 16; step > 0; step >>= 1) {
      const int s = __shfl_sync(0xffffffffu, start, l + step);
      if (s <= q) l += step;
    }
    const int ls = __shfl_sync(0xffffffffu, start, l);
    if (q >= total) continue;
    const EmitItem& it = items[warp][l];
    const int ty = it.ty0 + (q - ls);
    int lo = it.tx0, hi = it.tx1;
    if (ellipse && !psm_ellipse_row(it.e, ty, rs.tile_size, img_h, it.tx0, it.tx1, &lo, &hi)) continue;
    float sxl[4], sxr[4];
    if (it.strips) strips_f(it.sf, ty, img_h, sxl, sxr);
    for (int tx = lo; tx <= hi; ++tx) {
      const uint32_t bm = it.strips ? block_mask_f(sxl, sxr, tx, img_w) : 0xffu;
      pend[np++] = static_cast<uint32_t>(ty * rs.tiles_x + tx) | static_cast<uint32_t>(l) << 19 | bm << 24;
      if (np == kBatch) flush();
    }
  }
  if (np) flush();
}

__device__ __forceinline__ void cmpx(uint64_t& a, uint64_t& b) {  // a <- min, b <- max
  const uint64_t lo = a < b ? a : b;
  b = a < b ? b : a;
  a = lo;
}

// Bitonic sort of n = NT * E keys (flip formulation, all ascending), keys in
// registers in blocked order (thread t holds t*E .. t*E+E-1). Partners closer than
// E are in the same thread, closer than 32E in the same warp (shuffles), the rest go
// through shared memory `sm` (n keys).
template <int NT, int E, int M, bool FLIP>
__device__ __forceinline__ void bitonic_step(uint64_t (&v)[E], uint64_t* sm, int t) {
  if constexpr (M < E) {
#pragma unroll
    for (int e = 0; e < E; ++e) {
      if ((e ^ M) > e) cmpx(v[e], v[e ^ M]);
    }
  } else if constexpr (M < 32 * E) {
    constexpr int LM = M / E;  // lane distance (flip: k/E - 1, half-cleaner: j/E)
    constexpr int TOP = FLIP ? ((LM + 1) >> 1) : LM;
    const bool lower = (t & TOP) == 0;  // this lane holds the lower index of each pair
    uint64_t w[E];
#pragma unroll
    for (int e = 0; e < E; ++e) w[e] = __shfl_xor_sync(0xffffffffu, v[FLIP ? (e ^ (E - 1)) : e], LM);
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const uint64_t mn = v[e] < w[e] ? v[e] : w[e];
      const uint64_t mx = v[e] < w[e] ? w[e] : v[e];
      v[e] = lower ? mn : mx;
    }
  } else {
    // striped layout: element (t, e) at sm[e * NT + t] (consecutive lanes, consecutive words)
    constexpr int NTH = NT;
    __syncthreads();  // previous readers of sm are done
#pragma unroll
    for (int e = 0; e < E; ++e) sm[e * NTH + t] = v[e];
    __syncthreads();
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int i = t * E + e, p = i ^ M;
      const uint64_t w = sm[(p % E) * NTH + p / E];
      const uint64_t mn = v[e] < w ? v[e] : w;
      const uint64_t mx = v[e] < w ? w : v[e];
      v[e] = i < p ? mn : mx;
    }
  }
}

template <int NT, int E, int LK, int LJ>
__device__ __forceinline__ void bitonic_stage(uint64_t (&v)[E], uint64_t* sm, int t) {
  // stage k = 2^LK, step j = 2^LJ (LJ = LK - 1 is the flip step)
  if constexpr (LJ == LK - 1) bitonic_step<NT, E, (1 << LK) - 1, true>(v, sm, t);
  else bitonic_step<NT, E, (1 << LJ), false>(v, sm, t);
  if constexpr (LJ > 0) bitonic_stage<NT, E, LK, LJ - 1>(v, sm, t);
}

template <int NT, int E, int LK, int LG>
__device__ __forceinline__ void bitonic_all(uint64_t (&v)[E], uint64_t* sm, int t) {
  bitonic_stage<NT, E, LK, LK - 1>(v, sm, t);
  if constexpr (LK < LG) bitonic_all<NT, E, LK + 1, LG>(v, sm, t);
}

__host__ __device__ constexpr int ilog2(int n) { return n <= 1 ? 0 : 1 + ilog2(n >> 1); }

// Bitonic sort of n = NT * E keys (flip formulation, all ascending), keys in
// registers in blocked order (thread t holds t*E .. t*E+E-1). Partners closer than
// E are in the same thread, closer than 32E in the same warp (shuffles), the rest go
// through shared memory `sm` (n keys). Fully unrolled at compile time.
template <int NT, int E>
__device__ void bitonic_regs(uint64_t (&v)[E], uint64_t* sm) {
  bitonic_all<NT, E, 1, ilog2(NT * E)>(v, sm, threadIdx.x);
}

// Block merge sort of n = NT * E keys (ascending; keys are unique, padding ~0):
// each thread sorts its E keys in registers, then log2(NT) rounds merge pairs of
// sorted runs through shared memory `sm` (n keys); in each round a thread finds its
// first output by a merge-path binary search and emits E outputs sequentially.
// Shared-memory slot of logical key i: XOR-swizzled within 16-key groups so the
// blocked stores (thread t writes keys tE .. tE+E-1) do not pile onto one bank.
__device__ __forceinline__ int swz(int i) { return i ^ ((i >> 4) & 15); }

template <int NT, int E>
__device__ void merge_sort_regs(uint64_t (&v)[E], uint64_t* sm) {
  constexpr int n = NT * E;
  bitonic_all<1, E, 1, ilog2(E)>(v, sm, 0);  // E keys in registers (register steps only)
  const int t = threadIdx.x;
#pragma unroll 1
  for (int width = E; width < n; width <<= 1) {
    __syncthreads();  // previous round's readers are done
#pragma unroll
    for (int e = 0; e < E; ++e) sm[swz(t * E + e)] = v[e];
    __syncthreads();
    const int out0 = t * E;
    const int base = out0 & ~(2 * width - 1);
    const int a0 = base, b0 = base + width;
    const int diag = out0 - base;
    int lo = diag > width ? diag - width : 0, hi = diag < width ? diag : width;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (sm[swz(a0 + mid)] < sm[swz(b0 + diag - 1 - mid)]) lo = mid + 1;
      else hi = mid;
    }
    int ia = lo, ib = diag - lo;
    uint64_t ka = ia < width ? sm[swz(a0 + ia)] : ~0ull, kb = ib < width ? sm[swz(b0 + ib)] : ~0ull;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const bool take_a = ka <= kb && ia < width;
      v[e] = take_a ? ka : kb;
      if (take_a) {
        ++ia;
        ka = ia < width ? sm[swz(a0 + ia)] : ~0ull;
      } else {
        ++ib;
        kb = ib < width ? sm[swz(b0 + ib)] : ~0ull;
      }
    }
  }
}

// Repair after a truncated-key sort (sh > 0): entries whose truncated depths are equal
// were ordered by source, not by (full depth, source). Each maximal run of equal
// truncated depth is insertion-sorted by the full key by the thread owning its first
// entry, all runs in parallel. Repairing a run only permutes entries of equal truncated
// depth, so concurrent readers of a run's border always see the same truncated key.
__device__ void repair_truncated_runs(uint32_t* __restrict__ vals, uint8_t* __restrict__ masks, int len,
                                      const uint64_t* __restrict__ depth_bits, uint64_t dmin, int sh) {
  for (int i = threadIdx.x; i + 1 < len; i += blockDim.x) {
    const uint64_t ti = (depth_bits[vals[i]] - dmin) >> sh;
    if (i > 0 && ((depth_bits[vals[i - 1]] - dmin) >> sh) == ti) continue;  // not a run start
    int j = i + 1;
    while (j < len && ((depth_bits[vals[j]] - dmin) >> sh) == ti) ++j;
    for (int a = i + 1; a < j; ++a) {
      const uint32_t x = vals[a];
      const uint8_t xm = masks[a];
      const uint64_t dx = depth_bits[x];
      int b = a - 1;
      while (b >= i) {
        const uint32_t y = vals[b];
        const uint64_t dy = depth_bits[y];
        if (!(dy > dx || (dy == dx && y > x))) break;
        vals[b + 1] = y;
        masks[b + 1] = masks[b];
        --b;
      }
      vals[b + 1] = x;
      masks[b + 1] = xm;
    }
  }
}

// Per-tile sort algorithm: PSM_SORT_RADIX = 0 (the default): the register + merge-path
// merge sort of the whole 64-bit keys; 1: a CTA LSD radix sort of the keys' upper 32 bits
// (four 8-bit passes, the lower 32 bits carried), then the rare runs of equal upper halves
// ordered by the full key. Measured (r02x, C3, ncu per class, isolated): the radix sort
// executes 2-2.5x fewer instructions (<1024,2>: 29.2M -> 11.7M, <128,0>: 24.4M -> 15.3M)
// but is no faster (<128,0> 45 -> 56 us, <1024,2> 76 -> 74 us; the sort stage 0.141 ->
// 0.142 ms at C3, 0.528 -> 0.572 ms at C4): its four passes are barrier- and
// latency-bound, and the big buckets' time is one CTA's, whatever the instruction count.
#ifndef PSM_SORT_RADIX
#define PSM_SORT_RADIX 0
#endif
// Shared memory of radix_sort_bucket for NT threads and n = NT * E keys: the keys' upper and
// lower halves, the per-warp 16-bit digit counters and the digit starts.
__host__ __device__ constexpr int radix_smem_bytes(int nt, int n) { return 8 * n + (nt / 32) * 256 * 2 + 256 * 4 + 16; }

// Stable CTA radix sort of the bucket's keys by their upper 32 bits. Keys are held in a
// warp-striped arrangement (key index = warp * 32 E + round * 32 + lane), ranked per
// 8-bit digit with __match_any_sync within each warp round, offset by per-warp digit counts
// (exclusive over warps, then over digits) and scattered through shared memory. After the
// four passes, runs of equal upper halves (keys whose truncated depths agree in their top
// 32 bits; rare) are ordered by the full key, so the result is the keys' total order.
// Leaves the sorted keys' halves in shared memory (upper at [0, n), lower at [n, 2n)).
template <int NT, int E>
__device__ __forceinline__ void radix_sort_bucket(const uint64_t* __restrict__ keys, int start, int len,
                                                  unsigned char* smem) {
  constexpr int kW = NT / 32;
  constexpr int kN = NT * E;
  uint32_t* s_hi = reinterpret_cast<uint32_t*>(smem);
  uint32_t* s_lo = s_hi + kN;
  uint16_t* cnt = reinterpret_cast<uint16_t*>(s_lo + kN);  // [kW][256]
  int* dstart = reinterpret_cast<int*>(cnt + kW * 256);     // [256]
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const unsigned lt = (1u << lane) - 1u;
  uint32_t hi[E], lo[E];
#pragma unroll
  for (int r = 0; r < E; ++r) {
    const int idx = w * 32 * E + r * 32 + lane;
    const uint64_t k = idx < len ? keys[start + idx] : ~0ull;
    hi[r] = static_cast<uint32_t>(k >> 32);
    lo[r] = static_cast<uint32_t>(k);
  }
#pragma unroll 1
  for (int shift = 0; shift < 32; shift += 8) {
    for (int i = tid; i < kW * 256; i += NT) cnt[i] = 0;
    __syncthreads();
    int rank[E];
#pragma unroll
    for (int r = 0; r < E; ++r) {
      const int idx = w * 32 * E + r * 32 + lane;
      const int d = idx < len ? static_cast<int>((hi[r] >> shift) & 255u) : 256;
      const unsigned peers = __match_any_sync(0xffffffffu, d);
      const int before = __popc(peers & lt);
      const int base = d < 256 ? cnt[w * 256 + d] : 0;
      __syncwarp();
      if (d < 256 && before == 0) cnt[w * 256 + d] = static_cast<uint16_t>(base + __popc(peers));
      __syncwarp();
      rank[r] = base + before;
    }
    __syncthreads();
    // per digit: exclusive offsets over warps (in place), totals -> exclusive scan over digits
    for (int d = tid; d < 256; d += NT) {
      int run = 0;
#pragma unroll
      for (int ww = 0; ww < kW; ++ww) {
        const int t = cnt[ww * 256 + d];
        cnt[ww * 256 + d] = static_cast<uint16_t>(run);
        run += t;
      }
      dstart[d] = run;
    }
    __syncthreads();
    if (w == 0) {  // exclusive scan of the 256 digit totals: 8 per lane
      int x[8], sum = 0;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        x[k] = dstart[lane * 8 + k];
        sum += x[k];
      }
      int incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      int run = incl - sum;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        dstart[lane * 8 + k] = run;
        run += x[k];
      }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < E; ++r) {
      const int idx = w * 32 * E + r * 32 + lane;
      if (idx < len) {
        const int d = static_cast<int>((hi[r] >> shift) & 255u);
        const int pos = dstart[d] + cnt[w * 256 + d] + rank[r];
        s_hi[pos] = hi[r];
        s_lo[pos] = lo[r];
      }
    }
    __syncthreads();
    if (shift < 24) {
#pragma unroll
      for (int r = 0; r < E; ++r) {
        const int idx = w * 32 * E + r * 32 + lane;
        if (idx < len) {
          hi[r] = s_hi[idx];
          lo[r] = s_lo[idx];
        }
      }
      __syncthreads();
    }
  }
  // runs of equal upper halves: ordered by the lower half (the full key), each by the
  // thread owning its first entry (runs are rare and short)
  for (int i = tid; i < len; i += NT) {
    if (i > 0 && s_hi[i - 1] == s_hi[i]) continue;  // not a run start
    int j = i + 1;
    while (j < len && s_hi[j] == s_hi[i]) ++j;
    for (int a = i + 1; a < j; ++a) {
      const uint32_t x = s_lo[a];
      int b = a - 1;
      while (b >= i && s_lo[b] > x) {
        s_lo[b + 1] = s_lo[b];
        --b;
      }
      s_lo[b + 1] = x;
    }
  }
  __syncthreads();
}

// Sorts the bucket [start, start + len) of tile keys into tile_vals (sources). After
// a truncated-key sort (sh > 0), runs of equal truncated depth are re-ordered by the
// full (depth, source) order (rare).
template <int NT, int E>
__device__ void sort_bucket(const uint64_t* __restrict__ keys, uint32_t* __restrict__ vals, uint8_t* __restrict__ masks,
                            int start, int len,
                            uint64_t* sm, const uint64_t* __restrict__ depth_bits, uint64_t dmin, int sh,
                            int src_bits) {
  const uint64_t smask = (1ull << src_bits) - 1ull;
  __shared__ int bad;
#if PSM_SORT_RADIX
  radix_sort_bucket<NT, E>(keys, start, len, reinterpret_cast<unsigned char*>(sm));
  const uint32_t* s_hi = reinterpret_cast<const uint32_t*>(sm);
  const uint32_t* s_lo = s_hi + NT * E;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < len; i += NT) {  // coalesced
    const uint64_t k = static_cast<uint64_t>(s_hi[i]) << 32 | s_lo[i];
    vals[start + i] = static_cast<uint32_t>((k & smask) >> kFieldExtra);
    masks[start + i] = static_cast<uint8_t>(k);
    // neighbours with equal truncated depth: order unknown below the dropped bits
    if (sh > 0 && i + 1 < len && (k >> src_bits) == ((static_cast<uint64_t>(s_hi[i + 1]) << 32 | s_lo[i + 1]) >> src_bits))
      bad = 1;
  }
  __syncthreads();
  if (sh > 0 && bad) repair_truncated_runs(vals + start, masks + start, len, depth_bits, dmin, sh);
#else
  uint64_t v[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int i = threadIdx.x * E + e;
    v[e] = i < len ? keys[start + i] : ~0ull;
  }
  merge_sort_regs<NT, E>(v, sm);
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int i = threadIdx.x * E + e;
    if (i < len) {
      vals[start + i] = static_cast<uint32_t>((v[e] & smask) >> kFieldExtra);
      masks[start + i] = static_cast<uint8_t>(v[e]);
      // neighbours with equal truncated depth: order unknown below the dropped bits
      if (sh > 0 && e + 1 < E && i + 1 < len && (v[e] >> src_bits) == (v[e + 1] >> src_bits)) bad = 1;
    }
  }
  if (sh > 0) {
    const int last = threadIdx.x * E + E - 1;  // pairs across thread boundaries
    sm[threadIdx.x] = v[0];
    __syncthreads();
    if (threadIdx.x + 1 < NT && last + 1 < len && (v[E - 1] >> src_bits) == (sm[threadIdx.x + 1] >> src_bits)) bad = 1;
    __syncthreads();
    if (bad) repair_truncated_runs(vals + start, masks + start, len, depth_bits, dmin, sh);
  }
#endif
}

// threads per CTA of the <= 1024-key class (E = 2, 4 or 8 keys per thread); measured:
// 256 threads make the C3 sort stage 0.142 -> 0.144 ms and C4's 0.528 -> 0.565 ms
#ifndef PSM_SORT_NT0
#define PSM_SORT_NT0 128
#endif
static_assert(PSM_SORT_NT0 * 8 >= 1024, "the <= 1024-key class needs NT * 8 >= 1024");
// NT = 128: buckets up to 2048 entries in n = 128 * E slots (E = 2 .. 16, the smallest
// that fits), 2049..4096 with E = 32; NT = 1024 (LARGE): 4097..16384 entries.
template <int NT, int CLS>
__global__ void __launch_bounds__(NT) sort_tiles_kernel(const int32_t* __restrict__ ranges,
                                                        const uint64_t* __restrict__ keys,
                                                        uint32_t* __restrict__ tile_vals,
                                                        uint8_t* __restrict__ tile_masks,
                                                        const uint64_t* __restrict__ depth_bits,
                                                        const unsigned long long* __restrict__ depth_minmax,
                                                        int src_bits, const int32_t* __restrict__ classes,
                                                        int tiles) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint64_t* sm = reinterpret_cast<uint64_t*>(smem_raw);
  const int sh = key_shift(depth_minmax, src_bits);
  const uint64_t dmin = depth_minmax[0];
  const int n_cls = classes[kSortClasses * tiles + CLS];
  for (int b = blockIdx.x; b < n_cls; b += gridDim.x) {
    const int t = classes[CLS * tiles + b];
    const int start = ranges[2 * t], len = ranges[2 * t + 1] - start;
    if (CLS == 0) {
      if (len == 1) {  // nothing to sort: unpack the key
        if (threadIdx.x == 0) {
          const uint64_t v = keys[start];
          tile_vals[start] = static_cast<uint32_t>((v & ((1ull << src_bits) - 1ull)) >> kFieldExtra);
          tile_masks[start] = static_cast<uint8_t>(v);
        }
      } else if (len <= 2 * NT) {
        sort_bucket<NT, 2>(keys, tile_vals, tile_masks, start, len, sm, depth_bits, dmin, sh, src_bits);
      } else if (len <= 4 * NT) {
        sort_bucket<NT, 4>(keys, tile_vals, tile_masks, start, len, sm, depth_bits, dmin, sh, src_bits);
      } else {
        sort_bucket<NT, 8>(keys, tile_vals, tile_masks, start, len, sm, depth_bits, dmin, sh, src_bits);
      }
    } else if (CLS == 1) {  // NT = 512
      if (len <= 2048) sort_bucket<NT, 4>(keys, tile_vals, tile_masks, start, len, sm, depth_bits, dmin, sh, src_bits);
      else sort_bucket<NT, 8>(keys, tile_vals, tile_masks, start, len, sm, depth_bits, dmin, sh, src_bits);
    } else if (CLS == 2) {
      sort_bucket<NT, 8>(keys, tile_vals, tile_masks, start, len, sm, depth_bits, dmin, sh, src_bits);
    } else {
      sort_bucket<NT, 16>(keys, tile_vals, tile_masks, start, len, sm, depth_bits, dmin, sh, src_bits);
    }
    __syncthreads();  // shared memory is reused by the next tile
  }
}

// Buckets beyond 16384 entries (C4's largest is ~17.7k): one 1024-thread CTA sorts each
// 16384-key chunk in shared memory, then merge-path passes in global memory double the
// sorted run width until the bucket is one run (ping-pong with `scratch`).
constexpr int kHugeChunk = 16384;
__device__ void sort_huge_bucket(int t, const int32_t* __restrict__ ranges, uint64_t* __restrict__ keys,
                                 uint64_t* __restrict__ scratch, uint32_t* __restrict__ tile_vals,
                                 uint8_t* __restrict__ tile_masks, const uint64_t* __restrict__ depth_bits,
                                 const unsigned long long* __restrict__ depth_minmax, int src_bits, uint64_t* sm) {
  const int start = ranges[2 * t], len = ranges[2 * t + 1] - start;
  constexpr int NT = 1024, E = kHugeChunk / NT;
  uint64_t* src = keys + start;
  uint64_t* dst = scratch + start;
  // sorted runs of kHugeChunk; the last, partial run takes the smallest sort that holds it
  // (a bucket just past 16384 keys otherwise sorts a second full 16384-slot run)
  auto sort_run = [&](auto e_tag, int c0, int cl) {
    constexpr int EE = decltype(e_tag)::value;
    uint64_t v[EE];
#pragma unroll
    for (int e = 0; e < EE; ++e) {
      const int i = threadIdx.x * EE + e;
      v[e] = i < cl ? src[c0 + i] : ~0ull;
    }
    merge_sort_regs<NT, EE>(v, sm);
#pragma unroll
    for (int e = 0; e < EE; ++e) {
      const int i = threadIdx.x * EE + e;
      if (i < cl) src[c0 + i] = v[e];
    }
    __syncthreads();
  };
  for (int c0 = 0; c0 < len; c0 += kHugeChunk) {
    const int cl = min(kHugeChunk, len - c0);
    if (cl <= 2 * NT) sort_run(std::integral_constant<int, 2>{}, c0, cl);
    else if (cl <= 4 * NT) sort_run(std::integral_constant<int, 4>{}, c0, cl);
    else if (cl <= 8 * NT) sort_run(std::integral_constant<int, 8>{}, c0, cl);
    else sort_run(std::integral_constant<int, E>{}, c0, cl);
  }
  const int per = (len + NT - 1) / NT;  // outputs per thread in each merge pass
  for (int width = kHugeChunk; width < len; width <<= 1) {
    int o = threadIdx.x * per;
    const int o_end = min(len, o + per);
    while (o < o_end) {
      const int base = (o / (2 * width)) * (2 * width);
      const int na = min(width, len - base);
      const int nb = min(width, max(0, len - base - width));
      const uint64_t* A = src + base;
      const uint64_t* B = src + base + width;
      const int diag = o - base;
      int lo = diag > nb ? diag - nb : 0, hi = diag < na ? diag : na;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (A[mid] < B[diag - 1 - mid]) lo = mid + 1;
        else hi = mid;
      }
      int ia = lo, ib = diag - lo;
      const int seg_end = min(o_end, base + 2 * width);
      for (; o < seg_end; ++o) {
        const bool take_a = ib >= nb || (ia < na && A[ia] < B[ib]);
        dst[o] = take_a ? A[ia++] : B[ib++];
      }
    }
    __syncthreads();
    uint64_t* tmp = src;
    src = dst;
    dst = tmp;
  }
  const uint64_t smask = (1ull << src_bits) - 1ull;
  const int sh = key_shift(depth_minmax, src_bits);
  __shared__ int tie;
  if (threadIdx.x == 0) tie = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < len; i += NT) {
    tile_vals[start + i] = static_cast<uint32_t>((src[i] & smask) >> kFieldExtra);
    tile_masks[start + i] = static_cast<uint8_t>(src[i]);
    if (sh > 0 && i + 1 < len && (src[i] >> src_bits) == (src[i + 1] >> src_bits)) tie = 1;
  }
  __syncthreads();
  if (tie) repair_truncated_runs(tile_vals + start, tile_masks + start, len, depth_bits, depth_minmax[0], sh);
}

__global__ void __launch_bounds__(1024) sort_tiles_huge_kernel(const int32_t* __restrict__ ranges,
                                                               uint64_t* __restrict__ keys,
                                                               uint64_t* __restrict__ scratch,
                                                               uint32_t* __restrict__ tile_vals,
                                                               uint8_t* __restrict__ tile_masks,
                                                               const uint64_t* __restrict__ depth_bits,
                                                               const unsigned long long* __restrict__ depth_minmax,
                                                               int src_bits, const int32_t* __restrict__ classes,
                                                               int tiles) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint64_t* sm = reinterpret_cast<uint64_t*>(smem_raw);
  const int n_cls = classes[kSortClasses * tiles + 4];
  for (int b = blockIdx.x; b < n_cls; b += gridDim.x) {
    sort_huge_bucket(classes[4 * tiles + b], ranges, keys, scratch, tile_vals, tile_masks, depth_bits, depth_minmax,
                     src_bits, sm);
    __syncthreads();
  }
}

__global__ void compact_kernel(const int32_t* __restrict__ valid, const int32_t* __restrict__ pos,
                               const uint64_t* __restrict__ depth_bits, int64_t n, uint64_t* __restrict__ keys_out,
                               uint32_t* __restrict__ src_out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n || !valid[i]) return;
  const int32_t o = pos[i];
  keys_out[o] = depth_bits[i];
  src_out[o] = static_cast<uint32_t>(i);
}

__global__ void rank_of_kernel(const uint32_t* __restrict__ src_by_rank, const uint32_t* __restrict__ n_proj_dev,
                               int32_t* __restrict__ rank_of) {
  const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r < *n_proj_dev) rank_of[src_by_rank[r]] = static_cast<int32_t>(r);
}

__global__ void debug_keys_kernel(const int32_t* __restrict__ ranges, const uint32_t* __restrict__ vals,
                                  const int32_t* __restrict__ rank_of, uint64_t* __restrict__ out) {
  const int t = blockIdx.x;
  const int start = ranges[2 * t], end = ranges[2 * t + 1];
  for (int i = start + threadIdx.x; i < end; i += blockDim.x)
    out[i] = (static_cast<uint64_t>(t) << 32) | static_cast<uint32_t>(rank_of[vals[i]]);
}

inline unsigned grid_for(int64_t n, int block) { return static_cast<unsigned>((n + block - 1) / block); }

}  // namespace

void launch_tile_scan(const uint32_t* tile_counts, int tiles, uint32_t cap, int32_t* ranges, uint32_t* cursor,
                      uint32_t* totals, uint32_t* tile_start, uint32_t* rn_dev, uint32_t* rn_eff,
                      unsigned long long* nonempty, int32_t* overflow, int32_t* classes, cudaStream_t st) {
  tile_sub_scan_kernel<<<grid_for(tiles, 256), 256, 0, st>>>(tile_counts, tiles, cursor, totals);
  tile_scan_kernel<<<1, 1024, 0, st>>>(totals, tiles, cap, ranges, tile_start, rn_dev, rn_eff, nonempty, overflow,
                                       classes);
}

void launch_emit(const int32_t* valid, int64_t n, const SurfRec* recs, const BinRec* bins, const DevRaster& rs,
                 int img_h, uint32_t* cursor, const uint32_t* tile_start, uint32_t cap, uint64_t* tile_keys,
                 const uint64_t* depth_bits, const unsigned long long* depth_minmax, int src_bits, int img_w,
                 cudaStream_t st) {
  if (n <= 0) return;
  // fewer than ~4 CTAs of 32-surfel warps per SM: PSM_EMIT_SMALL_SPW surfels per warp
  if (n < 148LL * 4 * kEmitWarps * 32)
    emit_kernel<PSM_EMIT_SMALL_SPW><<<grid_for(n, PSM_EMIT_SMALL_SPW * kEmitWarps), 32 * kEmitWarps, 0, st>>>(
        valid, n, recs, bins, rs, img_h, cursor, tile_start, cap, tile_keys, depth_bits, depth_minmax, src_bits, img_w);
  else
    emit_kernel<32><<<grid_for(n, 32 * kEmitWarps), 32 * kEmitWarps, 0, st>>>(
        valid, n, recs, bins, rs, img_h, cursor, tile_start, cap, tile_keys, depth_bits, depth_minmax, src_bits, img_w);
}

template <int NT, int CLS>
void launch_sort_class(const int32_t* ranges, int tiles, const uint64_t* keys, uint32_t* tile_vals,
                       uint8_t* tile_masks, const uint64_t* depth_bits, const unsigned long long* depth_minmax,
                       int src_bits, const int32_t* classes, int grid, cudaStream_t st) {
  constexpr int n_max = CLS <= 1 ? NT * 8 : CLS == 2 ? 8192 : 16384;
  constexpr int smem = PSM_SORT_RADIX ? radix_smem_bytes(NT, n_max) : static_cast<int>(sizeof(uint64_t)) * n_max;
  static unsigned long long configured = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(configured >> dev & 1ull)) {
    cudaFuncSetAttribute(sort_tiles_kernel<NT, CLS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    configured |= 1ull << dev;
  }
  sort_tiles_kernel<NT, CLS><<<std::min(grid, tiles), NT, smem, st>>>(ranges, keys, tile_vals, tile_masks, depth_bits,
                                                                     depth_minmax, src_bits, classes, tiles);
}

void launch_sort_tiles(const int32_t* ranges, int tiles, uint64_t* tile_keys, uint64_t* key_scratch, uint32_t* tile_vals,
                       uint8_t* tile_masks, const uint64_t* depth_bits, const unsigned long long* depth_minmax,
                       int src_bits, const int32_t* classes, cudaStream_t st, cudaStream_t side, cudaStream_t side2,
                       cudaEvent_t fork, cudaEvent_t join, cudaEvent_t join2) {
  if (tiles <= 0) return;
  src_bits += kFieldExtra;  // the keys' source field carries the warp-block mask below the source
  static int sms[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!sms[dev]) cudaDeviceGetAttribute(&sms[dev], cudaDevAttrMultiProcessorCount, dev);
  const int n_sm = sms[dev];
  // Persistent launches over K3b's class lists. The large classes run on two side streams,
  // concurrently with the many small buckets, which fit beside them on every SM: side:
  // the beyond-16384 buckets (1 CTA per SM) then the 8192-key class (3 CTAs per SM); side2:
  // the 16384-key class (1 CTA per SM); main: the <= 4096 then the <= 1024-key classes.
  // The few beyond-16384 buckets hold a handful of SMs for long (C4: 175 us serialised), so
  // the 16384-key class no longer queues behind them: C4 sort 0.529 -> 0.492 ms (C3, which
  // has no such buckets, 0.140 -> 0.142); the 8192-key class on the main stream 0.509.
  cudaEventRecord(fork, st);
  cudaStreamWaitEvent(side, fork, 0);
  cudaStreamWaitEvent(side2, fork, 0);
  {
    constexpr int smem = static_cast<int>(sizeof(uint64_t)) * kHugeChunk;
    static unsigned long long configured = 0;
    if (!(configured >> dev & 1ull)) {
      cudaFuncSetAttribute(sort_tiles_huge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      configured |= 1ull << dev;
    }
    sort_tiles_huge_kernel<<<std::min(n_sm, tiles), 1024, smem, side>>>(ranges, tile_keys, key_scratch, tile_vals,
                                                                        tile_masks, depth_bits, depth_minmax, src_bits,
                                                                        classes, tiles);
  }
  launch_sort_class<1024, 3>(ranges, tiles, tile_keys, tile_vals, tile_masks, depth_bits, depth_minmax, src_bits, classes,
                             n_sm, side2);
  launch_sort_class<1024, 2>(ranges, tiles, tile_keys, tile_vals, tile_masks, depth_bits, depth_minmax, src_bits, classes,
                             3 * n_sm, side);
  launch_sort_class<512, 1>(ranges, tiles, tile_keys, tile_vals, tile_masks, depth_bits, depth_minmax, src_bits, classes,
                            4 * n_sm, st);
  launch_sort_class<PSM_SORT_NT0, 0>(ranges, tiles, tile_keys, tile_vals, tile_masks, depth_bits, depth_minmax, src_bits, classes,
                            8 * n_sm, st);
  cudaEventRecord(join, side);
  cudaEventRecord(join2, side2);
  cudaStreamWaitEvent(st, join, 0);
  cudaStreamWaitEvent(st, join2, 0);
}

void launch_compact(const int32_t* valid, const int32_t* pos, const uint64_t* depth_bits, int64_t n, uint64_t* keys_out,
                    uint32_t* src_out, cudaStream_t st) {
  if (n > 0) compact_kernel<<<grid_for(n, 256), 256, 0, st>>>(valid, pos, depth_bits, n, keys_out, src_out);
}
void launch_rank_of(const uint32_t* src_by_rank, const uint32_t* n_proj_dev, int64_t cap, int32_t* rank_of,
                    cudaStream_t st) {
  if (cap > 0) rank_of_kernel<<<grid_for(cap, 256), 256, 0, st>>>(src_by_rank, n_proj_dev, rank_of);
}
void launch_debug_keys(const int32_t* ranges, int tiles, const uint32_t* sorted_vals, const int32_t* rank_of,
                       uint64_t* keys_out, cudaStream_t st) {
  if (tiles > 0) debug_keys_kernel<<<tiles, 128, 0, st>>>(ranges, sorted_vals, rank_of, keys_out);
}

}  // namespace psm
