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
//                  (fp64 depth bits, source) with a bitonic network in shared
//                  memory (flip formulation, implicit +inf padding), so the
//                  result is the reference's list whatever order K4 produced.
//                  Buckets larger than 4096 entries fall back to the same network
//                  over global memory.
// Every count stays on the device; key buffers are capacity-checked (the host
// re-renders a frame whose RN-Total outgrew them, capi.cu).
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

// K3b: one CTA scans the tile totals: ranges, tile starts, RN-Total, non-empty tiles.
__global__ void __launch_bounds__(1024) tile_scan_kernel(const uint32_t* __restrict__ totals, int tiles, uint32_t cap,
                                                        int32_t* __restrict__ ranges, uint32_t* __restrict__ tile_start,
                                                        uint32_t* __restrict__ rn_dev, uint32_t* __restrict__ rn_eff,
                                                        unsigned long long* __restrict__ nonempty,
                                                        int32_t* __restrict__ overflow) {
  __shared__ uint32_t warp_sums[32];
  __shared__ uint32_t warp_ne[32];
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
    if (t < tiles) {
      const uint32_t v = totals[t];
      tile_start[t] = run;
      ranges[2 * t] = static_cast<int32_t>(min(run, cap));
      ranges[2 * t + 1] = static_cast<int32_t>(min(run + v, cap));
      run += v;
    }
  }
  if (tid == 0) {
    *rn_dev = all;
    *rn_eff = min(all, cap);
    *nonempty = all_ne;
    if (all > cap) atomicOr(overflow, 1);  // buckets past the capacity are dropped; the host re-renders
  }
}

__global__ void __launch_bounds__(256) emit_kernel(const int32_t* __restrict__ valid, int64_t n,
                                                   const SurfRec* __restrict__ recs, const BinRec* __restrict__ bins,
                                                   DevRaster rs, int img_h, uint32_t* __restrict__ cursor,
                                                   const uint32_t* __restrict__ tile_start, uint32_t cap,
                                                   uint32_t* __restrict__ tile_vals) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n || !valid[i]) return;
  const BinRec b = bins[i];
  if (b.tx0 > b.tx1 || b.ty0 > b.ty1) return;
  const bool ellipse = rs.binning == PSM_BIN_ELLIPSE;
  const double cx = recs[i].cx, cy = recs[i].cy;
  uint32_t* cur = cursor + static_cast<int64_t>(threadIdx.x & (kSplit - 1)) * rs.tiles_x * rs.tiles_y;
  for (int ty = b.ty0; ty <= b.ty1; ++ty) {
    int lo = b.tx0, hi = b.tx1;
    if (ellipse && !psm_ellipse_row(cx, cy, b.F00, b.F01, b.F11, rs.chi2, ty, rs.tile_size, img_h, b.tx0, b.tx1, &lo, &hi))
      continue;
    for (int tx = lo; tx <= hi; ++tx) {
      const int t = ty * rs.tiles_x + tx;
      const uint32_t o = __ldg(tile_start + t) + atomicAdd(cur + t, 1u);
      if (o < cap) tile_vals[o] = static_cast<uint32_t>(i);
    }
  }
}

// (key, source) total order of the reference's per-tile comparator (raster.cpp:78-83):
// positive fp64 depths order as their bit patterns.
__device__ __forceinline__ bool key_greater(uint64_t ka, uint32_t sa, uint64_t kb, uint32_t sb) {
  return ka > kb || (ka == kb && sa > sb);
}

// Bitonic sort (flip formulation) of `len` entries, all compare-exchanges ascending and
// entries at index >= len treated as +inf (never moved), over arrays K / S that are
// shared or global memory. Called by all threads of the CTA.
__device__ __forceinline__ void cmp_swap(uint64_t* keys, uint32_t* srcs, int lo, int hi) {
  const uint64_t ka = keys[lo], kb = keys[hi];
  const uint32_t sa = srcs[lo], sb = srcs[hi];
  if (key_greater(ka, sa, kb, sb)) {
    keys[lo] = kb; keys[hi] = ka;
    srcs[lo] = sb; srcs[hi] = sa;
  }
}

template <int NT>
__device__ void bitonic_sort(uint64_t* keys, uint32_t* srcs, int len) {
  int lg = 0;
  while ((1 << lg) < len) ++lg;
  const int half = 1 << (lg - 1);
  for (int lk = 1; lk <= lg; ++lk) {
    const int lh = lk - 1;  // log2(k / 2)
    for (int i = threadIdx.x; i < half; i += NT) {  // flip
      const int blk = i >> lh, off = i & ((1 << lh) - 1);
      const int lo = (blk << lk) + off, hi = (blk << lk) + (1 << lk) - 1 - off;
      if (hi < len) cmp_swap(keys, srcs, lo, hi);
    }
    __syncthreads();
    for (int lj = lk - 2; lj >= 0; --lj) {  // half-cleaners, j = 2^lj
      for (int i = threadIdx.x; i < half; i += NT) {
        const int lo = ((i >> lj) << (lj + 1)) + (i & ((1 << lj) - 1)), hi = lo + (1 << lj);
        if (hi < len) cmp_swap(keys, srcs, lo, hi);
      }
      __syncthreads();
    }
  }
}

// One CTA per tile in the size class (lo_len, hi_len]; the smem class loads the bucket's
// (depth bits, source) into shared memory, the last class sorts in global memory.
template <int NT, int CAP, bool GLOBAL>
__global__ void __launch_bounds__(NT) sort_tiles_kernel(const int32_t* __restrict__ ranges, int lo_len,
                                                        const uint64_t* __restrict__ depth_bits,
                                                        uint32_t* __restrict__ tile_vals, uint64_t* __restrict__ key_scratch) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int t = blockIdx.x;
  const int start = ranges[2 * t], len = ranges[2 * t + 1] - start;
  if (len <= lo_len || len <= 1 || (!GLOBAL && len > CAP)) return;
  if (!GLOBAL) {
    uint64_t* keys = reinterpret_cast<uint64_t*>(smem_raw);
    uint32_t* srcs = reinterpret_cast<uint32_t*>(smem_raw + sizeof(uint64_t) * CAP);
    for (int i = threadIdx.x; i < len; i += NT) {
      const uint32_t s = tile_vals[start + i];
      srcs[i] = s;
      keys[i] = __ldg(depth_bits + s);
    }
    __syncthreads();
    bitonic_sort<NT>(keys, srcs, len);
    for (int i = threadIdx.x; i < len; i += NT) tile_vals[start + i] = srcs[i];
  } else {
    uint64_t* keys = key_scratch + start;
    uint32_t* srcs = tile_vals + start;
    for (int i = threadIdx.x; i < len; i += NT) keys[i] = __ldg(depth_bits + srcs[i]);
    __syncthreads();
    bitonic_sort<NT>(keys, srcs, len);
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
                      unsigned long long* nonempty, int32_t* overflow, cudaStream_t st) {
  tile_sub_scan_kernel<<<grid_for(tiles, 256), 256, 0, st>>>(tile_counts, tiles, cursor, totals);
  tile_scan_kernel<<<1, 1024, 0, st>>>(totals, tiles, cap, ranges, tile_start, rn_dev, rn_eff, nonempty, overflow);
}

void launch_emit(const int32_t* valid, int64_t n, const SurfRec* recs, const BinRec* bins, const DevRaster& rs,
                 int img_h, uint32_t* cursor, const uint32_t* tile_start, uint32_t cap, uint32_t* tile_vals,
                 cudaStream_t st) {
  if (n > 0)
    emit_kernel<<<grid_for(n, 256), 256, 0, st>>>(valid, n, recs, bins, rs, img_h, cursor, tile_start, cap, tile_vals);
}

template <int NT, int CAP, bool GLOBAL>
void launch_sort_class(const int32_t* ranges, int tiles, int lo_len, const uint64_t* depth_bits, uint32_t* tile_vals,
                       uint64_t* key_scratch, cudaStream_t st) {
  constexpr int smem = GLOBAL ? 0 : static_cast<int>((sizeof(uint64_t) + sizeof(uint32_t)) * CAP);
  static unsigned long long configured = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (!GLOBAL && !(configured >> dev & 1ull)) {
    cudaFuncSetAttribute(sort_tiles_kernel<NT, CAP, GLOBAL>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    configured |= 1ull << dev;
  }
  sort_tiles_kernel<NT, CAP, GLOBAL><<<tiles, NT, smem, st>>>(ranges, lo_len, depth_bits, tile_vals, key_scratch);
}

void launch_sort_tiles(const int32_t* ranges, int tiles, const uint64_t* depth_bits, uint32_t* tile_vals,
                       uint64_t* key_scratch, cudaStream_t st) {
  if (tiles <= 0) return;
  launch_sort_class<256, 4096, false>(ranges, tiles, 0, depth_bits, tile_vals, key_scratch, st);       // 48 KB
  launch_sort_class<1024, 16384, false>(ranges, tiles, 4096, depth_bits, tile_vals, key_scratch, st);  // 192 KB
  launch_sort_class<1024, 0, true>(ranges, tiles, 16384, depth_bits, tile_vals, key_scratch, st);      // global
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
