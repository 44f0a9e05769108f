// binning.cu — K2..K6 glue kernels: compaction of projected surfels into
// (depth, source) sort input, per-rank tile counts, (tile, source) key
// emission in depth-rank order, and per-tile [start, end) ranges.
//
// Reference: bin_boxes (proj/src/raster.cpp:51-90). The reference pushes each
// projected index into every tile of its box and then std::sorts each tile by
// (sort_depth, source) (raster.cpp:77-83). Here the N surfels are sorted once by
// depth (stable radix sort of the fp64 bit pattern, source-ordered input, so
// ties keep source order), keys are emitted in that rank order, and a stable
// sort on the tile bits alone yields each tile's list already in
// (depth, source) order: the same lists, with one N-sized 64-bit sort and one
// RN-sized 12-13-bit sort instead of per-tile comparison sorts.
#include "psm_device.cuh"
#include "psm_ellipse.h"
#include "psm_kernels.h"

namespace psm {
namespace {

__global__ void compact_kernel(const int32_t* __restrict__ valid, const int32_t* __restrict__ pos,
                               const uint64_t* __restrict__ depth_bits, int64_t n, uint64_t* __restrict__ keys_out,
                               uint32_t* __restrict__ src_out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n || !valid[i]) return;
  const int32_t o = pos[i];
  keys_out[o] = depth_bits[i];
  src_out[o] = static_cast<uint32_t>(i);
}

__global__ void gather_counts_kernel(const uint32_t* __restrict__ src_by_rank, const int32_t* __restrict__ tile_cnt,
                                     const uint32_t* __restrict__ n_proj_dev, uint32_t* __restrict__ cnt_by_rank) {
  const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= *n_proj_dev) return;
  cnt_by_rank[r] = static_cast<uint32_t>(tile_cnt[src_by_rank[r]]);
}

__global__ void emit_kernel(const uint32_t* __restrict__ src_by_rank, const uint32_t* __restrict__ offsets,
                            const uint32_t* __restrict__ n_proj_dev, const SurfRec* __restrict__ recs,
                            const BinRec* __restrict__ bins, DevRaster rs, int img_h, uint32_t* __restrict__ tile_keys,
                            uint32_t* __restrict__ tile_vals, const uint32_t* __restrict__ rn_dev, uint32_t cap,
                            uint32_t* __restrict__ rn_eff, int32_t* __restrict__ overflow) {
  const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r == 0) {
    const uint32_t rn = *rn_dev;
    *rn_eff = rn < cap ? rn : cap;
    if (rn > cap) atomicOr(overflow, 1);  // keys beyond the capacity are dropped; the host re-renders
  }
  if (r >= *n_proj_dev) return;
  const uint32_t s = src_by_rank[r];
  const BinRec b = bins[s];
  if (b.tx0 > b.tx1 || b.ty0 > b.ty1) return;
  uint32_t o = offsets[r];
  const bool ellipse = rs.binning == PSM_BIN_ELLIPSE;
  const double cx = recs[s].cx, cy = recs[s].cy;
  for (int ty = b.ty0; ty <= b.ty1; ++ty) {
    int lo = b.tx0, hi = b.tx1;
    if (ellipse && !psm_ellipse_row(cx, cy, b.F00, b.F01, b.F11, rs.chi2, ty, rs.tile_size, img_h, b.tx0, b.tx1, &lo, &hi))
      continue;
    for (int tx = lo; tx <= hi; ++tx, ++o) {
      if (o < cap) {
        tile_keys[o] = static_cast<uint32_t>(ty * rs.tiles_x + tx);
        tile_vals[o] = s;
      }
    }
  }
}

__global__ void ranges_kernel(const uint32_t* __restrict__ keys, const uint32_t* __restrict__ rn_dev,
                              int32_t* __restrict__ ranges, unsigned long long* __restrict__ nonempty) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t rn = *rn_dev;
  bool first = false;
  if (i < rn) {
    const uint32_t t = keys[i];
    first = i == 0 || keys[i - 1] != t;
    if (first) ranges[2 * t] = static_cast<int32_t>(i);
    if (i == rn - 1 || keys[i + 1] != t) ranges[2 * t + 1] = static_cast<int32_t>(i + 1);
  }
  const unsigned cnt = __popc(__ballot_sync(0xffffffffu, first));
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(nonempty, static_cast<unsigned long long>(cnt));
}

__global__ void rank_of_kernel(const uint32_t* __restrict__ src_by_rank, const uint32_t* __restrict__ n_proj_dev,
                               int32_t* __restrict__ rank_of) {
  const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r < *n_proj_dev) rank_of[src_by_rank[r]] = static_cast<int32_t>(r);
}

__global__ void debug_keys_kernel(const uint32_t* __restrict__ tiles, const uint32_t* __restrict__ vals,
                                  const int32_t* __restrict__ rank_of, int64_t rn, uint64_t* __restrict__ out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < rn) out[i] = (static_cast<uint64_t>(tiles[i]) << 32) | static_cast<uint32_t>(rank_of[vals[i]]);
}

inline unsigned grid_for(int64_t n, int block) { return static_cast<unsigned>((n + block - 1) / block); }

}  // namespace

void launch_compact(const int32_t* valid, const int32_t* pos, const uint64_t* depth_bits, int64_t n, uint64_t* keys_out,
                    uint32_t* src_out, cudaStream_t st) {
  if (n > 0) compact_kernel<<<grid_for(n, 256), 256, 0, st>>>(valid, pos, depth_bits, n, keys_out, src_out);
}
void launch_gather_counts(const uint32_t* src_by_rank, const int32_t* tile_cnt, const uint32_t* n_proj_dev, int64_t cap,
                          uint32_t* cnt_by_rank, cudaStream_t st) {
  if (cap > 0) gather_counts_kernel<<<grid_for(cap, 256), 256, 0, st>>>(src_by_rank, tile_cnt, n_proj_dev, cnt_by_rank);
}
void launch_emit(const uint32_t* src_by_rank, const uint32_t* offsets, const uint32_t* n_proj_dev, int64_t cap_proj,
                 const SurfRec* recs, const BinRec* bins, const DevRaster& rs, int img_h, uint32_t* tile_keys,
                 uint32_t* tile_vals, const uint32_t* rn_dev, uint32_t cap_keys, uint32_t* rn_eff, int32_t* overflow,
                 cudaStream_t st) {
  emit_kernel<<<grid_for(cap_proj > 0 ? cap_proj : 1, 256), 256, 0, st>>>(
      src_by_rank, offsets, n_proj_dev, recs, bins, rs, img_h, tile_keys, tile_vals, rn_dev, cap_keys, rn_eff, overflow);
}
void launch_ranges(const uint32_t* sorted_tiles, const uint32_t* rn_dev, int64_t cap, int32_t* ranges,
                   unsigned long long* nonempty, cudaStream_t st) {
  if (cap > 0) ranges_kernel<<<grid_for(cap, 256), 256, 0, st>>>(sorted_tiles, rn_dev, ranges, nonempty);
}
void launch_rank_of(const uint32_t* src_by_rank, const uint32_t* n_proj_dev, int64_t cap, int32_t* rank_of,
                    cudaStream_t st) {
  if (cap > 0) rank_of_kernel<<<grid_for(cap, 256), 256, 0, st>>>(src_by_rank, n_proj_dev, rank_of);
}
void launch_debug_keys(const uint32_t* sorted_tiles, const uint32_t* sorted_vals, const int32_t* rank_of, int64_t rn,
                       uint64_t* keys_out, cudaStream_t st) {
  if (rn > 0) debug_keys_kernel<<<grid_for(rn, 256), 256, 0, st>>>(sorted_tiles, sorted_vals, rank_of, rn, keys_out);
}

}  // namespace psm
