// radix_sort.cu — hand-written stable LSD radix sort for the two sorts of the
// render pipeline (K2: surfels by fp64 depth bits, 64-bit keys; K5: (tile, surfel)
// assignments by tile id, 12-13 key bits), replacing the reference's per-tile
// std::sort by (sort_depth, source) (proj/src/raster.cpp:77-83).
//
// 8-bit digits, 4096 keys per CTA (256 threads x 16), three kernels per pass:
//   upsweep    per-CTA digit histogram (per-warp shared counters) -> hist[d][cta],
//              digit totals by atomics
//   scan       one CTA per digit: exclusive scan of hist[d][*] over CTAs plus the
//              digit's base (sum of smaller digits' totals)
//   downsweep  stable CTA-local ranking (__match_any_sync per 32-key round, warps
//              own contiguous 512-key runs), keys reordered in shared memory and
//              written out as coalesced per-digit runs
// The key count is read from device memory (no host round trip); grids are sized
// for the capacity and CTAs past the count exit. Input order is preserved among
// equal keys, so sorting source-ordered depth keys yields the reference's
// (sort_depth, source) order and sorting rank-ordered tile keys yields each
// tile's list in that order.
#include <cstdint>

#include "psm_device.cuh"
#include "psm_kernels.h"

namespace psm {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kItems = 16;
constexpr int kTileKeys = kThreads * kItems;  // 4096
constexpr int kRadix = 256;

template <typename K>
__device__ __forceinline__ int digit_of(K k, int shift) {
  return static_cast<int>((k >> shift) & 0xffu);
}

template <typename K>
__global__ void __launch_bounds__(kThreads) upsweep_kernel(const K* __restrict__ keys, const uint32_t* __restrict__ n_ptr,
                                                           int shift, uint32_t* __restrict__ hist,
                                                           uint32_t* __restrict__ totals, int max_ctas) {
  __shared__ uint32_t h[kWarps][kRadix];
  const uint32_t n = *n_ptr;
  const uint32_t start = blockIdx.x * kTileKeys;
  if (start >= n) return;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < kWarps * kRadix; i += kThreads) (&h[0][0])[i] = 0;
  __syncthreads();
  const uint32_t end = min(n, start + kTileKeys);
  for (uint32_t i = start + tid; i < end; i += kThreads) atomicAdd(&h[warp][digit_of(keys[i], shift)], 1u);
  __syncthreads();
  {
    const int d = tid;  // kThreads == kRadix
    uint32_t s = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) s += h[w][d];
    hist[d * max_ctas + blockIdx.x] = s;
    if (s) atomicAdd(totals + d, s);
  }
}

// One CTA per digit: hist[d][c] <- base(d) + sum_{c' < c} hist[d][c'].
__global__ void __launch_bounds__(1024) scan_kernel(uint32_t* __restrict__ hist, const uint32_t* __restrict__ totals,
                                                    const uint32_t* __restrict__ n_ptr, int max_ctas) {
  __shared__ uint32_t warp_sums[32];
  __shared__ uint32_t s_base;
  const int d = blockIdx.x;
  const uint32_t n = *n_ptr;
  const int nctas = static_cast<int>((n + kTileKeys - 1) / kTileKeys);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid < 32) {  // base = sum of totals of smaller digits
    uint32_t s = 0;
    for (int j = lane; j < d; j += 32) s += totals[j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) s_base = s;
  }
  __syncthreads();
  uint32_t carry = s_base;
  uint32_t* row = hist + static_cast<int64_t>(d) * max_ctas;
  for (int c0 = 0; c0 < nctas; c0 += 1024) {
    const int c = c0 + tid;
    const uint32_t v = c < nctas ? row[c] : 0u;
    uint32_t x = v;  // inclusive warp scan
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_sums[warp] = x;
    __syncthreads();
    if (warp == 0) {
      uint32_t ws = warp_sums[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, ws, o);
        if (lane >= o) ws += y;
      }
      warp_sums[lane] = ws;  // inclusive
    }
    __syncthreads();
    const uint32_t excl = x - v + (warp > 0 ? warp_sums[warp - 1] : 0u);
    if (c < nctas) row[c] = carry + excl;
    const uint32_t chunk_total = warp_sums[31];
    __syncthreads();
    carry += chunk_total;
  }
}

template <typename K>
struct SortSmem {
  K keys[kTileKeys];
  uint32_t vals[kTileKeys];
  uint32_t wcount[kWarps][kRadix];  // per-warp digit counts, then per-warp exclusive offsets
  uint32_t dstart[kRadix];          // CTA-local start of each digit's run
  uint32_t gbase[kRadix];           // global start of this CTA's run of each digit
  uint32_t scan_tmp[kWarps];
};

template <typename K>
__global__ void __launch_bounds__(kThreads) downsweep_kernel(const K* __restrict__ keys_in,
                                                             const uint32_t* __restrict__ vals_in,
                                                             K* __restrict__ keys_out, uint32_t* __restrict__ vals_out,
                                                             const uint32_t* __restrict__ n_ptr, int shift,
                                                             const uint32_t* __restrict__ hist, int max_ctas) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SortSmem<K>& sm = *reinterpret_cast<SortSmem<K>*>(smem_raw);
  const uint32_t n = *n_ptr;
  const uint32_t start = blockIdx.x * kTileKeys;
  if (start >= n) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < kWarps * kRadix; i += kThreads) (&sm.wcount[0][0])[i] = 0;
  __syncthreads();

  const unsigned lt_mask = (1u << lane) - 1u;
  K k[kItems];
  uint32_t v[kItems];
  uint32_t rank[kItems];
  const uint32_t wstart = start + warp * (kItems * 32);
#pragma unroll
  for (int r = 0; r < kItems; ++r) {
    const uint32_t idx = wstart + r * 32 + lane;
    const bool ok = idx < n;
    k[r] = ok ? keys_in[idx] : K(0);
    v[r] = ok ? vals_in[idx] : 0u;
    const int d = ok ? digit_of(k[r], shift) : kRadix;  // out-of-range keys form their own group
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    const uint32_t before = static_cast<uint32_t>(__popc(peers & lt_mask));
    const uint32_t base = ok ? sm.wcount[warp][d] : 0u;
    __syncwarp();
    if (ok && before == 0) sm.wcount[warp][d] = base + static_cast<uint32_t>(__popc(peers));
    __syncwarp();
    rank[r] = base + before;
  }
  __syncthreads();
  {  // per digit: exclusive offsets across warps; CTA totals -> exclusive scan across digits
    const int d = tid;
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      const uint32_t t = sm.wcount[w][d];
      sm.wcount[w][d] = run;
      run += t;
    }
    uint32_t x = run;  // inclusive scan of totals over d = tid
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) sm.scan_tmp[warp] = x;
    __syncthreads();
    uint32_t wpre = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w)
      if (w < warp) wpre += sm.scan_tmp[w];
    sm.dstart[d] = wpre + x - run;
    sm.gbase[d] = hist[d * max_ctas + blockIdx.x];
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kItems; ++r) {
    const uint32_t idx = wstart + r * 32 + lane;
    if (idx < n) {
      const int d = digit_of(k[r], shift);
      const uint32_t lp = sm.dstart[d] + sm.wcount[warp][d] + rank[r];
      sm.keys[lp] = k[r];
      sm.vals[lp] = v[r];
    }
  }
  __syncthreads();
  const uint32_t cnt = min(n - start, static_cast<uint32_t>(kTileKeys));
  for (uint32_t i = tid; i < cnt; i += kThreads) {
    const K key = sm.keys[i];
    const int d = digit_of(key, shift);
    const uint32_t o = sm.gbase[d] + (i - sm.dstart[d]);
    keys_out[o] = key;
    vals_out[o] = sm.vals[i];
  }
}

template <typename K>
void configure_downsweep() {
  static unsigned long long configured = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(configured >> dev & 1ull)) {
    cudaFuncSetAttribute(downsweep_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(sizeof(SortSmem<K>)));
    configured |= 1ull << dev;
  }
}

template <typename K>
void sort_pairs(K* keys, uint32_t* vals, K* keys_alt, uint32_t* vals_alt, const uint32_t* n_dev, int64_t cap,
                int begin_bit, int end_bit, uint32_t* hist, uint32_t* totals, cudaStream_t st, bool* result_in_alt) {
  const int max_ctas = static_cast<int>((cap + kTileKeys - 1) / kTileKeys);
  configure_downsweep<K>();
  K* kin = keys;
  uint32_t* vin = vals;
  K* kout = keys_alt;
  uint32_t* vout = vals_alt;
  bool in_alt = false;
  for (int shift = begin_bit; shift < end_bit; shift += 8) {
    cudaMemsetAsync(totals, 0, sizeof(uint32_t) * kRadix, st);
    if (max_ctas > 0) {
      upsweep_kernel<K><<<max_ctas, kThreads, 0, st>>>(kin, n_dev, shift, hist, totals, max_ctas);
      scan_kernel<<<kRadix, 1024, 0, st>>>(hist, totals, n_dev, max_ctas);
      downsweep_kernel<K><<<max_ctas, kThreads, sizeof(SortSmem<K>), st>>>(kin, vin, kout, vout, n_dev, shift, hist,
                                                                           max_ctas);
    }
    K* tk = kin; kin = kout; kout = tk;
    uint32_t* tv = vin; vin = vout; vout = tv;
    in_alt = !in_alt;
  }
  *result_in_alt = in_alt;
}

}  // namespace

size_t radix_hist_words(int64_t cap) { return static_cast<size_t>(kRadix) * ((cap + kTileKeys - 1) / kTileKeys) + 1; }

void radix_sort_u64(uint64_t* keys, uint32_t* vals, uint64_t* keys_alt, uint32_t* vals_alt, const uint32_t* n_dev,
                    int64_t cap, int begin_bit, int end_bit, uint32_t* hist, uint32_t* totals, cudaStream_t st,
                    bool* result_in_alt) {
  sort_pairs<uint64_t>(keys, vals, keys_alt, vals_alt, n_dev, cap, begin_bit, end_bit, hist, totals, st,
                       result_in_alt);
}

void radix_sort_u32(uint32_t* keys, uint32_t* vals, uint32_t* keys_alt, uint32_t* vals_alt, const uint32_t* n_dev,
                    int64_t cap, int begin_bit, int end_bit, uint32_t* hist, uint32_t* totals, cudaStream_t st,
                    bool* result_in_alt) {
  sort_pairs<uint32_t>(keys, vals, keys_alt, vals_alt, n_dev, cap, begin_bit, end_bit, hist, totals, st,
                       result_in_alt);
}

}  // namespace psm
