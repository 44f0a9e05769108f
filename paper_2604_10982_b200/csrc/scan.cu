// scan.cu — exclusive prefix sum of uint32 counts with a device-resident length,
// used for the projected-surfel compaction (valid flags -> compact positions)
// and for the per-rank tile counts (-> key offsets and RN-Total; the reference
// accumulates these by push_back, proj/src/raster.cpp:69-75,84-88).
// Three kernels: per-CTA sums (4096 items / CTA), one-CTA scan of the CTA sums
// (also writes the grand total), per-CTA scan + offset. No host round trip.
#include <cstdint>

#include "psm_device.cuh"
#include "psm_kernels.h"

namespace psm {
namespace {

constexpr int kThreads = 256;
constexpr int kItems = 16;
constexpr int kTile = kThreads * kItems;

__device__ __forceinline__ uint32_t block_exclusive(uint32_t v, uint32_t* warp_tmp, uint32_t* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tmp[warp] = x;
  __syncthreads();
  uint32_t pre = 0, all = 0;
  for (int w = 0; w < (kThreads >> 5); ++w) {
    const uint32_t t = warp_tmp[w];
    if (w < warp) pre += t;
    all += t;
  }
  __syncthreads();
  *total = all;
  return pre + x - v;
}

template <typename In>
__global__ void __launch_bounds__(kThreads) reduce_kernel(const In* __restrict__ in, const uint32_t* __restrict__ n_ptr,
                                                          int64_t n_fixed, uint32_t* __restrict__ cta_sums) {
  __shared__ uint32_t tmp[kThreads / 32];
  const int64_t n = n_ptr ? static_cast<int64_t>(*n_ptr) : n_fixed;
  const int64_t start = static_cast<int64_t>(blockIdx.x) * kTile;
  if (start >= n) return;
  uint32_t s = 0;
  const int64_t end = min(n, start + kTile);
  for (int64_t i = start + threadIdx.x; i < end; i += kThreads) s += static_cast<uint32_t>(in[i]);
  uint32_t total;
  block_exclusive(s, tmp, &total);
  if (threadIdx.x == 0) cta_sums[blockIdx.x] = total;
}

__global__ void __launch_bounds__(1024) cta_scan_kernel(uint32_t* __restrict__ cta_sums, const uint32_t* __restrict__ n_ptr,
                                                        int64_t n_fixed, uint32_t* __restrict__ total_out) {
  __shared__ uint32_t warp_sums[32];
  const int64_t n = n_ptr ? static_cast<int64_t>(*n_ptr) : n_fixed;
  const int nctas = static_cast<int>((n + kTile - 1) / kTile);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint32_t carry = 0;
  for (int c0 = 0; c0 < nctas; c0 += 1024) {
    const int c = c0 + tid;
    const uint32_t v = c < nctas ? cta_sums[c] : 0u;
    uint32_t x = v;
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
      warp_sums[lane] = ws;
    }
    __syncthreads();
    if (c < nctas) cta_sums[c] = carry + x - v + (warp > 0 ? warp_sums[warp - 1] : 0u);
    const uint32_t chunk = warp_sums[31];
    __syncthreads();
    carry += chunk;
  }
  if (tid == 0) *total_out = carry;
}

template <typename In>
__global__ void __launch_bounds__(kThreads) apply_kernel(const In* __restrict__ in, const uint32_t* __restrict__ n_ptr,
                                                         int64_t n_fixed, const uint32_t* __restrict__ cta_sums,
                                                         uint32_t* __restrict__ out) {
  __shared__ uint32_t tmp[kThreads / 32];
  const int64_t n = n_ptr ? static_cast<int64_t>(*n_ptr) : n_fixed;
  const int64_t start = static_cast<int64_t>(blockIdx.x) * kTile;
  if (start >= n) return;
  // each thread owns kItems consecutive items
  const int64_t base = start + static_cast<int64_t>(threadIdx.x) * kItems;
  uint32_t v[kItems];
  uint32_t s = 0;
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    v[j] = base + j < n ? static_cast<uint32_t>(in[base + j]) : 0u;
    s += v[j];
  }
  uint32_t total;
  uint32_t run = block_exclusive(s, tmp, &total) + cta_sums[blockIdx.x];
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    if (base + j < n) out[base + j] = run;
    run += v[j];
  }
}

template <typename In>
void scan_t(const In* in, const uint32_t* n_dev, int64_t n_fixed, int64_t cap, uint32_t* out, uint32_t* total_dev,
            uint32_t* cta_sums, cudaStream_t st) {
  const int64_t ctas = (cap + kTile - 1) / kTile;
  if (ctas <= 0) {
    cudaMemsetAsync(total_dev, 0, sizeof(uint32_t), st);
    return;
  }
  reduce_kernel<In><<<static_cast<unsigned>(ctas), kThreads, 0, st>>>(in, n_dev, n_fixed, cta_sums);
  cta_scan_kernel<<<1, 1024, 0, st>>>(cta_sums, n_dev, n_fixed, total_dev);
  apply_kernel<In><<<static_cast<unsigned>(ctas), kThreads, 0, st>>>(in, n_dev, n_fixed, cta_sums, out);
}

}  // namespace

size_t scan_cta_words(int64_t cap) { return static_cast<size_t>((cap + kTile - 1) / kTile) + 1; }

void exclusive_scan_i32(const int32_t* in, int64_t n, uint32_t* out, uint32_t* total_dev, uint32_t* cta_sums,
                        cudaStream_t st) {
  scan_t<int32_t>(in, nullptr, n, n, out, total_dev, cta_sums, st);
}

void exclusive_scan_u32_dev(const uint32_t* in, const uint32_t* n_dev, int64_t cap, uint32_t* out, uint32_t* total_dev,
                            uint32_t* cta_sums, cudaStream_t st) {
  scan_t<uint32_t>(in, n_dev, 0, cap, out, total_dev, cta_sums, st);
}

}  // namespace psm
