// labels.cu — assign_labels (proj/src/panoptic.cpp:36-91) on the device, SURVEY.md
// §8f row F2: one thread per surfel evaluates every alive query's attention
// A = sigmoid(f_q . f_ins) * exp(-1/2 d^T Sigma^-1 d) and the softmax over them with
// the shared psm_panoptic.h arithmetic (bit-identical to the oracle), then writes the
// scene's new feature rows [f_sem | dist] in fp32 (and fp64 for exact scenes).
//
// The A values of a surfel live in a column-major scratch (a * N + s), so a warp's
// accesses to one query are coalesced; the query table (features, means, inverse
// covariances) is read through the read-only cache by every thread alike.
#include <cstdint>

#include "psm_device.cuh"
#include "psm_kernels.h"
#include "psm_panoptic.h"

namespace psm {
namespace {

// Copies the alive-query table (features, means, inverse covariances: n_alive x
// (c_ins + 12) doubles) and psm_exp's table into shared memory.
__device__ __forceinline__ void stage_tables(const LabelParams& p, double* qs, uint64_t* tab) {
  const int words = p.n_alive * (p.c_ins + 12);
  for (int i = threadIdx.x; i < words; i += blockDim.x) qs[i] = p.q_feat[i];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) tab[i] = psm_exp_tab_dev[i];
  __syncthreads();
}

// The surfel's new row: f_sem columns (when not in place), then dist over all queries.
__device__ __forceinline__ void write_rows(const LabelParams& p, int64_t s, int best) {
  const int D = p.c_sem + p.n_q;
  float* row32 = p.feat_out + s * D;
  double* row64 = p.feat64_out ? p.feat64_out + s * D : nullptr;
  // f_sem columns carried over from the old rows (nothing to do when rewriting in place)
  for (int c = 0; c < (p.feat_out == p.feat_in ? 0 : p.c_sem); ++c) {
    row32[c] = p.feat_in[s * p.d_in + c];
    if (row64) row64[c] = p.feat64_in[s * p.d_in + c];
  }
  for (int q = 0; q < p.n_q; ++q) {
    const int a = p.alive_slot[q];
    double v = 0.0;
    if (a >= 0) v = p.scratch[static_cast<int64_t>(a) * p.n + s];
    row32[p.c_sem + q] = static_cast<float>(v);
    if (row64) row64[p.c_sem + q] = v;
    if (p.dist) p.dist[s * p.n_q + q] = v;
  }
  if (p.argmax) p.argmax[s] = best;
}

// General path: A values in the column-major global scratch (a * N + s); the query
// table in shared memory when it fits (kQsWords), else read through L1.
constexpr int kQsWords = 6144;  // 48 KB
__global__ void __launch_bounds__(256) assign_labels_kernel(LabelParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  uint64_t* tab = reinterpret_cast<uint64_t*>(smem);
  double* qs = reinterpret_cast<double*>(smem + 2048);
  const bool staged = p.n_alive * (p.c_ins + 12) <= kQsWords;
  if (staged) {
    stage_tables(p, qs, tab);
  } else {
    tab[threadIdx.x] = psm_exp_tab_dev[threadIdx.x];
    __syncthreads();
  }
  const int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s >= p.n) return;
  const double* fq = staged ? qs : p.q_feat;
  const double* mean = fq + p.n_alive * p.c_ins;
  const double* inv = mean + 3 * p.n_alive;
  int best = -1;
  if (p.n_alive > 0) {
    const double center[3] = {p.surfels[s * 13 + 0], p.surfels[s * 13 + 1], p.surfels[s * 13 + 2]};
    const int b = psm_assign_one(p.f_ins + s * p.c_ins, p.c_ins, center, p.n_alive, fq, mean, inv,
                                 p.scratch + s, p.n, tab);
    best = p.alive_index[b];
  }
  write_rows(p, s, best);
}

// Up to 32 alive queries: a warp keeps its 32 surfels' A values / probabilities in shared
// memory ([query][33] per warp, padded against bank conflicts) instead of the global
// scratch, and then writes the 32 rows cooperatively: lane = column, so every row store
// is one coalesced run (the per-thread row stores of the general path touch one 32-byte
// sector per lane and value). CI > 0: C_ins == CI at compile time, so the surfel's f_ins
// row is loaded once into registers and every query's dot is unrolled; the dynamic form
// re-reads the row through L1 for every query (C3p, 32 queries, C_ins 8: 0.89 -> 0.55 ms).
constexpr int kRowsMaxAlive = 32;
constexpr int kRowsWarps = 8;
template <int CI>
__global__ void __launch_bounds__(32 * kRowsWarps) assign_labels_rows_kernel(LabelParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  uint64_t* tab = reinterpret_cast<uint64_t*>(smem);
  double* vals = reinterpret_cast<double*>(smem + 2048);  // [warp][kRowsMaxAlive][33]
  double* qs = vals + kRowsWarps * kRowsMaxAlive * 33;
  stage_tables(p, qs, tab);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* wv = vals + warp * kRowsMaxAlive * 33;
  const int64_t s0 = (static_cast<int64_t>(blockIdx.x) * kRowsWarps + warp) * 32;
  const int64_t s = s0 + lane;
  const double* mean = qs + p.n_alive * p.c_ins;
  const double* inv = mean + 3 * p.n_alive;
  int best = -1;
  if (s < p.n && p.n_alive > 0) {
    const double center[3] = {p.surfels[s * 13 + 0], p.surfels[s * 13 + 1], p.surfels[s * 13 + 2]};
    int b;
    if constexpr (CI > 0) {
      double f[CI];
      const double2* row = reinterpret_cast<const double2*>(p.f_ins + s * CI);  // 16 B aligned: CI even
#pragma unroll
      for (int c = 0; c < CI / 2; ++c) {
        const double2 v = __ldg(row + c);
        f[2 * c] = v.x;
        f[2 * c + 1] = v.y;
      }
      b = psm_assign_one(f, CI, center, p.n_alive, qs, mean, inv, wv + lane, 33, tab);
    } else {
      b = psm_assign_one(p.f_ins + s * p.c_ins, p.c_ins, center, p.n_alive, qs, mean, inv, wv + lane, 33, tab);
    }
    best = p.alive_index[b];
  }
  if (s < p.n && p.argmax) p.argmax[s] = best;
  __syncwarp();
  const int D = p.c_sem + p.n_q;
  const bool carry = p.feat_out != p.feat_in;  // f_sem columns move to new rows
  for (int j = 0; j < 32; ++j) {
    const int64_t sj = s0 + j;
    if (sj >= p.n) break;
    float* row32 = p.feat_out + sj * D;
    double* row64 = p.feat64_out ? p.feat64_out + sj * D : nullptr;
    if (carry)
      for (int c = lane; c < p.c_sem; c += 32) {
        row32[c] = p.feat_in[sj * p.d_in + c];
        if (row64) row64[c] = p.feat64_in[sj * p.d_in + c];
      }
    for (int q = lane; q < p.n_q; q += 32) {
      const int a = p.alive_slot[q];
      const double v = a >= 0 ? wv[a * 33 + j] : 0.0;
      row32[p.c_sem + q] = static_cast<float>(v);
      if (row64) row64[p.c_sem + q] = v;
      if (p.dist) p.dist[sj * p.n_q + q] = v;
    }
  }
}

}  // namespace

void launch_assign_labels(const LabelParams& p, cudaStream_t st) {
  if (p.n <= 0) return;
  static unsigned long long configured = 0;  // one bit per device
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(configured >> dev & 1ull)) {
    const int most = 2048 + static_cast<int>(sizeof(double)) * kQsWords;
    cudaFuncSetAttribute(assign_labels_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, most);
    configured |= 1ull << dev;
  }
  const int words = p.n_alive * (p.c_ins + 12);
  if (p.n_alive <= kRowsMaxAlive && words <= kQsWords) {
    static unsigned long long configured_rows = 0;
    const int most = 2048 + static_cast<int>(sizeof(double)) * (kRowsWarps * kRowsMaxAlive * 33 + kQsWords);
    if (!(configured_rows >> dev & 1ull)) {
      cudaFuncSetAttribute(assign_labels_rows_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, most);
      cudaFuncSetAttribute(assign_labels_rows_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, most);
      cudaFuncSetAttribute(assign_labels_rows_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, most);
      configured_rows |= 1ull << dev;
    }
    const size_t smem = 2048 + sizeof(double) * (kRowsWarps * kRowsMaxAlive * 33 + words);
    const unsigned blocks = static_cast<unsigned>((p.n + 32 * kRowsWarps - 1) / (32 * kRowsWarps));
    if (p.c_ins == 8) assign_labels_rows_kernel<8><<<blocks, 32 * kRowsWarps, smem, st>>>(p);
    else if (p.c_ins == 16) assign_labels_rows_kernel<16><<<blocks, 32 * kRowsWarps, smem, st>>>(p);
    else assign_labels_rows_kernel<0><<<blocks, 32 * kRowsWarps, smem, st>>>(p);
    return;
  }
  const unsigned blocks = static_cast<unsigned>((p.n + 255) / 256);
  const size_t smem = 2048 + (words <= kQsWords ? sizeof(double) * words : 0);
  assign_labels_kernel<<<blocks, 256, smem, st>>>(p);
}

}  // namespace psm
