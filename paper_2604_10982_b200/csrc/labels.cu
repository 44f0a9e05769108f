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

__global__ void __launch_bounds__(256) assign_labels_kernel(LabelParams p) {
  const int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s >= p.n) return;
  const int D = p.c_sem + p.n_q;
  float* row32 = p.feat_out + s * D;
  double* row64 = p.feat64_out ? p.feat64_out + s * D : nullptr;
  // f_sem columns carried over from the old rows
  for (int c = 0; c < p.c_sem; ++c) {
    row32[c] = p.feat_in[s * p.d_in + c];
    if (row64) row64[c] = p.feat64_in[s * p.d_in + c];
  }
  int best = -1;
  if (p.n_alive > 0) {
    double center[3];
    center[0] = p.surfels[s * 13 + 0];
    center[1] = p.surfels[s * 13 + 1];
    center[2] = p.surfels[s * 13 + 2];
    const int b = psm_assign_one(p.f_ins + s * p.c_ins, p.c_ins, center, p.n_alive, p.q_feat, p.q_mean, p.q_inv,
                                 p.scratch + s, p.n, psm_exp_tab_dev);
    best = p.alive_index[b];
  }
  for (int q = 0; q < p.n_q; ++q) {
    const int a = p.alive_slot[q];
    const double v = a >= 0 ? p.scratch[static_cast<int64_t>(a) * p.n + s] : 0.0;
    row32[p.c_sem + q] = static_cast<float>(v);
    if (row64) row64[p.c_sem + q] = v;
    if (p.dist) p.dist[s * p.n_q + q] = v;
  }
  if (p.argmax) p.argmax[s] = best;
}

}  // namespace

void launch_assign_labels(const LabelParams& p, cudaStream_t st) {
  if (p.n <= 0) return;
  const unsigned blocks = static_cast<unsigned>((p.n + 255) / 256);
  assign_labels_kernel<<<blocks, 256, 0, st>>>(p);
}

}  // namespace psm
