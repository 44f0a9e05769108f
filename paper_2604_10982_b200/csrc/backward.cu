// backward.cu — the render backward on the device: the blending
// backward of the training pipeline (proj/src/pipeline.cpp:347-460) and the geometry
// chain project_surfel_backward (raster.cpp:179-203, psm_backward.h).
//
// The forward runs first in cache mode (blend.cu with lists_t): every pixel's
// contributors in blend order as (list position, transmittance before the blend), plus
// the Top-K positions — RenderCache::pixels (raster.cpp:399-403). Here one thread per
// pixel walks its contributors backwards exactly as pipeline.cpp:393-452 does:
// alpha, u, v are recomputed from the staged record with the forward's fp64
// arithmetic (so they are the forward's bits), the suffix of w_i <g, value_i> is seeded
// with the background term, and the per-surfel sums are fp64 atomics (their order, and
// so the last bits, differ from the reference's chunked merge). A second kernel chains
// each projected surfel's dL/dH^-1 to its centre, quaternion and scales.
#include <cstdint>

#include "psm_backward.h"
#include "psm_device.cuh"
#include "psm_exp.h"
#include "psm_kernels.h"

namespace psm {
namespace {

__global__ void __launch_bounds__(256) pixel_backward_kernel(BackwardParams p) {
  __shared__ __align__(16) uint64_t tab[256];
  tab[threadIdx.x] = psm_exp_tab_dev[threadIdx.x];
  __syncthreads();
  const int64_t pix = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t npx = static_cast<int64_t>(p.width) * p.height;
  if (pix >= npx) return;
  int m = p.blend_count[pix];
  if (m > p.list_cap) m = p.list_cap;  // the caller re-renders with a larger cap first
  if (m <= 0) return;
  const int x = static_cast<int>(pix % p.width), y = static_cast<int>(pix / p.width);
  const double rx = (x + 0.5 - p.cam_cx) / p.cam_fx;
  const double ry = (y + 0.5 - p.cam_cy) / p.cam_fy;
  const double zero3[3] = {0.0, 0.0, 0.0};
  const double* gc = p.g_color ? p.g_color + pix * 3 : zero3;
  const double* gf = (p.c_sem > 0 && p.g_sem) ? p.g_sem + pix * p.c_sem : nullptr;
  const double* gi = (p.n_q > 0 && p.g_ins) ? p.g_ins + pix * p.n_q : nullptr;
  const int D = p.c_sem + p.n_q;
  const bool sel_all = !(p.topk && m > p.k_sel);
  const int32_t* tk = p.topk_pos ? p.topk_pos + pix * p.k_sel : nullptr;
  const uint2* lst = p.lists + pix * p.list_cap;
  const double* lt = p.lists_t + pix * p.list_cap;

  // T after the last blend: the forward's chain continued from the stored T_{m-1}
  double t_end;
  {
    const int pos = static_cast<int>(lst[m - 1].x);
    const SurfRec& r = p.recs[__ldg(p.vals + pos)];
    const double w0 = r.h[0] * rx + r.h[1] * ry + r.h[2];
    const double w1 = r.h[3] * rx + r.h[4] * ry + r.h[5];
    const double w2 = r.h[6] * rx + r.h[7] * ry + r.h[8];
    const double rcp = 1.0 / w2;
    const double u = w0 * rcp, v = w1 * rcp;
    const double alpha = r.opacity * psm_exp_t(-0.5 * (u * u + v * v), tab);
    t_end = lt[m - 1] * (1.0 - alpha);
  }
  double suffix = t_end * (gc[0] * p.bg0 + gc[1] * p.bg1 + gc[2] * p.bg2);
  for (int j = m - 1; j >= 0; --j) {
    const int pos = static_cast<int>(lst[j].x);
    const double t_j = lt[j];
    const int64_t src = __ldg(p.vals + pos);
    const SurfRec& r = p.recs[src];
    const double* sf = p.surfels + src * 13;
    // the forward's alpha (blend.cu main loop, raster.cpp:383-392), bit for bit
    const double w0 = r.h[0] * rx + r.h[1] * ry + r.h[2];
    const double w1 = r.h[3] * rx + r.h[4] * ry + r.h[5];
    const double w2 = r.h[6] * rx + r.h[7] * ry + r.h[8];
    const double rcp = 1.0 / w2;
    const double u = w0 * rcp, v = w1 * rcp;
    const double d_sigma = psm_exp_t(-0.5 * (u * u + v * v), tab);
    const double alpha = r.opacity * d_sigma;
    const double w_j = alpha * t_j;

    double direct = gc[0] * sf[10] + gc[1] * sf[11] + gc[2] * sf[12];
    atomicAdd(p.d_color + src * 3 + 0, w_j * gc[0]);
    atomicAdd(p.d_color + src * 3 + 1, w_j * gc[1]);
    atomicAdd(p.d_color + src * 3 + 2, w_j * gc[2]);
    bool selected = sel_all;
    if (!selected && tk)
      for (int i = 0; i < p.k_sel; ++i) selected |= tk[i] == pos;
    if (selected && (gf || gi)) {
      const int64_t row = src * D;
      if (gf) {
        double dot = 0;
        for (int i = 0; i < p.c_sem; ++i) {
          const double f = p.feat64 ? p.feat64[row + i] : static_cast<double>(p.feat32[row + i]);
          dot += gf[i] * f;
          atomicAdd(p.d_fsem + src * p.c_sem + i, w_j * gf[i]);
        }
        direct += dot;
      }
      if (gi) {
        double dot = 0;
        for (int i = 0; i < p.n_q; ++i) {
          const double l = p.feat64 ? p.feat64[row + p.c_sem + i] : static_cast<double>(p.feat32[row + p.c_sem + i]);
          dot += gi[i] * l;
          atomicAdd(p.d_lab + src * p.n_q + i, w_j * gi[i]);
        }
        direct += dot;
      }
    }
    const double one_minus = 1.0 - alpha;
    const double g_alpha = t_j * direct - (one_minus > 0 ? suffix / one_minus : 0.0);
    suffix += w_j * direct;
    atomicAdd(p.d_opacity + src, d_sigma * g_alpha);
    const double g_dsigma = r.opacity * g_alpha;
    const double g_u = -u * d_sigma * g_dsigma;
    const double g_v = -v * d_sigma * g_dsigma;
    const double gw[3] = {g_u / w2, g_v / w2, -(u * g_u + v * g_v) / w2};
    const double ray[3] = {rx, ry, 1.0};
    double* gh = p.d_hinv + src * 9;
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) atomicAdd(gh + a * 3 + b, gw[a] * ray[b]);
  }
}

__global__ void __launch_bounds__(256) geom_backward_kernel(const double* __restrict__ surfels,
                                                            const SurfRec* __restrict__ recs,
                                                            const int32_t* __restrict__ valid, int64_t n,
                                                            DevCamera cam, const double* __restrict__ d_hinv,
                                                            double* __restrict__ d_center, double* __restrict__ d_rot,
                                                            double* __restrict__ d_scales) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double dc[3] = {0, 0, 0}, dq[4] = {0, 0, 0, 0}, ds[2] = {0, 0};
  if (valid[i]) {  // projected surfels only (pipeline.cpp:478)
    double rc[9], gh[9];
    for (int k = 0; k < 9; ++k) {
      rc[k] = cam.r[k];
      gh[k] = d_hinv[i * 9 + k];
    }
    psm_geom_backward(surfels + i * 13, rc, recs[i].h, gh, dc, dq, ds);
  }
  for (int k = 0; k < 3; ++k) d_center[i * 3 + k] = dc[k];
  for (int k = 0; k < 4; ++k) d_rot[i * 4 + k] = dq[k];
  for (int k = 0; k < 2; ++k) d_scales[i * 2 + k] = ds[k];
}

}  // namespace

void launch_pixel_backward(const BackwardParams& p, cudaStream_t st) {
  const int64_t npx = static_cast<int64_t>(p.width) * p.height;
  if (npx <= 0) return;
  pixel_backward_kernel<<<static_cast<unsigned>((npx + 255) / 256), 256, 0, st>>>(p);
}

void launch_geom_backward(const double* surfels, const SurfRec* recs, const int32_t* valid, int64_t n,
                          const DevCamera& cam, const double* d_hinv, double* d_center, double* d_rot,
                          double* d_scales, cudaStream_t st) {
  if (n <= 0) return;
  geom_backward_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(surfels, recs, valid, n, cam, d_hinv,
                                                                               d_center, d_rot, d_scales);
}

}  // namespace psm
