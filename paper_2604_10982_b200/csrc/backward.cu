// backward.cu — the render backward on the device: the blending
// backward of the training pipeline (proj/src/pipeline.cpp:347-460) and the geometry
// chain project_surfel_backward (raster.cpp:179-203, psm_backward.h).
//
// The forward runs first in cache mode (blend.cu with lists_t): every pixel's
// contributors in blend order as (list position, transmittance before the blend), plus
// the Top-K positions — RenderCache::pixels (raster.cpp:399-403). Here each warp takes an
// 8x4 pixel block of a tile and walks the union of its pixels' contributor lists from
// the back; every pixel does the reference's reverse step (pipeline.cpp:393-452): alpha,
// u, v recomputed from the staged record with the forward's fp64 arithmetic (so they
// are the forward's bits), the suffix of w_i <g, value_i> seeded with the background
// term. The per-surfel sums are reduced over the warp's pixels first and then added
// with one fp64 atomic per parameter (their order, and so the last bits, differ from
// the reference's chunked merge). A second kernel chains each projected surfel's
// dL/dH^-1 to its centre, quaternion and scales.
#include <cstdint>

#include "psm_backward.h"
#include "psm_device.cuh"
#include "psm_exp.h"
#include "psm_kernels.h"

namespace psm {
namespace {

// candidates owned by at most this many lanes add their terms lane by lane (no reduction).
// C3 pixel backward (ms): always reduce 3.62-3.66, <= 2 lanes 3.65, 4 3.61, 8 3.56-3.60,
// 12 3.60-3.62, 16 3.73, always direct 7.0 (fp64 atomics then dominate)
#ifndef PSM_BWD_DIRECT
#define PSM_BWD_DIRECT 8
#endif

// Sum over the warp of 16 per-lane values by recursive halving: after the five steps
// lane l holds the total of value (l >> 1) (both lanes of a pair hold it). 16 double
// shuffles instead of 16 x 5 for independent butterflies.
__device__ __forceinline__ double warp_sum16(double (&v)[16], int lane) {
#pragma unroll
  for (int k = 0; k < 8; ++k) {  // offset 16: keep half (by lane bit 4), receive the other half
    const bool hi = lane & 16;
    const double send = hi ? v[k] : v[k + 8];
    const double keep = hi ? v[k + 8] : v[k];
    v[k] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const bool hi = lane & 8;
    const double send = hi ? v[k] : v[k + 4];
    const double keep = hi ? v[k + 4] : v[k];
    v[k] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
  }
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const bool hi = lane & 4;
    const double send = hi ? v[k] : v[k + 2];
    const double keep = hi ? v[k + 2] : v[k];
    v[k] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
  }
  {
    const bool hi = lane & 2;
    const double send = hi ? v[0] : v[1];
    const double keep = hi ? v[1] : v[0];
    v[0] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
  }
  return v[0] + __shfl_xor_sync(0xffffffffu, v[0], 1);
}

__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

// One CTA per 16x16 tile, one warp per 8x4 pixel block (the forward's split), one lane
// per pixel. The warp walks the union of its pixels' contributor lists from the back
// (every list is a subsequence of the tile list, so the next candidate is the largest
// remaining list position over the lanes); the lanes owning the candidate do the
// reference's reverse step (pipeline.cpp:393-452) for their pixel, and the warp sums
// the candidate's gradient terms over its pixels before one atomic per parameter:
// colour 3, opacity 1, dL/dH^-1 9 (one lane each), and f_sem / label channels (lane
// per channel, for the pixels that selected the candidate).
// NCH: feature channel chunks of 32 handled per pass (ceil(D / 32), at most 4; wider rows
// take several passes).
template <int NCH>
__global__ void __launch_bounds__(256, 3) pixel_backward_kernel(BackwardParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint64_t* tab = reinterpret_cast<uint64_t*>(smem_raw);
  int* sel_pos = reinterpret_cast<int*>(tab + 256);  // [k_sel][256]: selected positions, descending
  tab[threadIdx.x] = psm_exp_tab_dev[threadIdx.x];
  const int tid = threadIdx.x, lane = tid & 31, blk = tid >> 5;
  const int tiles_x = (p.width + 15) / 16;
  const int tx = blockIdx.x % tiles_x, ty = blockIdx.x / tiles_x;
  const int x = tx * 16 + (blk & 1) * 8 + (lane & 7), y = ty * 16 + (blk >> 1) * 4 + (lane >> 3);
  const bool inside = x < p.width && y < p.height;
  const int64_t pix = inside ? static_cast<int64_t>(y) * p.width + x : 0;
  int m = inside ? p.blend_count[pix] : 0;
  if (m > p.list_cap) m = p.list_cap;  // the caller re-renders with a larger cap first
  const bool sel_all = !(p.topk && m > p.k_sel);
  int nsel = 0;
  if (!sel_all && p.topk_pos) {  // RenderCache::pixels' Top-K set, sorted by position, descending
    nsel = p.k_sel;
    for (int i = 0; i < nsel; ++i) {
      const int v = p.topk_pos[pix * p.k_sel + i];
      int k = i;
      while (k > 0 && sel_pos[(k - 1) * 256 + tid] < v) {
        sel_pos[k * 256 + tid] = sel_pos[(k - 1) * 256 + tid];
        --k;
      }
      sel_pos[k * 256 + tid] = v;
    }
  }
  __syncthreads();

  const double rx = (x + 0.5 - p.cam_cx) / p.cam_fx;
  const double ry = (y + 0.5 - p.cam_cy) / p.cam_fy;
  double gc0 = 0.0, gc1 = 0.0, gc2 = 0.0;
  if (p.g_color && inside) {
    gc0 = p.g_color[pix * 3 + 0];
    gc1 = p.g_color[pix * 3 + 1];
    gc2 = p.g_color[pix * 3 + 2];
  }
  const double* gf = p.c_sem > 0 ? p.g_sem : nullptr;  // kernel parameters: warp-uniform
  const double* gi = p.n_q > 0 ? p.g_ins : nullptr;
  const int cs = p.c_sem, nq = p.n_q, D = cs + nq;
  // this pixel's list: entry j at lst[32 j] / lt[32 j] (psm_list_index)
  const int64_t l0 = inside ? psm_list_index(x, y, p.width, p.list_cap, 0) : 0;
  const uint2* lst = p.lists + l0;
  const double* lt = p.lists_t + l0;

  // T after the last blend (the forward's chain continued from the stored T_{m-1}),
  // seeding the suffix with the background term
  double suffix = 0.0;
  if (m > 0) {
    const SurfRec& r = p.recs[__ldg(p.vals + lst[32 * (m - 1)].x)];
    const double w0 = r.h[0] * rx + r.h[1] * ry + r.h[2];
    const double w1 = r.h[3] * rx + r.h[4] * ry + r.h[5];
    const double w2 = r.h[6] * rx + r.h[7] * ry + r.h[8];
    const double rcp = 1.0 / w2;
    const double u = w0 * rcp, v = w1 * rcp;
    const double alpha = r.opacity * psm_exp_t(-0.5 * (u * u + v * v), tab);
    const double t_end = lt[32 * (m - 1)] * (1.0 - alpha);
    suffix = t_end * (gc0 * p.bg0 + gc1 * p.bg1 + gc2 * p.bg2);
  }
  // the lane's current contributor (position, T before it) and the next one, loaded a
  // step ahead so the walk's max-reduction does not wait on a fresh load
  int j = m - 1;
  int cur = j >= 0 ? static_cast<int>(lst[32 * (j)].x) : -1;
  double tcur = j >= 0 ? lt[32 * (j)] : 0.0;
  int nxt = j >= 1 ? static_cast<int>(lst[32 * (j - 1)].x) : -1;
  double tnxt = j >= 1 ? lt[32 * (j - 1)] : 0.0;
  int sp = 0;
  for (;;) {
    const int pos = __reduce_max_sync(0xffffffffu, cur);
    if (pos < 0) break;
    const bool mine = cur == pos;
    const uint32_t src = __ldg(p.vals + pos);
    const SurfRec& r = p.recs[src];
    // the forward's alpha (blend.cu, raster.cpp:383-392), bit for bit
    double u = 0, v = 0, rcp = 1, d_sigma = 0, alpha = 0, w_j = 0, t_j = 0;
    bool selected = false;
    if (mine) {
      t_j = tcur;
      const double w0 = r.h[0] * rx + r.h[1] * ry + r.h[2];
      const double w1 = r.h[3] * rx + r.h[4] * ry + r.h[5];
      const double w2 = r.h[6] * rx + r.h[7] * ry + r.h[8];
      rcp = 1.0 / w2;
      u = w0 * rcp;
      v = w1 * rcp;
      d_sigma = psm_exp_t(-0.5 * (u * u + v * v), tab);
      alpha = r.opacity * d_sigma;
      w_j = alpha * t_j;
      if (sel_all) {
        selected = true;
      } else if (sp < nsel && sel_pos[sp * 256 + tid] == pos) {
        selected = true;
        ++sp;
      }
    }
    // direct = <g_c, colour> + <g_sem, f_sem> + <g_ins, label> (pipeline.cpp:401-431)
    const double* sf = p.surfels + static_cast<int64_t>(src) * 13;
    double direct = mine ? gc0 * sf[10] + gc1 * sf[11] + gc2 * sf[12] : 0.0;
    const unsigned selm = __ballot_sync(0xffffffffu, selected);
    if (selm && (gf || gi)) {
      // Feature channels c = c0 + 32 ch + lane in groups of 4 chunks: per selected lane l,
      // its pixel's upstream gradient row is read once (coalesced), its weighted copy is
      // summed into the per-channel totals, and its dots with the candidate's row are
      // reduced over the warp (one reduction per dot for the whole group).
      const int64_t row = static_cast<int64_t>(src) * D;
      double dsem = 0.0, dins = 0.0;
      for (int c0 = 0; c0 < D; c0 += 32 * NCH) {
        double f[NCH], gacc[NCH];
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) {
          const int c = c0 + 32 * ch + lane;
          f[ch] = 0.0;
          gacc[ch] = 0.0;
          if (c < D) f[ch] = p.feat64 ? p.feat64[row + c] : static_cast<double>(p.feat32[row + c]);
        }
        for (unsigned mm = selm; mm;) {
          const int l = __ffs(mm) - 1;
          mm &= mm - 1;
          const int64_t pl = __shfl_sync(0xffffffffu, pix, l);
          const double wl = __shfl_sync(0xffffffffu, w_j, l);
          double g[NCH];
#pragma unroll
          for (int ch = 0; ch < NCH; ++ch) {
            const int c = c0 + 32 * ch + lane;
            g[ch] = 0.0;
            if (c < cs) {
              if (gf) g[ch] = gf[pl * cs + c];
            } else if (c < D) {
              if (gi) g[ch] = gi[pl * nq + (c - cs)];
            }
          }
          double ps = 0.0, pi = 0.0;
#pragma unroll
          for (int ch = 0; ch < NCH; ++ch) {
            const int c = c0 + 32 * ch + lane;
            gacc[ch] += wl * g[ch];
            if (c < cs) ps += g[ch] * f[ch];
            else pi += g[ch] * f[ch];
          }
          if (gf) ps = warp_sum(ps);
          if (gi) pi = warp_sum(pi);
          if (lane == l) {
            dsem += ps;
            dins += pi;
          }
        }
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) {
          const int c = c0 + 32 * ch + lane;
          if (c < cs) {
            if (gf) atomicAdd(p.d_fsem + static_cast<int64_t>(src) * cs + c, gacc[ch]);
          } else if (c < D) {
            if (gi) atomicAdd(p.d_lab + static_cast<int64_t>(src) * nq + (c - cs), gacc[ch]);
          }
        }
      }
      if (selected) {
        if (gf) direct += dsem;
        if (gi) direct += dins;
      }
    }
    double val[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) val[k] = 0.0;
    if (mine) {
      const double one_minus = 1.0 - alpha;
      const double g_alpha = t_j * direct - (one_minus > 0 ? suffix / one_minus : 0.0);
      suffix += w_j * direct;
      const double g_dsigma = r.opacity * g_alpha;
      const double g_u = -u * d_sigma * g_dsigma;
      const double g_v = -v * d_sigma * g_dsigma;
      // dL/dw = (g_u, g_v, -(u g_u + v g_v)) / w2 (pipeline.cpp:440-446), as products with
      // the forward's 1 / w2 (within an ulp of the quotients)
      const double gw[3] = {g_u * rcp, g_v * rcp, -(u * g_u + v * g_v) * rcp};
      const double ray[3] = {rx, ry, 1.0};
      val[0] = w_j * gc0;
      val[1] = w_j * gc1;
      val[2] = w_j * gc2;
      val[3] = d_sigma * g_alpha;
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) val[4 + a * 3 + b] = gw[a] * ray[b];
    }
    // few owners: each adds its own 13 terms; otherwise one warp reduction, one atomic each
    if (__popc(__ballot_sync(0xffffffffu, mine)) <= PSM_BWD_DIRECT) {
      if (mine) {
#pragma unroll
        for (int k = 0; k < 3; ++k) atomicAdd(p.d_color + static_cast<int64_t>(src) * 3 + k, val[k]);
        atomicAdd(p.d_opacity + src, val[3]);
#pragma unroll
        for (int k = 0; k < 9; ++k) atomicAdd(p.d_hinv + static_cast<int64_t>(src) * 9 + k, val[4 + k]);
      }
    } else {
      const double tot = warp_sum16(val, lane);
      const int k = lane >> 1;
      if (!(lane & 1) && k < 13) {
        double* dst = k < 3 ? p.d_color + static_cast<int64_t>(src) * 3 + k
                            : (k == 3 ? p.d_opacity + src : p.d_hinv + static_cast<int64_t>(src) * 9 + (k - 4));
        atomicAdd(dst, tot);
      }
    }
    if (mine) {
      --j;
      cur = nxt;
      tcur = tnxt;
      nxt = j >= 1 ? static_cast<int>(lst[32 * (j - 1)].x) : -1;
      tnxt = j >= 1 ? lt[32 * (j - 1)] : 0.0;
    }
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
  const int tiles = ((p.width + 15) / 16) * ((p.height + 15) / 16);
  const size_t smem = 256 * sizeof(uint64_t) + (p.topk ? static_cast<size_t>(p.k_sel) * 256 * sizeof(int) : 0);
  static unsigned long long configured = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(configured >> dev & 1ull)) {
    cudaFuncSetAttribute(pixel_backward_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2048 + 32 * 256 * 4);
    cudaFuncSetAttribute(pixel_backward_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2048 + 32 * 256 * 4);
    cudaFuncSetAttribute(pixel_backward_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2048 + 32 * 256 * 4);
    configured |= 1ull << dev;
  }
  const int nch = (p.c_sem + p.n_q + 31) / 32;
  if (nch <= 1) pixel_backward_kernel<1><<<tiles, 256, smem, st>>>(p);
  else if (nch <= 2) pixel_backward_kernel<2><<<tiles, 256, smem, st>>>(p);
  else pixel_backward_kernel<4><<<tiles, 256, smem, st>>>(p);
}

void launch_geom_backward(const double* surfels, const SurfRec* recs, const int32_t* valid, int64_t n,
                          const DevCamera& cam, const double* d_hinv, double* d_center, double* d_rot,
                          double* d_scales, cudaStream_t st) {
  if (n <= 0) return;
  geom_backward_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(surfels, recs, valid, n, cam, d_hinv,
                                                                               d_center, d_rot, d_scales);
}

}  // namespace psm
