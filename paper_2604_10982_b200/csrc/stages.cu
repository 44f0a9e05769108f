// stages.cu — the reference's stage functions as device-backed batch entry points
// (include/psm.h "Stage entry points"; reference: proj/include/psimap/raster.hpp:87-126):
//
//   psm_project_surfels  project_surfel            raster.cpp:94-142   (psm_project.cuh, shared with K1)
//   psm_bin_projected    bin_circle / bin_aabb     raster.cpp:51-90,144-152
//   psm_sample_alpha     sample_surfel_alpha +     raster.cpp:154-177
//                        evaluate_alpha
//   psm_topk_select      topk_select               raster.cpp:225-251
//
// They are not on the frame's hot path (the render pipeline inlines its own forms of
// these steps); they exist so that callers of the reference's stage API (acceptance.cpp,
// pipeline.cpp:387) drop in unchanged. Arithmetic follows the reference bit for bit
// (--fmad=false, psm_exp for glibc exp). Inputs and outputs are host arrays; device
// memory is per call (stream-ordered allocations on the context stream).
#include <algorithm>
#include <cstring>
#include <numeric>
#include <vector>

#include "psm_ctx.h"
#include "psm_ellipse.h"
#include "psm_exp.h"
#include "psm_kernels.h"
#include "psm_project.cuh"

namespace psm {
namespace {

int sfail(psm_ctx* ctx, int code, const char* msg) {
  if (ctx) ctx->err = msg;
  return code;
}

// Stream-ordered scratch for one call.
struct Tmp {
  cudaStream_t st;
  std::vector<void*> ps;
  explicit Tmp(cudaStream_t s) : st(s) {}
  ~Tmp() {
    for (void* p : ps) cudaFreeAsync(p, st);
  }
  template <class T>
  cudaError_t get(T** out, size_t count) {
    void* p = nullptr;
    const cudaError_t e = cudaMallocAsync(&p, sizeof(T) * (count > 0 ? count : 1), st);
    if (e == cudaSuccess) ps.push_back(p);
    *out = static_cast<T*>(p);
    return e;
  }
};

DevCamera dev_camera(const psm_camera* c) {
  DevCamera d;
  std::memcpy(d.r, c->r_cw, sizeof d.r);
  std::memcpy(d.t, c->t_cw, sizeof d.t);
  d.fx = c->fx; d.fy = c->fy; d.cx = c->cx; d.cy = c->cy;
  d.w = c->width; d.h = c->height;
  d.near_clip = c->near_clip; d.far_clip = c->far_clip;
  return d;
}

// ---------------------------------------------------------------- project_surfel
__global__ void project_batch_kernel(const double* __restrict__ s13, int64_t n, DevCamera cam, double chi2,
                                     psm_projected* __restrict__ out, int32_t* __restrict__ status,
                                     unsigned long long* __restrict__ first_bad) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  ProjFull f;
  const int st = psm_project(s13 + 13 * i, cam, chi2, f);
  status[i] = st > 0 ? 1 : 0;
  if (st < 0) atomicMin(first_bad, static_cast<unsigned long long>(i));
  if (st != 1) return;
  psm_projected p;
  p.source = -1;  // raster.cpp:140: the caller fills the scene index
  p.pad = 0;
  p.screen_center[0] = f.cx;
  p.screen_center[1] = f.cy;
  p.sigma[0] = f.sg00; p.sigma[1] = f.sg01; p.sigma[2] = f.sg01; p.sigma[3] = f.sg11;
  p.sort_depth = f.pc2;
  p.h[0] = f.a0; p.h[1] = f.a1; p.h[2] = f.a2;     // column 0: a
  p.h[3] = f.b0; p.h[4] = f.b1; p.h[5] = f.b2;     // column 1: b
  p.h[6] = f.pc0; p.h[7] = f.pc1; p.h[8] = f.pc2;  // column 2: p_cam
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) p.h_inv[c * 3 + r] = f.h[r * 3 + c];
  // finv << f(1,1), -f(0,1), -f(1,0), f(0,0); footprint_inv = finv / fdet (raster.cpp:132-136)
  p.footprint_inv[0] = f.F11 / f.fdet;
  p.footprint_inv[1] = -f.F01 / f.fdet;  // (1, 0): -f(1,0), f symmetric
  p.footprint_inv[2] = -f.F01 / f.fdet;  // (0, 1)
  p.footprint_inv[3] = f.F00 / f.fdet;
  p.normal_vis[0] = f.sgn * f.r02;
  p.normal_vis[1] = f.sgn * f.r12;
  p.normal_vis[2] = f.sgn * f.r22;
  out[i] = p;
}

// ---------------------------------------------------------------- bin_circle / bin_aabb
// Order-preserving unsigned key of a double (negative values reversed below positive ones).
__device__ __forceinline__ uint64_t order_key(double d) {
  const uint64_t b = static_cast<uint64_t>(__double_as_longlong(d));
  return (b >> 63) ? ~b : (b | (1ull << 63));
}

struct TileRect {
  int tx0, tx1, ty0, ty1;
};

// The box of bin_boxes (raster.cpp:59-68) from a ProjectedSurfel: circle_box
// (raster.cpp:37-41) or aabb_box (raster.cpp:43-49), both over footprint_cov(sigma).
__device__ __forceinline__ TileRect tile_rect(const psm_projected& p, int circle, double chi2_circle, double chi2,
                                              int ts, int tiles_x, int tiles_y) {
  const double f00 = p.sigma[0] + 0.3, f11 = p.sigma[3] + 0.3;
  const double f01 = p.sigma[2], f10 = p.sigma[1];
  double x0, x1, y0, y1;
  if (circle) {
    const double half_tr = 0.5 * (f00 + f11);
    const double det = f00 * f11 - f01 * f10;
    const double dd = half_tr * half_tr - det;
    const double disc = sqrt(dd < 0.0 ? 0.0 : dd);
    const double r = sqrt(chi2_circle * (half_tr + disc));
    x0 = p.screen_center[0] - r; x1 = p.screen_center[0] + r;
    y0 = p.screen_center[1] - r; y1 = p.screen_center[1] + r;
  } else {
    const double dx = sqrt(chi2 * f00), dy = sqrt(chi2 * f11);
    x0 = p.screen_center[0] - dx; x1 = p.screen_center[0] + dx;
    y0 = p.screen_center[1] - dy; y1 = p.screen_center[1] + dy;
  }
  TileRect t;
  t.tx0 = max(x86_cvt(floor(psm_div_tile(x0, ts))), 0);
  t.tx1 = min(x86_cvt(floor(psm_div_tile(x1, ts))), tiles_x - 1);
  t.ty0 = max(x86_cvt(floor(psm_div_tile(y0, ts))), 0);
  t.ty1 = min(x86_cvt(floor(psm_div_tile(y1, ts))), tiles_y - 1);
  return t;
}

// keys[j] / vals[j] for the j-th projected surfel in (source, index) order.
__global__ void bin_keys_kernel(const psm_projected* __restrict__ proj, const int32_t* __restrict__ by_source,
                                int64_t n, uint64_t* __restrict__ keys, uint32_t* __restrict__ vals) {
  const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int32_t i = by_source[j];
  keys[j] = order_key(proj[i].sort_depth);
  vals[j] = static_cast<uint32_t>(i);
}

// Per rank r (the (sort_depth, source) order): the number of tiles of the surfel's box.
__global__ void bin_count_kernel(const psm_projected* __restrict__ proj, const uint32_t* __restrict__ order,
                                 int64_t n, int circle, double chi2_circle, double chi2, int ts, int tiles_x,
                                 int tiles_y, int32_t* __restrict__ counts) {
  const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const TileRect t = tile_rect(proj[order[r]], circle, chi2_circle, chi2, ts, tiles_x, tiles_y);
  counts[r] = (t.tx0 <= t.tx1 && t.ty0 <= t.ty1) ? (t.tx1 - t.tx0 + 1) * (t.ty1 - t.ty0 + 1) : 0;
}

// (tile, projected index) pairs in rank order; per-tile counts.
__global__ void bin_emit_kernel(const psm_projected* __restrict__ proj, const uint32_t* __restrict__ order,
                                const uint32_t* __restrict__ offs, int64_t n, int circle, double chi2_circle,
                                double chi2, int ts, int tiles_x, int tiles_y, uint32_t* __restrict__ pair_tile,
                                uint32_t* __restrict__ pair_val, uint32_t* __restrict__ tile_counts) {
  const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const uint32_t i = order[r];
  const TileRect t = tile_rect(proj[i], circle, chi2_circle, chi2, ts, tiles_x, tiles_y);
  uint32_t o = offs[r];
  for (int ty = t.ty0; ty <= t.ty1; ++ty)
    for (int tx = t.tx0; tx <= t.tx1; ++tx) {
      const uint32_t tile = static_cast<uint32_t>(ty * tiles_x + tx);
      pair_tile[o] = tile;
      pair_val[o] = i;
      atomicAdd(tile_counts + tile, 1u);
      ++o;
    }
}

// ---------------------------------------------------------------- sample / evaluate alpha
__global__ void alpha_batch_kernel(const psm_projected* __restrict__ proj, const double* __restrict__ opacity,
                                   int64_t n_proj, const int32_t* __restrict__ idx, const double* __restrict__ px,
                                   const double* __restrict__ py, int64_t m, double cam_cx, double cam_cy,
                                   double cam_fx, double cam_fy, int support_cutoff, double chi2, double alpha_min,
                                   psm_alpha_sample* __restrict__ out, int32_t* __restrict__ bad) {
  const int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= m) return;
  psm_alpha_sample o;
  o.alpha = 0; o.u = 0; o.v = 0; o.w2 = 0; o.inside = 0; o.pad = 0;
  const int32_t k = idx[q];
  if (k < 0 || k >= n_proj) {
    atomicOr(bad, 1);
    out[q] = o;
    return;
  }
  const psm_projected& p = proj[k];
  const double x = px[q], y = py[q];
  bool pass = true;
  if (support_cutoff) {  // d.dot(footprint_inv * d) > chi2 (raster.cpp:157-160)
    const double d0 = x - p.screen_center[0], d1 = y - p.screen_center[1];
    const double fd0 = p.footprint_inv[0] * d0 + p.footprint_inv[2] * d1;
    const double fd1 = p.footprint_inv[1] * d0 + p.footprint_inv[3] * d1;
    pass = !(d0 * fd0 + d1 * fd1 > chi2);
  }
  if (pass) {
    // ray (raster.cpp:161), w = h_inv * ray (the 1.0 multiply is exact)
    const double rx = (x - cam_cx) / cam_fx, ry = (y - cam_cy) / cam_fy;
    const double* hi = p.h_inv;
    const double w0 = (hi[0] * rx + hi[3] * ry) + hi[6] * 1.0;
    const double w1 = (hi[1] * rx + hi[4] * ry) + hi[7] * 1.0;
    const double w2 = (hi[2] * rx + hi[5] * ry) + hi[8] * 1.0;
    if (w2 > 1e-14) {  // raster.cpp:163
      o.u = w0 / w2;
      o.v = w1 / w2;
      o.w2 = w2;
      o.inside = 1;
      const double a = opacity[k] * psm_exp(-0.5 * (o.u * o.u + o.v * o.v));  // raster.cpp:175
      o.alpha = a < alpha_min ? 0.0 : a;
    }
  }
  out[q] = o;
}

// ---------------------------------------------------------------- topk_select
// One thread per list: the reference's insertion select into a scratch of k entries.
__global__ void topk_batch_kernel(const double* __restrict__ w, const int32_t* __restrict__ proj,
                                  const int64_t* __restrict__ offs, int n_lists, int k, int32_t* __restrict__ best,
                                  int8_t* __restrict__ selected) {
  const int l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= n_lists) return;
  const int64_t b = offs[l], e = offs[l + 1];
  const int m = static_cast<int>(e - b);
  if (k >= m) {  // raster.cpp:228-231
    for (int i = 0; i < m; ++i) selected[b + i] = 1;
    return;
  }
  for (int i = 0; i < m; ++i) selected[b + i] = 0;
  int32_t* bs = best + b;  // scratch: list positions of the k best so far (k < m slots)
  auto before = [&](int a, int c) {  // raster.cpp:232-235
    if (w[b + a] != w[b + c]) return w[b + a] > w[b + c];
    return proj[b + a] < proj[b + c];
  };
  int filled = 0;
  for (int i = 0; i < m; ++i) {
    if (filled == k && !before(i, bs[k - 1])) continue;
    int pos = filled == k ? k - 1 : filled;
    if (filled < k) ++filled;
    while (pos > 0 && before(i, bs[pos - 1])) {
      bs[pos] = bs[pos - 1];
      --pos;
    }
    bs[pos] = i;
  }
  for (int i = 0; i < filled; ++i) selected[b + bs[i]] = 1;
}

int grid_for(int64_t n, int t) { return static_cast<int>((n + t - 1) / t); }

// ---------------------------------------------------------------- RenderCache
// RenderCache::pixels (raster.cpp:399-403): each pixel's contributors in blend order as
// (index into the projected list, alpha, u, v). The cache-mode forward recorded every
// contributor's tile-list position; alpha, u and v are recomputed from the staged record
// with the blend's own expressions (raster.cpp:369-390), so they are the reference's bits.
__global__ void cache_pixels_kernel(const uint2* __restrict__ lists, int list_cap, const int32_t* __restrict__ cnt,
                                    const int64_t* __restrict__ offs, const uint32_t* __restrict__ vals,
                                    const SurfRec* __restrict__ recs, const uint32_t* __restrict__ proj_of,
                                    int width, int height, double cam_cx, double cam_cy, double cam_fx,
                                    double cam_fy, psm_contribution* __restrict__ out) {
  const int64_t pix = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (pix >= static_cast<int64_t>(width) * height) return;
  const int x = static_cast<int>(pix % width), y = static_cast<int>(pix / width);
  const double px = x + 0.5, py = y + 0.5;
  const double rx = (px - cam_cx) / cam_fx;
  const double ry = (py - cam_cy) / cam_fy;
  const int m = cnt[pix] < list_cap ? cnt[pix] : list_cap;
  int64_t o = offs[pix];
  for (int k = 0; k < m; ++k, ++o) {
    const uint32_t src = vals[lists[psm_list_index(x, y, width, list_cap, k)].x];
    const SurfRec& r = recs[src];
    const double w0 = r.h[0] * rx + r.h[1] * ry + r.h[2];
    const double w1 = r.h[3] * rx + r.h[4] * ry + r.h[5];
    const double w2 = r.h[6] * rx + r.h[7] * ry + r.h[8];
    const double rcp = 1.0 / w2;
    const double u = w0 * rcp, v = w1 * rcp;
    psm_contribution c;
    c.proj = static_cast<int32_t>(proj_of[src]);
    c.pad = 0;
    c.alpha = r.opacity * psm_exp(-0.5 * (u * u + v * v));
    c.u = u;
    c.v = v;
    out[o] = c;
  }
}

// projected[proj_of[i]] = project_surfel(surfel i) with its source, for every projecting i
__global__ void cache_projected_kernel(const double* __restrict__ s13, int64_t n, DevCamera cam, double chi2,
                                       const int32_t* __restrict__ valid, const uint32_t* __restrict__ proj_of,
                                       psm_projected* __restrict__ out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n || !valid[i]) return;
  ProjFull f;
  if (psm_project(s13 + 13 * i, cam, chi2, f) != 1) return;
  psm_projected p;
  p.source = static_cast<int32_t>(i);
  p.pad = 0;
  p.screen_center[0] = f.cx;
  p.screen_center[1] = f.cy;
  p.sigma[0] = f.sg00; p.sigma[1] = f.sg01; p.sigma[2] = f.sg01; p.sigma[3] = f.sg11;
  p.sort_depth = f.pc2;
  p.h[0] = f.a0; p.h[1] = f.a1; p.h[2] = f.a2;
  p.h[3] = f.b0; p.h[4] = f.b1; p.h[5] = f.b2;
  p.h[6] = f.pc0; p.h[7] = f.pc1; p.h[8] = f.pc2;
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) p.h_inv[c * 3 + r] = f.h[r * 3 + c];
  p.footprint_inv[0] = f.F11 / f.fdet;
  p.footprint_inv[1] = -f.F01 / f.fdet;
  p.footprint_inv[2] = -f.F01 / f.fdet;
  p.footprint_inv[3] = f.F00 / f.fdet;
  p.normal_vis[0] = f.sgn * f.r02;
  p.normal_vis[1] = f.sgn * f.r12;
  p.normal_vis[2] = f.sgn * f.r22;
  out[proj_of[i]] = p;
}

__global__ void gather_proj_kernel(const uint32_t* __restrict__ vals, const uint32_t* __restrict__ proj_of, int64_t n,
                                   int32_t* __restrict__ out) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e < n) out[e] = static_cast<int32_t>(proj_of[vals[e]]);
}

}  // namespace

void launch_cache_pixels(const uint2* lists, int list_cap, const int32_t* cnt, const int64_t* offs,
                         const uint32_t* vals, const SurfRec* recs, const uint32_t* proj_of, int width, int height,
                         double cx, double cy, double fx, double fy, psm_contribution* out, cudaStream_t st) {
  const int64_t npx = static_cast<int64_t>(width) * height;
  if (npx > 0)
    cache_pixels_kernel<<<grid_for(npx, 128), 128, 0, st>>>(lists, list_cap, cnt, offs, vals, recs, proj_of, width,
                                                            height, cx, cy, fx, fy, out);
}
void launch_cache_projected(const double* s13, int64_t n, const DevCamera& cam, double chi2, const int32_t* valid,
                            const uint32_t* proj_of, psm_projected* out, cudaStream_t st) {
  if (n > 0) cache_projected_kernel<<<grid_for(n, 128), 128, 0, st>>>(s13, n, cam, chi2, valid, proj_of, out);
}
void launch_gather_proj(const uint32_t* vals, const uint32_t* proj_of, int64_t n, int32_t* out, cudaStream_t st) {
  if (n > 0) gather_proj_kernel<<<grid_for(n, 256), 256, 0, st>>>(vals, proj_of, n, out);
}
}  // namespace psm

using psm::sfail;

extern "C" {

int psm_project_surfels(psm_ctx* ctx, const double* surfels13, int64_t n, const psm_camera* cam,
                        const psm_raster_config* cfg, psm_projected* out, int32_t* status, int64_t* bad_index) {
  if (!ctx || !cam || !cfg || n < 0 || (n > 0 && (!surfels13 || !out || !status)))
    return sfail(ctx, PSM_EINVAL, "project_surfels: bad arguments");
  if (bad_index) *bad_index = -1;
  if (n == 0) return PSM_OK;
  PSM_CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  psm::Tmp tmp(st);
  double* ds;
  psm_projected* dp;
  int32_t* dst;
  unsigned long long* dbad;
  PSM_CUDA_TRY(tmp.get(&ds, static_cast<size_t>(n) * 13));
  PSM_CUDA_TRY(tmp.get(&dp, static_cast<size_t>(n)));
  PSM_CUDA_TRY(tmp.get(&dst, static_cast<size_t>(n)));
  PSM_CUDA_TRY(tmp.get(&dbad, 1));
  PSM_CUDA_TRY(cudaMemcpyAsync(ds, surfels13, sizeof(double) * 13 * n, cudaMemcpyHostToDevice, st));
  PSM_CUDA_TRY(cudaMemsetAsync(dbad, 0xff, sizeof(unsigned long long), st));
  psm::project_batch_kernel<<<psm::grid_for(n, 128), 128, 0, st>>>(ds, n, psm::dev_camera(cam), cfg->chi2, dp, dst,
                                                                   dbad);
  PSM_CUDA_TRY(cudaGetLastError());
  unsigned long long hbad = ~0ull;
  PSM_CUDA_TRY(cudaMemcpyAsync(status, dst, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, st));
  PSM_CUDA_TRY(cudaMemcpyAsync(out, dp, sizeof(psm_projected) * n, cudaMemcpyDeviceToHost, st));
  PSM_CUDA_TRY(cudaMemcpyAsync(&hbad, dbad, sizeof hbad, cudaMemcpyDeviceToHost, st));
  PSM_CUDA_TRY(cudaStreamSynchronize(st));
  if (hbad != ~0ull) {
    if (bad_index) *bad_index = static_cast<int64_t>(hbad);
    return sfail(ctx, PSM_EINVAL, "degenerate quaternion");
  }
  return PSM_OK;
}

int psm_bin_projected(psm_ctx* ctx, const psm_projected* projected, int64_t n, const psm_camera* cam,
                      const psm_raster_config* cfg, int32_t binning, double chi2, int32_t* tile_counts, int32_t* list,
                      int64_t cap, psm_counters* counters) {
  if (!ctx || !cam || !cfg || n < 0 || (n > 0 && !projected) || !tile_counts)
    return sfail(ctx, PSM_EINVAL, "bin_projected: bad arguments");
  if (binning != PSM_BIN_CIRCLE && binning != PSM_BIN_AABB) return sfail(ctx, PSM_EINVAL, "bin_projected: binning");
  if (cfg->tile_size <= 0 || cam->width <= 0 || cam->height <= 0) return sfail(ctx, PSM_EINVAL, "bin_projected: grid");
  if (n > 0x7fffffffLL) return sfail(ctx, PSM_EUNSUPPORTED, "bin_projected: more than 2^31 - 1 surfels");
  const int ts = cfg->tile_size;
  const int tiles_x = (cam->width + ts - 1) / ts, tiles_y = (cam->height + ts - 1) / ts;
  const int64_t tiles = static_cast<int64_t>(tiles_x) * tiles_y;
  PSM_CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  psm::Tmp tmp(st);
  // input order (source, index): the stable depth sort then gives (sort_depth, source) (raster.cpp:78-83)
  std::vector<int32_t> by_source(static_cast<size_t>(n));
  std::iota(by_source.begin(), by_source.end(), 0);
  std::stable_sort(by_source.begin(), by_source.end(),
                   [&](int32_t a, int32_t b) { return projected[a].source < projected[b].source; });
  psm_projected* dp;
  int32_t* dsrc;
  uint64_t *keys, *keys2;
  uint32_t *vals, *vals2, *hist, *totals, *n_dev, *offs, *scan_cta, *rn_dev, *tcount;
  int32_t* counts;
  const size_t nn = static_cast<size_t>(n > 0 ? n : 1);
  PSM_CUDA_TRY(tmp.get(&dp, nn));
  PSM_CUDA_TRY(tmp.get(&dsrc, nn));
  PSM_CUDA_TRY(tmp.get(&keys, nn));
  PSM_CUDA_TRY(tmp.get(&keys2, nn));
  PSM_CUDA_TRY(tmp.get(&vals, nn));
  PSM_CUDA_TRY(tmp.get(&vals2, nn));
  PSM_CUDA_TRY(tmp.get(&hist, psm::radix_hist_words(n) + 16));
  PSM_CUDA_TRY(tmp.get(&totals, 256));
  PSM_CUDA_TRY(tmp.get(&n_dev, 1));
  PSM_CUDA_TRY(tmp.get(&counts, nn));
  PSM_CUDA_TRY(tmp.get(&offs, nn));
  PSM_CUDA_TRY(tmp.get(&scan_cta, psm::scan_cta_words(n) + 8));
  PSM_CUDA_TRY(tmp.get(&rn_dev, 1));
  PSM_CUDA_TRY(tmp.get(&tcount, static_cast<size_t>(tiles)));
  PSM_CUDA_TRY(cudaMemsetAsync(tcount, 0, sizeof(uint32_t) * tiles, st));
  PSM_CUDA_TRY(cudaMemsetAsync(rn_dev, 0, sizeof(uint32_t), st));
  uint32_t rn = 0;
  const uint32_t* order = vals;
  if (n > 0) {
    PSM_CUDA_TRY(cudaMemcpyAsync(dp, projected, sizeof(psm_projected) * n, cudaMemcpyHostToDevice, st));
    PSM_CUDA_TRY(cudaMemcpyAsync(dsrc, by_source.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice, st));
    const uint32_t nu = static_cast<uint32_t>(n);
    PSM_CUDA_TRY(cudaMemcpyAsync(n_dev, &nu, sizeof nu, cudaMemcpyHostToDevice, st));
    psm::bin_keys_kernel<<<psm::grid_for(n, 256), 256, 0, st>>>(dp, dsrc, n, keys, vals);
    bool in_alt = false;
    psm::radix_sort_u64(keys, vals, keys2, vals2, n_dev, n, 0, 64, hist, totals, st, &in_alt);
    order = in_alt ? vals2 : vals;
    const int circle = binning == PSM_BIN_CIRCLE;
    psm::bin_count_kernel<<<psm::grid_for(n, 256), 256, 0, st>>>(dp, order, n, circle, cfg->chi2, chi2, ts, tiles_x,
                                                                 tiles_y, counts);
    psm::exclusive_scan_i32(counts, n, offs, rn_dev, scan_cta, st);
    PSM_CUDA_TRY(cudaGetLastError());
    PSM_CUDA_TRY(cudaMemcpyAsync(&rn, rn_dev, sizeof rn, cudaMemcpyDeviceToHost, st));
    PSM_CUDA_TRY(cudaStreamSynchronize(st));
  }
  std::vector<uint32_t> hcount(static_cast<size_t>(tiles), 0u);
  if (rn > 0) {
    uint32_t *ptile, *pval, *ptile2, *pval2, *hist2, *rn_n;
    PSM_CUDA_TRY(tmp.get(&ptile, rn));
    PSM_CUDA_TRY(tmp.get(&pval, rn));
    PSM_CUDA_TRY(tmp.get(&ptile2, rn));
    PSM_CUDA_TRY(tmp.get(&pval2, rn));
    PSM_CUDA_TRY(tmp.get(&hist2, psm::radix_hist_words(rn) + 16));
    PSM_CUDA_TRY(tmp.get(&rn_n, 1));
    PSM_CUDA_TRY(cudaMemcpyAsync(rn_n, &rn, sizeof rn, cudaMemcpyHostToDevice, st));
    psm::bin_emit_kernel<<<psm::grid_for(n, 128), 128, 0, st>>>(dp, order, offs, n, binning == PSM_BIN_CIRCLE,
                                                                cfg->chi2, chi2, ts, tiles_x, tiles_y, ptile, pval,
                                                                tcount);
    int bits = 1;
    while ((1ll << bits) < tiles) ++bits;
    bool in_alt = false;
    psm::radix_sort_u32(ptile, pval, ptile2, pval2, rn_n, rn, 0, bits, hist2, totals, st, &in_alt);
    PSM_CUDA_TRY(cudaGetLastError());
    PSM_CUDA_TRY(cudaMemcpyAsync(hcount.data(), tcount, sizeof(uint32_t) * tiles, cudaMemcpyDeviceToHost, st));
    if (list && cap >= static_cast<int64_t>(rn))
      PSM_CUDA_TRY(cudaMemcpyAsync(list, in_alt ? pval2 : pval, sizeof(uint32_t) * rn, cudaMemcpyDeviceToHost, st));
    PSM_CUDA_TRY(cudaStreamSynchronize(st));
  }
  int64_t nonempty = 0;
  for (int64_t t = 0; t < tiles; ++t) {
    tile_counts[t] = static_cast<int32_t>(hcount[t]);
    nonempty += hcount[t] > 0;
  }
  if (counters) {  // raster.cpp:75-88
    std::memset(counters, 0, sizeof *counters);
    counters->rn_total = rn;
    counters->rn_per_tile = nonempty > 0 ? static_cast<double>(rn) / nonempty : 0.0;
    counters->n_proj = n;
    counters->tiles_x = tiles_x;
    counters->tiles_y = tiles_y;
    counters->nonempty_tiles = nonempty;
  }
  return PSM_OK;
}

int psm_sample_alpha(psm_ctx* ctx, const psm_projected* projected, const double* opacity, int64_t n_projected,
                     const int32_t* proj_index, const double* px, const double* py, int64_t m,
                     const psm_camera* cam, const psm_raster_config* cfg, psm_alpha_sample* out) {
  if (!ctx || !cam || !cfg || m < 0 || n_projected < 0 ||
      (m > 0 && (!projected || !opacity || !proj_index || !px || !py || !out)))
    return sfail(ctx, PSM_EINVAL, "sample_alpha: bad arguments");
  if (m == 0) return PSM_OK;
  PSM_CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  psm::Tmp tmp(st);
  psm_projected* dp;
  double *dop, *dx, *dy;
  int32_t *di, *dbad;
  psm_alpha_sample* dout;
  const size_t np = static_cast<size_t>(n_projected), mm = static_cast<size_t>(m);
  PSM_CUDA_TRY(tmp.get(&dp, np));
  PSM_CUDA_TRY(tmp.get(&dop, np));
  PSM_CUDA_TRY(tmp.get(&di, mm));
  PSM_CUDA_TRY(tmp.get(&dx, mm));
  PSM_CUDA_TRY(tmp.get(&dy, mm));
  PSM_CUDA_TRY(tmp.get(&dout, mm));
  PSM_CUDA_TRY(tmp.get(&dbad, 1));
  if (np) {
    PSM_CUDA_TRY(cudaMemcpyAsync(dp, projected, sizeof(psm_projected) * np, cudaMemcpyHostToDevice, st));
    PSM_CUDA_TRY(cudaMemcpyAsync(dop, opacity, sizeof(double) * np, cudaMemcpyHostToDevice, st));
  }
  PSM_CUDA_TRY(cudaMemcpyAsync(di, proj_index, sizeof(int32_t) * mm, cudaMemcpyHostToDevice, st));
  PSM_CUDA_TRY(cudaMemcpyAsync(dx, px, sizeof(double) * mm, cudaMemcpyHostToDevice, st));
  PSM_CUDA_TRY(cudaMemcpyAsync(dy, py, sizeof(double) * mm, cudaMemcpyHostToDevice, st));
  PSM_CUDA_TRY(cudaMemsetAsync(dbad, 0, sizeof(int32_t), st));
  psm::alpha_batch_kernel<<<psm::grid_for(m, 128), 128, 0, st>>>(dp, dop, n_projected, di, dx, dy, m, cam->cx, cam->cy,
                                                                 cam->fx, cam->fy, cfg->support_cutoff != 0, cfg->chi2,
                                                                 cfg->alpha_min, dout, dbad);
  PSM_CUDA_TRY(cudaGetLastError());
  int32_t hbad = 0;
  PSM_CUDA_TRY(cudaMemcpyAsync(out, dout, sizeof(psm_alpha_sample) * mm, cudaMemcpyDeviceToHost, st));
  PSM_CUDA_TRY(cudaMemcpyAsync(&hbad, dbad, sizeof hbad, cudaMemcpyDeviceToHost, st));
  PSM_CUDA_TRY(cudaStreamSynchronize(st));
  return hbad ? sfail(ctx, PSM_EINVAL, "sample_alpha: projected index out of range") : PSM_OK;
}

int psm_topk_select(psm_ctx* ctx, const double* weights, const int32_t* proj, const int64_t* offsets,
                    int32_t n_lists, int32_t k, int8_t* selected) {
  if (!ctx || n_lists < 0 || !offsets || (n_lists > 0 && (!selected)))
    return sfail(ctx, PSM_EINVAL, "topk_select: bad arguments");
  if (n_lists == 0) return PSM_OK;
  const int64_t total = offsets[n_lists];
  if (offsets[0] != 0 || total < 0) return sfail(ctx, PSM_EINVAL, "topk_select: offsets");
  for (int32_t l = 0; l < n_lists; ++l)
    if (offsets[l + 1] < offsets[l]) return sfail(ctx, PSM_EINVAL, "topk_select: offsets");
  if (total > 0 && (!weights || !proj)) return sfail(ctx, PSM_EINVAL, "topk_select: bad arguments");
  if (k < 1) return sfail(ctx, PSM_EINVAL, "topk_select: k must be >= 1 (render uses max(top_k, 1))");
  PSM_CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  psm::Tmp tmp(st);
  double* dw;
  int32_t *dp, *best;
  int64_t* doff;
  int8_t* dsel;
  const size_t tt = static_cast<size_t>(total);
  PSM_CUDA_TRY(tmp.get(&dw, tt));
  PSM_CUDA_TRY(tmp.get(&dp, tt));
  PSM_CUDA_TRY(tmp.get(&best, tt));
  PSM_CUDA_TRY(tmp.get(&dsel, tt));
  PSM_CUDA_TRY(tmp.get(&doff, static_cast<size_t>(n_lists) + 1));
  if (tt) {
    PSM_CUDA_TRY(cudaMemcpyAsync(dw, weights, sizeof(double) * tt, cudaMemcpyHostToDevice, st));
    PSM_CUDA_TRY(cudaMemcpyAsync(dp, proj, sizeof(int32_t) * tt, cudaMemcpyHostToDevice, st));
  }
  PSM_CUDA_TRY(cudaMemcpyAsync(doff, offsets, sizeof(int64_t) * (n_lists + 1), cudaMemcpyHostToDevice, st));
  psm::topk_batch_kernel<<<psm::grid_for(n_lists, 128), 128, 0, st>>>(dw, dp, doff, n_lists, k, best, dsel);
  PSM_CUDA_TRY(cudaGetLastError());
  if (tt) PSM_CUDA_TRY(cudaMemcpyAsync(selected, dsel, tt, cudaMemcpyDeviceToHost, st));
  PSM_CUDA_TRY(cudaStreamSynchronize(st));
  return PSM_OK;
}

}  // extern "C"
