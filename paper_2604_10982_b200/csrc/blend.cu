// blend.cu — K7: tile-based front-to-back compositing with register Top-K and
// warp-cooperative feature accumulation (reference: the tile loop of
// render_into, proj/src/raster.cpp:355-506, and topk_select, raster.cpp:225-251).
//
// One CTA per 16x16 tile, one thread per pixel. The tile's depth-sorted list
// (vals[start, end) from the tile sort) is streamed through shared memory in
// batches of 256 records (each thread stages one 144 B SurfRec, nine 16 B
// loads); every pixel then walks the batch in list order with the reference's
// fp64 arithmetic (compiled --fmad=false, psm_exp), so its contributor
// sequence, transmittance and Top-K set are bit-identical to the oracle's. The
// CTA leaves the list once every pixel has hit T < t_min (__syncthreads_count).
//
// Top-K: each thread keeps the KMAX best (weight desc, source asc) entries in
// registers by an unrolled insertion network (the reference's insertion select,
// raster.cpp:238-249; proj order == source order). Selection only changes the
// result when m > K, as in the reference (raster.cpp:442).
// Features: after compositing, each warp walks its 32 pixels; the owning lane's
// (source, weight) slots are broadcast with __shfl_sync and all 32 lanes read the
// selected surfel's feature row (coalesced 128 B per load) and accumulate 32
// channels each, then write the pixel's HWC channel run in one coalesced store.
// Full blending with features keeps per-pixel (source, weight) lists in a global
// scratch (L2-resident; written and re-read by the same CTA).
#include <cstdint>

#include "psm_device.cuh"
#include "psm_exp.h"
#include "psm_kernels.h"

namespace psm {
namespace {

constexpr int kTile = 16;
constexpr int kThreads = kTile * kTile;
constexpr int kMaxNch = 16;  // feature dims per launch: 32 * 16 = 512

// before(a, b) of topk_select (raster.cpp:232-235), proj order == source order
__device__ __forceinline__ bool before(double wa, int sa, double wb, int sb) {
  return wa > wb || (wa == wb && sa < sb);
}

template <int KMAX, bool FULL_LIST, int NCH>
__global__ void __launch_bounds__(kThreads, 2) blend_kernel(BlendParams p) {
  __shared__ SurfRec srec[kThreads];
  __shared__ int32_t ssrc[kThreads];

  const int tile = blockIdx.x;
  const int tx = tile % p.tiles_x, ty = tile / p.tiles_x;
  const int tid = threadIdx.x;
  const int x = tx * kTile + (tid & (kTile - 1));
  const int y = ty * kTile + (tid >> 4);
  const bool inside = x < p.width && y < p.height;
  const int64_t pix = static_cast<int64_t>(y) * p.width + x;

  const double px = x + 0.5, py = y + 0.5;
  const double rx = (px - p.cam_cx) / p.cam_fx;  // division as in raster.cpp:370-371
  const double ry = (py - p.cam_cy) / p.cam_fy;

  double T = 1.0;
  int m = 0;
  bool done = !inside;
  double acc_r = 0, acc_g = 0, acc_b = 0, exp_depth = 0, dom_depth = 0, dom_w = 0, nx = 0, ny = 0, nz = 0;
  double sw[KMAX > 0 ? KMAX : 1];
  int ss[KMAX > 0 ? KMAX : 1];
#pragma unroll
  for (int i = 0; i < (KMAX > 0 ? KMAX : 1); ++i) {
    sw[i] = -1.0;
    ss[i] = 0x7fffffff;
  }

  const int start = p.ranges[2 * tile], end = p.ranges[2 * tile + 1];
  for (int base = start; base < end; base += kThreads) {
    const int cnt = min(kThreads, end - base);
    if (tid < cnt) {
      const int s = static_cast<int>(p.vals[base + tid]);
      ssrc[tid] = s;
      const float4* src4 = reinterpret_cast<const float4*>(p.recs + s);
      float4* dst4 = reinterpret_cast<float4*>(srec + tid);
#pragma unroll
      for (int k = 0; k < 9; ++k) dst4[k] = __ldg(src4 + k);
    }
    __syncthreads();
    if (!done) {
      for (int j = 0; j < cnt; ++j) {
        const SurfRec& r = srec[j];
        if (p.support_cutoff) {
          const double dx = px - r.cx;
          const double dy = py - r.cy;
          if (r.f00 * dx * dx + r.f01x2 * dx * dy + r.f11 * dy * dy > p.chi2) continue;  // raster.cpp:379
        }
        const double w0 = r.h[0] * rx + r.h[1] * ry + r.h[2];
        const double w1 = r.h[3] * rx + r.h[4] * ry + r.h[5];
        const double w2 = r.h[6] * rx + r.h[7] * ry + r.h[8];
        if (!(w2 > 1e-14)) continue;
        const double rcp = 1.0 / w2;
        const double u = w0 * rcp, v = w1 * rcp;
        const double alpha = r.opacity * psm_exp(-0.5 * (u * u + v * v));
        if (alpha < p.alpha_min || alpha <= 0.0) continue;
        const double wt = alpha * T;
        // colour / depth / normal always over the full list (raster.cpp:405-436)
        acc_r += wt * static_cast<double>(r.color[0]);
        acc_g += wt * static_cast<double>(r.color[1]);
        acc_b += wt * static_cast<double>(r.color[2]);
        exp_depth += wt * rcp;
        if (wt > dom_w) {
          dom_w = wt;
          dom_depth = rcp;
        }
        nx += wt * static_cast<double>(r.normal[0]);
        ny += wt * static_cast<double>(r.normal[1]);
        nz += wt * static_cast<double>(r.normal[2]);
        const int src = ssrc[j];
        if constexpr (KMAX > 0) {
          if (before(wt, src, sw[KMAX - 1], ss[KMAX - 1])) {
#pragma unroll
            for (int i = KMAX - 1; i > 0; --i) {
              if (before(wt, src, sw[i], ss[i])) {
                const bool above_prev = before(wt, src, sw[i - 1], ss[i - 1]);
                sw[i] = above_prev ? sw[i - 1] : wt;
                ss[i] = above_prev ? ss[i - 1] : src;
              }
            }
            if (before(wt, src, sw[0], ss[0])) {
              sw[0] = wt;
              ss[0] = src;
            }
          }
        }
        if constexpr (FULL_LIST) {
          if (m < p.list_cap)
            p.lists[pix * p.list_cap + m] = make_uint2(static_cast<uint32_t>(src), __float_as_uint(static_cast<float>(wt)));
        }
        T *= 1.0 - alpha;
        ++m;
        if (T < p.t_min) {
          done = true;
          break;
        }
      }
    }
    if (__syncthreads_count(done) == kThreads) break;  // also fences srec reuse
  }

  const int k_sel = p.k_sel;
  int blend_n = m;
  if constexpr (KMAX > 0) blend_n = m < k_sel ? m : k_sel;
  if (inside) {
    p.color[pix * 3 + 0] = static_cast<float>(acc_r + T * p.bg0);
    p.color[pix * 3 + 1] = static_cast<float>(acc_g + T * p.bg1);
    p.color[pix * 3 + 2] = static_cast<float>(acc_b + T * p.bg2);
    const bool rdn = p.render_depth_normal != 0;
    p.depth[pix * 2 + 0] = rdn ? static_cast<float>(exp_depth) : 0.f;
    p.depth[pix * 2 + 1] = rdn ? static_cast<float>(dom_depth) : 0.f;
    p.normal[pix * 3 + 0] = rdn ? static_cast<float>(nx) : 0.f;
    p.normal[pix * 3 + 1] = rdn ? static_cast<float>(ny) : 0.f;
    p.normal[pix * 3 + 2] = rdn ? static_cast<float>(nz) : 0.f;
    p.alpha_acc[pix] = static_cast<float>(1.0 - T);
    p.blend_count[pix] = m;
    if constexpr (KMAX > 0) {
      if (p.topk_dbg) {
#pragma unroll
        for (int i = 0; i < KMAX; ++i)
          if (i < k_sel) p.topk_dbg[pix * k_sel + i] = i < blend_n ? ss[i] : -1;
      }
    }
    if constexpr (FULL_LIST) {
      if (m > p.list_cap) atomicMax(p.list_overflow, m);
    }
    // ins_argmax stays -1 unless labels were accumulated (raster.cpp:292,497)
    if (p.n_q == 0 || blend_n == 0 || NCH == 0) p.ins_argmax[pix] = -1;
  }

  // blended_total (raster.cpp:459,502,506): one atomic per warp
  {
    unsigned long long bl = inside ? static_cast<unsigned long long>(blend_n) : 0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) bl += __shfl_xor_sync(0xffffffffu, bl, o);
    if ((tid & 31) == 0 && bl) atomicAdd(p.blended_total, bl);
  }

  // ---- feature / label planes (raster.cpp:456-499), warp-cooperative
  if constexpr (NCH > 0) {
    const int D = p.feat_dims;
    const int lane = tid & 31;
    const int warp_base = tid & ~31;
    for (int q = 0; q < 32; ++q) {
      const int qtid = warp_base + q;
      const int qx = tx * kTile + (qtid & (kTile - 1));
      const int qy = ty * kTile + (qtid >> 4);
      if (qx >= p.width || qy >= p.height) continue;  // warp-uniform
      const int64_t qpix = static_cast<int64_t>(qy) * p.width + qx;
      int nq = __shfl_sync(0xffffffffu, blend_n, q);
      if constexpr (FULL_LIST) nq = nq < p.list_cap ? nq : p.list_cap;
      float acc[NCH];
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch) acc[ch] = 0.f;
      if constexpr (KMAX > 0) {
#pragma unroll
        for (int i = 0; i < KMAX; ++i) {
          const int s = __shfl_sync(0xffffffffu, ss[i], q);
          const float w = __shfl_sync(0xffffffffu, static_cast<float>(sw[i]), q);
          if (i < nq) {
            const float* f = p.feat + static_cast<int64_t>(s) * D + lane;
#pragma unroll
            for (int ch = 0; ch < NCH; ++ch)
              if (lane + 32 * ch < D) acc[ch] += w * __ldg(f + 32 * ch);
          }
        }
      } else {
        const uint2* lst = p.lists + qpix * p.list_cap;
        for (int i = 0; i < nq; ++i) {
          const uint2 e = lst[i];
          const float w = __uint_as_float(e.y);
          const float* f = p.feat + static_cast<int64_t>(e.x) * D + lane;
#pragma unroll
          for (int ch = 0; ch < NCH; ++ch)
            if (lane + 32 * ch < D) acc[ch] += w * __ldg(f + 32 * ch);
        }
      }
      // lanes own channels lane + 32*ch of the pixel's HWC run: coalesced stores
      float best = 0.f;
      int best_i = 0x7fffffff;
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch) {
        const int c = lane + 32 * ch;
        if (c < D) {
          const float v = nq > 0 ? acc[ch] : 0.f;
          if (c < p.c_sem) {
            if (p.sem_feat) p.sem_feat[qpix * p.c_sem + c] = v;
          } else {
            const int qi = c - p.c_sem;
            if (p.ins_dist) p.ins_dist[qpix * p.n_q + qi] = v;
            if (best_i == 0x7fffffff || v > best) {  // first max within the lane (ascending index)
              best = v;
              best_i = qi;
            }
          }
        }
      }
      if (p.n_q > 0 && nq > 0) {
        // first-max argmax across lanes (raster.cpp:492-497): ties go to the lower index
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const float ob = __shfl_xor_sync(0xffffffffu, best, o);
          const int oi = __shfl_xor_sync(0xffffffffu, best_i, o);
          if (oi != 0x7fffffff && (best_i == 0x7fffffff || ob > best || (ob == best && oi < best_i))) {
            best = ob;
            best_i = oi;
          }
        }
        if (lane == 0) p.ins_argmax[qpix] = best_i;
      }
    }
  }
}

template <int KMAX, bool FULL, int NCH>
void launch_t(const BlendParams& p, int tiles, cudaStream_t st) {
  blend_kernel<KMAX, FULL, NCH><<<tiles, kThreads, 0, st>>>(p);
}

template <int KMAX, bool FULL>
void launch_nch(const BlendParams& p, int nch, int tiles, cudaStream_t st) {
  switch (nch) {
    case 0: launch_t<KMAX, FULL, 0>(p, tiles, st); break;
    case 1: launch_t<KMAX, FULL, 1>(p, tiles, st); break;
    case 2: launch_t<KMAX, FULL, 2>(p, tiles, st); break;
    case 3: launch_t<KMAX, FULL, 3>(p, tiles, st); break;
    case 4: launch_t<KMAX, FULL, 4>(p, tiles, st); break;
    case 8: launch_t<KMAX, FULL, 8>(p, tiles, st); break;
    default: launch_t<KMAX, FULL, 16>(p, tiles, st); break;
  }
}

}  // namespace

int blend_kmax_for(int k_sel) {
  if (k_sel <= 8) return 8;
  if (k_sel <= 16) return 16;
  if (k_sel <= 32) return 32;
  return -1;
}

int blend_nch_for(int feat_dims) {
  const int c = (feat_dims + 31) / 32;
  if (c <= 4) return c;
  if (c <= 8) return 8;
  if (c <= kMaxNch) return 16;
  return -1;
}

void launch_blend(const BlendParams& p, int tiles, bool topk, cudaStream_t st) {
  if (tiles <= 0) return;
  const int nch = blend_nch_for(p.feat_dims);
  if (!topk) {
    if (nch == 0) launch_t<0, false, 0>(p, tiles, st);
    else launch_nch<0, true>(p, nch, tiles, st);
    return;
  }
  switch (blend_kmax_for(p.k_sel)) {
    case 8: launch_nch<8, false>(p, nch, tiles, st); break;
    case 16: launch_nch<16, false>(p, nch, tiles, st); break;
    default: launch_nch<32, false>(p, nch, tiles, st); break;
  }
}

}  // namespace psm
