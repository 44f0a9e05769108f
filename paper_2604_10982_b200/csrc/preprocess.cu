// preprocess.cu — K1: per-surfel 2DGS ray-splat transform, culls, screen box
// and tile count (reference: project_surfel, proj/src/raster.cpp:94-142, plus
// the hot-record build raster.cpp:321-353 and the box of bin_boxes 51-68).
//
// One thread per surfel, source order. All decision arithmetic is fp64 with
// the reference's (Eigen's) operation order and no FMA contraction (this file
// is compiled with --fmad=false), so culls, boxes and the records the blend
// kernel decides on are bit-identical to the CPU oracle.
#include "psm_device.cuh"
#include "psm_ellipse.h"
#include "psm_kernels.h"

namespace psm {
namespace {

__device__ __forceinline__ double sum3(double a, double b, double c) { return (a + b) + c; }

// Adds one to the counter of every tile the surfel is binned to (bin_boxes,
// raster.cpp:59-74; Ellipse extension in psm_ellipse.h): the per-tile bucket sizes
// of the counting sort that replaces the reference's per-tile push_back. Each tile
// has kSplit sub-counters (sub-bucket = lane), laid out split-major, so the atomics
// of a hot tile (10k entries near the camera) spread over kSplit addresses.
__device__ __forceinline__ void count_tiles(const BinRec& b, double cx, double cy, const DevRaster& rs, int img_h,
                                            uint32_t* __restrict__ tile_counts) {
  if (b.tx0 > b.tx1 || b.ty0 > b.ty1) return;
  const bool ellipse = rs.binning == PSM_BIN_ELLIPSE;
  PsmEllipse e;
  if (ellipse) e = psm_ellipse_prep(cx, cy, b.F00, b.F01, b.F11, rs.chi2);
  for (int ty = b.ty0; ty <= b.ty1; ++ty) {
    int lo = b.tx0, hi = b.tx1;
    if (ellipse && !psm_ellipse_row(e, ty, rs.tile_size, img_h, b.tx0, b.tx1, &lo, &hi)) continue;
    uint32_t* row = tile_counts + static_cast<int64_t>(threadIdx.x & (kSplit - 1)) * rs.tiles_x * rs.tiles_y +
                    ty * rs.tiles_x;
    for (int tx = lo; tx <= hi; ++tx) atomicAdd(row + tx, 1u);
  }
}

// One surfel; returns whether it projects (then *db = its depth bit pattern).
__device__ __forceinline__ bool project_one(int64_t i, const double* __restrict__ s,
                                                          DevCamera cam, DevRaster rs, SurfRec* __restrict__ recs,
                                                          BinRec* __restrict__ bins,
                                                          uint64_t* __restrict__ depth_bits,
                                                          uint32_t* __restrict__ tile_counts,
                                                          int32_t* __restrict__ valid, 
                                                          uint64_t* db,
                                                          int32_t* __restrict__ err) {
  valid[i] = 0;

  // p_cam = r_cw * mu + t_cw (Camera::to_camera, core_types.hpp:51)
  const double mu0 = s[0], mu1 = s[1], mu2 = s[2];
  const double pc0 = sum3(cam.r[0] * mu0, cam.r[3] * mu1, cam.r[6] * mu2) + cam.t[0];
  const double pc1 = sum3(cam.r[1] * mu0, cam.r[4] * mu1, cam.r[7] * mu2) + cam.t[1];
  const double pc2 = sum3(cam.r[2] * mu0, cam.r[5] * mu1, cam.r[8] * mu2) + cam.t[2];
  if (!(pc2 > cam.near_clip) || !(pc2 < cam.far_clip)) return false;  // raster.cpp:97

  // rotation_from_quat (math_util.cpp:46-52): norm as Eigen's SSE2 Vector4d reduction
  const double qw = s[3], qx = s[4], qy = s[5], qz = s[6];
  const double qn = sqrt((qw * qw + qy * qy) + (qx * qx + qz * qz));
  if (!(qn > 1e-12) || !isfinite(qw) || !isfinite(qx) || !isfinite(qy) || !isfinite(qz)) {
    atomicOr(err, 1);  // the reference throws std::invalid_argument here
    return false;
  }
  const double w = qw / qn, x = qx / qn, y = qy / qn, z = qz / qn;
  // rotation_unit (math_util.cpp:16-23), R(row, col)
  const double r00 = 1 - 2 * (y * y + z * z), r01 = 2 * (x * y - w * z), r02 = 2 * (x * z + w * y);
  const double r10 = 2 * (x * y + w * z), r11 = 1 - 2 * (x * x + z * z), r12 = 2 * (y * z - w * x);
  const double r20 = 2 * (x * z - w * y), r21 = 2 * (y * z + w * x), r22 = 1 - 2 * (x * x + y * y);

  // a = r_cw (s1 R.col0), b = r_cw (s2 R.col1)  (raster.cpp:100-101)
  const double s1 = s[7], s2 = s[8];
  const double sa0 = s1 * r00, sa1 = s1 * r10, sa2 = s1 * r20;
  const double sb0 = s2 * r01, sb1 = s2 * r11, sb2 = s2 * r21;
  const double a0 = sum3(cam.r[0] * sa0, cam.r[3] * sa1, cam.r[6] * sa2);
  const double a1 = sum3(cam.r[1] * sa0, cam.r[4] * sa1, cam.r[7] * sa2);
  const double a2 = sum3(cam.r[2] * sa0, cam.r[5] * sa1, cam.r[8] * sa2);
  const double b0 = sum3(cam.r[0] * sb0, cam.r[3] * sb1, cam.r[6] * sb2);
  const double b1 = sum3(cam.r[1] * sb0, cam.r[4] * sb1, cam.r[7] * sb2);
  const double b2 = sum3(cam.r[2] * sb0, cam.r[5] * sb1, cam.r[8] * sb2);

  // H = [a b p_cam]; H(row, col): col0 = a, col1 = b, col2 = p
  const double m00 = a0, m10 = a1, m20 = a2;
  const double m01 = b0, m11 = b1, m21 = b2;
  const double m02 = pc0, m12 = pc1, m22 = pc2;
  // Matrix3d::determinant (Eigen bruteforce_det3_helper)
  const double det = m00 * (m11 * m22 - m12 * m21) - m01 * (m10 * m22 - m12 * m20) + m02 * (m10 * m21 - m11 * m20);
  const double na = sqrt(sum3(a0 * a0, a1 * a1, a2 * a2));
  const double nb = sqrt(sum3(b0 * b0, b1 * b1, b2 * b2));
  const double np = sqrt(sum3(pc0 * pc0, pc1 * pc1, pc2 * pc2));
  const double det_scale = na * nb * np;
  if (fabs(det) <= 1e-12 * (det_scale < 1e-30 ? 1e-30 : det_scale)) return false;  // grazing, std::max (raster.cpp:109)

  // Matrix3d::inverse: cofactors (cyclic), det from column 0, times 1/det
  const double c00 = m11 * m22 - m12 * m21;  // cof(0,0)
  const double c10 = m21 * m02 - m22 * m01;  // cof(1,0)
  const double c20 = m01 * m12 - m02 * m11;  // cof(2,0)
  const double idet = 1.0 / sum3(c00 * m00, c10 * m10, c20 * m20);
  const double c01 = m12 * m20 - m10 * m22;  // cof(0,1)
  const double c11 = m22 * m00 - m20 * m02;  // cof(1,1)
  const double c21 = m02 * m10 - m00 * m12;  // cof(2,1)
  const double c02 = m10 * m21 - m11 * m20;  // cof(0,2)
  const double c12 = m20 * m01 - m21 * m00;  // cof(1,2)
  const double c22 = m00 * m11 - m01 * m10;  // cof(2,2)
  SurfRec rec;
  // h_inv(r, c) = cof(c, r) * idet, stored row-major
  rec.h[0] = c00 * idet; rec.h[1] = c10 * idet; rec.h[2] = c20 * idet;
  rec.h[3] = c01 * idet; rec.h[4] = c11 * idet; rec.h[5] = c21 * idet;
  rec.h[6] = c02 * idet; rec.h[7] = c12 * idet; rec.h[8] = c22 * idet;

  const double zz = pc2;
  const double cx = cam.fx * pc0 / zz + cam.cx;
  const double cy = cam.fy * pc1 / zz + cam.cy;
  // Jacobian and Sigma' = B B^T (raster.cpp:119-125); the zero entries of jac drop out exactly
  const double j00 = cam.fx / zz, j02 = -cam.fx * pc0 / (zz * zz);
  const double j11 = cam.fy / zz, j12 = -cam.fy * pc1 / (zz * zz);
  const double bb00 = sum3(j00 * a0, 0.0 * a1, j02 * a2);
  const double bb10 = sum3(0.0 * a0, j11 * a1, j12 * a2);
  const double bb01 = sum3(j00 * b0, 0.0 * b1, j02 * b2);
  const double bb11 = sum3(0.0 * b0, j11 * b1, j12 * b2);
  const double sg00 = bb00 * bb00 + bb01 * bb01;
  const double sg01 = bb00 * bb10 + bb01 * bb11;
  const double sg11 = bb10 * bb10 + bb11 * bb11;

  // footprint_cov + circle_box off-screen cull (raster.cpp:127-130)
  const double F00 = sg00 + 0.3, F01 = sg01, F11 = sg11 + 0.3;
  const double half_tr = 0.5 * (F00 + F11);
  const double fdet = F00 * F11 - F01 * F01;
  const double dd = half_tr * half_tr - fdet;
  const double disc = sqrt(dd < 0.0 ? 0.0 : dd);  // std::max(., 0.0) keeps NaN
  const double rad = sqrt(rs.chi2 * (half_tr + disc));
  const double bx0 = cx - rad, bx1 = cx + rad, by0 = cy - rad, by1 = cy + rad;
  if (bx1 < 0 || bx0 > cam.w || by1 < 0 || by0 > cam.h) return false;

  // footprint_inv = adj(F) / det F (raster.cpp:132-136)
  rec.cx = cx;
  rec.cy = cy;
  rec.f00 = F11 / fdet;
  rec.f01x2 = 2.0 * (-F01 / fdet);
  rec.f11 = F00 / fdet;
  rec.opacity = s[9];
  rec.color[0] = static_cast<float>(s[10]);
  rec.color[1] = static_cast<float>(s[11]);
  rec.color[2] = static_cast<float>(s[12]);
  // normal_vis (raster.cpp:138-139): (center_world - mu) . n >= 0 ? n : -n
  const double cw0 = -sum3(cam.r[0] * cam.t[0], cam.r[1] * cam.t[1], cam.r[2] * cam.t[2]);
  const double cw1 = -sum3(cam.r[3] * cam.t[0], cam.r[4] * cam.t[1], cam.r[5] * cam.t[2]);
  const double cw2 = -sum3(cam.r[6] * cam.t[0], cam.r[7] * cam.t[1], cam.r[8] * cam.t[2]);
  const double side = sum3((cw0 - mu0) * r02, (cw1 - mu1) * r12, (cw2 - mu2) * r22);
  const double sgn = side >= 0 ? 1.0 : -1.0;
  rec.normal[0] = static_cast<float>(sgn * r02);
  rec.normal[1] = static_cast<float>(sgn * r12);
  rec.normal[2] = static_cast<float>(sgn * r22);
  recs[i] = rec;

  // binning box (circle_box or aabb_box), tile rectangle (raster.cpp:60-68)
  BinRec b;
  b.F00 = F00; b.F01 = F01; b.F11 = F11;
  double x0 = bx0, x1 = bx1, y0 = by0, y1 = by1;
  if (rs.binning != PSM_BIN_CIRCLE) {
    const double dx = sqrt(rs.chi2 * F00), dy = sqrt(rs.chi2 * F11);
    x0 = cx - dx; x1 = cx + dx; y0 = cy - dy; y1 = cy + dy;
  }
  const int ts = rs.tile_size;  // floor(x / ts) as raster.cpp:62-65 (exact reciprocal for 16)
  b.tx0 = max(x86_cvt(floor(psm_div_tile(x0, ts))), 0);
  b.tx1 = min(x86_cvt(floor(psm_div_tile(x1, ts))), rs.tiles_x - 1);
  b.ty0 = max(x86_cvt(floor(psm_div_tile(y0, ts))), 0);
  b.ty1 = min(x86_cvt(floor(psm_div_tile(y1, ts))), rs.tiles_y - 1);
  b.pad0 = b.pad1 = 0;
  bins[i] = b;
  depth_bits[i] = static_cast<uint64_t>(__double_as_longlong(zz));
  count_tiles(b, cx, cy, rs, cam.h, tile_counts);
  valid[i] = 1;
  *db = static_cast<uint64_t>(__double_as_longlong(zz));
  return true;
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }
constexpr int kPreSmem = 2 * 8 * 32 * 13 * static_cast<int>(sizeof(double));  // 53,248 B

// 2 CTAs per SM (126 registers, no spills) with the batch prefetch: C3 preprocess 0.130 ->
// 0.120 ms, C4 0.552 -> 0.505 ms; at 3 CTAs the persistent loop spills (0.150 ms)
#ifndef PSM_PRE_MINB
#define PSM_PRE_MINB 2
#endif
__global__ void __launch_bounds__(256, PSM_PRE_MINB) preprocess_kernel(const double* __restrict__ surfels13, int64_t n,
                                                          DevCamera cam, DevRaster rs, SurfRec* __restrict__ recs,
                                                          BinRec* __restrict__ bins,
                                                          uint64_t* __restrict__ depth_bits,
                                                          uint32_t* __restrict__ tile_counts,
                                                          int32_t* __restrict__ valid, uint32_t* __restrict__ n_proj,
                                                          unsigned long long* __restrict__ depth_minmax,
                                                          int32_t* __restrict__ err) {
  // Persistent: each warp walks 32-surfel batches (grid stride); a batch's 32 x 104 B
  // (contiguous) are staged through shared memory with coalesced 16-byte cp.async, the
  // next batch's copies in flight while this one is projected.
  extern __shared__ __align__(16) double stage[];  // [2][8 warps][32 * 13]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t n_batches = (n + 31) / 32, stride = static_cast<int64_t>(gridDim.x) * 8;
  auto issue = [&](int64_t bt, int buf) {
    if (bt < n_batches) {
      const int64_t w0 = bt * 32;
      const int nw = static_cast<int>(n - w0 < 32 ? n - w0 : 32);
      const double* src = surfels13 + 13 * w0;
      double* dst = stage + (buf * 8 + w) * (32 * 13);
      const int nv = (13 * nw) / 2;  // whole 16-byte pairs (13 * 32 is even)
#pragma unroll
      for (int k = 0; k < 7; ++k) {
        const int v = lane + 32 * k;
        if (v < nv) cp_async16(dst + 2 * v, src + 2 * v);
      }
      if ((13 * nw) % 2 && lane == 0) cp_async8(dst + 13 * nw - 1, src + 13 * nw - 1);
    }
    cp_async_commit();
  };
  unsigned long long lo = ~0ull, hi = 0ull;
  uint32_t n_ok = 0;
  int buf = 0;
  int64_t bt = static_cast<int64_t>(blockIdx.x) * 8 + w;
  issue(bt, 0);
  for (; bt < n_batches; bt += stride, buf ^= 1) {
    issue(bt + stride, buf ^ 1);
    cp_async_wait<1>();
    __syncwarp();
    const int64_t i = bt * 32 + lane;
    uint64_t db = 0;
    const bool ok = i < n && project_one(i, stage + (buf * 8 + w) * (32 * 13) + 13 * lane, cam, rs, recs, bins, depth_bits,
                                         tile_counts, valid, &db, err);
    if (ok) {
      lo = db < lo ? db : lo;
      hi = db > hi ? db : hi;
      ++n_ok;
    }
    __syncwarp();  // the buffer is refilled two batches later
  }
  cp_async_wait<0>();
  // n_proj and the frame's depth bit range (sort keys, binning.cu): a full-warp reduction
  // with identities for culled lanes, one atomic each per warp
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long l2 = __shfl_xor_sync(0xffffffffu, lo, o), h2 = __shfl_xor_sync(0xffffffffu, hi, o);
    lo = l2 < lo ? l2 : lo;
    hi = h2 > hi ? h2 : hi;
    n_ok += __shfl_xor_sync(0xffffffffu, n_ok, o);
  }
  if (lane == 0 && n_ok) {
    atomicAdd(n_proj, n_ok);
    atomicMin(depth_minmax, lo);
    atomicMax(depth_minmax + 1, hi);
  }
}

// Per-frame reset in one launch (instead of three memsets and a host-to-device copy):
// the 16 frame counters, the per-tile ranges, the split tile counters, and the depth
// range's (min, max) identities.
__global__ void frame_init_kernel(unsigned long long* __restrict__ small, int32_t* __restrict__ ranges, int n_ranges,
                                  uint32_t* __restrict__ tcounts, int n_counts,
                                  unsigned long long* __restrict__ dminmax) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x, stride = gridDim.x * blockDim.x;
  if (t < 16) small[t] = 0ull;
  if (dminmax && t < 2) dminmax[t] = t == 0 ? ~0ull : 0ull;
  for (int i = t; i < n_ranges; i += stride) ranges[i] = 0;
  for (int i = t; i < n_counts; i += stride) tcounts[i] = 0u;
}

}  // namespace

void launch_frame_init(unsigned long long* small, int32_t* ranges, int n_ranges, uint32_t* tcounts, int n_counts,
                       unsigned long long* dminmax, cudaStream_t stream) {
  const int work = n_ranges > n_counts ? n_ranges : n_counts;
  int blocks = (work + 255) / 256;
  blocks = blocks < 1 ? 1 : (blocks > 1184 ? 1184 : blocks);
  frame_init_kernel<<<blocks, 256, 0, stream>>>(small, ranges, n_ranges, tcounts, n_counts, dminmax);
}

void launch_preprocess(const double* surfels13, int64_t n, const DevCamera& cam, const DevRaster& rs, SurfRec* recs,
                       BinRec* bins, uint64_t* depth_bits, uint32_t* tile_counts, int32_t* valid,
                       uint32_t* n_proj, unsigned long long* depth_minmax, int32_t* err, cudaStream_t stream) {
  if (n <= 0) return;
  // persistent: every resident CTA, or fewer when the scene is smaller
  static int per_sm[64] = {}, sms[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!per_sm[dev]) {
    cudaDeviceGetAttribute(&sms[dev], cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(preprocess_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kPreSmem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[dev], preprocess_kernel, 256, kPreSmem);
    if (per_sm[dev] < 1) per_sm[dev] = 1;
  }
  const int64_t need = (n + 255) / 256;
  const int64_t resident = static_cast<int64_t>(per_sm[dev]) * sms[dev];
  const int64_t blocks = need < resident ? need : resident;
  preprocess_kernel<<<static_cast<unsigned>(blocks), 256, kPreSmem, stream>>>(surfels13, n, cam, rs, recs, bins, depth_bits,
                                                                       tile_counts, valid, n_proj, depth_minmax, err);
}

}  // namespace psm
