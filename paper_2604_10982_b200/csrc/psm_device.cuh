// psm_device.cuh — device-side records and launch helpers shared by the kernels.
//
// HBM layout (per frame, all fp64 geometry kept exact for decisions):
//   SurfRec  [N]  144 B, source-indexed: the reference's HotReject + HotGeom +
//                 colour + normal_vis (raster.cpp:324-353), packed so one record
//                 is nine 16-byte loads and the 5 support-test scalars share the
//                 first 48 bytes.
//   BinRec   [N]  64 B: the dilated covariance F (raster.cpp:19-24), the screen
//                 centre, the depth bits and the clamped tile rectangle of the
//                 active box (raster.cpp:59-68): everything K4 reads per surfel.
//   depth    [N]  uint64 bit pattern of sort_depth (positive doubles order as
//                 unsigned integers, so a radix sort reproduces (depth, source)).
#ifndef PSM_DEVICE_CUH
#define PSM_DEVICE_CUH

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/psm.h"

namespace psm {

struct __align__(16) SurfRec {
  double cx, cy;      // screen centre (raster.hpp:23)
  double f00, f01x2;  // footprint_inv(0,0), 2 * footprint_inv(0,1) (2x is exact)
  double f11, opacity;
  double h[9];        // h_inv row-major (raster.cpp:343)
  float color[3];     // Surfel::color (fp32: only blended, never decided on)
  float normal[3];    // normal_vis
};
static_assert(sizeof(SurfRec) == 144, "SurfRec must be 144 bytes");

struct __align__(16) BinRec {
  double F00, F01, F11;  // footprint_cov(sigma)
  double cx, cy;         // screen centre (the emit's ellipse rows and warp-block masks)
  uint64_t depth_bits;   // sort_depth's bit pattern (the emit's sort key)
  int32_t tx0, tx1, ty0, ty1;  // clamped tile rectangle of the binning box (empty if tx0 > tx1)
};
static_assert(sizeof(BinRec) == 64, "BinRec must be 64 bytes (one record per emit read)");

// Sub-buckets per tile for the counting sort's atomics (binning.cu).
constexpr int kSplit = 32;
// Bits below the source id in a tile sort key: the 8-bit warp-block live mask of the
// (surfel, tile) entry (psm_block_mask), carried through the sort beside the source.
constexpr int kFieldExtra = 8;
// K5 per-tile sort size classes (binning.cu); K3b writes their tile lists and the
// blend's tile order into one buffer of (kSortClasses + 2) x tiles ints.
constexpr int kSortClasses = 5;

// Camera by value in kernel parameters.
struct DevCamera {
  double r[9];  // column-major r_cw
  double t[3];
  double fx, fy, cx, cy;
  int32_t w, h;
  double near_clip, far_clip;
};

struct DevRaster {
  double chi2, alpha_min, t_min;
  double bg[3];
  int32_t support_cutoff, binning, render_depth_normal, tile_size;
  int32_t tiles_x, tiles_y;
};

// x86-64 cvttsd2si semantics for the reference's static_cast<int>(std::floor(...))
// (raster.cpp:61-64): out-of-range and NaN give INT_MIN.
__device__ __forceinline__ int x86_cvt(double v) {
  if (!(v > -2147483649.0 && v < 2147483648.0)) return INT32_MIN;
  return static_cast<int>(v);
}

#define PSM_CUDA_TRY(expr)                                                          \
  do {                                                                              \
    cudaError_t _e = (expr);                                                        \
    if (_e != cudaSuccess) return ::psm::fail_cuda(ctx, _e, #expr, __FILE__, __LINE__); \
  } while (0)

}  // namespace psm

#endif  // PSM_DEVICE_CUH
