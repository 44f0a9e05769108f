// psm_project.cuh — project_surfel (proj/src/raster.cpp:94-142) as one device function,
// shared by K1 (preprocess.cu, which packs its result into the blend's SurfRec and the
// binning's BinRec) and the stage entry point psm_project_surfels (stages.cu, which returns
// the whole ProjectedSurfel). All decision arithmetic is fp64 in the reference's (Eigen's)
// operation order; the files that include it compile with --fmad=false, so the results
// are bit-identical to the reference's x86-64 SSE2 build (tests/test_ref_pin.py pins the
// oracle to it; the GPU parity suite pins this code to the oracle).
#ifndef PSM_PROJECT_CUH
#define PSM_PROJECT_CUH

#include "psm_device.cuh"

namespace psm {

__device__ __forceinline__ double psm_sum3(double a, double b, double c) { return (a + b) + c; }

// Everything project_surfel computes for one surfel.
struct ProjFull {
  double pc0, pc1, pc2;          // p_cam (= H column 2); sort_depth = pc2
  double a0, a1, a2, b0, b1, b2; // H columns 0, 1
  double h[9];                   // h_inv, row-major
  double cx, cy;                 // screen_center
  double sg00, sg01, sg11;       // sigma (symmetric bit for bit: the products commute)
  double F00, F01, F11, fdet;    // footprint_cov(sigma) and its determinant
  double rad;                    // circle_box half-width sqrt(chi2 lambda_max(F))
  double r02, r12, r22, sgn;     // world normal (R column 2) and the normal_vis sign
};

// Returns 1 projected, 0 culled, -1 degenerate quaternion on a surfel that passed the
// depth cull (the reference throws std::invalid_argument there, math_util.cpp:48-50).
__device__ __forceinline__ int psm_project(const double* __restrict__ s, const DevCamera& cam, double chi2,
                                           ProjFull& o) {
  // p_cam = r_cw * mu + t_cw (Camera::to_camera, core_types.hpp:51)
  const double mu0 = s[0], mu1 = s[1], mu2 = s[2];
  o.pc0 = psm_sum3(cam.r[0] * mu0, cam.r[3] * mu1, cam.r[6] * mu2) + cam.t[0];
  o.pc1 = psm_sum3(cam.r[1] * mu0, cam.r[4] * mu1, cam.r[7] * mu2) + cam.t[1];
  o.pc2 = psm_sum3(cam.r[2] * mu0, cam.r[5] * mu1, cam.r[8] * mu2) + cam.t[2];
  const double pc0 = o.pc0, pc1 = o.pc1, pc2 = o.pc2;
  if (!(pc2 > cam.near_clip) || !(pc2 < cam.far_clip)) return 0;  // raster.cpp:97

  // rotation_from_quat (math_util.cpp:46-52): norm as Eigen's SSE2 Vector4d reduction
  const double qw = s[3], qx = s[4], qy = s[5], qz = s[6];
  const double qn = sqrt((qw * qw + qy * qy) + (qx * qx + qz * qz));
  if (!(qn > 1e-12) || !isfinite(qw) || !isfinite(qx) || !isfinite(qy) || !isfinite(qz)) return -1;
  const double w = qw / qn, x = qx / qn, y = qy / qn, z = qz / qn;
  // rotation_unit (math_util.cpp:16-23), R(row, col)
  const double r00 = 1 - 2 * (y * y + z * z), r01 = 2 * (x * y - w * z);
  const double r10 = 2 * (x * y + w * z), r11 = 1 - 2 * (x * x + z * z);
  const double r20 = 2 * (x * z - w * y), r21 = 2 * (y * z + w * x);
  o.r02 = 2 * (x * z + w * y);
  o.r12 = 2 * (y * z - w * x);
  o.r22 = 1 - 2 * (x * x + y * y);

  // a = r_cw (s1 R.col0), b = r_cw (s2 R.col1)  (raster.cpp:100-101)
  const double s1 = s[7], s2 = s[8];
  const double sa0 = s1 * r00, sa1 = s1 * r10, sa2 = s1 * r20;
  const double sb0 = s2 * r01, sb1 = s2 * r11, sb2 = s2 * r21;
  const double a0 = psm_sum3(cam.r[0] * sa0, cam.r[3] * sa1, cam.r[6] * sa2);
  const double a1 = psm_sum3(cam.r[1] * sa0, cam.r[4] * sa1, cam.r[7] * sa2);
  const double a2 = psm_sum3(cam.r[2] * sa0, cam.r[5] * sa1, cam.r[8] * sa2);
  const double b0 = psm_sum3(cam.r[0] * sb0, cam.r[3] * sb1, cam.r[6] * sb2);
  const double b1 = psm_sum3(cam.r[1] * sb0, cam.r[4] * sb1, cam.r[7] * sb2);
  const double b2 = psm_sum3(cam.r[2] * sb0, cam.r[5] * sb1, cam.r[8] * sb2);
  o.a0 = a0; o.a1 = a1; o.a2 = a2;
  o.b0 = b0; o.b1 = b1; o.b2 = b2;

  // H = [a b p_cam]; H(row, col): col0 = a, col1 = b, col2 = p
  const double m00 = a0, m10 = a1, m20 = a2;
  const double m01 = b0, m11 = b1, m21 = b2;
  const double m02 = pc0, m12 = pc1, m22 = pc2;
  // Matrix3d::determinant (Eigen bruteforce_det3_helper)
  const double det = m00 * (m11 * m22 - m12 * m21) - m01 * (m10 * m22 - m12 * m20) + m02 * (m10 * m21 - m11 * m20);
  const double na = sqrt(psm_sum3(a0 * a0, a1 * a1, a2 * a2));
  const double nb = sqrt(psm_sum3(b0 * b0, b1 * b1, b2 * b2));
  const double np = sqrt(psm_sum3(pc0 * pc0, pc1 * pc1, pc2 * pc2));
  const double det_scale = na * nb * np;
  if (fabs(det) <= 1e-12 * (det_scale < 1e-30 ? 1e-30 : det_scale)) return 0;  // grazing, std::max (raster.cpp:109)

  // Matrix3d::inverse: cofactors (cyclic), det from column 0, times 1/det
  const double c00 = m11 * m22 - m12 * m21;  // cof(0,0)
  const double c10 = m21 * m02 - m22 * m01;  // cof(1,0)
  const double c20 = m01 * m12 - m02 * m11;  // cof(2,0)
  const double idet = 1.0 / psm_sum3(c00 * m00, c10 * m10, c20 * m20);
  const double c01 = m12 * m20 - m10 * m22;  // cof(0,1)
  const double c11 = m22 * m00 - m20 * m02;  // cof(1,1)
  const double c21 = m02 * m10 - m00 * m12;  // cof(2,1)
  const double c02 = m10 * m21 - m11 * m20;  // cof(0,2)
  const double c12 = m20 * m01 - m21 * m00;  // cof(1,2)
  const double c22 = m00 * m11 - m01 * m10;  // cof(2,2)
  // h_inv(r, c) = cof(c, r) * idet, stored row-major
  o.h[0] = c00 * idet; o.h[1] = c10 * idet; o.h[2] = c20 * idet;
  o.h[3] = c01 * idet; o.h[4] = c11 * idet; o.h[5] = c21 * idet;
  o.h[6] = c02 * idet; o.h[7] = c12 * idet; o.h[8] = c22 * idet;

  const double zz = pc2;
  o.cx = cam.fx * pc0 / zz + cam.cx;
  o.cy = cam.fy * pc1 / zz + cam.cy;
  // Jacobian and Sigma' = B B^T (raster.cpp:119-125); the zero entries of jac drop out exactly
  const double j00 = cam.fx / zz, j02 = -cam.fx * pc0 / (zz * zz);
  const double j11 = cam.fy / zz, j12 = -cam.fy * pc1 / (zz * zz);
  const double bb00 = psm_sum3(j00 * a0, 0.0 * a1, j02 * a2);
  const double bb10 = psm_sum3(0.0 * a0, j11 * a1, j12 * a2);
  const double bb01 = psm_sum3(j00 * b0, 0.0 * b1, j02 * b2);
  const double bb11 = psm_sum3(0.0 * b0, j11 * b1, j12 * b2);
  o.sg00 = bb00 * bb00 + bb01 * bb01;
  o.sg01 = bb00 * bb10 + bb01 * bb11;
  o.sg11 = bb10 * bb10 + bb11 * bb11;

  // footprint_cov + circle_box off-screen cull (raster.cpp:127-130)
  o.F00 = o.sg00 + 0.3;
  o.F01 = o.sg01;
  o.F11 = o.sg11 + 0.3;
  const double half_tr = 0.5 * (o.F00 + o.F11);
  o.fdet = o.F00 * o.F11 - o.F01 * o.F01;
  const double dd = half_tr * half_tr - o.fdet;
  const double disc = sqrt(dd < 0.0 ? 0.0 : dd);  // std::max(., 0.0) keeps NaN
  o.rad = sqrt(chi2 * (half_tr + disc));
  if (o.cx + o.rad < 0 || o.cx - o.rad > cam.w || o.cy + o.rad < 0 || o.cy - o.rad > cam.h) return 0;

  // normal_vis (raster.cpp:138-139): (center_world - mu) . n >= 0 ? n : -n
  const double cw0 = -psm_sum3(cam.r[0] * cam.t[0], cam.r[1] * cam.t[1], cam.r[2] * cam.t[2]);
  const double cw1 = -psm_sum3(cam.r[3] * cam.t[0], cam.r[4] * cam.t[1], cam.r[5] * cam.t[2]);
  const double cw2 = -psm_sum3(cam.r[6] * cam.t[0], cam.r[7] * cam.t[1], cam.r[8] * cam.t[2]);
  const double side = psm_sum3((cw0 - mu0) * o.r02, (cw1 - mu1) * o.r12, (cw2 - mu2) * o.r22);
  o.sgn = side >= 0 ? 1.0 : -1.0;
  return 1;
}

}  // namespace psm

#endif  // PSM_PROJECT_CUH
