// psm_backward.h — project_surfel_backward (proj/src/raster.cpp:179-203) with the
// quaternion Jacobian (rotation_from_quat_jacobian, math_util.cpp:54-71), shared by the
// CUDA backward (backward.cu) and the CPU oracle. The blending backward's per-surfel
// dL/dH^-1 (pipeline.cpp:447-449) is chained through H = [r_cw s1 R e1, r_cw s2 R e2, p_cam]
// to the centre, quaternion and scales.
//
// Layout: s13 = [centre 3, quaternion w,x,y,z 4, scales 2, opacity, colour 3];
// r_cw column-major (Eigen Matrix3d); h_inv and g_hinv row-major (r * 3 + c).
// Sums are left to right ((a + b) + c), as the restated Eigen products elsewhere.
#ifndef PSM_BACKWARD_H
#define PSM_BACKWARD_H

#if defined(__CUDACC__)
#define PSM_BHD __host__ __device__ __forceinline__
#else
#define PSM_BHD static inline
#include <math.h>
#endif

// rotation_unit (math_util.cpp:16-23), column-major out
PSM_BHD void psm_rot_unit(double w, double x, double y, double z, double* r) {
  r[0] = 1 - 2 * (y * y + z * z); r[3] = 2 * (x * y - w * z); r[6] = 2 * (x * z + w * y);
  r[1] = 2 * (x * y + w * z); r[4] = 1 - 2 * (x * x + z * z); r[7] = 2 * (y * z - w * x);
  r[2] = 2 * (x * z - w * y); r[5] = 2 * (y * z + w * x); r[8] = 1 - 2 * (x * x + y * y);
}

// rotation_unit_grads (math_util.cpp:26-42): d R / d n_j, column-major, j = w, x, y, z
PSM_BHD void psm_rot_unit_grads(double w, double x, double y, double z, double g[4][9]) {
  // g[0]: [0, -2z, 2y; 2z, 0, -2x; -2y, 2x, 0] (rows), stored column-major
  g[0][0] = 0;      g[0][3] = -2 * z; g[0][6] = 2 * y;
  g[0][1] = 2 * z;  g[0][4] = 0;      g[0][7] = -2 * x;
  g[0][2] = -2 * y; g[0][5] = 2 * x;  g[0][8] = 0;
  g[1][0] = 0;      g[1][3] = 2 * y;  g[1][6] = 2 * z;
  g[1][1] = 2 * y;  g[1][4] = -4 * x; g[1][7] = -2 * w;
  g[1][2] = 2 * z;  g[1][5] = 2 * w;  g[1][8] = -4 * x;
  g[2][0] = -4 * y; g[2][3] = 2 * x;  g[2][6] = 2 * w;
  g[2][1] = 2 * x;  g[2][4] = 0;      g[2][7] = 2 * z;
  g[2][2] = -2 * w; g[2][5] = 2 * z;  g[2][8] = -4 * y;
  g[3][0] = -4 * z; g[3][3] = -2 * w; g[3][6] = 2 * x;
  g[3][1] = 2 * w;  g[3][4] = -4 * z; g[3][7] = 2 * y;
  g[3][2] = 2 * x;  g[3][5] = 2 * y;  g[3][8] = 0;
}

// d L / d (centre, quaternion, scales) of one projected surfel from d L / d H^-1.
PSM_BHD void psm_geom_backward(const double* s13, const double* r_cw, const double* h_inv, const double* g_hinv,
                               double* d_center, double* d_rot, double* d_scales) {
  // g_h = -H^-T g H^-T  (A = H^-T, A(r, c) = h_inv[c * 3 + r])
  double t1[9], gh[9];  // row-major
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c)
      t1[r * 3 + c] = ((-h_inv[0 * 3 + r]) * g_hinv[0 * 3 + c] + (-h_inv[1 * 3 + r]) * g_hinv[1 * 3 + c]) +
                      (-h_inv[2 * 3 + r]) * g_hinv[2 * 3 + c];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c)
      gh[r * 3 + c] = (t1[r * 3 + 0] * h_inv[c * 3 + 0] + t1[r * 3 + 1] * h_inv[c * 3 + 1]) + t1[r * 3 + 2] * h_inv[c * 3 + 2];
  // rotation_from_quat_jacobian (the reference throws on a degenerate quaternion; the
  // surfel projected, so the forward already validated it)
  const double* q = s13 + 3;
  const double norm = sqrt((q[0] * q[0] + q[2] * q[2]) + (q[1] * q[1] + q[3] * q[3]));
  const double n[4] = {q[0] / norm, q[1] / norm, q[2] / norm, q[3] / norm};
  double rs[9], gn[4][9], dr[4][9];
  psm_rot_unit(n[0], n[1], n[2], n[3], rs);
  psm_rot_unit_grads(n[0], n[1], n[2], n[3], gn);
  for (int i = 0; i < 4; ++i)
    for (int e = 0; e < 9; ++e) {
      double acc = 0.0;
      for (int j = 0; j < 4; ++j) {
        const double dn = ((i == j ? 1.0 : 0.0) - n[i] * n[j]) / norm;
        acc = acc + gn[j][e] * dn;
      }
      dr[i][e] = acc;
    }
  const double ga[3] = {gh[0], gh[3], gh[6]}, gb[3] = {gh[1], gh[4], gh[7]}, gc[3] = {gh[2], gh[5], gh[8]};
  // d_center = r_cw^T g_c
  for (int i = 0; i < 3; ++i)
    d_center[i] = (r_cw[i * 3 + 0] * gc[0] + r_cw[i * 3 + 1] * gc[1]) + r_cw[i * 3 + 2] * gc[2];
  // d_scales: g_a . (r_cw R e0), g_b . (r_cw R e1)
  double a0[3], a1[3];
  for (int i = 0; i < 3; ++i) {
    a0[i] = (r_cw[0 * 3 + i] * rs[0] + r_cw[1 * 3 + i] * rs[1]) + r_cw[2 * 3 + i] * rs[2];
    a1[i] = (r_cw[0 * 3 + i] * rs[3] + r_cw[1 * 3 + i] * rs[4]) + r_cw[2 * 3 + i] * rs[5];
  }
  d_scales[0] = (ga[0] * a0[0] + ga[1] * a0[1]) + ga[2] * a0[2];
  d_scales[1] = (gb[0] * a1[0] + gb[1] * a1[1]) + gb[2] * a1[2];
  // g_tu = s1 r_cw^T g_a, g_tv = s2 r_cw^T g_b; d_rot[i] = g_tu . dR_i e0 + g_tv . dR_i e1
  double tu[3], tv[3];
  for (int i = 0; i < 3; ++i) {
    tu[i] = s13[7] * ((r_cw[i * 3 + 0] * ga[0] + r_cw[i * 3 + 1] * ga[1]) + r_cw[i * 3 + 2] * ga[2]);
    tv[i] = s13[8] * ((r_cw[i * 3 + 0] * gb[0] + r_cw[i * 3 + 1] * gb[1]) + r_cw[i * 3 + 2] * gb[2]);
  }
  for (int i = 0; i < 4; ++i)
    d_rot[i] = ((tu[0] * dr[i][0] + tu[1] * dr[i][1]) + tu[2] * dr[i][2]) +
               ((tv[0] * dr[i][3] + tv[1] * dr[i][4]) + tv[2] * dr[i][5]);
}

#endif  // PSM_BACKWARD_H
