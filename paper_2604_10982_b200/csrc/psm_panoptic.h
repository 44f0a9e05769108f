// psm_panoptic.h — the panoptic label assignment of Ψ-Map, shared verbatim by the
// CUDA kernel (labels.cu) and the CPU oracle so both produce the same bits.
//
// assign_labels (proj/src/panoptic.cpp:36-91): for every surfel s and alive query a
//   A(a, s) = sigmoid(f_q(a) . f_ins(s)) * exp(-1/2 d^T Sigma_a^-1 d),  d = mu_s - mean_a
// (attention_map, panoptic.cpp:32-34), then a softmax over the alive queries,
//   dist(a, s) = exp(A - A_max) / sum_b exp(A_b - A_max),
// and argmax(s) = the first alive query with the largest A (ties to the lower index).
// Dead queries keep dist 0. Sigma_a^-1 comes from an LLT of the symmetrised
// covariance, retried with an eps*I floor when it is not positive definite
// (panoptic.cpp:53-62).
//
// Evaluation order is Eigen 3.4's on x86-64 SSE2 without FMA: the feature dot is a
// dynamic-size vectorised reduction (psm_dot_dyn), the 3x3 products are left-to-right
// sums, the LLT is llt_inplace::unblocked and its solve against the identity goes
// through triangular_solve_matrix (psm_llt3_inverse). tests/test_ref_pin.py checks the
// oracle against the reference's panoptic.cpp / metrics.cpp compiled in oracle/_ref
// (with oracle/eigen_min modelling the same Eigen code paths); the reference's
// test_panoptic.cpp:86-183 cases are ported in tests/test_panoptic_oracle.py. GPU and
// oracle agree bit for bit. exp is psm_exp (glibc-exact); compile without contraction.
#ifndef PSM_PANOPTIC_H
#define PSM_PANOPTIC_H

#include <stdint.h>

#include "psm_exp.h"

#if defined(__CUDACC__)
#define PSM_PHD __host__ __device__ __forceinline__
#else
#define PSM_PHD static inline
#include <math.h>
#endif

// psm_exp_t with its common range unbranched: psm_exp_main always, the full function only
// when the argument is outside it (psm_exp_main_ok); same value as psm_exp_t(x, tab).
PSM_PHD double psm_exp_q(double x, const uint64_t* tab) {
  double y = psm_exp_main(x, tab);
  if (!psm_exp_main_ok(x)) y = psm_exp_t(x, tab);
  return y;
}

// Which exps of assign_labels take psm_exp_q: bit 0 the sigmoid's, bit 1 the softmax's,
// bit 2 the Mahalanobis term's (the others psm_exp_t; the values are identical). C3p
// (32 queries), frames/s with the branch-free sigmoid: none 434, sigmoid 445, sigmoid +
// softmax 442, all three 456.
#ifndef PSM_LABEL_EXPQ
#define PSM_LABEL_EXPQ 7
#endif
PSM_PHD double psm_label_exp(double x, const uint64_t* tab, int which) {
  return (PSM_LABEL_EXPQ >> which & 1) ? psm_exp_q(x, tab) : psm_exp_t(x, tab);
}

// sigmoid (math_util.cpp:122-128): x >= 0: 1 / (1 + exp(-x)), else e / (1 + e) with
// e = exp(x). One exp and one division whatever the sign, so that a warp whose lanes
// disagree on it does not run both branches.
PSM_PHD double psm_sigmoid_t(double x, const uint64_t* tab) {
  const bool pos = x >= 0;
  const double e = psm_label_exp(pos ? -x : x, tab, 0);
  return (pos ? 1.0 : e) / (1.0 + e);
}

// Lower Cholesky of a symmetric 3x3 (column-major a[c*3 + r]); 0 if not positive definite.
PSM_PHD int psm_llt3(const double* a, double* l) {
  for (int i = 0; i < 9; ++i) l[i] = 0.0;
  for (int k = 0; k < 3; ++k) {
    double x = a[k * 3 + k];
    if (k == 1) x -= l[0 * 3 + 1] * l[0 * 3 + 1];
    if (k == 2) x -= l[0 * 3 + 2] * l[0 * 3 + 2] + l[1 * 3 + 2] * l[1 * 3 + 2];
    if (x <= 0.0) return 0;  // llt_inplace::unblocked's test (a NaN pivot passes, as there)
    x = sqrt(x);
    l[k * 3 + k] = x;
    for (int i = k + 1; i < 3; ++i) {
      double v = a[k * 3 + i];
      if (k == 1) v -= l[0 * 3 + i] * l[0 * 3 + 1];
      if (k == 2) v -= l[0 * 3 + i] * l[0 * 3 + 2] + l[1 * 3 + i] * l[1 * 3 + 2];
      l[k * 3 + i] = v / x;
    }
  }
  return 1;
}

// X = (L L^T)^-1 = llt.solve(Identity) in Eigen's order: a 3x3 right-hand side goes
// through triangular_solve_matrix, column by column. Lower solve (L column-major):
// x_i *= 1 / l_ii, then x_r -= x_i l_ri below it. Upper solve (L^T, row-major) from the
// last row up: b = 0 + sum over the solved rows in column order, x_i = (x_i - b) / l_ii
// as a multiply by the reciprocal.
PSM_PHD void psm_llt3_inverse(const double* l, double* inv) {
  for (int c = 0; c < 3; ++c) {
    double x[3] = {c == 0 ? 1.0 : 0.0, c == 1 ? 1.0 : 0.0, c == 2 ? 1.0 : 0.0};
    for (int i = 0; i < 3; ++i) {
      const double a = 1.0 / l[i * 3 + i];
      x[i] = x[i] * a;
      for (int r = i + 1; r < 3; ++r) x[r] = x[r] - x[i] * l[i * 3 + r];
    }
    for (int k = 0; k < 3; ++k) {
      const int i = 2 - k;
      const double a = 1.0 / l[i * 3 + i];
      double b = 0.0;
      for (int t = 0; t < k; ++t) b = b + l[i * 3 + (i + 1 + t)] * x[i + 1 + t];
      x[i] = (x[i] - b) * a;
    }
    inv[c * 3 + 0] = x[0];
    inv[c * 3 + 1] = x[1];
    inv[c * 3 + 2] = x[2];
  }
}

// VectorXd::dot in Eigen's order (redux_impl, LinearVectorizedTraversal, NoUnrolling,
// 2-wide packets, aligned start): the products accumulate in two packet sums over
// 4-element strides, one more packet when two remain, the two lanes are added, then
// the odd tail.
PSM_PHD double psm_dot_dyn(const double* a, const double* b, int n) {
  const int aligned = (n / 2) * 2, aligned2 = (n / 4) * 4;
  if (!aligned) return n > 0 ? a[0] * b[0] : 0.0;
  double p0 = a[0] * b[0], p1 = a[1] * b[1];
  if (aligned > 2) {
    double q0 = a[2] * b[2], q1 = a[3] * b[3];
    for (int i = 4; i < aligned2; i += 4) {
      p0 = p0 + a[i] * b[i];
      p1 = p1 + a[i + 1] * b[i + 1];
      q0 = q0 + a[i + 2] * b[i + 2];
      q1 = q1 + a[i + 3] * b[i + 3];
    }
    p0 = p0 + q0;
    p1 = p1 + q1;
    if (aligned > aligned2) {
      p0 = p0 + a[aligned2] * b[aligned2];
      p1 = p1 + a[aligned2 + 1] * b[aligned2 + 1];
    }
  }
  double res = p0 + p1;
  for (int i = aligned; i < n; ++i) res = res + a[i] * b[i];
  return res;
}

// Sigma^-1 of a query covariance (panoptic.cpp:53-62), column-major in and out.
PSM_PHD void psm_query_inverse(const double* cov, double* inv) {
  double s[9], l[9];
  for (int c = 0; c < 3; ++c)
    for (int r = 0; r < 3; ++r) s[c * 3 + r] = 0.5 * (cov[c * 3 + r] + cov[r * 3 + c]);
  if (!psm_llt3(s, l)) {
    const double tr = (s[0] + s[4]) + s[8];
    const double eps = 1e-8 * (tr > 1e-12 ? tr : 1e-12);
    s[0] += eps;
    s[4] += eps;
    s[8] += eps;
    psm_llt3(s, l);  // as the reference, the retry's outcome is used unchecked
  }
  psm_llt3_inverse(l, inv);
}

// One surfel against the n_alive alive queries: fq[a * c_ins + c], mean[a * 3 + i],
// inv[a * 9 + c * 3 + r] (column-major). Writes A to a_vals[a * a_stride] and then the
// softmax probability over it (in place); returns the argmax among the alive queries.
PSM_PHD int psm_assign_one(const double* f_ins, int c_ins, const double* center, int n_alive, const double* fq,
                           const double* mean, const double* inv, double* a_vals, int64_t a_stride,
                           const uint64_t* tab) {
  double a_max = -1;
  for (int a = 0; a < n_alive; ++a) {
    const double sim = psm_sigmoid_t(psm_dot_dyn(fq + a * c_ins, f_ins, c_ins), tab);
    const double d0 = center[0] - mean[a * 3 + 0];
    const double d1 = center[1] - mean[a * 3 + 1];
    const double d2 = center[2] - mean[a * 3 + 2];
    const double* m = inv + a * 9;
    const double v0 = (m[0] * d0 + m[3] * d1) + m[6] * d2;
    const double v1 = (m[1] * d0 + m[4] * d1) + m[7] * d2;
    const double v2 = (m[2] * d0 + m[5] * d1) + m[8] * d2;
    const double q = (d0 * v0 + d1 * v1) + d2 * v2;
    const double geo = psm_label_exp(-0.5 * q, tab, 2);
    const double av = sim * geo;
    a_vals[a * a_stride] = av;
    a_max = av > a_max ? av : a_max;  // std::max(a_max, av)
  }
  // exp(A - A_max) is evaluated once per query (the reference evaluates the same
  // argument twice, panoptic.cpp:79,83; exp is deterministic, so the values agree)
  double denom = 0;
  int best = 0;
  double best_a = a_vals[0];
  for (int a = 0; a < n_alive; ++a) {
    const double av = a_vals[a * a_stride];
    if (av > best_a) {
      best = a;
      best_a = av;
    }
    const double e = psm_label_exp(av - a_max, tab, 1);
    a_vals[a * a_stride] = e;
    denom += e;
  }
  for (int a = 0; a < n_alive; ++a) a_vals[a * a_stride] = a_vals[a * a_stride] / denom;
  return best;
}

#endif  // PSM_PANOPTIC_H
