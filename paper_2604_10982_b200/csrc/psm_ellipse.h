// psm_ellipse.h — "Precise Tile Intersection" as an exact support-ellipse vs
// tile test (north-star extension of bin_aabb, proj/src/raster.cpp:43-49,149-152).
//
// The reference keeps a surfel in every tile its AABB [cx +- sqrt(chi2 F00),
// cy +- sqrt(chi2 F11)] touches (F = Sigma' + 0.3 I, raster.cpp:17-24). A pixel
// only ever uses a candidate whose support test d^T F^-1 d <= chi2 passes at
// its pixel centre (raster.cpp:375-382), so a tile whose pixel centres all lie
// outside the ellipse can be dropped without changing any output. This header
// computes, per tile row of the AABB, the contiguous run of tiles whose
// pixel-centre rectangle meets the (slightly inflated) ellipse:
//   for fixed dy the ellipse's x-extent is  (F01/F11) dy +- sqrt((k F11 - dy^2) det F) / F11,
//   its right edge is concave in dy with maximum at dy* = F01 sqrt(k / F00)
//   (left edge convex, minimum at -dy*), so the extent over a strip of rows is
//   the edge evaluated at dy* clamped into the strip.
// Margins (relative 1e-6 on chi2, 1e-3 px on the interval) make the test
// conservative against the fp64 rounding of the per-pixel support test;
// tests/test_oracle_kat.py::test_ellipse_binning_conservative checks it
// exhaustively. Ill-conditioned footprints fall back to the AABB row.
// Shared verbatim by the CUDA kernels and the oracle so both produce the same
// tile lists.
#ifndef PSM_ELLIPSE_H
#define PSM_ELLIPSE_H

#if defined(__CUDACC__)
#define PSM_EHD __host__ __device__ __forceinline__
#else
#define PSM_EHD static inline
#include <math.h>
#endif

// x / ts. For a power-of-two tile size the quotient is exact-scaled, so multiplying by
// the (exact) reciprocal gives the identical double without a division.
PSM_EHD double psm_div_tile(double x, int ts) { return (ts & (ts - 1)) == 0 ? x * (1.0 / ts) : x / ts; }

// Per-surfel constants of the row test (computed once per surfel, used per tile row).
struct PsmEllipse {
  double cx, cy;
  double ymax;   // sqrt(k F11): y half-extent
  double slope;  // F01 / F11: centre line x = slope * dy
  double dstar;  // F01 sqrt(k / F00): dy of the rightmost point
  double kf11;   // k F11
  double q;      // det F / F11^2: half-width(dy) = sqrt((k F11 - dy^2) q)
  int ok;        // 0: degenerate / ill-conditioned -> every AABB row is kept
};

PSM_EHD PsmEllipse psm_ellipse_prep(double cx, double cy, double f00, double f01, double f11, double chi2) {
  PsmEllipse e;
  const double k = chi2 * 1.000001 + 1e-9;
  const double det = f00 * f11 - f01 * f01;
  const double tr = f00 + f11;
  e.cx = cx;
  e.cy = cy;
  e.ok = (det > 0.0) && (tr * tr < 1e12 * det);
  e.ymax = e.ok ? sqrt(k * f11) : 0.0;
  e.slope = e.ok ? f01 / f11 : 0.0;
  e.dstar = e.ok ? f01 * sqrt(k / f00) : 0.0;
  e.kf11 = k * f11;
  e.q = e.ok ? det / (f11 * f11) : 0.0;
  return e;
}

// x-extent [*xl, *xr] (with the 1e-3 px margin) of the ellipse over the rows of pixel
// centres y in [y_lo, y_hi]. Returns 0 if the strip misses the ellipse's y-extent.
// Requires e.ok.
PSM_EHD int psm_ellipse_span(const PsmEllipse& e, double y_lo, double y_hi, double* xl, double* xr) {
  double dlo = y_lo - e.cy;
  double dhi = y_hi - e.cy;
  if (dlo < -e.ymax) dlo = -e.ymax;
  if (dhi > e.ymax) dhi = e.ymax;
  if (dlo > dhi + 1e-3) return 0;  // strip misses the ellipse's y-extent
  double dr = e.dstar;             // maximiser of the right edge, clamped into the strip
  if (dr < dlo) dr = dlo;
  if (dr > dhi) dr = dhi;
  double dl = -e.dstar;            // minimiser of the left edge
  if (dl < dlo) dl = dlo;
  if (dl > dhi) dl = dhi;
  double rr = e.kf11 - dr * dr;
  double rl = e.kf11 - dl * dl;
  if (rr < 0.0) rr = 0.0;
  if (rl < 0.0) rl = 0.0;
  *xr = e.cx + e.slope * dr + sqrt(rr * e.q) + 1e-3;
  *xl = e.cx + e.slope * dl - sqrt(rl * e.q) - 1e-3;
  return 1;
}

// Tile-column run [*tx_lo, *tx_hi] of tile row `ty` met by the ellipse, intersected
// with the AABB columns [ax0, ax1]. Returns 0 if the row is empty.
PSM_EHD int psm_ellipse_row(const PsmEllipse& e, int ty, int ts, int height, int ax0, int ax1, int* tx_lo,
                            int* tx_hi) {
  if (!e.ok) {  // degenerate / ill-conditioned: keep the AABB row
    *tx_lo = ax0;
    *tx_hi = ax1;
    return ax0 <= ax1;
  }
  const double y_lo = ty * ts + 0.5;
  int y_end = ty * ts + ts;
  if (y_end > height) y_end = height;
  const double y_hi = y_end - 0.5;
  double xl, xr;
  if (!psm_ellipse_span(e, y_lo, y_hi, &xl, &xr)) return 0;
  // tiles whose pixel-centre span [tx*ts + 0.5, tx*ts + ts - 0.5] meets [xl, xr]
  double lo = ceil(psm_div_tile(xl - (ts - 0.5), ts));
  double hi = floor(psm_div_tile(xr - 0.5, ts));
  if (!(lo == lo) || !(hi == hi)) {  // NaN anywhere: keep the AABB row
    lo = ax0;
    hi = ax1;
  }
  if (lo < ax0) lo = ax0;
  if (hi > ax1) hi = ax1;
  if (lo > hi) return 0;
  *tx_lo = static_cast<int>(lo);
  *tx_hi = static_cast<int>(hi);
  return 1;
}

#endif  // PSM_ELLIPSE_H
