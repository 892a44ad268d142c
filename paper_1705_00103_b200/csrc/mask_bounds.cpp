// Host estimate of the spectral bounds of D^-1 A for a generic 5-point mask
// (the numeric fallback NEXT-4 needs; the paper's closed forms,
// P:78-84 / P:100-106, only cover the Cartesian stencils).
//
// D^-1 A = I - N with (N x)_k = sum_q a_q x_q, a_q = -c_q / c_C over the
// interior neighbours q in {W, E, S, N} (the Dirichlet ghosts drop out).  The
// 5-point graph of the grid is bipartite (every neighbour flips the parity of
// i + j), so if N v = mu v then N (s v) = -mu (s v) with s = (-1)^(i+j): the
// spectrum of N is symmetric about 0 and that of D^-1 A about 1.  Hence
//     kappa_min = 1 - rho(N),   kappa_max = 1 + rho(N),
// and only rho(N) has to be estimated.  Power iteration from the positive,
// smooth vector sin(pi i/(nx+1)) sin(pi j/(ny+1)) (the exact dominant
// eigenvector of the Cartesian mask, close to it for smooth coefficients):
// rho ~ ||N x|| / ||x||.  Both +rho and -rho eigen-components are scaled by
// rho, so the norm ratio converges to rho even when x has a component on the
// checkerboard eigenvector.  The ratio approaches rho from below for a
// symmetrisable N: kappa_min is then slightly over-estimated (the caller may
// shrink it; Chebyshev weights on a slightly too short interval still
// converge, only more slowly).
#include "internal.h"

#include <cmath>
#include <vector>

namespace cjm {

bool mask_spectral_bounds(int nx, int ny, const double* cW, const double* cE, const double* cS,
                          const double* cN, const double* cC, long long ldc, int iters,
                          double* kmin, double* kmax) {
  if (nx < 1 || ny < 1 || ldc < nx || !cW || !cE || !cS || !cN || !cC || iters < 1) return false;
  const size_t n = (size_t)nx * ny;
  std::vector<double> a(4 * n), x(n), y(n);
  for (int j = 0; j < ny; ++j)
    for (int i = 0; i < nx; ++i) {
      const long long k = (long long)j * ldc + i;
      const double cc = cC[k];
      if (!(cc != 0.0) || !std::isfinite(cc)) return false;
      const size_t e = (size_t)j * nx + i;
      // interior couplings only: ghost neighbours carry Dirichlet data
      a[4 * e + 0] = i > 0 ? -cW[k] / cc : 0.0;
      a[4 * e + 1] = i + 1 < nx ? -cE[k] / cc : 0.0;
      a[4 * e + 2] = j > 0 ? -cS[k] / cc : 0.0;
      a[4 * e + 3] = j + 1 < ny ? -cN[k] / cc : 0.0;
      x[e] = std::sin(M_PI * (i + 1) / (nx + 1.0)) * std::sin(M_PI * (j + 1) / (ny + 1.0));
    }
  auto apply = [&](const std::vector<double>& in, std::vector<double>& out) {
    for (int j = 0; j < ny; ++j)
      for (int i = 0; i < nx; ++i) {
        const size_t e = (size_t)j * nx + i;
        double s = 0.0;
        if (i > 0) s += a[4 * e + 0] * in[e - 1];
        if (i + 1 < nx) s += a[4 * e + 1] * in[e + 1];
        if (j > 0) s += a[4 * e + 2] * in[e - nx];
        if (j + 1 < ny) s += a[4 * e + 3] * in[e + nx];
        out[e] = s;
      }
  };
  auto norm = [](const std::vector<double>& v) {
    double s = 0.0;
    for (double q : v) s += q * q;
    return std::sqrt(s);
  };
  double nrm = norm(x), rho = 0.0;
  for (int it = 0; it < iters; ++it) {
    for (double& q : x) q /= nrm;
    apply(x, y);
    nrm = norm(y);
    rho = nrm;                    // ||N x|| with ||x|| = 1
    if (!(nrm > 0.0) || !std::isfinite(nrm)) return false;
    x.swap(y);
  }
  if (!(rho < 1.0)) return false;  // D^-1 A not positive definite: CJM does not apply
  *kmin = 1.0 - rho;
  *kmax = 1.0 + rho;
  return true;
}

// Square (2m+1)^2 masks (cjm_mask_bounds_n): no bipartite symmetry, so both
// ends are estimated.  B = D^-1 A, (B x)_k = x_k - sum_q a_q x_{k+q} over the
// interior neighbours (a_q = -c_q / c_C).  kappa_max: power iteration on B
// (the norm ratio ||B x|| / ||x||, from below for a symmetrisable B);
// kappa_min: power iteration on sigma I - B with sigma = kappa_max (its
// dominant eigenvalue is sigma - kappa_min).  Both start from the smooth
// positive vector; cost 2 x iters x nx x ny x (2m+1)^2 on one host core.
bool mask_spectral_bounds_n(int m, int nx, int ny, const double* const* c, long long ldc,
                            int iters, double* kmin, double* kmax) {
  if (m < 1 || m > 2 || nx < 1 || ny < 1 || ldc < nx || !c || iters < 1) return false;
  const int S = 2 * m + 1, QC = m * S + m;
  if (!c[QC]) return false;
  const size_t n = (size_t)nx * ny;
  std::vector<double> x0(n), x(n), y(n);
  for (int j = 0; j < ny; ++j)
    for (int i = 0; i < nx; ++i) {
      const double cc = c[QC][(long long)j * ldc + i];
      if (!(cc != 0.0) || !std::isfinite(cc)) return false;
      x0[(size_t)j * nx + i] =
          std::sin(M_PI * (i + 1) / (nx + 1.0)) * std::sin(M_PI * (j + 1) / (ny + 1.0));
    }
  // out = shift * in - B in
  auto apply = [&](double shift, const std::vector<double>& in, std::vector<double>& out) {
    for (int j = 0; j < ny; ++j)
      for (int i = 0; i < nx; ++i) {
        const long long k = (long long)j * ldc + i;
        const size_t e = (size_t)j * nx + i;
        const double cc = c[QC][k];
        double s = 0.0;
        for (int q = 0; q < S * S; ++q) {
          if (q == QC || !c[q]) continue;
          const int ii = i + q % S - m, jj = j + q / S - m;
          if (ii < 0 || ii >= nx || jj < 0 || jj >= ny) continue;   // Dirichlet ghost
          s += (-c[q][k] / cc) * in[(size_t)jj * nx + ii];
        }
        out[e] = shift * in[e] - (in[e] - s);
      }
  };
  auto norm = [](const std::vector<double>& v) {
    double s = 0.0;
    for (double q : v) s += q * q;
    return std::sqrt(s);
  };
  auto power = [&](double shift, double sign, double* lam) {
    x = x0;
    double nrm = norm(x);
    for (int it = 0; it < iters; ++it) {
      for (double& q : x) q /= nrm;
      apply(shift, x, y);
      for (double& q : y) q *= sign;
      nrm = norm(y);
      if (!(nrm > 0.0) || !std::isfinite(nrm)) return false;
      x.swap(y);
    }
    *lam = nrm;
    return true;
  };
  double lmax = 0.0, mu = 0.0;
  if (!power(0.0, -1.0, &lmax)) return false;          // ||B x||: 0 I - B, sign flipped
  if (!power(lmax, 1.0, &mu)) return false;             // ||(lmax I - B) x||
  const double lmin = lmax - mu;
  if (!(lmin > 0.0) || !(lmax > lmin)) return false;    // not positive definite: CJM does not apply
  *kmin = lmin;
  *kmax = lmax;
  return true;
}

}  // namespace cjm
