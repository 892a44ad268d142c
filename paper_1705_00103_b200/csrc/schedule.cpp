// Host weight scheduler of the CJM.
//
// kappa bounds  : P:100-106 (Eq. kmkM9p), P:126-134 (17-pt), classical 5-pt
//                 (S:249-257), evaluated at N = unknowns + 1 (DESIGN R1)
// cycle length  : M_min = ceil(acosh(1/tol) / acosh(mu)), mu = (kmax+kmin)/
//                 (kmax-kmin) ("depends on ... the required tolerance";
//                 S:292), acosh(mu) via log1p (DESIGN R5); P = min 2^a 3^b >= M
//                 (CJM_ORDER_LEBEDEV2: P = min 2^a >= M)
// ordering      : generalised Lebedev-Finogenov recursion (DESIGN R3)
// weights       : w = 1/(kmin + (kmax-kmin) sin^2(t pi / 4P))  (the
//                 half-angle form of S:292's 2/[(kmax+kmin)-(kmax-kmin)cos])
//
// The floating-point expressions follow DESIGN R5 literally (same operations
// in the same order) so that the weights are reproducible bit for bit.
#include "internal.h"

#include <cmath>
#include <cstdint>
#include <vector>

namespace cjm {

int stencil_reach(int stencil) {
  switch (stencil) {
    case 5: case 9: return 1;
    case 17: return 2;
    default: return 0;
  }
}

static inline double sq_sin(double a) {
  const double s = std::sin(a);
  return s * s;
}

bool spectral_bounds(int stencil, int nx, int ny, double* kmin, double* kmax) {
  const double Nx = double(nx) + 1.0;  // mesh intervals (DESIGN R1)
  const double Ny = double(ny) + 1.0;
  const double ax = M_PI / (2.0 * Nx), ay = M_PI / (2.0 * Ny);  // pi / 2N
  const double bx = M_PI / Nx, by = M_PI / Ny;                  // pi / N
  switch (stencil) {
    case 5:
      *kmin = sq_sin(ax) + sq_sin(ay);
      *kmax = 2.0;
      return true;
    case 9:
      *kmin = (4.0 / 5.0) * (sq_sin(ax) + sq_sin(ay)) +
              (1.0 / 5.0) * (sq_sin(ax + ay) + sq_sin(ax - ay));
      *kmax = 8.0 / 5.0;
      return true;
    case 17:  // P:128-133 (garbled braces read as DESIGN R2)
      *kmin = -(4.0 / 75.0) * (sq_sin(bx) + sq_sin(by)) +
              (64.0 / 75.0) * (sq_sin(ax) + sq_sin(ay)) -
              (1.0 / 75.0) * (sq_sin(bx + by) + sq_sin(bx - by)) +
              (16.0 / 75.0) * (sq_sin(ax + ay) + sq_sin(ax - ay));
      *kmax = 128.0 / 75.0;
      return true;
    default:
      return false;
  }
}

long long chebyshev_degree(double kmin, double kmax, double tol) {
  const double x = 2.0 * kmin / (kmax - kmin);             // mu - 1
  const double acosh_mu = std::log1p(x + std::sqrt(x * (2.0 + x)));
  double m = std::ceil(std::acosh(1.0 / tol) / acosh_mu);
  return m < 1.0 ? 1 : (long long)m;
}

long long smooth_cycle_length(long long m, int* a_out, int* b_out) {
  // enumerate 3^b, then the smallest power of two lifting it to >= m
  long long best = -1;
  int ba = 0, bb = 0;
  long long p3 = 1;
  for (int b = 0; b < 40; ++b) {
    long long v = p3;
    int a = 0;
    while (v < m) { v *= 2; ++a; }
    if (best < 0 || v < best) { best = v; ba = a; bb = b; }
    if (p3 >= m) break;
    p3 *= 3;
  }
  *a_out = ba;
  *b_out = bb;
  return best;
}

std::vector<long long> lebedev23_order(int a, int b) {
  std::vector<long long> cur{1}, next;
  long long m = 1;
  for (int f_idx = 0; f_idx < a + b; ++f_idx) {
    const int f = f_idx < b ? 3 : 2;   // factors of 3 first (DESIGN R3)
    next.clear();
    next.reserve(cur.size() * f);
    for (long long t : cur) {
      next.push_back(t);
      next.push_back(4 * m - t);
      if (f == 3) next.push_back(4 * m + t);
    }
    cur.swap(next);
    m *= f;
  }
  return cur;
}

bool build_schedule_bounds(double kmin, double kmax, double tol, int order, Schedule* s) {
  if (!(kmin > 0.0 && kmax > kmin) || !std::isfinite(kmax)) return false;
  s->kmin = kmin;
  s->kmax = kmax;
  s->m_min = chebyshev_degree(s->kmin, s->kmax, tol);
  int a = 0, b = 0;
  s->P = smooth_cycle_length(s->m_min, &a, &b);
  if (order == 2) {   // power-of-two cycle: P = smallest 2^a >= M_min
    a = 0;
    b = 0;
    for (s->P = 1; s->P < s->m_min; s->P *= 2) ++a;
  }
  if (order == 0 || order == 2) {
    s->t = lebedev23_order(a, b);
  } else if (order == 1) {  // ascending weights = descending zero index
    s->t.resize(s->P);
    for (long long k = 0; k < s->P; ++k) s->t[k] = 2 * (s->P - k) - 1;
  } else {
    return false;
  }
  s->w.resize(s->P);
  const double span = s->kmax - s->kmin;
  for (long long k = 0; k < s->P; ++k) {
    const double theta = (M_PI * double(s->t[k])) / (4.0 * double(s->P));
    const double sn = std::sin(theta);
    s->w[k] = 1.0 / (s->kmin + span * (sn * sn));
  }
  return true;
}

bool build_schedule(int stencil, int nx, int ny, double tol, int order, Schedule* s) {
  double kmin = 0, kmax = 0;
  if (!spectral_bounds(stencil, nx, ny, &kmin, &kmax)) return false;
  return build_schedule_bounds(kmin, kmax, tol, order, s);
}

}  // namespace cjm
