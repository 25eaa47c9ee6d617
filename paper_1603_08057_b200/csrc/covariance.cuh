// Covariance entries Sigma(theta) and Sigma_i = dSigma/dtheta_i, evaluated on the fly.
//
//   Sigma_jk = sigma2 * k(r_jk) + nugget * [j == k]            (index delta, R-H/R-I)
//   rq        k = (1 + r^2 / (2 alpha rho^2))^-alpha
//   matern12  k = exp(-s),                s = r / rho            P:912-917 (nu = 1/2)
//   matern32  k = (1 + s) exp(-s),        s = sqrt(3) r / rho
//   matern52  k = (1 + s + s^2/3) exp(-s), s = sqrt(5) r / rho
//   sqexp     k = exp(-r^2 / (2 rho^2))   (alpha -> inf RQ limit; test family)
// Derivatives by the chain rule; d/dalpha of RQ uses a 5-term series of
// u/(alpha+u) - log1p(u/alpha) when u/alpha < 1e-3 (the direct form cancels).
#pragma once
#include <cuda_runtime.h>

namespace rsf {

enum Family { FAM_RQ = 0, FAM_M12 = 1, FAM_M32 = 2, FAM_M52 = 3, FAM_SQEXP = 4 };
// which matrix: -1 Sigma, else the theta component (rsf_param)
enum Which { W_SIGMA = -1, W_RHO = 0, W_SIGMA2 = 1, W_NUGGET = 2, W_ALPHA = 3, W_RHO2 = 4 };

struct KParams {
  int family;
  double rho, sigma2, nugget, alpha;
  double rho2 = 0.0;   // > 0: anisotropic per-axis lengths (rho, rho2), scaled distance of P:704-708
};

__host__ __device__ inline double k_unit(const KParams& p, double r) {
  switch (p.family) {
    case FAM_RQ: {
      double u = r * r / (2.0 * p.rho * p.rho);
      return exp(-p.alpha * log1p(u / p.alpha));
    }
    case FAM_M12: return exp(-r / p.rho);
    case FAM_M32: {
      double s = 1.7320508075688772 * r / p.rho;
      return (1.0 + s) * exp(-s);
    }
    case FAM_M52: {
      double s = 2.23606797749979 * r / p.rho;
      return (1.0 + s + s * s * (1.0 / 3.0)) * exp(-s);
    }
    default: return exp(-r * r / (2.0 * p.rho * p.rho));
  }
}

__host__ __device__ inline double dk_rho(const KParams& p, double r) {
  switch (p.family) {
    case FAM_RQ: {
      double u = r * r / (2.0 * p.rho * p.rho);
      return (r * r / (p.rho * p.rho * p.rho)) * exp((-p.alpha - 1.0) * log1p(u / p.alpha));
    }
    case FAM_M12: {
      double s = r / p.rho;
      return (s / p.rho) * exp(-s);
    }
    case FAM_M32: {
      double s = 1.7320508075688772 * r / p.rho;
      return (s * s / p.rho) * exp(-s);
    }
    case FAM_M52: {
      double s = 2.23606797749979 * r / p.rho;
      return s * s * (1.0 + s) * exp(-s) / (3.0 * p.rho);
    }
    default: return (r * r / (p.rho * p.rho * p.rho)) * exp(-r * r / (2.0 * p.rho * p.rho));
  }
}

__host__ __device__ inline double dk_alpha(const KParams& p, double r) {
  double u = r * r / (2.0 * p.rho * p.rho);
  double x = u / p.alpha;
  double k = exp(-p.alpha * log1p(x));
  double br;
  if (x < 1e-3) {
    // sum_{j>=2} (-1)^(j+1) (j-1)/j x^j
    br = x * x * (-0.5 + x * (2.0 / 3.0 + x * (-0.75 + x * (0.8 + x * (-5.0 / 6.0)))));
  } else {
    br = u / (p.alpha + u) - log1p(x);
  }
  return k * br;
}

// entry of the matrix `which` between two points at distance r; `same` = same index
__host__ __device__ inline double entry(const KParams& p, int which, double r, bool same) {
  switch (which) {
    case W_SIGMA: return same ? p.sigma2 + p.nugget : p.sigma2 * k_unit(p, r);
    case W_RHO: return same ? 0.0 : p.sigma2 * dk_rho(p, r);
    case W_SIGMA2: return same ? 1.0 : k_unit(p, r);
    case W_NUGGET: return same ? 1.0 : 0.0;
    default: return (same || p.family != FAM_RQ) ? 0.0 : p.sigma2 * dk_alpha(p, r);
  }
}

// d k(q) / d rho at rho = 1, divided by q^2 (finite as q -> 0 except for matern12, where the
// factor dx^2 / q of the caller keeps the product bounded)
__host__ __device__ inline double dk_rho_over_q2(const KParams& p, double q) {
  switch (p.family) {
    case FAM_RQ: return exp((-p.alpha - 1.0) * log1p(q * q / (2.0 * p.alpha)));
    case FAM_M12: return q > 0.0 ? exp(-q) / q : 0.0;
    case FAM_M32: return 3.0 * exp(-1.7320508075688772 * q);
    case FAM_M52: { const double s = 2.23606797749979 * q; return (5.0 / 3.0) * (1.0 + s) * exp(-s); }
    default: return exp(-0.5 * q * q);
  }
}

// entry between two points with coordinate differences (dx, dy).  Isotropic (rho2 == 0): the
// family of k(r / rho).  Anisotropic: q = ||x - y||_theta = sqrt(dx^2/rho^2 +
// dy^2/rho2^2) and k(q) is the family at unit length; d/d rho_1 = k'(q) dq/drho_1 with
// dq/drho_1 = -dx^2 / (rho_1^3 q), i.e. (dk/drho|_{rho=1} / q^2) * dx^2 / rho_1^3.
__host__ __device__ inline double entry_xy(const KParams& p, int which, double dx, double dy, bool same) {
  if (!(p.rho2 > 0.0)) return entry(p, which, sqrt(dx * dx + dy * dy), same);
  const double ax = dx / p.rho, ay = dy / p.rho2;
  const double q = sqrt(ax * ax + ay * ay);
  KParams u = p;
  u.rho = 1.0;
  switch (which) {
    case W_SIGMA: return same ? p.sigma2 + p.nugget : p.sigma2 * k_unit(u, q);
    case W_SIGMA2: return same ? 1.0 : k_unit(u, q);
    case W_NUGGET: return same ? 1.0 : 0.0;
    case W_RHO: return same ? 0.0 : p.sigma2 * dk_rho_over_q2(u, q) * dx * dx / (p.rho * p.rho * p.rho);
    case W_RHO2: return same ? 0.0 : p.sigma2 * dk_rho_over_q2(u, q) * dy * dy / (p.rho2 * p.rho2 * p.rho2);
    default: return (same || p.family != FAM_RQ) ? 0.0 : p.sigma2 * dk_alpha(u, q);
  }
}

}  // namespace rsf
