// host_tables.cpp — fp64 table arithmetic on the host (see host_tables.hpp).
// Each routine follows the reference's operation order so its outputs are
// bitwise the reference's; citations are to /root/reference/proj/src.
#include "host_tables.hpp"

#include <algorithm>
#include <cmath>
#include <string>

#include "ermc_b200.hpp"

namespace ermc_host {

namespace {
constexpr double kPiH = ermc::kPi;
constexpr double kSigmaH = ermc::kSigma;

void check_bands(int nb, const double* lo, const double* hi) {
  // validate_bands (spectral.cpp:80-89)
  if (nb <= 0) throw ermc::Error("SpectralModel: no bands");
  for (int n = 0; n < nb; ++n) {
    if (hi[n] <= lo[n])
      throw ermc::Error("SpectralModel: band " + std::to_string(n) +
                        " has non-positive width");
    if (n > 0 && lo[n] < hi[n - 1] - 1e-9)
      throw ermc::Error("SpectralModel: bands overlap at index " +
                        std::to_string(n));
  }
}

double sigma_t4(double t) { return kSigmaH * t * t * t * t; }
}  // namespace

std::string fmt_double(double v) { return std::to_string(v); }

TableView make_view_unchecked(const ermc_model_t& m) {
  TableView v;
  v.nb = m.n_bands;
  v.nq = m.n_quad;
  v.nt = m.n_temps;
  v.nu_lo = m.band_nu_lo;
  v.nu_hi = m.band_nu_hi;
  v.g_weights = m.g_weights;
  v.temps = m.temp_grid;
  v.k = m.k_table;
  v.ib = m.ib_table;
  // Uniform temperature grids get a direct-index lookup (spectral.cpp:119-129).
  if (v.nt >= 2) {
    v.t0 = v.temps[0];
    v.dt = v.temps[1] - v.temps[0];
    v.uniform = true;
    for (int t = 1; t < v.nt; ++t)
      if (std::abs(v.temps[t] - (v.t0 + t * v.dt)) > 1e-9 * v.dt) {
        v.uniform = false;
        break;
      }
  }
  return v;
}

TableView make_view(const ermc_model_t& m) {
  check_bands(m.n_bands, m.band_nu_lo, m.band_nu_hi);
  if (m.n_temps <= 0) throw ermc::Error("SpectralModel: empty temperature grid");
  for (int t = 1; t < m.n_temps; ++t)
    if (m.temp_grid[t] <= m.temp_grid[t - 1])
      throw ermc::Error("SpectralModel: temperature grid must be ascending");
  double wsum = 0.0;
  for (int g = 0; g < m.n_quad; ++g) wsum += m.g_weights[g];
  if (std::abs(wsum - 1.0) > 1e-12)
    throw ermc::Error("SpectralModel: quadrature weights must sum to 1");
  const size_t nk = static_cast<size_t>(m.n_bands) * m.n_quad * m.n_temps;
  for (size_t i = 0; i < nk; ++i)
    if (m.k_table[i] < 0.0 || !std::isfinite(m.k_table[i]))
      throw ermc::Error("SpectralModel: k_table entries must be non-negative");
  return make_view_unchecked(m);
}

Lookup lookup(const TableView& v, double T) {
  // SpectralModel::lookup (spectral.cpp:148-177)
  if (!(T >= v.temps[0] && T <= v.temps[v.nt - 1]))
    throw ermc::Error("temperature " + fmt_double(T) +
                      " K outside table range [" + fmt_double(v.temps[0]) +
                      ", " + fmt_double(v.temps[v.nt - 1]) + "]");
  if (v.nt < 2) return {0, 0.0};  // single node (the reference reads node -1)
  const double* tg = v.temps;
  if (v.uniform) {
    int lo = static_cast<int>((T - v.t0) / v.dt);
    lo = std::clamp(lo, 0, v.nt - 2);
    double frac = (T - tg[lo]) / (tg[lo + 1] - tg[lo]);
    if (frac < 0.0 && lo > 0) {
      --lo;
      frac = (T - tg[lo]) / (tg[lo + 1] - tg[lo]);
    } else if (frac > 1.0 && lo < v.nt - 2) {
      ++lo;
      frac = (T - tg[lo]) / (tg[lo + 1] - tg[lo]);
    }
    return {lo, frac};
  }
  const int hi = static_cast<int>(std::upper_bound(tg, tg + v.nt, T) - tg);
  if (hi == 0) return {0, 0.0};
  if (hi == v.nt) return {v.nt - 2, 1.0};
  const int lo = hi - 1;
  return {lo, (T - tg[lo]) / (tg[hi] - tg[lo])};
}

double interp_k(const TableView& v, int n, int g, double T) {
  const Lookup l = lookup(v, T);
  const double a = v.k_node(n, g, l.idx);
  if (l.frac == 0.0) return a;
  return a + l.frac * (v.k_node(n, g, l.idx + 1) - a);
}

double interp_ib(const TableView& v, int n, double T) {
  const Lookup l = lookup(v, T);
  const double a = v.ib_node(n, l.idx);
  if (l.frac == 0.0) return a;
  return a + l.frac * (v.ib_node(n, l.idx + 1) - a);
}

double planck_mean(const TableView& v, double T) {
  // spectral.cpp:207-218
  lookup(v, T);
  if (T <= 0.0) return 0.0;
  double sum = 0.0;
  for (int n = 0; n < v.nb; ++n) {
    double gk = 0.0;
    for (int g = 0; g < v.nq; ++g) gk += v.g_weights[g] * interp_k(v, n, g, T);
    sum += kPiH * (v.nu_hi[n] - v.nu_lo[n]) * interp_ib(v, n, T) * gk;
  }
  return sum / sigma_t4(T);
}

std::vector<double> kp_nodes(const TableView& v) {
  // spectral.cpp:131-145
  std::vector<double> kp(v.nt, 0.0);
  for (int t = 0; t < v.nt; ++t) {
    const double T = v.temps[t];
    if (T <= 0.0) continue;
    double sum = 0.0;
    for (int n = 0; n < v.nb; ++n) {
      double gk = 0.0;
      for (int g = 0; g < v.nq; ++g) gk += v.g_weights[g] * v.k_node(n, g, t);
      sum += kPiH * (v.nu_hi[n] - v.nu_lo[n]) * v.ib_node(n, t) * gk;
    }
    kp[t] = sum / sigma_t4(T);
  }
  return kp;
}

void build_cdfs(const TableView& v, double t_max, double* band_cdf,
                double* quad_cdf) {
  // spectral.cpp:306-354 — emission-weighted importance sampling at T_max.
  std::vector<double> weight(v.nb);
  double total = 0.0;
  for (int n = 0; n < v.nb; ++n) {
    double gk = 0.0;
    for (int g = 0; g < v.nq; ++g)
      gk += v.g_weights[g] * interp_k(v, n, g, t_max);
    weight[n] = kPiH * (v.nu_hi[n] - v.nu_lo[n]) * interp_ib(v, n, t_max) * gk;
    total += weight[n];
  }
  if (!(total > 0.0))
    throw ermc::Error("build_cdfs: medium is transparent at T_max (kappa_p = 0)");
  double cum = 0.0;
  for (int n = 0; n < v.nb; ++n) {
    cum += weight[n] / total;
    band_cdf[n] = cum;
  }
  band_cdf[v.nb - 1] = 1.0;

  std::vector<double> w(v.nq);
  for (int n = 0; n < v.nb; ++n) {
    double gsum = 0.0;
    for (int g = 0; g < v.nq; ++g) {
      w[g] = v.g_weights[g] * interp_k(v, n, g, t_max);
      gsum += w[g];
    }
    if (gsum <= 0.0) {  // unreachable band: keep a valid CDF
      for (int g = 0; g < v.nq; ++g) w[g] = v.g_weights[g];
      gsum = 1.0;
    }
    double c = 0.0;
    double* row = quad_cdf + static_cast<size_t>(n) * v.nq;
    for (int g = 0; g < v.nq; ++g) {
      c += w[g] / gsum;
      row[g] = c;
    }
    row[v.nq - 1] = 1.0;
  }
}

double planck_intensity_checked(double nu, double T) {
  // spectral.cpp:62-70, per cm^-1
  if (nu <= 0.0) throw ermc::Error("planck_intensity: wavenumber must be positive");
  if (T <= 0.0) throw ermc::Error("planck_intensity: temperature must be positive");
  const double nu_m = nu * 100.0;
  const double x = ermc::kPlanckC2 * nu_m / T;
  return 100.0 * ermc::kPlanckC1 * nu_m * nu_m * nu_m / std::expm1(x);
}

}  // namespace ermc_host
