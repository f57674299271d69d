// host_tables.hpp — host-side table arithmetic shared by the C-ABI (which
// precomputes everything the trace kernel consumes) and the C++ API
// (SpectralModel members). All functions reproduce the reference's fp64
// operation order so that T_max-derived inputs are bitwise the reference's.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "ermc_b200.h"

namespace ermc_host {

// Read-only view of a model's tables plus the uniform-grid detection the
// reference does in its SpectralModel constructor (spectral.cpp:119-129).
struct TableView {
  int nb = 0, nq = 0, nt = 0;
  const double* nu_lo = nullptr;
  const double* nu_hi = nullptr;
  const double* g_weights = nullptr;
  const double* temps = nullptr;
  const double* k = nullptr;   // [nb][nq][nt]
  const double* ib = nullptr;  // [nb][nt]
  bool uniform = false;
  double t0 = 0.0, dt = 1.0;

  double k_node(int n, int g, int t) const {
    return k[(static_cast<size_t>(n) * nq + g) * nt + t];
  }
  double ib_node(int n, int t) const {
    return ib[static_cast<size_t>(n) * nt + t];
  }
};

// Builds the view and validates like SpectralModel's constructor
// (spectral.cpp:80-117); throws ermc::Error.
TableView make_view(const ermc_model_t& m);
// Same without validation (for already-validated SpectralModel objects).
TableView make_view_unchecked(const ermc_model_t& m);

struct Lookup {
  int idx;
  double frac;
};
Lookup lookup(const TableView& v, double temperature);  // throws out of range
double interp_k(const TableView& v, int n, int g, double temperature);
double interp_ib(const TableView& v, int n, double temperature);
double planck_mean(const TableView& v, double temperature);
// kp at every node (constructor, spectral.cpp:131-145).
std::vector<double> kp_nodes(const TableView& v);
// build_cdfs (spectral.cpp:306-354): band_cdf[nb], quad_cdf[nb*nq].
void build_cdfs(const TableView& v, double t_max, double* band_cdf,
                double* quad_cdf);

// Band blackbody with the cold-wall limit folded in.
double planck_intensity_checked(double nu, double temperature);

// Error text helpers shared with the reference's formatting.
std::string fmt_double(double v);  // std::to_string

}  // namespace ermc_host
