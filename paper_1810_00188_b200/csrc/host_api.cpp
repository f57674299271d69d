// host_api.cpp — the ermc:: C++ API (include/ermc_b200.hpp).
//
// Setup objects (grids, boundaries, spectral tables and their builders) are
// host data, restated from the reference's documented behaviour with its
// fp64 operation order so that tables built here are bitwise the
// reference's (pinned by tests/test_host_parity.py). ermc::solve forwards to
// the C-ABI, which runs every cell and ray on the GPU.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <string>
#include <utility>

#include "ermc_b200.hpp"
#include "host_tables.hpp"

namespace ermc {

// ---------------------------------------------------------------- geometry

double CartesianGrid::min_spacing() const { return std::min({dx, dy, dz}); }

void CartesianGrid::validate() const {
  if (nx < 1 || ny < 1 || nz < 1)
    throw Error("CartesianGrid: cell counts must be >= 1");
  if (dx <= 0.0 || dy <= 0.0 || dz <= 0.0)
    throw Error("CartesianGrid: spacings must be positive");
}

void BoundarySpec::validate() const {
  for (int a = 0; a < 3; ++a) {
    if (periodic(a)) continue;
    for (const Wall& w : {lo[a], hi[a]}) {
      if (w.emissivity < 0.0 || w.emissivity > 1.0)
        throw Error("BoundarySpec: wall emissivity must be in [0,1]");
      if (w.temperature < 0.0)
        throw Error("BoundarySpec: wall temperature must be >= 0");
    }
  }
}

double TemperatureField::max_value() const {
  return *std::max_element(values.begin(), values.end());
}
double TemperatureField::min_value() const {
  return *std::min_element(values.begin(), values.end());
}

void TemperatureField::validate() const {
  grid.validate();
  if (static_cast<std::int64_t>(values.size()) != grid.cell_count())
    throw Error("TemperatureField: value count does not match grid");
  for (double v : values)
    if (!(v > 0.0)) throw Error("TemperatureField: temperatures must be positive");
}

TemperatureField restrict_field(const TemperatureField& fine, int ratio) {
  if (ratio < 2) throw Error("restrict_field: ratio must be >= 2");
  const CartesianGrid& f = fine.grid;
  TemperatureField out;
  CartesianGrid& c = out.grid;
  c.nx = (f.nx + ratio - 1) / ratio;
  c.ny = (f.ny + ratio - 1) / ratio;
  c.nz = (f.nz + ratio - 1) / ratio;
  c.dx = f.extent(0) / c.nx;
  c.dy = f.extent(1) / c.ny;
  c.dz = f.extent(2) / c.nz;
  c.origin = f.origin;
  out.values.resize(c.cell_count());
  for (int ci = 0; ci < c.nx; ++ci)
    for (int cj = 0; cj < c.ny; ++cj)
      for (int ck = 0; ck < c.nz; ++ck) {
        double sum = 0.0;
        int n = 0;
        const int i1 = std::min((ci + 1) * ratio, f.nx);
        const int j1 = std::min((cj + 1) * ratio, f.ny);
        const int k1 = std::min((ck + 1) * ratio, f.nz);
        for (int i = ci * ratio; i < i1; ++i)
          for (int j = cj * ratio; j < j1; ++j)
            for (int k = ck * ratio; k < k1; ++k, ++n) sum += fine.values[f.linear(i, j, k)];
        out.values[c.linear(ci, cj, ck)] = sum / n;
      }
  return out;
}

GridHierarchy build_hierarchy(const CartesianGrid& grid,
                              const std::vector<double>& field, int n_levels,
                              int ratio, int steps_per_level) {
  grid.validate();
  if (n_levels < 1) throw Error("build_hierarchy: n_levels must be >= 1");
  if (n_levels > 1 && ratio < 2) throw Error("build_hierarchy: ratio must be >= 2");
  if (static_cast<std::int64_t>(field.size()) != grid.cell_count())
    throw Error("build_hierarchy: field size does not match grid");
  GridHierarchy h;
  TemperatureField level{grid, field};
  h.grids.push_back(grid);
  h.fields.push_back(field);
  for (int l = 1; l < n_levels; ++l) {
    const CartesianGrid& g = h.grids.back();
    if (g.nx == 1 && g.ny == 1 && g.nz == 1)
      throw Error("build_hierarchy: cannot coarsen below one cell; achievable "
                  "depth is " + std::to_string(l));
    level = restrict_field(level, ratio);
    h.grids.push_back(level.grid);
    h.fields.push_back(level.values);
  }
  h.step_caps.assign(n_levels, steps_per_level);
  h.step_caps.back() = -1;
  return h;
}

std::array<int, 3> locate(const CartesianGrid& grid, const Vec3& p) {
  std::array<int, 3> idx{};
  for (int a = 0; a < 3; ++a) {
    const double rel = (p[a] - grid.origin[a]) / grid.spacing(a);
    int i = static_cast<int>(std::floor(rel));
    const int n = grid.count(a);
    if (i < 0 || i >= n) {
      if (rel >= -1e-9 && i < 0)
        i = 0;
      else if (rel <= n + 1e-9 && i >= n)
        i = n - 1;
      else
        throw Error("locate: point outside domain on axis " + std::to_string(a));
    }
    idx[a] = i;
  }
  return idx;
}

std::array<int, 3> locate(const CartesianGrid& grid, const Vec3& p,
                          const Vec3& dir) {
  const double e = geom_eps(grid);
  return locate(grid, {p[0] + e * dir[0], p[1] + e * dir[1], p[2] + e * dir[2]});
}

// ---------------------------------------------------------------- spectral

FaceCrossing face_distances(const CartesianGrid& grid, const Vec3& pos, const Vec3& dir,
                            int i, int j, int k) {
  FaceCrossing fc;
  const int idx[3] = {i, j, k};
  for (int a = 0; a < 3; ++a) {
    if (dir[a] == 0.0) {
      fc.df[a] = kInf;
      continue;
    }
    const double face = grid.origin[a] + (idx[a] + (dir[a] > 0.0 ? 1 : 0)) * grid.spacing(a);
    fc.df[a] = (face - pos[a]) / dir[a];
  }
  fc.ds = fc.df[0];
  for (int a = 1; a < 3; ++a)
    if (fc.df[a] < fc.ds) {
      fc.ds = fc.df[a];
      fc.axis = a;
    }
  fc.ds = std::max(fc.ds, 0.0);
  return fc;
}

QuadratureSet QuadratureSet::gauss_legendre(int n) {
  if (n < 1) throw Error("gauss_legendre: need at least one point");
  QuadratureSet q;
  q.g_points.assign(n, 0.0);
  q.weights.assign(n, 0.0);
  // Newton on P_n from the asymptotic root guess; map (-1,1) -> (0,1).
  for (int r = 0; r < n; ++r) {
    double x = std::cos(kPi * (r + 0.75) / (n + 0.5));
    double deriv = 0.0;
    for (int it = 0; it < 100; ++it) {
      double pm1 = 1.0, p = x;
      for (int j = 2; j <= n; ++j) {
        const double pn = ((2 * j - 1) * x * p - (j - 1) * pm1) / j;
        pm1 = p;
        p = pn;
      }
      deriv = n * (x * p - pm1) / (x * x - 1.0);
      const double step = p / deriv;
      x -= step;
      if (std::abs(step) < 1e-15) break;
    }
    q.g_points[n - 1 - r] = 0.5 * (x + 1.0);
    q.weights[n - 1 - r] = 1.0 / ((1.0 - x * x) * deriv * deriv);
  }
  return q;
}

QuadratureSet QuadratureSet::single_point() {
  QuadratureSet q;
  q.g_points = {0.5};
  q.weights = {1.0};
  return q;
}

void LineSpectrum::validate() const {
  if (nu_grid.size() < 2) throw Error("LineSpectrum: need at least 2 samples");
  for (size_t s = 1; s < nu_grid.size(); ++s)
    if (nu_grid[s] <= nu_grid[s - 1])
      throw Error("LineSpectrum: nu_grid must be strictly increasing");
  if (temps.empty() || kappa.size() != temps.size())
    throw Error("LineSpectrum: one kappa row per temperature node");
  for (const auto& row : kappa) {
    if (row.size() != nu_grid.size()) throw Error("LineSpectrum: kappa row size mismatch");
    for (double v : row)
      if (v < 0.0 || !std::isfinite(v))
        throw Error("LineSpectrum: kappa must be finite and non-negative");
  }
}

double planck_intensity(double nu, double temperature) {
  return ermc_host::planck_intensity_checked(nu, temperature);
}

namespace {

double band_blackbody(const NarrowBand& b, double t) {
  return t <= 0.0 ? 0.0 : planck_intensity(b.nu_center, t);
}

void check_band_list(const std::vector<NarrowBand>& bands) {
  if (bands.empty()) throw Error("SpectralModel: no bands");
  for (size_t n = 0; n < bands.size(); ++n) {
    if (bands[n].nu_hi <= bands[n].nu_lo)
      throw Error("SpectralModel: band " + std::to_string(n) +
                  " has non-positive width");
    if (n > 0 && bands[n].nu_lo < bands[n - 1].nu_hi - 1e-9)
      throw Error("SpectralModel: bands overlap at index " + std::to_string(n));
  }
}

}  // namespace

SpectralModel::SpectralModel(std::vector<NarrowBand> bands,
                             QuadratureSet quadrature,
                             std::vector<double> temp_grid,
                             std::vector<double> k_table,
                             std::vector<double> ib_table)
    : bands_(std::move(bands)),
      quadrature_(std::move(quadrature)),
      temp_grid_(std::move(temp_grid)),
      k_table_(std::move(k_table)),
      ib_table_(std::move(ib_table)) {
  check_band_list(bands_);
  if (temp_grid_.empty()) throw Error("SpectralModel: empty temperature grid");
  for (size_t t = 1; t < temp_grid_.size(); ++t)
    if (temp_grid_[t] <= temp_grid_[t - 1])
      throw Error("SpectralModel: temperature grid must be ascending");
  const double wsum = std::accumulate(quadrature_.weights.begin(),
                                      quadrature_.weights.end(), 0.0);
  if (std::abs(wsum - 1.0) > 1e-12)
    throw Error("SpectralModel: quadrature weights must sum to 1");
  if (quadrature_.weights.size() != quadrature_.g_points.size() ||
      k_table_.size() != bands_.size() * quadrature_.count() * temp_grid_.size() ||
      ib_table_.size() != bands_.size() * temp_grid_.size())
    throw Error("SpectralModel: table size mismatch");
  for (double k : k_table_)
    if (k < 0.0 || !std::isfinite(k))
      throw Error("SpectralModel: k_table entries must be non-negative");
  nu_lo_.resize(bands_.size());
  nu_hi_.resize(bands_.size());
  nu_center_.resize(bands_.size());
  for (size_t n = 0; n < bands_.size(); ++n) {
    nu_lo_[n] = bands_[n].nu_lo;
    nu_hi_[n] = bands_[n].nu_hi;
    nu_center_[n] = bands_[n].nu_center;
  }
  kp_table_ = ermc_host::kp_nodes(ermc_host::make_view_unchecked(c_view()));
}

ermc_model_t SpectralModel::c_view() const {
  ermc_model_t m{};
  m.n_bands = n_bands();
  m.n_quad = n_quad();
  m.n_temps = n_temps();
  m.band_nu_lo = nu_lo_.data();
  m.band_nu_hi = nu_hi_.data();
  m.band_nu_center = nu_center_.data();
  m.g_points = quadrature_.g_points.data();
  m.g_weights = quadrature_.weights.data();
  m.temp_grid = temp_grid_.data();
  m.k_table = k_table_.data();
  m.ib_table = ib_table_.data();
  return m;
}

namespace {
ermc_host::TableView view_of(const SpectralModel& m) {
  if (m.n_bands() == 0) throw Error("SpectralModel: no bands");
  return ermc_host::make_view_unchecked(m.c_view());
}
}  // namespace

double SpectralModel::interp_k(int band, int g, double t) const {
  return ermc_host::interp_k(view_of(*this), band, g, t);
}
double SpectralModel::interp_ib(int band, double t) const {
  return ermc_host::interp_ib(view_of(*this), band, t);
}
void SpectralModel::interp_pair(int band, int g, double t, double* k,
                                double* ib) const {
  const ermc_host::TableView v = view_of(*this);
  *k = ermc_host::interp_k(v, band, g, t);
  *ib = ermc_host::interp_ib(v, band, t);
}
double SpectralModel::planck_mean(double t) const {
  return ermc_host::planck_mean(view_of(*this), t);
}

SpectralModel build_k_distribution(const LineSpectrum& spectrum,
                                   const std::vector<NarrowBand>& bands,
                                   const QuadratureSet& quadrature) {
  spectrum.validate();
  check_band_list(bands);
  const std::vector<double>& nu = spectrum.nu_grid;
  const size_t ns = nu.size();
  const int nt = static_cast<int>(spectrum.temps.size());
  const int nq = quadrature.count();
  std::vector<double> k_table(bands.size() * nq * nt);
  std::vector<double> ib_table(bands.size() * nt);
  // Trapezoid share of each spectral sample.
  std::vector<double> share(ns);
  for (size_t s = 0; s < ns; ++s) {
    const double a = s == 0 ? nu[0] : 0.5 * (nu[s - 1] + nu[s]);
    const double b = s + 1 == ns ? nu[ns - 1] : 0.5 * (nu[s] + nu[s + 1]);
    share[s] = b - a;
  }
  std::vector<std::pair<double, double>> kw;
  std::vector<double> gpos;
  for (size_t n = 0; n < bands.size(); ++n) {
    std::vector<size_t> members;
    for (size_t s = 0; s < ns; ++s)
      if (nu[s] >= bands[n].nu_lo && nu[s] < bands[n].nu_hi) members.push_back(s);
    if (members.size() < 2)
      throw Error("build_k_distribution: band [" + std::to_string(bands[n].nu_lo) +
                  ", " + std::to_string(bands[n].nu_hi) +
                  "] cm^-1 has fewer than 2 spectral samples");
    for (int t = 0; t < nt; ++t) {
      // g(k): samples sorted by kappa, cumulative share at sample midpoints.
      kw.clear();
      double wtot = 0.0;
      for (size_t s : members) {
        kw.emplace_back(spectrum.kappa[t][s], share[s]);
        wtot += share[s];
      }
      std::sort(kw.begin(), kw.end());
      gpos.assign(kw.size(), 0.0);
      double cum = 0.0;
      for (size_t s = 0; s < kw.size(); ++s) {
        gpos[s] = (cum + 0.5 * kw[s].second) / wtot;
        cum += kw[s].second;
      }
      for (int g = 0; g < nq; ++g) {
        const double a = quadrature.g_points[g];
        double value;
        if (a <= gpos.front()) {
          value = kw.front().first;
        } else if (a >= gpos.back()) {
          value = kw.back().first;
        } else {
          const size_t hi = std::upper_bound(gpos.begin(), gpos.end(), a) - gpos.begin();
          const size_t lo = hi - 1;
          const double f = (a - gpos[lo]) / (gpos[hi] - gpos[lo]);
          value = kw[lo].first + f * (kw[hi].first - kw[lo].first);
        }
        k_table[(n * nq + g) * nt + t] = value;
      }
      ib_table[n * nt + t] = band_blackbody(bands[n], spectrum.temps[t]);
    }
  }
  return SpectralModel(bands, quadrature, spectrum.temps, std::move(k_table),
                       std::move(ib_table));
}

SpectralModel grey_model(double kappa, const std::vector<NarrowBand>& bands,
                         const std::vector<double>& temp_grid,
                         const QuadratureSet& quadrature) {
  if (kappa < 0.0) throw Error("grey_model: kappa must be non-negative");
  check_band_list(bands);
  const size_t nt = temp_grid.size();
  std::vector<double> k_table(bands.size() * quadrature.count() * nt, kappa);
  std::vector<double> ib_table(bands.size() * nt);
  for (size_t n = 0; n < bands.size(); ++n)
    for (size_t t = 0; t < nt; ++t) ib_table[n * nt + t] = band_blackbody(bands[n], temp_grid[t]);
  return SpectralModel(bands, quadrature, temp_grid, std::move(k_table),
                       std::move(ib_table));
}

SamplingCdfs build_cdfs(const SpectralModel& model, double t_max) {
  const ermc_host::TableView v = view_of(model);
  std::vector<double> band(v.nb), quad(static_cast<size_t>(v.nb) * v.nq);
  ermc_host::build_cdfs(v, t_max, band.data(), quad.data());
  SamplingCdfs c;
  c.t_max = t_max;
  c.band_cdf = std::move(band);
  c.quad_cdf.resize(v.nb);
  for (int n = 0; n < v.nb; ++n)
    c.quad_cdf[n].assign(quad.begin() + static_cast<size_t>(n) * v.nq,
                         quad.begin() + static_cast<size_t>(n + 1) * v.nq);
  return c;
}

std::vector<NarrowBand> make_bands(double nu_lo, double nu_hi, int n) {
  if (n < 1 || nu_hi <= nu_lo) throw Error("make_bands: invalid partition");
  std::vector<NarrowBand> out(n);
  const double w = (nu_hi - nu_lo) / n;
  for (int i = 0; i < n; ++i) {
    NarrowBand& b = out[i];
    b.nu_lo = nu_lo + i * w;
    b.nu_hi = nu_lo + (i + 1) * w;
    b.nu_center = 0.5 * (b.nu_lo + b.nu_hi);
  }
  out.back().nu_hi = nu_hi;
  return out;
}

std::vector<NarrowBand> make_planck_bands(double t_lo, double t_hi, int n) {
  if (t_lo <= 0.0 || t_hi < t_lo) throw Error("make_planck_bands: need 0 < t_lo <= t_hi");
  if (n < 8) throw Error("make_planck_bands: need at least 8 bands");
  // x = c2 nu / T spans [0.05, 35] over [t_lo, t_hi]: geometric partition.
  const double scale = 100.0 * kPlanckC2;
  const double first = 0.05 * t_lo / scale;
  const double last = 35.0 * t_hi / scale;
  const double ratio = std::pow(last / first, 1.0 / n);
  std::vector<NarrowBand> out(n);
  double edge = first;
  for (int i = 0; i < n; ++i) {
    const double next = i + 1 == n ? last : edge * ratio;
    out[i] = {edge, next, std::sqrt(edge * next)};
    edge = next;
  }
  return out;
}

std::vector<double> make_temp_grid(double t_lo, double t_hi, double spacing) {
  if (t_lo < 0.0 || t_hi <= t_lo || spacing <= 0.0)
    throw Error("make_temp_grid: invalid range");
  const int n = static_cast<int>(std::ceil((t_hi - t_lo) / spacing));
  std::vector<double> g;
  g.reserve(n + 1);
  for (int i = 0; i < n; ++i) g.push_back(t_lo + i * spacing);
  g.push_back(t_hi);
  return g;
}

LineSpectrum elsasser_spectrum(const ElsasserParams& p,
                               const std::vector<double>& temps) {
  if (p.nu_hi <= p.nu_lo || p.line_spacing <= 0.0 || p.half_width <= 0.0 ||
      p.resolution <= 0.0)
    throw Error("elsasser_spectrum: invalid parameters");
  for (double t : temps)
    if (t <= 0.0) throw Error("elsasser_spectrum: temperatures must be positive");
  LineSpectrum out;
  out.temps = temps;
  const int ns = static_cast<int>(std::floor((p.nu_hi - p.nu_lo) / p.resolution)) + 1;
  out.nu_grid.resize(ns);
  for (int s = 0; s < ns; ++s) out.nu_grid[s] = p.nu_lo + s * p.resolution;
  // Regular Lorentz comb, five line spacings of margin past each edge.
  std::vector<double> lines;
  for (double c = p.nu_lo - 5.0 * p.line_spacing; c < p.nu_hi + 5.0 * p.line_spacing;
       c += p.line_spacing)
    lines.push_back(c + 0.5 * p.line_spacing);
  out.kappa.assign(temps.size(), std::vector<double>(ns));
  const double gam = p.half_width;
  for (size_t t = 0; t < temps.size(); ++t) {
    const double st = p.strength * std::pow(p.t_ref / temps[t], 1.5);
    std::vector<double>& row = out.kappa[t];
    for (int s = 0; s < ns; ++s) {
      double k = p.continuum;
      for (double c : lines) {
        const double d = out.nu_grid[s] - c;
        k += st / kPi * gam / (d * d + gam * gam);
      }
      row[s] = k;
    }
  }
  return out;
}

// ------------------------------------------------------------------ solver

void SolveConfig::validate() const {
  if (rays_per_cell < 1) throw Error("SolveConfig: rays_per_cell must be >= 1");
  if (!(tolerance > 0.0 && tolerance < 1.0))
    throw Error("SolveConfig: tolerance must be in (0,1)");
  if (n_levels < 1) throw Error("SolveConfig: n_levels must be >= 1");
  if (steps_per_level < 1) throw Error("SolveConfig: steps_per_level must be >= 1");
  if (max_steps < 1) throw Error("SolveConfig: max_steps must be >= 1");
  if (workers < 0) throw Error("SolveConfig: workers must be >= 0");
}

ermc_config_t SolveConfig::c_view() const {
  ermc_config_t c;
  ermc_b200_config_default(&c);
  c.rays_per_cell = rays_per_cell;
  c.n_levels = n_levels;
  c.tolerance = tolerance;
  c.seed = seed;
  c.max_steps = max_steps;
  c.sorting = sorting ? 1 : 0;
  c.steps_per_level = steps_per_level;
  c.coarsen_ratio = coarsen_ratio;
  c.volume_sampling = volume_sampling ? 1 : 0;
  c.specular_walls = specular_walls ? 1 : 0;
  c.workers = workers;
  c.precision = static_cast<int32_t>(precision);
  c.device = device;
  c.n_devices = n_devices;
  return c;
}

namespace {
ermc_grid_t grid_view(const CartesianGrid& g) {
  ermc_grid_t o{};
  o.nx = g.nx;
  o.ny = g.ny;
  o.nz = g.nz;
  o.dx = g.dx;
  o.dy = g.dy;
  o.dz = g.dz;
  for (int a = 0; a < 3; ++a) o.origin[a] = g.origin[a];
  return o;
}

ermc_boundary_t boundary_view(const BoundarySpec& b) {
  ermc_boundary_t o{};
  for (int a = 0; a < 3; ++a) {
    o.kind[a] = b.periodic(a) ? ERMC_AXIS_PERIODIC : ERMC_AXIS_WALL;
    o.lo_temperature[a] = b.lo[a].temperature;
    o.lo_emissivity[a] = b.lo[a].emissivity;
    o.hi_temperature[a] = b.hi[a].temperature;
    o.hi_emissivity[a] = b.hi[a].emissivity;
  }
  return o;
}
}  // namespace

SolutionField solve(const CartesianGrid& grid, const TemperatureField& field,
                    const BoundarySpec& boundary, const SpectralModel& model,
                    const SolveConfig& config) {
  // Validation order of solver.cpp:39-58; the O(N) field checks that need
  // the whole array run on the GPU inside ermc_b200_solve.
  config.validate();
  grid.validate();
  field.grid.validate();
  if (static_cast<std::int64_t>(field.values.size()) != field.grid.cell_count())
    throw Error("TemperatureField: value count does not match grid");
  if (model.n_bands() == 0) throw Error("SpectralModel: no bands");
  if (field.grid.cell_count() != grid.cell_count()) {
    // Mismatched shapes cannot be handed to the device; finish the
    // reference's remaining checks on the host in its order.
    field.validate();
    boundary.validate();
    throw Error("solve: temperature field does not match the grid");
  }
  SolutionField out;
  out.grid = grid;
  out.q_r.assign(grid.cell_count(), 0.0);
  out.std_dev.assign(grid.cell_count(), 0.0);
  out.steps_per_level.assign(config.n_levels, 0);
  ermc_grid_t g = grid_view(grid);
  ermc_boundary_t b = boundary_view(boundary);
  ermc_model_t m = model.c_view();
  ermc_config_t c = config.c_view();
  ermc_solution_t s{out.q_r.data(), out.std_dev.data(), out.steps_per_level.data(), 0, 0.0};
  char err[1024] = {0};
  if (ermc_b200_solve(&g, field.values.data(), &b, &m, &c, &s, err, sizeof(err)) != 0)
    throw Error(err);
  out.total_steps = s.total_steps;
  out.wall_time = s.wall_time;
  return out;
}

namespace {
// The keyed stream of sampling.cpp:13-29 (MurmurHash3 fmix64 chain).
std::uint64_t fmix64(std::uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdULL;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ULL;
  x ^= x >> 33;
  return x;
}
double keyed_uniform(std::uint64_t seed, std::uint64_t cell, std::uint32_t ray,
                     std::uint32_t draw) {
  std::uint64_t h = fmix64(seed + 0x9e3779b97f4a7c15ULL);
  h = fmix64(h ^ cell);
  h = fmix64(h ^ ((static_cast<std::uint64_t>(ray) << 32) | draw));
  return static_cast<double>(h >> 11) * 0x1.0p-53;
}
int cdf_index(const std::vector<double>& cdf, double u) {
  const auto it = std::upper_bound(cdf.begin(), cdf.end(), u);
  const int i = static_cast<int>(it - cdf.begin());
  return std::min(i, static_cast<int>(cdf.size()) - 1);
}
}  // namespace

// ---- the per-ray API (reference sampling.cpp, tracer.cpp) -----------------
double uniform(const RandomKey& key) {
  return keyed_uniform(key.seed, key.cell_id, key.ray_id, key.draw_id);
}

std::pair<int, int> sample_band(double r_n, double r_g, const SamplingCdfs& cdfs) {
  const int n = cdf_index(cdfs.band_cdf, r_n);
  return {n, cdf_index(cdfs.quad_cdf[n], r_g)};
}

namespace {
void check_rc(int rc, const char* err) {
  if (rc != 0) throw Error(err);
}
}  // namespace

Direction sample_direction(double r_theta, double r_phi) {
  double out[5];
  char err[512] = {0};
  check_rc(ermc_b200_sample_direction(1, &r_theta, &r_phi, out, err, sizeof err), err);
  Direction d;
  d.theta = out[0];
  d.phi = out[1];
  d.unit = {out[2], out[3], out[4]};
  return d;
}

double absorptivity(double kappa, double ds) {
  double out = 0.0;
  char err[512] = {0};
  check_rc(ermc_b200_absorptivity(1, &kappa, &ds, &out, err, sizeof err), err);
  return out;
}

RayState init_ray(const CellIndex& cell, std::uint32_t ray_id, std::uint64_t seed,
                  const SpectralModel& model, const SamplingCdfs& cdfs,
                  const GridHierarchy& hierarchy, bool volume_sampling) {
  if (hierarchy.grids.empty()) throw Error("init_ray: empty grid hierarchy");
  const int nb = model.n_bands(), nq = model.n_quad();
  if (static_cast<int>(cdfs.band_cdf.size()) != nb ||
      static_cast<int>(cdfs.quad_cdf.size()) != nb)
    throw Error("init_ray: sampling CDFs do not match the spectral model");
  std::vector<double> quad(static_cast<size_t>(nb) * nq);
  for (int n = 0; n < nb; ++n) {
    if (static_cast<int>(cdfs.quad_cdf[n].size()) != nq)
      throw Error("init_ray: sampling CDFs do not match the spectral model");
    std::copy(cdfs.quad_cdf[n].begin(), cdfs.quad_cdf[n].end(), quad.begin() + n * nq);
  }
  const ermc_grid_t g = grid_view(hierarchy.grids[0]);
  const ermc_model_t m = model.c_view();
  const int32_t c[3] = {cell.i, cell.j, cell.k};
  ermc_ray_state_t st{};
  char err[1024] = {0};
  check_rc(ermc_b200_init_rays(&g, hierarchy.fields[0].data(), &m, cdfs.band_cdf.data(),
                               quad.data(), cdfs.t_max, seed, volume_sampling ? 1 : 0, 1, c,
                               &ray_id, &st, err, sizeof err),
           err);
  RayState r;
  r.pos = {st.pos[0], st.pos[1], st.pos[2]};
  r.dir = {st.dir[0], st.dir[1], st.dir[2]};
  r.cell = CellIndex{st.cell[0], st.cell[1], st.cell[2], st.cell[3]};
  r.transmissivity = st.transmissivity;
  r.band = st.band;
  r.quad = st.quad;
  r.prefactor = st.prefactor;
  r.ib_source = st.ib_source;
  r.reflections = st.reflections;
  r.seed = st.seed;
  r.cell_id = st.cell_id;
  r.ray_id = st.ray_id;
  r.next_draw = st.next_draw;
  return r;
}

MarchResult march(RayState ray, const GridHierarchy& hierarchy, const SpectralModel& model,
                  const BoundarySpec& boundary, double q_emission, const TraceOptions& options) {
  const int nl = hierarchy.n_levels();
  if (nl < 1 || static_cast<int>(hierarchy.fields.size()) != nl)
    throw Error("march: invalid grid hierarchy");
  std::vector<ermc_grid_t> grids(nl);
  std::vector<const double*> fields(nl);
  std::vector<int32_t> caps(nl);
  for (int l = 0; l < nl; ++l) {
    grids[l] = grid_view(hierarchy.grids[l]);
    fields[l] = hierarchy.fields[l].data();
    caps[l] = l < static_cast<int>(hierarchy.step_caps.size()) ? hierarchy.step_caps[l] : -1;
  }
  ermc_ray_state_t st{};
  for (int a = 0; a < 3; ++a) {
    st.pos[a] = ray.pos[a];
    st.dir[a] = ray.dir[a];
  }
  st.cell[0] = ray.cell.i;
  st.cell[1] = ray.cell.j;
  st.cell[2] = ray.cell.k;
  st.cell[3] = ray.cell.level;
  st.transmissivity = ray.transmissivity;
  st.band = ray.band;
  st.quad = ray.quad;
  st.prefactor = ray.prefactor;
  st.ib_source = ray.ib_source;
  st.reflections = ray.reflections;
  st.seed = ray.seed;
  st.cell_id = ray.cell_id;
  st.ray_id = ray.ray_id;
  st.next_draw = ray.next_draw;
  const ermc_model_t m = model.c_view();
  const ermc_boundary_t b = boundary_view(boundary);
  ermc_ray_result_t res{};
  std::vector<std::int64_t> level_steps(nl, 0);
  char err[1024] = {0};
  check_rc(ermc_b200_march_rays(nl, grids.data(), fields.data(), caps.data(), &m, &b,
                                q_emission, options.tolerance, options.max_steps,
                                options.specular_walls ? 1 : 0, 1, &st, &res,
                                level_steps.data(), err, sizeof err),
           err);
  MarchResult out;
  out.q_contribution = res.q_contribution;
  out.steps = res.steps;
  out.steps_per_level = level_steps;
  out.terminated_by = static_cast<Termination>(res.terminated_by);
  out.reflections = res.reflections;
  out.weight_absorbed = res.weight_absorbed;
  out.weight_walls = res.weight_walls;
  out.weight_residual = res.weight_residual;
  return out;
}

std::vector<PlanEntry> presample_and_sort(std::uint64_t cell_id, std::uint32_t n_rays,
                                          std::uint64_t seed, const SamplingCdfs& cdfs,
                                          const SpectralModel& model) {
  std::vector<PlanEntry> plan(n_rays);
  for (std::uint32_t r = 0; r < n_rays; ++r) {
    const int n = cdf_index(cdfs.band_cdf, keyed_uniform(seed, cell_id, r, 2));
    const int g = cdf_index(cdfs.quad_cdf[n], keyed_uniform(seed, cell_id, r, 3));
    plan[r] = PlanEntry{r, n, g, model.interp_k(n, g, cdfs.t_max)};
  }
  std::stable_sort(plan.begin(), plan.end(),
                   [](const PlanEntry& a, const PlanEntry& b) { return a.k_sort < b.k_sort; });
  return plan;
}

// Line-by-line model (reference oracles.cpp:232-264): every spectral sample
// becomes its own band — edges at the midpoints between samples, the outer
// edges mirrored half a spacing out — with a single g point, so the solve
// samples wavenumbers directly. The GPU solve then runs unchanged with
// n_bands = number of samples (8001 for the default Elsasser spectrum).
SpectralModel lbl_model(const LineSpectrum& spectrum, std::size_t memory_cap_bytes) {
  spectrum.validate();
  const std::vector<double>& nu = spectrum.nu_grid;
  const size_t ns = nu.size();
  const size_t nt = spectrum.temps.size();
  const size_t need = ns * nt * 2 * sizeof(double);
  if (need > memory_cap_bytes)
    throw Error("lbl_model: tables would need " + std::to_string(need) +
                " bytes; coarsen the spectrum or raise the cap");
  std::vector<NarrowBand> bands(ns);
  for (size_t s = 0; s < ns; ++s) {
    NarrowBand& b = bands[s];
    b.nu_center = nu[s];
    b.nu_lo = s > 0 ? 0.5 * (nu[s - 1] + nu[s]) : nu[0] - 0.5 * (nu[1] - nu[0]);
    b.nu_hi = s + 1 < ns ? 0.5 * (nu[s] + nu[s + 1])
                         : nu[ns - 1] + 0.5 * (nu[ns - 1] - nu[ns - 2]);
  }
  std::vector<double> k_table(ns * nt), ib_table(ns * nt);
  for (size_t s = 0; s < ns; ++s) {
    double* krow = k_table.data() + s * nt;
    double* irow = ib_table.data() + s * nt;
    for (size_t t = 0; t < nt; ++t) {
      krow[t] = spectrum.kappa[t][s];
      irow[t] = band_blackbody(bands[s], spectrum.temps[t]);
    }
  }
  return SpectralModel(std::move(bands), QuadratureSet::single_point(), spectrum.temps,
                       std::move(k_table), std::move(ib_table));
}

// lbl_reference (reference oracles.cpp:266-274): the line-by-line solve, on
// the GPU like every other solve.
SolutionField lbl_reference(const CartesianGrid& grid, const TemperatureField& field,
                            const BoundarySpec& boundary, const LineSpectrum& spectrum,
                            const SolveConfig& config, std::size_t memory_cap_bytes) {
  const SpectralModel model = lbl_model(spectrum, memory_cap_bytes);
  return solve(grid, field, boundary, model, config);
}

StepCensus step_census(const SolutionField& solution, const CartesianGrid& grid,
                       const TemperatureField& field,
                       const BoundarySpec& boundary,
                       const SpectralModel& model, const SolveConfig& config) {
  StepCensus c;
  c.steps_per_level = solution.steps_per_level;
  c.total_steps = solution.total_steps;
  if (config.n_levels == 1) return c;
  SolveConfig single = config;
  single.n_levels = 1;
  const SolutionField base = solve(grid, field, boundary, model, single);
  c.saved_ratio = static_cast<double>(base.total_steps) / solution.total_steps;
  return c;
}

}  // namespace ermc
