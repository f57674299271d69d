// ermc_b200.hpp — C++ host API of the B200 ERMC solver, source-compatible
// with the reference's public headers for the solve path (namespace ermc):
//   proj/include/ermc/{constants,errors,geometry,spectral,solver,io}.hpp
// Client code written against the reference's ermc::solve compiles against
// this header unchanged; the solve itself runs on the GPU through the C-ABI
// in ermc_b200.h (no CPU fallback exists).
//
// Not provided (out of the hot-path scope): the per-ray
// sampling/tracer API (init_ray, march — they exist only inside the trace
// kernel; tests drive them through ermc_b200_trace_rays), the verification
// cases and analytic oracles, and the CLI.
#pragma once

#include <array>
#include <cstddef>
#include <cstdint>
#include <iosfwd>
#include <limits>
#include <map>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "ermc_b200.h"

namespace ermc {

// ---- constants.hpp / errors.hpp -------------------------------------------
inline constexpr double kSigma = 5.670374419e-8;              // W m^-2 K^-4
inline constexpr double kPlanckC1 = 1.1910429723971884e-16;   // 2hc^2
inline constexpr double kPlanckC2 = 1.4387768775039337e-2;    // hc/kB
inline constexpr double kPi = 3.14159265358979323846;

struct Error : std::runtime_error {
  explicit Error(const std::string& what) : std::runtime_error(what) {}
};

// ---- geometry.hpp ----------------------------------------------------------
using Vec3 = std::array<double, 3>;

struct CartesianGrid {
  int nx = 1, ny = 1, nz = 1;
  double dx = 1.0, dy = 1.0, dz = 1.0;
  Vec3 origin = {0.0, 0.0, 0.0};

  int count(int axis) const { return axis == 0 ? nx : axis == 1 ? ny : nz; }
  double spacing(int axis) const { return axis == 0 ? dx : axis == 1 ? dy : dz; }
  double extent(int axis) const { return count(axis) * spacing(axis); }
  std::int64_t cell_count() const {
    return static_cast<std::int64_t>(nx) * ny * nz;
  }
  std::int64_t linear(int i, int j, int k) const {  // k-fastest
    return (static_cast<std::int64_t>(i) * ny + j) * nz + k;
  }
  Vec3 cell_center(int i, int j, int k) const {
    return {origin[0] + (i + 0.5) * dx, origin[1] + (j + 0.5) * dy,
            origin[2] + (k + 0.5) * dz};
  }
  double cell_volume() const { return dx * dy * dz; }
  double min_spacing() const;
  void validate() const;
};

enum class AxisKind { periodic, wall };

struct Wall {
  double temperature = 0.0;  // K
  double emissivity = 1.0;   // [0,1]
};

struct BoundarySpec {
  std::array<AxisKind, 3> kind = {AxisKind::wall, AxisKind::wall,
                                  AxisKind::wall};
  std::array<Wall, 3> lo;
  std::array<Wall, 3> hi;
  void validate() const;
  bool periodic(int axis) const { return kind[axis] == AxisKind::periodic; }
};

struct TemperatureField {
  CartesianGrid grid;
  std::vector<double> values;  // k-fastest
  double at(int i, int j, int k) const { return values[grid.linear(i, j, k)]; }
  double max_value() const;
  double min_value() const;
  void validate() const;
};

struct CellIndex {
  int i = 0, j = 0, k = 0;
  int level = 0;
};

struct GridHierarchy {
  std::vector<CartesianGrid> grids;
  std::vector<std::vector<double>> fields;
  std::vector<int> step_caps;
  int n_levels() const { return static_cast<int>(grids.size()); }
  double temperature(const CellIndex& c) const {
    return fields[c.level][grids[c.level].linear(c.i, c.j, c.k)];
  }
};

// Host restatements for API compatibility; the solve builds its levels on
// the GPU (kernel K3, bitwise the same values).
GridHierarchy build_hierarchy(const CartesianGrid& grid,
                              const std::vector<double>& field, int n_levels,
                              int ratio, int steps_per_level);
TemperatureField restrict_field(const TemperatureField& fine, int ratio);
std::array<int, 3> locate(const CartesianGrid& grid, const Vec3& point);
std::array<int, 3> locate(const CartesianGrid& grid, const Vec3& point,
                          const Vec3& dir);

inline constexpr double kInf = std::numeric_limits<double>::infinity();

// face_distances (reference geometry.hpp:100-109): distance to the next cell
// face along each axis, the minimum (clamped at 0) and its axis, ties x < y < z
// — the first step of Dda::setup / march's step selection (tracer.cpp:103-113).
struct FaceCrossing {
  std::array<double, 3> df;
  double ds = 0.0;
  int axis = 0;
};
FaceCrossing face_distances(const CartesianGrid& grid, const Vec3& pos, const Vec3& dir,
                            int i, int j, int k);
inline double geom_eps(const CartesianGrid& grid) {
  return 1e-12 * grid.min_spacing();
}

// ---- spectral.hpp ----------------------------------------------------------
struct NarrowBand {
  double nu_lo = 0.0;
  double nu_hi = 0.0;
  double nu_center = 0.0;
  double delta_nu() const { return nu_hi - nu_lo; }
};

struct QuadratureSet {
  std::vector<double> g_points;
  std::vector<double> weights;
  int count() const { return static_cast<int>(g_points.size()); }
  static QuadratureSet gauss_legendre(int n);
  static QuadratureSet single_point();
};

struct LineSpectrum {
  std::vector<double> nu_grid;
  std::vector<double> temps;
  std::vector<std::vector<double>> kappa;  // [t][s]
  void validate() const;
};

struct SamplingCdfs {
  std::vector<double> band_cdf;
  std::vector<std::vector<double>> quad_cdf;
  double t_max = 0.0;
};

class SpectralModel {
 public:
  SpectralModel() = default;
  SpectralModel(std::vector<NarrowBand> bands, QuadratureSet quadrature,
                std::vector<double> temp_grid, std::vector<double> k_table,
                std::vector<double> ib_table);

  int n_bands() const { return static_cast<int>(bands_.size()); }
  int n_quad() const { return quadrature_.count(); }
  int n_temps() const { return static_cast<int>(temp_grid_.size()); }
  const std::vector<NarrowBand>& bands() const { return bands_; }
  const QuadratureSet& quadrature() const { return quadrature_; }
  const std::vector<double>& temp_grid() const { return temp_grid_; }
  const std::vector<double>& k_table() const { return k_table_; }
  const std::vector<double>& ib_table() const { return ib_table_; }
  const std::vector<double>& kp_table() const { return kp_table_; }
  double t_min() const { return temp_grid_.front(); }
  double t_max_table() const { return temp_grid_.back(); }

  double interp_k(int band, int g, double temperature) const;
  double interp_ib(int band, double temperature) const;
  void interp_pair(int band, int g, double temperature, double* k,
                   double* ib) const;
  double planck_mean(double temperature) const;

  double k_at_node(int band, int g, int t) const {
    return k_table_[(static_cast<size_t>(band) * n_quad() + g) * n_temps() + t];
  }
  double ib_at_node(int band, int t) const {
    return ib_table_[static_cast<size_t>(band) * n_temps() + t];
  }

  // Borrowed C descriptor of the tables (valid while *this lives).
  ermc_model_t c_view() const;

 private:
  std::vector<NarrowBand> bands_;
  QuadratureSet quadrature_;
  std::vector<double> temp_grid_;
  std::vector<double> k_table_;   // [band][g][T]
  std::vector<double> ib_table_;  // [band][T]
  std::vector<double> kp_table_;  // [T]
  // Column views for c_view().
  std::vector<double> nu_lo_, nu_hi_, nu_center_;
};

double planck_intensity(double nu, double temperature);
SpectralModel build_k_distribution(const LineSpectrum& spectrum,
                                   const std::vector<NarrowBand>& bands,
                                   const QuadratureSet& quadrature);
SpectralModel grey_model(double kappa, const std::vector<NarrowBand>& bands,
                         const std::vector<double>& temp_grid,
                         const QuadratureSet& quadrature = QuadratureSet::single_point());
SamplingCdfs build_cdfs(const SpectralModel& model, double t_max);
std::vector<NarrowBand> make_bands(double nu_lo, double nu_hi, int n);
std::vector<NarrowBand> make_planck_bands(double t_lo, double t_hi, int n);
std::vector<double> make_temp_grid(double t_lo, double t_hi, double spacing);

struct ElsasserParams {
  double nu_lo = 200.0;
  double nu_hi = 2200.0;
  double line_spacing = 20.0;
  double strength = 30.0;
  double half_width = 1.0;
  double continuum = 0.01;
  double t_ref = 1000.0;
  double resolution = 0.25;
};
LineSpectrum elsasser_spectrum(const ElsasserParams& params,
                               const std::vector<double>& temps);

// ---- solver.hpp ------------------------------------------------------------
enum class Precision { fp64 = ERMC_PRECISION_FP64, fp32 = ERMC_PRECISION_FP32 };

struct SolveConfig {
  int rays_per_cell = 2000;
  double tolerance = 1e-4;
  std::uint64_t seed = 0;
  bool sorting = false;
  int n_levels = 1;
  int steps_per_level = 5;
  int coarsen_ratio = 2;
  std::int64_t max_steps = 100000;
  bool volume_sampling = false;
  bool specular_walls = false;
  int workers = 0;  // accepted for compatibility; the GPU ignores it
  // B200 extensions (defaults keep reference semantics):
  Precision precision = Precision::fp64;
  int device = -1;  // CUDA ordinal, -1 = current device
  int n_devices = 1;  // GPUs one solve spreads over (ermc_config_t::n_devices)

  void validate() const;
  ermc_config_t c_view() const;
};

struct SolutionField {
  CartesianGrid grid;
  std::vector<double> q_r;
  std::vector<double> std_dev;
  std::vector<std::int64_t> steps_per_level;
  std::int64_t total_steps = 0;
  double wall_time = 0.0;
};

// ---- sampling.hpp / tracer.hpp: the per-ray API --------------------------
// The reference's per-ray functions (sampling.hpp:13-58, tracer.hpp:12-42).
// init_ray, march, sample_direction and absorptivity run the trace kernels'
// device code on the GPU, one ray per call (ermc_b200_init_rays,
// _march_rays, _sample_direction, _absorptivity); uniform and sample_band
// are the integer hash and CDF search the GPU solve and presample_and_sort
// share (pure functions, bitwise the device's).
struct RandomKey {
  std::uint64_t seed = 0;
  std::uint64_t cell_id = 0;
  std::uint32_t ray_id = 0;
  std::uint32_t draw_id = 0;
};
double uniform(const RandomKey& key);

struct Direction {
  double theta = 0.0;
  double phi = 0.0;
  Vec3 unit = {0.0, 0.0, 1.0};
};
Direction sample_direction(double r_theta, double r_phi);
std::pair<int, int> sample_band(double r_n, double r_g, const SamplingCdfs& cdfs);

struct RayState {
  Vec3 pos = {0.0, 0.0, 0.0};
  Vec3 dir = {0.0, 0.0, 1.0};
  CellIndex cell;
  double transmissivity = 1.0;
  int band = 0;
  int quad = 0;
  double prefactor = 1.0;
  double ib_source = 0.0;
  int reflections = 0;
  std::uint64_t seed = 0;
  std::uint64_t cell_id = 0;
  std::uint32_t ray_id = 0;
  std::uint32_t next_draw = 0;
};
RayState init_ray(const CellIndex& cell, std::uint32_t ray_id, std::uint64_t seed,
                  const SpectralModel& model, const SamplingCdfs& cdfs,
                  const GridHierarchy& hierarchy, bool volume_sampling = false);

enum class Termination { tolerance, wall_absorbed, step_cap };

struct MarchResult {
  double q_contribution = 0.0;
  std::int64_t steps = 0;
  std::vector<std::int64_t> steps_per_level;
  Termination terminated_by = Termination::tolerance;
  int reflections = 0;
  double weight_absorbed = 0.0;
  double weight_walls = 0.0;
  double weight_residual = 0.0;
};

struct TraceOptions {
  double tolerance = 1e-4;
  std::int64_t max_steps = 100000;
  bool specular_walls = false;
};

MarchResult march(RayState ray, const GridHierarchy& hierarchy, const SpectralModel& model,
                  const BoundarySpec& boundary, double q_emission, const TraceOptions& options);
double absorptivity(double kappa, double ds);

// presample_and_sort (reference solver.hpp:39-50, solver.cpp:62-80): the
// (band, g) of every ray of a cell from its keyed draws 2 and 3, ordered by
// k(n, g, T_max) ascending (stable). Host utility; the GPU solve applies the
// same order as its dispatch schedule (dispatch.cu), which never changes a
// result.
struct PlanEntry {
  std::uint32_t ray_id = 0;
  int band = 0;
  int quad = 0;
  double k_sort = 0.0;
};
std::vector<PlanEntry> presample_and_sort(std::uint64_t cell_id, std::uint32_t n_rays,
                                          std::uint64_t seed, const SamplingCdfs& cdfs,
                                          const SpectralModel& model);

// Runs the whole solve on the GPU (ermc_b200_solve). Throws ermc::Error
// with the reference's messages.
SolutionField solve(const CartesianGrid& grid, const TemperatureField& field,
                    const BoundarySpec& boundary, const SpectralModel& model,
                    const SolveConfig& config);

struct StepCensus {
  std::vector<std::int64_t> steps_per_level;
  std::int64_t total_steps = 0;
  double saved_ratio = 1.0;
};
StepCensus step_census(const SolutionField& solution, const CartesianGrid& grid,
                       const TemperatureField& field,
                       const BoundarySpec& boundary,
                       const SpectralModel& model, const SolveConfig& config);

// ---- oracles.hpp (the line-by-line path only) -------------------------------
// lbl_model / lbl_reference (reference oracles.hpp:50-59): one band per
// spectral sample, one g point; lbl_reference solves it on the GPU.
SpectralModel lbl_model(const LineSpectrum& spectrum,
                        std::size_t memory_cap_bytes = std::size_t(2) << 30);
SolutionField lbl_reference(const CartesianGrid& grid, const TemperatureField& field,
                            const BoundarySpec& boundary, const LineSpectrum& spectrum,
                            const SolveConfig& config,
                            std::size_t memory_cap_bytes = std::size_t(2) << 30);

// ---- io.hpp ----------------------------------------------------------------
void write_ktab(const std::string& path, const SpectralModel& model);
SpectralModel read_ktab(const std::string& path);
void write_tfld(const std::string& path, const TemperatureField& field);
TemperatureField read_tfld(const std::string& path);
void write_qrf(const std::string& path, const SolutionField& solution);
SolutionField read_qrf(const std::string& path);

class Config {
 public:
  static Config parse_file(const std::string& path);
  static Config parse(std::istream& in, const std::string& name);
  bool has(const std::string& key) const;
  std::string get(const std::string& key) const;
  std::string get_or(const std::string& key, const std::string& fallback) const;
  double get_double(const std::string& key, double fallback) const;
  std::int64_t get_int(const std::string& key, std::int64_t fallback) const;
  bool get_bool(const std::string& key, bool fallback) const;
  void set(const std::string& key, const std::string& value);
  const std::map<std::string, std::string>& entries() const { return entries_; }

 private:
  std::map<std::string, std::string> entries_;
};

struct LineList {
  std::vector<double> nu_center;
  std::vector<double> strength;
  std::vector<double> half_width;
  double t_ref = 1000.0;
  double strength_exponent = 1.5;
};
LineList read_line_list(const std::string& path);
LineSpectrum evaluate_line_list(const LineList& lines, double resolution,
                                double continuum,
                                const std::vector<double>& temps);

std::string file_hash(const std::string& path);

}  // namespace ermc
