// ref_shim.cpp — TEST INFRASTRUCTURE ONLY (the checker, never the product).
//
// A thin C shim over the UNMODIFIED reference library, compiled from the
// sources under /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libermc_ref.so. It takes the same plain-C descriptors as the
// product boundary (include/ermc_b200.h) so tests and bench.py's CPU arm can
// drive the reference and the GPU path with identical inputs.
//
// Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl
// reference) may load this library.

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "ermc/constants.hpp"
#include "ermc/errors.hpp"
#include "ermc/geometry.hpp"
#include "ermc/sampling.hpp"
#include "ermc/solver.hpp"
#include "ermc/spectral.hpp"
#include "ermc/tracer.hpp"
#include "ermc_b200.h"

namespace {

void put_err(char* buf, size_t len, const char* msg) {
  if (!buf || len == 0) return;
  std::snprintf(buf, len, "%s", msg);
}

ermc::CartesianGrid to_grid(const ermc_grid_t* g) {
  ermc::CartesianGrid out;
  out.nx = g->nx;
  out.ny = g->ny;
  out.nz = g->nz;
  out.dx = g->dx;
  out.dy = g->dy;
  out.dz = g->dz;
  out.origin = {g->origin[0], g->origin[1], g->origin[2]};
  return out;
}

ermc::BoundarySpec to_boundary(const ermc_boundary_t* b) {
  ermc::BoundarySpec out;
  for (int a = 0; a < 3; ++a) {
    out.kind[a] = b->kind[a] == ERMC_AXIS_PERIODIC ? ermc::AxisKind::periodic
                                                   : ermc::AxisKind::wall;
    out.lo[a] = {b->lo_temperature[a], b->lo_emissivity[a]};
    out.hi[a] = {b->hi_temperature[a], b->hi_emissivity[a]};
  }
  return out;
}

ermc::SpectralModel to_model(const ermc_model_t* m) {
  std::vector<ermc::NarrowBand> bands(m->n_bands);
  for (int n = 0; n < m->n_bands; ++n)
    bands[n] = {m->band_nu_lo[n], m->band_nu_hi[n], m->band_nu_center[n]};
  ermc::QuadratureSet q;
  q.g_points.assign(m->g_points, m->g_points + m->n_quad);
  q.weights.assign(m->g_weights, m->g_weights + m->n_quad);
  std::vector<double> temps(m->temp_grid, m->temp_grid + m->n_temps);
  size_t nk = static_cast<size_t>(m->n_bands) * m->n_quad * m->n_temps;
  std::vector<double> k(m->k_table, m->k_table + nk);
  std::vector<double> ib(m->ib_table,
                         m->ib_table + static_cast<size_t>(m->n_bands) * m->n_temps);
  return ermc::SpectralModel(std::move(bands), std::move(q), std::move(temps),
                             std::move(k), std::move(ib));
}

ermc::SolveConfig to_config(const ermc_config_t* c) {
  ermc::SolveConfig out;
  out.rays_per_cell = c->rays_per_cell;
  out.tolerance = c->tolerance;
  out.seed = c->seed;
  out.sorting = c->sorting != 0;
  out.n_levels = c->n_levels;
  out.steps_per_level = c->steps_per_level;
  out.coarsen_ratio = c->coarsen_ratio;
  out.max_steps = c->max_steps;
  out.volume_sampling = c->volume_sampling != 0;
  out.specular_walls = c->specular_walls != 0;
  out.workers = c->workers;
  return out;
}

ermc::TemperatureField to_field(const ermc::CartesianGrid& g, const double* t) {
  ermc::TemperatureField f;
  f.grid = g;
  f.values.assign(t, t + g.cell_count());
  return f;
}

}  // namespace

extern "C" {

int ref_solve(const ermc_grid_t* grid, const double* temperature,
              const ermc_boundary_t* boundary, const ermc_model_t* model,
              const ermc_config_t* config, ermc_solution_t* out, char* errbuf,
              size_t errlen) {
  try {
    ermc::CartesianGrid g = to_grid(grid);
    ermc::SolutionField s =
        ermc::solve(g, to_field(g, temperature), to_boundary(boundary),
                    to_model(model), to_config(config));
    std::copy(s.q_r.begin(), s.q_r.end(), out->q_r);
    std::copy(s.std_dev.begin(), s.std_dev.end(), out->std_dev);
    std::copy(s.steps_per_level.begin(), s.steps_per_level.end(),
              out->steps_per_level);
    out->total_steps = s.total_steps;
    out->wall_time = s.wall_time;
    return 0;
  } catch (const std::exception& e) {
    put_err(errbuf, errlen, e.what());
    return 1;
  }
}

// Cell-subset replay of solver.cpp:118-156 through the public
// build_cdfs / planck_mean / build_hierarchy / init_ray / march API:
// bitwise identical to solve() for the selected cells.
// steps_per_level receives the per-level sum over the selected cells.
// cell_steps (nullable) receives each selected cell's march steps summed
// over its rays and levels.
int ref_solve_cells_ex(const ermc_grid_t* grid, const double* temperature,
                       const ermc_boundary_t* boundary, const ermc_model_t* model,
                       const ermc_config_t* config, int64_t n_sel,
                       const int64_t* cells, double* q_r, double* std_dev,
                       int64_t* steps_per_level, int64_t* cell_steps,
                       int32_t n_threads, double* wall_time, char* errbuf,
                       size_t errlen) {
  try {
    auto t0 = std::chrono::steady_clock::now();
    ermc::CartesianGrid g = to_grid(grid);
    ermc::TemperatureField field = to_field(g, temperature);
    ermc::BoundarySpec b = to_boundary(boundary);
    ermc::SpectralModel m = to_model(model);
    ermc::SolveConfig cfg = to_config(config);
    double t_max = field.max_value();
    for (int a = 0; a < 3; ++a) {
      if (b.periodic(a)) continue;
      t_max = std::max({t_max, b.lo[a].temperature, b.hi[a].temperature});
    }
    ermc::SamplingCdfs cdfs = ermc::build_cdfs(m, t_max);
    double kp = m.planck_mean(t_max);
    int n_rays = cfg.rays_per_cell;
    double qe = 4.0 * kp * ermc::kSigma * t_max * t_max * t_max * t_max / n_rays;
    ermc::GridHierarchy h = ermc::build_hierarchy(
        g, field.values, cfg.n_levels, cfg.coarsen_ratio, cfg.steps_per_level);
    ermc::TraceOptions opt{cfg.tolerance, cfg.max_steps, cfg.specular_walls};
    int nt = std::max(1, n_threads);
    if (cell_steps) std::fill(cell_steps, cell_steps + n_sel, int64_t{0});
    std::vector<std::vector<int64_t>> steps(nt, std::vector<int64_t>(cfg.n_levels, 0));
    std::vector<std::string> errors(nt);
    auto work = [&](int w) {
      try {
        std::vector<double> per_ray(n_rays);
        for (int64_t s = w; s < n_sel; s += nt) {
          int64_t c = cells[s];
          ermc::CellIndex cell;
          cell.i = static_cast<int>(c / (static_cast<int64_t>(g.ny) * g.nz));
          cell.j = static_cast<int>((c / g.nz) % g.ny);
          cell.k = static_cast<int>(c % g.nz);
          for (int r = 0; r < n_rays; ++r) {
            ermc::RayState ray = ermc::init_ray(cell, r, cfg.seed, m, cdfs, h,
                                                cfg.volume_sampling);
            ermc::MarchResult res = ermc::march(ray, h, m, b, qe, opt);
            per_ray[r] = res.q_contribution;
            for (int l = 0; l < cfg.n_levels; ++l)
              steps[w][l] += res.steps_per_level[l];
            if (cell_steps) cell_steps[s] += res.steps;
          }
          double sum = 0.0, mean = 0.0, m2 = 0.0;
          for (int r = 0; r < n_rays; ++r) {
            double x = per_ray[r];
            sum += x;
            double delta = x - mean;
            mean += delta / (r + 1);
            m2 += delta * (x - mean);
          }
          q_r[s] = sum;
          std_dev[s] = n_rays > 1 ? std::sqrt(m2 * n_rays / (n_rays - 1.0)) : 0.0;
        }
      } catch (const std::exception& e) {
        errors[w] = e.what();
      }
    };
    // wall_time covers the per-cell trace loop only (threads start -> join),
    // not the O(N) setup copies above, so small samples time the march.
    auto t_trace = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int w = 0; w < nt; ++w) pool.emplace_back(work, w);
    for (auto& t : pool) t.join();
    t0 = t_trace;
    for (auto& e : errors)
      if (!e.empty()) throw ermc::Error(e);
    for (int l = 0; l < cfg.n_levels; ++l) {
      steps_per_level[l] = 0;
      for (int w = 0; w < nt; ++w) steps_per_level[l] += steps[w][l];
    }
    if (wall_time)
      *wall_time = std::chrono::duration<double>(
                       std::chrono::steady_clock::now() - t0).count();
    return 0;
  } catch (const std::exception& e) {
    put_err(errbuf, errlen, e.what());
    return 1;
  }
}

int ref_solve_cells(const ermc_grid_t* grid, const double* temperature,
                    const ermc_boundary_t* boundary, const ermc_model_t* model,
                    const ermc_config_t* config, int64_t n_sel,
                    const int64_t* cells, double* q_r, double* std_dev,
                    int64_t* steps_per_level, int32_t n_threads,
                    double* wall_time, char* errbuf, size_t errlen) {
  return ref_solve_cells_ex(grid, temperature, boundary, model, config, n_sel,
                            cells, q_r, std_dev, steps_per_level, nullptr,
                            n_threads, wall_time, errbuf, errlen);
}

int ref_trace_rays(const ermc_grid_t* grid, const double* temperature,
                   const ermc_boundary_t* boundary, const ermc_model_t* model,
                   const ermc_config_t* config, double t_max, double q_emission,
                   int64_t n, const int64_t* cell_ids, const uint32_t* ray_ids,
                   const double* dir_override, ermc_ray_result_t* out,
                   int64_t* level_steps, char* errbuf, size_t errlen) {
  try {
    ermc::CartesianGrid g = to_grid(grid);
    ermc::TemperatureField field = to_field(g, temperature);
    ermc::BoundarySpec b = to_boundary(boundary);
    ermc::SpectralModel m = to_model(model);
    ermc::SolveConfig cfg = to_config(config);
    ermc::SamplingCdfs cdfs = ermc::build_cdfs(m, t_max);
    ermc::GridHierarchy h = ermc::build_hierarchy(
        g, field.values, cfg.n_levels, cfg.coarsen_ratio, cfg.steps_per_level);
    ermc::TraceOptions opt{cfg.tolerance, cfg.max_steps, cfg.specular_walls};
    for (int64_t s = 0; s < n; ++s) {
      int64_t c = cell_ids[s];
      ermc::CellIndex cell;
      cell.i = static_cast<int>(c / (static_cast<int64_t>(g.ny) * g.nz));
      cell.j = static_cast<int>((c / g.nz) % g.ny);
      cell.k = static_cast<int>(c % g.nz);
      ermc::RayState ray = ermc::init_ray(cell, ray_ids[s], cfg.seed, m, cdfs,
                                          h, cfg.volume_sampling);
      if (dir_override)
        ray.dir = {dir_override[3 * s], dir_override[3 * s + 1],
                   dir_override[3 * s + 2]};
      ermc::MarchResult r = ermc::march(ray, h, m, b, q_emission, opt);
      ermc_ray_result_t& o = out[s];
      std::memset(&o, 0, sizeof(o));
      o.q_contribution = r.q_contribution;
      o.weight_absorbed = r.weight_absorbed;
      o.weight_walls = r.weight_walls;
      o.weight_residual = r.weight_residual;
      for (int a = 0; a < 3; ++a) o.dir[a] = ray.dir[a];
      o.prefactor = ray.prefactor;
      o.ib_source = ray.ib_source;
      o.steps = r.steps;
      o.terminated_by = static_cast<int32_t>(r.terminated_by);
      o.reflections = r.reflections;
      o.band = ray.band;
      o.quad = ray.quad;
      o.next_draw = ray.next_draw;
      if (level_steps)
        for (int l = 0; l < cfg.n_levels; ++l)
          level_steps[s * cfg.n_levels + l] = r.steps_per_level[l];
    }
    return 0;
  } catch (const std::exception& e) {
    put_err(errbuf, errlen, e.what());
    return 1;
  }
}

int ref_build_cdfs(const ermc_model_t* model, double t_max, double* band_cdf,
                   double* quad_cdf, char* errbuf, size_t errlen) {
  try {
    ermc::SpectralModel m = to_model(model);
    ermc::SamplingCdfs c = ermc::build_cdfs(m, t_max);
    for (int n = 0; n < m.n_bands(); ++n) {
      band_cdf[n] = c.band_cdf[n];
      for (int q = 0; q < m.n_quad(); ++q)
        quad_cdf[n * m.n_quad() + q] = c.quad_cdf[n][q];
    }
    return 0;
  } catch (const std::exception& e) {
    put_err(errbuf, errlen, e.what());
    return 1;
  }
}

int ref_planck_mean(const ermc_model_t* model, double t, double* out,
                    char* errbuf, size_t errlen) {
  try {
    *out = to_model(model).planck_mean(t);
    return 0;
  } catch (const std::exception& e) {
    put_err(errbuf, errlen, e.what());
    return 1;
  }
}

int ref_interp(const ermc_model_t* model, int band, int g, double t,
               double* k_out, double* ib_out, char* errbuf, size_t errlen) {
  try {
    ermc::SpectralModel m = to_model(model);
    m.interp_pair(band, g, t, k_out, ib_out);
    return 0;
  } catch (const std::exception& e) {
    put_err(errbuf, errlen, e.what());
    return 1;
  }
}

double ref_uniform(uint64_t seed, uint64_t cell, uint32_t ray, uint32_t draw) {
  return ermc::uniform({seed, cell, ray, draw});
}

// Level fields of build_hierarchy (geometry.cpp:84-110), concatenated.
int ref_build_hierarchy(const ermc_grid_t* grid, const double* temperature,
                        int n_levels, int ratio, ermc_grid_t* grids_out,
                        double* fields_out, int64_t cap, char* errbuf,
                        size_t errlen) {
  try {
    ermc::CartesianGrid g = to_grid(grid);
    std::vector<double> f(temperature, temperature + g.cell_count());
    ermc::GridHierarchy h = ermc::build_hierarchy(g, f, n_levels, ratio, 5);
    int64_t off = 0;
    for (int l = 0; l < h.n_levels(); ++l) {
      const auto& lg = h.grids[l];
      grids_out[l] = {lg.nx, lg.ny, lg.nz, 0, lg.dx, lg.dy, lg.dz,
                      {lg.origin[0], lg.origin[1], lg.origin[2]}};
      if (off + static_cast<int64_t>(h.fields[l].size()) > cap)
        throw ermc::Error("ref_build_hierarchy: output too small");
      std::copy(h.fields[l].begin(), h.fields[l].end(), fields_out + off);
      off += h.fields[l].size();
    }
    return 0;
  } catch (const std::exception& e) {
    put_err(errbuf, errlen, e.what());
    return 1;
  }
}

}  // extern "C"
