/*
 * ermc_b200.h — C-ABI drop-in boundary for the ERMC per-cell solve on B200.
 *
 * The reference exposes the hot path as one C++ free function,
 *   ermc::SolutionField ermc::solve(const CartesianGrid&, const TemperatureField&,
 *                                   const BoundarySpec&, const SpectralModel&,
 *                                   const SolveConfig&)
 * (reference proj/include/ermc/solver.hpp:55-57, proj/src/solver.cpp:82-180),
 * bound to Python as _ermc.solve (proj/python/bindings.cpp:145-147).
 * This header restates those inputs as plain C descriptors (no C++ or torch
 * types) so any FFI (ctypes, cgo, JNI, N-API) can bind it.
 *
 * Error convention: every entry point returns 0 on success and non-zero on
 * failure, with a NUL-terminated message in errbuf. The message text is the
 * one the reference puts into ermc::Error (proj/include/ermc/errors.hpp:8-10),
 * so a host wrapper can rethrow it verbatim.
 *
 * Layouts are the reference's: temperature k-fastest (geometry.hpp:25-27),
 * k_table [band][g][T] and ib_table [band][T] (spectral.hpp:81-86).
 */
#ifndef ERMC_B200_H
#define ERMC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ERMC_B200_ABI_VERSION 2

/* CartesianGrid (reference geometry.hpp:13-36). */
typedef struct ermc_grid {
  int32_t nx, ny, nz;
  int32_t reserved0;
  double dx, dy, dz;
  double origin[3];
} ermc_grid_t;

/* AxisKind (reference geometry.hpp:38): periodic = 0, wall = 1. */
enum { ERMC_AXIS_PERIODIC = 0, ERMC_AXIS_WALL = 1 };

/* BoundarySpec + Wall (reference geometry.hpp:40-54). */
typedef struct ermc_boundary {
  int32_t kind[3];
  int32_t reserved0;
  double lo_temperature[3];
  double lo_emissivity[3];
  double hi_temperature[3];
  double hi_emissivity[3];
} ermc_boundary_t;

/* SpectralModel tables (reference spectral.hpp:55-110). Borrowed pointers. */
typedef struct ermc_model {
  int32_t n_bands, n_quad, n_temps;
  int32_t reserved0;
  const double* band_nu_lo;     /* [n_bands] */
  const double* band_nu_hi;     /* [n_bands] */
  const double* band_nu_center; /* [n_bands] */
  const double* g_points;       /* [n_quad] */
  const double* g_weights;      /* [n_quad] */
  const double* temp_grid;      /* [n_temps], ascending */
  const double* k_table;        /* [n_bands][n_quad][n_temps] */
  const double* ib_table;       /* [n_bands][n_temps] */
} ermc_model_t;

/* Arithmetic of the trace kernel. */
enum {
  ERMC_PRECISION_FP64 = 0, /* reference arithmetic, per-cell parity */
  ERMC_PRECISION_FP32 = 1  /* fp32 ray state, statistical (3 sigma) parity */
};

/* SolveConfig (reference solver.hpp:12-26) plus device fields. */
typedef struct ermc_config {
  int32_t rays_per_cell;
  int32_t n_levels;
  double tolerance;
  uint64_t seed;
  int64_t max_steps;
  int32_t sorting;
  int32_t steps_per_level;
  int32_t coarsen_ratio;
  int32_t volume_sampling;
  int32_t specular_walls;
  int32_t workers;   /* accepted and validated (>= 0); the GPU ignores it */
  int32_t precision; /* ERMC_PRECISION_* */
  int32_t device;    /* CUDA ordinal, -1 = current */
  /* One-shot solves (ermc_b200_solve / _solve_range) split their cell range
   * into n_devices contiguous parts solved concurrently, part p on device
   * (device + p) mod (visible devices), each with a replicated T field —
   * the GPU form of the reference's worker chunks (solver.cpp:159-170).
   * Results are byte-identical for any n_devices. 0 or 1 = one device.
   * Sessions always use one device. */
  int32_t n_devices;
  int32_t reserved0;
} ermc_config_t;

/* Fills the reference SolveConfig defaults (solver.hpp:12-26). */
void ermc_b200_config_default(ermc_config_t* cfg);

/* SolutionField (reference solver.hpp:28-35). Caller-owned host buffers:
 * q_r and std_dev hold the solved cell range, steps_per_level n_levels. */
typedef struct ermc_solution {
  double* q_r;
  double* std_dev;
  int64_t* steps_per_level;
  int64_t total_steps;
  double wall_time; /* seconds, host clock around the whole call */
} ermc_solution_t;

/*
 * Full solve, host buffers in and out (replaces ermc::solve,
 * reference solver.cpp:82-180). Validation errors are reported before any
 * kernel runs, with the reference's messages (solver.cpp:14-58).
 */
int ermc_b200_solve(const ermc_grid_t* grid, const double* temperature,
                    const ermc_boundary_t* boundary, const ermc_model_t* model,
                    const ermc_config_t* config, ermc_solution_t* out,
                    char* errbuf, size_t errlen);

/*
 * Solve only linear cells [cell_lo, cell_hi) — one x-slab of a multi-GPU
 * partition (the reference's worker chunks, solver.cpp:163-167). Outputs
 * hold cell_hi - cell_lo values. Results per cell are bitwise those of the
 * full solve.
 */
int ermc_b200_solve_range(const ermc_grid_t* grid, const double* temperature,
                          const ermc_boundary_t* boundary,
                          const ermc_model_t* model,
                          const ermc_config_t* config, int64_t cell_lo,
                          int64_t cell_hi, ermc_solution_t* out, char* errbuf,
                          size_t errlen);

/* ---- Device-resident sessions (inputs stay in HBM between solves). ---- */

typedef struct ermc_session ermc_session_t;

/* Creates a session bound to config->device: uploads the tables, validates
 * the static inputs. The field is supplied separately. */
ermc_session_t* ermc_b200_session_create(const ermc_grid_t* grid,
                                         const ermc_boundary_t* boundary,
                                         const ermc_model_t* model,
                                         const ermc_config_t* config,
                                         char* errbuf, size_t errlen);
void ermc_b200_session_destroy(ermc_session_t* s);

/* Sets the temperature field from host memory (is_device = 0, pageable or
 * pinned) or from a device pointer on the session's device (is_device = 1).
 * Copies are issued on `stream` (cudaStream_t, NULL = legacy default). */
int ermc_b200_session_set_field(ermc_session_t* s, const double* temperature,
                                int is_device, void* stream, char* errbuf,
                                size_t errlen);

/*
 * Solves cells [cell_lo, cell_hi) on `stream` into DEVICE buffers
 * d_q_r / d_std_dev (cell_hi - cell_lo doubles each). steps_per_level
 * (host, n_levels) receives the counters; the call synchronises `stream`
 * once after the trace to read the error word and counters.
 */
int ermc_b200_session_solve(ermc_session_t* s, int64_t cell_lo,
                            int64_t cell_hi, double* d_q_r, double* d_std_dev,
                            int64_t* steps_per_level, void* stream,
                            char* errbuf, size_t errlen);

/* Asynchronous session_solve (the DNS coupling of PAPER.md:354,553: the host
 * keeps computing while the radiation solve runs). session_solve_async
 * validates the field and computes T_max (a short host wait for one device
 * reduction), enqueues the sort, trace and reduction on `stream` and returns;
 * session_wait blocks until they are done, then reports the step counts or
 * the error the solve raised, exactly as session_solve would. One solve may
 * be pending per session; wait before destroying the session or its stream. */
int ermc_b200_session_solve_async(ermc_session_t* s, int64_t cell_lo,
                                  int64_t cell_hi, double* d_q_r, double* d_std_dev,
                                  void* stream, char* errbuf, size_t errlen);
int ermc_b200_session_wait(ermc_session_t* s, int64_t* steps_per_level,
                           char* errbuf, size_t errlen);

/* session_solve with the all-gather fused into the per-cell reduction: each
 * cell's Q_r / sigma is stored into all n_out (<= 8) full-field buffers —
 * this device's and peer GPUs' (mapped with ermc_b200_ipc_open) — at its
 * global linear index, by the reduction kernel itself (NVLink stores on a
 * B200 node). After every rank's call and a barrier each buffer holds the
 * whole field. Replaces the reference's single-process result assembly. */
int ermc_b200_session_solve_scatter(ermc_session_t* s, int64_t cell_lo,
                                    int64_t cell_hi, double* const* d_q_full,
                                    double* const* d_sd_full, int32_t n_out,
                                    int64_t* steps_per_level, void* stream,
                                    char* errbuf, size_t errlen);

/* Device buffers shareable across processes (cudaMalloc'd, so their CUDA IPC
 * handles address the buffer itself). No reference counterpart: the
 * reference solver is one process (solver.cpp:106-170). */
int ermc_b200_device_alloc(int device, size_t bytes, void** d_ptr, char* errbuf,
                           size_t errlen);
int ermc_b200_device_free(void* d_ptr);
/* CUDA IPC export / map / unmap of such a buffer (64-byte handles). */
int ermc_b200_ipc_export(const void* d_ptr, uint8_t handle[64], char* errbuf,
                         size_t errlen);
int ermc_b200_ipc_open(const uint8_t handle[64], void** d_ptr, char* errbuf,
                       size_t errlen);
int ermc_b200_ipc_close(void* d_ptr);

/* Per-kernel device times (CUDA events on the launch stream) of the last
 * session_solve, milliseconds: [0] validate+T_max, [1] restrict + the
 * narrow-band sort of the dispatch order, [2] trace (all chunks),
 * [3] per-cell reduce. Also the launch count. */
int ermc_b200_session_timings(const ermc_session_t* s, double* ms4,
                              int32_t* n_launches);

/* ---- Test hook: trace explicit rays (reference init_ray + march). ---- */

typedef struct ermc_ray_result {
  double q_contribution;
  double weight_absorbed;
  double weight_walls;
  double weight_residual;
  double dir[3];      /* initial direction actually traced */
  double prefactor;   /* R_I */
  double ib_source;
  int64_t steps;
  int32_t terminated_by; /* 0 tolerance, 1 wall_absorbed, 2 step_cap */
  int32_t reflections;
  int32_t band, quad;
  uint32_t next_draw; /* draws consumed */
  int32_t reserved0;
} ermc_ray_result_t;

/*
 * Runs init_ray + march (reference sampling.cpp:55-96, tracer.cpp:57-194)
 * on the GPU for n explicit (cell, ray) pairs with the given T_max-derived
 * sampling setup and q_emission. If dir_override is non-NULL it holds
 * 3*n doubles replacing the sampled directions (the reference's two-cell
 * KAT overrides ray.dir, test_tracer.cpp:65-66). steps_per_level of each
 * ray are written to level_steps[n * n_levels] when non-NULL.
 */
int ermc_b200_trace_rays(const ermc_grid_t* grid, const double* temperature,
                         const ermc_boundary_t* boundary,
                         const ermc_model_t* model, const ermc_config_t* config,
                         double t_max, double q_emission, int64_t n,
                         const int64_t* cell_ids, const uint32_t* ray_ids,
                         const double* dir_override, ermc_ray_result_t* out,
                         int64_t* level_steps, char* errbuf, size_t errlen);

/* ---- The per-ray API of the reference (sampling.hpp, tracer.hpp), on the
 * GPU. Each call runs the device code of the trace kernels on n explicit
 * rays; the C++ API (ermc_b200.hpp: sample_direction, init_ray, march,
 * absorptivity) wraps them one ray at a time. ---- */

/* RayState (reference sampling.hpp:36-51): cell = {i, j, k, level}. */
typedef struct ermc_ray_state {
  double pos[3];
  double dir[3];
  int32_t cell[4];
  double transmissivity;
  int32_t band, quad;
  double prefactor;   /* R_I */
  double ib_source;
  int32_t reflections;
  int32_t reserved0;
  uint64_t seed;
  uint64_t cell_id;
  uint32_t ray_id;
  uint32_t next_draw;
} ermc_ray_state_t;

/* sample_direction (reference sampling.cpp:31-40) for n draw pairs:
 * out[5 i + 0..4] = theta, phi, unit[0..2]. */
int ermc_b200_sample_direction(int64_t n, const double* r_theta, const double* r_phi,
                               double* out, char* errbuf, size_t errlen);
/* absorptivity (reference tracer.cpp:11-13): out[i] = -expm1(-kappa[i] ds[i]). */
int ermc_b200_absorptivity(int64_t n, const double* kappa, const double* ds, double* out,
                           char* errbuf, size_t errlen);
/* init_ray (reference sampling.cpp:55-96) for n (cell, ray) pairs on the
 * level-0 grid / field, with the given sampling CDFs (band_cdf[n_bands],
 * quad_cdf[n_bands * n_quad]) built at t_max. cells = 3 n (i, j, k). */
int ermc_b200_init_rays(const ermc_grid_t* grid, const double* temperature,
                        const ermc_model_t* model, const double* band_cdf,
                        const double* quad_cdf, double t_max, uint64_t seed,
                        int32_t volume_sampling, int64_t n, const int32_t* cells,
                        const uint32_t* ray_ids, ermc_ray_state_t* out, char* errbuf,
                        size_t errlen);
/* march (reference tracer.cpp:57-194) of n ray states through a grid
 * hierarchy given level by level (grids[l], fields[l] k-fastest,
 * step_caps[l], -1 = uncapped), with TraceOptions {tolerance, max_steps,
 * specular}. out: q_contribution, weights, steps, termination, reflections;
 * level_steps[n * n_levels] when non-NULL. */
int ermc_b200_march_rays(int32_t n_levels, const ermc_grid_t* grids,
                         const double* const* fields, const int32_t* step_caps,
                         const ermc_model_t* model, const ermc_boundary_t* boundary,
                         double q_emission, double tolerance, int64_t max_steps,
                         int32_t specular, int64_t n, const ermc_ray_state_t* rays,
                         ermc_ray_result_t* out, int64_t* level_steps, char* errbuf,
                         size_t errlen);

/* ---- Host setup the kernel consumes (bitwise the reference's). ---- */

/* build_cdfs (reference spectral.cpp:306-354): band_cdf[n_bands],
 * quad_cdf[n_bands*n_quad]. */
int ermc_b200_build_cdfs(const ermc_model_t* model, double t_max,
                         double* band_cdf, double* quad_cdf, char* errbuf,
                         size_t errlen);
/* SpectralModel::planck_mean (reference spectral.cpp:207-218). */
int ermc_b200_planck_mean(const ermc_model_t* model, double temperature,
                          double* out, char* errbuf, size_t errlen);
/* The keyed uniform draw (reference sampling.cpp:13-29), evaluated on the
 * GPU for n keys; used by tests to pin the device RNG. */
int ermc_b200_uniform_device(uint64_t seed, int64_t n, const uint64_t* cell_ids,
                             const uint32_t* ray_ids, const uint32_t* draw_ids,
                             double* out, char* errbuf, size_t errlen);

/* Number of visible CUDA devices (0 when none); never fails. */
int ermc_b200_device_count(void);
/* ABI version for loaders. */
int ermc_b200_abi_version(void);
/* The solve entry points keep freed device buffers in a per-device cache
 * (up to a third of the device memory) so repeated one-shot solves do not
 * pay cudaMalloc/cudaFree; this returns the cached blocks of `device`
 * (-1 = current) to the driver. No reference counterpart (the reference
 * has no device memory). Returns 0. */
int ermc_b200_release_cached_memory(int device);

/* L2 bandwidth probe (measurement only; no reference counterpart): reads
 * an L2-resident buffer of `bytes` (1 MiB .. ~64 MiB) on `device` (-1 =
 * current). mode 0: streaming 16-byte ld.global.cg sweeps, `iters` times;
 * mode 1: independent hashed 8-byte gathers, one 32-byte sector each,
 * counted as sector bytes. *gbs = bytes moved / kernel time (CUDA events).
 * The denominator of bench.py's roofline.l2. */
int ermc_b200_probe_l2(int device, size_t bytes, int iters, int mode, double* gbs,
                       char* errbuf, size_t errlen);

#ifdef __cplusplus
}
#endif

#endif /* ERMC_B200_H */
