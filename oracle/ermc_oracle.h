/*
 * ermc_oracle.h — TEST INFRASTRUCTURE ONLY: a plain-C restatement of the
 * reference's ERMC solve path, used as the checker (never the product).
 *
 * Restates /root/reference/proj/src: sampling.cpp:13-96 (keyed RNG,
 * direction / band sampling, init_ray), tracer.cpp:11-194 (march),
 * solver.cpp:27-155 (T_max, QE, per-cell Welford), spectral.cpp:148-218,
 * 306-354 (lookup, interpolation, Planck mean, CDFs), geometry.cpp:51-138
 * (restriction, locate) and oracles.cpp:13-128 + expint.cpp:10-48 (the
 * analytic grey-slab oracle). Pinned bitwise against the reference library
 * compiled into oracle/_ref (tests/test_oracle.py) and against committed
 * golden vectors (tests/golden/).
 *
 * Descriptors are the product's C-ABI structs (include/ermc_b200.h).
 */
#ifndef ERMC_ORACLE_H
#define ERMC_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#include "../include/ermc_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

double oracle_uniform(uint64_t seed, uint64_t cell, uint32_t ray, uint32_t draw);

int oracle_build_cdfs(const ermc_model_t* m, double t_max, double* band_cdf,
                      double* quad_cdf, char* err, size_t errlen);
int oracle_planck_mean(const ermc_model_t* m, double t, double* out, char* err,
                       size_t errlen);

/* Solve cells [cell_lo, cell_hi) with n_threads pthreads (cells striped). */
int oracle_solve(const ermc_grid_t* g, const double* temperature,
                 const ermc_boundary_t* b, const ermc_model_t* m,
                 const ermc_config_t* c, int64_t cell_lo, int64_t cell_hi,
                 double* q_r, double* std_dev, int64_t* steps_per_level,
                 int n_threads, char* err, size_t errlen);

/* Explicit rays at a given T_max and q_emission (tracer KAT replays). */
int oracle_trace_rays(const ermc_grid_t* g, const double* temperature,
                      const ermc_boundary_t* b, const ermc_model_t* m,
                      const ermc_config_t* c, double t_max, double qe, int64_t n,
                      const int64_t* cells, const uint32_t* rays,
                      const double* dirs, ermc_ray_result_t* out, char* err,
                      size_t errlen);

/* Temperature profiles of the reference case library (cases.cpp:11-15). */
enum {
  ORACLE_PROFILE_CONST = 0, /* T = t_const */
  ORACLE_PROFILE_LIN1 = 1,  /* 500 + 1000 x */
  ORACLE_PROFILE_LIN2 = 2,  /* 295 + 10 x */
  ORACLE_PROFILE_PARAB = 3  /* 500 - 2000 x^2 + 2000 x */
};
double oracle_profile(int profile, double t_const, double x);

/* Analytic grey slab Q^R(x) (oracles.cpp:73-128): exponential-integral
 * kernels with a reflection series for grey walls. */
int oracle_slab(double length, int profile, double t_const, double kappa,
                double t_lo, double eps_lo, double t_hi, double eps_hi,
                const double* x, int nx, int refine, double* q, char* err,
                size_t errlen);

/* Restatement of the fp64 lean kernel's expm1 and its distance to glibc. */
double oracle_expm1_lean(double x);
double oracle_expm1_lean_max_ulp(long n, long* n_differ);

double oracle_expint_e1(double x);
double oracle_expint_e2(double x);
double oracle_expint_e3(double x);

#ifdef __cplusplus
}
#endif

#endif
