// trace_common.cuh — parameter blocks shared by the host launcher
// (capi.cu) and the trace kernels (trace_fp64.cu, trace_fp32.cu).
//
// Everything the kernel needs is precomputed on the host with the reference's
// own arithmetic (bitwise): per-level grid constants, T_max-derived sampling
// CDFs, k(n,g,T_max) and Ib(n,T_max), wall blackbodies per (face, band),
// the emission weight QE and the seed hash. The kernel then only marches.
#pragma once

#include <cstdint>

#include "ermc_b200.h"  // ermc_ray_state_t (the per-ray API's state)

namespace ermc_dev {

constexpr int kMaxLevels = 16;
constexpr int kMaxSmemCdf = 2048;  // sampling CDFs staged in shared memory up to
                                   // this many doubles (16 KB; 119 x 16 needs 2023)
// Guide tables of the staged CDFs (sample_band_cdf): the band CDF is split
// in kGuideBand equal buckets of [0, 1), each g CDF in kGuideQuad; a bucket
// holds upper_bound(cdf, bucket start), where the search for any r in the
// bucket can start.
constexpr int kGuideBand = 64;
constexpr int kGuideQuad = 16;

// Division by a loop-invariant divisor d >= 1 for numerators n < 2^31:
// q = (umulhi(n, m) + n) >> s with s = ceil(log2 d),
// m = floor(2^32 (2^s - d) / d) + 1 (Granlund-Montgomery); 3 instructions
// instead of the ~18 of a runtime 32-bit division.
struct FastDiv {
  uint32_t d, m, s, pad;
};

// One multigrid level (reference GridHierarchy, geometry.hpp:74-83).
struct LevelDesc {
  int32_t n[3];      // cells per axis
  int32_t cap;       // steps before demotion; -1 = uncapped (coarsest level)
  double d[3];       // spacing per axis
  double rd[3];      // RN(1 / spacing): Markstein divisions by the spacing
  double origin[3];  // grid origin
  double extent[3];  // n * d, computed as CartesianGrid::extent
  double eps;        // geom_eps = 1e-12 * min spacing (geometry.hpp:114-116)
  const double* field;   // fp64 temperature, k-fastest
  const float* field32;  // fp32 copy for the fast kernel (may be null)
  const float* field32b;   // fp32 in 2x2x2 micro-bricks (even grids, lean kernel)
  const double* field64b;  // fp64 in 2x2x2 micro-bricks (even grids, lean kernel)
  // Table coordinates of every cell (lean fp64 tracers, see TraceParams::cw_*):
  // (lo << cw_shift) | m, where lo is the reference lookup's interval and
  // m * 2^-cw_scale_exp == T - t[lo] exactly.
  const uint64_t* cellw;
  // Step budget of a ray on this level (set_level_budgets): the steps it can
  // take here before it demotes or reaches max_steps, counted from its first
  // step on the level; budget_demotes = 1 when the budget ends in a demotion.
  int32_t budget;
  int32_t budget_demotes;
};

// Error codes raised on the device; the host re-traces the failing ray
// through the debug kernel to build the reference's message.
enum DevError : int32_t {
  kErrNone = 0,
  kErrNonFinite = 1,      // tracer.cpp:134-138
  kErrTableRange = 2,     // spectral.cpp:149-153
  kErrTransparent = 3,    // sampling.cpp:91-93
  kErrLocate = 4,         // geometry.cpp:119-127
};

struct TraceParams {
  // ---- geometry ----
  int32_t n_levels;
  int32_t periodic[3];
  int32_t periodic_mask;     // bit a set when axis a is periodic
  LevelDesc lv[kMaxLevels];
  double wall_eps[6];        // face = 2*axis + (hi ? 1 : 0)
  const double* wall_ib;     // [6][n_bands] interp_ib(band, T_wall) or 0

  // ---- spectral tables ----
  int32_t n_bands, n_quad, n_temps;
  int32_t uniform_temps;     // SpectralModel uniform fast path (spectral.cpp:119-129)
  double t0, dt;             // uniform grid origin and step
  const double* temps;       // [n_temps]
  const double* k;           // [n_bands][n_quad][n_temps]
  const double* ib;          // [n_bands][n_temps]
  const double* band_cdf;    // [n_bands]
  const double* quad_cdf;    // [n_bands][n_quad]
  const double* k_max;       // [n_bands][n_quad]  k(n,g,T_max)
  const double* ib_max;      // [n_bands]          Ib(n,T_max)
  // Packed fp64 tables of the fast single-level kernel (values are copies, so
  // interpolation stays bitwise the reference's):
  const double4* tint;       // [n_temps-1] {t_lo, t_hi - t_lo, 1/(t_hi - t_lo), 0}
  const double4* iv64;       // [n_bands*n_quad][n_temps-1] {k_lo, k_hi, ib_lo, ib_hi}
  double inv_dt;             // 1/dt for the table-index estimate
  double inv_w;              // RN(1 / dt): tint's reciprocal when tint_arith
  int32_t cdf_smem;          // lean kernels stage in shared memory: 0 nothing, 1 the
                             // sampling CDFs + their guide tables, 2 the guides only
                             // (large CDFs stay in L1-cached global memory)
  const uint8_t* cdf_guide;  // [kGuideBand + n_bands * kGuideQuad] (with cdf_smem)
  int32_t tint_arith;        // every node is exactly l*dt + t0 and every width
                             // exactly dt, so tint[l] is computed, not loaded
  double t_first, t_last;    // table range
  // Cell words (LevelDesc::cellw): the lookup's (lo, frac) precomputed per
  // cell once per field. frac = RN(m / cw_dt) with cw_dt = dt * 2^s and
  // cw_rdt = RN(1 / cw_dt) (Markstein: the reference's RN((T - t[lo]) / dt),
  // bitwise; the builder checks it cell by cell).
  int32_t carveout;          // shared-memory carveout request: -1 driver default,
                             // 0 the smallest that holds the resident blocks, > 0 percent
  int32_t cellw;             // 1: the lean fp64 tracers read cell words
  int32_t cw_shift;          // lo = w >> cw_shift (64 - bits of the interval index)
  double cw_dt, cw_rdt;

  // ---- fp32 fast-path tables (trace_fp32.cu) ----
  const float4* iv32;        // [n_bands*n_quad][n_temps-1] {k_lo, k_hi-k_lo, ib_lo, ib_hi-ib_lo}
  const float* wall_ibn32;   // [6][n_bands] wall Ib / Ib(n, T_last)
  float inv_dt32;            // 1/dt for the fp32 lookup (uniform grids only)
  float t0_32;
  float tol32;               // tolerance as float
  float u0_32;               // -t0 / dt as float (table coordinate offset)

  // ---- march options (TraceOptions, tracer.hpp:26-30) ----
  double qe;                 // 4 kappa_p(T_max) sigma T_max^4 / R (solver.cpp:92-93)
  double tol;
  int64_t max_steps;
  int32_t specular;
  int32_t volume_sampling;
  uint64_t h_seed;           // mix64(seed + 0x9e3779b97f4a7c15) (sampling.cpp:25)
  int32_t rays;              // rays per cell

  // ---- per-ray setup helpers (bitwise the reference's arithmetic) ----
  FastDiv div_rays, div_nyz, div_nz;  // work id -> (cell, ray); level-0 cell decode
  FastDiv div_row;  // interval row -> band: n_quad * (n_temps - 1)
  const double2* pref_den;   // [n_bands*n_quad] {k(n,g,T_max) Ib(n,T_max), RN(1 / that)}

  // ---- work decomposition ----
  int32_t refill_threshold;  // idle lanes before a warp regenerates rays
  int32_t inner_steps;       // march steps between two pool checks
  int32_t lean;              // fp64: 1 = lean tracer (per-axis records in smem)
  int32_t brick;             // lean tracers read the micro-brick field copy
  int32_t track_pos;         // 0 when every wall is black (positions never read)
  int64_t cell_base;         // first global linear cell of this chunk
  int64_t n_cells;           // cells in this chunk
  uint64_t n_work;           // n_cells * rays (ray work items)
  const uint32_t* perm;      // dispatch order of the work ids (narrow-band
                             // sorted, dispatch.cu) or null = cell-major
  unsigned long long* work_counter;
  double* q_ray;             // [rays][n_cells] per-ray q contributions
  unsigned long long* steps_per_level;  // [n_levels]
  unsigned long long* err_key;          // ~(min failing work item) (0 = none)
  int32_t* err_code;
};

// Per-level step budgets (LevelDesc::budget) from the caps and max_steps, in
// the order of the reference's checks (tracer.cpp:88-101): a ray stops at
// max_steps before it demotes. Host side, after the levels and max_steps are
// set.
inline void set_level_budgets(TraceParams& P) {
  const long long ms = P.max_steps < 0x7fffffffLL ? P.max_steps : 0x7fffffffLL;
  long long start = 0;  // steps taken on the finer levels when a ray arrives
  for (int l = 0; l < P.n_levels; ++l) {
    LevelDesc& L = P.lv[l];
    const bool capped = L.cap >= 0 && l + 1 < P.n_levels;
    const long long left = ms > start ? ms - start : 0;
    const bool demotes = capped && start + L.cap < ms;
    L.budget = static_cast<int32_t>(demotes ? L.cap : left);
    L.budget_demotes = demotes ? 1 : 0;
    if (!demotes) {  // no ray gets past this level
      for (int k = l + 1; k < P.n_levels; ++k) {
        P.lv[k].budget = 0;
        P.lv[k].budget_demotes = 0;
      }
      break;
    }
    start += L.cap;
  }
}

// Full-field output buffers of the fused reduce + all-gather (K2 scatter).
constexpr int kMaxScatter = 8;
struct ScatterOut {
  double* q[kMaxScatter];
  double* sd[kMaxScatter];
  int32_t n;
};

// Debug / test record of one traced ray (ermc_ray_result_t mirror).
struct RayRecord {
  double q;
  double w_abs, w_walls, w_res;
  double dir[3];
  double prefactor, ib_source;
  int64_t steps;
  int32_t term, reflections, band, quad;
  uint32_t next_draw;
  int32_t err;
  double err_value;   // offending temperature / coordinate
  int32_t err_axis;
  int32_t pad;
};

#ifdef __CUDACC__
// L1 / shared-memory split of a trace kernel. The driver's default for these
// kernels is the 132 KB shared-memory configuration (ncu
// launch__shared_mem_config_size), although their resident blocks need far
// less: the smallest configuration that holds `blocks` blocks (their dynamic
// and static shared memory plus the 1 KB the driver reserves per block)
// leaves the rest of the 256 KB to the L1 that caches the gathers.
inline cudaError_t set_trace_carveout(const void* fn, int grid, size_t dyn_smem, int request) {
  if (request < 0) return cudaSuccess;
  int pct = request;
  if (pct == 0) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, fn);
    const int blocks = (grid + sms - 1) / sms;
    const size_t need = static_cast<size_t>(blocks) * (dyn_smem + fa.sharedSizeBytes + 1024);
    pct = static_cast<int>((need * 100 + 228 * 1024 - 1) / (228 * 1024));
    if (pct > 100) pct = 100;
  }
  return cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
}
#endif

}  // namespace ermc_dev
