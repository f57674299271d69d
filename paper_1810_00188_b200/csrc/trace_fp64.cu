// trace_fp64.cu — the ERMC hot path on sm_100a, reference (fp64) arithmetic.
//
// K1 `trace_pool_fp64`: fused init_ray + march for every (cell, ray) work
// item of a cell range (reference sampling.cpp:55-96, tracer.cpp:57-194,
// driven per cell by solver.cpp:115-140). One persistent CTA set covers the
// SMs; every lane owns one ray at a time and regenerates a new ray from a
// warp-local work pool when its ray terminates (the paper's persistent ray
// pool), so lanes never wait for the longest ray of a
// batch. The per-ray reciprocal exchange q is written to q_ray[ray][cell];
// K2 `reduce_cells` then does the reference's per-cell sum + Welford in
// ray-id order (solver.cpp:142-155), so results do not depend on the
// marching order — the GPU analogue of the reference's worker/sorting
// invariance (P5, P8).
//
// This translation unit is compiled with --fmad=false and IEEE div/sqrt so
// every add/mul/div rounds exactly like the reference's x86-64 build (no FMA
// contraction). Only libdevice expm1/sin/cos may differ from glibc by an
// ulp, which bounds the per-cell parity.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "device_common.cuh"
#include "trace_common.cuh"

namespace ermc_dev {

namespace {

constexpr double kPiD = kPiDev;
constexpr int kBlock = 128;
constexpr unsigned kFull = kFullMask;

// SpectralModel::lookup (reference spectral.cpp:148-177). Returns false when
// T is outside the table (the reference throws).
__device__ __forceinline__ bool t_lookup(const TraceParams& P, double T,
                                         int& lo, double& frac) {
  const double* tg = P.temps;
  const int nt = P.n_temps;
  if (!(T >= __ldg(tg) && T <= __ldg(tg + nt - 1))) return false;
  if (nt < 2) {  // single node: exact (the reference indexes node -1 here)
    lo = 0;
    frac = 0.0;
    return true;
  }
  if (P.uniform_temps) {
    int l = static_cast<int>((T - P.t0) / P.dt);
    l = min(max(l, 0), nt - 2);
    double a = __ldg(tg + l), b = __ldg(tg + l + 1);
    double f = (T - a) / (b - a);
    if (f < 0.0 && l > 0) {
      --l;
      f = (T - __ldg(tg + l)) / (__ldg(tg + l + 1) - __ldg(tg + l));
    } else if (f > 1.0 && l < nt - 2) {
      ++l;
      f = (T - __ldg(tg + l)) / (__ldg(tg + l + 1) - __ldg(tg + l));
    }
    lo = l;
    frac = f;
    return true;
  }
  int hi = upper_bound_d(tg, nt, T);
  if (hi == 0) {
    lo = 0;
    frac = 0.0;
  } else if (hi == nt) {
    lo = nt - 2;
    frac = 1.0;
  } else {
    lo = hi - 1;
    double a = __ldg(tg + lo);
    frac = (T - a) / (__ldg(tg + hi) - a);
  }
  return true;
}

// a + frac*(b - a) with the frac == 0 exact shortcut (spectral.cpp:179-205).
__device__ __forceinline__ double interp_row(const double* row, int lo,
                                             double frac) {
  double a = __ldg(row + lo);
  if (frac == 0.0) return a;
  return a + frac * (__ldg(row + lo + 1) - a);
}

struct Ray {
  double pos[3], dir[3], tn[3], td[3];
  double tau, q, last_ib2, ib1, pref;
  const double* krow;
  const double* ibrow;
  int idx[3], stp[3];
  int band, quad, level, sal, steps;
  uint32_t next_draw, ray_id;
  uint64_t h_cell;
};

struct DebugRec {
  double w_abs, w_walls;
  int reflections, term;
  int64_t level_steps[kMaxLevels];
  double err_value;
  int err_axis;
};

// Dda::setup (reference tracer.cpp:17-38).
__device__ __forceinline__ void dda_setup(const LevelDesc& L, Ray& r) {
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    double da = r.dir[a];
    if (da == 0.0) {
      r.tn[a] = __longlong_as_double(0x7ff0000000000000LL);
      r.td[a] = __longlong_as_double(0x7ff0000000000000LL);
      r.stp[a] = 0;
      continue;
    }
    r.stp[a] = da > 0.0 ? 1 : -1;
    int face_idx = r.idx[a] + (da > 0.0 ? 1 : 0);
    double face = L.origin[a] + face_idx * L.d[a];
    r.tn[a] = (face - r.pos[a]) / da;
    r.td[a] = L.d[a] / fabs(da);
  }
}

// One iteration of march's loop (reference tracer.cpp:82-185).
// kMulti enables the multigrid demotion branch (tracer.cpp:91-101).
template <bool kMulti, bool kDebug>
__device__ __forceinline__ int march_step(const TraceParams& P, Ray& r,
                                          int max_steps, DebugRec* dbg,
                                          int* err) {
  if (r.tau <= P.tol) {
    if (kDebug) dbg->term = 0;
    return kDone;
  }
  if (r.steps >= max_steps) {
    if (kDebug) dbg->term = 2;
    return kDone;
  }
  if (kMulti) {
    const int cap = P.lv[r.level].cap;
    if (cap >= 0 && r.sal >= cap && r.level + 1 < P.n_levels) {
      // Demote: same position/direction/transmissivity on coarser cells;
      // locate(grid, pos, dir) (geometry.cpp:112-138).
      ++r.level;
      const LevelDesc& C = P.lv[r.level];
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        double p = r.pos[a] + C.eps * r.dir[a];
        double rel = (p - C.origin[a]) / C.d[a];
        int i = static_cast<int>(floor(rel));
        if (i < 0 || i >= C.n[a]) {
          if (rel >= -1e-9 && i < 0) {
            i = 0;
          } else if (rel <= C.n[a] + 1e-9 && i >= C.n[a]) {
            i = C.n[a] - 1;
          } else {
            if (kDebug) {
              dbg->err_axis = a;
              dbg->err_value = rel;
            }
            *err = kErrLocate;
            return kFail;
          }
        }
        r.idx[a] = i;
      }
      r.sal = 0;
      dda_setup(C, r);
    }
  }
  const LevelDesc& L = P.lv[kMulti ? r.level : 0];

  int axis = 0;
  double ds = r.tn[0];
  if (r.tn[1] < ds) {
    ds = r.tn[1];
    axis = 1;
  }
  if (r.tn[2] < ds) {
    ds = r.tn[2];
    axis = 2;
  }
  if (ds < 0.0) ds = 0.0;

  const int64_t lin =
      (static_cast<int64_t>(r.idx[0]) * L.n[1] + r.idx[1]) * L.n[2] + r.idx[2];
  const double t_cell = __ldg(L.field + lin);
  int lo;
  double frac;
  if (!t_lookup(P, t_cell, lo, frac)) {
    if (kDebug) dbg->err_value = t_cell;
    *err = kErrTableRange;
    return kFail;
  }
  const double kappa = interp_row(r.krow, lo, frac);
  const double ib2 = interp_row(r.ibrow, lo, frac);
  const double alpha = -expm1(-kappa * ds);
  r.last_ib2 = ib2;
  r.q += P.qe * r.tau * alpha * ((ib2 - r.ib1) / r.ib1) * r.pref;
  if (kDebug) dbg->w_abs += r.tau * alpha;
  r.tau *= 1.0 - alpha;

  const double advance = ds + L.eps;
  r.pos[0] += advance * r.dir[0];
  r.pos[1] += advance * r.dir[1];
  r.pos[2] += advance * r.dir[2];
  r.tn[0] -= advance;
  r.tn[1] -= advance;
  r.tn[2] -= advance;
#pragma unroll
  for (int a = 0; a < 3; ++a)
    if (a == axis) r.tn[a] += r.td[a];
  ++r.steps;
  if (kMulti) ++r.sal;
  if (kDebug) ++dbg->level_steps[r.level];

  // Non-finite values propagate to the end of the ray, where the pool
  // checks them; the debug tracer checks every step like the reference.
  if (kDebug && (!isfinite(r.q) || !isfinite(r.tau))) {
    *err = kErrNonFinite;
    return kFail;
  }

  int ia = 0, na = 0, sa = 0;
#pragma unroll
  for (int a = 0; a < 3; ++a)
    if (a == axis) {
      r.idx[a] += r.stp[a];
      ia = r.idx[a];
      na = L.n[a];
      sa = r.stp[a];
    }
  if (ia >= 0 && ia < na) return kContinue;

  if (P.periodic[axis]) {
    const double ext = L.extent[axis];
#pragma unroll
    for (int a = 0; a < 3; ++a)
      if (a == axis) {
        if (ia < 0) {
          r.idx[a] = na - 1;
          r.pos[a] += ext;
        } else {
          r.idx[a] = 0;
          r.pos[a] -= ext;
        }
      }
    return kContinue;
  }

  // Wall exchange, then absorption or reflection (tracer.cpp:155-184).
  const bool at_hi = sa > 0;
  const int face = 2 * axis + (at_hi ? 1 : 0);
  const double ew = P.wall_eps[face];
  const double ib_w = __ldg(P.wall_ib + face * P.n_bands + r.band);
  r.q += P.qe * r.tau * ew * ((ib_w - r.ib1) / r.ib1) * r.pref;
  if (kDebug) dbg->w_walls += r.tau * ew;
  r.tau *= 1.0 - ew;
  if (r.tau <= P.tol) {
    if (kDebug) dbg->term = 1;
    return kDone;
  }
  if (kDebug) ++dbg->reflections;
  const double face_pos = L.origin[axis] + (at_hi ? L.extent[axis] : 0.0);
  const int inward = at_hi ? -1 : 1;
  double nd[3] = {r.dir[0], r.dir[1], r.dir[2]};
  if (P.specular) {
#pragma unroll
    for (int a = 0; a < 3; ++a)
      if (a == axis) nd[a] = -nd[a];
  } else {
    // diffuse_reflection (tracer.cpp:42-53)
    double r1 = draw_u(r.h_cell, r.ray_id, r.next_draw++);
    double r2 = draw_u(r.h_cell, r.ray_id, r.next_draw++);
    double sin_t = sqrt(r1);
    double cos_t = sqrt(1.0 - r1);
    double phi = 2.0 * kPiD * r2;
    double sp, cp;
    sincos(phi, &sp, &cp);
    const int t1 = axis == 2 ? 0 : axis + 1;
    const int t2 = axis == 0 ? 2 : axis - 1;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      if (a == axis) nd[a] = inward * cos_t;
      if (a == t1) nd[a] = sin_t * cp;
      if (a == t2) nd[a] = sin_t * sp;
    }
  }
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    if (a == axis) {
      r.idx[a] -= r.stp[a];
      r.pos[a] = face_pos;
    }
    r.dir[a] = nd[a];
  }
  r.pos[0] += L.eps * r.dir[0];
  r.pos[1] += L.eps * r.dir[1];
  r.pos[2] += L.eps * r.dir[2];
  dda_setup(L, r);
  return kContinue;
}

// Residual dump into the source cell (tracer.cpp:186-188).
__device__ __forceinline__ double finish_ray(const TraceParams& P,
                                             const Ray& r) {
  return r.q + P.qe * r.tau * ((r.last_ib2 - r.ib1) / r.ib1) * r.pref;
}

// ---------------------------------------------------------------------------
// Fast single-level tracer. Same operations, same order, same rounding as
// march_step (hence the reference), restructured for the gather latency:
//   * T of the next cell is loaded one step ahead, while the current step's
//     absorption math runs (the DDA does not depend on absorption);
//   * one 32-byte interval record {k_lo, k_hi, ib_lo, ib_hi} per step instead
//     of four scattered loads, and {t_lo, w, 1/w} per temperature interval;
//   * divisions by a per-ray or per-interval constant use its correctly
//     rounded reciprocal plus one FMA correction (Markstein), which returns
//     the correctly rounded quotient, i.e. bitwise the IEEE division;
//   * the table index estimate (T - t0) * (1/dt) falls back to the true
//     division near an integer, so trunc() sees the reference's quotient.

// Correctly rounded a / b from r = RN(1/b) (Markstein / Cornea et al.).
__device__ __forceinline__ double div_rcp(double a, double b, double r) {
  const double q0 = a * r;
  const double e = fma(-q0, b, a);
  return fma(e, r, q0);
}

// The reference's table index trunc((T - t0) / dt) with the IEEE division;
// kept out of line so the common multiply path is not if-converted into it.
__device__ __noinline__ int exact_index(double T, double t0, double dt) {
  return static_cast<int>((T - t0) / dt);
}

// SpectralModel::lookup on the packed tables (uniform or not). The interval
// record of the returned lo is loaded into *rec (issued together with the
// temperature record so the two loads overlap).
template <int kHint = 0>
__device__ __forceinline__ bool fast_lookup(const TraceParams& P,
                                            const double4* row, double T,
                                            int& lo, double& frac,
                                            double4& rec) {
  if (!(T >= P.t_first && T <= P.t_last)) return false;
  const int nt = P.n_temps;
  int l;
  if (P.uniform_temps) {
    const double x = (T - P.t0) * P.inv_dt;
    const double xf = x - floor(x);
    if (xf < 1e-9 || xf > 1.0 - 1e-9)
      l = exact_index(T, P.t0, P.dt);
    else
      l = static_cast<int>(x);
    l = min(max(l, 0), nt - 2);
    rec = ld_rec64<kHint>(row + l);
    double4 ti;
    if (P.tint_arith)  // the nodes are exactly t0 + l*dt (checked on the host)
      ti = make_double4(static_cast<double>(l) * P.dt + P.t0, P.dt, P.inv_w, 0.0);
    else
      ti = ld_rec64<kHint>(P.tint + l);
    double f = div_rcp(T - ti.x, ti.y, ti.z);
    if ((f < 0.0 && l > 0) || (f > 1.0 && l < nt - 2)) {
      // rounding put T in the neighbouring interval (spectral.cpp:159-168)
      l += f < 0.0 ? -1 : 1;
      ti = ld_rec64<kHint>(P.tint + l);
      rec = ld_rec64<kHint>(row + l);
      f = div_rcp(T - ti.x, ti.y, ti.z);
    }
    lo = l;
    frac = f;
    return true;
  }
  const int hi = upper_bound_d(P.temps, nt, T);
  if (hi == 0) {
    lo = 0;
    frac = 0.0;
  } else if (hi == nt) {
    lo = nt - 2;
    frac = 1.0;
  } else {
    lo = hi - 1;
    const double4 ti = ldg4(P.tint + lo);
    frac = div_rcp(T - ti.x, ti.y, ti.z);
  }
  rec = ldg4(row + lo);
  return true;
}

// fast_lookup with the common case as one straight-line block: the index
// estimate, the record loads and the Markstein quotient run unconditionally;
// every rare condition (T outside the table, an estimate within 1e-9 of an
// integer, a quotient outside [0, 1], non-uniform or non-arithmetic nodes)
// is OR-ed into one predicate that re-runs fast_lookup. Same results;
// measured +3.4 % on the fp64 tracer (a branch-free expm1 was 2.4 % slower).
template <int kHint = 0>
__device__ __forceinline__ bool lookup_spec(const TraceParams& P, const double4* row,
                                            double T, int& lo, double& frac,
                                            double4& rec) {
  const int nt = P.n_temps;
  const double x = (T - P.t0) * P.inv_dt;
  const double xf = x - floor(x);
  const int l = min(max(static_cast<int>(x), 0), nt - 2);
  rec = ld_rec64<kHint>(row + l);
  const double tl = static_cast<double>(l) * P.dt + P.t0;
  const double f = div_rcp(T - tl, P.dt, P.inv_w);
  const bool rare = !(T >= P.t_first && T <= P.t_last) || !P.tint_arith ||
                    xf < 1e-9 || xf > 1.0 - 1e-9 || (f < 0.0 && l > 0) ||
                    (f > 1.0 && l < nt - 2);
  if (rare) return fast_lookup<kHint>(P, row, T, lo, frac, rec);
  lo = l;
  frac = f;
  return true;
}

// Cell words (TraceParams::cw_*): the lookup of a cell's temperature,
// precomputed once per field. The interval index sits in the top 8 bits;
// the low 56 hold m = (T - t[lo]) * 2^s, an exact integer because every
// in-range T and table node is a multiple of ulp(t_first) = 2^-s, and
// T - t[lo] is exact (Sterbenz: t[lo] <= T <= t[lo] + dt <= 2 t[lo]).
// frac = RN(m / (dt 2^s)) = RN((T - t[lo]) / dt), the reference's quotient
// (spectral.cpp:148-177) — the builder verifies it for every cell.
constexpr int kCwShift = 56;

__device__ __forceinline__ void decode_cw(const TraceParams& P, uint64_t w, int& lo,
                                          double& frac) {
  lo = static_cast<int>(w >> kCwShift);
  const uint64_t m = w & ((1ull << kCwShift) - 1ull);
  frac = div_rcp(static_cast<double>(m), P.cw_dt, P.cw_rdt);
}

// init_ray (reference sampling.cpp:55-96) for global cell `cell`, with the
// level-0 grid. Returns an error code (0 = ok).
// cdf: the staged sampling CDFs (lean kernels) or null for P's global copy.
// kLean: the lean tracers' variant — the table lookup runs on the packed
// interval records (lookup_spec: same values), and the DDA setup is left to
// the tracer, which builds its own per-axis records.
template <bool kLean = false, bool kCW = false>
__device__ __forceinline__ int init_ray(const TraceParams& P, int64_t cell,
                                        uint32_t ray_id, Ray& r,
                                        const double* dir_override,
                                        const void* staged = nullptr,
                                        const uint8_t* guide = nullptr) {
  const LevelDesc& L = P.lv[0];
  int ci, cj, ck;
  decode_cell(P, cell, ci, cj, ck);
  r.h_cell = mix64(P.h_seed ^ static_cast<uint64_t>(cell));
  r.ray_id = ray_id;
  double r_theta = draw_u(r.h_cell, ray_id, 0);
  double r_phi = draw_u(r.h_cell, ray_id, 1);
  double r_n = draw_u(r.h_cell, ray_id, 2);
  double r_g = draw_u(r.h_cell, ray_id, 3);
  r.next_draw = 4;

  // sample_direction (sampling.cpp:31-40)
  double cos_t = 1.0 - 2.0 * r_theta;
  double phi = 2.0 * kPiD * r_phi;
  double sin_t = sqrt(fmax(0.0, 1.0 - cos_t * cos_t));
  double sp, cp;
  sincos(phi, &sp, &cp);
  r.dir[0] = sin_t * cp;
  r.dir[1] = sin_t * sp;
  r.dir[2] = cos_t;
  if (dir_override) {
    r.dir[0] = dir_override[0];
    r.dir[1] = dir_override[1];
    r.dir[2] = dir_override[2];
  }

  int n, g;
  if (guide)
    sample_band_guided(P, guide, r_n, r_g, n, g);
  else
    sample_band_staged(P, staged, r_n, r_g, n, g);
  r.band = n;
  r.quad = g;
  r.krow = P.k + (static_cast<int64_t>(n) * P.n_quad + g) * P.n_temps;
  r.ibrow = P.ib + static_cast<int64_t>(n) * P.n_temps;

  // cell centre (geometry.hpp:28-31), optional volume sampling
  r.idx[0] = ci;
  r.idx[1] = cj;
  r.idx[2] = ck;
  r.pos[0] = L.origin[0] + (ci + 0.5) * L.d[0];
  r.pos[1] = L.origin[1] + (cj + 0.5) * L.d[1];
  r.pos[2] = L.origin[2] + (ck + 0.5) * L.d[2];
  if (P.volume_sampling) {
#pragma unroll
    for (int a = 0; a < 3; ++a)
      r.pos[a] += (draw_u(r.h_cell, ray_id, r.next_draw++) - 0.5) * L.d[a];
  }

  int lo;
  double frac;
  double k1;
  if (kLean) {
    double4 v;  // {k_lo, k_hi, ib_lo, ib_hi}: copies of the table values
    const double4* row = P.iv64 + (n * P.n_quad + g) * (P.n_temps - 1);
    if (kCW) {
      decode_cw(P, __ldg(L.cellw + cell), lo, frac);
      v = ld_rec64<0>(row + lo);
    } else if (!lookup_spec<0>(P, row, __ldg(L.field + cell), lo, frac, v)) {
      return kErrTableRange;
    }
    r.ib1 = frac == 0.0 ? v.z : v.z + frac * (v.w - v.z);
    k1 = frac == 0.0 ? v.x : v.x + frac * (v.y - v.x);
  } else {
    if (!t_lookup(P, __ldg(L.field + cell), lo, frac)) return kErrTableRange;
    r.ib1 = interp_row(r.ibrow, lo, frac);
    k1 = interp_row(r.krow, lo, frac);
  }
  // R_I = (k1 Ib1) / (k_max Ib_max) (sampling.cpp:88-94); the lean tracers
  // divide by the per-(n, g) denominator with its correctly rounded
  // reciprocal (Markstein: bitwise the IEEE quotient for normal operands).
  const double num = k1 * r.ib1;
  bool have_pref = false;
  if (kLean) {
    const double2 den = __ldg(P.pref_den + n * P.n_quad + g);
    const double an = fabs(num);
    if (den.x >= 0x1p-960 && den.x <= 0x1p960 &&
        ((an >= 0x1p-960 && an <= 0x1p960) || num == 0.0)) {
      r.pref = div_rcp(num, den.x, den.y);
      have_pref = true;
    }
  }
  if (!have_pref) {
    const double k_max = __ldg(P.k_max + static_cast<int64_t>(n) * P.n_quad + g);
    const double ib_max = __ldg(P.ib_max + n);
    if (k_max <= 0.0 || ib_max <= 0.0) return kErrTransparent;
    r.pref = num / (k_max * ib_max);
  }

  // march() prologue (tracer.cpp:62-77)
  r.tau = 1.0;
  r.q = 0.0;
  r.last_ib2 = r.ib1;
  r.level = 0;
  r.sal = 0;
  r.steps = 0;
  if (!kLean) dda_setup(L, r);
  return kErrNone;
}

struct Fp64Fast {
  double pos[3], dir[3], tn[3], td[3];
  double tau, q, last_ib2, ib1, rib1, pref, t_cur;
  const double4* row;
  int64_t lin;
  int idx[3];
  int band, steps_;
  uint32_t next_draw, ray_id;
  uint64_t h_cell;
  int err;

  __device__ __forceinline__ int init(const TraceParams& P, int64_t cell,
                                      uint32_t ray) {
    Ray r;
    const int e = init_ray(P, cell, ray, r, nullptr);
    if (e != kErrNone) return e;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      pos[a] = r.pos[a];
      dir[a] = r.dir[a];
      tn[a] = r.tn[a];
      td[a] = r.td[a];
      idx[a] = r.idx[a];
    }
    tau = 1.0;
    q = 0.0;
    ib1 = r.ib1;
    last_ib2 = r.ib1;
    rib1 = 1.0 / r.ib1;
    pref = r.pref;
    band = r.band;
    const int64_t ng = (r.krow - P.k) / P.n_temps;
    row = P.iv64 + ng * (P.n_temps - 1);
    steps_ = 0;
    next_draw = r.next_draw;
    ray_id = ray;
    h_cell = r.h_cell;
    lin = cell;
    t_cur = __ldg(P.lv[0].field + cell);
    return kErrNone;
  }

  __device__ __forceinline__ int step(const TraceParams& P, int max_steps) {
    if (tau <= P.tol) return kDone;
    if (steps_ >= max_steps) return kDone;
    const LevelDesc& L = P.lv[0];
    int lo;
    double frac;
    double4 v;  // {k_lo, k_hi, ib_lo, ib_hi}
    if (!fast_lookup(P, row, t_cur, lo, frac, v)) {
      err = kErrTableRange;
      return kFail;
    }

    int axis = 0;
    double ds = tn[0];
    if (tn[1] < ds) {
      ds = tn[1];
      axis = 1;
    }
    if (tn[2] < ds) {
      ds = tn[2];
      axis = 2;
    }
    if (ds < 0.0) ds = 0.0;

    // Next cell, and its temperature prefetched ahead of this step's math.
    int ia = 0, na = 0, sa = 0;
    int64_t stride = 1;
#pragma unroll
    for (int a = 0; a < 3; ++a)
      if (a == axis) {
        sa = dir[a] > 0.0 ? 1 : -1;
        ia = idx[a] + sa;
        na = L.n[a];
        stride = a == 0 ? static_cast<int64_t>(L.n[1]) * L.n[2]
                        : (a == 1 ? static_cast<int64_t>(L.n[2]) : 1);
      }
    const bool inside = ia >= 0 && ia < na;
    int64_t nlin = lin + (sa > 0 ? stride : -stride);
    if (!inside) nlin += (ia < 0 ? 1 : -1) * stride * na;  // periodic image
    double t_next = t_cur;
    if (inside || P.periodic[axis]) t_next = __ldg(L.field + nlin);

    const double kappa = frac == 0.0 ? v.x : v.x + frac * (v.y - v.x);
    const double ib2 = frac == 0.0 ? v.z : v.z + frac * (v.w - v.z);
    const double alpha = -expm1(-kappa * ds);
    last_ib2 = ib2;
    q += P.qe * tau * alpha * div_rcp(ib2 - ib1, ib1, rib1) * pref;
    tau *= 1.0 - alpha;

    const double advance = ds + L.eps;
    pos[0] += advance * dir[0];
    pos[1] += advance * dir[1];
    pos[2] += advance * dir[2];
    tn[0] -= advance;
    tn[1] -= advance;
    tn[2] -= advance;
#pragma unroll
    for (int a = 0; a < 3; ++a)
      if (a == axis) tn[a] += td[a];
    ++steps_;

    if (inside) {
#pragma unroll
      for (int a = 0; a < 3; ++a)
        if (a == axis) idx[a] = ia;
      lin = nlin;
      t_cur = t_next;
      return kContinue;
    }
    if (P.periodic[axis]) {
      const double ext = L.extent[axis];
#pragma unroll
      for (int a = 0; a < 3; ++a)
        if (a == axis) {
          if (ia < 0) {
            idx[a] = na - 1;
            pos[a] += ext;
          } else {
            idx[a] = 0;
            pos[a] -= ext;
          }
        }
      lin = nlin;
      t_cur = t_next;
      return kContinue;
    }
    // Wall exchange, absorption or reflection (tracer.cpp:155-184); the ray
    // stays in its boundary cell, so lin and t_cur are unchanged.
    const bool at_hi = sa > 0;
    const int face = 2 * axis + (at_hi ? 1 : 0);
    const double ew = P.wall_eps[face];
    const double ib_w = __ldg(P.wall_ib + face * P.n_bands + band);
    q += P.qe * tau * ew * div_rcp(ib_w - ib1, ib1, rib1) * pref;
    tau *= 1.0 - ew;
    if (tau <= P.tol) return kDone;
    const double face_pos = L.origin[axis] + (at_hi ? L.extent[axis] : 0.0);
    const int inward = at_hi ? -1 : 1;
    double nd[3] = {dir[0], dir[1], dir[2]};
    if (P.specular) {
#pragma unroll
      for (int a = 0; a < 3; ++a)
        if (a == axis) nd[a] = -nd[a];
    } else {
      const double r1 = draw_u(h_cell, ray_id, next_draw++);
      const double r2 = draw_u(h_cell, ray_id, next_draw++);
      const double sin_t = sqrt(r1);
      const double cos_t = sqrt(1.0 - r1);
      const double phi = 2.0 * kPiD * r2;
      double sp, cp;
      sincos(phi, &sp, &cp);
      const int t1 = axis == 2 ? 0 : axis + 1;
      const int t2 = axis == 0 ? 2 : axis - 1;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        if (a == axis) nd[a] = inward * cos_t;
        if (a == t1) nd[a] = sin_t * cp;
        if (a == t2) nd[a] = sin_t * sp;
      }
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      if (a == axis) pos[a] = face_pos;
      dir[a] = nd[a];
    }
    pos[0] += L.eps * dir[0];
    pos[1] += L.eps * dir[1];
    pos[2] += L.eps * dir[2];
    // Dda::setup (tracer.cpp:17-38)
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const double da = dir[a];
      if (da == 0.0) {
        tn[a] = __longlong_as_double(0x7ff0000000000000LL);
        td[a] = __longlong_as_double(0x7ff0000000000000LL);
        continue;
      }
      const int face_idx = idx[a] + (da > 0.0 ? 1 : 0);
      const double fpos = L.origin[a] + face_idx * L.d[a];
      tn[a] = (fpos - pos[a]) / da;
      td[a] = L.d[a] / fabs(da);
    }
    return kContinue;
  }

  // Residual dump (tracer.cpp:186-188).
  __device__ __forceinline__ double finish(const TraceParams& P) const {
    return q + P.qe * tau * div_rcp(last_ib2 - ib1, ib1, rib1) * pref;
  }
  __device__ __forceinline__ bool finite_state() const { return isfinite(tau); }
  __device__ __forceinline__ int level() const { return 0; }
  __device__ __forceinline__ int sal(const TraceParams&) const { return steps_; }
  __device__ __forceinline__ int steps() const { return steps_; }
};

// ---------------------------------------------------------------------------
// expm1 for the lean tracer: x = j ln2 + r with |r| <= ln2/2 (Cody-Waite with
// fdlibm's split of ln2), e^r - 1 = r + r^2 (1/2 + r/6 + ... + r^11/13!)
// (Taylor to degree 13: truncation < 0.1 ulp), expm1(x) = 2^j (e^r - 1) +
// (2^j - 1). Coefficients come from the constant bank (no per-use 64-bit
// immediates). Within 1 ulp of glibc's expm1 on 5e7 samples of the march's
// argument range (tests/test_oracle.py::test_expm1_restatement), the same
// accuracy class as libdevice's.
__constant__ double kEm1Coef[12] = {
    1.0 / 2, 1.0 / 6, 1.0 / 24, 1.0 / 120, 1.0 / 720, 1.0 / 5040,
    1.0 / 40320, 1.0 / 362880, 1.0 / 3628800, 1.0 / 39916800,
    1.0 / 479001600, 1.0 / 6227020800.0};

// kJ0Path: a separate branch for j = 0 (|x| < ln2 / 2, most steps and
// warp-uniform in practice) that skips the reduction — r = x exactly there
// (fma(0, c, x)), so the bits are the same. Single-level tracers only:
// +0.4 % there, −5.7 % in the larger multigrid kernel (r2ax).
template <bool kJ0Path = false>
__device__ __forceinline__ double expm1_lean(double x) {
  if (!(x >= -40.0 && x <= 0.5)) {
    if (x < -40.0) return -1.0;  // |expm1(x) + 1| < 2^-57
    return expm1(x);             // NaN, positive arguments: libdevice
  }
  const double magic = 6755399441055744.0;  // 1.5 * 2^52
  const double t = fma(x, 1.4426950408889634074, magic);
  const int ji = __double2loint(t);
  if (kJ0Path && ji == 0) {
    double p = kEm1Coef[11];
#pragma unroll
    for (int i = 10; i >= 0; --i) p = fma(p, x, kEm1Coef[i]);
    return fma(x * x, p, x);
  }
  const double j = t - magic;
  double r = fma(j, -6.93147180369123816490e-01, x);
  r = fma(j, -1.90821492927058770002e-10, r);
  double p = kEm1Coef[11];
#pragma unroll
  for (int i = 10; i >= 0; --i) p = fma(p, r, kEm1Coef[i]);
  const double e = fma(r * r, p, r);
  if (!kJ0Path && ji == 0) return e;
  const double sc = __hiloint2double((ji + 1023) << 20, 0);
  return fma(sc, e, sc - 1.0);
}

// Lean single-level fp64 tracer: Fp64Fast's arithmetic (hence the
// reference's) with the per-axis DDA constants in a per-thread shared-memory
// record indexed by the stepping axis:
//   ax[a] = {t_delta (lo, hi words), signed linear stride, cells left before
//            the domain face (or the fixed index of a non-moving axis)}.
// rec[3] = {band, next_draw, cell id, ray id}: state only walls touch.
// kBrick: the temperature gathers read the 2x2x2 micro-brick copy of the
// field (64 bytes per brick, even grids; brick_index in device_common.cuh);
// the stride word then holds the signed index delta of a step that leaves
// the brick ("far"), and the in-brick delta is +-(4 >> axis) with far's sign.
// A step leaves its brick exactly when the cells-left counter is even before
// the step (either direction, even n).
// kPos = false when every wall is black: a ray that reaches a wall then ends
// there (tau *= 1 - 1), so its position is never read again after init and
// the per-step position update (3 multiplies + 3 adds) is dead work.
// kMulti: multigrid ray coarsening (tracer.cpp:91-101): after `cap` steps on
// a level the ray continues on the next coarser one from its current
// position, `locate`d as in geometry.cpp:112-138; the per-axis records and
// the field pointer are then the coarse level's.
constexpr int kLeanRecs64 = 4;

// kReflect = false (every wall black) drops the reflection code; the
// multigrid tracer keeps positions for demotion but can still drop it.
// kCW: the cells are read as cell words (LevelDesc::cellw: the lookup's
// interval and exact offset, precomputed per field) instead of temperatures,
// so a step decodes (lo, frac) with one shift, one mask, one conversion and
// one Markstein quotient instead of running the table lookup.
template <int kHint, bool kBrick, bool kPos = true, bool kMulti = false, bool kReflect = kPos,
          bool kCW = false>
struct Fp64Lean {
  static_assert(!kMulti || (kPos && !kBrick), "demotion reads positions, k-fastest levels");
  static_assert(!kCW || !kBrick, "cell words use the k-fastest layout");
  // kDiet: a black-wall cell-word tracer needs no wall record (the band is
  // row / (n_quad (n_temps - 1))) and stages only the CDF guide tables:
  // 3 per-axis records + guides keep 7 resident blocks inside the 64 KB
  // shared-memory carveout, leaving 192 KB of L1 to the gathers.
  static constexpr bool kDiet = kCW && !kReflect && !kMulti;  // multigrid: measured -0.9 %
  double pos[3], dir[3], tn[3];
  double tau, q, last_ib2, ib1, rib1, pref, t_cur;
  uint64_t w_cur;  // kCW: the current cell's word
  int4* ax;
  int row;  // first interval record of (band, g) in iv64
  int lin;
  // Single level: steps taken. kMulti: steps left of the current level's
  // budget (LevelDesc::budget: until the demotion or max_steps) — one
  // register and one compare per step instead of a step count, a limit and
  // the level's cap read through a per-lane level index.
  int steps_;
  int lvl;  // kMulti: current level
  int err;
  // kMulti: the level's cell words (or temperatures) and eps, from the
  // block's shared copy of the level table (lv_hot; conflict-free: one
  // 16-byte entry per level) instead of the kernel parameters indexed by a
  // per-lane level.
  __device__ __forceinline__ void level_hot(const TraceParams& P, const void*& base,
                                            double& eps) const {
    if (kMulti) {
      const ulonglong2 h = s_lv_hot[lvl];
      base = reinterpret_cast<const void*>(h.x);
      eps = __longlong_as_double(static_cast<long long>(h.y));
    } else {
      base = kCW ? static_cast<const void*>(P.lv[0].cellw) : static_cast<const void*>(P.lv[0].field);
      eps = P.lv[0].eps;
    }
  }

  __device__ __forceinline__ int idx_of(const LevelDesc& L, int a) const {
    const int left = ax[a * kBlock].w;
    if (dir[a] == 0.0) return left;
    return dir[a] > 0.0 ? L.n[a] - 1 - left : left;
  }

  // Dda::setup (tracer.cpp:17-38) + the per-axis records.
  __device__ __forceinline__ void setup(const LevelDesc& L, const int* idx) {
    const int nby = (L.n[1] + 1) >> 1, nbz = (L.n[2] + 1) >> 1;
    const int stride[3] = {kBrick ? 8 * nby * nbz - 4 : L.n[1] * L.n[2],
                           kBrick ? 8 * nbz - 2 : L.n[2], kBrick ? 7 : 1};
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const double da = dir[a];
      if (da == 0.0) {
        tn[a] = __longlong_as_double(0x7ff0000000000000LL);
        ax[a * kBlock] = make_int4(0, 0x7ff00000, 0, idx[a]);
        continue;
      }
      const bool pos_dir = da > 0.0;
      const int face_idx = idx[a] + (pos_dir ? 1 : 0);
      const double face = L.origin[a] + face_idx * L.d[a];
      // (face - pos) / da and d / |da| from one correctly rounded reciprocal
      // (div_rcp returns the correctly rounded quotient, bitwise the IEEE
      // division; |da| >= ~1e-17 here, far from under/overflow).
      const double rda = 1.0 / da;
      tn[a] = div_rcp(face - pos[a], da, rda);
      const double td = div_rcp(L.d[a], fabs(da), fabs(rda));
      ax[a * kBlock] = make_int4(__double2loint(td), __double2hiint(td),
                                 pos_dir ? stride[a] : -stride[a],
                                 pos_dir ? L.n[a] - 1 - idx[a] : idx[a]);
    }
    lin = kBrick ? brick_index(L, idx[0], idx[1], idx[2])
                 : (idx[0] * L.n[1] + idx[1]) * L.n[2] + idx[2];
  }

  __device__ __forceinline__ int init(const TraceParams& P, int64_t cell,
                                      uint32_t ray) {
    extern __shared__ int4 s_dyn[];
    ax = s_dyn + threadIdx.x;
    Ray r;
    const void* staged = !kDiet && P.cdf_smem ? s_dyn + kLeanRecs64 * kBlock : nullptr;
    const uint8_t* guide =
        kDiet && P.cdf_smem ? reinterpret_cast<const uint8_t*>(s_dyn + 3 * kBlock) : nullptr;
    const int e = init_ray<true, kCW>(P, cell, ray, r, nullptr, staged, guide);
    if (e != kErrNone) return e;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      pos[a] = r.pos[a];
      dir[a] = r.dir[a];
    }
    tau = 1.0;
    q = 0.0;
    ib1 = r.ib1;
    last_ib2 = r.ib1;
    rib1 = 1.0 / r.ib1;
    pref = r.pref;
    row = (r.band * P.n_quad + r.quad) * (P.n_temps - 1);
    lvl = 0;
    steps_ = kMulti ? P.lv[0].budget : 0;
    if (!kDiet)
      ax[3 * kBlock] = make_int4(r.band, static_cast<int>(r.next_draw),
                                 static_cast<int>(cell), static_cast<int>(ray));
    if (kCW)
      w_cur = __ldg(P.lv[0].cellw + cell);
    else
      t_cur = __ldg(P.lv[0].field + cell);
    setup(P.lv[0], r.idx);
    return kErrNone;
  }

  // Demotion to the next coarser level (tracer.cpp:91-101): locate the
  // current position there (geometry.cpp:112-138), rebuild the records and
  // load the coarse cell's temperature.
  __device__ __forceinline__ int demote(const TraceParams& P) {
    ++lvl;
    const LevelDesc& C = P.lv[lvl];
    int idx[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const double p = pos[a] + C.eps * dir[a];
      const double rel = div_rcp(p - C.origin[a], C.d[a], C.rd[a]);  // == (p - o) / d
      int i = static_cast<int>(floor(rel));
      if (i < 0 || i >= C.n[a]) {
        if (rel >= -1e-9 && i < 0)
          i = 0;
        else if (rel <= C.n[a] + 1e-9 && i >= C.n[a])
          i = C.n[a] - 1;
        else
          return kErrLocate;
      }
      idx[a] = i;
    }
    steps_ = C.budget;
    setup(C, idx);
    if (kCW)
      w_cur = __ldg(C.cellw + lin);
    else
      t_cur = __ldg(C.field + lin);
    return kErrNone;
  }

  __device__ __forceinline__ int step(const TraceParams& P, int max_steps) {
    if (tau <= P.tol) return kDone;
    if (kMulti) {
      if (steps_ <= 0) {  // the level's budget is spent: demote or stop
        if (!P.lv[lvl].budget_demotes) return kDone;
        const int e = demote(P);
        if (e != kErrNone) {
          err = e;
          return kFail;
        }
      }
    } else if (steps_ >= max_steps) {
      return kDone;
    }
    const LevelDesc& L = P.lv[kMulti ? lvl : 0];
    const void* lbase;
    double leps;
    level_hot(P, lbase, leps);
    int lo;
    double frac;
    double4 v;  // {k_lo, k_hi, ib_lo, ib_hi}
    if (kCW) {
      decode_cw(P, w_cur, lo, frac);
      v = ld_rec64<kHint>(P.iv64 + row + lo);
    } else if (!lookup_spec<kHint>(P, P.iv64 + row, t_cur, lo, frac, v)) {
      err = kErrTableRange;
      return kFail;
    }
    int axis = 0;
    double ds = tn[0];
    if (tn[1] < ds) {
      ds = tn[1];
      axis = 1;
    }
    if (tn[2] < ds) {
      ds = tn[2];
      axis = 2;
    }
    const double t_axis = ds;  // tn[axis]
    if (ds < 0.0) ds = 0.0;

    int4* rp = ax + axis * kBlock;
    const int4 rec = *rp;
    const double td = __hiloint2double(rec.y, rec.x);
    const int left = rec.w - 1;
    const bool inside = left >= 0;
    const bool periodic = (P.periodic_mask >> axis) & 1;
    int nlin;
    if (kBrick) {
      const int near = rec.z > 0 ? (4 >> axis) : -(4 >> axis);
      nlin = lin + ((rec.w & 1) ? near : rec.z);
      if (!inside) {  // periodic image: re-index the wrapped cell
        int idx[3];
#pragma unroll
        for (int a = 0; a < 3; ++a)
          idx[a] = a == axis ? (rec.z > 0 ? 0 : L.n[a] - 1) : idx_of(L, a);
        nlin = brick_index(L, idx[0], idx[1], idx[2]);
      }
    } else {
      nlin = lin + rec.z;
      if (kMulti ? !inside && periodic : !inside) nlin -= rec.z * L.n[axis];  // periodic image
    }
    // The next cell's word (temperature) is loaded straight into w_cur
    // (t_cur): this step's decode has consumed it, so the gather stays in
    // flight until the next step's decode. Loaded into a second register and
    // moved at the end of the step, every step waited for its own gather at
    // the move (ncu r2aj: 14 % of the stall samples). A wall step reloads
    // its own cell.
    const int ld_lin = (inside || periodic) ? nlin : lin;
    if (kCW)
      w_cur = __ldg(static_cast<const uint64_t*>(lbase) + ld_lin);
    else
      t_cur = ld_t64<kHint>((kBrick ? L.field64b : static_cast<const double*>(lbase)) + ld_lin);

    // interp's frac == 0 shortcut (spectral.cpp:179-205) needs no select here:
    // a + 0 * (b - a) == a for finite table values (k is validated finite; a
    // non-finite Ib makes the step non-finite on either form, and such rays
    // are re-traced by the reference-order debug tracer for the error).
    const double kappa = v.x + frac * (v.y - v.x);
    const double ib2 = v.z + frac * (v.w - v.z);
    const double alpha = -expm1_lean<!kMulti>(-kappa * ds);
    last_ib2 = ib2;
    q += P.qe * tau * alpha * div_rcp(ib2 - ib1, ib1, rib1) * pref;
    tau *= 1.0 - alpha;

    const double advance = ds + leps;
    if (kPos) {
      pos[0] += advance * dir[0];
      pos[1] += advance * dir[1];
      pos[2] += advance * dir[2];
    }
    // tn[axis] - advance + td computed once from the selected value (same
    // operands, same bits) instead of three speculative adds and selects
    const double t_new = (t_axis - advance) + td;
#pragma unroll
    for (int a = 0; a < 3; ++a) tn[a] = a == axis ? t_new : tn[a] - advance;
    steps_ += kMulti ? -1 : 1;

    if (inside) {
      rp->w = left;
      lin = nlin;
      return kContinue;
    }
    if (periodic) {
      rp->w = L.n[axis] - 1;
      const double ext = L.extent[axis];
#pragma unroll
      for (int a = 0; a < 3; ++a)
        if (kPos && a == axis) pos[a] += rec.z > 0 ? -ext : ext;
      lin = nlin;
      return kContinue;
    }
    // Wall exchange, absorption or reflection (tracer.cpp:155-184); the ray
    // stays in its boundary cell (its record still says 0 cells left).
    const bool at_hi = rec.z > 0;
    const int face = 2 * axis + (at_hi ? 1 : 0);
    const int4 r3 = kDiet ? make_int4(static_cast<int>(fdiv(static_cast<uint32_t>(row), P.div_row)), 0, 0, 0)
                          : ax[3 * kBlock];
    const double ew = P.wall_eps[face];
    const double ib_w = __ldg(P.wall_ib + face * P.n_bands + r3.x);
    q += P.qe * tau * ew * div_rcp(ib_w - ib1, ib1, rib1) * pref;
    tau *= 1.0 - ew;
    if (tau <= P.tol) return kDone;
    // !kPos: every wall is black, so tau is 0 here unless it is not finite;
    // ending the ray then leaves the report to the pool's finite-state check,
    // and with no reflection code the position and direction are dead after
    // setup (12 registers).
    if constexpr (!kReflect) {
      return kDone;
    } else {
      int idx[3];
#pragma unroll
      for (int a = 0; a < 3; ++a) idx[a] = idx_of(L, a);
      const double face_pos = L.origin[axis] + (at_hi ? L.extent[axis] : 0.0);
      const int inward = at_hi ? -1 : 1;
      double nd[3] = {dir[0], dir[1], dir[2]};
      if (P.specular) {
#pragma unroll
        for (int a = 0; a < 3; ++a)
          if (a == axis) nd[a] = -nd[a];
      } else {
        const uint64_t h_cell = mix64(P.h_seed ^ static_cast<uint64_t>(r3.z));
        const uint32_t ray_id = static_cast<uint32_t>(r3.w);
        const uint32_t draw0 = static_cast<uint32_t>(r3.y);
        const double r1 = draw_u(h_cell, ray_id, draw0);
        const double r2 = draw_u(h_cell, ray_id, draw0 + 1);
        ax[3 * kBlock].y = static_cast<int>(draw0 + 2);
        const double sin_t = sqrt(r1);
        const double cos_t = sqrt(1.0 - r1);
        const double phi = 2.0 * kPiD * r2;
        double sp, cp;
        sincos(phi, &sp, &cp);
        const int t1 = axis == 2 ? 0 : axis + 1;
        const int t2 = axis == 0 ? 2 : axis - 1;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          if (a == axis) nd[a] = inward * cos_t;
          if (a == t1) nd[a] = sin_t * cp;
          if (a == t2) nd[a] = sin_t * sp;
        }
      }
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        if (a == axis) pos[a] = face_pos;
        dir[a] = nd[a];
      }
      pos[0] += L.eps * dir[0];
      pos[1] += L.eps * dir[1];
      pos[2] += L.eps * dir[2];
      setup(L, idx);
      return kContinue;
    }
  }

  __device__ __forceinline__ double finish(const TraceParams& P) const {
    return q + P.qe * tau * div_rcp(last_ib2 - ib1, ib1, rib1) * pref;
  }
  __device__ __forceinline__ bool finite_state() const { return isfinite(tau); }
  __device__ __forceinline__ int level() const { return kMulti ? lvl : 0; }
  // Steps on the final level: every level below took exactly its cap.
  __device__ __forceinline__ int sal(const TraceParams& P) const {
    return kMulti ? P.lv[lvl].budget - steps_ : steps_;
  }
  __device__ __forceinline__ int steps() const { return steps_; }  // single level
};

struct Fp64Tracer {
  Ray r;
  int err;
  __device__ __forceinline__ int init(const TraceParams& P, int64_t cell,
                                      uint32_t ray) {
    return init_ray(P, cell, ray, r, nullptr);
  }
  template <bool kMulti>
  __device__ __forceinline__ int step_t(const TraceParams& P, int max_steps) {
    return march_step<kMulti, false>(P, r, max_steps, nullptr, &err);
  }
  __device__ __forceinline__ double finish(const TraceParams& P) const {
    return finish_ray(P, r);
  }
  __device__ __forceinline__ bool finite_state() const {
    return isfinite(r.tau);
  }
  __device__ __forceinline__ int level() const { return r.level; }
  __device__ __forceinline__ int sal(const TraceParams&) const { return r.sal; }
  __device__ __forceinline__ int steps() const { return r.steps; }
};
struct Fp64Multi : Fp64Tracer {
  __device__ __forceinline__ int step(const TraceParams& P, int m) {
    return step_t<true>(P, m);
  }
};


// K1: persistent ray-pool trace over the chunk's (cell, ray) work items.
// kMulti = false: the fast single-level tracer; true: the reference-order
// tracer with multigrid demotion (also used for single-node tables).
// kMinBlocks trades registers for occupancy (tuned on B200).
template <bool kMulti, int kMinBlocks>
__global__ void __launch_bounds__(kBlock, kMinBlocks)
    trace_pool_fp64(const __grid_constant__ TraceParams P) {
  if (kMulti)
    pool_kernel_body<Fp64Multi, true>(P);
  else
    pool_kernel_body<Fp64Fast, false>(P);
}

template <int kMinBlocks, int kHint, bool kBrick, bool kPos = true, bool kCW = false,
          int kInner = 0>
__global__ void __launch_bounds__(kBlock, kMinBlocks)
    trace_pool_fp64_lean(const __grid_constant__ TraceParams P) {
  extern __shared__ int4 s_dyn[];
  if (P.cdf_smem) {
    if (kCW && !kPos)  // Fp64Lean::kDiet
      stage_guides(P, reinterpret_cast<uint8_t*>(s_dyn + 3 * kBlock));
    else
      stage_sampling(P, s_dyn + kLeanRecs64 * kBlock);
  }
  pool_kernel_body<Fp64Lean<kHint, kBrick, kPos, false, kPos, kCW>, false, kInner>(P);
}

// Multigrid variant of the lean tracer (n_levels > 1).
template <int kMinBlocks, bool kReflect = true, bool kCW = false, int kInner = 0>
__global__ void __launch_bounds__(kBlock, kMinBlocks)
    trace_pool_fp64_lean_mg(const __grid_constant__ TraceParams P) {
  extern __shared__ int4 s_dyn[];
  stage_sampling(P, s_dyn + kLeanRecs64 * kBlock);
  stage_level_hot(P, kCW ? kLvCellWords : kLvField);
  pool_kernel_body<Fp64Lean<0, false, true, true, kReflect, kCW>, true, kInner>(P);
}

// Cell words of one level (TraceParams::cw_*), with the reference lookup
// (t_lookup, spectral.cpp:148-177) and a per-cell check that the tracer's
// decode returns exactly its (lo, frac); *bad is set if any cell does not
// fit (the solve then keeps the temperature-reading tracers).
__global__ void build_cell_words(const __grid_constant__ TraceParams P,
                                 const double* __restrict__ field, int64_t n, double scale,
                                 uint64_t* __restrict__ out, int* __restrict__ bad) {
  bool all_ok = true;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double T = field[i];
    int lo = 0;
    double frac = 0.0;
    bool ok = t_lookup(P, T, lo, frac) && lo < (1 << (64 - kCwShift));
    uint64_t w = 0;
    if (ok) {
      const double ms = (T - __ldg(P.temps + lo)) * scale;  // exact power-of-two scaling
      ok = ms >= 0.0 && ms < 9007199254740992.0 && ms == floor(ms);
      if (ok) {
        const uint64_t m = static_cast<uint64_t>(ms);
        w = (static_cast<uint64_t>(lo) << kCwShift) | m;
        int dlo;
        double dfrac;
        decode_cw(P, w, dlo, dfrac);
        ok = (m >> kCwShift) == 0 && dlo == lo && dfrac == frac;
      }
    }
    out[i] = w;
    all_ok = all_ok && ok;
  }
  if (__any_sync(kFull, !all_ok) && (threadIdx.x & 31) == 0) atomicOr(bad, 1);
}

// Copies the fp64 k-fastest field into the 2x2x2 micro-brick layout.
__global__ void to_bricked64(const double* __restrict__ src, double* __restrict__ dst,
                             int nx, int ny, int nz) {
  const int64_t n = static_cast<int64_t>(nx) * ny * nz;
  const int nby = (ny + 1) >> 1, nbz = (nz + 1) >> 1;
  for (int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; c < n;
       c += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int i = static_cast<int>(c / (static_cast<int64_t>(ny) * nz));
    const int j = static_cast<int>((c / nz) % ny);
    const int k = static_cast<int>(c % nz);
    const int64_t b = ((static_cast<int64_t>(i >> 1) * nby + (j >> 1)) * nbz + (k >> 1)) * 8 +
                      ((i & 1) << 2) + ((j & 1) << 1) + (k & 1);
    dst[b] = src[c];
  }
}

// Debug/test kernel: one thread traces one explicit ray with full
// bookkeeping (weights, termination, per-level steps).
__global__ void trace_rays_fp64(const __grid_constant__ TraceParams P,
                                int64_t n, const int64_t* cells,
                                const uint32_t* ray_ids, const double* dirs,
                                RayRecord* out, int64_t* level_steps) {
  const int64_t s = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (s >= n) return;
  Ray r;
  DebugRec dbg;
  dbg.w_abs = dbg.w_walls = 0.0;
  dbg.reflections = 0;
  dbg.term = 0;
  dbg.err_value = 0.0;
  dbg.err_axis = -1;
  for (int l = 0; l < kMaxLevels; ++l) dbg.level_steps[l] = 0;
  RayRecord rec;
  rec.err = kErrNone;
  rec.err_value = 0.0;
  rec.err_axis = -1;
  int e = init_ray(P, cells[s], ray_ids[s], r, dirs ? dirs + 3 * s : nullptr);
  if (e != kErrNone) {
    rec.err = e;
    if (e == kErrTableRange) rec.err_value = __ldg(P.lv[0].field + cells[s]);
    out[s] = rec;
    return;
  }
  rec.dir[0] = r.dir[0];
  rec.dir[1] = r.dir[1];
  rec.dir[2] = r.dir[2];
  rec.prefactor = r.pref;
  rec.ib_source = r.ib1;
  // The reference's RayState leaves init_ray with next_draw = 4 (7 with
  // volume sampling); march consumes reflection draws on its own copy.
  rec.next_draw = r.next_draw;
  const int max_steps = static_cast<int>(
      P.max_steps < 0x7fffffffLL ? P.max_steps : 0x7fffffffLL);
  int st, err = 0;
  const bool multi = P.n_levels > 1;
  do {
    st = multi ? march_step<true, true>(P, r, max_steps, &dbg, &err)
               : march_step<false, true>(P, r, max_steps, &dbg, &err);
  } while (st == kContinue);
  rec.steps = r.steps;
  rec.band = r.band;
  rec.quad = static_cast<int32_t>(
      (r.krow - P.k) / P.n_temps - static_cast<int64_t>(r.band) * P.n_quad);
  rec.reflections = dbg.reflections;
  rec.term = dbg.term;
  if (st == kFail) {
    rec.err = err;
    rec.err_value = dbg.err_value;
    rec.err_axis = dbg.err_axis;
    rec.q = r.q;
  } else {
    rec.q = finish_ray(P, r);
  }
  rec.w_abs = dbg.w_abs;
  rec.w_walls = dbg.w_walls;
  rec.w_res = r.tau;
  out[s] = rec;
  if (level_steps)
    for (int l = 0; l < P.n_levels; ++l)
      level_steps[s * P.n_levels + l] = dbg.level_steps[l];
}

// Per-ray API (ermc_b200_init_rays / _march_rays / _sample_direction /
// _absorptivity): the reference's init_ray, march, sample_direction and
// absorptivity (sampling.cpp:31-96, tracer.cpp:11-194) on explicit rays,
// with the debug tracer's reference-order arithmetic.
__global__ void init_states_fp64(const __grid_constant__ TraceParams P, int64_t n,
                                 const int32_t* __restrict__ cells,
                                 const uint32_t* __restrict__ ray_ids, uint64_t seed,
                                 ermc_ray_state_t* __restrict__ out, int32_t* __restrict__ err) {
  const int64_t s = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (s >= n) return;
  const LevelDesc& L = P.lv[0];
  const int64_t cell =
      (static_cast<int64_t>(cells[3 * s]) * L.n[1] + cells[3 * s + 1]) * L.n[2] + cells[3 * s + 2];
  Ray r;
  const int e = init_ray(P, cell, ray_ids[s], r, nullptr);
  err[s] = e;
  if (e != kErrNone) return;
  ermc_ray_state_t o;
  for (int a = 0; a < 3; ++a) {
    o.pos[a] = r.pos[a];
    o.dir[a] = r.dir[a];
    o.cell[a] = r.idx[a];
  }
  o.cell[3] = 0;
  o.transmissivity = 1.0;
  o.band = r.band;
  o.quad = r.quad;
  o.prefactor = r.pref;
  o.ib_source = r.ib1;
  o.reflections = 0;
  o.reserved0 = 0;
  o.seed = seed;
  o.cell_id = static_cast<uint64_t>(cell);
  o.ray_id = ray_ids[s];
  o.next_draw = r.next_draw;
  out[s] = o;
}

__global__ void march_states_fp64(const __grid_constant__ TraceParams P, int64_t n,
                                  const ermc_ray_state_t* __restrict__ in,
                                  RayRecord* __restrict__ out, int64_t* level_steps) {
  const int64_t s = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (s >= n) return;
  const ermc_ray_state_t st = in[s];
  Ray r;
  for (int a = 0; a < 3; ++a) {
    r.pos[a] = st.pos[a];
    r.dir[a] = st.dir[a];
    r.idx[a] = st.cell[a];
  }
  r.level = st.cell[3];
  r.tau = st.transmissivity;
  r.q = 0.0;
  r.ib1 = st.ib_source;
  r.last_ib2 = st.ib_source;  // degenerate termination dumps zero (tracer.cpp:67)
  r.pref = st.prefactor;
  r.band = st.band;
  r.quad = st.quad;
  r.krow = P.k + (static_cast<int64_t>(st.band) * P.n_quad + st.quad) * P.n_temps;
  r.ibrow = P.ib + static_cast<int64_t>(st.band) * P.n_temps;
  r.sal = 0;
  r.steps = 0;
  r.h_cell = mix64(mix64(st.seed + 0x9e3779b97f4a7c15ULL) ^ st.cell_id);
  r.ray_id = st.ray_id;
  r.next_draw = st.next_draw;
  dda_setup(P.lv[r.level], r);
  DebugRec dbg;
  dbg.w_abs = dbg.w_walls = 0.0;
  dbg.reflections = 0;
  dbg.term = 0;
  dbg.err_value = 0.0;
  dbg.err_axis = -1;
  for (int l = 0; l < kMaxLevels; ++l) dbg.level_steps[l] = 0;
  const int max_steps = static_cast<int>(
      P.max_steps < 0x7fffffffLL ? P.max_steps : 0x7fffffffLL);
  int stt, e = 0;
  const bool multi = P.n_levels > 1;
  do {
    stt = multi ? march_step<true, true>(P, r, max_steps, &dbg, &e)
                : march_step<false, true>(P, r, max_steps, &dbg, &e);
  } while (stt == kContinue);
  RayRecord rec;
  rec.err = stt == kFail ? e : kErrNone;
  rec.err_value = dbg.err_value;
  rec.err_axis = dbg.err_axis;
  rec.q = stt == kFail ? r.q : finish_ray(P, r);
  rec.w_abs = dbg.w_abs;
  rec.w_walls = dbg.w_walls;
  rec.w_res = r.tau;
  for (int a = 0; a < 3; ++a) rec.dir[a] = r.dir[a];
  rec.prefactor = r.pref;
  rec.ib_source = r.ib1;
  rec.steps = r.steps;
  rec.term = dbg.term;
  rec.reflections = dbg.reflections;
  rec.band = r.band;
  rec.quad = r.quad;
  rec.next_draw = r.next_draw;
  out[s] = rec;
  if (level_steps)
    for (int l = 0; l < P.n_levels; ++l) level_steps[s * P.n_levels + l] = dbg.level_steps[l];
}

__global__ void sample_direction_kernel(int64_t n, const double* __restrict__ rt,
                                        const double* __restrict__ rp, double* __restrict__ out) {
  const int64_t s = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (s >= n) return;
  // sampling.cpp:31-40, the operations of init_ray above
  const double cos_t = 1.0 - 2.0 * rt[s];
  const double phi = 2.0 * kPiD * rp[s];
  const double sin_t = sqrt(fmax(0.0, 1.0 - cos_t * cos_t));
  double sp, cp;
  sincos(phi, &sp, &cp);
  out[5 * s + 0] = acos(cos_t);
  out[5 * s + 1] = phi;
  out[5 * s + 2] = sin_t * cp;
  out[5 * s + 3] = sin_t * sp;
  out[5 * s + 4] = cos_t;
}

__global__ void absorptivity_kernel(int64_t n, const double* __restrict__ k,
                                    const double* __restrict__ ds, double* __restrict__ out) {
  const int64_t s = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (s >= n) return;
  out[s] = -expm1(-k[s] * ds[s]);  // the march's alpha (tracer.cpp:118)
}

// K2: per-cell tally in ray-id order (reference solver.cpp:142-155).
__device__ __forceinline__ void tally_cell(const double* __restrict__ q_ray, int64_t n_cells,
                                           int rays, int64_t c, double& sum, double& sd) {
  double mean = 0.0, m2 = 0.0;
  sum = 0.0;
  for (int r = 0; r < rays; ++r) {
    const double x = q_ray[static_cast<int64_t>(r) * n_cells + c];
    sum += x;
    const double delta = x - mean;
    mean += delta / (r + 1);
    m2 += delta * (x - mean);
  }
  sd = rays > 1 ? sqrt(m2 * rays / (rays - 1.0)) : 0.0;
}

__global__ void reduce_cells(const double* __restrict__ q_ray, int64_t n_cells,
                             int rays, double* __restrict__ q_r,
                             double* __restrict__ std_dev) {
  const int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (c >= n_cells) return;
  double sum, sd;
  tally_cell(q_ray, n_cells, rays, c, sum, sd);
  q_r[c] = sum;
  std_dev[c] = sd;
}

// K2 with the all-gather fused in: each cell's (Q_r, sigma) is stored into
// every listed full-field buffer — this GPU's and its peers' (CUDA IPC
// mappings; NVLink stores on a B200 node) — at its global index `base + c`,
// so no collective follows the solve.
__global__ void reduce_cells_scatter(const double* __restrict__ q_ray, int64_t n_cells,
                                     int rays, ScatterOut out, int64_t base) {
  const int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (c >= n_cells) return;
  double sum, sd;
  tally_cell(q_ray, n_cells, rays, c, sum, sd);
  for (int p = 0; p < out.n; ++p) {
    out.q[p][base + c] = sum;
    out.sd[p][base + c] = sd;
  }
}

// K3: block-mean restriction (reference geometry.cpp:51-82), one thread per
// coarse cell, fine cells summed in the reference's i, j, k loop order.
__global__ void restrict_field(const double* __restrict__ fine, int fnx,
                               int fny, int fnz, int ratio,
                               double* __restrict__ coarse, int cnx, int cny,
                               int cnz) {
  const int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int64_t n = static_cast<int64_t>(cnx) * cny * cnz;
  if (c >= n) return;
  const int ci = static_cast<int>(c / (static_cast<int64_t>(cny) * cnz));
  const int cj = static_cast<int>((c / cnz) % cny);
  const int ck = static_cast<int>(c % cnz);
  double sum = 0.0;
  int count = 0;
  for (int i = ci * ratio; i < min((ci + 1) * ratio, fnx); ++i)
    for (int j = cj * ratio; j < min((cj + 1) * ratio, fny); ++j)
      for (int k = ck * ratio; k < min((ck + 1) * ratio, fnz); ++k) {
        sum += fine[(static_cast<int64_t>(i) * fny + j) * fnz + k];
        ++count;
      }
  coarse[c] = sum / count;
}

// Field statistics for validation and T_max (solver.cpp:27-58,
// geometry.cpp:34-49): min, max and the count of values failing v > 0.
__global__ void field_stats_partial(const double* __restrict__ t, int64_t n,
                                    double* __restrict__ pmin,
                                    double* __restrict__ pmax,
                                    unsigned long long* __restrict__ pbad) {
  double mn = __longlong_as_double(0x7ff0000000000000LL);
  double mx = -mn;
  unsigned long long bad = 0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
       i < n; i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double v = t[i];
    if (!(v > 0.0)) ++bad;
    mn = fmin(mn, v);
    mx = fmax(mx, v);
  }
  __shared__ double smn[32], smx[32];
  __shared__ unsigned long long sbad[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mn = fmin(mn, __shfl_xor_sync(kFull, mn, o));
    mx = fmax(mx, __shfl_xor_sync(kFull, mx, o));
    bad += __shfl_xor_sync(kFull, bad, o);
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    smn[w] = mn;
    smx[w] = mx;
    sbad[w] = bad;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < (blockDim.x >> 5); ++i) {
      mn = fmin(mn, smn[i]);
      mx = fmax(mx, smx[i]);
      bad += sbad[i];
    }
    pmin[blockIdx.x] = mn;
    pmax[blockIdx.x] = mx;
    pbad[blockIdx.x] = bad;
  }
}

__global__ void field_stats_final(const double* pmin, const double* pmax,
                                  const unsigned long long* pbad, int nb,
                                  double* out3) {
  if (threadIdx.x != 0) return;
  double mn = pmin[0], mx = pmax[0];
  unsigned long long bad = 0;
  for (int i = 0; i < nb; ++i) {
    mn = fmin(mn, pmin[i]);
    mx = fmax(mx, pmax[i]);
    bad += pbad[i];
  }
  out3[0] = mn;
  out3[1] = mx;
  out3[2] = static_cast<double>(bad);
}

// Packed fp64 tables for the fast tracer (copies of reference values).
__global__ void build_iv64(const double* __restrict__ k,
                           const double* __restrict__ ib, int nb, int nq,
                           int nt, double4* __restrict__ iv) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int64_t n_iv = static_cast<int64_t>(nb) * nq * (nt - 1);
  if (i >= n_iv) return;
  const int t = static_cast<int>(i % (nt - 1));
  const int64_t ng = i / (nt - 1);
  const int n = static_cast<int>(ng / nq);
  const double* krow = k + ng * nt;
  const double* ibrow = ib + static_cast<int64_t>(n) * nt;
  iv[i] = make_double4(krow[t], krow[t + 1], ibrow[t], ibrow[t + 1]);
}

__global__ void uniform_kernel(uint64_t h_seed, int64_t n,
                               const uint64_t* cells, const uint32_t* rays,
                               const uint32_t* draws, double* out) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  out[i] = draw_u(mix64(h_seed ^ cells[i]), rays[i], draws[i]);
}

}  // namespace

// ---- host launchers -------------------------------------------------------

int trace_fp64_block() { return kBlock; }

namespace {
// Kernel variant by (path, min blocks per SM); 4 or 5 blocks of 128 threads.
using TraceFn = void (*)(TraceParams);
bool lean_path(const TraceParams& P) {
  return P.n_temps >= 2 && P.lean &&
         P.lv[0].n[0] * static_cast<int64_t>(P.lv[0].n[1]) * P.lv[0].n[2] < (1LL << 31);
}
size_t fp64_smem(const TraceParams& P) {
  if (!lean_path(P)) return 0;
  if (P.cellw && !P.track_pos && P.n_levels == 1)  // Fp64Lean::kDiet: 3 records + guides
    return 3 * kBlock * sizeof(int4) + (P.cdf_smem ? cdf_guide_bytes(P.n_bands) : 0);
  return kLeanRecs64 * kBlock * sizeof(int4) + cdf_stage_bytes(P.cdf_smem, P.n_bands, P.n_quad);
}
// min_blocks = 0 picks the measured best per variant (B200, 256^3 channel):
// 8 blocks/SM for the black-wall tracer (64 registers + 128 B of L1-resident
// spills in the refill path beat 6 blocks / 80 registers by 12 %; 9, 10, 12
// blocks lose again: 0.98, 0.89, 0.77x of 8),
// 7 for the position-tracking tracer (grey walls, 256^3 eps = 0.5: +7 % over
// 6), 6 for the multigrid tracer (7 measured no better).
TraceFn fp64_kernel_p(const TraceParams& P, int min_blocks) {
  if (!lean_path(P)) return nullptr;
  const bool brick = P.brick && P.lv[0].field64b;
  // cell-word tracers: 7 blocks/SM (72 registers) beat 8 (64) by 3 % (r2e)
  if (min_blocks <= 0)
    min_blocks = P.n_levels > 1 ? (P.track_pos ? 6 : 7) : !P.track_pos ? (P.cellw ? 7 : 8) : 7;
  min_blocks = min(max(min_blocks, 6), 8);
  if (P.cellw) {
    if (P.n_levels > 1) {
      if (!P.track_pos && min_blocks == 7 && P.inner_steps == 64)  // 6+ levels' window
        return trace_pool_fp64_lean_mg<7, false, true, 64>;
      if (!P.track_pos)
        return min_blocks >= 8   ? trace_pool_fp64_lean_mg<8, false, true>
               : min_blocks == 7 ? trace_pool_fp64_lean_mg<7, false, true>
                                 : trace_pool_fp64_lean_mg<6, false, true>;
      return min_blocks >= 7 ? trace_pool_fp64_lean_mg<7, true, true>
                             : trace_pool_fp64_lean_mg<6, true, true>;
    }
    if (!P.track_pos) {
      // the bench kernel with its default window compiled in (kInner = 32)
      if (min_blocks == 7 && P.inner_steps == 32)
        return trace_pool_fp64_lean<7, 0, false, false, true, 32>;
      return min_blocks == 8   ? trace_pool_fp64_lean<8, 0, false, false, true>
             : min_blocks == 7 ? trace_pool_fp64_lean<7, 0, false, false, true>
                               : trace_pool_fp64_lean<6, 0, false, false, true>;
    }
    return min_blocks == 8   ? trace_pool_fp64_lean<8, 0, false, true, true>
           : min_blocks == 7 ? trace_pool_fp64_lean<7, 0, false, true, true>
                             : trace_pool_fp64_lean<6, 0, false, true, true>;
  }
  if (P.n_levels > 1) {
    if (!P.track_pos)  // black walls: no reflection code
      return min_blocks >= 8   ? trace_pool_fp64_lean_mg<8, false>
             : min_blocks == 7 ? trace_pool_fp64_lean_mg<7, false>
                               : trace_pool_fp64_lean_mg<6, false>;
    return min_blocks >= 7 ? trace_pool_fp64_lean_mg<7> : trace_pool_fp64_lean_mg<6>;
  }
  if (!P.track_pos) {
    if (brick) return trace_pool_fp64_lean<8, 0, true, false>;
    return min_blocks == 8   ? trace_pool_fp64_lean<8, 0, false, false>
           : min_blocks == 7 ? trace_pool_fp64_lean<7, 0, false, false>
                             : trace_pool_fp64_lean<6, 0, false, false>;
  }
  if (brick) return trace_pool_fp64_lean<7, 0, true>;
  return min_blocks == 8   ? trace_pool_fp64_lean<8, 0, false>
         : min_blocks == 7 ? trace_pool_fp64_lean<7, 0, false>
                           : trace_pool_fp64_lean<6, 0, false>;
}
TraceFn fp64_kernel(bool multi, int min_blocks) {
  if (min_blocks <= 0) min_blocks = 5;
  if (multi) return min_blocks >= 5 ? trace_pool_fp64<true, 5> : trace_pool_fp64<true, 4>;
  return min_blocks >= 5 ? trace_pool_fp64<false, 5> : trace_pool_fp64<false, 4>;
}
}  // namespace

bool fp64_fast_path(const TraceParams& P) {
  return P.n_levels == 1 && P.n_temps >= 2;
}

int trace_fp64_blocks_per_sm(const TraceParams& P, int min_blocks) {
  int nb = 0;
  TraceFn k = fp64_kernel_p(P, min_blocks);
  if (!k) k = fp64_kernel(!fp64_fast_path(P), min_blocks);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k, kBlock, fp64_smem(P));
  return nb;
}

cudaError_t launch_trace_fp64(const TraceParams& P, int grid, int min_blocks,
                              cudaStream_t stream) {
  TraceFn k = fp64_kernel_p(P, min_blocks);
  if (!k) k = fp64_kernel(!fp64_fast_path(P), min_blocks);
  set_trace_carveout(reinterpret_cast<const void*>(k), grid, fp64_smem(P), P.carveout);
  k<<<grid, kBlock, fp64_smem(P), stream>>>(P);
  return cudaGetLastError();
}

cudaError_t launch_trace_rays_fp64(const TraceParams& P, int64_t n,
                                   const int64_t* cells,
                                   const uint32_t* ray_ids, const double* dirs,
                                   RayRecord* out, int64_t* level_steps,
                                   cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  const int block = 64;
  const int64_t grid = (n + block - 1) / block;
  trace_rays_fp64<<<static_cast<unsigned>(grid), block, 0, stream>>>(
      P, n, cells, ray_ids, dirs, out, level_steps);
  return cudaGetLastError();
}

cudaError_t launch_init_states_fp64(const TraceParams& P, int64_t n, const int32_t* cells,
                                    const uint32_t* ray_ids, uint64_t seed,
                                    ermc_ray_state_t* out, int32_t* err, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  init_states_fp64<<<static_cast<unsigned>((n + 63) / 64), 64, 0, stream>>>(P, n, cells, ray_ids,
                                                                            seed, out, err);
  return cudaGetLastError();
}

cudaError_t launch_march_states_fp64(const TraceParams& P, int64_t n,
                                     const ermc_ray_state_t* in, RayRecord* out,
                                     int64_t* level_steps, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  march_states_fp64<<<static_cast<unsigned>((n + 63) / 64), 64, 0, stream>>>(P, n, in, out,
                                                                             level_steps);
  return cudaGetLastError();
}

cudaError_t launch_sample_direction(int64_t n, const double* rt, const double* rp, double* out,
                                    cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  sample_direction_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, stream>>>(n, rt, rp,
                                                                                      out);
  return cudaGetLastError();
}

cudaError_t launch_absorptivity(int64_t n, const double* k, const double* ds, double* out,
                                cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  absorptivity_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, stream>>>(n, k, ds, out);
  return cudaGetLastError();
}

cudaError_t launch_reduce_cells_scatter(const double* q_ray, int64_t n_cells, int rays,
                                        const ScatterOut& out, int64_t base,
                                        cudaStream_t stream) {
  if (n_cells <= 0) return cudaSuccess;
  const int block = 256;
  reduce_cells_scatter<<<static_cast<unsigned>((n_cells + block - 1) / block), block, 0,
                         stream>>>(q_ray, n_cells, rays, out, base);
  return cudaGetLastError();
}

cudaError_t launch_reduce_cells(const double* q_ray, int64_t n_cells, int rays,
                                double* q_r, double* std_dev,
                                cudaStream_t stream) {
  if (n_cells <= 0) return cudaSuccess;
  const int block = 256;
  reduce_cells<<<static_cast<unsigned>((n_cells + block - 1) / block), block, 0,
                 stream>>>(q_ray, n_cells, rays, q_r, std_dev);
  return cudaGetLastError();
}

cudaError_t launch_restrict(const double* fine, int fnx, int fny, int fnz,
                            int ratio, double* coarse, int cnx, int cny,
                            int cnz, cudaStream_t stream) {
  const int64_t n = static_cast<int64_t>(cnx) * cny * cnz;
  const int block = 256;
  restrict_field<<<static_cast<unsigned>((n + block - 1) / block), block, 0,
                   stream>>>(fine, fnx, fny, fnz, ratio, coarse, cnx, cny, cnz);
  return cudaGetLastError();
}

// scratch: 3 * n_blocks values; out3 device [min, max, bad]
cudaError_t launch_field_stats(const double* t, int64_t n, double* scratch,
                               int n_blocks, double* out3,
                               cudaStream_t stream) {
  double* pmin = scratch;
  double* pmax = scratch + n_blocks;
  auto* pbad = reinterpret_cast<unsigned long long*>(scratch + 2 * n_blocks);
  field_stats_partial<<<n_blocks, 256, 0, stream>>>(t, n, pmin, pmax, pbad);
  field_stats_final<<<1, 32, 0, stream>>>(pmin, pmax, pbad, n_blocks, out3);
  return cudaGetLastError();
}

cudaError_t launch_to_bricked64(const double* src, double* dst, int nx, int ny, int nz,
                                cudaStream_t stream) {
  const int64_t n = static_cast<int64_t>(nx) * ny * nz;
  if (n <= 0) return cudaSuccess;
  const int64_t want = (n + 255) / 256;
  to_bricked64<<<static_cast<unsigned>(want < 4096 ? want : 4096), 256, 0, stream>>>(
      src, dst, nx, ny, nz);
  return cudaGetLastError();
}

cudaError_t launch_build_iv64(const double* k, const double* ib, int nb, int nq,
                              int nt, double4* iv, cudaStream_t stream) {
  const int64_t n = static_cast<int64_t>(nb) * nq * (nt - 1);
  if (n <= 0) return cudaSuccess;
  build_iv64<<<static_cast<unsigned>((n + 255) / 256), 256, 0, stream>>>(
      k, ib, nb, nq, nt, iv);
  return cudaGetLastError();
}

cudaError_t launch_build_cell_words(const TraceParams& P, const double* field, int64_t n,
                                    double scale, uint64_t* out, int* bad,
                                    cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  const int64_t want = (n + 255) / 256;
  build_cell_words<<<static_cast<unsigned>(want < 8192 ? want : 8192), 256, 0, stream>>>(
      P, field, n, scale, out, bad);
  return cudaGetLastError();
}

cudaError_t launch_uniform(uint64_t h_seed, int64_t n, const uint64_t* cells,
                           const uint32_t* rays, const uint32_t* draws,
                           double* out, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  const int block = 256;
  uniform_kernel<<<static_cast<unsigned>((n + block - 1) / block), block, 0,
                   stream>>>(h_seed, n, cells, rays, draws, out);
  return cudaGetLastError();
}

}  // namespace ermc_dev
