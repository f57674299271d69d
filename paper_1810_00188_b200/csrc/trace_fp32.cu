// trace_fp32.cu — fast variant of the ERMC trace kernel (precision = fp32).
//
// Same work decomposition, RNG keys and (band, g) sampling as the fp64
// kernel (every ray is the reference's ray: the draws and the CDF
// inversion stay exact), but the march runs in fp32 with a layout built
// for the gather roofline:
//   * T as fp32 (64 MiB at 256^3: L2-resident on a 126 MB L2);
//   * one 16-byte float4 per (band, g, T-interval):
//       {k_lo, k_hi - k_lo, ibn_lo, ibn_hi - ibn_lo},  ibn = Ib / Ib(T_last)
//     so a step is one 4-byte T gather + one 16-byte table load (the 20 B/step
//     of BASELINE.md's roofline);
//   * Amanatides-Woo in absolute ray parameters (one add per step), with
//     the running position re-based at wraps/reflections;
//   * the reciprocal exchange accumulated as tau*alpha*(ibn2 - ibn1) and
//     scaled once per ray by QE * k1/k_max * Ib(T_last)/Ib_max (in fp64).
// Parity contract: statistical — per cell within 3 sigma of the fp64 path
// (north_star), total steps within 1e-3.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "device_common.cuh"
#include "trace_common.cuh"

namespace ermc_dev {

namespace {

constexpr int kBlock32 = 128;

// 1 - exp(-x) for x >= 0: Taylor near 0 (no cancellation), ex2 otherwise.
// Both forms evaluated and selected: lanes of a warp straddle 0.125.
__device__ __forceinline__ float absorb32(float x) {
  const float big = 1.0f - __expf(-x);
  float p = fmaf(x, -1.0f / 120.0f, 1.0f / 24.0f);
  p = fmaf(x, -p, 1.0f / 6.0f);
  p = fmaf(x, -p, 0.5f);
  p = fmaf(x, -p, 1.0f);
  return x < 0.125f ? x * p : big;
}

// locate (geometry.cpp:112-138) of a demoted ray on level C, axis a. The
// reference nudges the position by eps * dir (1e-12 of a cell) so that a
// ray sitting on a coarse face — every other fine face it crosses — lands in
// the cell it is moving into; in fp32 that nudge is below resolution, so a
// coordinate within 8 ulps of a face is resolved by the direction instead
// (otherwise the ray would take an extra zero-length step back across it).
__device__ __forceinline__ int locate32(const LevelDesc& C, int a, float p, float d) {
  const float rel = (p - static_cast<float>(C.origin[a])) / static_cast<float>(C.d[a]);
  const float fl = floorf(rel);
  const float fr = rel - fl;
  const float tie = 8.0f * 1.1920929e-7f * fmaxf(fabsf(rel), 1.0f);
  int i = static_cast<int>(fl);
  if (d > 0.0f && fr > 1.0f - tie) ++i;
  else if (d < 0.0f && fr < tie) --i;
  return min(max(i, 0), C.n[a] - 1);
}

// Sampling CDFs staged after the lean kernels' 3 x kBlock32 per-axis records.
constexpr int kRecs32 = 3;
__device__ __forceinline__ const void* staged_cdf(const TraceParams& P) {
  extern __shared__ int4 s_dyn[];
  return P.cdf_smem ? s_dyn + kRecs32 * kBlock32 : nullptr;
}
__device__ __forceinline__ void stage_cdfs32(const TraceParams& P) {
  extern __shared__ int4 s_dyn[];
  stage_sampling(P, s_dyn + kRecs32 * kBlock32);
}

struct Fp32Tracer {
  float p0[3];   // position at s = 0
  float dir[3];
  float tn[3];   // absolute ray parameter of the next face on each axis
  float td[3];
  float s;       // current ray parameter
  float tau, acc, ib1n, last_ib2n;
  double cq;     // QE * k1/k_max * Ib(T_last)/Ib_max  (per ray)
  const float4* row;
  int idx[3], stp[3];
  int lin;       // linear index of the current cell
  float t_cur;   // its temperature (prefetched one step ahead)
  int band, lvl, sal_, steps_;
  uint32_t next_draw, ray_id;
  uint64_t h_cell;
  int err;

  __device__ __forceinline__ void setup(const LevelDesc& L) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const float da = dir[a];
      if (da == 0.0f) {
        tn[a] = __int_as_float(0x7f800000);
        td[a] = __int_as_float(0x7f800000);
        stp[a] = 0;
        continue;
      }
      const float inv = 1.0f / da;
      stp[a] = da > 0.0f ? 1 : -1;
      const float face = static_cast<float>(
          L.origin[a] + (idx[a] + (da > 0.0f ? 1 : 0)) * L.d[a]);
      tn[a] = (face - p0[a]) * inv;
      td[a] = static_cast<float>(L.d[a]) * fabsf(inv);
    }
    s = 0.0f;
    lin = (idx[0] * L.n[1] + idx[1]) * L.n[2] + idx[2];
  }

  // Position at the current parameter; re-base so s = 0.
  __device__ __forceinline__ void rebase() {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      p0[a] = fmaf(s, dir[a], p0[a]);
      tn[a] -= s;
    }
    s = 0.0f;
  }

  // cdf: sampling CDFs staged in shared memory by the lean kernels, or null.
  __device__ __forceinline__ int init(const TraceParams& P, int64_t cell,
                                      uint32_t ray, const void* cdf = nullptr) {
    const LevelDesc& L = P.lv[0];
    int ci, cj, ck;
    decode_cell(P, cell, ci, cj, ck);
    h_cell = mix64(P.h_seed ^ static_cast<uint64_t>(cell));
    ray_id = ray;
    const double r_theta = draw_u(h_cell, ray, 0);
    const double r_phi = draw_u(h_cell, ray, 1);
    const double r_n = draw_u(h_cell, ray, 2);
    const double r_g = draw_u(h_cell, ray, 3);
    next_draw = 4;
    const float cos_t = static_cast<float>(1.0 - 2.0 * r_theta);
    const float sin_t = sqrtf(fmaxf(0.0f, 1.0f - cos_t * cos_t));
    float sp, cp;
    sincospif(static_cast<float>(2.0 * r_phi), &sp, &cp);
    dir[0] = sin_t * cp;
    dir[1] = sin_t * sp;
    dir[2] = cos_t;
    int n, g;
    sample_band_staged(P, cdf, r_n, r_g, n, g);
    band = n;
    const int nt1 = P.n_temps - 1;
    row = P.iv32 + (static_cast<int64_t>(n) * P.n_quad + g) * nt1;
    idx[0] = ci;
    idx[1] = cj;
    idx[2] = ck;
    double pos[3] = {L.origin[0] + (ci + 0.5) * L.d[0],
                     L.origin[1] + (cj + 0.5) * L.d[1],
                     L.origin[2] + (ck + 0.5) * L.d[2]};
    if (P.volume_sampling) {
#pragma unroll
      for (int a = 0; a < 3; ++a)
        pos[a] += (draw_u(h_cell, ray, next_draw++) - 0.5) * L.d[a];
    }
    p0[0] = static_cast<float>(pos[0]);
    p0[1] = static_cast<float>(pos[1]);
    p0[2] = static_cast<float>(pos[2]);
    const float t_cell = __ldg(L.field32 + cell);
    float u = fmaf(t_cell, P.inv_dt32, -P.t0_32 * P.inv_dt32);
    int lo = min(max(static_cast<int>(u), 0), nt1 - 1);
    const float f = u - static_cast<float>(lo);
    const float4 v = __ldg(row + lo);
    const float k1 = fmaf(f, v.y, v.x);
    ib1n = fmaf(f, v.w, v.z);
    last_ib2n = ib1n;
    const double kmax = __ldg(P.k_max + static_cast<int64_t>(n) * P.n_quad + g);
    const double ibmax = __ldg(P.ib_max + n);
    if (kmax <= 0.0 || ibmax <= 0.0) return kErrTransparent;
    // R_I / Ib1 * QE with Ib normalised by Ib(T_last): see file header.
    const double ib_last = __ldg(P.ib + static_cast<int64_t>(n) * P.n_temps + nt1);
    cq = P.qe * static_cast<double>(k1) / kmax * (ib_last / ibmax);
    tau = 1.0f;
    acc = 0.0f;
    lvl = 0;
    sal_ = 0;
    steps_ = 0;
    setup(L);
    t_cur = t_cell;
    return kErrNone;
  }

  template <bool kMulti>
  __device__ __forceinline__ int step_t(const TraceParams& P, int max_steps) {
    if (tau <= P.tol32) return kDone;
    if (steps_ >= max_steps) return kDone;
    if (kMulti) {
      const int cap = P.lv[lvl].cap;
      if (cap >= 0 && sal_ >= cap && lvl + 1 < P.n_levels) {
        ++lvl;
        const LevelDesc& C = P.lv[lvl];
        rebase();
#pragma unroll
        for (int a = 0; a < 3; ++a) idx[a] = locate32(C, a, p0[a], dir[a]);
        sal_ = 0;
        setup(C);
        t_cur = __ldg(C.field32 + lin);
      }
    }
    const LevelDesc& L = P.lv[kMulti ? lvl : 0];
    // table record of the current cell (its T arrived during the last step)
    const float u = fmaf(t_cur, P.inv_dt32, -P.t0_32 * P.inv_dt32);
    const int lo = min(max(static_cast<int>(u), 0), P.n_temps - 2);
    const float f = u - static_cast<float>(lo);
    const float4 v = __ldg(row + lo);

    int axis = 0;
    float tmin = tn[0];
    if (tn[1] < tmin) {
      tmin = tn[1];
      axis = 1;
    }
    if (tn[2] < tmin) {
      tmin = tn[2];
      axis = 2;
    }
    const float ds = fmaxf(tmin - s, 0.0f);
    s = fmaxf(tmin, s);

    // next cell; its T is fetched now, ahead of this step's math
    int ia = 0, na = 0, sa = 0, stride = 1;
#pragma unroll
    for (int a = 0; a < 3; ++a)
      if (a == axis) {
        sa = stp[a];
        ia = idx[a] + sa;
        na = L.n[a];
        stride = a == 0 ? L.n[1] * L.n[2] : (a == 1 ? L.n[2] : 1);
        tn[a] += td[a];
      }
    const bool inside = ia >= 0 && ia < na;
    int nlin = lin + (sa > 0 ? stride : -stride);
    if (!inside) nlin += (ia < 0 ? 1 : -1) * stride * na;  // periodic image
    float t_next = t_cur;
    if (inside || P.periodic[axis]) t_next = __ldg(L.field32 + nlin);

    const float kappa = fmaf(f, v.y, v.x);
    const float ib2n = fmaf(f, v.w, v.z);
    const float alpha = absorb32(kappa * ds);
    last_ib2n = ib2n;
    const float ta = tau * alpha;
    acc = fmaf(ta, ib2n - ib1n, acc);
    tau -= ta;
    ++steps_;
    if (kMulti) ++sal_;

    if (inside) {
#pragma unroll
      for (int a = 0; a < 3; ++a)
        if (a == axis) idx[a] = ia;
      lin = nlin;
      t_cur = t_next;
      return kContinue;
    }
    if (P.periodic[axis]) {
      rebase();
      const float ext = static_cast<float>(L.extent[axis]);
#pragma unroll
      for (int a = 0; a < 3; ++a)
        if (a == axis) {
          if (ia < 0) {
            idx[a] = na - 1;
            p0[a] += ext;
          } else {
            idx[a] = 0;
            p0[a] -= ext;
          }
        }
      lin = nlin;
      t_cur = t_next;
      return kContinue;
    }

    // wall exchange (tracer.cpp:155-165); the ray stays in its cell
    const bool at_hi = sa > 0;
    const int face = 2 * axis + (at_hi ? 1 : 0);
    const float ew = static_cast<float>(P.wall_eps[face]);
    const float ibw = __ldg(P.wall_ibn32 + face * P.n_bands + band);
    const float tw = tau * ew;
    acc = fmaf(tw, ibw - ib1n, acc);
    tau -= tw;
    if (tau <= P.tol32) return kDone;
    // reflection (tracer.cpp:167-182)
    rebase();
    const float face_pos = static_cast<float>(
        L.origin[axis] + (at_hi ? L.extent[axis] : 0.0));
    float nd[3] = {dir[0], dir[1], dir[2]};
    if (P.specular) {
#pragma unroll
      for (int a = 0; a < 3; ++a)
        if (a == axis) nd[a] = -nd[a];
    } else {
      const double r1 = draw_u(h_cell, ray_id, next_draw++);
      const double r2 = draw_u(h_cell, ray_id, next_draw++);
      const float sin_t = sqrtf(static_cast<float>(r1));
      const float cos_t = sqrtf(static_cast<float>(1.0 - r1));
      float sp, cp;
      sincospif(static_cast<float>(2.0 * r2), &sp, &cp);
      const int t1 = axis == 2 ? 0 : axis + 1;
      const int t2 = axis == 0 ? 2 : axis - 1;
      const float inward = at_hi ? -1.0f : 1.0f;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        if (a == axis) nd[a] = inward * cos_t;
        if (a == t1) nd[a] = sin_t * cp;
        if (a == t2) nd[a] = sin_t * sp;
      }
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      if (a == axis) p0[a] = face_pos;
      dir[a] = nd[a];
    }
    setup(L);
    return kContinue;
  }

  __device__ __forceinline__ double finish(const TraceParams&) const {
    const float a = fmaf(tau, last_ib2n - ib1n, acc);
    return cq * static_cast<double>(a);
  }
  __device__ __forceinline__ bool finite_state() const {
    return isfinite(tau) && isfinite(acc);
  }
  __device__ __forceinline__ int level() const { return lvl; }
  __device__ __forceinline__ int sal(const TraceParams&) const { return sal_; }
  __device__ __forceinline__ int steps() const { return steps_; }
};

// Lean single-level tracer: the per-axis constants of the DDA live in a
// per-thread shared-memory record indexed by the stepping axis,
//   ax[a] = {t_delta (float bits), signed linear stride, cells left before
//            the domain face, wrap delta (-stride * n) or the fixed index of
//            a non-moving axis},
// so one LDS.128 replaces the predicated per-axis selects and param-space
// loads of a register-only DDA; `lin` carries the cell index.
// kMulti: multigrid ray coarsening (tracer.cpp:91-101) with Fp32Tracer's
// demotion arithmetic; the records and field pointer then follow the level.
// kReflect = false (every wall black): no reflection code.
template <int kHint, bool kMulti = false, bool kReflect = true>
struct Fp32Lean {
  // multigrid level counters in 64-bit registers: measured ~3 % faster here
  static constexpr bool kWideLevelSteps = true;
  float p0[3], dir[3], tn[3];
  float s, tau, acc, ib1n, last_ib2n, t_cur;
  double cq;
  const float4* row;
  int4* ax;  // &s_ax[0][threadIdx.x]; axis a at ax[a * kBlock32]
  int lin, band, steps_;
  // kMulti: current level, and min(demotion step, max_steps) (Fp64Lean)
  int lvl, limit_;
  uint32_t next_draw, ray_id;
  uint64_t h_cell;
  int err;

  __device__ __forceinline__ int idx_of(const LevelDesc& L, int a) const {
    const int4 r = ax[a * kBlock32];
    if (dir[a] == 0.0f) return r.w;
    return dir[a] > 0.0f ? L.n[a] - 1 - r.z : r.z;
  }

  __device__ __forceinline__ void setup(const LevelDesc& L, const int* idx) {
    const int stride[3] = {L.n[1] * L.n[2], L.n[2], 1};
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const float da = dir[a];
      if (da == 0.0f) {
        tn[a] = __int_as_float(0x7f800000);
        ax[a * kBlock32] = make_int4(0x7f800000, 0, 0x7fffffff, idx[a]);
        continue;
      }
      const float inv = 1.0f / da;
      const bool pos = da > 0.0f;
      const float face =
          static_cast<float>(L.origin[a] + (idx[a] + (pos ? 1 : 0)) * L.d[a]);
      tn[a] = (face - p0[a]) * inv;
      const float td = static_cast<float>(L.d[a]) * fabsf(inv);
      const int dl = pos ? stride[a] : -stride[a];
      ax[a * kBlock32] = make_int4(__float_as_int(td), dl,
                                   pos ? L.n[a] - 1 - idx[a] : idx[a], -dl * L.n[a]);
    }
    s = 0.0f;
    lin = (idx[0] * L.n[1] + idx[1]) * L.n[2] + idx[2];
  }

  __device__ __forceinline__ void rebase() {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      p0[a] = fmaf(s, dir[a], p0[a]);
      tn[a] -= s;
    }
    s = 0.0f;
  }

  __device__ __forceinline__ int init(const TraceParams& P, int64_t cell,
                                      uint32_t ray) {
    extern __shared__ int4 s_dyn[];
    ax = s_dyn + threadIdx.x;
    Fp32Tracer base;
    const int e = base.init(P, cell, ray, staged_cdf(P));
    if (e != kErrNone) return e;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      p0[a] = base.p0[a];
      dir[a] = base.dir[a];
    }
    tau = 1.0f;
    acc = 0.0f;
    ib1n = base.ib1n;
    last_ib2n = base.ib1n;
    cq = base.cq;
    row = base.row;
    band = base.band;
    steps_ = 0;
    lvl = 0;
    if (kMulti) limit_ = level_limit(P, 0);
    next_draw = base.next_draw;
    ray_id = ray;
    h_cell = base.h_cell;
    t_cur = base.t_cur;
    setup(P.lv[0], base.idx);
    return kErrNone;
  }

  // Demotion to the next coarser level (Fp32Tracer::step_t's arithmetic).
  __device__ __forceinline__ void demote(const TraceParams& P) {
    ++lvl;
    const LevelDesc& C = P.lv[lvl];
    rebase();
    int idx[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) idx[a] = locate32(C, a, p0[a], dir[a]);
    limit_ = level_limit(P, lvl);
    setup(C, idx);
    t_cur = __ldg(C.field32 + lin);
  }

  __device__ __forceinline__ int level_limit(const TraceParams& P, int l) const {
    const int ms = static_cast<int>(P.max_steps < 0x7fffffffLL ? P.max_steps : 0x7fffffffLL);
    const int cap = P.lv[l].cap;
    if (cap < 0 || l + 1 >= P.n_levels) return ms;
    const long long d = static_cast<long long>(steps_) + cap;
    return d < ms ? static_cast<int>(d) : ms;
  }

  __device__ __forceinline__ int step(const TraceParams& P, int max_steps) {
    if (tau <= P.tol32) return kDone;
    if (kMulti) {
      if (steps_ >= limit_) {
        if (steps_ >= max_steps) return kDone;
        demote(P);
      }
    } else if (steps_ >= max_steps) {
      return kDone;
    }
    const LevelDesc& L = P.lv[kMulti ? lvl : 0];
    // kMulti: the level's fp32 field from the block's level table (s_lv_hot)
    const float* field32 =
        kMulti ? reinterpret_cast<const float*>(s_lv_hot[lvl].x) : P.lv[0].field32;
    // table record of the current cell (its T arrived during the last step)
    const float u = fmaf(t_cur, P.inv_dt32, P.u0_32);
    const int lo = min(static_cast<int>(u), P.n_temps - 2);
    const float f = u - static_cast<float>(lo);
    const float4 v = ld_rec32<kHint>(row + lo);

    int axis = 0;
    float tmin = tn[0];
    if (tn[1] < tmin) {
      tmin = tn[1];
      axis = 1;
    }
    if (tn[2] < tmin) {
      tmin = tn[2];
      axis = 2;
    }
    const float ds = fmaxf(tmin - s, 0.0f);
    s = fmaxf(tmin, s);

    int4* rp = ax + axis * kBlock32;
    const int4 r = *rp;
    const float td = __int_as_float(r.x);
#pragma unroll
    for (int a = 0; a < 3; ++a)
      if (a == axis) tn[a] += td;
    const int left = r.z - 1;
    const bool inside = left >= 0;
    const int nlin = lin + r.y + (inside ? 0 : r.w);  // periodic image if outside
    // next cell's temperature straight into t_cur (see Fp64Lean::step)
    t_cur = ld_t32<kHint>(field32 + ((inside || P.periodic[axis]) ? nlin : lin));

    const float kappa = fmaf(f, v.y, v.x);
    const float ib2n = fmaf(f, v.w, v.z);
    const float alpha = absorb32(kappa * ds);
    last_ib2n = ib2n;
    const float ta = tau * alpha;
    acc = fmaf(ta, ib2n - ib1n, acc);
    tau -= ta;
    ++steps_;

    if (inside) {
      rp->z = left;
      lin = nlin;
      return kContinue;
    }
    if (P.periodic[axis]) {
      rp->z = L.n[axis] - 1;
      rebase();
      const float ext = static_cast<float>(L.extent[axis]);
#pragma unroll
      for (int a = 0; a < 3; ++a)
        if (a == axis) p0[a] += r.y > 0 ? -ext : ext;
      lin = nlin;
      return kContinue;
    }
    // wall exchange (tracer.cpp:155-165); the ray stays in its cell
    const bool at_hi = r.y > 0;
    const int face = 2 * axis + (at_hi ? 1 : 0);
    const float ew = static_cast<float>(P.wall_eps[face]);
    const float ibw = __ldg(P.wall_ibn32 + face * P.n_bands + band);
    const float tw = tau * ew;
    acc = fmaf(tw, ibw - ib1n, acc);
    tau -= tw;
    if (tau <= P.tol32) return kDone;
    if constexpr (!kReflect) {  // black walls: tau is 0 here unless non-finite
      return kDone;
    } else {
      // reflection (tracer.cpp:167-182)
      int idx[3];
#pragma unroll
      for (int a = 0; a < 3; ++a) idx[a] = idx_of(L, a);  // rp->z still 0: the boundary cell
      rebase();
      const float face_pos =
          static_cast<float>(L.origin[axis] + (at_hi ? L.extent[axis] : 0.0));
      float nd[3] = {dir[0], dir[1], dir[2]};
      if (P.specular) {
#pragma unroll
        for (int a = 0; a < 3; ++a)
          if (a == axis) nd[a] = -nd[a];
      } else {
        const double r1 = draw_u(h_cell, ray_id, next_draw++);
        const double r2 = draw_u(h_cell, ray_id, next_draw++);
        const float sin_t = sqrtf(static_cast<float>(r1));
        const float cos_t = sqrtf(static_cast<float>(1.0 - r1));
        float sp, cp;
        sincospif(static_cast<float>(2.0 * r2), &sp, &cp);
        const int t1 = axis == 2 ? 0 : axis + 1;
        const int t2 = axis == 0 ? 2 : axis - 1;
        const float inward = at_hi ? -1.0f : 1.0f;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          if (a == axis) nd[a] = inward * cos_t;
          if (a == t1) nd[a] = sin_t * cp;
          if (a == t2) nd[a] = sin_t * sp;
        }
      }
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        if (a == axis) p0[a] = face_pos;
        dir[a] = nd[a];
      }
      setup(L, idx);
      return kContinue;
    }
  }

  __device__ __forceinline__ double finish(const TraceParams&) const {
    return cq * static_cast<double>(fmaf(tau, last_ib2n - ib1n, acc));
  }
  __device__ __forceinline__ bool finite_state() const {
    return isfinite(tau) && isfinite(acc);
  }
  __device__ __forceinline__ int level() const { return kMulti ? lvl : 0; }
  // Steps on the final level: every level below took exactly its cap.
  __device__ __forceinline__ int sal(const TraceParams& P) const {
    int s = steps_;
    if (kMulti)
      for (int l = 0; l < lvl; ++l) s -= P.lv[l].cap;
    return s;
  }
  __device__ __forceinline__ int steps() const { return steps_; }
};

// Micro-brick variant of the lean tracer (grids with even dimensions): the
// fp32 field is stored in 2x2x2 bricks (one 32-byte sector each) and the
// per-axis record carries the two signed index deltas of a step,
//   rec[a] = {t_delta bits, cells left before the face, delta inside a brick,
//             delta across a brick face}   (moving axis)
//            {inf, INT_MAX, 0, fixed index}                 (non-moving axis).
// With even n a step leaves its brick exactly when the cells-left counter is
// even before the step, for either direction.
// kPos = false when every wall is black: a wall hit ends the ray, so the
// position (p0) and direction are dead after setup and periodic re-basing
// only shifts the ray parameter (frees 6 registers; see Fp64Lean).
// kB: brick edge (2: 2x2x2 bricks = one 32-byte sector; 4: 4x4x4 = 256 B).
template <int kHint, bool kPos = true, int kB = 2>
struct Fp32Brick {
  float p0[3], dir[3], tn[3];
  float s, tau, acc, ib1n, last_ib2n, t_cur;
  double cq;
  const float4* row;
  // Per-axis records in two shared arrays so no access conflicts on banks:
  //   axr[a] = {t_delta bits, cross-brick delta "far"}  (8 B: one LDS.64)
  //            {inf, fixed index}                        (non-moving axis)
  //   axl[a] = cells left before the face               (4 B, read + written)
  // The in-brick delta is +-(4 >> a) with far's sign.
  int2* axr;
  int* axl;
  int lin, band, steps_;
  uint32_t next_draw, ray_id;
  uint64_t h_cell;
  int err;

  __device__ __forceinline__ int idx_of(const LevelDesc& L, int a) const {
    if (dir[a] == 0.0f) return axr[a * kBlock32].y;
    const int left = axl[a * kBlock32];
    return dir[a] > 0.0f ? L.n[a] - 1 - left : left;
  }

  __device__ __forceinline__ void setup(const LevelDesc& L, const int* idx) {
    constexpr int kV = kB * kB * kB;
    const int nby = L.n[1] / kB, nbz = L.n[2] / kB;
    const int bs[3] = {nby * nbz, nbz, 1};
    const int sn[3] = {kB * kB, kB, 1};
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const float da = dir[a];
      if (da == 0.0f) {
        tn[a] = __int_as_float(0x7f800000);
        axr[a * kBlock32] = make_int2(0x7f800000, idx[a]);
        axl[a * kBlock32] = 0x7fffffff;
        continue;
      }
      const float inv = 1.0f / da;
      const bool up = da > 0.0f;
      const float face =
          static_cast<float>(L.origin[a] + (idx[a] + (up ? 1 : 0)) * L.d[a]);
      tn[a] = (face - p0[a]) * inv;
      const float td = static_cast<float>(L.d[a]) * fabsf(inv);
      const int far = up ? kV * bs[a] - (kB - 1) * sn[a] : (kB - 1) * sn[a] - kV * bs[a];
      axr[a * kBlock32] = make_int2(__float_as_int(td), far);
      axl[a * kBlock32] = up ? L.n[a] - 1 - idx[a] : idx[a];
    }
    s = 0.0f;
    lin = brick_index_b<kB>(L, idx[0], idx[1], idx[2]);
  }

  __device__ __forceinline__ void rebase() {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      if (kPos) p0[a] = fmaf(s, dir[a], p0[a]);
      tn[a] -= s;
    }
    s = 0.0f;
  }

  __device__ __forceinline__ int init(const TraceParams& P, int64_t cell,
                                      uint32_t ray) {
    extern __shared__ int4 s_dyn[];
    axr = reinterpret_cast<int2*>(s_dyn) + threadIdx.x;
    axl = reinterpret_cast<int*>(reinterpret_cast<int2*>(s_dyn) + 3 * kBlock32) + threadIdx.x;
    Fp32Tracer base;
    const int e = base.init(P, cell, ray, staged_cdf(P));
    if (e != kErrNone) return e;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      p0[a] = base.p0[a];
      dir[a] = base.dir[a];
    }
    tau = 1.0f;
    acc = 0.0f;
    ib1n = base.ib1n;
    last_ib2n = base.ib1n;
    cq = base.cq;
    row = base.row;
    band = base.band;
    steps_ = 0;
    next_draw = base.next_draw;
    ray_id = ray;
    h_cell = base.h_cell;
    t_cur = base.t_cur;  // the same value as the brick copy's
    setup(P.lv[0], base.idx);
    return kErrNone;
  }

  __device__ __forceinline__ int step(const TraceParams& P, int max_steps) {
    if (tau <= P.tol32) return kDone;
    if (steps_ >= max_steps) return kDone;
    const LevelDesc& L = P.lv[0];
    const float u = fmaf(t_cur, P.inv_dt32, P.u0_32);
    const int lo = min(static_cast<int>(u), P.n_temps - 2);
    const float f = u - static_cast<float>(lo);
    const float4 v = ld_rec32<kHint>(row + lo);

    int axis = 0;
    float tmin = tn[0];
    if (tn[1] < tmin) {
      tmin = tn[1];
      axis = 1;
    }
    if (tn[2] < tmin) {
      tmin = tn[2];
      axis = 2;
    }
    const float ds = fmaxf(tmin - s, 0.0f);
    s = fmaxf(tmin, s);

    const int2 r = axr[axis * kBlock32];
    int* lp = axl + axis * kBlock32;
    const int left0 = *lp;
    const float td = __int_as_float(r.x);
    const int far = r.y;
#pragma unroll
    for (int a = 0; a < 3; ++a)
      if (a == axis) tn[a] += td;
    const int left = left0 - 1;
    const bool inside = left >= 0;
    const bool periodic = (P.periodic_mask >> axis) & 1;
    // the step leaves its brick when the cells-left counter is a multiple of kB
    const int near = kB == 2 ? (4 >> axis) : (16 >> (2 * axis));
    int nlin = lin + ((left0 & (kB - 1)) ? (far > 0 ? near : -near) : far);
    if (!inside && periodic) {
      int idx[3];
#pragma unroll
      for (int a = 0; a < 3; ++a)
        idx[a] = a == axis ? (far > 0 ? 0 : L.n[a] - 1) : idx_of(L, a);
      nlin = brick_index_b<kB>(L, idx[0], idx[1], idx[2]);
    }
    // next cell's temperature straight into t_cur (see Fp64Lean::step)
    t_cur = ld_t32<kHint>(L.field32b + ((inside || periodic) ? nlin : lin));

    const float kappa = fmaf(f, v.y, v.x);
    const float ib2n = fmaf(f, v.w, v.z);
    const float alpha = absorb32(kappa * ds);
    last_ib2n = ib2n;
    const float ta = tau * alpha;
    acc = fmaf(ta, ib2n - ib1n, acc);
    tau -= ta;
    ++steps_;

    if (inside) {
      *lp = left;
      lin = nlin;
      return kContinue;
    }
    if (periodic) {
      *lp = L.n[axis] - 1;
      rebase();
      const float ext = static_cast<float>(L.extent[axis]);
#pragma unroll
      for (int a = 0; a < 3; ++a)
        if (kPos && a == axis) p0[a] += far > 0 ? -ext : ext;
      lin = nlin;
      return kContinue;
    }
    // wall exchange (tracer.cpp:155-165); the ray stays in its cell
    const bool at_hi = far > 0;
    const int face = 2 * axis + (at_hi ? 1 : 0);
    const float ew = static_cast<float>(P.wall_eps[face]);
    const float ibw = __ldg(P.wall_ibn32 + face * P.n_bands + band);
    const float tw = tau * ew;
    acc = fmaf(tw, ibw - ib1n, acc);
    tau -= tw;
    if (tau <= P.tol32) return kDone;
    if constexpr (!kPos) {  // black walls: tau is 0 here unless non-finite
      return kDone;
    } else {
      // reflection (tracer.cpp:167-182)
      int idx[3];
#pragma unroll
      for (int a = 0; a < 3; ++a) idx[a] = idx_of(L, a);  // left still 0: the boundary cell
      rebase();
      const float face_pos =
          static_cast<float>(L.origin[axis] + (at_hi ? L.extent[axis] : 0.0));
      float nd[3] = {dir[0], dir[1], dir[2]};
      if (P.specular) {
#pragma unroll
        for (int a = 0; a < 3; ++a)
          if (a == axis) nd[a] = -nd[a];
      } else {
        const double r1 = draw_u(h_cell, ray_id, next_draw++);
        const double r2 = draw_u(h_cell, ray_id, next_draw++);
        const float sin_t = sqrtf(static_cast<float>(r1));
        const float cos_t = sqrtf(static_cast<float>(1.0 - r1));
        float sp, cp;
        sincospif(static_cast<float>(2.0 * r2), &sp, &cp);
        const int t1 = axis == 2 ? 0 : axis + 1;
        const int t2 = axis == 0 ? 2 : axis - 1;
        const float inward = at_hi ? -1.0f : 1.0f;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          if (a == axis) nd[a] = inward * cos_t;
          if (a == t1) nd[a] = sin_t * cp;
          if (a == t2) nd[a] = sin_t * sp;
        }
      }
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        if (a == axis) p0[a] = face_pos;
        dir[a] = nd[a];
      }
      setup(L, idx);
      return kContinue;
    }
  }

  __device__ __forceinline__ double finish(const TraceParams&) const {
    return cq * static_cast<double>(fmaf(tau, last_ib2n - ib1n, acc));
  }
  __device__ __forceinline__ bool finite_state() const {
    return isfinite(tau) && isfinite(acc);
  }
  __device__ __forceinline__ int level() const { return 0; }
  __device__ __forceinline__ int sal(const TraceParams&) const { return steps_; }
  __device__ __forceinline__ int steps() const { return steps_; }
};

template <int kMinBlocks, int kHint, bool kPos = true, int kB = 2, int kInner = 0>
__global__ void __launch_bounds__(kBlock32, kMinBlocks)
    trace_pool_fp32_brick(const __grid_constant__ TraceParams P) {
  stage_cdfs32(P);
  pool_kernel_body<Fp32Brick<kHint, kPos, kB>, false, kInner>(P);
}

// Converts the fp64 k-fastest field to the fp32 micro-brick layout (edge b).
__global__ void to_fp32_bricked(const double* __restrict__ src, float* __restrict__ dst,
                                int nx, int ny, int nz, int b) {
  const int64_t n = static_cast<int64_t>(nx) * ny * nz;
  const int nby = ny / b, nbz = nz / b;
  for (int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; c < n;
       c += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int i = static_cast<int>(c / (static_cast<int64_t>(ny) * nz));
    const int j = static_cast<int>((c / nz) % ny);
    const int k = static_cast<int>(c % nz);
    const int64_t idx = ((static_cast<int64_t>(i / b) * nby + (j / b)) * nbz + (k / b)) * (b * b * b) +
                        ((i % b) * b + (j % b)) * b + (k % b);
    dst[idx] = static_cast<float>(src[c]);
  }
}

template <int kMinBlocks, int kHint>
__global__ void __launch_bounds__(kBlock32, kMinBlocks)
    trace_pool_fp32_lean(const __grid_constant__ TraceParams P) {
  stage_cdfs32(P);
  pool_kernel_body<Fp32Lean<kHint>, false>(P);
}

// Multigrid variant of the lean tracer (n_levels > 1).
template <int kMinBlocks, bool kReflect = true>
__global__ void __launch_bounds__(kBlock32, kMinBlocks)
    trace_pool_fp32_lean_mg(const __grid_constant__ TraceParams P) {
  stage_cdfs32(P);
  stage_level_hot(P, kLvField32);
  pool_kernel_body<Fp32Lean<0, true, kReflect>, true>(P);
}

struct Fp32Multi : Fp32Tracer {
  __device__ __forceinline__ int step(const TraceParams& P, int m) {
    return step_t<true>(P, m);
  }
};

// Multigrid variant (levels > 1): the register-DDA tracer with demotion.
template <int kMinBlocks>
__global__ void __launch_bounds__(kBlock32, kMinBlocks)
    trace_pool_fp32(const __grid_constant__ TraceParams P) {
  pool_kernel_body<Fp32Multi, true>(P);
}

// {k_lo, k_hi - k_lo, ibn_lo, ibn_hi - ibn_lo} per (band, g, interval),
// ibn = Ib / Ib(n, T_last).
__global__ void build_iv32(const double* __restrict__ k,
                           const double* __restrict__ ib, int nb, int nq,
                           int nt, float4* __restrict__ iv) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int64_t n_iv = static_cast<int64_t>(nb) * nq * (nt - 1);
  if (i >= n_iv) return;
  const int t = static_cast<int>(i % (nt - 1));
  const int64_t ng = i / (nt - 1);
  const int n = static_cast<int>(ng / nq);
  const double* krow = k + ng * nt;
  const double* ibrow = ib + static_cast<int64_t>(n) * nt;
  const double ilast = ibrow[nt - 1];
  const double s = ilast > 0.0 ? 1.0 / ilast : 0.0;
  const double b0 = ibrow[t] * s, b1 = ibrow[t + 1] * s;
  iv[i] = make_float4(static_cast<float>(krow[t]),
                      static_cast<float>(krow[t + 1] - krow[t]),
                      static_cast<float>(b0), static_cast<float>(b1 - b0));
}

__global__ void to_fp32(const double* __restrict__ src, float* __restrict__ dst,
                        int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
       i < n; i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    dst[i] = static_cast<float>(src[i]);
}

}  // namespace

int trace_fp32_block() { return kBlock32; }

namespace {
using TraceFn32 = void (*)(TraceParams);
bool fp32_lean(const TraceParams& P) { return P.lean != 0; }
size_t fp32_smem(const TraceParams& P) {
  if (!fp32_lean(P)) return 0;
  return kRecs32 * kBlock32 * sizeof(int4) +
         cdf_stage_bytes(P.cdf_smem, P.n_bands, P.n_quad);
}
TraceFn32 fp32_kernel(const TraceParams& P, int min_blocks) {
  // 8 blocks/SM (64 registers) measured best; 10 and 12 lose (0.98, 0.92x).
  const bool eight = min_blocks >= 8;
  if (fp32_lean(P) && P.n_levels > 1) {
    if (!P.track_pos) return eight ? trace_pool_fp32_lean_mg<8, false> : trace_pool_fp32_lean_mg<6, false>;
    return eight ? trace_pool_fp32_lean_mg<8> : trace_pool_fp32_lean_mg<6>;
  }
  if (fp32_lean(P) && P.brick) {
    if (!P.track_pos && P.brick == 4) return trace_pool_fp32_brick<8, 0, false, 4>;
    if (!P.track_pos) {
      if (eight && P.inner_steps == 48)  // the default window compiled in
        return trace_pool_fp32_brick<8, 0, false, 2, 48>;
      return eight ? trace_pool_fp32_brick<8, 0, false> : trace_pool_fp32_brick<6, 0, false>;
    }
    return eight ? trace_pool_fp32_brick<8, 0> : trace_pool_fp32_brick<6, 0>;
  }
  if (fp32_lean(P)) return eight ? trace_pool_fp32_lean<8, 0> : trace_pool_fp32_lean<6, 0>;
  return eight ? trace_pool_fp32<8> : trace_pool_fp32<6>;
}
}  // namespace

int trace_fp32_blocks_per_sm(const TraceParams& P, int min_blocks) {
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fp32_kernel(P, min_blocks), kBlock32,
                                                fp32_smem(P));
  return nb;
}

cudaError_t launch_trace_fp32(const TraceParams& P, int grid, int min_blocks,
                              cudaStream_t stream) {
  const auto k = fp32_kernel(P, min_blocks);
  set_trace_carveout(reinterpret_cast<const void*>(k), grid, fp32_smem(P), P.carveout);
  k<<<grid, kBlock32, fp32_smem(P), stream>>>(P);
  return cudaGetLastError();
}

cudaError_t launch_build_iv32(const double* k, const double* ib, int nb, int nq,
                              int nt, float4* iv, cudaStream_t stream) {
  const int64_t n = static_cast<int64_t>(nb) * nq * (nt - 1);
  if (n <= 0) return cudaSuccess;
  build_iv32<<<static_cast<unsigned>((n + 255) / 256), 256, 0, stream>>>(
      k, ib, nb, nq, nt, iv);
  return cudaGetLastError();
}

cudaError_t launch_to_fp32_bricked(const double* src, float* dst, int nx, int ny,
                                   int nz, int b, cudaStream_t stream) {
  to_fp32_bricked<<<1184, 256, 0, stream>>>(src, dst, nx, ny, nz, b);
  return cudaGetLastError();
}

cudaError_t launch_to_fp32(const double* src, float* dst, int64_t n,
                           cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  to_fp32<<<1184, 256, 0, stream>>>(src, dst, n);
  return cudaGetLastError();
}

}  // namespace ermc_dev
