// device_common.cuh — pieces shared by the fp64 and fp32 trace kernels:
// the keyed RNG, CDF inversion, cell decode and the persistent ray-pool
// scheduler (the paper's persistent ray pool).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "trace_common.cuh"

namespace ermc_dev {

constexpr unsigned kFullMask = 0xffffffffu;
constexpr double kPiDev = 3.14159265358979323846;

enum StepStatus : int { kContinue = 0, kDone = 1, kFail = 2 };

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  // MurmurHash3 fmix64 finaliser (reference sampling.cpp:13-20).
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdULL;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ULL;
  x ^= x >> 33;
  return x;
}

// uniform(RandomKey) with the seed and cell hashes hoisted out of the draw
// (reference sampling.cpp:24-29): h_cell = mix64(mix64(seed + phi) ^ cell).
__device__ __forceinline__ double draw_u(uint64_t h_cell, uint32_t ray,
                                         uint32_t draw) {
  const uint64_t h =
      mix64(h_cell ^ ((static_cast<uint64_t>(ray) << 32) | draw));
  return static_cast<double>(h >> 11) * 0x1.0p-53;
}

// One 32-byte read-only load (LDG.E.ENL2.256 on sm_100a): a whole interval
// record in one sector.
__device__ __forceinline__ double4 ldg4(const double4* p) {
  double4 r;
  asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
      : "=d"(r.x), "=d"(r.y), "=d"(r.z), "=d"(r.w)
      : "l"(p));
  return r;
}

// Cache-hinted read-only loads for the march; the kernels instantiate
// kHint = 0 (the hinted variants measured 5-27 % slower on B200, see
// profiles/ROUND1.md) (kHint: 0 = plain LDG.CONSTANT,
// 1 = temperature gathers bypass L1 allocation, 2 = temperature gathers evict
// first; for kHint >= 1 the interval records are kept with evict_last).
template <int kHint>
__device__ __forceinline__ float ld_t32(const float* p) {
  float r;
  if (kHint == 1)
    asm("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(r) : "l"(p));
  else if (kHint == 2)
    asm("ld.global.nc.L1::evict_first.f32 %0, [%1];" : "=f"(r) : "l"(p));
  else
    r = __ldg(p);
  return r;
}
template <int kHint>
__device__ __forceinline__ double ld_t64(const double* p) {
  double r;
  if (kHint == 1)
    asm("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(r) : "l"(p));
  else if (kHint == 2)
    asm("ld.global.nc.L1::evict_first.f64 %0, [%1];" : "=d"(r) : "l"(p));
  else
    r = __ldg(p);
  return r;
}
template <int kHint>
__device__ __forceinline__ float4 ld_rec32(const float4* p) {
  if (kHint == 0) return __ldg(p);
  float4 r;
  asm("ld.global.nc.L1::evict_last.v4.f32 {%0,%1,%2,%3}, [%4];"
      : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
      : "l"(p));
  return r;
}
template <int kHint>
__device__ __forceinline__ double4 ld_rec64(const double4* p) {
  double4 r;
  if (kHint == 0)
    asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
        : "=d"(r.x), "=d"(r.y), "=d"(r.z), "=d"(r.w)
        : "l"(p));
  else
    asm("ld.global.nc.L1::evict_last.v4.f64 {%0,%1,%2,%3}, [%4];"
        : "=d"(r.x), "=d"(r.y), "=d"(r.z), "=d"(r.w)
        : "l"(p));
  return r;
}

// Element index of cell (i, j, k) in the 2x2x2 micro-brick layout: bricks in
// k-fastest order, cells inside a brick as (i&1, j&1, k&1) -> 4i + 2j + k.
// A brick of fp32 values is one 32-byte sector; a ray step stays inside its
// brick with probability ~1/2, so consecutive gathers share L1 sectors.
__device__ __forceinline__ int brick_index(const LevelDesc& L, int i, int j, int k) {
  const int nby = (L.n[1] + 1) >> 1, nbz = (L.n[2] + 1) >> 1;
  return (((i >> 1) * nby + (j >> 1)) * nbz + (k >> 1)) * 8 + ((i & 1) << 2) +
         ((j & 1) << 1) + (k & 1);
}

// The same for kB^3 bricks (kB = 2 or 4; grid dimensions divisible by kB).
template <int kB>
__device__ __forceinline__ int brick_index_b(const LevelDesc& L, int i, int j, int k) {
  const int nby = L.n[1] / kB, nbz = L.n[2] / kB;
  return (((i / kB) * nby + (j / kB)) * nbz + (k / kB)) * (kB * kB * kB) +
         ((i % kB) * kB + (j % kB)) * kB + (k % kB);
}

// std::upper_bound over a short ascending array (sampling.cpp:44-51).
__device__ __forceinline__ int upper_bound_d(const double* a, int n, double x) {
  int first = 0, count = n;
  while (count > 0) {
    const int step = count >> 1;
    const int it = first + step;
    if (!(x < __ldg(a + it))) {
      first = it + 1;
      count -= step + 1;
    } else {
      count = step;
    }
  }
  return first;
}

// std::upper_bound over an array in shared or global memory (generic loads).
__device__ __forceinline__ int upper_bound_gen(const double* a, int n, double x) {
  int first = 0, count = n;
  while (count > 0) {
    const int step = count >> 1;
    if (!(x < a[first + step])) {
      first += step + 1;
      count -= step + 1;
    } else {
      count = step;
    }
  }
  return first;
}

// Band / g CDFs staged in shared memory by the lean trace kernels when they
// fit (P.cdf_smem): init's two binary searches then cost shared-memory
// latency instead of dependent global loads. Layout: band_cdf[nb] then
// quad_cdf[nb][nq], right after the kernel's per-thread records.

// Bytes of the staged CDFs and their guide tables (16-byte multiple).
__host__ __device__ inline size_t cdf_guide_bytes(int nb) {
  return (static_cast<size_t>(kGuideBand) + static_cast<size_t>(nb) * kGuideQuad + 15) / 16 * 16;
}
__host__ __device__ inline size_t cdf_smem_bytes(int nb, int nq) {
  return static_cast<size_t>(nb) * (1 + nq) * sizeof(double) + cdf_guide_bytes(nb);
}
// Staged bytes for a TraceParams::cdf_smem mode.
__host__ __device__ inline size_t cdf_stage_bytes(int mode, int nb, int nq) {
  return mode == 1 ? cdf_smem_bytes(nb, nq) : mode == 2 ? cdf_guide_bytes(nb) : 0;
}

__device__ __forceinline__ void stage_cdfs(const TraceParams& P, double* dst) {
  const int nb = P.n_bands, n = nb + nb * P.n_quad;
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    dst[i] = i < nb ? P.band_cdf[i] : P.quad_cdf[i - nb];
  uint8_t* gdst = reinterpret_cast<uint8_t*>(dst + n);
  for (int i = threadIdx.x; i < kGuideBand + nb * kGuideQuad; i += blockDim.x)
    gdst[i] = P.cdf_guide[i];
  __syncthreads();
}

// sample_band (sampling.cpp:42-53) on the staged CDFs: upper_bound by a
// linear scan from the guide bucket's start (the same index: upper_bound is
// monotone in r and r >= bucket start; ~1-2 compares instead of log2 n).
// r * 64 and r * 16 are exact, so the bucket of r is floor(r * G).
__device__ __forceinline__ void sample_band_cdf(const TraceParams& P, const double* cdf,
                                                double r_n, double r_g, int& n, int& g) {
  const int nb = P.n_bands, nq = P.n_quad;
  const uint8_t* guide = reinterpret_cast<const uint8_t*>(cdf + nb + nb * nq);
  n = guide[static_cast<int>(r_n * kGuideBand)];
  while (n < nb && !(r_n < cdf[n])) ++n;
  if (n >= nb) n = nb - 1;
  const double* qc = cdf + nb + n * nq;
  g = guide[kGuideBand + n * kGuideQuad + static_cast<int>(r_g * kGuideQuad)];
  while (g < nq && !(r_g < qc[g])) ++g;
  if (g >= nq) g = nq - 1;
}

// The same with only the guide tables staged (in shared memory) and the
// CDF values read through the read-only path (L1): the lean black-wall
// tracers keep their shared memory small enough for a 64 KB carveout.
__device__ __forceinline__ void sample_band_guided(const TraceParams& P, const uint8_t* guide,
                                                   double r_n, double r_g, int& n, int& g) {
  const int nb = P.n_bands, nq = P.n_quad;
  n = guide[static_cast<int>(r_n * kGuideBand)];
  while (n < nb && !(r_n < __ldg(P.band_cdf + n))) ++n;
  if (n >= nb) n = nb - 1;
  const double* qc = P.quad_cdf + n * nq;
  g = guide[kGuideBand + n * kGuideQuad + static_cast<int>(r_g * kGuideQuad)];
  while (g < nq && !(r_g < __ldg(qc + g))) ++g;
  if (g >= nq) g = nq - 1;
}

// Stages per P.cdf_smem at `dst` (after the kernel's per-thread records).
__device__ __forceinline__ void stage_guides(const TraceParams& P, uint8_t* dst);
__device__ __forceinline__ void stage_sampling(const TraceParams& P, void* dst) {
  if (P.cdf_smem == 1) stage_cdfs(P, reinterpret_cast<double*>(dst));
  else if (P.cdf_smem == 2) stage_guides(P, reinterpret_cast<uint8_t*>(dst));
}
// sample_band for the staged mode: `staged` points at what stage_sampling
// wrote (null: nothing staged).
__device__ __forceinline__ void sample_band_guided(const TraceParams& P, const uint8_t* guide,
                                                   double r_n, double r_g, int& n, int& g);
__device__ __forceinline__ void sample_band_staged(const TraceParams& P, const void* staged,
                                                   double r_n, double r_g, int& n, int& g);
__device__ __forceinline__ void stage_guides(const TraceParams& P, uint8_t* dst) {
  for (int i = threadIdx.x; i < kGuideBand + P.n_bands * kGuideQuad; i += blockDim.x)
    dst[i] = P.cdf_guide[i];
  __syncthreads();
}

// sample_band (reference sampling.cpp:42-53).
__device__ __forceinline__ void sample_band(const TraceParams& P, double r_n,
                                            double r_g, int& n, int& g) {
  n = upper_bound_d(P.band_cdf, P.n_bands, r_n);
  if (n >= P.n_bands) n = P.n_bands - 1;
  g = upper_bound_d(P.quad_cdf + static_cast<int64_t>(n) * P.n_quad, P.n_quad,
                    r_g);
  if (g >= P.n_quad) g = P.n_quad - 1;
}

__device__ __forceinline__ void sample_band_staged(const TraceParams& P, const void* staged,
                                                   double r_n, double r_g, int& n, int& g) {
  if (staged && P.cdf_smem == 1)
    sample_band_cdf(P, reinterpret_cast<const double*>(staged), r_n, r_g, n, g);
  else if (staged && P.cdf_smem == 2)
    sample_band_guided(P, reinterpret_cast<const uint8_t*>(staged), r_n, r_g, n, g);
  else
    sample_band(P, r_n, r_g, n, g);
}


__device__ __forceinline__ uint32_t fdiv(uint32_t n, const FastDiv& f) {
  return (__umulhi(n, f.m) + n) >> f.s;
}

// Linear k-fastest index of a level-0 cell -> (i, j, k) (reference
// solver.cpp:120-122); invariant-divisor divisions below 2^31 cells.
__device__ __forceinline__ void decode_cell(const TraceParams& P, int64_t cell,
                                            int& ci, int& cj, int& ck) {
  const LevelDesc& L = P.lv[0];
  const int64_t nyz = static_cast<int64_t>(L.n[1]) * L.n[2];
  if (cell < 0x7fffffffLL && nyz < 0x7fffffffLL) {
    const uint32_t c = static_cast<uint32_t>(cell);
    const uint32_t i = fdiv(c, P.div_nyz);
    const uint32_t rem = c - i * static_cast<uint32_t>(nyz);
    const uint32_t j = fdiv(rem, P.div_nz);
    ci = static_cast<int>(i);
    cj = static_cast<int>(j);
    ck = static_cast<int>(rem - j * static_cast<uint32_t>(L.n[2]));
  } else {
    ci = static_cast<int>(cell / nyz);
    cj = static_cast<int>((cell / L.n[2]) % L.n[1]);
    ck = static_cast<int>(cell % L.n[2]);
  }
}

// Records the smallest failing work id of the chunk: the word holds ~key
// (0 = no error; the counters are zeroed before the launch), so the maximum
// of the complements is the minimum key.
__device__ __forceinline__ void raise_error(const TraceParams& P, uint64_t key,
                                            int code) {
  const unsigned long long enc = ~static_cast<unsigned long long>(key);
  const unsigned long long old = atomicMax(P.err_key, enc);
  if (old < enc) atomicExch(P.err_code, code);
}

// Tracer::kWideLevelSteps (optional): the multigrid per-level step counter
// is 64-bit instead of 32-bit (a register-allocation choice, measured per
// tracer).
template <class T, class = void>
struct wide_level_steps : std::false_type {};
template <class T>
struct wide_level_steps<T, std::void_t<decltype(T::kWideLevelSteps)>>
    : std::integral_constant<bool, T::kWideLevelSteps> {};

// Per-level values a multigrid step reads (the level's cell words or
// temperatures, and its eps), one 16-byte entry per level in shared memory:
// lanes on different levels read distinct banks, and the step needs no
// kernel-parameter load indexed by a per-lane level (those serialise in the
// constant cache and cost a dependent load per step). Staged by the
// multigrid kernels before pool_kernel_body's barrier.
__shared__ ulonglong2 s_lv_hot[kMaxLevels];

enum LevelData { kLvCellWords, kLvField, kLvField32 };
__device__ __forceinline__ void stage_level_hot(const TraceParams& P, LevelData what) {
  if (threadIdx.x < static_cast<unsigned>(P.n_levels)) {
    const LevelDesc& L = P.lv[threadIdx.x];
    const void* base = what == kLvCellWords ? static_cast<const void*>(L.cellw)
                       : what == kLvField   ? static_cast<const void*>(L.field)
                                            : static_cast<const void*>(L.field32);
    s_lv_hot[threadIdx.x] = make_ulonglong2(reinterpret_cast<unsigned long long>(base),
                                            static_cast<unsigned long long>(
                                                __double_as_longlong(L.eps)));
  }
}

// Persistent ray pool. Every lane owns one ray; when at least
// refill_threshold lanes of a warp are idle they take the next work items
// (positions in the dispatch order: P.perm, or cell-major (cell, ray) ids)
// from a warp-local pool, refilled with one
// atomic per `kBatch` items from the chunk's global queue. Terminated rays
// write their q to q_ray[ray][cell]; the per-cell reduction runs later in
// ray-id order, so the schedule never changes a bit of the result.
//
// Tracer interface:
//   int init(const TraceParams&, int64_t cell, uint32_t ray)  -> DevError
//   int step(const TraceParams&, int max_steps)               -> StepStatus
//   double finish(const TraceParams&)       residual dump, final q
//   int err;  int level();  int sal(const TraceParams&);  int steps();
// kInner > 0: march steps per pool check fixed at compile time (the host
// launches such a kernel only when P.inner_steps == kInner): the loop bound
// is then an immediate, not a parameter load and compare per step.
template <class Tracer, bool kMulti, int kInner = 0>
__device__ __forceinline__ void run_pool(const TraceParams& P,
                                         unsigned long long* s_steps) {
  // Work ids are 32-bit: the host keeps every chunk below 2^31 items.
  constexpr uint32_t kBatch = 128;
  const unsigned lane = threadIdx.x & 31u;
  const unsigned lt_mask = (1u << lane) - 1u;
  const uint32_t rays = static_cast<uint32_t>(P.rays);
  const uint32_t n_work = static_cast<uint32_t>(P.n_work);
  const int max_steps = static_cast<int>(
      P.max_steps < 0x7fffffffLL ? P.max_steps : 0x7fffffffLL);

  Tracer tr;
  bool active = false;
  uint32_t my_work = 0;
  uint32_t pool_next = 0, pool_end = 0;
  bool exhausted = false;
  unsigned long long my_steps = 0;
  uint32_t lvl_steps = 0;  // kMulti: lane l accumulates level l (l < n_levels)

  while (true) {
    const unsigned idle = __ballot_sync(kFullMask, !active);
    const uint32_t n_idle = __popc(idle);
    const bool can_get = pool_next < pool_end || !exhausted;
    if (can_get && (n_idle >= static_cast<uint32_t>(P.refill_threshold) ||
                    idle == kFullMask)) {
      const uint32_t avail = pool_end - pool_next;
      uint32_t nb = 0, nb_end = 0;
      if (avail < n_idle && !exhausted) {
        unsigned long long b = 0;
        if (lane == 0) b = atomicAdd(P.work_counter, kBatch);
        b = __shfl_sync(kFullMask, b, 0);
        if (b >= n_work) {
          exhausted = true;
        } else {
          nb = static_cast<uint32_t>(b);
          nb_end = b + kBatch < n_work ? nb + kBatch : n_work;
        }
      }
      if (!active) {
        const uint32_t rank = __popc(idle & lt_mask);
        uint32_t w = 0xffffffffu;
        if (rank < avail)
          w = pool_next + rank;
        else if (rank - avail < nb_end - nb)
          w = nb + (rank - avail);
        if (w != 0xffffffffu) {
          if (P.perm) w = __ldg(P.perm + w);  // narrow-band sorted order
          const uint32_t cell = fdiv(w, P.div_rays);
          my_work = w;
          const int e = tr.init(P, P.cell_base + cell, w - cell * rays);
          if (e == kErrNone)
            active = true;
          else
            raise_error(P, w, e);
        }
      }
      if (avail >= n_idle) {
        pool_next += n_idle;
      } else if (nb_end > nb) {
        uint32_t take = n_idle - avail;
        if (take > nb_end - nb) take = nb_end - nb;
        pool_next = nb + take;
        pool_end = nb_end;
      } else {
        pool_next = pool_end;
      }
    }
    if (__ballot_sync(kFullMask, active) == 0u && exhausted &&
        pool_next >= pool_end)
      break;
    int done_lvl = -1;  // kMulti: final level of a ray that just ended
    uint32_t done_sal = 0;
    if (active) {
      // Several march steps per pool check: amortises the ballots; a lane
      // whose ray ends early idles for < inner_steps iterations.
      int st = kContinue;
      if constexpr (kMulti) {
        const int inner = kInner > 0 ? kInner : P.inner_steps;
        // not unrolled: the demotion makes the step body large (i-cache)
#pragma unroll 1
        for (int s = 0; s < inner && st == kContinue; ++s)
          st = tr.step(P, max_steps);
      } else {
        const int inner = kInner > 0 ? kInner : P.inner_steps;  // +1.5 % fp64 (r2az)
#pragma unroll 4  // vs 2: +0.2 % fp64, +0.15 % fp32 (r2bc); vs 1: +0.2 % / +0.6 %
        for (int s = 0; s < inner && st == kContinue; ++s)
          st = tr.step(P, max_steps);
      }
      if (st != kContinue) {
        active = false;
        if (st == kDone) {
          const double q = tr.finish(P);
          if (isfinite(q) && tr.finite_state()) {
            const uint32_t cell = fdiv(my_work, P.div_rays);
            const uint32_t ray = my_work - cell * rays;
            // streaming store: keep the L2 for the temperature field
            __stcs(P.q_ray + static_cast<uint64_t>(ray) * P.n_cells + cell, q);
            if (kMulti) {
              done_lvl = tr.level();
              done_sal = static_cast<uint32_t>(tr.sal(P));
            } else {
              my_steps += static_cast<unsigned long long>(tr.steps());
            }
          } else {
            raise_error(P, my_work, kErrNonFinite);
          }
        } else {
          raise_error(P, my_work, tr.err);
        }
      }
    }
    // Per-level step counts of the rays that just ended: a ray that ended on
    // level L took cap_l steps on every level l < L and sal on L. Summed per
    // warp here (converged) instead of one shared-memory 64-bit atomic per
    // ray and level — those compile to CAS loops that, contended by every
    // warp of the block, took ~20 % of the multigrid kernel's time.
    if (kMulti && __any_sync(kFullMask, done_lvl >= 0)) {
      for (int l = 0; l < P.n_levels; ++l) {
        const uint32_t c = done_lvl > l    ? static_cast<uint32_t>(P.lv[l].cap)
                           : done_lvl == l ? done_sal
                                           : 0u;
        const uint32_t lo = __reduce_add_sync(kFullMask, c & 0xffffu);
        const uint32_t hi = __reduce_add_sync(kFullMask, c >> 16);
        if (lane == static_cast<unsigned>(l)) {
          const unsigned long long add = lo + (static_cast<unsigned long long>(hi) << 16);
          if (wide_level_steps<Tracer>::value) {
            my_steps += add;
          } else if (lvl_steps + add >= 0x80000000ull) {  // keep the register 32-bit
            atomicAdd(&s_steps[l], lvl_steps + add);
            lvl_steps = 0;
          } else {
            lvl_steps += static_cast<uint32_t>(add);
          }
        }
      }
    }
  }
  if (!kMulti) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
      my_steps += __shfl_xor_sync(kFullMask, my_steps, o);
    if (lane == 0) atomicAdd(&s_steps[0], my_steps);
  } else {
    const unsigned long long v = wide_level_steps<Tracer>::value ? my_steps : lvl_steps;
    if (lane < static_cast<unsigned>(P.n_levels) && v != 0ull) atomicAdd(&s_steps[lane], v);
  }
}

// Common kernel prologue/epilogue around run_pool.
template <class Tracer, bool kMulti, int kInner = 0>
__device__ __forceinline__ void pool_kernel_body(const TraceParams& P) {
  __shared__ unsigned long long s_steps[kMaxLevels];
  if (threadIdx.x < kMaxLevels) s_steps[threadIdx.x] = 0ull;
  __syncthreads();
  run_pool<Tracer, kMulti, kInner>(P, s_steps);
  __syncthreads();
  if (threadIdx.x < static_cast<unsigned>(P.n_levels) &&
      s_steps[threadIdx.x] != 0ull)
    atomicAdd(P.steps_per_level + threadIdx.x, s_steps[threadIdx.x]);
}

}  // namespace ermc_dev
