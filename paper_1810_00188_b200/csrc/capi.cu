// capi.cu — implementation of the C-ABI boundary (include/ermc_b200.h).
//
// Host orchestration of reference solve() (solver.cpp:82-180) on one B200:
//   validate (device min/max/positivity pass + host checks, same messages
//   and order as solver.cpp:39-58) -> T_max -> build_cdfs / planck_mean / QE
//   on the host (bitwise the reference's) -> multigrid levels (K3) ->
//   chunked persistent trace (K1) -> per-cell reduce (K2).
// The only CPU work is O(n_bands * n_quad) table setup; every cell and ray
// is processed on the GPU. There is no CPU fallback: without a device every
// solve entry point returns an error.
#include <cuda_runtime.h>

#include <algorithm>
#include <numeric>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <thread>
#include <unordered_map>
#include <map>
#include <string>
#include <vector>

#include "ermc_b200.h"
#include "ermc_b200.hpp"
#include "host_tables.hpp"
#include "trace_common.cuh"

namespace ermc_dev {
int trace_fp64_blocks_per_sm(const TraceParams& P, int min_blocks);
cudaError_t launch_trace_fp64(const TraceParams& P, int grid, int min_blocks,
                              cudaStream_t s);
int trace_fp32_blocks_per_sm(const TraceParams& P, int min_blocks);
cudaError_t launch_trace_fp32(const TraceParams& P, int grid, int min_blocks,
                              cudaStream_t s);
cudaError_t launch_build_iv64(const double* k, const double* ib, int nb,
                              int nq, int nt, double4* iv, cudaStream_t s);
cudaError_t launch_trace_rays_fp64(const TraceParams& P, int64_t n,
                                   const int64_t* cells, const uint32_t* rays,
                                   const double* dirs, RayRecord* out,
                                   int64_t* level_steps, cudaStream_t s);
cudaError_t launch_reduce_cells_scatter(const double* q_ray, int64_t n_cells, int rays,
                                        const ScatterOut& out, int64_t base, cudaStream_t s);
cudaError_t launch_reduce_cells(const double* q_ray, int64_t n_cells, int rays,
                                double* q_r, double* std_dev, cudaStream_t s);
cudaError_t launch_restrict(const double* fine, int fnx, int fny, int fnz,
                            int ratio, double* coarse, int cnx, int cny,
                            int cnz, cudaStream_t s);
cudaError_t launch_field_stats(const double* t, int64_t n, double* scratch,
                               int n_blocks, double* out3, cudaStream_t s);
cudaError_t launch_uniform(uint64_t h_seed, int64_t n, const uint64_t* cells,
                           const uint32_t* rays, const uint32_t* draws,
                           double* out, cudaStream_t s);
cudaError_t launch_build_iv32(const double* k, const double* ib, int nb,
                              int nq, int nt, float4* iv, cudaStream_t s);
cudaError_t launch_to_fp32(const double* src, float* dst, int64_t n,
                           cudaStream_t s);
cudaError_t launch_to_fp32_bricked(const double* src, float* dst, int nx, int ny,
                                   int nz, int b, cudaStream_t s);
cudaError_t launch_to_bricked64(const double* src, double* dst, int nx, int ny, int nz,
                                cudaStream_t s);
cudaError_t launch_build_cell_words(const TraceParams& P, const double* field, int64_t n,
                                    double scale, uint64_t* out, int* bad, cudaStream_t s);
cudaError_t launch_init_states_fp64(const TraceParams& P, int64_t n, const int32_t* cells,
                                    const uint32_t* ray_ids, uint64_t seed,
                                    ermc_ray_state_t* out, int32_t* err, cudaStream_t s);
cudaError_t launch_march_states_fp64(const TraceParams& P, int64_t n,
                                     const ermc_ray_state_t* in, RayRecord* out,
                                     int64_t* level_steps, cudaStream_t s);
cudaError_t launch_sample_direction(int64_t n, const double* rt, const double* rp, double* out,
                                    cudaStream_t s);
cudaError_t launch_absorptivity(int64_t n, const double* k, const double* ds, double* out,
                                cudaStream_t s);
int sort_max_bins();
int sort_max_tile_items();
cudaError_t launch_ng_sort(const TraceParams& P, const int32_t* row_rank, int n_rows,
                           int dir_bins, int tile_cells, int block, uint32_t* packed,
                           uint32_t* perm, cudaStream_t s);
}  // namespace ermc_dev

using ermc::Error;

namespace {

constexpr int kStatsBlocks = 592;  // 4 x 148 SMs

uint64_t mix64_host(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdULL;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ULL;
  x ^= x >> 33;
  return x;
}

void put_err(char* buf, size_t len, const std::string& msg) {
  if (!buf || len == 0) return;
  std::snprintf(buf, len, "%s", msg.c_str());
}

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw Error(std::string("CUDA error in ") + what + ": " +
                cudaGetErrorString(e));
}

// RAII device-current switch.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (dev >= 0 && dev != prev) cuda_check(cudaSetDevice(dev), "cudaSetDevice");
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

// Process-wide caching allocator for device buffers. A one-shot solve
// (ermc_b200_solve*) builds and drops a whole session — the field, the
// per-ray scratch (8.6 GB at 256^3, R = 64), the dispatch order — so
// without a cache every call pays cudaMalloc/cudaFree of all of it. Freed
// blocks are kept per device (best fit within 2x of the request) up to a cap
// of a third of the device memory; ermc_b200_release_cached_memory() returns
// them. Every solve path synchronises its stream before its buffers are
// released (session_solve_impl, solve_host, ~ermc_session), so a cached
// block is never handed out while a kernel may still touch it.
class DevicePool {
 public:
  static DevicePool& get() {
    static DevicePool* pool = new DevicePool();  // never destroyed: no CUDA calls at exit
    return *pool;
  }
  void* alloc(size_t bytes) {
    int dev = 0;
    cudaGetDevice(&dev);
    {
      std::lock_guard<std::mutex> lk(mu_);
      auto& fl = free_[dev];
      auto it = fl.lower_bound(bytes);
      if (it != fl.end() && it->first <= 2 * bytes + (size_t(1) << 20)) {
        void* p = it->second;
        cached_[dev] -= it->first;
        size_[p] = it->first;
        fl.erase(it);
        return p;
      }
    }
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e != cudaSuccess) {
      cudaGetLastError();
      release(dev);
      cuda_check(cudaMalloc(&p, bytes), "cudaMalloc");
    }
    std::lock_guard<std::mutex> lk(mu_);
    size_[p] = bytes;
    return p;
  }
  void free(void* p) {
    if (!p) return;
    int dev = 0;
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) == cudaSuccess) dev = a.device;
    cudaGetLastError();
    std::lock_guard<std::mutex> lk(mu_);
    auto it = size_.find(p);
    const size_t bytes = it == size_.end() ? 0 : it->second;
    if (it != size_.end()) size_.erase(it);
    free_[dev].emplace(bytes, p);
    cached_[dev] += bytes;
    trim_locked(dev);
  }
  void release(int dev) {
    std::lock_guard<std::mutex> lk(mu_);
    DeviceGuard g(dev);
    for (auto& kv : free_[dev]) cudaFree(kv.second);
    free_[dev].clear();
    cached_[dev] = 0;
  }

 private:
  void trim_locked(int dev) {
    if (cap_.find(dev) == cap_.end()) {
      size_t fr = 0, tot = 0;
      DeviceGuard g(dev);
      cudaMemGetInfo(&fr, &tot);
      cap_[dev] = tot / 3;
    }
    auto& fl = free_[dev];
    while (cached_[dev] > cap_[dev] && !fl.empty()) {
      auto last = std::prev(fl.end());
      DeviceGuard g(dev);
      cudaFree(last->second);
      cached_[dev] -= last->first;
      fl.erase(last);
    }
  }
  std::mutex mu_;
  std::map<int, std::multimap<size_t, void*>> free_;
  std::map<int, size_t> cached_, cap_;
  std::unordered_map<void*, size_t> size_;
};

// Pinned host words for the solve's counters (so their copies stay
// asynchronous). cudaMallocHost / cudaFreeHost are slow and the latter
// synchronises the device, so blocks are recycled process-wide instead of
// being allocated per session (one-shot solves create a session per call).
class PinnedPool {
 public:
  static PinnedPool& get() {
    static PinnedPool* pool = new PinnedPool();  // never destroyed
    return *pool;
  }
  unsigned long long* alloc(size_t words, size_t* got) {
    {
      std::lock_guard<std::mutex> lk(mu_);
      for (size_t i = 0; i < free_.size(); ++i)
        if (free_[i].second >= words) {
          auto b = free_[i];
          free_.erase(free_.begin() + static_cast<long>(i));
          *got = b.second;
          return b.first;
        }
    }
    const size_t n = std::max<size_t>(words, 4096);
    void* p = nullptr;
    cuda_check(cudaMallocHost(&p, n * sizeof(unsigned long long)), "cudaMallocHost");
    *got = n;
    return static_cast<unsigned long long*>(p);
  }
  void free(unsigned long long* p, size_t words) {
    if (!p) return;
    std::lock_guard<std::mutex> lk(mu_);
    free_.emplace_back(p, words);
  }

 private:
  std::mutex mu_;
  std::vector<std::pair<unsigned long long*, size_t>> free_;
};

template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { reset(); }
  void reset() {
    if (p) DevicePool::get().free(p);
    p = nullptr;
    n = 0;
  }
  void ensure(size_t count) {
    if (count <= n && p) return;
    reset();
    p = static_cast<T*>(DevicePool::get().alloc(std::max<size_t>(count, 1) * sizeof(T)));
    n = count;
  }
  void upload(const T* src, size_t count, cudaStream_t s) {
    ensure(count);
    if (count)
      cuda_check(cudaMemcpyAsync(p, src, count * sizeof(T),
                                 cudaMemcpyHostToDevice, s),
                 "cudaMemcpyAsync H2D");
  }
};

void validate_config(const ermc_config_t& c) {
  // SolveConfig::validate (solver.cpp:14-23)
  if (c.rays_per_cell < 1) throw Error("SolveConfig: rays_per_cell must be >= 1");
  if (!(c.tolerance > 0.0 && c.tolerance < 1.0))
    throw Error("SolveConfig: tolerance must be in (0,1)");
  if (c.n_levels < 1) throw Error("SolveConfig: n_levels must be >= 1");
  if (c.steps_per_level < 1)
    throw Error("SolveConfig: steps_per_level must be >= 1");
  if (c.max_steps < 1) throw Error("SolveConfig: max_steps must be >= 1");
  if (c.workers < 0) throw Error("SolveConfig: workers must be >= 0");
  if (c.precision != ERMC_PRECISION_FP64 && c.precision != ERMC_PRECISION_FP32)
    throw Error("SolveConfig: precision must be fp64 (0) or fp32 (1)");
  if (c.n_devices < 0) throw Error("ermc_b200: n_devices must be >= 0");
  if (c.n_levels > ermc_dev::kMaxLevels)
    throw Error("SolveConfig: n_levels above the GPU limit of " +
                std::to_string(ermc_dev::kMaxLevels));
}

void validate_grid(const ermc_grid_t& g) {
  // CartesianGrid::validate (geometry.cpp:15-20)
  if (g.nx < 1 || g.ny < 1 || g.nz < 1)
    throw Error("CartesianGrid: cell counts must be >= 1");
  if (g.dx <= 0.0 || g.dy <= 0.0 || g.dz <= 0.0)
    throw Error("CartesianGrid: spacings must be positive");
}

void validate_boundary(const ermc_boundary_t& b) {
  // BoundarySpec::validate (geometry.cpp:22-32)
  for (int a = 0; a < 3; ++a) {
    if (b.kind[a] == ERMC_AXIS_PERIODIC) continue;
    const double t[2] = {b.lo_temperature[a], b.hi_temperature[a]};
    const double e[2] = {b.lo_emissivity[a], b.hi_emissivity[a]};
    for (int s = 0; s < 2; ++s) {
      if (e[s] < 0.0 || e[s] > 1.0)
        throw Error("BoundarySpec: wall emissivity must be in [0,1]");
      if (t[s] < 0.0) throw Error("BoundarySpec: wall temperature must be >= 0");
    }
  }
}

double spacing(const ermc_grid_t& g, int a) {
  return a == 0 ? g.dx : a == 1 ? g.dy : g.dz;
}
int count(const ermc_grid_t& g, int a) { return a == 0 ? g.nx : a == 1 ? g.ny : g.nz; }
int64_t cells_of(const ermc_grid_t& g) {
  return static_cast<int64_t>(g.nx) * g.ny * g.nz;
}

struct Timing {
  cudaEvent_t a = nullptr, b = nullptr;
};

// Scheduling knobs (defaults tuned on B200; ERMC_* environment variables
// override them for experiments — they never change results).
struct Tune {
  int inner_steps = 32;    // fp64 march steps per pool check
  int inner_steps32 = 48;  // fp32
  int inner_steps_mg = 48;    // multigrid (n_levels > 1), fp64: measured -1..-4 % time
  int inner_steps32_mg = 64;  // multigrid, fp32: measured -1 %
  int refill = 8;
  int fp64_min_blocks = 0;  // 0 = per-tracer default (trace_fp64.cu)
  int fp32_min_blocks = 8;
  int lean = 1;
  int brick = 1;    // fp32: micro-brick field copy (measured +4 %)
  int brick64 = 0;  // fp64: micro-brick field copy (measured neutral; off saves 8 B/cell)
  int sort = 1;  // narrow-band sorted dispatch (dispatch.cu)
  int track_pos = 0;  // 1 forces the position-tracking fp64 kernel
  int tint_arith = 1;  // compute exact-uniform temperature records (fp64)
  int cdf_smem = 1;    // stage the sampling CDFs in shared memory (lean kernels)
  int sort_tile_items = 1 << 16;
  // cubic sort tiles (edge in cells; 0 = linear tiles, -1 = the largest edge
  // with edge^3 * R <= 2^16 for single-level solves (10 at R = 64: +0.6 %
  // over linear, r2bk/r2bl), linear for multigrid (−1.2 % there, r2bn))
  int sort_block = -1;
  int sort_dirs = 32;  // direction bins inside each spectral row (1, 8, 32: +1.9 % at 32)
  int cellw = 1;       // fp64 lean tracers read precomputed cell words (trace_fp64.cu)
  int carveout = 0;    // trace kernels: smallest shared-memory carveout (-1 driver default)
};
int env_int(const char* name, int fallback) {
  const char* v = std::getenv(name);
  return v && *v ? std::atoi(v) : fallback;
}
const Tune& tune() {
  static const Tune t = [] {
    Tune x;
    x.inner_steps = std::max(1, env_int("ERMC_INNER_STEPS", x.inner_steps));
    x.inner_steps32 = std::max(1, env_int("ERMC_INNER_STEPS32", x.inner_steps32));
    x.inner_steps_mg = std::max(1, env_int("ERMC_INNER_STEPS_MG", x.inner_steps_mg));
    x.inner_steps32_mg = std::max(1, env_int("ERMC_INNER_STEPS32_MG", x.inner_steps32_mg));
    x.refill = std::max(1, std::min(32, env_int("ERMC_REFILL", x.refill)));
    x.fp64_min_blocks = env_int("ERMC_FP64_MINB", x.fp64_min_blocks);
    x.fp32_min_blocks = env_int("ERMC_FP32_MINB", x.fp32_min_blocks);
    x.lean = env_int("ERMC_LEAN", x.lean);
    x.brick = env_int("ERMC_BRICK", x.brick);
    x.brick64 = env_int("ERMC_BRICK64", x.brick64);
    x.sort = env_int("ERMC_SORT", x.sort);
    x.track_pos = env_int("ERMC_TRACK_POS", x.track_pos);
    x.tint_arith = env_int("ERMC_TINT_ARITH", x.tint_arith);
    x.cdf_smem = env_int("ERMC_CDF_SMEM", x.cdf_smem);
    x.sort_tile_items = std::max(1, env_int("ERMC_SORT_TILE", x.sort_tile_items));
    x.sort_dirs = std::max(1, env_int("ERMC_SORT_DIRS", x.sort_dirs));
    x.sort_block = std::max(-1, env_int("ERMC_SORT_BLOCK", x.sort_block));
    x.cellw = env_int("ERMC_CELLW", x.cellw);
    x.carveout = env_int("ERMC_CARVEOUT", x.carveout);
    return x;
  }();
  return t;
}

}  // namespace

struct ermc_session {
  int device = 0;
  int n_sm = 148;
  ermc_grid_t grid{};
  ermc_boundary_t boundary{};
  ermc_config_t config{};
  // owning host copies of the model tables
  std::vector<double> nu_lo, nu_hi, nu_c, gp, gw, temps, k, ib;
  ermc_model_t model{};
  ermc_host::TableView view;
  int64_t n_cells = 0;

  DevBuf<double> d_temps, d_k, d_ib, d_wall_ib, d_band_cdf, d_quad_cdf, d_kmax,
      d_ibmax;
  DevBuf<float> d_wall_ibn32;
  DevBuf<double4> d_tint, d_iv64;
  DevBuf<double2> d_pref_den;
  DevBuf<uint8_t> d_cdf_guide;
  DevBuf<double> d_field;
  std::vector<std::unique_ptr<DevBuf<double>>> d_levels;  // levels >= 1
  std::vector<ermc_grid_t> level_grids;
  DevBuf<float> d_field32;
  DevBuf<float> d_field32b;
  int fp32_brick_edge = 0;  // layout of d_field32b (2 or 4)
  DevBuf<double> d_field64b;
  // cell words of every level (fp64 lean tracers); valid until set_field
  std::vector<std::unique_ptr<DevBuf<uint64_t>>> d_cellw;
  DevBuf<int> d_cw_bad;
  bool cellw_valid = false, cellw_ok = false;
  std::vector<std::unique_ptr<DevBuf<float>>> d_levels32;
  DevBuf<float4> d_iv32;
  bool iv32_ready = false;
  DevBuf<double> d_qray;
  // narrow-band sorted dispatch: row rank by k(n,g,T_max), keys, order
  DevBuf<int32_t> d_row_rank;
  DevBuf<uint32_t> d_keys;  // per work id: row rank << 16 | rank in its bin
  DevBuf<uint32_t> d_perm;
  DevBuf<unsigned long long> d_counters;  // per chunk: work, err key
  DevBuf<int32_t> d_errcode;
  DevBuf<unsigned long long> d_steps;
  DevBuf<double> d_stats_scratch, d_stats;
  bool field_set = false;
  bool levels_valid = false;  // coarse levels match the current field

  double ms[4] = {0, 0, 0, 0};
  // A solve enqueued but not yet waited for (session_solve_async): its
  // stream, events, chunking, parameters (to describe a failing ray) and the
  // pinned host words its counters are copied into.
  struct Pending {
    bool active = false;
    cudaStream_t st = nullptr;
    int64_t lo = 0, chunk_cells = 0, n_chunks = 0;
    int rays = 0;
    ermc_dev::TraceParams P{};
    std::vector<Timing> tt, tr, ts;
  } pending;
  unsigned long long* h_words = nullptr;  // pinned: counters, codes, steps
  size_t h_words_n = 0;
  int32_t launches = 0;
  std::mutex mu;
  size_t qray_budget_bytes = 0;
  bool tables_finite = true;  // every k / Ib table entry finite (lean tracers allowed)
  // Marks the last asynchronous work (set_field's copy) so the destructor can
  // wait for it before the buffers return to the pool.
  cudaEvent_t last_work = nullptr;
  ~ermc_session() {
    if (pending.active) {  // never waited for: finish the work before the
      DeviceGuard g(device);  // buffers go back to the pool
      cudaStreamSynchronize(pending.st);
    }
    PinnedPool::get().free(h_words, h_words_n);
    if (last_work) {
      DeviceGuard g(device);
      cudaEventSynchronize(last_work);
      cudaEventDestroy(last_work);
    }
  }
};

namespace {

void copy_model(ermc_session* s, const ermc_model_t& m) {
  s->nu_lo.assign(m.band_nu_lo, m.band_nu_lo + m.n_bands);
  s->nu_hi.assign(m.band_nu_hi, m.band_nu_hi + m.n_bands);
  s->nu_c.assign(m.band_nu_center, m.band_nu_center + m.n_bands);
  s->gp.assign(m.g_points, m.g_points + m.n_quad);
  s->gw.assign(m.g_weights, m.g_weights + m.n_quad);
  s->temps.assign(m.temp_grid, m.temp_grid + m.n_temps);
  const size_t nk = static_cast<size_t>(m.n_bands) * m.n_quad * m.n_temps;
  s->k.assign(m.k_table, m.k_table + nk);
  s->ib.assign(m.ib_table, m.ib_table + static_cast<size_t>(m.n_bands) * m.n_temps);
  s->model = m;
  s->model.band_nu_lo = s->nu_lo.data();
  s->model.band_nu_hi = s->nu_hi.data();
  s->model.band_nu_center = s->nu_c.data();
  s->model.g_points = s->gp.data();
  s->model.g_weights = s->gw.data();
  s->model.temp_grid = s->temps.data();
  s->model.k_table = s->k.data();
  s->model.ib_table = s->ib.data();
  s->view = ermc_host::make_view_unchecked(s->model);
  // The lean tracers drop interp's frac == 0 shortcut (a + 0 * (b - a) == a
  // only for finite b): with any non-finite table entry the solve runs the
  // reference-order tracers, which keep it (spectral.cpp:179-205).
  s->tables_finite = std::all_of(s->k.begin(), s->k.end(), [](double x) { return std::isfinite(x); }) &&
                     std::all_of(s->ib.begin(), s->ib.end(), [](double x) { return std::isfinite(x); });
}

ermc_session* create_session(const ermc_grid_t* grid,
                             const ermc_boundary_t* boundary,
                             const ermc_model_t* model,
                             const ermc_config_t* config) {
  if (!grid || !boundary || !model || !config)
    throw Error("ermc_b200: null descriptor");
  int n_dev = 0;
  if (cudaGetDeviceCount(&n_dev) != cudaSuccess || n_dev == 0) {
    cudaGetLastError();
    throw Error("ermc_b200: no CUDA device available (the solver has no CPU path)");
  }
  ermc_host::make_view(*model);  // SpectralModel constructor checks
  validate_config(*config);
  validate_grid(*grid);
  auto s = std::make_unique<ermc_session>();
  int dev = config->device;
  if (dev < 0) cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
  if (dev >= n_dev) throw Error("ermc_b200: device ordinal out of range");
  s->device = dev;
  DeviceGuard guard(dev);
  cuda_check(cudaDeviceGetAttribute(&s->n_sm, cudaDevAttrMultiProcessorCount, dev),
             "cudaDeviceGetAttribute");
  s->grid = *grid;
  s->boundary = *boundary;
  s->config = *config;
  copy_model(s.get(), *model);
  s->n_cells = cells_of(*grid);
  size_t free_b = 0, total_b = 0;
  cuda_check(cudaMemGetInfo(&free_b, &total_b), "cudaMemGetInfo");
  s->qray_budget_bytes = std::min<size_t>(free_b / 4, size_t(16) << 30);
  // Test hook: a small per-ray buffer budget forces many chunks (bytes).
  if (const char* e = std::getenv("ERMC_QRAY_BUDGET")) {
    const long long v = std::atoll(e);
    if (v > 0) s->qray_budget_bytes = static_cast<size_t>(v);
  }

  cudaStream_t st = nullptr;
  s->d_temps.upload(s->temps.data(), s->temps.size(), st);
  s->d_k.upload(s->k.data(), s->k.size(), st);
  s->d_ib.upload(s->ib.data(), s->ib.size(), st);
  {
    // Packed fp64 tables (copies of reference values + exact reciprocals).
    const ermc_host::TableView& v = s->view;
    if (v.nt >= 2) {
      std::vector<double4> tint(v.nt - 1);
      for (int l = 0; l + 1 < v.nt; ++l) {
        const double w = v.temps[l + 1] - v.temps[l];
        tint[l] = make_double4(v.temps[l], w, 1.0 / w, 0.0);
      }
      s->d_tint.upload(tint.data(), tint.size(), st);
      s->d_iv64.ensure(static_cast<size_t>(v.nb) * v.nq * (v.nt - 1));
      cuda_check(ermc_dev::launch_build_iv64(s->d_k.p, s->d_ib.p, v.nb, v.nq, v.nt,
                                             s->d_iv64.p, st),
                 "build_iv64");
    }
  }
  s->d_field.ensure(static_cast<size_t>(s->n_cells));
  s->d_stats_scratch.ensure(3 * kStatsBlocks);
  s->d_stats.ensure(3);
  s->d_steps.ensure(ermc_dev::kMaxLevels);
  cuda_check(cudaStreamSynchronize(st), "upload tables");
  return s.release();
}

// Per-level grids of build_hierarchy (geometry.cpp:84-110), host side.
std::vector<ermc_grid_t> level_grids(const ermc_grid_t& g0, int n_levels,
                                     int ratio) {
  std::vector<ermc_grid_t> out{g0};
  if (n_levels > 1 && ratio < 2)
    throw Error("build_hierarchy: ratio must be >= 2");
  for (int l = 1; l < n_levels; ++l) {
    const ermc_grid_t& f = out.back();
    if (f.nx == 1 && f.ny == 1 && f.nz == 1)
      throw Error("build_hierarchy: cannot coarsen below one cell; achievable "
                  "depth is " + std::to_string(l));
    ermc_grid_t c = f;
    c.nx = (f.nx + ratio - 1) / ratio;
    c.ny = (f.ny + ratio - 1) / ratio;
    c.nz = (f.nz + ratio - 1) / ratio;
    c.dx = (f.nx * f.dx) / c.nx;  // fg.extent(0) / cg.nx
    c.dy = (f.ny * f.dy) / c.ny;
    c.dz = (f.nz * f.dz) / c.nz;
    out.push_back(c);
  }
  return out;
}

struct Prepared {
  ermc_dev::TraceParams P{};
  double t_max = 0.0;
  double qe = 0.0;
  std::vector<double> band_cdf, quad_cdf, kmax, ibmax, wall_ib;
  std::vector<double2> pref_den;
  std::vector<float> wall_ibn32;
  bool sorted = false;  // narrow-band sorted dispatch enabled for this solve
};

// Device stats pass + the reference's validation order (solver.cpp:39-58)
// for the field-dependent checks; returns T_max (solver.cpp:27-37).
double validate_field_and_tmax(ermc_session* s, cudaStream_t st) {
  Timing t;
  cudaEventCreate(&t.a);
  cudaEventCreate(&t.b);
  cudaEventRecord(t.a, st);
  cuda_check(ermc_dev::launch_field_stats(s->d_field.p, s->n_cells,
                                          s->d_stats_scratch.p, kStatsBlocks,
                                          s->d_stats.p, st),
             "field_stats");
  s->launches += 2;
  cudaEventRecord(t.b, st);
  double h[3];
  cuda_check(cudaMemcpyAsync(h, s->d_stats.p, sizeof(h), cudaMemcpyDeviceToHost, st),
             "stats D2H");
  cuda_check(cudaStreamSynchronize(st), "stats sync");
  float ms = 0.f;
  cudaEventElapsedTime(&ms, t.a, t.b);
  s->ms[0] += ms;
  cudaEventDestroy(t.a);
  cudaEventDestroy(t.b);
  const double fmin_v = h[0], fmax_v = h[1];
  if (h[2] > 0.0) throw Error("TemperatureField: temperatures must be positive");
  validate_boundary(s->boundary);
  const double lo = s->temps.front(), hi = s->temps.back();
  if (fmin_v < lo || fmax_v > hi)
    throw Error("solve: field temperatures outside spectral table range");
  const ermc_boundary_t& b = s->boundary;
  for (int a = 0; a < 3; ++a) {
    if (b.kind[a] == ERMC_AXIS_PERIODIC) continue;
    for (double wt : {b.lo_temperature[a], b.hi_temperature[a]})
      if (wt != 0.0 && (wt < lo || wt > hi))
        throw Error("solve: wall temperature outside spectral table range");
  }
  double t_max = fmax_v;
  for (int a = 0; a < 3; ++a) {
    if (b.kind[a] == ERMC_AXIS_PERIODIC) continue;
    t_max = std::max({t_max, b.lo_temperature[a], b.hi_temperature[a]});
  }
  return t_max;
}

// Host setup for a given T_max and QE: CDFs, T_max interpolants, wall
// blackbodies, level descriptors (restricting coarse levels on device).
void prepare(ermc_session* s, Prepared& pr, double t_max, double qe,
             bool build_levels, cudaStream_t st) {
  const ermc_host::TableView& v = s->view;
  const ermc_config_t& c = s->config;
  pr.t_max = t_max;
  pr.qe = qe;
  pr.band_cdf.assign(v.nb, 0.0);
  pr.quad_cdf.assign(static_cast<size_t>(v.nb) * v.nq, 0.0);
  ermc_host::build_cdfs(v, t_max, pr.band_cdf.data(), pr.quad_cdf.data());
  std::vector<ermc_grid_t> grids = level_grids(s->grid, c.n_levels, c.coarsen_ratio);

  pr.kmax.resize(static_cast<size_t>(v.nb) * v.nq);
  pr.ibmax.resize(v.nb);
  for (int n = 0; n < v.nb; ++n) {
    pr.ibmax[n] = ermc_host::interp_ib(v, n, t_max);
    for (int g = 0; g < v.nq; ++g)
      pr.kmax[static_cast<size_t>(n) * v.nq + g] = ermc_host::interp_k(v, n, g, t_max);
  }
  // Dispatch order of the spectral rows: k(n, g, T_max) ascending, ties in
  // (n, g) order — the reference's presample_and_sort key (solver.cpp:62-80).
  const int n_rows = v.nb * v.nq;
  pr.sorted = tune().sort && n_rows <= ermc_dev::sort_max_bins() &&
              c.rays_per_cell <= ermc_dev::sort_max_tile_items();
  if (pr.sorted) {
    std::vector<int32_t> order(n_rows), rank(n_rows);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(),
                     [&](int32_t a, int32_t b) { return pr.kmax[a] < pr.kmax[b]; });
    for (int i = 0; i < n_rows; ++i) rank[order[i]] = i;
    s->d_row_rank.upload(rank.data(), rank.size(), st);
  }
  pr.wall_ib.assign(6 * static_cast<size_t>(v.nb), 0.0);
  const ermc_boundary_t& b = s->boundary;
  for (int a = 0; a < 3; ++a) {
    if (b.kind[a] == ERMC_AXIS_PERIODIC) continue;
    const double wt[2] = {b.lo_temperature[a], b.hi_temperature[a]};
    for (int side = 0; side < 2; ++side)
      if (wt[side] > 0.0)
        for (int n = 0; n < v.nb; ++n)
          pr.wall_ib[(2 * a + side) * static_cast<size_t>(v.nb) + n] =
              ermc_host::interp_ib(v, n, wt[side]);
  }
  {  // guide tables of the staged CDFs (device_common.cuh sample_band_cdf)
    std::vector<uint8_t> guide(ermc_dev::kGuideBand + static_cast<size_t>(v.nb) *
                                                          ermc_dev::kGuideQuad);
    for (int k = 0; k < ermc_dev::kGuideBand; ++k)
      guide[k] = static_cast<uint8_t>(std::min<ptrdiff_t>(
          255, std::upper_bound(pr.band_cdf.begin(), pr.band_cdf.end(),
                                static_cast<double>(k) / ermc_dev::kGuideBand) -
                   pr.band_cdf.begin()));
    for (int n = 0; n < v.nb; ++n) {
      auto q0 = pr.quad_cdf.begin() + static_cast<ptrdiff_t>(n) * v.nq;
      for (int k = 0; k < ermc_dev::kGuideQuad; ++k)
        guide[ermc_dev::kGuideBand + n * ermc_dev::kGuideQuad + k] = static_cast<uint8_t>(
            std::min<ptrdiff_t>(255, std::upper_bound(q0, q0 + v.nq,
                                                      static_cast<double>(k) /
                                                          ermc_dev::kGuideQuad) -
                                         q0));
    }
    s->d_cdf_guide.upload(guide.data(), guide.size(), st);
  }
  s->d_band_cdf.upload(pr.band_cdf.data(), pr.band_cdf.size(), st);
  s->d_quad_cdf.upload(pr.quad_cdf.data(), pr.quad_cdf.size(), st);
  s->d_kmax.upload(pr.kmax.data(), pr.kmax.size(), st);
  s->d_ibmax.upload(pr.ibmax.data(), pr.ibmax.size(), st);
  // R_I denominators k(n,g,T_max) Ib(n,T_max) (sampling.cpp:93) and their
  // correctly rounded reciprocals; non-positive ones keep the IEEE path.
  pr.pref_den.resize(pr.kmax.size());
  for (int n = 0; n < v.nb; ++n)
    for (int g = 0; g < v.nq; ++g) {
      const size_t i = static_cast<size_t>(n) * v.nq + g;
      const double d = pr.kmax[i] * pr.ibmax[n];
      pr.pref_den[i] = make_double2(pr.kmax[i] > 0.0 && pr.ibmax[n] > 0.0 ? d : 0.0,
                                    d > 0.0 ? 1.0 / d : 0.0);
    }
  s->d_pref_den.upload(pr.pref_den.data(), pr.pref_den.size(), st);
  s->d_wall_ib.upload(pr.wall_ib.data(), pr.wall_ib.size(), st);
  // fp32 kernel: wall blackbodies normalised like its interval table.
  pr.wall_ibn32.assign(pr.wall_ib.size(), 0.0f);
  for (int f = 0; f < 6; ++f)
    for (int n = 0; n < v.nb; ++n) {
      const double last = v.ib_node(n, v.nt - 1);
      const size_t i = static_cast<size_t>(f) * v.nb + n;
      pr.wall_ibn32[i] = last > 0.0 ? static_cast<float>(pr.wall_ib[i] / last) : 0.0f;
    }
  s->d_wall_ibn32.upload(pr.wall_ibn32.data(), pr.wall_ibn32.size(), st);

  // Multigrid levels (K3), restricted level by level like build_hierarchy.
  if (build_levels && !s->levels_valid) {
    Timing t;
    cudaEventCreate(&t.a);
    cudaEventCreate(&t.b);
    cudaEventRecord(t.a, st);
    s->d_levels.resize(grids.size());
    for (size_t l = 1; l < grids.size(); ++l) {
      if (!s->d_levels[l]) s->d_levels[l] = std::make_unique<DevBuf<double>>();
      s->d_levels[l]->ensure(static_cast<size_t>(cells_of(grids[l])));
      const double* fine = l == 1 ? s->d_field.p : s->d_levels[l - 1]->p;
      const ermc_grid_t& f = grids[l - 1];
      const ermc_grid_t& cg = grids[l];
      cuda_check(ermc_dev::launch_restrict(fine, f.nx, f.ny, f.nz,
                                           c.coarsen_ratio, s->d_levels[l]->p,
                                           cg.nx, cg.ny, cg.nz, st),
                 "restrict");
      ++s->launches;
    }
    cudaEventRecord(t.b, st);
    cudaEventSynchronize(t.b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, t.a, t.b);
    s->ms[1] += ms;
    cudaEventDestroy(t.a);
    cudaEventDestroy(t.b);
    s->levels_valid = true;
    s->level_grids = grids;
  }

  ermc_dev::TraceParams& P = pr.P;
  std::memset(&P, 0, sizeof(P));
  P.n_levels = c.n_levels;
  for (int a = 0; a < 3; ++a) {
    P.periodic[a] = b.kind[a] == ERMC_AXIS_PERIODIC;
    P.periodic_mask |= P.periodic[a] << a;
  }
  for (int l = 0; l < c.n_levels; ++l) {
    const ermc_grid_t& g = grids[l];
    ermc_dev::LevelDesc& L = P.lv[l];
    for (int a = 0; a < 3; ++a) {
      L.n[a] = count(g, a);
      L.d[a] = spacing(g, a);
      L.rd[a] = 1.0 / L.d[a];
      L.origin[a] = g.origin[a];
      L.extent[a] = count(g, a) * spacing(g, a);
    }
    L.eps = 1e-12 * std::min({g.dx, g.dy, g.dz});
    L.cap = (l + 1 == c.n_levels) ? -1 : c.steps_per_level;
    L.field = l == 0 ? s->d_field.p : (s->d_levels.size() > size_t(l) && s->d_levels[l] ? s->d_levels[l]->p : nullptr);
    L.field32 = nullptr;
  }
  for (int a = 0; a < 3; ++a) {
    P.wall_eps[2 * a] = b.lo_emissivity[a];
    P.wall_eps[2 * a + 1] = b.hi_emissivity[a];
  }
  P.wall_ib = s->d_wall_ib.p;
  P.wall_ibn32 = s->d_wall_ibn32.p;
  P.n_bands = v.nb;
  P.n_quad = v.nq;
  P.n_temps = v.nt;
  P.uniform_temps = v.uniform ? 1 : 0;
  P.t0 = v.t0;
  P.dt = v.dt;
  P.temps = s->d_temps.p;
  P.k = s->d_k.p;
  P.ib = s->d_ib.p;
  P.band_cdf = s->d_band_cdf.p;
  P.quad_cdf = s->d_quad_cdf.p;
  P.k_max = s->d_kmax.p;
  P.pref_den = s->d_pref_den.p;
  {
    auto fast_div = [](uint32_t d) {
      ermc_dev::FastDiv f{};
      f.d = d;
      uint32_t sh = 0;
      while ((1ull << sh) < d) ++sh;
      f.s = sh;
      f.m = static_cast<uint32_t>(((1ull << 32) * ((1ull << sh) - d)) / d + 1);
      return f;
    };
    const ermc_grid_t& g0 = s->grid;
    const uint64_t nyz = static_cast<uint64_t>(g0.ny) * g0.nz;
    P.div_rays = fast_div(static_cast<uint32_t>(c.rays_per_cell));
    P.div_nyz = fast_div(nyz < (1ull << 31) ? static_cast<uint32_t>(nyz) : 1u);
    P.div_nz = fast_div(static_cast<uint32_t>(g0.nz));
    P.div_row = fast_div(static_cast<uint32_t>(std::max(1, s->view.nq * (s->view.nt - 1))));
  }
  P.ib_max = s->d_ibmax.p;
  P.qe = qe;
  P.tol = c.tolerance;
  P.max_steps = c.max_steps;
  ermc_dev::set_level_budgets(P);
  P.specular = c.specular_walls;
  P.volume_sampling = c.volume_sampling;
  P.h_seed = mix64_host(c.seed + 0x9e3779b97f4a7c15ULL);
  P.rays = c.rays_per_cell;
  P.refill_threshold = tune().refill;
  // multigrid windows: 48 steps; 64 from 6 levels on, where rays are ~22
  // steps long (7 levels: 9.14e10 vs 8.96e10 trace steps/s; 4 levels prefer
  // 48: 8.79e10 vs 8.74e10 — r2aa/r2ab)
  P.inner_steps = c.n_levels > 1
                      ? (std::getenv("ERMC_INNER_STEPS_MG") == nullptr && c.n_levels >= 6
                             ? 64
                             : tune().inner_steps_mg)
                      : tune().inner_steps;
  P.lean = tune().lean && s->tables_finite;
  P.carveout = tune().carveout;
  P.tol32 = static_cast<float>(c.tolerance);
  P.tint = s->d_tint.p;
  P.iv64 = s->d_iv64.p;
  P.inv_dt = 1.0 / v.dt;
  // tint[l] = {temps[l], temps[l+1] - temps[l], RN(1/width)}: when every node
  // is exactly l*dt + t0 (the kernel's expression, same two roundings) and
  // every width exactly dt, the record is computed in the kernel instead of
  // gathered (make_temp_grid's integer grids qualify).
  P.inv_w = 1.0 / v.dt;
  P.tint_arith = v.uniform && v.nt >= 2 && tune().tint_arith;
  for (int l = 0; P.tint_arith && l + 1 < v.nt; ++l) {
    const volatile double node = static_cast<double>(l) * v.dt;
    if (node + v.t0 != v.temps[l] || v.temps[l + 1] - v.temps[l] != v.dt) P.tint_arith = 0;
  }
  P.t_first = v.temps[0];
  P.t_last = v.temps[v.nt - 1];
  P.steps_per_level = s->d_steps.p;
  // Staged sampling tables (device_common.cuh stage_sampling): the CDFs +
  // guide tables while they are small (<= 4 KB), else the guides only — a
  // 119-band CDF (16 KB) in every block took the L1 from the gathers
  // (fp32, 119 x 16: L1 hit rate 0.4 %). ERMC_CDF_SMEM: 0 off, 1 this
  // choice, 2 guides only, 3 CDFs + guides whenever they fit 16 KB.
  {
    const int mode = tune().cdf_smem;
    const int len = v.nb * (1 + v.nq);
    const bool guides = v.nb <= 255 && v.nq <= 255;
    P.cdf_smem = !guides || mode == 0 ? 0
                 : mode == 2          ? 2
                 : mode == 3          ? (len <= ermc_dev::kMaxSmemCdf ? 1 : 2)
                                      : (len <= 512 ? 1 : 2);
  }
  P.cdf_guide = s->d_cdf_guide.p;
  // Positions matter after a wall only if some wall can reflect.
  P.track_pos = 0;
  for (int a = 0; a < 3; ++a)
    if (b.kind[a] != ERMC_AXIS_PERIODIC &&
        (b.lo_emissivity[a] != 1.0 || b.hi_emissivity[a] != 1.0))
      P.track_pos = 1;
  if (tune().track_pos) P.track_pos = 1;
}

double q_emission(const ermc_session* s, double t_max) {
  // solver.cpp:90-93
  const double kp = ermc_host::planck_mean(s->view, t_max);
  return 4.0 * kp * ermc::kSigma * t_max * t_max * t_max * t_max /
         s->config.rays_per_cell;
}

std::string error_message(const ermc_session* s, const ermc_dev::RayRecord& r,
                          int64_t cell, uint32_t ray) {
  switch (r.err) {
    case ermc_dev::kErrNonFinite:
      return "march: non-finite value at cell " + std::to_string(cell) +
             " ray " + std::to_string(ray) + " step " + std::to_string(r.steps);
    case ermc_dev::kErrTableRange:
      return "temperature " + ermc_host::fmt_double(r.err_value) +
             " K outside table range [" + ermc_host::fmt_double(s->temps.front()) +
             ", " + ermc_host::fmt_double(s->temps.back()) + "]";
    case ermc_dev::kErrTransparent:
      return "init_ray: sampled a transparent point at T_max; spectral tables "
             "are inconsistent with the sampling CDFs";
    case ermc_dev::kErrLocate:
      return "locate: point outside domain on axis " + std::to_string(r.err_axis);
    default:
      return "ermc_b200: device error " + std::to_string(r.err);
  }
}

// Re-traces one failing ray with the debug kernel to recover the message.
std::string describe_failure(ermc_session* s, const ermc_dev::TraceParams& P,
                             int64_t cell, uint32_t ray, cudaStream_t st) {
  DevBuf<int64_t> dc;
  DevBuf<uint32_t> dr;
  DevBuf<ermc_dev::RayRecord> drec;
  dc.upload(&cell, 1, st);
  dr.upload(&ray, 1, st);
  drec.ensure(1);
  cuda_check(ermc_dev::launch_trace_rays_fp64(P, 1, dc.p, dr.p, nullptr, drec.p,
                                              nullptr, st),
             "trace_rays");
  ermc_dev::RayRecord rec{};
  cuda_check(cudaMemcpyAsync(&rec, drec.p, sizeof(rec), cudaMemcpyDeviceToHost, st),
             "D2H");
  cuda_check(cudaStreamSynchronize(st), "sync");
  return error_message(s, rec, cell, ray);
}

void ensure_fp32_inputs(ermc_session* s, ermc_dev::TraceParams& P,
                        cudaStream_t st);

// fp64 lean tracer: the micro-brick copy of the field (even grids, one level).
void ensure_fp64_brick(ermc_session* s, ermc_dev::TraceParams& P, cudaStream_t st) {
  const ermc_grid_t& g0 = s->grid;
  const bool even = g0.nx % 2 == 0 && g0.ny % 2 == 0 && g0.nz % 2 == 0;
  P.brick = (tune().brick64 && even && s->config.n_levels == 1 &&
             s->n_cells < (int64_t(1) << 31)) ? 1 : 0;
  if (!P.brick) return;
  if (!s->d_field64b.p) {
    s->d_field64b.ensure(static_cast<size_t>(s->n_cells));
    cuda_check(ermc_dev::launch_to_bricked64(s->d_field.p, s->d_field64b.p, g0.nx, g0.ny,
                                             g0.nz, st),
               "to_bricked64");
    ++s->launches;
  }
  P.lv[0].field64b = s->d_field64b.p;
}

// fp64 lean tracers: cell words of every level (trace_fp64.cu decode_cw), built
// once per field. They need an exactly arithmetic temperature grid (the
// kernel's dt), at most 256 intervals, and every in-range T - t[lo] to be an
// integer multiple of 2^-s below 2^53 * 2^-s with s = 52 - floor(log2 t_first);
// the builder checks every cell and the solve keeps the temperature-reading
// tracers if one does not fit.
void ensure_cell_words(ermc_session* s, ermc_dev::TraceParams& P, cudaStream_t st) {
  const ermc_host::TableView& v = s->view;
  P.cellw = 0;
  if (!tune().cellw || !P.lean || P.brick || !P.tint_arith || v.nt < 2 || v.nt - 1 > 256 ||
      !(v.temps[0] > 0.0))
    return;
  int e = 0;
  std::frexp(v.temps[0], &e);              // t_first = f 2^e, f in [0.5, 1)
  const double scale = std::ldexp(1.0, 52 - (e - 1));  // 1 / ulp(t_first)
  const double cw_dt = v.dt * scale;
  if (!(cw_dt < 9007199254740992.0)) return;  // m must convert exactly
  P.cw_shift = 56;
  P.cw_dt = cw_dt;
  P.cw_rdt = 1.0 / cw_dt;
  if (!s->cellw_valid) {
    Timing t;
    cudaEventCreate(&t.a);
    cudaEventCreate(&t.b);
    cudaEventRecord(t.a, st);
    const size_t nl = s->level_grids.size();
    s->d_cellw.resize(nl);
    s->d_cw_bad.ensure(1);
    cuda_check(cudaMemsetAsync(s->d_cw_bad.p, 0, sizeof(int), st), "memset");
    for (size_t l = 0; l < nl; ++l) {
      if (!s->d_cellw[l]) s->d_cellw[l] = std::make_unique<DevBuf<uint64_t>>();
      const int64_t n = cells_of(s->level_grids[l]);
      s->d_cellw[l]->ensure(static_cast<size_t>(n));
      const double* field = l == 0 ? s->d_field.p : s->d_levels[l]->p;
      cuda_check(ermc_dev::launch_build_cell_words(P, field, n, scale, s->d_cellw[l]->p,
                                                   s->d_cw_bad.p, st),
                 "build_cell_words");
      ++s->launches;
    }
    cudaEventRecord(t.b, st);
    int bad = 0;
    cuda_check(cudaMemcpyAsync(&bad, s->d_cw_bad.p, sizeof(int), cudaMemcpyDeviceToHost, st),
               "D2H");
    cuda_check(cudaStreamSynchronize(st), "cell words");
    float ms = 0.f;
    cudaEventElapsedTime(&ms, t.a, t.b);
    s->ms[0] += ms;
    cudaEventDestroy(t.a);
    cudaEventDestroy(t.b);
    s->cellw_valid = true;
    s->cellw_ok = bad == 0;
  }
  if (!s->cellw_ok) return;
  for (size_t l = 0; l < s->d_cellw.size(); ++l) P.lv[l].cellw = s->d_cellw[l]->p;
  P.cellw = 1;
}

// Core solve of [lo, hi) into device outputs.
// scatter: write each cell's result into these full-field buffers at its
// global index instead of d_q / d_sd (the fused all-gather).
void session_enqueue(ermc_session* s, int64_t lo, int64_t hi, double* d_q,
                     double* d_sd, cudaStream_t st,
                     const ermc_dev::ScatterOut* scatter = nullptr) {
  if (s->pending.active) throw Error("ermc_b200: a solve is pending on this session; wait first");
  if (!s->field_set) throw Error("ermc_b200: temperature field not set");
  if (lo < 0 || hi > s->n_cells || lo > hi)
    throw Error("ermc_b200: cell range outside the grid");
  for (double& m : s->ms) m = 0.0;
  s->launches = 0;
  DeviceGuard guard(s->device);
  // set_field may have copied on another stream: order the solve after it.
  if (s->last_work) cuda_check(cudaStreamWaitEvent(st, s->last_work, 0), "stream wait");
  const double t_max = validate_field_and_tmax(s, st);
  Prepared pr;
  // build_cdfs (inside prepare) may throw before the hierarchy checks, as
  // in solver.cpp:88-96; planck_mean cannot fail for an in-range T_max.
  const double qe = q_emission(s, t_max);
  prepare(s, pr, t_max, qe, /*build_levels=*/true, st);
  ermc_dev::TraceParams& P = pr.P;
  const bool fp32 = s->config.precision == ERMC_PRECISION_FP32;
  if (fp32) {
    P.inner_steps = P.n_levels > 1 ? tune().inner_steps32_mg : tune().inner_steps32;
    ensure_fp32_inputs(s, P, st);
  }
  else {
    ensure_fp64_brick(s, P, st);
    ensure_cell_words(s, P, st);
  }

  const int R = s->config.rays_per_cell;
  const int64_t total_cells = hi - lo;
  // Chunk so the per-ray buffer stays within budget and work ids fit 31 bits.
  const size_t item_bytes = sizeof(double) + (pr.sorted ? 2 * sizeof(uint32_t) : 0);
  const uint64_t max_items = std::min<uint64_t>(
      (1ull << 31) - 1, std::max<uint64_t>(s->qray_budget_bytes / item_bytes, R));
  int64_t chunk_cells = std::max<int64_t>(1, static_cast<int64_t>(max_items / R));
  chunk_cells = std::min<int64_t>(chunk_cells, std::max<int64_t>(total_cells, 1));
  {  // whole x-planes per chunk when possible (cubic sort tiles need them)
    const int64_t plane = static_cast<int64_t>(s->grid.ny) * s->grid.nz;
    if (chunk_cells < total_cells && chunk_cells >= plane) chunk_cells -= chunk_cells % plane;
  }
  const int64_t n_chunks = total_cells == 0 ? 0 : (total_cells + chunk_cells - 1) / chunk_cells;
  s->d_qray.ensure(static_cast<size_t>(chunk_cells) * R);
  const int n_rows = s->view.nb * s->view.nq;
  if (pr.sorted) {
    s->d_keys.ensure(static_cast<size_t>(chunk_cells) * R);
    s->d_perm.ensure(static_cast<size_t>(chunk_cells) * R);
  }
  // <= 2^16 work ids per sort tile (whole cells); cubic tiles of the largest
  // edge in {ERMC_SORT_BLOCK, /2, ...} with edge^3 * R <= 2^16 (0 = linear)
  const int tile_cells = std::max(
      1, std::min(tune().sort_tile_items, ermc_dev::sort_max_tile_items()) / R);
  int sort_block = tune().sort_block;
  if (sort_block < 0 && s->config.n_levels > 1) {
    sort_block = 0;  // multigrid: the cubic tiles' slower sort is not repaid (r2bn)
  } else if (sort_block < 0) {  // auto: the largest cube of whole cells in a tile
    sort_block = 1;
    while (static_cast<int64_t>(sort_block + 1) * (sort_block + 1) * (sort_block + 1) * R <=
           (int64_t(1) << 16))
      ++sort_block;
    if (sort_block < 2) sort_block = 0;
  }
  while (sort_block > 1 &&
         static_cast<int64_t>(sort_block) * sort_block * sort_block * R > (int64_t(1) << 16))
    sort_block /= 2;
  s->d_counters.ensure(2 * std::max<int64_t>(n_chunks, 1));
  s->d_errcode.ensure(std::max<int64_t>(n_chunks, 1));
  cuda_check(cudaMemsetAsync(s->d_counters.p, 0,
                             2 * std::max<int64_t>(n_chunks, 1) * sizeof(unsigned long long), st),
             "memset");
  cuda_check(cudaMemsetAsync(s->d_errcode.p, 0, std::max<int64_t>(n_chunks, 1) * sizeof(int32_t), st),
             "memset");
  cuda_check(cudaMemsetAsync(s->d_steps.p, 0, ermc_dev::kMaxLevels * sizeof(unsigned long long), st),
             "memset");
  const int min_blocks = fp32 ? tune().fp32_min_blocks : tune().fp64_min_blocks;
  const int bps = fp32 ? ermc_dev::trace_fp32_blocks_per_sm(P, min_blocks)
                       : ermc_dev::trace_fp64_blocks_per_sm(P, min_blocks);
  const int grid = std::max(1, bps) * s->n_sm;

  std::vector<Timing> tt(n_chunks), tr(n_chunks), ts(n_chunks);
  for (int64_t ch = 0; ch < n_chunks; ++ch) {
    const int64_t c0 = lo + ch * chunk_cells;
    const int64_t nc = std::min<int64_t>(chunk_cells, hi - c0);
    P.cell_base = c0;
    P.n_cells = nc;
    P.n_work = static_cast<uint64_t>(nc) * R;
    P.work_counter = s->d_counters.p + 2 * ch;
    P.err_key = s->d_counters.p + 2 * ch + 1;
    P.err_code = s->d_errcode.p + ch;
    P.q_ray = s->d_qray.p;
    P.perm = nullptr;
    if (pr.sorted) {
      cudaEventCreate(&ts[ch].a);
      cudaEventCreate(&ts[ch].b);
      cudaEventRecord(ts[ch].a, st);
      cuda_check(ermc_dev::launch_ng_sort(P, s->d_row_rank.p, n_rows, tune().sort_dirs,
                                          tile_cells, sort_block, s->d_keys.p,
                                          s->d_perm.p, st),
                 "narrow-band sort");
      cudaEventRecord(ts[ch].b, st);
      s->launches += 1;
      P.perm = s->d_perm.p;
    }
    cudaEventCreate(&tt[ch].a);
    cudaEventCreate(&tt[ch].b);
    cudaEventCreate(&tr[ch].a);
    cudaEventCreate(&tr[ch].b);
    cudaEventRecord(tt[ch].a, st);
    cuda_check(fp32 ? ermc_dev::launch_trace_fp32(P, grid, min_blocks, st)
                    : ermc_dev::launch_trace_fp64(P, grid, min_blocks, st),
               "trace");
    cudaEventRecord(tt[ch].b, st);
    cudaEventRecord(tr[ch].a, st);
    cuda_check(scatter ? ermc_dev::launch_reduce_cells_scatter(s->d_qray.p, nc, R, *scatter, c0, st)
                       : ermc_dev::launch_reduce_cells(s->d_qray.p, nc, R, d_q + (c0 - lo),
                                                       d_sd + (c0 - lo), st),
               "reduce");
    cudaEventRecord(tr[ch].b, st);
    s->launches += 2;
  }
  // Counters, error codes and step counts into pinned host words (so the
  // copies stay asynchronous); session_finish reads them after the stream.
  const size_t n_cnt = 2 * static_cast<size_t>(std::max<int64_t>(n_chunks, 1));
  const size_t n_codes = static_cast<size_t>(std::max<int64_t>(n_chunks, 1));
  const size_t need = n_cnt + n_codes + ermc_dev::kMaxLevels;
  if (s->h_words_n < need) {
    PinnedPool::get().free(s->h_words, s->h_words_n);
    s->h_words = PinnedPool::get().alloc(need, &s->h_words_n);
  }
  cuda_check(cudaMemcpyAsync(s->h_words, s->d_counters.p, n_cnt * sizeof(unsigned long long),
                             cudaMemcpyDeviceToHost, st),
             "D2H");
  cuda_check(cudaMemcpyAsync(s->h_words + n_cnt, s->d_errcode.p, n_codes * sizeof(int32_t),
                             cudaMemcpyDeviceToHost, st),
             "D2H");
  cuda_check(cudaMemcpyAsync(s->h_words + n_cnt + n_codes, s->d_steps.p,
                             ermc_dev::kMaxLevels * sizeof(unsigned long long),
                             cudaMemcpyDeviceToHost, st),
             "D2H");
  auto& pd = s->pending;
  pd.active = true;
  pd.st = st;
  pd.lo = lo;
  pd.chunk_cells = chunk_cells;
  pd.n_chunks = n_chunks;
  pd.rays = R;
  pd.P = P;
  pd.tt = std::move(tt);
  pd.tr = std::move(tr);
  pd.ts = std::move(ts);
}

// Waits for the enqueued solve: kernel times, the error word (a failing ray
// is re-traced by the debug kernel for the reference's message), step counts.
void session_finish(ermc_session* s, int64_t* steps_out) {
  auto& pd = s->pending;
  if (!pd.active) throw Error("ermc_b200: no solve pending on this session");
  pd.active = false;
  DeviceGuard guard(s->device);
  cudaStream_t st = pd.st;
  cuda_check(cudaStreamSynchronize(st), "trace sync");
  const int64_t n_chunks = pd.n_chunks;
  const size_t n_cnt = 2 * static_cast<size_t>(std::max<int64_t>(n_chunks, 1));
  const size_t n_codes = static_cast<size_t>(std::max<int64_t>(n_chunks, 1));
  const unsigned long long* counters = s->h_words;
  const unsigned long long* steps = s->h_words + n_cnt + n_codes;
  for (int64_t ch = 0; ch < n_chunks; ++ch) {
    float a = 0.f, b = 0.f;
    cudaEventElapsedTime(&a, pd.tt[ch].a, pd.tt[ch].b);
    cudaEventElapsedTime(&b, pd.tr[ch].a, pd.tr[ch].b);
    s->ms[2] += a;
    s->ms[3] += b;
    if (pd.ts[ch].a) {
      float c = 0.f;
      cudaEventElapsedTime(&c, pd.ts[ch].a, pd.ts[ch].b);
      s->ms[1] += c;
      cudaEventDestroy(pd.ts[ch].a);
      cudaEventDestroy(pd.ts[ch].b);
    }
    cudaEventDestroy(pd.tt[ch].a);
    cudaEventDestroy(pd.tt[ch].b);
    cudaEventDestroy(pd.tr[ch].a);
    cudaEventDestroy(pd.tr[ch].b);
  }
  const int R = pd.rays;
  for (int64_t ch = 0; ch < n_chunks; ++ch) {
    const unsigned long long key = counters[2 * ch + 1];
    if (key == 0ull) continue;  // raise_error stores ~(failing work id)
    const int64_t c0 = pd.lo + ch * pd.chunk_cells;
    const uint64_t w = ~key;
    const int64_t cell = c0 + static_cast<int64_t>(w / R);
    const uint32_t ray = static_cast<uint32_t>(w % R);
    // Describe with the fp64 debug tracer (reference arithmetic).
    ermc_dev::TraceParams P = pd.P;
    P.lv[0].field = s->d_field.p;
    throw Error(describe_failure(s, P, cell, ray, st));
  }
  for (int l = 0; l < s->config.n_levels; ++l)
    steps_out[l] = static_cast<int64_t>(steps[l]);
}

void session_solve_impl(ermc_session* s, int64_t lo, int64_t hi, double* d_q,
                        double* d_sd, int64_t* steps_out, cudaStream_t st,
                        const ermc_dev::ScatterOut* scatter = nullptr) {
  session_enqueue(s, lo, hi, d_q, d_sd, st, scatter);
  session_finish(s, steps_out);
}

void set_field_impl(ermc_session* s, const double* t, int is_device,
                    cudaStream_t st) {
  // The pending solve reads d_field and the derived fp32 / brick copies that
  // this call overwrites and frees.
  if (s->pending.active)
    throw Error("ermc_b200: a solve is pending on this session; wait before set_field");
  DeviceGuard guard(s->device);
  s->d_field.ensure(static_cast<size_t>(s->n_cells));
  cuda_check(cudaMemcpyAsync(s->d_field.p, t, s->n_cells * sizeof(double),
                             is_device ? cudaMemcpyDeviceToDevice
                                       : cudaMemcpyHostToDevice,
                             st),
             "set_field copy");
  if (!s->last_work)
    cuda_check(cudaEventCreateWithFlags(&s->last_work, cudaEventDisableTiming), "event");
  cuda_check(cudaEventRecord(s->last_work, st), "event record");
  s->field_set = true;
  s->levels_valid = false;
  s->iv32_ready = s->iv32_ready;  // tables unchanged
  s->d_levels32.clear();
  s->cellw_valid = false;
  s->d_field32.reset();
  s->d_field32b.reset();
  s->d_field64b.reset();
}

void ensure_fp32_inputs(ermc_session* s, ermc_dev::TraceParams& P,
                        cudaStream_t st) {
  const ermc_host::TableView& v = s->view;
  if (v.nt < 2 || !v.uniform)
    throw Error("ermc_b200: the fp32 kernel needs a uniform temperature grid "
                "with at least 2 nodes; use precision=fp64");
  if (!s->tables_finite)
    throw Error("ermc_b200: the fp32 kernel needs finite k / Ib tables; use precision=fp64");
  for (const ermc_grid_t& g : s->level_grids)
    if (cells_of(g) >= (int64_t(1) << 31))
      throw Error("ermc_b200: the fp32 kernel supports grids below 2^31 "
                  "cells; use precision=fp64");
  if (!s->iv32_ready) {
    s->d_iv32.ensure(static_cast<size_t>(v.nb) * v.nq * (v.nt - 1));
    cuda_check(ermc_dev::launch_build_iv32(s->d_k.p, s->d_ib.p, v.nb, v.nq, v.nt,
                                           s->d_iv32.p, st),
               "build_iv32");
    ++s->launches;
    s->iv32_ready = true;
  }
  if (!s->d_field32.p) {
    s->d_field32.ensure(static_cast<size_t>(s->n_cells));
    cuda_check(ermc_dev::launch_to_fp32(s->d_field.p, s->d_field32.p, s->n_cells, st),
               "to_fp32");
    ++s->launches;
  }
  P.lv[0].field32 = s->d_field32.p;
  const ermc_grid_t& g0 = s->grid;
  // brick edge: ERMC_BRICK=4 asks for 4^3 bricks (dimensions divisible by 4),
  // otherwise 2^3 bricks on even grids
  auto divisible = [&](int b) { return g0.nx % b == 0 && g0.ny % b == 0 && g0.nz % b == 0; };
  int edge = 0;
  if (tune().brick && s->config.n_levels == 1) {
    if (tune().brick == 4 && divisible(4) && !P.track_pos) edge = 4;
    else if (divisible(2)) edge = 2;
  }
  if (s->fp32_brick_edge != edge) s->d_field32b.reset();  // layout changed
  s->fp32_brick_edge = edge;
  P.brick = edge;
  if (P.brick) {
    if (!s->d_field32b.p) {
      s->d_field32b.ensure(static_cast<size_t>(s->n_cells));
      cuda_check(ermc_dev::launch_to_fp32_bricked(s->d_field.p, s->d_field32b.p, g0.nx,
                                                  g0.ny, g0.nz, edge, st),
                 "to_fp32_bricked");
      ++s->launches;
    }
    P.lv[0].field32b = s->d_field32b.p;
  }
  s->d_levels32.resize(s->config.n_levels);
  for (int l = 1; l < s->config.n_levels; ++l) {
    const int64_t n = cells_of(s->level_grids[l]);
    if (!s->d_levels32[l]) {
      s->d_levels32[l] = std::make_unique<DevBuf<float>>();
      s->d_levels32[l]->ensure(static_cast<size_t>(n));
      cuda_check(ermc_dev::launch_to_fp32(s->d_levels[l]->p, s->d_levels32[l]->p, n, st),
                 "to_fp32");
      ++s->launches;
    }
    P.lv[l].field32 = s->d_levels32[l]->p;
  }
  P.iv32 = s->d_iv32.p;
  P.inv_dt32 = static_cast<float>(1.0 / v.dt);
  P.t0_32 = static_cast<float>(v.t0);
  P.u0_32 = -P.t0_32 * P.inv_dt32;
}

template <typename F>
int guarded(char* errbuf, size_t errlen, F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    put_err(errbuf, errlen, e.what());
    return 1;
  } catch (...) {
    put_err(errbuf, errlen, "ermc_b200: unknown error");
    return 1;
  }
}

// One part of a one-shot solve on config->device: session, H2D of the whole
// T field (replicated per device), solve of [lo, hi), D2H of Q_r / sigma
// into q_out / sd_out. Throws ermc::Error.
void solve_part(const ermc_grid_t* grid, const double* temperature,
                const ermc_boundary_t* boundary, const ermc_model_t* model,
                const ermc_config_t* config, int64_t lo, int64_t hi, double* q_out,
                double* sd_out, int64_t* steps_out) {
  const auto t0 = std::chrono::steady_clock::now();
  // ERMC_HOST_PROFILE=1: phase times of this call on stderr (diagnostics).
  static const bool prof = env_int("ERMC_HOST_PROFILE", 0) != 0;
  auto mark = [&](const char* what) {
    if (!prof) return;
    std::fprintf(stderr, "ermc_b200 solve_host: %-12s %9.3f ms\n", what,
                 std::chrono::duration<double, std::milli>(
                     std::chrono::steady_clock::now() - t0).count());
  };
  std::unique_ptr<ermc_session> s(create_session(grid, boundary, model, config));
  mark("session");
  DeviceGuard guard(s->device);
  cudaStream_t st;
  cuda_check(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "stream");
  struct StreamGuard {
    cudaStream_t s;
    ~StreamGuard() { cudaStreamDestroy(s); }
  } sg{st};
  set_field_impl(s.get(), temperature, 0, st);
  if (prof) cudaStreamSynchronize(st);
  mark("h2d field");
  const int64_t n = hi - lo;
  DevBuf<double> dq, dsd;
  dq.ensure(static_cast<size_t>(std::max<int64_t>(n, 1)));
  dsd.ensure(static_cast<size_t>(std::max<int64_t>(n, 1)));
  session_solve_impl(s.get(), lo, hi, dq.p, dsd.p, steps_out, st);
  mark("solve");
  if (n > 0) {
    cuda_check(cudaMemcpyAsync(q_out, dq.p, n * sizeof(double), cudaMemcpyDeviceToHost, st),
               "D2H q_r");
    cuda_check(cudaMemcpyAsync(sd_out, dsd.p, n * sizeof(double), cudaMemcpyDeviceToHost, st),
               "D2H std_dev");
  }
  cuda_check(cudaStreamSynchronize(st), "sync");
  mark("d2h q, sigma");
  dq.reset();
  dsd.reset();
  s.reset();
  mark("teardown");
}

// Host-buffer entry points (ermc_b200_solve / _solve_range): the range is
// split into config->n_devices contiguous parts solved concurrently, one
// host thread per part (the reference's worker chunks, solver.cpp:159-170,
// with a GPU per chunk). Each cell is computed identically wherever it runs,
// so the result does not depend on the split. The error reported is the one
// of the lowest failing part — the cells a single worker reaches first.
int solve_host(const ermc_grid_t* grid, const double* temperature,
               const ermc_boundary_t* boundary, const ermc_model_t* model,
               const ermc_config_t* config, int64_t lo, int64_t hi,
               ermc_solution_t* out, char* errbuf, size_t errlen) {
  return guarded(errbuf, errlen, [&] {
    const auto t0 = std::chrono::steady_clock::now();
    if (!out) throw Error("ermc_b200: null solution");
    if (!config) throw Error("ermc_b200: null descriptor");
    if (config->n_devices < 0) throw Error("ermc_b200: n_devices must be >= 0");
    const int parts = std::max(1, config->n_devices);
    const int n_levels = std::max(1, config->n_levels);
    std::vector<int64_t> steps(static_cast<size_t>(parts) * n_levels, 0);
    if (parts == 1) {
      solve_part(grid, temperature, boundary, model, config, lo, hi, out->q_r, out->std_dev,
                 steps.data());
    } else {
      int n_dev = 0;
      if (cudaGetDeviceCount(&n_dev) != cudaSuccess || n_dev == 0) {
        cudaGetLastError();
        throw Error("ermc_b200: no CUDA device available (the solver has no CPU path)");
      }
      int base = config->device;
      if (base < 0) cuda_check(cudaGetDevice(&base), "cudaGetDevice");
      if (base >= n_dev) throw Error("ermc_b200: device ordinal out of range");
      const int64_t n = hi - lo;
      std::vector<std::string> errors(parts);
      std::vector<std::thread> pool;
      for (int p = 0; p < parts; ++p) {
        const int64_t a = lo + n * p / parts, b = lo + n * (p + 1) / parts;
        pool.emplace_back([&, p, a, b] {
          try {
            ermc_config_t c = *config;
            c.device = (base + p) % n_dev;
            c.n_devices = 1;
            solve_part(grid, temperature, boundary, model, &c, a, b, out->q_r + (a - lo),
                       out->std_dev + (a - lo), steps.data() + static_cast<size_t>(p) * n_levels);
          } catch (const std::exception& e) {
            errors[p] = e.what();
            if (errors[p].empty()) errors[p] = "ermc_b200: unknown error";
          } catch (...) {
            errors[p] = "ermc_b200: unknown error";
          }
        });
      }
      for (auto& t : pool) t.join();
      for (const std::string& e : errors)
        if (!e.empty()) throw Error(e);
    }
    int64_t total = 0;
    for (int l = 0; l < n_levels; ++l) {
      int64_t v = 0;
      for (int p = 0; p < parts; ++p) v += steps[static_cast<size_t>(p) * n_levels + l];
      out->steps_per_level[l] = v;
      total += v;
    }
    out->total_steps = total;
    out->wall_time = std::chrono::duration<double>(
                         std::chrono::steady_clock::now() - t0).count();
  });
}

}  // namespace

extern "C" {

void ermc_b200_config_default(ermc_config_t* c) {
  std::memset(c, 0, sizeof(*c));
  c->rays_per_cell = 2000;
  c->n_levels = 1;
  c->tolerance = 1e-4;
  c->seed = 0;
  c->max_steps = 100000;
  c->sorting = 0;
  c->n_devices = 1;
  c->steps_per_level = 5;
  c->coarsen_ratio = 2;
  c->volume_sampling = 0;
  c->specular_walls = 0;
  c->workers = 0;
  c->precision = ERMC_PRECISION_FP64;
  c->device = -1;
}

int ermc_b200_solve(const ermc_grid_t* grid, const double* temperature,
                    const ermc_boundary_t* boundary, const ermc_model_t* model,
                    const ermc_config_t* config, ermc_solution_t* out,
                    char* errbuf, size_t errlen) {
  const int64_t n = grid ? cells_of(*grid) : 0;
  return solve_host(grid, temperature, boundary, model, config, 0, n, out,
                    errbuf, errlen);
}

int ermc_b200_solve_range(const ermc_grid_t* grid, const double* temperature,
                          const ermc_boundary_t* boundary,
                          const ermc_model_t* model,
                          const ermc_config_t* config, int64_t cell_lo,
                          int64_t cell_hi, ermc_solution_t* out, char* errbuf,
                          size_t errlen) {
  return solve_host(grid, temperature, boundary, model, config, cell_lo,
                    cell_hi, out, errbuf, errlen);
}

ermc_session_t* ermc_b200_session_create(const ermc_grid_t* grid,
                                         const ermc_boundary_t* boundary,
                                         const ermc_model_t* model,
                                         const ermc_config_t* config,
                                         char* errbuf, size_t errlen) {
  ermc_session* s = nullptr;
  guarded(errbuf, errlen, [&] { s = create_session(grid, boundary, model, config); });
  return s;
}

void ermc_b200_session_destroy(ermc_session_t* s) {
  if (!s) return;
  {
    DeviceGuard guard(s->device);
    delete s;
  }
}

int ermc_b200_session_set_field(ermc_session_t* s, const double* temperature,
                                int is_device, void* stream, char* errbuf,
                                size_t errlen) {
  return guarded(errbuf, errlen, [&] {
    if (!s || !temperature) throw Error("ermc_b200: null argument");
    std::lock_guard<std::mutex> lk(s->mu);
    set_field_impl(s, temperature, is_device, static_cast<cudaStream_t>(stream));
  });
}

int ermc_b200_session_solve(ermc_session_t* s, int64_t cell_lo,
                            int64_t cell_hi, double* d_q_r, double* d_std_dev,
                            int64_t* steps_per_level, void* stream,
                            char* errbuf, size_t errlen) {
  return guarded(errbuf, errlen, [&] {
    if (!s || !steps_per_level) throw Error("ermc_b200: null argument");
    std::lock_guard<std::mutex> lk(s->mu);
    session_solve_impl(s, cell_lo, cell_hi, d_q_r, d_std_dev, steps_per_level,
                       static_cast<cudaStream_t>(stream));
  });
}

int ermc_b200_session_solve_scatter(ermc_session_t* s, int64_t cell_lo, int64_t cell_hi,
                                    double* const* d_q_full, double* const* d_sd_full,
                                    int32_t n_out, int64_t* steps_per_level, void* stream,
                                    char* errbuf, size_t errlen) {
  return guarded(errbuf, errlen, [&] {
    if (!s || !steps_per_level || !d_q_full || !d_sd_full) throw Error("ermc_b200: null argument");
    if (n_out < 1 || n_out > ermc_dev::kMaxScatter)
      throw Error("ermc_b200: n_out must be in [1, " + std::to_string(ermc_dev::kMaxScatter) + "]");
    ermc_dev::ScatterOut out{};
    out.n = n_out;
    for (int p = 0; p < n_out; ++p) {
      if (!d_q_full[p] || !d_sd_full[p]) throw Error("ermc_b200: null output buffer");
      out.q[p] = d_q_full[p];
      out.sd[p] = d_sd_full[p];
    }
    std::lock_guard<std::mutex> lk(s->mu);
    session_solve_impl(s, cell_lo, cell_hi, nullptr, nullptr, steps_per_level,
                       static_cast<cudaStream_t>(stream), &out);
  });
}

int ermc_b200_device_alloc(int device, size_t bytes, void** d_ptr, char* errbuf,
                           size_t errlen) {
  return guarded(errbuf, errlen, [&] {
    if (!d_ptr) throw Error("ermc_b200: null argument");
    DeviceGuard g(device);
    cuda_check(cudaMalloc(d_ptr, std::max<size_t>(bytes, 1)), "cudaMalloc");
  });
}

int ermc_b200_device_free(void* d_ptr) {
  return cudaFree(d_ptr) == cudaSuccess ? 0 : 1;
}

int ermc_b200_ipc_export(const void* d_ptr, uint8_t handle[64], char* errbuf, size_t errlen) {
  return guarded(errbuf, errlen, [&] {
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
    cudaIpcMemHandle_t h;
    cuda_check(cudaIpcGetMemHandle(&h, const_cast<void*>(d_ptr)), "cudaIpcGetMemHandle");
    std::memcpy(handle, &h, 64);
  });
}

int ermc_b200_ipc_open(const uint8_t handle[64], void** d_ptr, char* errbuf, size_t errlen) {
  return guarded(errbuf, errlen, [&] {
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, 64);
    cuda_check(cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess),
               "cudaIpcOpenMemHandle");
  });
}

int ermc_b200_ipc_close(void* d_ptr) {
  return cudaIpcCloseMemHandle(d_ptr) == cudaSuccess ? 0 : 1;
}

int ermc_b200_session_solve_async(ermc_session_t* s, int64_t cell_lo, int64_t cell_hi,
                                  double* d_q_r, double* d_std_dev, void* stream,
                                  char* errbuf, size_t errlen) {
  return guarded(errbuf, errlen, [&] {
    if (!s) throw Error("ermc_b200: null argument");
    std::lock_guard<std::mutex> lk(s->mu);
    session_enqueue(s, cell_lo, cell_hi, d_q_r, d_std_dev, static_cast<cudaStream_t>(stream));
  });
}

int ermc_b200_session_wait(ermc_session_t* s, int64_t* steps_per_level, char* errbuf,
                           size_t errlen) {
  return guarded(errbuf, errlen, [&] {
    if (!s || !steps_per_level) throw Error("ermc_b200: null argument");
    std::lock_guard<std::mutex> lk(s->mu);
    session_finish(s, steps_per_level);
  });
}

int ermc_b200_session_timings(const ermc_session_t* s, double* ms4,
                              int32_t* n_launches) {
  if (!s) return 1;
  for (int i = 0; i < 4; ++i) ms4[i] = s->ms[i];
  if (n_launches) *n_launches = s->launches;
  return 0;
}

int ermc_b200_trace_rays(const ermc_grid_t* grid, const double* temperature,
                         const ermc_boundary_t* boundary,
                         const ermc_model_t* model, const ermc_config_t* config,
                         double t_max, double q_emission, int64_t n,
                         const int64_t* cell_ids, const uint32_t* ray_ids,
                         const double* dir_override, ermc_ray_result_t* out,
                         int64_t* level_steps, char* errbuf, size_t errlen) {
  return guarded(errbuf, errlen, [&] {
    std::unique_ptr<ermc_session> s(create_session(grid, boundary, model, config));
    DeviceGuard guard(s->device);
    cudaStream_t st = nullptr;
    set_field_impl(s.get(), temperature, 0, st);
    Prepared pr;
    prepare(s.get(), pr, t_max, q_emission, true, st);
    DevBuf<int64_t> dc;
    DevBuf<uint32_t> dr;
    DevBuf<double> dd;
    DevBuf<ermc_dev::RayRecord> drec;
    DevBuf<int64_t> dls;
    dc.upload(cell_ids, n, st);
    dr.upload(ray_ids, n, st);
    if (dir_override) dd.upload(dir_override, 3 * n, st);
    drec.ensure(n);
    if (level_steps) dls.ensure(static_cast<size_t>(n) * config->n_levels);
    cuda_check(ermc_dev::launch_trace_rays_fp64(pr.P, n, dc.p, dr.p,
                                                dir_override ? dd.p : nullptr,
                                                drec.p, level_steps ? dls.p : nullptr, st),
               "trace_rays");
    std::vector<ermc_dev::RayRecord> recs(n);
    cuda_check(cudaMemcpy(recs.data(), drec.p, n * sizeof(ermc_dev::RayRecord),
                          cudaMemcpyDeviceToHost), "D2H");
    if (level_steps)
      cuda_check(cudaMemcpy(level_steps, dls.p, n * config->n_levels * sizeof(int64_t),
                            cudaMemcpyDeviceToHost), "D2H");
    for (int64_t i = 0; i < n; ++i) {
      const ermc_dev::RayRecord& r = recs[i];
      if (r.err != ermc_dev::kErrNone)
        throw Error(error_message(s.get(), r, cell_ids[i], ray_ids[i]));
      ermc_ray_result_t& o = out[i];
      std::memset(&o, 0, sizeof(o));
      o.q_contribution = r.q;
      o.weight_absorbed = r.w_abs;
      o.weight_walls = r.w_walls;
      o.weight_residual = r.w_res;
      for (int a = 0; a < 3; ++a) o.dir[a] = r.dir[a];
      o.prefactor = r.prefactor;
      o.ib_source = r.ib_source;
      o.steps = r.steps;
      o.terminated_by = r.term;
      o.reflections = r.reflections;
      o.band = r.band;
      o.quad = r.quad;
      o.next_draw = r.next_draw;
    }
  });
}

namespace {
void require_device() {
  int n_dev = 0;
  if (cudaGetDeviceCount(&n_dev) != cudaSuccess || n_dev == 0) {
    cudaGetLastError();
    throw Error("ermc_b200: no CUDA device available (the solver has no CPU path)");
  }
}

// The reference's RayRecord -> ermc_ray_result_t (ermc_b200_trace_rays too).
void copy_result(const ermc_dev::RayRecord& r, ermc_ray_result_t& o) {
  std::memset(&o, 0, sizeof(o));
  o.q_contribution = r.q;
  o.weight_absorbed = r.w_abs;
  o.weight_walls = r.w_walls;
  o.weight_residual = r.w_res;
  for (int a = 0; a < 3; ++a) o.dir[a] = r.dir[a];
  o.prefactor = r.prefactor;
  o.ib_source = r.ib_source;
  o.steps = r.steps;
  o.terminated_by = r.term;
  o.reflections = r.reflections;
  o.band = r.band;
  o.quad = r.quad;
  o.next_draw = r.next_draw;
}
}  // namespace

int ermc_b200_sample_direction(int64_t n, const double* r_theta, const double* r_phi,
                               double* out, char* errbuf, size_t errlen) {
  return guarded(errbuf, errlen, [&] {
    require_device();
    if (n <= 0) return;
    cudaStream_t st = nullptr;
    DevBuf<double> a, b, o;
    a.upload(r_theta, n, st);
    b.upload(r_phi, n, st);
    o.ensure(5 * static_cast<size_t>(n));
    cuda_check(ermc_dev::launch_sample_direction(n, a.p, b.p, o.p, st), "sample_direction");
    cuda_check(cudaMemcpy(out, o.p, 5 * n * sizeof(double), cudaMemcpyDeviceToHost), "D2H");
  });
}

int ermc_b200_absorptivity(int64_t n, const double* kappa, const double* ds, double* out,
                           char* errbuf, size_t errlen) {
  return guarded(errbuf, errlen, [&] {
    require_device();
    if (n <= 0) return;
    cudaStream_t st = nullptr;
    DevBuf<double> a, b, o;
    a.upload(kappa, n, st);
    b.upload(ds, n, st);
    o.ensure(n);
    cuda_check(ermc_dev::launch_absorptivity(n, a.p, b.p, o.p, st), "absorptivity");
    cuda_check(cudaMemcpy(out, o.p, n * sizeof(double), cudaMemcpyDeviceToHost), "D2H");
  });
}

int ermc_b200_init_rays(const ermc_grid_t* grid, const double* temperature,
                        const ermc_model_t* model, const double* band_cdf,
                        const double* quad_cdf, double t_max, uint64_t seed,
                        int32_t volume_sampling, int64_t n, const int32_t* cells,
                        const uint32_t* ray_ids, ermc_ray_state_t* out, char* errbuf,
                        size_t errlen) {
  return guarded(errbuf, errlen, [&] {
    ermc_config_t cfg;
    ermc_b200_config_default(&cfg);
    cfg.rays_per_cell = 1;
    cfg.seed = seed;
    cfg.volume_sampling = volume_sampling;
    ermc_boundary_t b{};  // init_ray reads no wall
    for (int a = 0; a < 3; ++a) {
      b.kind[a] = ERMC_AXIS_PERIODIC;
      b.lo_emissivity[a] = b.hi_emissivity[a] = 1.0;
    }
    std::unique_ptr<ermc_session> s(create_session(grid, &b, model, &cfg));
    DeviceGuard guard(s->device);
    cudaStream_t st = nullptr;
    set_field_impl(s.get(), temperature, 0, st);
    Prepared pr;
    prepare(s.get(), pr, t_max, 1.0, false, st);
    // the caller's CDFs (a SamplingCdfs need not come from build_cdfs)
    const ermc_host::TableView& v = s->view;
    s->d_band_cdf.upload(band_cdf, v.nb, st);
    s->d_quad_cdf.upload(quad_cdf, static_cast<size_t>(v.nb) * v.nq, st);
    pr.P.band_cdf = s->d_band_cdf.p;
    pr.P.quad_cdf = s->d_quad_cdf.p;
    DevBuf<int32_t> dc, de;
    DevBuf<uint32_t> dr;
    DevBuf<ermc_ray_state_t> dout;
    dc.upload(cells, 3 * static_cast<size_t>(n), st);
    dr.upload(ray_ids, n, st);
    de.ensure(n);
    dout.ensure(n);
    cuda_check(ermc_dev::launch_init_states_fp64(pr.P, n, dc.p, dr.p, seed, dout.p, de.p, st),
               "init_rays");
    std::vector<int32_t> errs(n);
    cuda_check(cudaMemcpy(errs.data(), de.p, n * sizeof(int32_t), cudaMemcpyDeviceToHost),
               "D2H");
    for (int64_t i = 0; i < n; ++i)
      if (errs[i] != ermc_dev::kErrNone) {
        ermc_dev::RayRecord rec{};
        rec.err = errs[i];
        rec.err_value = temperature[(static_cast<int64_t>(cells[3 * i]) * grid->ny +
                                     cells[3 * i + 1]) * grid->nz + cells[3 * i + 2]];
        throw Error(error_message(s.get(), rec, 0, ray_ids[i]));
      }
    cuda_check(cudaMemcpy(out, dout.p, n * sizeof(ermc_ray_state_t), cudaMemcpyDeviceToHost),
               "D2H");
  });
}

int ermc_b200_march_rays(int32_t n_levels, const ermc_grid_t* grids,
                         const double* const* fields, const int32_t* step_caps,
                         const ermc_model_t* model, const ermc_boundary_t* boundary,
                         double q_emission, double tolerance, int64_t max_steps,
                         int32_t specular, int64_t n, const ermc_ray_state_t* rays,
                         ermc_ray_result_t* out, int64_t* level_steps, char* errbuf,
                         size_t errlen) {
  return guarded(errbuf, errlen, [&] {
    if (n_levels < 1 || n_levels > ermc_dev::kMaxLevels)
      throw Error("march: hierarchy must have 1 to 16 levels");
    ermc_config_t cfg;
    ermc_b200_config_default(&cfg);
    cfg.rays_per_cell = 1;
    std::unique_ptr<ermc_session> s(create_session(&grids[0], boundary, model, &cfg));
    DeviceGuard guard(s->device);
    cudaStream_t st = nullptr;
    set_field_impl(s.get(), fields[0], 0, st);
    Prepared pr;
    prepare(s.get(), pr, s->temps.back(), q_emission, false, st);  // T_max: CDFs unused
    ermc_dev::TraceParams& P = pr.P;
    // the caller's hierarchy, level by level (GridHierarchy, geometry.hpp:74-83)
    std::vector<DevBuf<double>> lv(n_levels);
    P.n_levels = n_levels;
    for (int l = 0; l < n_levels; ++l) {
      const ermc_grid_t& g = grids[l];
      validate_grid(g);
      ermc_dev::LevelDesc& L = P.lv[l];
      for (int a = 0; a < 3; ++a) {
        L.n[a] = count(g, a);
        L.d[a] = spacing(g, a);
        L.rd[a] = 1.0 / L.d[a];
        L.origin[a] = g.origin[a];
        L.extent[a] = count(g, a) * spacing(g, a);
      }
      L.eps = 1e-12 * std::min({g.dx, g.dy, g.dz});
      L.cap = step_caps[l];
      if (l == 0) {
        L.field = s->d_field.p;
      } else {
        lv[l].upload(fields[l], static_cast<size_t>(cells_of(g)), st);
        L.field = lv[l].p;
      }
    }
    P.qe = q_emission;
    P.tol = tolerance;
    P.max_steps = max_steps;
    ermc_dev::set_level_budgets(P);
    P.specular = specular;
    DevBuf<ermc_ray_state_t> din;
    DevBuf<ermc_dev::RayRecord> drec;
    DevBuf<int64_t> dls;
    din.upload(rays, n, st);
    drec.ensure(n);
    if (level_steps) dls.ensure(static_cast<size_t>(n) * n_levels);
    cuda_check(ermc_dev::launch_march_states_fp64(P, n, din.p, drec.p,
                                                  level_steps ? dls.p : nullptr, st),
               "march_rays");
    std::vector<ermc_dev::RayRecord> recs(n);
    cuda_check(cudaMemcpy(recs.data(), drec.p, n * sizeof(ermc_dev::RayRecord),
                          cudaMemcpyDeviceToHost), "D2H");
    if (level_steps)
      cuda_check(cudaMemcpy(level_steps, dls.p, n * n_levels * sizeof(int64_t),
                            cudaMemcpyDeviceToHost), "D2H");
    for (int64_t i = 0; i < n; ++i) {
      if (recs[i].err != ermc_dev::kErrNone)
        throw Error(error_message(s.get(), recs[i], static_cast<int64_t>(rays[i].cell_id),
                                  rays[i].ray_id));
      copy_result(recs[i], out[i]);
    }
  });
}

int ermc_b200_build_cdfs(const ermc_model_t* model, double t_max,
                         double* band_cdf, double* quad_cdf, char* errbuf,
                         size_t errlen) {
  return guarded(errbuf, errlen, [&] {
    ermc_host::TableView v = ermc_host::make_view(*model);
    ermc_host::build_cdfs(v, t_max, band_cdf, quad_cdf);
  });
}

int ermc_b200_planck_mean(const ermc_model_t* model, double temperature,
                          double* out, char* errbuf, size_t errlen) {
  return guarded(errbuf, errlen, [&] {
    ermc_host::TableView v = ermc_host::make_view(*model);
    *out = ermc_host::planck_mean(v, temperature);
  });
}

int ermc_b200_uniform_device(uint64_t seed, int64_t n, const uint64_t* cell_ids,
                             const uint32_t* ray_ids, const uint32_t* draw_ids,
                             double* out, char* errbuf, size_t errlen) {
  return guarded(errbuf, errlen, [&] {
    int n_dev = 0;
    if (cudaGetDeviceCount(&n_dev) != cudaSuccess || n_dev == 0) {
      cudaGetLastError();
      throw Error("ermc_b200: no CUDA device available (the solver has no CPU path)");
    }
    cudaStream_t st = nullptr;
    DevBuf<uint64_t> dc;
    DevBuf<uint32_t> dr, dd;
    DevBuf<double> dout;
    dc.upload(cell_ids, n, st);
    dr.upload(ray_ids, n, st);
    dd.upload(draw_ids, n, st);
    dout.ensure(n);
    cuda_check(ermc_dev::launch_uniform(mix64_host(seed + 0x9e3779b97f4a7c15ULL), n,
                                        dc.p, dr.p, dd.p, dout.p, st),
               "uniform");
    cuda_check(cudaMemcpy(out, dout.p, n * sizeof(double), cudaMemcpyDeviceToHost),
               "D2H");
  });
}

int ermc_b200_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int ermc_b200_abi_version(void) { return ERMC_B200_ABI_VERSION; }

int ermc_b200_release_cached_memory(int device) {
  int dev = device;
  if (dev < 0 && cudaGetDevice(&dev) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  DevicePool::get().release(dev);
  return 0;
}

}  // extern "C"
