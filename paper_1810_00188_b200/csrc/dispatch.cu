// dispatch.cu — narrow-band sorted ray dispatch (the paper's "narrow-band
// sorting"; the reference's presample_and_sort,
// solver.cpp:62-80, as a GPU scheduling pass).
//
// Every (cell, ray) work item of a chunk draws its (band, g) pair from the
// reference's keyed stream (draws 2 and 3, sampling.cpp:42-53, 77-78) before
// any ray is traced. A counting sort then orders the work ids by
// k(band, g, T_max) ascending — the reference's sort key — with ties kept in
// (band, g) order, so the trace kernel's persistent ray pool hands
// consecutive lanes rays of the same spectral row:
//   * the per-step interval-record gathers of a warp land on one table row
//     (a few cache lines instead of one line per lane — the L1 wavefront
//     count of the record load was the kernel's largest cost);
//   * rays of similar optical thickness, hence similar length, run side by
//     side (the paper's divergence argument).
// The order never changes a result: each ray still writes q_ray[ray][cell]
// and K2 reduces in ray-id order (P5 byte-identity with sorting on or off).
//
// K4 ng_tile_sort: per spatial tile of whole cells, the key (rank of the
// ray's spectral row) of every work id, a shared-memory counting sort, and
// the tile's slice of the dispatch order.
#include <cuda_runtime.h>

#include <cstdint>

#include "device_common.cuh"

namespace ermc_dev {

constexpr int kSortBlock = 512;
constexpr int kMaxSortBins = 8192;  // >= the 8001 rows of a line-by-line model

namespace {

// std::upper_bound (sampling.cpp:44-51) over a CDF in shared or global memory.
__device__ __forceinline__ int upper_bound_any(const double* a, int n, double x) {
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

// One block per spatial tile of `tile_items` work ids (whole cells). The sort
// is local to the tile — a shared-memory counting sort writing the tile's
// own slice of perm — so it needs no global atomics, and the dispatch order
// keeps the cell-major order's spatial locality: the rays in flight at any
// time start from a couple of neighbouring tiles, so their temperature
// gathers share the L2 the way unsorted rays do, while consecutive lanes
// draw the same spectral row.
//   pass 1: key and the item's rank inside its bin (the shared atomic's old
//           value), packed as key << 16 | rank (tile_items <= 2^16);
//   scan:   bin offsets;
//   pass 2: perm[tile + offset[key] + rank] = id — no atomics.
// Dynamic shared memory: n_bins counters, kSortBlock partial sums, and the
// band / g CDFs when they fit (cdf_len > 0).
// Tile geometry. Linear: tile t = work ids [t * items, (t + 1) * items).
// Blocked (the chunk is whole x-planes): tile t = a bx^3 block of cells —
// (tx, ty, tz) in x-major block order, clipped at the chunk's faces — so the
// rays that share a spectral row and direction bin also start within a few
// cells of each other and their temperature gathers share cache lines.
struct TileGeom {
  uint32_t items;     // linear: work ids per tile
  int b;              // blocked: block edge (0 = linear tiles)
  int nx, ny, nz;     // blocked: chunk planes, grid ny, nz
  int nby, nbz;       // blocked: blocks along y, z
};

// Work id of item u of tile t, the tile's first dispatch position, its item
// count.
struct TileMap {
  const TileGeom& g;
  uint32_t rays;
  uint32_t t;
  int tx, ty, tz, cx, cy, cz;
  __device__ TileMap(const TileGeom& geo, uint32_t r, uint32_t tile, uint32_t n_work)
      : g(geo), rays(r), t(tile) {
    if (g.b == 0) {
      tx = ty = tz = cx = cy = cz = 0;
      return;
    }
    tz = static_cast<int>(t % g.nbz);
    ty = static_cast<int>((t / g.nbz) % g.nby);
    tx = static_cast<int>(t / (g.nbz * g.nby));
    cx = min(g.b, g.nx - tx * g.b);
    cy = min(g.b, g.ny - ty * g.b);
    cz = min(g.b, g.nz - tz * g.b);
  }
  __device__ uint32_t first(uint32_t n_work) const {
    if (g.b == 0) return t * g.items;
    const uint64_t cells = static_cast<uint64_t>(tx) * g.b * g.ny * g.nz +
                           static_cast<uint64_t>(cx) * (static_cast<uint64_t>(ty) * g.b * g.nz +
                                                        static_cast<uint64_t>(cy) * tz * g.b);
    return static_cast<uint32_t>(cells * rays);
  }
  __device__ uint32_t count(uint32_t n_work) const {
    if (g.b == 0) return min(n_work - t * g.items, g.items);
    return static_cast<uint32_t>(cx * cy * cz) * rays;
  }
  __device__ uint32_t work(uint32_t u, uint32_t n_work) const {
    if (g.b == 0) return t * g.items + u;
    const uint32_t lc = u / rays, ray = u - lc * rays;
    const int dk = static_cast<int>(lc % cz);
    const int dj = static_cast<int>((lc / cz) % cy);
    const int di = static_cast<int>(lc / (cz * cy));
    const uint32_t cell = (static_cast<uint32_t>(tx * g.b + di) * g.ny + (ty * g.b + dj)) * g.nz +
                          (tz * g.b + dk);
    return cell * rays + ray;
  }
};

__global__ void __launch_bounds__(kSortBlock)
    ng_tile_sort(const __grid_constant__ TraceParams P, const int32_t* __restrict__ row_rank,
                 int n_bins, int dir_bins, int cdf_len, TileGeom geo,
                 uint32_t* __restrict__ packed,
                 uint32_t* __restrict__ perm) {
  extern __shared__ __align__(8) unsigned char s_raw[];
  double* s_cdf = reinterpret_cast<double*>(s_raw);
  unsigned int* s_cur = reinterpret_cast<unsigned int*>(
      s_raw + (cdf_len && P.cdf_smem ? cdf_smem_bytes(P.n_bands, P.n_quad)
                                     : cdf_len * sizeof(double)));
  unsigned int* s_part = s_cur + n_bins;
  const uint32_t n = static_cast<uint32_t>(P.n_work);
  const uint32_t rays = static_cast<uint32_t>(P.rays);
  const TileMap tm(geo, rays, blockIdx.x, n);
  const uint32_t t0 = tm.first(n);
  const uint32_t cnt = tm.count(n);
  const int nb = P.n_bands, nq = P.n_quad;
  for (int b = threadIdx.x; b < n_bins; b += blockDim.x) s_cur[b] = 0u;
  // the staged CDFs carry their guide tables (trace kernels' layout) when
  // the session built them (P.cdf_smem)
  const bool guided = cdf_len && P.cdf_smem;
  for (int b = threadIdx.x; b < cdf_len; b += blockDim.x)
    s_cdf[b] = b < nb ? P.band_cdf[b] : P.quad_cdf[b - nb];
  if (guided) {
    uint8_t* gdst = reinterpret_cast<uint8_t*>(s_cdf + cdf_len);
    for (int i = threadIdx.x; i < kGuideBand + nb * kGuideQuad; i += blockDim.x)
      gdst[i] = P.cdf_guide[i];
  }
  __syncthreads();
  const double* band_cdf = cdf_len ? s_cdf : P.band_cdf;
  const double* quad_cdf = cdf_len ? s_cdf + nb : P.quad_cdf;
  for (uint32_t u = threadIdx.x; u < cnt; u += blockDim.x) {
    const uint32_t w = tm.work(u, n);
    // sample_band on draws 2 and 3 of the ray's key (sampling.cpp:42-53, 77-78)
    const uint32_t c = fdiv(w, P.div_rays);
    const uint32_t ray = w - c * rays;
    const uint64_t h_cell =
        mix64(P.h_seed ^ static_cast<uint64_t>(P.cell_base + static_cast<int64_t>(c)));
    int bn, g;
    if (guided) {
      sample_band_cdf(P, s_cdf, draw_u(h_cell, ray, 2), draw_u(h_cell, ray, 3), bn, g);
    } else {
      bn = upper_bound_any(band_cdf, nb, draw_u(h_cell, ray, 2));
      if (bn >= nb) bn = nb - 1;
      g = upper_bound_any(quad_cdf + bn * nq, nq, draw_u(h_cell, ray, 3));
      if (g >= nq) g = nq - 1;
    }
    unsigned key = static_cast<unsigned>(__ldg(row_rank + bn * nq + g));
    if (dir_bins > 1) {
      // Direction bin from draws 0 and 1 (sampling.cpp:31-40): cos(theta) =
      // 1 - 2 u0 and phi = 2 pi u1, binned uniformly in u0 and u1, so rays of
      // one spectral row that travel alike sit in adjacent lanes.
      const int nth = dir_bins >= 32 ? 4 : 2;
      const int nph = dir_bins / nth;
      const int bt = min(static_cast<int>(draw_u(h_cell, ray, 0) * nth), nth - 1);
      const int bp = min(static_cast<int>(draw_u(h_cell, ray, 1) * nph), nph - 1);
      key = key * dir_bins + bt * nph + bp;
    }
    const unsigned rank = atomicAdd(&s_cur[key], 1u);
    packed[w] = key << 16 | rank;
  }
  __syncthreads();
  // exclusive scan of the counts in place: per-thread segments, then a
  // serial scan of the kSortBlock segment sums
  const int per = (n_bins + kSortBlock - 1) / kSortBlock;
  const int b0 = threadIdx.x * per;
  const int b1 = min(n_bins, b0 + per);
  unsigned int sum = 0;
  for (int b = b0; b < b1; ++b) sum += s_cur[b];
  s_part[threadIdx.x] = sum;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int run = 0;
    for (int t = 0; t < kSortBlock; ++t) {
      const unsigned int v = s_part[t];
      s_part[t] = run;
      run += v;
    }
  }
  __syncthreads();
  unsigned int run = s_part[threadIdx.x];
  for (int b = b0; b < b1; ++b) {
    const unsigned int v = s_cur[b];
    s_cur[b] = run;
    run += v;
  }
  __syncthreads();
  for (uint32_t u = threadIdx.x; u < cnt; u += blockDim.x) {
    const uint32_t w = tm.work(u, n);
    const uint32_t kr = packed[w];
    perm[t0 + s_cur[kr >> 16] + (kr & 0xffffu)] = w;
  }
}

}  // namespace

int sort_max_bins() { return kMaxSortBins; }
int sort_max_tile_items() { return 1 << 16; }

// tile_cells: cells per linear tile; block: edge of the cubic tiles when the
// chunk is whole x-planes (0 = linear tiles).
cudaError_t launch_ng_sort(const TraceParams& P, const int32_t* row_rank, int n_rows,
                           int dir_bins, int tile_cells, int block, uint32_t* packed,
                           uint32_t* perm, cudaStream_t s) {
  while (dir_bins > 1 && n_rows * dir_bins > kMaxSortBins) dir_bins /= 2;
  const int n_bins = n_rows * dir_bins;
  if (P.n_work == 0) return cudaSuccess;
  const uint32_t rays = static_cast<uint32_t>(P.rays);
  const uint32_t tile_items = static_cast<uint32_t>(tile_cells) * rays;
  if (n_bins > kMaxSortBins || tile_items > (1u << 16)) return cudaErrorInvalidValue;
  TileGeom geo{tile_items, 0, 0, 0, 0, 0, 0};
  const int64_t plane = static_cast<int64_t>(P.lv[0].n[1]) * P.lv[0].n[2];
  if (block > 0 && P.cell_base % plane == 0 && P.n_cells % plane == 0 &&
      static_cast<uint64_t>(block) * block * block * rays <= (1u << 16)) {
    geo.b = block;
    geo.nx = static_cast<int>(P.n_cells / plane);
    geo.ny = P.lv[0].n[1];
    geo.nz = P.lv[0].n[2];
    geo.nby = (geo.ny + block - 1) / block;
    geo.nbz = (geo.nz + block - 1) / block;
  }
  const int cdf_total = P.n_bands + P.n_bands * P.n_quad;
  const int cdf_len = cdf_total <= 4096 ? cdf_total : 0;
  const size_t cdf_bytes = cdf_len && P.cdf_smem ? cdf_smem_bytes(P.n_bands, P.n_quad)
                                                 : cdf_len * sizeof(double);
  const size_t smem = cdf_bytes + (n_bins + kSortBlock) * sizeof(unsigned int);
  if (smem > 48 * 1024) {
    const cudaError_t e = cudaFuncSetAttribute(
        ng_tile_sort, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  const uint32_t n = static_cast<uint32_t>(P.n_work);
  const uint32_t tiles = geo.b ? static_cast<uint32_t>((geo.nx + geo.b - 1) / geo.b) * geo.nby * geo.nbz
                               : (n + tile_items - 1) / tile_items;
  ng_tile_sort<<<tiles, kSortBlock, smem, s>>>(P, row_rank, n_bins, dir_bins, cdf_len, geo,
                                               packed, perm);
  return cudaGetLastError();
}

}  // namespace ermc_dev
