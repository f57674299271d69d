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

constexpr int kSortBlock = 256;
constexpr int kMaxSortBins = 8192;  // >= the 8001 rows of a line-by-line model

namespace {

__device__ __forceinline__ uint32_t work_key(const TraceParams& P,
                                             const int32_t* __restrict__ row_rank,
                                             uint32_t w) {
  const uint32_t rays = static_cast<uint32_t>(P.rays);
  const uint32_t c = w / rays;
  const uint32_t ray = w - c * rays;
  const uint64_t h_cell =
      mix64(P.h_seed ^ static_cast<uint64_t>(P.cell_base + static_cast<int64_t>(c)));
  int n, g;
  sample_band(P, draw_u(h_cell, ray, 2), draw_u(h_cell, ray, 3), n, g);
  return static_cast<uint32_t>(__ldg(row_rank + n * P.n_quad + g));
}

// One block per spatial tile of `tile_cells` whole cells (tile_cells * R
// work ids). The sort is local to the tile: keys, histogram, scan and
// scatter all stay in shared memory and the tile's own slice of perm, so it
// needs no global atomics, and the dispatch order keeps the cell-major
// order's spatial locality — the rays in flight at any time start from a
// couple of neighbouring tiles, so their temperature gathers share the L2
// the way unsorted rays do — while consecutive lanes draw the same row.
__global__ void __launch_bounds__(kSortBlock)
    ng_tile_sort(const __grid_constant__ TraceParams P, const int32_t* __restrict__ row_rank,
                 int n_bins, uint32_t tile_items, uint16_t* __restrict__ keys,
                 uint32_t* __restrict__ perm) {
  __shared__ unsigned int s_cur[kMaxSortBins];
  __shared__ unsigned int s_part[kSortBlock];
  const unsigned lane = threadIdx.x & 31u;
  const unsigned lt = (1u << lane) - 1u;
  const uint32_t n = static_cast<uint32_t>(P.n_work);
  const uint32_t t0 = blockIdx.x * tile_items;
  const uint32_t t1 = min(n, t0 + tile_items);
  for (int b = threadIdx.x; b < n_bins; b += blockDim.x) s_cur[b] = 0u;
  __syncthreads();
  // keys + histogram (warp-aggregated shared atomics: hot rows are common)
  for (uint32_t base = t0; base < t1; base += blockDim.x) {
    const uint32_t w = base + threadIdx.x;
    const bool valid = w < t1;
    const unsigned key = valid ? work_key(P, row_rank, w) : 0xffffffffu;
    const unsigned peers = __match_any_sync(kFullMask, key);
    if (valid) {
      keys[w] = static_cast<uint16_t>(key);
      if (lane == static_cast<unsigned>(__ffs(peers) - 1)) atomicAdd(&s_cur[key], __popc(peers));
    }
  }
  __syncthreads();
  // exclusive scan of the histogram in place: per-thread segments, then a
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
  // scatter into the tile's slice of perm (ascending ids inside a warp)
  for (uint32_t base = t0; base < t1; base += blockDim.x) {
    const uint32_t w = base + threadIdx.x;
    const bool valid = w < t1;
    const unsigned key = valid ? keys[w] : 0xffffffffu;
    const unsigned peers = __match_any_sync(kFullMask, key);
    const int leader = __ffs(peers) - 1;
    unsigned int pos = 0;
    if (valid && static_cast<int>(lane) == leader) pos = atomicAdd(&s_cur[key], __popc(peers));
    pos = __shfl_sync(kFullMask, pos, leader);
    if (valid) perm[t0 + pos + __popc(peers & lt)] = w;
  }
}

}  // namespace

int sort_max_bins() { return kMaxSortBins; }

cudaError_t launch_ng_sort(const TraceParams& P, const int32_t* row_rank, int n_bins,
                           int tile_cells, uint16_t* keys, uint32_t* perm, cudaStream_t s) {
  if (P.n_work == 0) return cudaSuccess;
  if (n_bins > kMaxSortBins) return cudaErrorInvalidValue;
  const uint32_t tile_items = static_cast<uint32_t>(tile_cells) * static_cast<uint32_t>(P.rays);
  const uint32_t n = static_cast<uint32_t>(P.n_work);
  const uint32_t tiles = (n + tile_items - 1) / tile_items;
  ng_tile_sort<<<tiles, kSortBlock, 0, s>>>(P, row_rank, n_bins, tile_items, keys, perm);
  return cudaGetLastError();
}

}  // namespace ermc_dev
