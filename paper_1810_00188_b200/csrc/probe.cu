// L2 bandwidth probe: the denominator of the L2 roofline bench.py reports
// beside the HBM one ("also report the L2 fraction using a
// measured L2 bandwidth"). No reference counterpart — the reference has no
// device; this is measurement plumbing of the C-ABI, not part of a solve.
//
// mode 0 (stream): every thread reads 16-byte vectors with ld.global.cg
//   (cached in L2 only, so no L1 hit can inflate the figure) in a
//   grid-stride sweep over an L2-resident buffer, `iters` sweeps.
// mode 1 (gather): every thread reads one 8-byte word at a hashed position
//   per load, i.e. one 32-byte L2 sector per request — the access pattern of
//   the trace kernel's temperature gather. Reported as sector bytes/s.
// One CTA per SM x 8 (148 SMs), 512 threads.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstring>

#include "ermc_b200.h"

namespace {

__global__ void __launch_bounds__(512) l2_stream(const uint4* __restrict__ buf, size_t n_vec,
                                                 int iters, uint32_t* __restrict__ sink) {
  uint32_t acc = 0;
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  for (int it = 0; it < iters; ++it) {
    for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n_vec; i += stride) {
      uint4 v = __ldcg(buf + i);
      acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
  }
  if (acc == 0x9e3779b9u) sink[0] = acc;  // keeps the loads alive
}

__global__ void __launch_bounds__(512) l2_gather(const uint64_t* __restrict__ buf,
                                                 uint64_t n_words, int loads,
                                                 uint32_t* __restrict__ sink) {
  uint64_t acc = 0;
  uint64_t h = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) * 0x9e3779b97f4a7c15ull + 1;
  for (int i = 0; i < loads; ++i) {
    h ^= h >> 29;
    h *= 0xbf58476d1ce4e5b9ull;
    h ^= h >> 32;
    acc += __ldcg(buf + (h % n_words));  // the next address depends on no load: MLP-limited only
  }
  if (acc == 0x9e3779b9ull) sink[0] = uint32_t(acc);
}

void put(char* errbuf, size_t errlen, const char* msg) {
  if (errbuf && errlen) {
    std::strncpy(errbuf, msg, errlen - 1);
    errbuf[errlen - 1] = '\0';
  }
}

}  // namespace

extern "C" int ermc_b200_probe_l2(int device, size_t bytes, int iters, int mode, double* gbs,
                                  char* errbuf, size_t errlen) {
  if (!gbs || bytes < (1u << 20) || iters < 1 || (mode != 0 && mode != 1)) {
    put(errbuf, errlen, "ermc_b200_probe_l2: invalid arguments");
    return 1;
  }
  int prev = 0;
  cudaGetDevice(&prev);
  if (device >= 0 && cudaSetDevice(device) != cudaSuccess) {
    cudaGetLastError();
    put(errbuf, errlen, "ermc_b200_probe_l2: no such device");
    return 1;
  }
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device < 0 ? prev : device);
  void* buf = nullptr;
  uint32_t* sink = nullptr;
  cudaStream_t st = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  int rc = 0;
  do {
    if (cudaMalloc(&buf, bytes) != cudaSuccess || cudaMalloc(&sink, 64) != cudaSuccess ||
        cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreate(&e0) != cudaSuccess || cudaEventCreate(&e1) != cudaSuccess) {
      rc = 1;
      break;
    }
    cudaMemsetAsync(buf, 0x5a, bytes, st);
    const int blocks = sms * 8, threads = 512;
    const size_t n_vec = bytes / sizeof(uint4);
    const uint64_t n_words = bytes / sizeof(uint64_t);
    const int loads = 256;
    auto launch = [&]() {
      if (mode == 0)
        l2_stream<<<blocks, threads, 0, st>>>(static_cast<const uint4*>(buf), n_vec, iters, sink);
      else
        l2_gather<<<blocks, threads, 0, st>>>(static_cast<const uint64_t*>(buf), n_words,
                                              loads * iters, sink);
    };
    launch();  // warm: the buffer becomes L2-resident
    launch();
    cudaEventRecord(e0, st);
    launch();
    cudaEventRecord(e1, st);
    if (cudaEventSynchronize(e1) != cudaSuccess) {
      rc = 1;
      break;
    }
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double moved = mode == 0 ? double(n_vec) * sizeof(uint4) * iters
                                   : double(blocks) * threads * loads * iters * 32.0;
    *gbs = moved / (double(ms) * 1e-3) / 1e9;
  } while (false);
  cudaError_t err = cudaGetLastError();
  if (rc || err != cudaSuccess) {
    char msg[256];
    std::snprintf(msg, sizeof msg, "ermc_b200_probe_l2: %s", cudaGetErrorString(err));
    put(errbuf, errlen, msg);
    rc = 1;
  }
  if (e0) cudaEventDestroy(e0);
  if (e1) cudaEventDestroy(e1);
  if (st) cudaStreamDestroy(st);
  if (sink) cudaFree(sink);
  if (buf) cudaFree(buf);
  cudaSetDevice(prev);
  return rc;
}
