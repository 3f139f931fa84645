// Calibration probe: per-SM streaming bandwidth of 1-D bulk copies (cp.async.bulk) with a
// ring of `stages` x `chunk` bytes in flight, versus plain 128-bit vector loads.
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2512_12977_b200/csrc/vlc_ptx.cuh"
using namespace vlc;

__global__ void bulk_stream(const uint8_t* src, long bytes_per_cta, int chunk, int stages, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + stages * chunk);
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) mbar_init(&full[s], 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const uint8_t* base = src + (long)blockIdx.x * bytes_per_cta;
  const long n = bytes_per_cta / chunk;
  const uint64_t pol = policy_evict_first();
  unsigned long long acc = 0;
  long issued = 0;
  for (; issued < n && issued < stages; ++issued) {
    mbar_expect_tx(&full[issued], chunk);
    bulk_load(sm + issued * chunk, base + issued * chunk, chunk, &full[issued], pol);
  }
  for (long i = 0; i < n; ++i) {
    const int s = i % stages;
    mbar_wait(&full[s], (i / stages) & 1);
    acc += sm[s * chunk + (i & 63)];
    if (issued < n) {
      mbar_expect_tx(&full[s], chunk);
      bulk_load(sm + s * chunk, base + issued * chunk, chunk, &full[s], pol);
      ++issued;
    }
  }
  sink[blockIdx.x] = acc;
}

__global__ void ldg_stream(const uint4* src, long vec_per_cta, unsigned long long* sink) {
  const uint4* base = src + (long)blockIdx.x * vec_per_cta;
  unsigned acc = 0;
#pragma unroll 8
  for (long i = threadIdx.x; i < vec_per_cta; i += blockDim.x) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(base + i));
    acc ^= v.x ^ v.w;
  }
  if (acc == 0x12345) sink[blockIdx.x] = acc;
}

extern "C" int probe_bulk(const void* src, long bytes_per_cta, int chunk, int stages, int ctas, void* sink, cudaStream_t s) {
  const int smem = stages * chunk + stages * 8 + 64;
  cudaFuncSetAttribute(bulk_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
  bulk_stream<<<ctas, 32, smem, s>>>((const uint8_t*)src, bytes_per_cta, chunk, stages, (unsigned long long*)sink);
  return (int)cudaGetLastError();
}
extern "C" int probe_ldg(const void* src, long bytes_per_cta, int ctas, int threads, void* sink, cudaStream_t s) {
  ldg_stream<<<ctas, threads, 0, s>>>((const uint4*)src, bytes_per_cta / 16, (unsigned long long*)sink);
  return (int)cudaGetLastError();
}
