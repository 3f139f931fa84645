// Calibration probe: per-SM streaming bandwidth of 1-D bulk copies (cp.async.bulk) with a
// ring of `stages` x `chunk` bytes in flight, versus plain 128-bit vector loads.
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2512_12977_b200/csrc/vlc_ptx.cuh"
using namespace vlc;

__global__ void bulk_stream(const uint8_t* src, long bytes_per_cta, int chunk, int stages, unsigned long long* sink,
                            long wrap = 0, int shared = 0) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + stages * chunk);
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) mbar_init(&full[s], 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  // wrap > 0: the CTA re-reads a window of `wrap` bytes (L2-resident after the first pass); shared: all
  // CTAs read the same window
  const uint8_t* base = src + (wrap > 0 ? (shared ? 0 : (long)blockIdx.x * wrap) : (long)blockIdx.x * bytes_per_cta);
  auto at = [&](long i) { return base + (wrap > 0 ? (i * chunk) % wrap : i * chunk); };
  const long n = bytes_per_cta / chunk;
  const uint64_t pol = wrap > 0 ? policy_evict_normal() : policy_evict_first();
  unsigned long long acc = 0;
  long issued = 0;
  for (; issued < n && issued < stages; ++issued) {
    mbar_expect_tx(&full[issued], chunk);
    bulk_load(sm + issued * chunk, at(issued), chunk, &full[issued], pol);
  }
  for (long i = 0; i < n; ++i) {
    const int s = i % stages;
    mbar_wait(&full[s], (i / stages) & 1);
    acc += sm[s * chunk + (i & 63)];
    if (issued < n) {
      mbar_expect_tx(&full[s], chunk);
      bulk_load(sm + s * chunk, at(issued), chunk, &full[s], pol);
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

// ---------------------------------------------------------------- tcgen05 issue-rate probe
// One CTA, operands = whatever is in smem (timing only).  variant bits:
//  1: commit to an mbarrier after every group of 8 MMAs (else once at the end)
//  2: wait that mbarrier before the next group (serialising, like a 1-deep pipeline)
__global__ void mma_probe(int n, int groups, int variant, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) tmem_alloc<512>(&tslot);
  if (threadIdx.x == 32) { mbar_init(&bar, 1); fence_barrier_init(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (warp == 1 && lane == 0) {
    const uint32_t idesc = make_idesc_bf16(128, n, 0, 0);
    const uint32_t a = smem_u32(sm), b = smem_u32(sm + 32768);
    long long t0 = clock64();
    for (int g = 0; g < groups; ++g) {
      for (int k = 0; k < 8; ++k) {
        const uint64_t ad = make_sdesc(a + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024, 128);
        const uint64_t bd = make_sdesc(b + (k >> 2) * 32768 + (k & 3) * 32, 16, 1024, 128);
        tc_mma_f16(tmem, ad, bd, idesc, (g | k) ? 1u : 0u);
      }
      if (variant & 1) tc_commit(&bar);
      if (variant & 2) { mbar_wait(&bar, g & 1); tc_fence_after(); }
    }
    long long t1 = clock64();
    tc_commit(&bar);
    mbar_wait(&bar, (variant & 1) ? (groups & 1) : 0);
    long long t2 = clock64();
    if (blockIdx.x == 0) {
      out[0] = t1 - t0;  // issue loop
      out[1] = t2 - t0;  // until all MMAs complete
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<512>(tmem); }
}

extern "C" int probe_mma(int n, int groups, int variant, void* out, cudaStream_t s, int ctas) {
  cudaFuncSetAttribute(mma_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  mma_probe<<<ctas, 128, 200 * 1024, s>>>(n, groups, variant, (unsigned long long*)out);
  return (int)cudaGetLastError();
}

extern "C" int probe_bulk_l2(const void* src, long bytes_per_cta, int chunk, int stages, int ctas, long wrap, int shared,
                             void* sink, cudaStream_t s) {
  const int smem = stages * chunk + stages * 8 + 64;
  cudaFuncSetAttribute(bulk_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
  bulk_stream<<<ctas, 32, smem, s>>>((const uint8_t*)src, bytes_per_cta, chunk, stages, (unsigned long long*)sink,
                                     wrap, shared);
  return (int)cudaGetLastError();
}
