// Calibration probe: per-SM streaming bandwidth of 1-D bulk copies (cp.async.bulk) with a
// ring of `stages` x `chunk` bytes in flight, versus plain 128-bit vector loads.
#include <cstdint>
#include <cuda.h>
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


// Tensor-map (cp.async.bulk.tensor.2d) variant: rows of 128 B (64 bf16), box of chunk / 128 rows (<= 256),
// 128-byte swizzle; `issuers` warps each run an independent ring of stages / issuers slots over their own
// rows (issuers > 1 also for the 1-D variant below: does the SM's TMA unit overlap ops of several issuers?)
__global__ void tensor_stream(const __grid_constant__ CUtensorMap map, long rows_per_cta, int box_rows, int stages,
                              int issuers, int tensor, const uint8_t* src, unsigned long long* sink, long wrap_rows) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const int chunk = box_rows * 128;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + stages * chunk);
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) mbar_init(&full[s], 1);
    fence_barrier_init();
  }
  __syncthreads();
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) != 0 || w >= issuers) return;
  const int per = stages / issuers;                 // this issuer's slots [w * per, (w + 1) * per)
  const long n = rows_per_cta / box_rows / issuers; // ops of this issuer
  const uint64_t pol = policy_evict_normal();
  auto row_of = [&](long i) { return ((long)blockIdx.x * 0 + (i * issuers + w) * box_rows) % wrap_rows; };
  auto issue = [&](int s, long i) {
    mbar_expect_tx(&full[s], chunk);
    if (tensor) tma_load_2d(sm + s * chunk, &map, &full[s], 0, (int)row_of(i), pol);
    else bulk_load(sm + s * chunk, src + row_of(i) * 128, chunk, &full[s], pol);
  };
  long issued = 0;
  for (; issued < n && issued < per; ++issued) issue(w * per + (int)issued, issued);
  unsigned long long acc = 0;
  for (long i = 0; i < n; ++i) {
    const int s = w * per + (int)(i % per);
    mbar_wait(&full[s], (i / per) & 1);
    acc += sm[s * chunk + (i & 63)];
    if (issued < n) issue(s, issued++);
  }
  sink[blockIdx.x * 8 + w] = acc;
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
extern "C" int probe_tensor(const void* src, long rows_total, long rows_per_cta, int box_rows, int stages, int issuers,
                            int tensor, int ctas, void* sink, cudaStream_t s) {
  static EncFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess) return -1;
    fn = reinterpret_cast<EncFn>(p);
  }
  CUtensorMap m;
  cuuint64_t dims[2] = {64, (cuuint64_t)rows_total};
  cuuint64_t strides[1] = {128};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  if (fn(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(src), dims, strides, box, es,
         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return -2;
  const int smem = stages * box_rows * 128 + stages * 8 + 64;
  cudaFuncSetAttribute(tensor_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
  tensor_stream<<<ctas, 32 * issuers, smem, s>>>(m, rows_per_cta, box_rows, stages, issuers, tensor,
                                                 (const uint8_t*)src, (unsigned long long*)sink, rows_total);
  return (int)cudaGetLastError();
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

// ---------------------------------------------------------------- tcgen05 cta_group::2 issue-rate probe
// One cluster of 2 CTAs (an SM pair), operands = whatever is in smem (timing only): the leader issues
// groups of 8 UMMAs M = 256 (128 rows per SM), N = n split over the pair, K = 16 each.
__global__ void __cluster_dims__(2, 1, 1) mma2_probe(int n, int groups, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  if (warp == 0) tmem_alloc2<512>(&tslot);
  if (threadIdx.x == 32) { mbar_init(&bar, 1); fence_barrier_init(); }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (rank == 0 && warp == 1 && lane == 0) {
    const uint32_t idesc = make_idesc_bf16(256, n, 0, 0);
    const uint32_t a = smem_u32(sm), b = smem_u32(sm + 32768);
    const int atom_b = (n / 2) * 128;
    long long t0 = clock64();
    for (int g = 0; g < groups; ++g) {
      for (int k = 0; k < 8; ++k) {
        const uint64_t ad = make_sdesc(a + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024, 128);
        const uint64_t bd = make_sdesc(b + (k >> 2) * atom_b + (k & 3) * 32, 16, 1024, 128);
        tc_mma2_f16(tmem, ad, bd, idesc, (g | k) ? 1u : 0u);
      }
    }
    long long t1 = clock64();
    tc_commit2_mc(&bar, 3);
    mbar_wait(&bar, 0);
    long long t2 = clock64();
    out[0] = t1 - t0;
    out[1] = t2 - t0;
  }
  if (rank == 1 && threadIdx.x == 32) mbar_wait(&bar, 0);
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  if (warp == 0) { tc_fence_after(); tmem_dealloc2<512>(tmem); }
}

extern "C" int probe_mma2(int n, int groups, void* out, cudaStream_t s) {
  cudaFuncSetAttribute(mma2_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  mma2_probe<<<2, 128, 200 * 1024, s>>>(n, groups, (unsigned long long*)out);
  return (int)cudaGetLastError();
}
