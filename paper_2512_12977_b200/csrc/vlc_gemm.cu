// Weight-streaming tcgen05 GEMM for the recomputed rows of the reuse prefill.
//
//   acc[f, j] = sum_k W[f, k] * X[j, k]          (swap-AB: weights on UMMA M)
//
// W is the layer weight stored K-major on device ([n_out, k] with k contiguous),
// X the activations of the c computed tokens ([rows, k], bf16).  A CTA owns a
// 128-row weight tile and one <=256-token tile; the K range may be split across
// CTAs (split-K, deterministic "last CTA reduces").  One elected thread issues
// the TMA loads (warp 0) and another the tcgen05.mma chain into TMEM (warp 1);
// four epilogue warps read TMEM with tcgen05.ld and apply the fused epilogue:
//   QKV_ROPE  Q/K rotated at the token's position (engine.py:176-180), K/V scattered
//             into the request KV cache rows, pre-RoPE K kept for the result
//   RESID     x += acc (fp32 residual, engine.py:183,185)
//   SWIGLU    silu(gate) * up -> bf16 (model.py:262-265)
//   F32       logits (engine.py:187)
//   BIAS_ADD  encoder patch embedding + bias + positional rows (model.py:316)
//   QKV_PLAIN encoder projections (model.py:318)
#include "vlc_internal.h"

namespace vlc {

constexpr int GEMM_THREADS = 192;
constexpr int GEMM_BM = 128;
constexpr int GEMM_BK = 64;

__device__ __forceinline__ float silu_f(float g) { return g / (1.0f + expf(-g)); }

__device__ __forceinline__ void store_bf16(void* base, long idx, float v) {
  reinterpret_cast<__nv_bfloat16*>(base)[idx] = __float2bfloat16_rn(v);
}

// Apply the epilogue to 16 consecutive token columns (j0 .. j0+15) of this thread's
// weight row f.  Per-token metadata is fetched once per warp (lane i loads token j0+i,
// then broadcast with shuffles) and every global load of the chunk is issued before
// any store, so the chunk costs ~one memory round trip instead of sixteen.
__device__ __forceinline__ void epilogue_chunk(const GemmEpi& e, int f, int j0, const float* v) {
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int hb = lane & 16;  // metadata of token j0+i lives in lane hb+i (half-warps may differ in j0)
  const int jl = j0 + (lane & 15);
  const bool jl_ok = jl < e.m_tokens;
  const int m1_l = (e.map1 && jl_ok) ? __ldg(e.map1 + jl) : jl;
  const int m2_l = (e.map2 && jl_ok) ? __ldg(e.map2 + jl) : jl;
  const int ps_l = (e.pos && jl_ok) ? __ldg(e.pos + jl) : 0;
  const int nv = min(16, e.m_tokens - j0);
  const bool row_ok = f < e.n_valid;
  switch (e.kind) {
    case EPI_F32: {
      float* __restrict__ o = reinterpret_cast<float*>(e.out) + f;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int r = __shfl_sync(FULL, m1_l, hb + i);
        if (row_ok && i < nv) o[(long)r * e.ldo] = v[i];
      }
      break;
    }
    case EPI_RESID: {
      float* __restrict__ o = reinterpret_cast<float*>(e.out) + f;
      float old[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) old[i] = (row_ok && i < nv) ? o[(long)(j0 + i) * e.ldo] : 0.f;
#pragma unroll
      for (int i = 0; i < 16; ++i)
        if (row_ok && i < nv) o[(long)(j0 + i) * e.ldo] = old[i] + v[i];
      break;
    }
    case EPI_BF16: {
#pragma unroll
      for (int i = 0; i < 16; ++i)
        if (row_ok && i < nv) store_bf16(e.out, (long)(j0 + i) * e.ldo + f, v[i]);
      break;
    }
    case EPI_BIAS_ADD: {
      const float b = (e.bias && row_ok) ? __ldg(e.bias + f) : 0.f;
      float a[16];
#pragma unroll
      for (int i = 0; i < 16; ++i)
        a[i] = (e.add && row_ok && i < nv) ? __ldg(e.add + (long)(j0 + i) * e.ld_add + f) : 0.f;
      float* __restrict__ o = reinterpret_cast<float*>(e.out) + f;
#pragma unroll
      for (int i = 0; i < 16; ++i)
        if (row_ok && i < nv) o[(long)(j0 + i) * e.ldo] = (v[i] + b) + a[i];
      break;
    }
    case EPI_SWIGLU: {
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const float up = __shfl_xor_sync(FULL, v[i], 1);
        if (row_ok && i < nv && (f & 1) == 0) store_bf16(e.out, (long)(j0 + i) * e.ldo + (f >> 1), silu_f(v[i]) * up);
      }
      break;
    }
    case EPI_QKV_PLAIN: {
      const int sec = f / e.seg, r = f - sec * e.seg;
      void* dst = sec == 0 ? e.out : sec == 1 ? e.out2 : e.out3;
      const int ld = sec == 0 ? e.ldo : sec == 1 ? e.ld2 : e.ld3;
#pragma unroll
      for (int i = 0; i < 16; ++i)
        if (row_ok && i < nv) store_bf16(dst, (long)(j0 + i) * ld + r, v[i]);
      break;
    }
    case EPI_QKV_ROPE: {
      const int sec = f / e.seg, r = f - sec * e.seg;
      float partner[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) partner[i] = __shfl_xor_sync(FULL, v[i], 1);
      if (sec == 2) {  // V: not permuted, not rotated
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int kr = __shfl_sync(FULL, m2_l, hb + i);
          if (row_ok && i < nv) store_bf16(e.out3, (long)kr * e.ld3 + r, v[i]);
        }
        break;
      }
      const int half = e.hd >> 1;
      const int head = r / e.hd, w = r - head * e.hd, t = w >> 1, odd = w & 1;
      const int feat = head * e.hd + (odd ? t + half : t);
      float c[16], sn[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int p = __shfl_sync(FULL, ps_l, hb + i);
        const long tab = (long)p * e.tab_ld + t;
        c[i] = row_ok ? __ldg(e.cos_tab + tab) : 0.f;
        sn[i] = row_ok ? __ldg(e.sin_tab + tab) : 0.f;
      }
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const float a = odd ? partner[i] : v[i], b = odd ? v[i] : partner[i];
        const float rot = odd ? (b * c[i] + a * sn[i]) : (a * c[i] - b * sn[i]);
        const int q_row = __shfl_sync(FULL, m1_l, hb + i);
        const int kv_row = __shfl_sync(FULL, m2_l, hb + i);
        if (!(row_ok && i < nv)) continue;
        if (sec == 0) {
          store_bf16(e.out, (long)q_row * e.ldo + feat, rot);
        } else {
          if (e.out4) store_bf16(e.out4, (long)(j0 + i) * e.ld4 + feat, v[i]);
          store_bf16(e.out2, (long)kv_row * e.ld2 + feat, rot);
        }
      }
      break;
    }
    default:
      break;
  }
}

// ------------------------------------------------------------------ stream-K schedule
struct SkSched {
  long long U;   // total work units = tiles * KB
  int G;         // CTAs (all co-resident: cooperative launch)
  int KB;        // k-blocks per tile
  int m_tiles;
  __device__ __forceinline__ long long u0(int g) const { return U * g / G; }
  __device__ __forceinline__ int cta_of(long long u) const {
    int g = (int)((u * G) / U);
    while (g + 1 < G && u0(g + 1) <= u) ++g;
    while (g > 0 && u0(g) > u) --g;
    return g;
  }
};

constexpr int SK_MAX_PART = 8;  // participants per split tile

__global__ void __launch_bounds__(GEMM_THREADS, 1)
    gemm_bf16_tc(const __grid_constant__ CUtensorMap map_w, const __grid_constant__ CUtensorMap map_x,
                 GemmEpi epi, SkSched sk, int n_tile, int stages, float* ws, int* counters) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int a_bytes = GEMM_BM * GEMM_BK * 2;
  const int b_bytes = n_tile * GEMM_BK * 2;
  uint8_t* sa = smem;
  uint8_t* sb = smem + stages * a_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(sb + stages * b_bytes);
  uint64_t* empty = full + stages;
  uint64_t* acc_full = empty + stages;   // [2]
  uint64_t* acc_empty = acc_full + 2;    // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const uint32_t warp = warp_id(), lane = lane_id();
  const int g = blockIdx.x;
  const long long u_begin = sk.u0(g), u_end = sk.u0(g + 1);
  const int t_first = (int)(u_begin / sk.KB);
  const int t_last = (u_end > u_begin) ? (int)((u_end - 1) / sk.KB) : t_first - 1;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&map_w);
    tma_prefetch(&map_x);
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&acc_full[s], 1);
      mbar_init(&acc_empty[s], 128);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol_w = policy_evict_first();
      const uint64_t pol_x = policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      for (int t = t_first; t <= t_last; ++t) {
        const long long tb = (long long)t * sk.KB;
        const int kb_lo = (int)(max(u_begin, tb) - tb), kb_hi = (int)(min(u_end, tb + sk.KB) - tb);
        const int m0 = (t % sk.m_tiles) * GEMM_BM, tok0 = (t / sk.m_tiles) * n_tile;
        for (int kb = kb_lo; kb < kb_hi; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_expect_tx(&full[stage], a_bytes + b_bytes);
          tma_load_2d(sa + stage * a_bytes, &map_w, &full[stage], kb * GEMM_BK, m0, pol_w);
          tma_load_2d(sb + stage * b_bytes, &map_x, &full[stage], kb * GEMM_BK, tok0, pol_x);
          if (++stage == stages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = make_idesc_bf16(GEMM_BM, n_tile, 0, 0);
      int stage = 0;
      uint32_t phase = 0;
      int seg = 0;
      for (int t = t_first; t <= t_last; ++t, ++seg) {
        const long long tb = (long long)t * sk.KB;
        const int nkb = (int)(min(u_end, tb + sk.KB) - max(u_begin, tb));
        const int slot = seg & 1;
        mbar_wait(&acc_empty[slot], ((seg >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + slot * 256;
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(sa + stage * a_bytes);
          const uint32_t b_addr = smem_u32(sb + stage * b_bytes);
#pragma unroll
          for (int k = 0; k < GEMM_BK / 16; ++k) {
            const uint64_t ad = make_sdesc(a_addr + k * 32, 16, 1024, 128);
            const uint64_t bd = make_sdesc(b_addr + k * 32, 16, 1024, 128);
            tc_mma_f16(d, ad, bd, idesc, (kb > 0 || k > 0) ? 1u : 0u);
          }
          tc_commit(&empty[stage]);
          if (++stage == stages) { stage = 0; phase ^= 1; }
        }
        tc_commit(&acc_full[slot]);
      }
    }
    __syncwarp();
  } else {
    // ---------------- epilogue warps 2..5 (threads 64..191)
    const int quad = warp & 3;
    const int row = quad * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    const int nchunks = n_tile / 16;
    int seg = 0;
    for (int t = t_first; t <= t_last; ++t, ++seg) {
      const long long tb = (long long)t * sk.KB;
      const int gf = sk.cta_of(tb), gl = sk.cta_of(tb + sk.KB - 1);
      const int m0 = (t % sk.m_tiles) * GEMM_BM, tok0 = (t / sk.m_tiles) * n_tile;
      const int slot = seg & 1;
      mbar_wait(&acc_full[slot], (seg >> 1) & 1);
      tc_fence_after();
      const uint32_t d = tmem + slot * 256 + lane_off;
      if (gf == gl) {
        for (int c = 0; c < nchunks; ++c) {
          float v[16];
          tmem_ld16(d + c * 16, v);
          tmem_wait_ld();
          epilogue_chunk(epi, m0 + row, tok0 + c * 16, v);
        }
        tc_fence_before();
        mbar_arrive(&acc_empty[slot]);
      } else {
        float* part = ws + (((long)gf * SK_MAX_PART + (g - gf)) * GEMM_BM + row) * (long)n_tile;
        for (int c = 0; c < nchunks; ++c) {
          float v[16];
          tmem_ld16(d + c * 16, v);
          tmem_wait_ld();
          float4* dst = reinterpret_cast<float4*>(part + c * 16);
#pragma unroll
          for (int q = 0; q < 4; ++q) __stcg(dst + q, make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]));
        }
        tc_fence_before();
        mbar_arrive(&acc_empty[slot]);
        __threadfence();
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (threadIdx.x == 64) atomicAdd(&counters[2 * gf], 1);
      }
    }
    // ---- parallel fixup of the split tiles this CTA touched (first and/or last segment)
    for (int t = t_first; t <= t_last; ++t) {
      const long long tb = (long long)t * sk.KB;
      const int gf = sk.cta_of(tb), gl = sk.cta_of(tb + sk.KB - 1);
      if (gf == gl) continue;
      const int nseg = gl - gf + 1, p = g - gf;
      if (threadIdx.x == 64) {
        volatile int* cnt = counters + 2 * gf;
        while (*cnt < nseg) __nanosleep(64);
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      __threadfence();
      const int m0 = (t % sk.m_tiles) * GEMM_BM, tok0 = (t / sk.m_tiles) * n_tile;
      const int u_lo = p * 8 / nseg, u_hi = (p + 1) * 8 / nseg;   // 16-row units owned by this CTA
      const int nu = u_hi - u_lo;
      const int total = nu * nchunks;
      const int half = lane >> 4;
      const float* base = ws + (long)gf * SK_MAX_PART * GEMM_BM * n_tile;
      const long pstride = (long)GEMM_BM * n_tile;
      for (int pr = quad; pr < (total + 1) / 2; pr += 4) {
        const int w = 2 * pr + half;
        const bool ok = w < total;
        const int unit = u_lo + (ok ? w % nu : 0), chunk = ok ? w / nu : 0;
        const int r = unit * 16 + (lane & 15);
        float v[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = 0.f;
        if (ok) {
          for (int s = 0; s < nseg; ++s) {
            const float4* src = reinterpret_cast<const float4*>(base + s * pstride + (long)r * n_tile + chunk * 16);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const float4 x = __ldcg(src + q);
              v[4 * q] += x.x; v[4 * q + 1] += x.y; v[4 * q + 2] += x.z; v[4 * q + 3] += x.w;
            }
          }
        }
        epilogue_chunk(epi, ok ? m0 + r : 0x7fffffff, tok0 + chunk * 16, v);
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (threadIdx.x == 64) {
        if (atomicAdd(&counters[2 * gf + 1], 1) == nseg - 1) {
          counters[2 * gf] = 0;
          counters[2 * gf + 1] = 0;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

int g_stage_override = 0;

static int gemm_pick_stages(int n_tile) {
  if (g_stage_override > 0) return g_stage_override;
  const int per = GEMM_BM * GEMM_BK * 2 + n_tile * GEMM_BK * 2;
  int s = (200 * 1024) / per;
  if (s > 8) s = 8;
  if (s < 2) s = 2;
  return s;
}

static int gemm_smem_bytes(int n_tile, int stages) {
  return 1024 + stages * (GEMM_BM * GEMM_BK * 2 + n_tile * GEMM_BK * 2) + (2 * stages + 4) * 8 + 16;
}

static int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

// ws must hold G * SK_MAX_PART * 128 * n_tile floats; counters 2 * G ints (zero).
cudaError_t launch_gemm(const void* W, int n_pad, int k_pad, const void* X, int x_rows_cap,
                        int m_tokens, const GemmEpi& epi, int max_ctas, float* ws, size_t ws_bytes,
                        int* counters, cudaStream_t stream) {
  if (m_tokens <= 0) return cudaSuccess;
  const int KB = k_pad / GEMM_BK;
  const int m_tiles = n_pad / GEMM_BM;
  int n_tile = m_tokens >= 256 ? 256 : ((m_tokens + 15) / 16) * 16;
  if (n_tile < 16) n_tile = 16;
  const int tok_tiles = (m_tokens + n_tile - 1) / n_tile;
  const long long U = (long long)m_tiles * tok_tiles * KB;
  int G = num_sms();
  if (max_ctas > 0 && max_ctas < G) G = max_ctas;
  const int min_units = (KB + 5) / 6;  // keeps <= 8 participants per split tile
  if ((long long)G * min_units > U) G = (int)(U / min_units);
  if (G < 1) G = 1;
  const size_t need = (size_t)G * SK_MAX_PART * GEMM_BM * n_tile * sizeof(float);
  if (need > ws_bytes || counters == nullptr) {
    // no workspace: one CTA per tile, never split
    if (U / KB <= num_sms()) G = (int)(U / KB);
    else return cudaErrorInvalidValue;
  }
  CUtensorMap mw, mx;
  cudaError_t err = make_tmap_2d(&mw, W, k_pad, n_pad, (uint64_t)k_pad * 2, GEMM_BK, GEMM_BM, 128);
  if (err != cudaSuccess) return err;
  err = make_tmap_2d(&mx, X, k_pad, x_rows_cap, (uint64_t)k_pad * 2, GEMM_BK, n_tile, 128);
  if (err != cudaSuccess) return err;
  const int stages = gemm_pick_stages(n_tile);
  const int smem = gemm_smem_bytes(n_tile, stages);
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(gemm_bf16_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
    attr_set = true;
  }
  SkSched sk{U, G, KB, m_tiles};
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(G);
  cfg.blockDim = dim3(GEMM_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, gemm_bf16_tc, mw, mx, epi, sk, n_tile, stages, ws, counters);
}

}  // namespace vlc
