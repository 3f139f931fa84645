// Mixed attention of the reuse prefill (engine.py:179-182, model.py:268-291):
// the recomputed queries of one request attend, causally by ABSOLUTE position,
// over every key of the request -- cached keys re-rotated by kv_relocate and
// fresh keys written by the QKV epilogue.  Flash-style on tcgen05:
//   S = Q K^T  (UMMA 128x128xHD, accumulator in TMEM)
//   softmax in registers (one thread per query row, exp2 domain, lazy rescale)
//   O += P V   (P staged in smem K-major, V consumed MN-major, O in TMEM)
// One CTA = (request, head, <=128 queries, key range); key ranges may be split
// across CTAs, merged by attn_combine.
#include "vlc_internal.h"

namespace vlc {

constexpr int ATT_THREADS = 192;
constexpr int ATT_STAGES = 2;

template <int HD>
struct AttnCfg {
  static constexpr int ATOM_E = HD < 64 ? HD : 64;        // elements per swizzled row
  static constexpr int SWZ = ATOM_E * 2;                  // swizzle width in bytes
  static constexpr int N_ATOMS = HD / ATOM_E;
  static constexpr int TILE_BYTES = 128 * HD * 2;         // 128 rows x HD
  static constexpr int ATOM_BYTES = 128 * SWZ;
  static constexpr int P_BYTES = 128 * 128 * 2;
  static constexpr int SMEM = 1024 + TILE_BYTES * (1 + 2 * ATT_STAGES) + P_BYTES + 256;
};

template <int HD>
__global__ void __launch_bounds__(ATT_THREADS, 1)
    attn_fwd_tc(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_k,
                const __grid_constant__ CUtensorMap map_v, vlc_attn_args a) {
  using C = AttnCfg<HD>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sK = sQ + C::TILE_BYTES;
  uint8_t* sV = sK + ATT_STAGES * C::TILE_BYTES;
  uint8_t* sP = sV + ATT_STAGES * C::TILE_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sP + C::P_BYTES);
  uint64_t* q_full = bars;
  uint64_t* kv_full = bars + 1;
  uint64_t* kv_empty = kv_full + ATT_STAGES;
  uint64_t* s_full = kv_empty + ATT_STAGES;
  uint64_t* s_free = s_full + 1;
  uint64_t* p_full = s_free + 1;
  uint64_t* o_done = p_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_done + 1);

  const int* it = a.items + blockIdx.x * 8;
  const int q_row0 = it[0], n_q = it[1], head = it[2], kv_row0 = it[3];
  const int key_begin = it[4], key_end = it[5], slot = it[6];
  const int n_kt = (key_end - key_begin + 127) / 128;

  const uint32_t warp = warp_id(), lane = lane_id();
  if (warp == 0 && lane == 0) {
    tma_prefetch(&map_q);
    tma_prefetch(&map_k);
    tma_prefetch(&map_v);
    mbar_init(q_full, 1);
    for (int s = 0; s < ATT_STAGES; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(s_free, 128);
    mbar_init(p_full, 128);
    mbar_init(o_done, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<256>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tmem_s = tmem, tmem_o = tmem + 128;

  if (warp == 0) {
    if (lane == 0 && n_kt > 0) {
      const uint64_t pol_q = policy_evict_first();
      const uint64_t pol_kv = policy_evict_normal();
      mbar_expect_tx(q_full, C::TILE_BYTES);
#pragma unroll
      for (int at = 0; at < C::N_ATOMS; ++at)
        tma_load_2d(sQ + at * C::ATOM_BYTES, &map_q, q_full, head * HD + at * C::ATOM_E, q_row0, pol_q);
      for (int j = 0; j < n_kt; ++j) {
        const int st = j % ATT_STAGES;
        mbar_wait(&kv_empty[st], ((j / ATT_STAGES) & 1) ^ 1);
        mbar_expect_tx(&kv_full[st], 2 * C::TILE_BYTES);
        const int krow = kv_row0 + key_begin + j * 128;
#pragma unroll
        for (int at = 0; at < C::N_ATOMS; ++at) {
          tma_load_3d(sK + st * C::TILE_BYTES + at * C::ATOM_BYTES, &map_k, &kv_full[st],
                      head * HD + at * C::ATOM_E, krow, a.layer, pol_kv);
          tma_load_3d(sV + st * C::TILE_BYTES + at * C::ATOM_BYTES, &map_v, &kv_full[st],
                      head * HD + at * C::ATOM_E, krow, a.layer, pol_kv);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && n_kt > 0) {
      const uint32_t idesc_s = make_idesc_bf16(128, 128, 0, 0);
      const uint32_t idesc_o = make_idesc_bf16(128, HD, 0, 1);
      const uint32_t q_addr = smem_u32(sQ);
      mbar_wait(q_full, 0);
      auto issue_s = [&](int j) {
        const int st = j % ATT_STAGES;
        mbar_wait(&kv_full[st], (j / ATT_STAGES) & 1);
        tc_fence_after();
        const uint32_t k_addr = smem_u32(sK + st * C::TILE_BYTES);
#pragma unroll
        for (int k = 0; k < HD / 16; ++k) {
          const int at = (k * 16) / C::ATOM_E;
          const uint32_t off = at * C::ATOM_BYTES + ((k * 16) % C::ATOM_E) * 2;
          const uint64_t ad = make_sdesc(q_addr + off, 16, 8 * C::SWZ, C::SWZ);
          const uint64_t bd = make_sdesc(k_addr + off, 16, 8 * C::SWZ, C::SWZ);
          tc_mma_f16(tmem_s, ad, bd, idesc_s, k > 0 ? 1u : 0u);
        }
        tc_commit(s_full);
      };
      issue_s(0);
      const uint32_t p_addr = smem_u32(sP);
      for (int j = 0; j < n_kt; ++j) {
        if (j + 1 < n_kt) {
          mbar_wait(s_free, j & 1);
          tc_fence_after();
          issue_s(j + 1);
        }
        mbar_wait(p_full, j & 1);
        tc_fence_after();
        const int st = j % ATT_STAGES;
        const uint32_t v_addr = smem_u32(sV + st * C::TILE_BYTES);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint64_t ad = make_sdesc(p_addr + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024, 128);
          const uint64_t bd = make_sdesc(v_addr + k * 16 * C::SWZ, C::ATOM_BYTES, 8 * C::SWZ, C::SWZ);
          tc_mma_f16(tmem_o, ad, bd, idesc_o, (j > 0 || k > 0) ? 1u : 0u);
        }
        tc_commit(o_done);
        tc_commit(&kv_empty[st]);
      }
    }
    __syncwarp();
  } else {
    // ---------------- softmax / correction / epilogue warps
    const int quad = warp & 3;
    const int r = quad * 32 + lane;
    const bool q_valid = r < n_q;
    const int qp = q_valid ? a.qpos[q_row0 + r] : -1;
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    const float NEG_INF = -INFINITY;
    float m_run = NEG_INF, l_run = 0.f;
    uint8_t* prow = sP + r * 128;
    const int sw = r & 7;
    for (int j = 0; j < n_kt; ++j) {
      const int k0 = key_begin + j * 128;
      float s[128];
      mbar_wait(s_full, j & 1);
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld32(tmem_s + lane_off + c * 32, s + c * 32);
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(s_free);
      float tmax = NEG_INF;
      const int lim = min(qp, key_end - 1) - k0;  // columns <= lim are visible
#pragma unroll
      for (int i = 0; i < 128; ++i) {
        s[i] = (i <= lim) ? s[i] * a.scale_log2 : NEG_INF;
        tmax = fmaxf(tmax, s[i]);
      }
      if (j > 0) {
        mbar_wait(o_done, (j - 1) & 1);
        tc_fence_after();
      }
      const float m_new = fmaxf(m_run, tmax);
      const bool need = m_new > m_run + 8.0f;  // lazy rescale (true when m_run = -inf)
      const bool has_o = m_run != NEG_INF;
      if (__any_sync(0xffffffffu, need && has_o)) {
        const float sc = (need && has_o) ? exp2f(m_run - m_new) : 1.0f;
#pragma unroll
        for (int c = 0; c < HD / 16; ++c) {
          float o[16];
          tmem_ld16(tmem_o + lane_off + c * 16, o);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 16; ++i) o[i] *= sc;
          tmem_st16(tmem_o + lane_off + c * 16, o);
        }
        tmem_wait_st();
      }
      if (need) {
        l_run = has_o ? l_run * exp2f(m_run - m_new) : 0.f;
        m_run = m_new;
      }
      const bool any = m_run != NEG_INF;
      float lsum = 0.f;
#pragma unroll
      for (int c16 = 0; c16 < 16; ++c16) {
        uint32_t pk[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float p0 = any ? exp2f(s[c16 * 8 + 2 * q] - m_run) : 0.f;
          const float p1 = any ? exp2f(s[c16 * 8 + 2 * q + 1] - m_run) : 0.f;
          lsum += p0 + p1;
          pk[q] = pack_bf16(p0, p1);
        }
        const int atom = c16 >> 3, ch = (c16 & 7) ^ sw;
        *reinterpret_cast<uint4*>(prow + atom * 16384 + ch * 16) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
      }
      l_run += lsum;
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(p_full);
    }
    if (n_kt > 0) {
      mbar_wait(o_done, (n_kt - 1) & 1);
      tc_fence_after();
    }
    if (slot < 0) {
      const float inv = (l_run > 0.f) ? 1.0f / l_run : 0.f;
      __nv_bfloat16* orow = q_valid ? reinterpret_cast<__nv_bfloat16*>(a.out) +
                                          (long)a.rowof[q_row0 + r] * a.ldo + head * HD
                                    : nullptr;
#pragma unroll
      for (int c = 0; c < HD / 16; ++c) {
        float o[16];
        if (n_kt > 0) {
          tmem_ld16(tmem_o + lane_off + c * 16, o);
          tmem_wait_ld();
        } else {
#pragma unroll
          for (int i = 0; i < 16; ++i) o[i] = 0.f;
        }
        if (q_valid) {
          uint32_t pk[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) pk[q] = pack_bf16(o[2 * q] * inv, o[2 * q + 1] * inv);
          uint4* dst = reinterpret_cast<uint4*>(orow + c * 16);
          dst[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
          dst[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
        }
      }
    } else {
      float* wo = a.ws_o + ((long)slot * 128 + r) * HD;
#pragma unroll
      for (int c = 0; c < HD / 16; ++c) {
        float o[16];
        if (n_kt > 0) {
          tmem_ld16(tmem_o + lane_off + c * 16, o);
          tmem_wait_ld();
        } else {
#pragma unroll
          for (int i = 0; i < 16; ++i) o[i] = 0.f;
        }
        if (q_valid) {
          float4* dst = reinterpret_cast<float4*>(wo + c * 16);
#pragma unroll
          for (int q = 0; q < 4; ++q) dst[q] = make_float4(o[4 * q], o[4 * q + 1], o[4 * q + 2], o[4 * q + 3]);
        }
      }
      if (q_valid) {
        a.ws_ml[((long)slot * 128 + r) * 2] = m_run;
        a.ws_ml[((long)slot * 128 + r) * 2 + 1] = l_run;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<256>(tmem);
  }
}

// Merge split-KV partials: O = sum_s 2^(m_s-M) O_s / sum_s 2^(m_s-M) l_s.
// Block = one combine item; thread = (query row, 4 output columns).
template <int HD>
__global__ void __launch_bounds__(256) attn_combine_kernel(vlc_attn_args a) {
  const int* it = a.comb + blockIdx.x * 8;
  const int q_row0 = it[0], n_q = it[1], head = it[2], slot0 = it[3], ns = it[4];
  constexpr int C4 = HD / 4;
  for (int w = threadIdx.x; w < 128 * C4; w += blockDim.x) {
    const int r = w / C4, c4 = w - r * C4;
    if (r >= n_q) break;
    float M = -INFINITY;
    for (int s = 0; s < ns; ++s) M = fmaxf(M, __ldg(a.ws_ml + ((long)(slot0 + s) * 128 + r) * 2));
    float L = 0.f;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int s = 0; s < ns; ++s) {
      const long base = (long)(slot0 + s) * 128 + r;
      const float m = __ldg(a.ws_ml + base * 2), l = __ldg(a.ws_ml + base * 2 + 1);
      const float wgt = (m == -INFINITY) ? 0.f : exp2f(m - M);
      L += wgt * l;
      const float4 o = __ldg(reinterpret_cast<const float4*>(a.ws_o + base * HD) + c4);
      acc.x += wgt * o.x; acc.y += wgt * o.y; acc.z += wgt * o.z; acc.w += wgt * o.w;
    }
    const float inv = L > 0.f ? 1.0f / L : 0.f;
    __nv_bfloat16* orow = reinterpret_cast<__nv_bfloat16*>(a.out) + (long)a.rowof[q_row0 + r] * a.ldo + head * HD;
    uint2 pk = make_uint2(pack_bf16(acc.x * inv, acc.y * inv), pack_bf16(acc.z * inv, acc.w * inv));
    *reinterpret_cast<uint2*>(orow + c4 * 4) = pk;
  }
}

template <int HD>
static cudaError_t launch_attn_hd(const vlc_attn_args& a, cudaStream_t stream) {
  using C = AttnCfg<HD>;
  CUtensorMap mq, mk, mv;
  cudaError_t e = make_tmap_2d(&mq, a.q, a.kv, a.q_rows_cap, (uint64_t)a.kv * 2, C::ATOM_E, 128, C::SWZ);
  if (e != cudaSuccess) return e;
  e = make_tmap_3d(&mk, a.kc, a.kv, a.kv_rows_cap, a.layers_cap, (uint64_t)a.kv * 2,
                   (uint64_t)a.kv * 2 * a.kv_rows_cap, C::ATOM_E, 128, 1, C::SWZ);
  if (e != cudaSuccess) return e;
  e = make_tmap_3d(&mv, a.vc, a.kv, a.kv_rows_cap, a.layers_cap, (uint64_t)a.kv * 2,
                   (uint64_t)a.kv * 2 * a.kv_rows_cap, C::ATOM_E, 128, 1, C::SWZ);
  if (e != cudaSuccess) return e;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attn_fwd_tc<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    attr = true;
  }
  attn_fwd_tc<HD><<<a.n_items, ATT_THREADS, C::SMEM, stream>>>(mq, mk, mv, a);
  return cudaGetLastError();
}

// ===================================================================== ping-pong kernel
// CTA = (request, head, key range) for up to 256 queries = two 128-query tiles A and B.
// Warp 0: TMA (Q once, then 64-key K/V tiles through a 3-stage ring); warp 1: tcgen05.mma
// issue; warps 2-5 softmax A, warps 6-9 softmax B.  While one group runs its softmax the
// tensor core works on the other group's S / PV.  TMEM: S_A, S_B (64 cols fp32), P_A, P_B
// (32 cols of packed bf16 pairs, the A operand of the PV MMA), O_A, O_B (HD cols fp32).
constexpr int PP_THREADS = 320;
// Softmax warps per (query tile, TMEM row quadrant): SW = 1 -> one thread per query row and all KT
// columns (10 warps); SW = 2 (VAR 0x4000) -> two threads per row, KT/2 columns each, row max
// exchanged through shared memory (20 warps: 2 control + 16 softmax + 2 idle = 5 per scheduler,
// so the per-scheduler register file allows 96 registers per thread).
// ONE (VAR 0x8000): a single query tile per CTA with S double-buffered in TMEM (S(j+1) is computed
// while the softmax works on S(j)) and SW = 4 threads per row (32 columns each; 0x4000: 2).
template <int VAR>
struct PPRoles {
  static constexpr bool ONE = (VAR & 0x8000) != 0;
  static constexpr int SW = ONE ? ((VAR & 0x4000) ? 2 : 4) : ((VAR & 0x4000) ? 2 : 1);
  static constexpr int NTILE = ONE ? 1 : 2;
  static constexpr int SOFT_WARPS = 4 * SW * NTILE;
  static constexpr int THREADS = SOFT_WARPS <= 8 ? PP_THREADS : 640;   // 10 or 20 warps
  static constexpr int XM_BYTES = SW == 1 ? 0 : 2 * NTILE * SW * 128 * 4;   // [parity][tile][part][row]
};
// Experiment instrumentation.  The buffers travel as kernel parameters (constant bank), so a
// disabled trace costs a predicated branch, not a global load on the softmax critical path.
static unsigned long long* h_attn_dbg = nullptr;    // per-CTA phase timestamps
static unsigned long long* h_attn_trace = nullptr;  // per-iteration event times of CTA 0
__device__ __forceinline__ void adbg(unsigned long long* dbgp, int slot) {
  if (dbgp) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    dbgp[blockIdx.x * 8 + slot] = t;
  }
}
void set_attn_debug_buffer(unsigned long long* p) { h_attn_dbg = p; }
__device__ __forceinline__ void atrace(unsigned long long* trc, int slot) {   // SM clock (CTA 0 only)
  if (trc && blockIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));
    trc[slot] = t;
  }
}
void set_attn_trace_buffer(unsigned long long* p) { h_attn_trace = p; }
// VAR 0x400: per-phase cycle counts summed over all CTAs into g_attn_trace[256 + slot]
__device__ __forceinline__ long long clk() { long long c; asm volatile("mov.u64 %0, %%clock64;" : "=l"(c)); return c; }
#define PH(on, slot, t)                                                               \
  do {                                                                                \
    if (on) {                                                                         \
      const long long t2_ = clk();                                                    \
      atomicAdd(&trc[256 + (slot)], (unsigned long long)(t2_ - (t)));        \
      t = t2_;                                                                        \
    }                                                                                 \
  } while (0)
// KT = keys per tile.  KT = 64: S double-buffered per query tile (S runs two tiles ahead).
// KT = 128 (hd 128): one 128-column S buffer per query tile (TMEM: S_A, S_B, O_A, O_B = 512
// columns), half the MMA instructions and barrier round trips per key; the ping-pong between
// the two query tiles hides the S(j) -> softmax -> PV(j) -> S(j+1) chain of each tile.
int g_attn_kt = 128;   // tuning key 12: key tile of the hd-128 kernel (64 or 128)
int g_attn_var = 0;    // tuning key 15: softmax variant of the hd-128 / 128-key kernel (see VAR below;
                       // 0 = default two-threads-per-row kernel, 100 = one thread per row)

template <int HD, int KT, bool PSM_ = false, int XM_BYTES = 0, bool ONE = false>
struct PPCfg {
  static constexpr bool DB = KT == 64 || ONE;
  // PSM: P staged in shared memory (SS MMA for PV) instead of aliased over S in TMEM, so S(j+1)
  // can be issued as soon as the softmax has read S(j) into registers (KT = 128 only)
  static constexpr bool PSM = PSM_ && KT == 128;
  static constexpr int P_BYTES = PSM ? 128 * KT * 2 : 0;
  static constexpr int ATOM_E = HD < 64 ? HD : 64;
  static constexpr int SWZ = ATOM_E * 2;
  static constexpr int N_ATOMS = HD / ATOM_E;
  static constexpr int Q_BYTES = 128 * HD * 2;
  static constexpr int Q_ATOM = 128 * SWZ;
  static constexpr int KV_BYTES = KT * HD * 2;
  static constexpr int KV_ATOM = KT * SWZ;
  // K/V ring as deep as shared memory allows (<= 8): the softmax warps wait on S, i.e. on K/V
  // loads, when the ring is shallow (ncu: s_full wait was the top stall at 3 stages)
  // Separate K and V rings: K(j) is consumed by S(j), a softmax ahead of PV(j), so K gets the
  // extra stage (KT = 128: K 3 deep, V 2 deep) -- with one shared 2-deep ring the S issue waited
  // on the HBM latency of K(j+1), loaded only once PV(j-1) had freed its slot.
  static constexpr int BAR_BYTES = 512;
  static constexpr int RING = 232448 - 1024 - BAR_BYTES - 2 * Q_BYTES - P_BYTES - XM_BYTES;
  static constexpr int VST_FIT = RING / (2 * KV_BYTES);
  static constexpr int VST = VST_FIT > 8 ? 8 : VST_FIT;
  static constexpr int KST_FIT = (RING - VST * KV_BYTES) / KV_BYTES;
  static constexpr int KST = KST_FIT > 8 ? 8 : KST_FIT;
  static constexpr int SMEM = 1024 + 2 * Q_BYTES + (KST + VST) * KV_BYTES + P_BYTES + XM_BYTES + BAR_BYTES;
  static_assert(VST >= 2 && KST >= VST, "K / V rings");
  static_assert((KST + VST) * KV_BYTES >= 2 * 128 * HD * 4, "split partials are staged in the K/V ring");
  static_assert((KST + VST) * KV_BYTES >= 256 * 8 * 12 + 256 * 4, "merge tables live in the K/V ring");
  // TMEM: S[x][buf] (KT fp32 cols; P bf16 pairs aliased in its first KT/2 cols), O[x] (HD cols)
  __device__ static constexpr uint32_t s_col(int x, int b) {
    return ONE ? 128u * b : (DB ? 64u * (2 * x + b) : 128u * x);
  }
  __device__ static constexpr uint32_t o_col(int x) { return 256u + (uint32_t)(HD > 64 ? HD : 64) * x; }
  __device__ static constexpr int sbuf(int j) { return DB ? (j & 1) : 0; }          // S buffer of tile j
  __device__ static constexpr uint32_t sphase(int j) { return DB ? ((j >> 1) & 1) : (j & 1); }
};

// VAR (softmax variants, tuning key 15): bit 0 = three-input max, bits 4-6 = pairs of every 8 whose
// exponentials run as poly_exp2 on the FMA pipe; bits 1 / 2 = timing experiments only (no exp2 /
// no O rescale: wrong results).
template <int HD, int KT, int VAR = 0>
__global__ void __launch_bounds__(PPRoles<VAR>::THREADS, 1)
    attn_pp_kernel(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_k,
                   const __grid_constant__ CUtensorMap map_v, vlc_attn_args a, unsigned long long* dbgp,
                   unsigned long long* trc) {
  using R = PPRoles<VAR>;
  using C = PPCfg<HD, KT, (VAR & 0x1000) != 0, R::XM_BYTES, R::ONE>;
  constexpr bool PSM = C::PSM;
  constexpr int SW = R::SW, NTH = R::THREADS;
  static_assert(!R::ONE || KT == 128, "single-tile mode: 128-key tiles");
  // OSPLIT (VAR 0x20000, single tile, two threads per row): each column half of the row keeps its
  // own running max / sum and its own O accumulator (O0, O1 in the TMEM columns the second tile
  // would use), so the per-iteration row-max exchange disappears; the halves merge once at the end.
  constexpr bool OSPLIT = (VAR & 0x20000) != 0;
  static_assert(!OSPLIT || (R::ONE && SW == 2 && HD == 128), "O split: single tile, two threads per row");
  static_assert(!(PSM && SW == 2), "P-in-smem is a one-warp-per-row variant");
  static_assert(SW == 1 || KT == 128, "two threads per row: 128-key tiles");
  constexpr int PP_KT = KT;
  constexpr int POLY = (VAR >> 4) & 7;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;                                   // [2][Q_BYTES]
  uint8_t* sK = sQ + 2 * C::Q_BYTES;                    // [ST][KV_BYTES]
  uint8_t* sV = sK + C::KST * C::KV_BYTES;              // [VST][KV_BYTES]
  uint8_t* sP = sV + C::VST * C::KV_BYTES;              // [P_BYTES] (PSM)
  float* xm = reinterpret_cast<float*>(sP + C::P_BYTES);  // [XM_BYTES] (SW = 2) row-max exchange
  uint64_t* bars = reinterpret_cast<uint64_t*>(sP + C::P_BYTES + R::XM_BYTES);
  uint64_t* q_full = bars;
  uint64_t* k_full = bars + 1;
  uint64_t* k_empty = k_full + C::KST;
  uint64_t* v_full = k_empty + C::KST;
  uint64_t* v_empty = v_full + C::VST;
  uint64_t* s_full = v_empty + C::VST;   // [2 tiles][2 buffers]
  uint64_t* p_full = s_full + 4;         // [2 tiles][2 S buffers]: P(j) of tile x in buffer j&1
  uint64_t* o_done = p_full + 4;         // [2]
  uint64_t* all_done = o_done + 2;       // every MMA of the CTA complete (K/V ring reusable)
  uint64_t* s_free = all_done + 1;       // [2] PSM: S(j) of tile x read into registers
  uint64_t* p_free = s_free + 2;         // [2] PSM: PV of P-buffer use u complete (alternating)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(p_free + 2);

  const int* it = a.items + blockIdx.x * 8;
  const int q_row0 = it[0], nq = it[1], head = it[2], kv_row0 = it[3];
  const int kb = it[4], ke = it[5], group = it[6];
  const int part = it[7] >> 8, nsplit = it[7] & 0xff;
  const int nq_t[2] = {min(nq, 128), R::ONE ? 0 : max(0, nq - 128)};   // ONE: items carry <= 128 queries
  int nt_t[2];
#pragma unroll
  for (int x = 0; x < 2; ++x) {
    int e = -1;
    if (nq_t[x] > 0) e = min(ke, a.qpos[q_row0 + x * 128 + nq_t[x] - 1] + 1);
    nt_t[x] = e > kb ? (e - kb + PP_KT - 1) / PP_KT : 0;
  }
  const int nt = max(nt_t[0], nt_t[1]);
  // PSM: the single P buffer is used in the order (j, tile A), (j, tile B), ...; use index of (x, j)
  auto p_use = [&](int x, int j) { return min(j, nt_t[0]) + min(j, nt_t[1]) + ((x == 1 && j < nt_t[0]) ? 1 : 0); };

  const uint32_t warp = warp_id(), lane = lane_id();
  if (warp == 0 && lane == 0) {
    adbg(dbgp, 0);
    tma_prefetch(&map_q);
    tma_prefetch(&map_k);
    tma_prefetch(&map_v);
    mbar_init(q_full, 1);
    for (int s = 0; s < C::KST; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < C::VST; ++s) {
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    for (int x = 0; x < 4; ++x) mbar_init(&s_full[x], 1);
    for (int x = 0; x < 4; ++x) mbar_init(&p_full[x], 128 * SW);
    for (int x = 0; x < 2; ++x) {
      mbar_init(&o_done[x], 1);
    }
    mbar_init(all_done, 1);
    for (int x = 0; x < 2; ++x) {
      mbar_init(&s_free[x], 128);
      mbar_init(&p_free[x], 1);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();                 // Q / K / V / work lists come from the previous kernels
  if (threadIdx.x == 0) pdl_trigger();

  if (warp == 0) {
    if (lane == 0 && nt > 0) {
      const uint64_t pol_q = policy_evict_first();
      const uint64_t pol_kv = policy_evict_normal();
      mbar_expect_tx(q_full, (nq_t[1] > 0 ? 2 : 1) * C::Q_BYTES);
      for (int x = 0; x < 2; ++x)   // one op per Q tile: 3-D view {atom elems, rows, atoms}
        if (nq_t[x] > 0)
          tma_load_3d(sQ + x * C::Q_BYTES, &map_q, q_full, 0, q_row0 + x * 128, head * C::N_ATOMS, pol_q);
      auto load_k = [&](int j) {   // one op per K / V tile: 4-D {elems, keys, atoms, layer}
        const int st = j % C::KST;
        mbar_wait(&k_empty[st], ((j / C::KST) & 1) ^ 1);
        mbar_expect_tx(&k_full[st], C::KV_BYTES);
        tma_load_4d(sK + st * C::KV_BYTES, &map_k, &k_full[st], 0, kv_row0 + kb + j * PP_KT, head * C::N_ATOMS,
                    a.layer, pol_kv);
      };
      auto load_v = [&](int j) {
        const int st = j % C::VST;
        mbar_wait(&v_empty[st], ((j / C::VST) & 1) ^ 1);
        if (j < 32) atrace(trc, 128 + j);
        mbar_expect_tx(&v_full[st], C::KV_BYTES);
        tma_load_4d(sV + st * C::KV_BYTES, &map_v, &v_full[st], 0, kv_row0 + kb + j * PP_KT, head * C::N_ATOMS,
                    a.layer, pol_kv);
      };
      // K runs KST-1 tiles ahead of V
      for (int j = 0; j < C::KST - 1 && j < nt; ++j) load_k(j);
      for (int j = 0; j < nt; ++j) {
        if (j + C::KST - 1 < nt) load_k(j + C::KST - 1);
        load_v(j);
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && nt > 0) {
      const uint32_t idesc_s = make_idesc_bf16(128, PP_KT, 0, 0);
      const uint32_t idesc_o = make_idesc_bf16(128, HD, 0, 1);
      mbar_wait(q_full, 0);
      adbg(dbgp, 1);
      auto issue_s = [&](int x, int j) {   // S[x][j&1] = Q_x K_j^T
        const int st = j % C::KST;
        mbar_wait(&k_full[st], (j / C::KST) & 1);
        tc_fence_after();
        const uint32_t q_addr = smem_u32(sQ + x * C::Q_BYTES);
        const uint32_t k_addr = smem_u32(sK + st * C::KV_BYTES);
#pragma unroll
        for (int k = 0; k < HD / 16; ++k) {
          const int at = (k * 16) / C::ATOM_E;
          const uint32_t eoff = ((k * 16) % C::ATOM_E) * 2;
          const uint64_t ad = make_sdesc(q_addr + at * C::Q_ATOM + eoff, 16, 8 * C::SWZ, C::SWZ);
          const uint64_t bd = make_sdesc(k_addr + at * C::KV_ATOM + eoff, 16, 8 * C::SWZ, C::SWZ);
          if (!(VAR & 0x200)) tc_mma_f16(tmem + C::s_col(x, C::sbuf(j)), ad, bd, idesc_s, k > 0 ? 1u : 0u);
        }
        tc_commit(&s_full[2 * x + C::sbuf(j)]);
      };
      auto issue_pv = [&](int x, int j) {  // O_x += P_x(j) V_j, P from TMEM (aliased in S[x][j&1])
        const int st = j % C::VST;
        const uint32_t v_addr = smem_u32(sV + st * C::KV_BYTES);
#pragma unroll
        for (int k = 0; k < PP_KT / 16; ++k) {
          const uint64_t bd = make_sdesc(v_addr + k * 16 * C::SWZ, C::KV_ATOM, 8 * C::SWZ, C::SWZ);
          if (!(VAR & 0x200)) {
            if (OSPLIT)   // keys of column half k>>2 accumulate into O_(k>>2); P of half h at S cols 64h..
              tc_mma_f16_ts(tmem + C::o_col(k >> 2), tmem + C::s_col(x, C::sbuf(j)) + k * 8 + (k >> 2) * 32, bd,
                            idesc_o, (j > 0 || (k & 3) > 0) ? 1u : 0u);
            else
              tc_mma_f16_ts(tmem + C::o_col(x), tmem + C::s_col(x, C::sbuf(j)) + k * 8, bd, idesc_o,
                            (j > 0 || k > 0) ? 1u : 0u);
          }
        }
        tc_commit(&o_done[x]);
      };
      if constexpr (PSM) {
        // S_x(j+1) as soon as the softmax has read S_x(j); PV_x(j) (P from smem) when P_x(j) is
        // written; P-buffer use u releases the buffer through p_free[u & 1]
        for (int x = 0; x < 2; ++x)
          if (0 < nt_t[x]) issue_s(x, 0);
        tc_commit(&k_empty[0]);
        const uint32_t p_addr = smem_u32(sP);
        for (int j = 0; j < nt; ++j) {
          for (int x = 0; x < 2; ++x)
            if (j + 1 < nt_t[x]) {
              mbar_wait(&s_free[x], j & 1);
              tc_fence_after();
              issue_s(x, j + 1);
            }
          if (j + 1 < nt) tc_commit(&k_empty[(j + 1) % C::KST]);
          const int st = j % C::VST;
          mbar_wait(&v_full[st], (j / C::VST) & 1);
          tc_fence_after();
          const uint32_t v_addr = smem_u32(sV + st * C::KV_BYTES);
          for (int x = 0; x < 2; ++x) {
            if (j >= nt_t[x]) continue;
            mbar_wait(&p_full[2 * x], j & 1);
            tc_fence_after();
#pragma unroll
            for (int k = 0; k < PP_KT / 16; ++k) {
              const uint64_t ad = make_sdesc(p_addr + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024, 128);
              const uint64_t bd = make_sdesc(v_addr + k * 16 * C::SWZ, C::KV_ATOM, 8 * C::SWZ, C::SWZ);
              tc_mma_f16(tmem + C::o_col(x), ad, bd, idesc_o, (j > 0 || k > 0) ? 1u : 0u);
            }
            tc_commit(&p_free[p_use(x, j) & 1]);
            tc_commit(&o_done[x]);
          }
          tc_commit(&v_empty[st]);
        }
        tc_commit(all_done);
        adbg(dbgp, 2);
      }
      // DB: S runs two tiles ahead of the softmax (double-buffered per query tile); otherwise one
      // tile ahead: S(j+1) is issued right after PV(j), which frees the single S/P buffer
      constexpr int AHEAD = C::DB ? 2 : 1;
      if (!PSM) {
      for (int j = 0; j < AHEAD; ++j) {
        for (int x = 0; x < 2; ++x)
          if (j < nt_t[x]) issue_s(x, j);
        if (j < nt) tc_commit(&k_empty[j % C::KST]);
      }
      for (int j = 0; j < nt; ++j) {
        mbar_wait(&v_full[j % C::VST], (j / C::VST) & 1);
        tc_fence_after();
        for (int x = 0; x < 2; ++x) {
          if (j >= nt_t[x]) continue;
          const bool ph = (VAR & 0x400) && trc;
          long long tph = ph ? clk() : 0;
          mbar_wait(&p_full[2 * x + C::sbuf(j)], C::sphase(j));
          tc_fence_after();
          PH(ph, 16 + x * 4 + 0, tph);
          if (j < 16) atrace(trc, 64 + j * 4 + 2 * x);
          issue_pv(x, j);
          PH(ph, 16 + x * 4 + 1, tph);
          if (j + AHEAD < nt_t[x]) issue_s(x, j + AHEAD);   // in-order after PV(j): reuses P(j)'s columns
          PH(ph, 16 + x * 4 + 2, tph);
          if (j < 16) atrace(trc, 64 + j * 4 + 2 * x + 1);
        }
        tc_commit(&v_empty[j % C::VST]);
        if (j + AHEAD < nt) tc_commit(&k_empty[(j + AHEAD) % C::KST]);
      }
      tc_commit(all_done);
      adbg(dbgp, 2);
      }
    }
    __syncwarp();
  } else if (warp < 2 + R::SOFT_WARPS) {
    // ---------------- softmax groups: warps 2.. -> tile A, then tile B (SW warps per quadrant)
    const int x = (warp - 2) / (4 * SW);
    const int hh = SW == 1 ? 0 : ((warp - 2) >> 2) % SW;   // column part of the row
    constexpr int CW = KT / SW, OW = HD / SW;              // S / O columns of this thread
    const int quad = warp & 3;
    const int r = quad * 32 + lane;
    const bool q_valid = r < nq_t[x];
    const int qp = q_valid ? a.qpos[q_row0 + x * 128 + r] : -1;
    const int ntx = nt_t[x];
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    const uint32_t tO = tmem + C::o_col(OSPLIT ? hh : x) + lane_off;   // OSPLIT: this half's O
    const float NEG_INF = -INFINITY;
    float m_run = NEG_INF, l_run = 0.f;
    for (int j = 0; j < ntx; ++j) {
      const int k0 = kb + j * PP_KT;
      const uint32_t tS = tmem + C::s_col(x, C::sbuf(j)) + lane_off;
      float s[CW];
      const bool ph = (VAR & 0x400) && r == 0 && hh == 0 && trc;
      long long tph = ph ? clk() : 0;
      mbar_wait(&s_full[2 * x + C::sbuf(j)], C::sphase(j));
      tc_fence_after();
      PH(ph, x * 8 + 0, tph);
      if (VAR & 0x100) {                      // experiment: no softmax work at all
        tc_fence_before();
        if (PSM) mbar_arrive(&s_free[x]);
        mbar_arrive(&p_full[2 * x + C::sbuf(j)]);
        continue;
      }
      const bool tr = trc && r == 0 && hh == 0 && j < 16;
      if (tr) atrace(trc, (x ? 160 : 0) + j * 4);
#pragma unroll
      for (int c = 0; c < CW / 32; ++c) tmem_ld32(tS + hh * CW + 32 * c, s + 32 * c);
      tmem_wait_ld();
      if (PSM) {                                  // S(j) is in registers: S(j+1) may overwrite it
        tc_fence_before();
        mbar_arrive(&s_free[x]);
      }
      PH(ph, x * 8 + 1, tph);
      if (tr) atrace(trc, (x ? 160 : 0) + j * 4 + 1);
      // scores stay raw (scale folded into the exp2 FFMA); masked keys -> -inf; reductions in
      // 4 independent chains (only 2 softmax warps per scheduler: latency, not issue, binds)
      const int lim = min(qp, ke - 1) - k0 - hh * CW;
      if (lim < CW - 1) {
#pragma unroll
        for (int i = 0; i < CW; ++i) s[i] = (i <= lim) ? s[i] : NEG_INF;
      }
      float mx4[4] = {NEG_INF, NEG_INF, NEG_INF, NEG_INF};
      if (VAR & 1) {
#pragma unroll
        for (int i = 0; i < CW; i += 2) mx4[(i >> 1) & 3] = fmax3(mx4[(i >> 1) & 3], s[i], s[i + 1]);
      } else {
#pragma unroll
        for (int i = 0; i < CW; ++i) mx4[i & 3] = fmaxf(mx4[i & 3], s[i]);
      }
      float pmax = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3]));
      if constexpr (SW > 1 && !OSPLIT) {
        // the other row parts' maxima; the barrier also orders every part's S reads before any P
        // write into S's columns (P of an upper part lands in a lower part's S columns)
        float* xb = xm + ((j & 1) * R::NTILE + x) * (SW * 128);
        xb[hh * 128 + r] = pmax;
        tc_fence_before();
        asm volatile("bar.sync %0, %1;" ::"r"(1 + x), "r"(128 * SW) : "memory");
        tc_fence_after();
#pragma unroll
        for (int o = 1; o < SW; ++o) pmax = fmaxf(pmax, xb[((hh + o) % SW) * 128 + r]);
      }
      const float tmax = pmax * a.scale_log2;
      const float m_new = fmaxf(m_run, tmax);
      const bool need = m_new > m_run + 8.0f;
      const bool has_o = m_run != NEG_INF;
      // O is only touched when some row rescales; P(j) goes to S buffer j&1, whose previous P
      // (PV(j-2)) is complete because S(j) was issued after it.  So PV(j-1) is waited for only
      // when rescaling, and on the last tile (so that the final wait below is unambiguous):
      // o_done has completed j-1 or j phases here (S(j) done => PV(j-2) done).
      PH(ph, x * 8 + 2, tph);
      const bool resc = (VAR & 4) ? false : __any_sync(0xffffffffu, need && has_o);
      if (C::DB && j > 0 && (resc || j == ntx - 1)) {   // !DB: S(j) done => PV(j-1) done already
        mbar_wait(&o_done[x], (j - 1) & 1);
        tc_fence_after();
      }
      // PSM: S(j) done => PV(j-2) done (issued earlier), so o_done has j-1 or j completions here
      if (PSM && j > 0 && resc) {
        mbar_wait(&o_done[x], (j - 1) & 1);
        tc_fence_after();
      }
      if (resc) {
        const float sc = (need && has_o) ? fast_exp2(m_run - m_new) : 1.0f;
        constexpr int RW = OSPLIT ? HD : OW;          // O columns this thread rescales
        const uint32_t tR = OSPLIT ? tO : tO + hh * OW;
#pragma unroll
        for (int c = 0; c < RW / 16; ++c) {
          float o[16];
          tmem_ld16(tR + c * 16, o);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 16; ++i) o[i] *= sc;
          tmem_st16(tR + c * 16, o);
        }
        tmem_wait_st();
      }
      if (need) {
        l_run = has_o ? l_run * fast_exp2(m_run - m_new) : 0.f;
        m_run = m_new;
      }
      PH(ph, x * 8 + 3, tph);
      const bool any = m_run != NEG_INF;
      const float nm = any ? -m_run : NEG_INF;     // all-masked row: every p = exp2(-inf) = 0
      // P packed in place into s[0, KT/2) (slot i is free once pairs 2i, 2i+1 are read)
      float ls4[4] = {0.f, 0.f, 0.f, 0.f};
      if constexpr ((VAR & 0x10000) != 0) {    // two exponentials per MUFU op (f16x2), fp32 sums
        const float2 sc2 = make_float2(a.scale_log2, a.scale_log2), nm2 = make_float2(nm, nm);
        float2 l2[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
        for (int i = 0; i < CW / 2; ++i) {
          const float2 xx = ffma2(make_float2(s[2 * i], s[2 * i + 1]), sc2, nm2);
          const float2 pp = exp2_f16x2(xx.x, xx.y);
          l2[i & 3] = fadd2(l2[i & 3], pp);
          s[i] = __uint_as_float(pack_bf16(pp.x, pp.y));
        }
        const float2 la = fadd2(l2[0], l2[1]), lb = fadd2(l2[2], l2[3]);
        ls4[0] = la.x; ls4[1] = la.y; ls4[2] = lb.x; ls4[3] = lb.y;
      } else if constexpr ((VAR & 0x2000) != 0) {     // packed-pair FFMA2 / FADD2
        const float2 sc2 = make_float2(a.scale_log2, a.scale_log2), nm2 = make_float2(nm, nm);
        float2 l2[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
        for (int i = 0; i < CW / 2; ++i) {
          const float2 xx = ffma2(make_float2(s[2 * i], s[2 * i + 1]), sc2, nm2);
          const float2 pp = make_float2(fast_exp2(xx.x), fast_exp2(xx.y));
          l2[i & 3] = fadd2(l2[i & 3], pp);
          s[i] = __uint_as_float(pack_bf16(pp.x, pp.y));
        }
        const float2 la = fadd2(l2[0], l2[1]), lb = fadd2(l2[2], l2[3]);
        ls4[0] = la.x; ls4[1] = la.y; ls4[2] = lb.x; ls4[3] = lb.y;
      } else
#pragma unroll
      for (int i = 0; i < CW / 2; ++i) {
        // POLY of every 8 pairs on the FMA pipe, the rest on the MUFU (both pipes busy)
        const float x0 = fmaf(s[2 * i], a.scale_log2, nm), x1 = fmaf(s[2 * i + 1], a.scale_log2, nm);
        float p0, p1;
        if (VAR & 2) {
          p0 = x0; p1 = x1;                                   // experiment: no exponential at all
        } else if ((i & 7) < POLY) {
          p0 = poly_exp2(x0); p1 = poly_exp2(x1);
        } else {
          p0 = fast_exp2(x0); p1 = fast_exp2(x1);
        }
        ls4[i & 3] += p0 + p1;
        s[i] = __uint_as_float(pack_bf16(p0, p1));
      }
      l_run += (ls4[0] + ls4[1]) + (ls4[2] + ls4[3]);
      PH(ph, x * 8 + 4, tph);
      if (tr) atrace(trc, (x ? 160 : 0) + j * 4 + 2);
      if constexpr (PSM) {
        // P(j) -> the shared P buffer (SW128 K-major: 2 atoms of 64 keys, 16-byte chunk c of row r
        // at c ^ (r & 7)) once its previous use (the other tile's or own PV) has completed.  Use
        // u-1 shares p_free[(u-1) & 1] only with u-3, which this thread has already seen complete.
        const int u = p_use(x, j);
        if (u > 0) mbar_wait(&p_free[(u - 1) & 1], ((u - 1) >> 1) & 1);
        uint8_t* prow = sP + r * 128;
#pragma unroll
        for (int c = 0; c < PP_KT / 8; ++c)
          *reinterpret_cast<uint4*>(prow + (c >> 3) * 16384 + (((c & 7) ^ (r & 7)) << 4)) =
              make_uint4(__float_as_uint(s[4 * c]), __float_as_uint(s[4 * c + 1]), __float_as_uint(s[4 * c + 2]),
                         __float_as_uint(s[4 * c + 3]));
        fence_proxy_async_smem();
        mbar_arrive(&p_full[2 * x]);
      } else {
        if constexpr (CW >= 64) {
#pragma unroll
          // P(j) over S(j)'s first cols (OSPLIT: over this half's own S columns -- no exchange barrier
          // orders the other half's S reads)
          for (int c = 0; c < CW / 64; ++c) tmem_st32f(tS + hh * (OSPLIT ? CW : CW / 2) + 32 * c, s + 32 * c);
        } else {
          tmem_st16(tS + hh * (CW / 2), s);
        }
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(&p_full[2 * x + C::sbuf(j)]);   // per-buffer barrier: softmax may run a tile ahead
      }
      PH(ph, x * 8 + 5, tph);
      if (ph) atomicAdd(&trc[256 + x * 8 + 7], 1ull);
      if (tr) atrace(trc, (x ? 160 : 0) + j * 4 + 3);
    }
    if (ntx > 0) {   // o_done has completed ntx-1 or ntx phases here
      mbar_wait(&o_done[x], (ntx - 1) & 1);
      tc_fence_after();
    }
    float w_own = 1.f, w_oth = 0.f;   // OSPLIT: weights of O_own / O_other in the merged row
    if constexpr (OSPLIT) {
      // merge the two halves' (max, sum): M = max, w_h = 2^(m_h - M), L = w0 l0 + w1 l1
      xm[hh * 128 + r] = m_run;
      xm[256 + hh * 128 + r] = l_run;
      asm volatile("bar.sync %0, %1;" ::"r"(1 + x), "r"(256) : "memory");
      const float m_o = xm[(1 - hh) * 128 + r], l_o = xm[256 + (1 - hh) * 128 + r];
      const float M = fmaxf(m_run, m_o);
      w_own = m_run == -INFINITY ? 0.f : fast_exp2(m_run - M);
      w_oth = m_o == -INFINITY ? 0.f : fast_exp2(m_o - M);
      l_run = w_own * l_run + w_oth * l_o;
      m_run = M;
    } else if constexpr (SW > 1) {   // row sum = all parts' sums (exchange buffer of iteration ntx: free)
      float* xb = xm + ((ntx & 1) * R::NTILE + x) * (SW * 128);
      xb[hh * 128 + r] = l_run;
      asm volatile("bar.sync %0, %1;" ::"r"(1 + x), "r"(128 * SW) : "memory");
      float lt = l_run;
#pragma unroll
      for (int o = 1; o < SW; ++o) lt += xb[((hh + o) % SW) * 128 + r];
      l_run = lt;
    }
    if (r == 0 && hh == 0) adbg(dbgp, 3 + x);
    const int qrow = q_row0 + x * 128 + r;
    // 16 O columns (chunk c of this thread's OW) of the row: OSPLIT merges O_own and O_other
    auto load_o = [&](int c, float* o) {
      if constexpr (OSPLIT) {
        float o2[16];
        tmem_ld16(tmem + C::o_col(hh) + lane_off + hh * OW + c * 16, o);
        tmem_ld16(tmem + C::o_col(1 - hh) + lane_off + hh * OW + c * 16, o2);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 16; ++i) o[i] = w_own * o[i] + w_oth * o2[i];
      } else {
        tmem_ld16(tO + hh * OW + c * 16, o);
        tmem_wait_ld();
      }
    };
    if (group < 0) {
      const float inv = (l_run > 0.f) ? 1.0f / l_run : 0.f;
      const int orow_i = q_valid ? a.rowof[qrow] : 0;
      __nv_bfloat16* obase = reinterpret_cast<__nv_bfloat16*>(a.out);
#pragma unroll
      for (int c = 0; c < OW / 16; ++c) {
        float o[16];
        if (ntx > 0) {
          load_o(c, o);
        } else {
#pragma unroll
          for (int i = 0; i < 16; ++i) o[i] = 0.f;
        }
        if (q_valid) {
          uint32_t pkk[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) pkk[q] = pack_bf16(o[2 * q] * inv, o[2 * q + 1] * inv);
          const int col = head * HD + hh * OW + c * 16;
          const long o0 = a.pk_rows > 0 ? packed_off(orow_i, col, a.pk_rows, a.pk_kb) : (long)orow_i * a.ldo + col;
          const long o1 = a.pk_rows > 0 ? packed_off(orow_i, col + 8, a.pk_rows, a.pk_kb) : o0 + 8;
          *reinterpret_cast<uint4*>(obase + o0) = make_uint4(pkk[0], pkk[1], pkk[2], pkk[3]);
          *reinterpret_cast<uint4*>(obase + o1) = make_uint4(pkk[4], pkk[5], pkk[6], pkk[7]);
        }
      }
    } else {
      // Split partial: once every MMA of the CTA is complete the K/V ring is free; stage this
      // tile's fp32 O rows there (row-major, float4 slot c4 stored at c4 ^ (row & 7): bank-conflict
      // free, same layout in ws_o) and write them with one bulk copy (full-line writes; per-thread
      // 16-byte row stores at a 512-byte stride were L2-transaction bound).
      const long prow0 = ((long)group * 8 + part) * 256 + x * 128;
      {
        if (nt > 0) mbar_wait(all_done, 0);
        tc_fence_after();
        float4* stg = reinterpret_cast<float4*>(sK) + x * 128 * (HD / 4) + r * (HD / 4);
#pragma unroll
        for (int c = 0; c < OW / 16; ++c) {
          float o[16];
          if (ntx > 0) {
            load_o(c, o);
          } else {
#pragma unroll
            for (int i = 0; i < 16; ++i) o[i] = 0.f;
          }
          const int c4 = (hh * OW / 16 + c) * 4;
#pragma unroll
          for (int q = 0; q < 4; ++q)
            stg[(c4 + q) ^ (r & 7)] = make_float4(o[4 * q], o[4 * q + 1], o[4 * q + 2], o[4 * q + 3]);
        }
        fence_proxy_async_smem();
        asm volatile("bar.sync %0, %1;" ::"r"(1 + x), "r"(128 * SW) : "memory");
        if (quad == 0 && lane == 0 && hh == 0 && nq_t[x] > 0)
          bulk_store_wait(a.ws_o + prow0 * HD, reinterpret_cast<float4*>(sK) + x * 128 * (HD / 4),
                          (uint32_t)(nq_t[x] * HD * 4));
      }
      if (q_valid && hh == 0) __stcg(reinterpret_cast<float2*>(a.ws_ml) + prow0 + r, make_float2(m_run, l_run));
      __threadfence();
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
  if (group < 0) return;
  // ---------------- parallel merge of the nsplit partials (all CTAs of the group co-resident).
  // This CTA merges rows [r_lo, r_hi) of the group.  Pass 1: one thread per (row, split) reads
  // (m, l); one thread per row turns them into normalised split weights (smem, in the K/V ring,
  // free once this CTA's partials are written).  Pass 2: one thread per (row, float4 of the head), all split loads independent --
  // no dependent L2 round trips per row.
  if (threadIdx.x == 0) {
    atomicAdd(&a.counters[group], 1);
    volatile int* cnt = a.counters + group;
    while (*cnt < nsplit) __nanosleep(32);
  }
  __syncthreads();
  __threadfence();
  if (threadIdx.x == 0) adbg(dbgp, 5);
  const int r_lo = nq * part / nsplit, r_hi = nq * (part + 1) / nsplit;
  const int nr = max(0, r_hi - r_lo);
  float2* s_ml = reinterpret_cast<float2*>(sK);                 // [nr][8]
  float* s_w = reinterpret_cast<float*>(s_ml + 256 * 8);        // [nr][8] weight / L
  int* s_orow = reinterpret_cast<int*>(s_w + 256 * 8);          // [nr]
  const long gbase = (long)group * 8 * 256;
  for (int t = threadIdx.x; t < nr * 8; t += NTH) {
    const int rr = t >> 3, s2 = t & 7;
    s_ml[t] = s2 < nsplit ? __ldcg(reinterpret_cast<const float2*>(a.ws_ml) + gbase + s2 * 256 + r_lo + rr)
                          : make_float2(-INFINITY, 0.f);
  }
  for (int rr = threadIdx.x; rr < nr; rr += NTH) s_orow[rr] = a.rowof[q_row0 + r_lo + rr];
  __syncthreads();
  for (int rr = threadIdx.x; rr < nr; rr += NTH) {
    float M = -INFINITY;
#pragma unroll
    for (int s2 = 0; s2 < 8; ++s2) M = fmaxf(M, s_ml[rr * 8 + s2].x);
    float w[8], L = 0.f;
#pragma unroll
    for (int s2 = 0; s2 < 8; ++s2) {
      const float2 ml = s_ml[rr * 8 + s2];
      w[s2] = ml.x == -INFINITY ? 0.f : exp2f(ml.x - M);
      L += w[s2] * ml.y;
    }
    const float inv = L > 0.f ? 1.0f / L : 0.f;
#pragma unroll
    for (int s2 = 0; s2 < 8; ++s2) s_w[rr * 8 + s2] = w[s2] * inv;
  }
  __syncthreads();
  constexpr int C4 = HD / 4;
  for (int t = threadIdx.x; t < nr * C4; t += NTH) {
    const int rr = t / C4, c4 = t % C4;
    const int row = r_lo + rr;                                   // row within the group's 256
    const float4* src = reinterpret_cast<const float4*>(a.ws_o) + (gbase + row) * C4 + (c4 ^ (row & 7));
    float4 xs[8];
#pragma unroll
    for (int s2 = 0; s2 < 8; ++s2)
      if (s2 < nsplit) xs[s2] = __ldcg(src + (long)s2 * 256 * C4);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int s2 = 0; s2 < 8; ++s2) {
      if (s2 >= nsplit) break;
      const float w = s_w[rr * 8 + s2];
      acc.x += w * xs[s2].x; acc.y += w * xs[s2].y; acc.z += w * xs[s2].z; acc.w += w * xs[s2].w;
    }
    const int orow_i = s_orow[rr], col = head * HD + c4 * 4;
    const long off = a.pk_rows > 0 ? packed_off(orow_i, col, a.pk_rows, a.pk_kb) : (long)orow_i * a.ldo + col;
    *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(a.out) + off) =
        make_uint2(pack_bf16(acc.x, acc.y), pack_bf16(acc.z, acc.w));
  }
  __syncthreads();
  if (threadIdx.x == 0) adbg(dbgp, 6);
  if (threadIdx.x == 0) {
    if (atomicAdd(&a.counters[a.ws_slots + group], 1) == nsplit - 1) {
      a.counters[group] = 0;
      a.counters[a.ws_slots + group] = 0;
    }
  }
}

int g_attn_min_smem = 0;

template <int HD, int KT, int VAR = 0>
static cudaError_t launch_pp_hd(const vlc_attn_args& a, cudaStream_t stream, bool coop) {
  using C = PPCfg<HD, KT, (VAR & 0x1000) != 0, PPRoles<VAR>::XM_BYTES, PPRoles<VAR>::ONE>;
  CUtensorMap mq, mk, mv;
  // Q: {atom elems, rows, atoms} box {ATOM_E, 128, N_ATOMS}: one op = both swizzle atoms of a tile
  cudaError_t e = make_tmap_3d(&mq, a.q, C::ATOM_E, a.q_rows_cap, a.kv / C::ATOM_E, (uint64_t)a.kv * 2,
                               (uint64_t)C::SWZ, C::ATOM_E, 128, C::N_ATOMS, C::SWZ);
  if (e != cudaSuccess) return e;
  const uint64_t dims[4] = {(uint64_t)C::ATOM_E, (uint64_t)a.kv_rows_cap, (uint64_t)(a.kv / C::ATOM_E),
                            (uint64_t)a.layers_cap};
  const uint64_t strides[3] = {(uint64_t)a.kv * 2, (uint64_t)C::SWZ, (uint64_t)a.kv * 2 * a.kv_rows_cap};
  const uint32_t box[4] = {(uint32_t)C::ATOM_E, (uint32_t)KT, (uint32_t)C::N_ATOMS, 1};
  e = make_tmap_4d(&mk, a.kc, dims, strides, box, C::SWZ);
  if (e != cudaSuccess) return e;
  e = make_tmap_4d(&mv, a.vc, dims, strides, box, C::SWZ);
  if (e != cudaSuccess) return e;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attn_pp_kernel<HD, KT, VAR>, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
    attr = true;
  }
  const int smem = C::SMEM > g_attn_min_smem ? C::SMEM : g_attn_min_smem;
  return launch_chain(attn_pp_kernel<HD, KT, VAR>, dim3(a.n_items), dim3(PPRoles<VAR>::THREADS), smem, stream, coop, mq, mk, mv, a,
                      h_attn_dbg, h_attn_trace);
}

cudaError_t launch_attention_pp(const vlc_attn_args& a, cudaStream_t stream, bool coop) {
  if (a.n_items <= 0) return cudaSuccess;
  switch (a.head_dim) {
    case 16: return launch_pp_hd<16, 64>(a, stream, coop);
    case 32: return launch_pp_hd<32, 64>(a, stream, coop);
    case 64: return launch_pp_hd<64, 64>(a, stream, coop);
    case 128:
      if (g_attn_kt == 64) return launch_pp_hd<128, 64>(a, stream, coop);
      switch (g_attn_var) {
        case 1: return launch_pp_hd<128, 128, 0x01>(a, stream, coop);
        case 2: return launch_pp_hd<128, 128, 0x21>(a, stream, coop);
        case 3: return launch_pp_hd<128, 128, 0x31>(a, stream, coop);
        case 4: return launch_pp_hd<128, 128, 0x41>(a, stream, coop);
        case 5: return launch_pp_hd<128, 128, 0x03>(a, stream, coop);
        case 6: return launch_pp_hd<128, 128, 0x05>(a, stream, coop);
        case 7: return launch_pp_hd<128, 128, 0x07>(a, stream, coop);
        case 8: return launch_pp_hd<128, 128, 0x100>(a, stream, coop);
        case 9: return launch_pp_hd<128, 128, 0x200>(a, stream, coop);
        case 10: return launch_pp_hd<128, 128, 0x300>(a, stream, coop);
        case 11: return launch_pp_hd<128, 128, 0x400>(a, stream, coop);
        case 20: return launch_pp_hd<128, 128, 0x2001>(a, stream, coop);
        case 22: return launch_pp_hd<128, 128, 0x4000>(a, stream, coop);
        case 23: return launch_pp_hd<128, 128, 0x4001>(a, stream, coop);
        case 24: return launch_pp_hd<128, 128, 0x4400>(a, stream, coop);
        case 25: return launch_pp_hd<128, 128, 0x4021>(a, stream, coop);
        case 26: return launch_pp_hd<128, 128, 0x4031>(a, stream, coop);
        case 27: return launch_pp_hd<128, 128, 0x4041>(a, stream, coop);
        case 28: return launch_pp_hd<128, 128, 0x4051>(a, stream, coop);
        case 21: return launch_pp_hd<128, 128, 0x2401>(a, stream, coop);
        case 16: return launch_pp_hd<128, 128, 0x1000>(a, stream, coop);
        case 17: return launch_pp_hd<128, 128, 0x1001>(a, stream, coop);
        case 18: return launch_pp_hd<128, 128, 0x1100>(a, stream, coop);
        case 19: return launch_pp_hd<128, 128, 0x1400>(a, stream, coop);
        case 100: return launch_pp_hd<128, 128, 0x0>(a, stream, coop);     // one warp per row quadrant
        case 30: return launch_pp_hd<128, 128, 0x8001>(a, stream, coop);   // single tile, S double-buffered
        case 31: return launch_pp_hd<128, 128, 0x8401>(a, stream, coop);
        case 32: return launch_pp_hd<128, 128, 0x8021>(a, stream, coop);
        case 33: return launch_pp_hd<128, 128, 0x8031>(a, stream, coop);
        case 34: return launch_pp_hd<128, 128, 0x8041>(a, stream, coop);
        case 35: return launch_pp_hd<128, 128, 0xA001>(a, stream, coop);
        case 36: return launch_pp_hd<128, 128, 0xC001>(a, stream, coop);   // single tile, two threads per row
        case 37: return launch_pp_hd<128, 128, 0x1C001>(a, stream, coop);  // + f16x2 exponentials
        case 38: return launch_pp_hd<128, 128, 0x18001>(a, stream, coop);  // single tile, SW 4, f16x2
        case 39: return launch_pp_hd<128, 128, 0x2C001>(a, stream, coop);  // single tile, SW 2, O per half
        // default: two threads per query row (PPRoles SW = 2), three-input max -- measured
        // 32.4 -> 31.8 us standalone, 5.25 -> 5.16 ms C3 TTFT (profiles/r1_attention_softmax_variants.txt)
        default: return launch_pp_hd<128, 128, 0x4001>(a, stream, coop);
      }
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_attention(const vlc_attn_args& a, cudaStream_t stream) {
  if (a.n_items <= 0) return cudaSuccess;
  switch (a.head_dim) {
    case 16: return launch_attn_hd<16>(a, stream);
    case 32: return launch_attn_hd<32>(a, stream);
    case 64: return launch_attn_hd<64>(a, stream);
    case 128: return launch_attn_hd<128>(a, stream);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_attn_combine(const vlc_attn_args& a, cudaStream_t stream) {
  if (a.n_comb <= 0) return cudaSuccess;
  switch (a.head_dim) {
    case 16: attn_combine_kernel<16><<<a.n_comb, 256, 0, stream>>>(a); break;
    case 32: attn_combine_kernel<32><<<a.n_comb, 256, 0, stream>>>(a); break;
    case 64: attn_combine_kernel<64><<<a.n_comb, 256, 0, stream>>>(a); break;
    case 128: attn_combine_kernel<128><<<a.n_comb, 256, 0, stream>>>(a); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace vlc
