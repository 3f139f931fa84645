// CTA-pair (cta_group::2) stream-K tcgen05 GEMM: the projections of the reuse prefill
// (QKV, O, gate/up, down, LM head at c ~ 100-256 recomputed rows).
//
//   acc[f, j] = sum_k W[f, k] * X[j, k]        (swap-AB: weights on UMMA M = 256 per pair)
//
// Why a pair: at c ~ 240 tokens a single-CTA GEMM is bound by its SM's shared-memory traffic --
// every operand byte is written once by the bulk copy and read once by the UMMA (~128 B/clk per
// SM), and a 128-row weight tile drags ~1.9 activation bytes through shared memory per weight byte.
// In a CTA pair each SM loads its own 128 weight rows but only HALF of the token rows of each
// activation k-block, and the pair's tensor cores read each half once for both SMs: per-SM
// shared-memory bytes per weight byte drop from ~3.8 to ~2.
// Why stream-K: a one-wave projection has too few 256-row tiles to cover the SMs (QKV at C3:
// 42 tiles for 74 pairs), so the work units are (256-row tile, 128-wide k-block) and pair p takes
// the contiguous unit range [U p / P, U (p + 1) / P): every SM streams ~1/148 of the weights.
//
// A pair's range is a sequence of tile SEGMENTS, each accumulated in one of two TMEM slots (the
// epilogue of one overlaps the mainloop of the next).  The segment holding a tile's k-block 0
// OWNS the tile; every other segment of that tile is the FIRST segment of a later pair's range,
// so it finishes early: it stores its fp32 partial ([tokens][128 rows], one slot per CTA) and bumps
// the tile's flag, and the owner adds the partials in its epilogue before the fused write.
// RESID tiles need no fix-up: each segment reduces straight into the fp32 residual (red.add).
// The owner only ever waits on CTAs of LATER pairs, which never wait themselves before storing
// their partial, so the schedule cannot deadlock even if the pairs are not all co-resident.
//
// Roles (both CTAs run the same warps):
//   warp 0 lane 0   producer: own weight rows (one 32 KB bulk copy per 128-wide k-block) and
//                   own token half (two bulk copies, one per 64-column swizzle atom); the first ring
//                   pass of weights is issued before griddepcontrol.wait (PDL)
//   warp 1 lane 0   leader CTA: waits for its own stage and the peer's relay, issues
//                   tcgen05.mma.cta_group::2 (M = 256), commits stage / accumulator barriers
//                   to both CTAs (multicast); peer CTA: relays "stage landed" to the leader
//   warps 2-9       epilogue of this CTA's 128 accumulator rows (TMEM lanes): TMEM -> smem stage ->
//                   coalesced token-major writes (write_chunk of vlc_gemm_epi.cuh)
#include "vlc_internal.h"
#include "vlc_gemm_epi.cuh"

namespace vlc {

constexpr int PAIR_EPI_WARPS = 8;
constexpr int PAIR_THREADS = 64 + 32 * PAIR_EPI_WARPS;
constexpr int PAIR_FLAG = 12288;   // counters[PAIR_FLAG + 2 t + rank]: finished partials of tile t (t < 2048)

struct PairSched {
  int m_tiles2;   // 256-row weight tiles
  int tok_tiles;
  int KB;         // 128-wide k-blocks
  int n_pairs;
  long long U;    // units: m_tiles2 * tok_tiles * KB
  unsigned long long* dbg;   // per-CTA phase timestamps (experiments; nullptr)
  __device__ __forceinline__ long long u0(int p) const { return U * p / n_pairs; }
  __device__ __forceinline__ int pair_of(long long u) const {
    int p = (int)((u * n_pairs) / U);
    while (p + 1 < n_pairs && u0(p + 1) <= u) ++p;
    while (p > 0 && u0(p) > u) --p;
    return p;
  }
};
#ifdef VLC_PAIR_TRACE   // experiment builds only: per-unit stamps [cta][64 units][4] in the debug buffer
#define PTR(u, k)                                                                          \
  do {                                                                                     \
    if (sc.dbg && (u) < 64) {                                                              \
      unsigned long long t_;                                                               \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                               \
      sc.dbg[4096 + ((long)blockIdx.x * 64 + (u)) * 4 + (k)] = t_;                         \
    }                                                                                      \
  } while (0)
#else
#define PTR(u, k) do { } while (0)
#endif
#define PDBG(slot)                                                                        \
  do {                                                                                    \
    if (sc.dbg) {                                                                         \
      unsigned long long t_;                                                              \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                              \
      sc.dbg[blockIdx.x * 8 + (slot)] = t_;                                               \
    }                                                                                     \
  } while (0)

template <int KIND>
__global__ void __launch_bounds__(PAIR_THREADS, 1)
    gemm_pair_tc(const uint8_t* __restrict__ wp, const uint8_t* __restrict__ xp, GemmEpi epi, PairSched sc,
                 int n_tile, int stages, float* __restrict__ ws, int* __restrict__ counters) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int half = n_tile >> 1;                 // token rows held by this CTA
  const int a_bytes = 128 * 128 * 2;            // 32 KB: own 128 weight rows x 128 k
  const int atom_b = half * 128;                // one 64-column atom of the token half
  const int b_bytes = 2 * atom_b;
  uint8_t* sa = smem;
  uint8_t* sb = smem + stages * a_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(sb + stages * b_bytes);
  uint64_t* empty = full + stages;
  uint64_t* peer_full = empty + stages;
  uint64_t* acc_full = peer_full + stages;     // [2]
  uint64_t* acc_empty = acc_full + 2;          // [2] leader: this CTA's epilogue released the slot
  uint64_t* acc_empty_peer = acc_empty + 2;    // [2] leader: the peer's epilogue released it
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty_peer + 2);
  float* stage_all = reinterpret_cast<float*>(                  // [2][32][128] fp32, 128-B aligned
      (reinterpret_cast<uintptr_t>(acc_empty_peer + 2) + 8 + 127) & ~uintptr_t(127));

  const uint32_t warp = warp_id(), lane = lane_id();
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int pair = blockIdx.x >> 1;
  const long long u_begin = sc.u0(pair), u_end = sc.u0(pair + 1);
  const int t_first = (int)(u_begin / sc.KB);
  const int t_last = u_end > u_begin ? (int)((u_end - 1) / sc.KB) : t_first - 1;
  // k-block range [lo, hi) of tile t inside this pair's units
  auto kb_range = [&](int t, int& lo, int& hi) {
    const long long tb = (long long)t * sc.KB;
    lo = (int)(max(u_begin, tb) - tb);
    hi = (int)(min(u_end, tb + sc.KB) - tb);
  };

  if (warp == 0 && lane == 0) {
    PDBG(0);
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
      mbar_init(&peer_full[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&acc_full[s], 1);
      mbar_init(&acc_empty[s], 1);
      mbar_init(&acc_empty_peer[s], 1);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc2<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();          // the peer's barriers exist before any remote arrive
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // weight rows of k-block kb of tile t (this CTA's 128 of the 256) / its token half
  auto w_src = [&](int t, int kb) -> const uint8_t* {
    return wp + ((long)(2 * (t % sc.m_tiles2) + rank) * sc.KB + kb) * a_bytes;
  };
  auto x_src = [&](int t, int kb) -> const uint8_t* {
    return xp + ((long)(t / sc.m_tiles2) * sc.KB + kb) * (2L * n_tile * 128) + (long)rank * atom_b;
  };

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol_w = policy_evict_first();
      const uint64_t pol_x = policy_evict_last();
      // weights first (independent of the previous kernel), activations after griddepcontrol.wait
      int pre = 0;
      for (int t = t_first; t <= t_last && pre < stages; ++t) {
        int lo, hi;
        kb_range(t, lo, hi);
        for (int kb = lo; kb < hi && pre < stages; ++kb, ++pre) {
          mbar_expect_tx(&full[pre], a_bytes + b_bytes);
          bulk_load(sa + pre * a_bytes, w_src(t, kb), a_bytes, &full[pre], pol_w);
        }
      }
      pdl_wait();
      PDBG(1);
      int stage = 0, u = 0;
      uint32_t phase = 0;
      for (int t = t_first; t <= t_last; ++t) {
        int lo, hi;
        kb_range(t, lo, hi);
        for (int kb = lo; kb < hi; ++kb, ++u) {
          if (u >= pre) {
            mbar_wait(&empty[stage], phase ^ 1);
            mbar_expect_tx(&full[stage], a_bytes + b_bytes);
            bulk_load(sa + stage * a_bytes, w_src(t, kb), a_bytes, &full[stage], pol_w);
          }
          const uint8_t* xb = x_src(t, kb);
          bulk_load(sb + stage * b_bytes, xb, atom_b, &full[stage], pol_x);
          bulk_load(sb + stage * b_bytes + atom_b, xb + (long)n_tile * 128, atom_b, &full[stage], pol_x);
          PTR(u, 0);
          if (++stage == stages) { stage = 0; phase ^= 1; }
        }
      }
      PDBG(2);
    }
  } else if (warp == 1) {
    if (lane == 0) {
      if (!leader) {
        // relay: tell the leader each stage of this CTA has landed
        int stage = 0;
        uint32_t phase = 0;
        for (long long u = u_begin; u < u_end; ++u) {
          mbar_wait(&full[stage], phase);
          PTR((int)(u - u_begin), 1);
          mbar_arrive_remote(mapa_shared(&peer_full[stage], 0));
          if (++stage == stages) { stage = 0; phase ^= 1; }
        }
      } else {
        const uint32_t idesc = make_idesc_bf16(256, n_tile, 0, 0);
        int stage = 0, seg = 0;
        uint32_t phase = 0;
        int uu = 0;   // unit index within the range (trace)
        for (int t = t_first; t <= t_last; ++t, ++seg) {
          int lo, hi;
          kb_range(t, lo, hi);
          const int slot = seg & 1;
          const uint32_t ap = ((seg >> 1) & 1) ^ 1;
          mbar_wait(&acc_empty[slot], ap);
          mbar_wait_cluster(&acc_empty_peer[slot], ap);
          tc_fence_after();
          const uint32_t d = tmem + slot * 256;
          for (int kb = lo; kb < hi; ++kb) {
            mbar_wait(&full[stage], phase);
            PTR(uu, 1);
            mbar_wait_cluster(&peer_full[stage], phase);
            PTR(uu, 2);
            tc_fence_after();
            const uint32_t a_addr = smem_u32(sa + stage * a_bytes);
            const uint32_t b_addr = smem_u32(sb + stage * b_bytes);
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              const int at = k >> 2;
              const uint64_t ad = make_sdesc(a_addr + at * (128 * 128) + (k & 3) * 32, 16, 1024, 128);
              const uint64_t bd = make_sdesc(b_addr + at * atom_b + (k & 3) * 32, 16, 1024, 128);
              tc_mma2_f16(d, ad, bd, idesc, (kb > lo || k > 0) ? 1u : 0u);
            }
            tc_commit2_mc(&empty[stage], 3);
            PTR(uu, 3);
            ++uu;
            if (++stage == stages) { stage = 0; phase ^= 1; }
          }
          tc_commit2_mc(&acc_full[slot], 3);
        }
      }
    }
    __syncwarp();
  } else {
    pdl_wait();
    if (threadIdx.x == 64) pdl_trigger();
    // ---------------- epilogue: this CTA's 128 accumulator rows; group eg takes alternate
    // 32-token chunks; TMEM -> smem stage -> coalesced token-major writes (write_chunk)
    const int quad = warp & 3;
    const int eg = (warp - 2) >> 2;
    const int row = quad * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    float* stage_buf = stage_all + eg * 32 * 128;
    const int bar_id = 1 + eg;
    const bool lead_thr = threadIdx.x == 64;
    const long pslot = (long)n_tile * 128;                 // floats per partial slot
    int seg = 0;
    for (int t = t_first; t <= t_last; ++t, ++seg) {
      int lo, hi;
      kb_range(t, lo, hi);
      const int slot = seg & 1;
      const int m0 = (t % sc.m_tiles2) * 256 + rank * 128, tok0 = (t / sc.m_tiles2) * n_tile;
      const long long tb = (long long)t * sc.KB;
      const int p_own = sc.pair_of(tb), p_end = sc.pair_of(tb + sc.KB - 1);
      const bool split = KIND != EPI_RESID && p_end > p_own;   // RESID partials: red.add into x
      const bool owner = lo == 0;
      int* flag = counters + PAIR_FLAG + 2 * t + rank;
      if (split && owner) {
        // every later participant's partial is in L2 before its flag increment
        if (lead_thr) {
          volatile int* f = flag;
          while (*f < p_end - p_own) __nanosleep(32);
        }
        asm volatile("bar.sync 3, 256;" ::: "memory");
        __threadfence();
        if (lead_thr) PDBG(4);
      }
      mbar_wait(&acc_full[slot], (seg >> 1) & 1);
      tc_fence_after();
      if (lead_thr) PDBG(seg == 0 ? 5 : 3);
      const uint32_t d = tmem + slot * 256 + lane_off;
      const int nch = (n_tile + 31) / 32;
      float* part = ws + (long)blockIdx.x * pslot;
      for (int ci = eg; ci < nch; ci += 2) {
        const int c = ci * 32;
        float v[32];
        tmem_ld32(d + c, v);
        tmem_wait_ld();
        if (split && owner) {
          for (int q = p_own + 1; q <= p_end; ++q) {
            const float* pp = ws + (long)(2 * q + rank) * pslot + (long)c * 128 + row;
#pragma unroll
            for (int jj = 0; jj < 32; ++jj) v[jj] += __ldcg(pp + jj * 128);
          }
        }
#pragma unroll
        for (int jj = 0; jj < 32; ++jj) stage_buf[jj * 128 + row] = v[jj];
        asm volatile("bar.sync %0, 128;" ::"r"(bar_id) : "memory");
        const int jmax = min(32, n_tile - c);
        if (split && !owner) {
          for (int jj = quad; jj < jmax; jj += 4)
            __stcg(reinterpret_cast<float4*>(part + (long)(c + jj) * 128) + lane,
                   *reinterpret_cast<const float4*>(stage_buf + jj * 128 + 4 * lane));
        } else {
          const int jv = min(jmax, epi.m_tokens - tok0 - c);
          write_chunk<KIND>(epi, m0 + 4 * lane, tok0 + c, quad, jv, stage_buf + 4 * lane);
        }
        asm volatile("bar.sync %0, 128;" ::"r"(bar_id) : "memory");
      }
      tc_fence_before();
      if (split && !owner) __threadfence();                  // the partial is visible before the flag
      asm volatile("bar.sync 3, 256;" ::: "memory");   // all 256 epilogue threads drained the slot
      if (lead_thr) {
        if (leader) mbar_arrive(&acc_empty[slot]);
        else mbar_arrive_remote(mapa_shared(&acc_empty_peer[slot], 0));
        if (split) {
          if (owner) *flag = 0;                          // every participant has arrived: re-arm
          else atomicAdd(flag, 1);
        }
      }
    }
    if (lead_thr) PDBG(6);
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();          // the leader's MMAs read this CTA's smem / write its TMEM
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc2<512>(tmem);
  }
}

static int pair_stages(int n_tile) {
  const int per = 128 * 128 * 2 + n_tile * 128;   // 32 KB weights + half of the token rows (2 atoms)
  int s = (222 * 1024 - 32 * 1024) / per;
  return s > 8 ? 8 : (s < 2 ? 2 : s);
}

static int pair_smem(int n_tile, int stages) {
  return 1024 + stages * (128 * 128 * 2 + n_tile * 128) + (3 * stages + 6) * 8 + 8 + 128 + 2 * 32 * 128 * 4;
}

// Launchable when the weight rows form whole 256-row tiles and the token tile splits into two
// 8-row-aligned halves; returns cudaErrorNotSupported otherwise (caller falls back).
// ws: >= 2 * pairs * n_tile * 128 floats (split partials); counters: PAIR_FLAG + 2 * tiles ints, zero.
cudaError_t launch_gemm_pair(const void* W, int n_pad, int k_pad, const void* X, int x_rows_cap, int m_tokens,
                             const GemmEpi& epi, int max_pairs, float* ws, size_t ws_bytes, int* counters,
                             cudaStream_t stream) {
  const int n_tile = gemm_row_tile(n_pad, m_tokens);
  if (n_tile > 256) return cudaErrorNotSupported;
  if (n_pad % 256 || k_pad % 128 || n_tile % 16 || n_tile < 32) return cudaErrorNotSupported;
  const int tok_tiles = (m_tokens + n_tile - 1) / n_tile;
  if (x_rows_cap < tok_tiles * n_tile) return cudaErrorInvalidValue;
  const int stages = pair_stages(n_tile);
  const int smem = pair_smem(n_tile, stages);
  PairSched sc{n_pad / 256, tok_tiles, k_pad / 128, 0, 0, debug_buffer()};
  const long long tiles = (long long)sc.m_tiles2 * tok_tiles;
  sc.U = tiles * sc.KB;
  int pairs = 74;
  cudaLaunchConfig_t cfg{};
  cfg.blockDim = dim3(PAIR_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  int na = 1;
  if (g_pdl) {
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    na = 2;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  if (max_pairs > 0 && max_pairs < pairs) pairs = max_pairs;
  if ((long long)pairs * 2 > sc.U) pairs = (int)(sc.U / 2 > 0 ? sc.U / 2 : 1);   // >= 2 k-blocks per pair
  // split tiles of non-RESID kinds need the partial slots and flags; without them every pair owns
  // whole tiles (pairs divides tiles: tile-aligned unit ranges)
  const bool fix_ok = counters != nullptr && ws != nullptr &&
                      (size_t)2 * pairs * n_tile * 128 * sizeof(float) <= ws_bytes && PAIR_FLAG + 2 * tiles <= 16384;
  if (epi.kind != EPI_RESID && !fix_ok) {
    if (pairs > tiles) pairs = (int)tiles;
    while (pairs > 1 && tiles % pairs) --pairs;
  }
  sc.n_pairs = pairs;
  cfg.gridDim = dim3(2 * pairs);
  const uint8_t* wpp = reinterpret_cast<const uint8_t*>(W);
  const uint8_t* xpp = reinterpret_cast<const uint8_t*>(X);
#define VLC_PAIR_KIND(K)                                                                                 \
  case K: {                                                                                              \
    static bool attr = false;                                                                            \
    if (!attr) {                                                                                         \
      cudaFuncSetAttribute(gemm_pair_tc<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);        \
      cudaFuncSetAttribute(gemm_pair_tc<K>, cudaFuncAttributeNonPortableClusterSizeAllowed, 0);          \
      attr = true;                                                                                       \
    }                                                                                                    \
    return cudaLaunchKernelEx(&cfg, gemm_pair_tc<K>, wpp, xpp, epi, sc, n_tile, stages, ws, counters);  \
  }
  switch (epi.kind) {
    VLC_PAIR_KIND(EPI_F32)
    VLC_PAIR_KIND(EPI_RESID)
    VLC_PAIR_KIND(EPI_BF16)
    VLC_PAIR_KIND(EPI_BIAS_ADD)
    VLC_PAIR_KIND(EPI_SWIGLU)
    VLC_PAIR_KIND(EPI_QKV_PLAIN)
    VLC_PAIR_KIND(EPI_QKV_ROPE)
    default:
      return cudaErrorNotSupported;
  }
#undef VLC_PAIR_KIND
}

}  // namespace vlc
