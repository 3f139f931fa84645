// CTA-pair (cta_group::2) tcgen05 GEMM for the token-heavy projections of the reuse prefill
// (QKV, gate/up, LM head at c ~ 100-256 recomputed rows).
//
//   acc[f, j] = sum_k W[f, k] * X[j, k]        (swap-AB: weights on UMMA M = 256 per pair)
//
// Why: at c ~ 240 tokens a 128-row weight tile streams ~1.9 activation bytes per weight byte
// into its SM, and the single-CTA GEMM runs at the per-SM L2->SM ingress limit (~110 GB/s per
// SM measured, tools/gemm_epi_bench.py).  In a CTA pair each SM loads its own 128 weight rows
// but only HALF of the token rows of each activation k-block; the pair's tensor cores read both
// halves from the two SMs' shared memory.  Per-SM ingress per weight byte drops from 2.9 to 1.9
// bytes and the smaller stages fit one more pipeline stage.
//
// Roles (both CTAs run the same warps):
//   warp 0 lane 0   producer: own weight rows (one 32 KB bulk copy per 128-wide k-block) and
//                   own token half (two bulk copies, one per 64-column swizzle atom)
//   warp 1 lane 0   leader CTA: waits for its own stage and the peer's relay, issues
//                   tcgen05.mma.cta_group::2 (M = 256), commits stage / accumulator barriers
//                   to both CTAs (multicast); peer CTA: relays "stage landed" to the leader
//   warps 2-9       epilogue of this CTA's 128 accumulator rows (TMEM lanes), as vlc_gemm.cu
// Tiles (256 weight rows x <= 256 tokens) are assigned round-robin to pairs; no split-K, the
// accumulator is double-buffered so a pair's epilogue overlaps its next tile's mainloop.
#include "vlc_internal.h"
#include "vlc_gemm_epi.cuh"

namespace vlc {

constexpr int PAIR_EPI_WARPS = 8;
constexpr int PAIR_THREADS = 64 + 32 * PAIR_EPI_WARPS;

struct PairSched {
  int m_tiles2;   // 256-row weight tiles
  int tok_tiles;
  int KB;         // 128-wide k-blocks
  int n_pairs;
  unsigned long long* dbg;   // per-CTA phase timestamps (experiments; nullptr)
};
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
                 int n_tile, int stages) {
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
  const int n_tiles = sc.m_tiles2 * sc.tok_tiles;

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

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol_w = policy_evict_first();
      const uint64_t pol_x = policy_evict_last();
      // weights first (independent of the previous kernel), activations after griddepcontrol.wait
      int pre = 0;
      for (int t = pair; t < n_tiles && pre < stages; t += sc.n_pairs) {
        const uint8_t* wsrc = wp + (long)(2 * (t % sc.m_tiles2) + rank) * sc.KB * a_bytes;
        for (int kb = 0; kb < sc.KB && pre < stages; ++kb, ++pre) {
          mbar_expect_tx(&full[pre], a_bytes + b_bytes);
          bulk_load(sa + pre * a_bytes, wsrc + (long)kb * a_bytes, a_bytes, &full[pre], pol_w);
        }
      }
      pdl_wait();
      PDBG(1);
      int stage = 0, u = 0;
      uint32_t phase = 0;
      for (int t = pair; t < n_tiles; t += sc.n_pairs) {
        const uint8_t* wsrc = wp + (long)(2 * (t % sc.m_tiles2) + rank) * sc.KB * a_bytes;
        const uint8_t* xsrc = xp + (long)(t / sc.m_tiles2) * sc.KB * (2L * n_tile * 128) + (long)rank * atom_b;
        for (int kb = 0; kb < sc.KB; ++kb, ++u) {
          if (u >= pre) {
            mbar_wait(&empty[stage], phase ^ 1);
            mbar_expect_tx(&full[stage], a_bytes + b_bytes);
            bulk_load(sa + stage * a_bytes, wsrc + (long)kb * a_bytes, a_bytes, &full[stage], pol_w);
          }
          const uint8_t* xb = xsrc + (long)kb * (2L * n_tile * 128);
          bulk_load(sb + stage * b_bytes, xb, atom_b, &full[stage], pol_x);
          bulk_load(sb + stage * b_bytes + atom_b, xb + (long)n_tile * 128, atom_b, &full[stage], pol_x);
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
        for (int t = pair; t < n_tiles; t += sc.n_pairs)
          for (int kb = 0; kb < sc.KB; ++kb) {
            mbar_wait(&full[stage], phase);
            mbar_arrive_remote(mapa_shared(&peer_full[stage], 0));
            if (++stage == stages) { stage = 0; phase ^= 1; }
          }
      } else {
        const uint32_t idesc = make_idesc_bf16(256, n_tile, 0, 0);
        int stage = 0, seg = 0;
        uint32_t phase = 0;
        for (int t = pair; t < n_tiles; t += sc.n_pairs, ++seg) {
          const int slot = seg & 1;
          const uint32_t ap = ((seg >> 1) & 1) ^ 1;
          mbar_wait(&acc_empty[slot], ap);
          mbar_wait_cluster(&acc_empty_peer[slot], ap);
          tc_fence_after();
          const uint32_t d = tmem + slot * 256;
          for (int kb = 0; kb < sc.KB; ++kb) {
            mbar_wait(&full[stage], phase);
            mbar_wait_cluster(&peer_full[stage], phase);
            tc_fence_after();
            const uint32_t a_addr = smem_u32(sa + stage * a_bytes);
            const uint32_t b_addr = smem_u32(sb + stage * b_bytes);
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              const int at = k >> 2;
              const uint64_t ad = make_sdesc(a_addr + at * (128 * 128) + (k & 3) * 32, 16, 1024, 128);
              const uint64_t bd = make_sdesc(b_addr + at * atom_b + (k & 3) * 32, 16, 1024, 128);
              tc_mma2_f16(d, ad, bd, idesc, (kb > 0 || k > 0) ? 1u : 0u);
            }
            tc_commit2_mc(&empty[stage], 3);
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
    int seg = 0;
    for (int t = pair; t < n_tiles; t += sc.n_pairs, ++seg) {
      const int slot = seg & 1;
      const int m0 = (t % sc.m_tiles2) * 256 + rank * 128, tok0 = (t / sc.m_tiles2) * n_tile;
      mbar_wait(&acc_full[slot], (seg >> 1) & 1);
      tc_fence_after();
      if (threadIdx.x == 64) PDBG(3);
      const uint32_t d = tmem + slot * 256 + lane_off;
      const int nch = (n_tile + 31) / 32;
      for (int ci = eg; ci < nch; ci += 2) {
        const int c = ci * 32;
        float v[32];
        tmem_ld32(d + c, v);
        tmem_wait_ld();
#pragma unroll
        for (int jj = 0; jj < 32; ++jj) stage_buf[jj * 128 + row] = v[jj];
        asm volatile("bar.sync %0, 128;" ::"r"(bar_id) : "memory");
        const int jv = min(min(32, n_tile - c), epi.m_tokens - tok0 - c);
        write_chunk<KIND>(epi, m0 + 4 * lane, tok0 + c, quad, jv, stage_buf + 4 * lane);
        asm volatile("bar.sync %0, 128;" ::"r"(bar_id) : "memory");
      }
      tc_fence_before();
      asm volatile("bar.sync 3, 256;" ::: "memory");   // all 256 epilogue threads drained the slot
      if (threadIdx.x == 64) {
        if (leader) mbar_arrive(&acc_empty[slot]);
        else mbar_arrive_remote(mapa_shared(&acc_empty_peer[slot], 0));
      }
    }
    if (threadIdx.x == 64) PDBG(6);
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
cudaError_t launch_gemm_pair(const void* W, int n_pad, int k_pad, const void* X, int x_rows_cap, int m_tokens,
                             const GemmEpi& epi, int max_pairs, cudaStream_t stream) {
  const int n_tile = gemm_row_tile(m_tokens);
  if (n_pad % 256 || k_pad % 128 || n_tile % 16 || n_tile < 32) return cudaErrorNotSupported;
  const int tok_tiles = (m_tokens + n_tile - 1) / n_tile;
  if (x_rows_cap < tok_tiles * n_tile) return cudaErrorInvalidValue;
  int sms = 0, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  PairSched sc{n_pad / 256, tok_tiles, k_pad / 128, 0, debug_buffer()};
  const int tiles = sc.m_tiles2 * tok_tiles;
  int pairs = (sms > 0 ? sms : 148) / 2;
  if (max_pairs > 0 && max_pairs < pairs) pairs = max_pairs;
  if (tiles < pairs) pairs = tiles;
  sc.n_pairs = pairs;
  const int stages = pair_stages(n_tile);
  const int smem = pair_smem(n_tile, stages);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2 * pairs);
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
    return cudaLaunchKernelEx(&cfg, gemm_pair_tc<K>, wpp, xpp, epi, sc, n_tile, stages);                \
  }
  switch (epi.kind) {
    VLC_PAIR_KIND(EPI_F32)
    VLC_PAIR_KIND(EPI_BF16)
    VLC_PAIR_KIND(EPI_BIAS_ADD)
    VLC_PAIR_KIND(EPI_SWIGLU)
    VLC_PAIR_KIND(EPI_QKV_PLAIN)
    VLC_PAIR_KIND(EPI_QKV_ROPE)
    default:
      return cudaErrorNotSupported;   // RESID keeps the stream-K single-CTA kernel (red.add partials)
  }
#undef VLC_PAIR_KIND
}

}  // namespace vlc
