// Paged attention of the reuse prefill (K6; model.py:274-291, engine.py:179-182).
//
// The recomputed queries of one layer attend over ALL n keys of their request.  The keys are
// described as a list of 64-key CHUNKS (contiguous positions), each read from one of two places:
//   * the request's K/V rows (kc / vc, [layer][row][kv]): text and recomputed tokens, whose K the
//     QKV epilogue already rotated to its position -- and the few cached rows that share a chunk
//     with recomputed ones (relocated there by vlc_kv_relocate);
//   * a page of the store's pool (pool_k / pool_v, [row][kv]): cached image tokens, K rotated at the
//     position it was CACHED at (o + t).  At its new position s + t the reference re-rotates the
//     pre-RoPE key (engine.py:180); since RoPE rotations compose, R(s + t) k = R(D) R(o + t) k with
//     D = s - o the image's shift, and q . R(D) K = (R(-D) q) . K.  So instead of re-rotating every
//     cached key (per layer, per key), the CTA rotates its 128 queries ONCE by -D (four ROTATION
//     warps, fp32 tables of model.py:129-134) into a second Q buffer and multiplies the store chunks
//     against it; request chunks use the queries as they are.  A chunk's D rides in the upper bits
//     of its length word; a tile never pairs store chunks of two images (host padding), and when the
//     CTA's key range reaches the next image the rotation warps redo the rotation for its D once the
//     MMAs on the previous one are complete (q1_free / q1_ready).
// So the cached K/V of an image cross HBM once per layer, read-only, straight from the store: the
// gather + re-rotation + scatter of vlc_kv_relocate disappears into the consumer.
//
// CTA = (request, head, <= 128 position-sorted queries, range of 128-key tiles); tile j of an item
// = chunks chunk0 + 2j, 2j + 1 (the host pads every list to an even length).  Warp 0 issues the
// TMA loads (Q once; per K / V tile 2 chunks x the head's swizzle atoms), warp 1 the tcgen05.mma
// chain, warps 2-9 run the online softmax (two threads per query row, one per 64-key chunk, each
// with its own running max / sum and O accumulator in TMEM, merged once at the end), warps 10-13
// rotate the queries for the store chunks.  A 128-key tile whose two chunks need different query
// buffers is multiplied as two N = 64 halves.  S is double-buffered in TMEM: S(j+2) is issued after PV(j), so the
// tensor pipe computes S(j+1) while the softmax works on S(j).  P (bf16) overwrites S in TMEM and
// feeds O += P V as a TS-MMA.  Key ranges of long query tiles are split over co-resident CTAs that
// merge their fp32 partials in-kernel (group >= 0).
#include "vlc_internal.h"

namespace vlc {

constexpr int PA_CHUNK = 64;                 // keys per chunk (= store page rows / 64-row box)
constexpr int PA_KT = 128;                   // keys per tile (two chunks)
constexpr int PA_SOFT_WARPS = 8;             // 4 TMEM lane quadrants x 2 chunk halves
constexpr int PA_ROT_WARPS = 4;
constexpr int PA_WARPS = 2 + PA_SOFT_WARPS + PA_ROT_WARPS;
constexpr int PA_THREADS = 32 * PA_WARPS;    // 448
constexpr int PA_SMEM_MAX = 232448;

template <int HD>
struct PaCfg {
  static constexpr int ATOM_E = HD < 64 ? HD : 64;       // elements per swizzle atom row
  static constexpr int SWZ = ATOM_E * 2;                 // swizzle span (bytes): 32 / 64 / 128
  static constexpr int SWZ_B = SWZ == 128 ? 3 : (SWZ == 64 ? 2 : 1);
  static constexpr int N_ATOMS = HD / ATOM_E;
  static constexpr int Q_BYTES = 128 * HD * 2;
  static constexpr int Q_ATOM = 128 * SWZ;
  static constexpr int KV_BYTES = PA_KT * HD * 2;        // one 128-key tile
  static constexpr int KV_ATOM = PA_KT * SWZ;            // [atom][128 rows][SWZ]
  static constexpr int CH_ATOM_BYTES = PA_CHUNK * SWZ;   // one chunk's rows of one atom
  static constexpr int BAR_BYTES = 512;
  static constexpr int XM_BYTES = 2 * 2 * 128 * 4;       // merge exchange: [m | l][half][row] (in the V ring)
  static constexpr int RING = PA_SMEM_MAX - 1024 - BAR_BYTES - 2 * Q_BYTES;
  static constexpr int VST_FIT = RING / (2 * KV_BYTES);
  static constexpr int VST = VST_FIT > 6 ? 6 : VST_FIT;
  static constexpr int KST_FIT = (RING - VST * KV_BYTES) / KV_BYTES;
  static constexpr int KST = KST_FIT > 6 ? 6 : KST_FIT;
  static constexpr int SMEM = 1024 + 2 * Q_BYTES + (KST + VST) * KV_BYTES + BAR_BYTES;
  static_assert(VST * KV_BYTES >= XM_BYTES, "merge exchange lives in the V ring");
  static_assert(VST >= 2 && KST >= VST, "K / V rings");
  static_assert((KST + VST) * KV_BYTES >= 128 * HD * 4, "split partials are staged in the K/V ring");
  static_assert((KST + VST) * KV_BYTES >= 256 * 8 * 12 + 256 * 4, "merge tables live in the K/V ring");
  // TMEM: S[b] at 128 b (b = 0, 1: KT fp32 columns, P bf16 pairs over its first half of each chunk's
  // columns); O_h (h = chunk half) at 256 + 128 h (HD columns)
  __device__ static constexpr uint32_t s_col(int b) { return 128u * b; }
  __device__ static constexpr uint32_t o_col(int h) { return 256u + 128u * h; }
};

// byte offset of the 16-byte group q (dims 8q .. 8q+7) of row r (0..127) in a [atom][128][SWZ]
// tile, after the TMA / UMMA swizzle (Swizzle<B,4,3>: address bits [4, 4+B) ^= bits [7, 7+B))
template <int HD>
__device__ __forceinline__ uint32_t pa_swz_off(int r, int q) {
  using C = PaCfg<HD>;
  constexpr int GPA = C::ATOM_E / 8;                      // 16-byte groups per atom row
  const uint32_t lin = (uint32_t)((q / GPA) * C::KV_ATOM + r * C::SWZ + (q % GPA) * 16);
  return lin ^ (((lin >> 7) & ((1u << C::SWZ_B) - 1)) << 4);
}

template <int N>
__device__ __forceinline__ void tmem_ld_n(uint32_t taddr, float* v) {
  if constexpr (N == 16) {
    tmem_ld16(taddr, v);
  } else {
    static_assert(N == 8, "8 or 16 columns");
    uint32_t* r = reinterpret_cast<uint32_t*>(v);
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                   "=r"(r[7])
                 : "r"(taddr));
  }
}

// timing trace (a.trace != NULL only in timing studies): slot s of this CTA's 64 stamps
#define PA_TRACE(s)                                                                        \
  do {                                                                                     \
    if (a.trace) {                                                                         \
      unsigned long long t_;                                                               \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                               \
      a.trace[blockIdx.x * 64 + (s)] = t_;                                                 \
    }                                                                                      \
  } while (0)

template <int HD>
__global__ void __launch_bounds__(PA_THREADS, 1)
    attn_paged_kernel(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_kc,
                      const __grid_constant__ CUtensorMap map_vc, const __grid_constant__ CUtensorMap map_pk,
                      const __grid_constant__ CUtensorMap map_pv, vlc_attn_paged_args a) {
  using C = PaCfg<HD>;
  constexpr int CW = PA_CHUNK;            // S columns per softmax thread (one chunk)
  constexpr int OW = HD / 2;              // O columns per thread in the final store
  constexpr int OC = OW >= 16 ? 16 : OW;  // TMEM load width of the final store
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sQ1 = sQ + C::Q_BYTES;         // queries rotated by -D for the store chunks
  uint8_t* sK = sQ1 + C::Q_BYTES;
  uint8_t* sV = sK + C::KST * C::KV_BYTES;
  float* xm = reinterpret_cast<float*>(sV);   // used once every PV has completed
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + C::VST * C::KV_BYTES);
  uint64_t* q_full = bars;
  uint64_t* k_full = q_full + 1;          // [KST] TMA landed
  uint64_t* q1_ready = k_full + C::KST;   // rotated queries written (one phase per image run)
  uint64_t* q1_free = q1_ready + 1;       // every MMA on the previous run's rotated queries complete
  uint64_t* k_empty = q1_free + 1;        // [KST] S MMA done with the slot
  uint64_t* v_full = k_empty + C::KST;    // [VST]
  uint64_t* v_empty = v_full + C::VST;    // [VST]
  uint64_t* s_full = v_empty + C::VST;    // [2] S buffer b complete
  uint64_t* p_full = s_full + 2;          // [2] P written over S buffer b (all 256 softmax threads)
  uint64_t* o_done = p_full + 2;          // PV(j) complete (one phase per tile)
  uint64_t* all_done = o_done + 1;        // every MMA of the CTA complete (K/V ring reusable)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(all_done + 1);

  const int* it = a.items + blockIdx.x * 8;
  const int q_row0 = it[0], nq = it[1], head = it[2], chunk0 = it[3];
  const int tb = it[4], te = it[5], group = it[6];
  const int part = it[7] >> 8, nsplit = it[7] & 0xff;
  const int nt = te - tb;
  const int4* chunks = reinterpret_cast<const int4*>(a.chunks) + chunk0 + 2 * tb;   // this item's tiles

  const uint32_t warp = warp_id(), lane = lane_id();
  if (warp == 0 && lane == 0) {
    tma_prefetch(&map_q);
    tma_prefetch(&map_kc);
    tma_prefetch(&map_vc);
    tma_prefetch(&map_pk);
    tma_prefetch(&map_pv);
    mbar_init(q_full, 1);
    mbar_init(q1_ready, 32 * PA_ROT_WARPS);
    mbar_init(q1_free, 1);
    for (int s = 0; s < C::KST; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < C::VST; ++s) {
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&s_full[b], 1);
      mbar_init(&p_full[b], 32 * PA_SOFT_WARPS);
    }
    mbar_init(o_done, 1);
    mbar_init(all_done, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // Programmatic dependent launch: Q and the request K / V rows come from the QKV GEMM before this
  // kernel, so the producer waits for it (griddepcontrol.wait) -- but only after it has issued the
  // loads of the leading tiles whose chunks are all store pages (cached K / V, independent of it),
  // and the rotation warps work on those while the GEMM drains.  The softmax warps wait as well
  // (they write the attention output); the MMA warp only consumes shared memory / TMEM.
  if (warp >= 2 && warp < 2 + PA_SOFT_WARPS) {
    pdl_wait();
    if (threadIdx.x == 64) pdl_trigger();
  }
  if (threadIdx.x == 0) PA_TRACE(0);

  if (warp == 0) {
    // ---------------- TMA producer
    if (lane == 0 && nt > 0) {
      const uint64_t pol_q = policy_evict_first();
      const uint64_t pol_kv = policy_evict_normal();
      // one op per (chunk, atom): [atom][128 rows][SWZ] with chunk h in rows 64h .. 64h + 63
      auto load_tile = [&](uint8_t* dst, uint64_t* bar, int j, bool is_k) {
        mbar_expect_tx(bar, C::KV_BYTES);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int4 ch = chunks[2 * j + h];
#pragma unroll
          for (int at = 0; at < C::N_ATOMS; ++at) {
            uint8_t* d = dst + at * C::KV_ATOM + h * C::CH_ATOM_BYTES;
            if (ch.w < 0)          // request rows (kc / vc of this layer)
              tma_load_4d(d, is_k ? &map_kc : &map_vc, bar, 0, ch.z, head * C::N_ATOMS + at, a.layer, pol_kv);
            else                   // store page: pool row = page * P + offset
              tma_load_3d(d, is_k ? &map_pk : &map_pv, bar, 0, a.page_table[ch.z] * a.page_rows + ch.w,
                          head * C::N_ATOMS + at, pol_kv);
          }
        }
      };
      auto load_k = [&](int j) {
        const int st = j % C::KST;
        mbar_wait(&k_empty[st], ((j / C::KST) & 1) ^ 1);
        load_tile(sK + st * C::KV_BYTES, &k_full[st], j, true);
      };
      auto load_v = [&](int j) {
        const int st = j % C::VST;
        mbar_wait(&v_empty[st], ((j / C::VST) & 1) ^ 1);
        load_tile(sV + st * C::KV_BYTES, &v_full[st], j, false);
      };
      // leading store-only tiles before griddepcontrol.wait (their K / V do not depend on the GEMM)
      auto store_only = [&](int j) { return chunks[2 * j].w >= 0 && chunks[2 * j + 1].w >= 0; };
      int jk = 0, jv = 0;
      while (jk < C::KST - 1 && jk < nt && store_only(jk)) load_k(jk++);
      while (jv < C::VST && jv < jk) load_v(jv++);
      pdl_wait();
      mbar_expect_tx(q_full, C::Q_BYTES);
      tma_load_3d(sQ, &map_q, q_full, 0, q_row0, head * C::N_ATOMS, pol_q);
      // K runs KST - 1 tiles ahead of V (S(j) needs K(j) a softmax before PV(j) needs V(j))
      for (; jk < C::KST - 1 && jk < nt; ++jk) load_k(jk);
      for (int j = 0; j < nt; ++j) {
        if (j + C::KST - 1 < nt) load_k(j + C::KST - 1);
        if (j >= jv) load_v(j);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issue (one thread)
    if (lane == 0 && nt > 0) {
      const uint32_t idesc_s = make_idesc_bf16(128, PA_KT, 0, 0);
      const uint32_t idesc_h = make_idesc_bf16(128, PA_CHUNK, 0, 0);
      const uint32_t idesc_o = make_idesc_bf16(128, HD, 0, 1);
      mbar_wait(q_full, 0);
      PA_TRACE(1);
      int run = -1, run_d = 0;      // image run of the rotated queries in use
      auto issue_s = [&](int j) {   // S[j & 1] = Q K_j^T (store chunks against the rotated queries)
        const int st = j % C::KST;
        const int4 c0 = chunks[2 * j], c1 = chunks[2 * j + 1];
        const bool s0 = c0.w >= 0, s1 = c1.w >= 0;
        if (s0 || s1) {
          const int dj = (s0 ? c0.y : c1.y) >> 8;
          if (run < 0 || dj != run_d) {          // a new image: its rotation, after the old one's MMAs
            if (run >= 0) tc_commit(q1_free);
            ++run;
            run_d = dj;
            mbar_wait(q1_ready, run & 1);
          }
        }
        mbar_wait(&k_full[st], (j / C::KST) & 1);
        tc_fence_after();
        const uint32_t k_addr = smem_u32(sK + st * C::KV_BYTES);
        if (s0 == s1) {
          const uint32_t q_addr = smem_u32(s0 ? sQ1 : sQ);
#pragma unroll
          for (int k = 0; k < HD / 16; ++k) {
            const int at = (k * 16) / C::ATOM_E;
            const uint32_t eoff = ((k * 16) % C::ATOM_E) * 2;
            const uint64_t ad = make_sdesc(q_addr + at * C::Q_ATOM + eoff, 16, 8 * C::SWZ, C::SWZ);
            const uint64_t bd = make_sdesc(k_addr + at * C::KV_ATOM + eoff, 16, 8 * C::SWZ, C::SWZ);
            tc_mma_f16(tmem + C::s_col(j & 1), ad, bd, idesc_s, k > 0 ? 1u : 0u);
          }
        } else {
          // mixed tile: chunk h (key rows 64h ..) against its own query buffer, N = 64 each
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const uint32_t q_addr = smem_u32((h ? s1 : s0) ? sQ1 : sQ);
#pragma unroll
            for (int k = 0; k < HD / 16; ++k) {
              const int at = (k * 16) / C::ATOM_E;
              const uint32_t eoff = ((k * 16) % C::ATOM_E) * 2;
              const uint64_t ad = make_sdesc(q_addr + at * C::Q_ATOM + eoff, 16, 8 * C::SWZ, C::SWZ);
              const uint64_t bd = make_sdesc(k_addr + at * C::KV_ATOM + h * C::CH_ATOM_BYTES + eoff, 16,
                                             8 * C::SWZ, C::SWZ);
              tc_mma_f16(tmem + C::s_col(j & 1) + h * PA_CHUNK, ad, bd, idesc_h, k > 0 ? 1u : 0u);
            }
          }
        }
        tc_commit(&s_full[j & 1]);
        if (j + C::KST < nt) tc_commit(&k_empty[st]);   // the slot's next load waits on this
      };
      auto issue_pv = [&](int j) {  // O_h += P_h(j) V_h(j): chunk half h's keys into its own O
        const int st = j % C::VST;
        const uint32_t v_addr = smem_u32(sV + st * C::KV_BYTES);
#pragma unroll
        for (int k = 0; k < PA_KT / 16; ++k) {   // 16 keys per step; steps 0-3 chunk 0, 4-7 chunk 1
          const int h = k >> 2;
          const uint64_t bd = make_sdesc(v_addr + k * 16 * C::SWZ, C::KV_ATOM, 8 * C::SWZ, C::SWZ);
          // P of half h (bf16 pairs) sits in S columns [64 h, 64 h + 32)
          tc_mma_f16_ts(tmem + C::o_col(h), tmem + C::s_col(j & 1) + h * 64 + (k & 3) * 8, bd, idesc_o,
                        (j > 0 || (k & 3) > 0) ? 1u : 0u);
        }
        tc_commit(o_done);
        if (j + C::VST < nt) tc_commit(&v_empty[st]);
      };
      issue_s(0);
      if (nt > 1) issue_s(1);
      for (int j = 0; j < nt; ++j) {
        mbar_wait(&v_full[j % C::VST], (j / C::VST) & 1);
        mbar_wait(&p_full[j & 1], (j >> 1) & 1);
        tc_fence_after();
        issue_pv(j);
        if (j + 2 < nt) issue_s(j + 2);       // in order after PV(j): reuses P(j)'s TMEM columns
      }
      tc_commit(all_done);
    }
    __syncwarp();
  } else if (warp >= 2 + PA_SOFT_WARPS) {
    // ---------------- rotation warps: the queries rotated by -D for the store chunks (sQ1)
    // D = the shift of the image whose store chunks the tile reads; redone per image run of the range.
    // Lane -> two adjacent frequencies (f0, f0 + 1) of the head: one 4-byte word of the lower half row
    // (dims f0, f0 + 1) and one of the upper half (f0 + HD/2, ...); a warp covers RPW whole rows per
    // step (one 128-byte wavefront per access).  R(-D): (a, b) -> (a cos + b sin, b cos - a sin) with
    // cos / sin of D * theta from the fp32 tables (row |D|; sin flips sign for D < 0), in fp32, one
    // bf16 rounding.
    constexpr int LPR = HD / 4;                               // lanes per row
    constexpr int RPW = 32 / LPR;                             // rows per warp step
    constexpr int HALF = HD / 2;
    constexpr int STEPS = 128 / (PA_ROT_WARPS * RPW);
    constexpr int B = STEPS < 8 ? STEPS : 8;                  // rows per batch: loads, math, stores
    const int wr = (int)warp - (2 + PA_SOFT_WARPS);
    const int f0 = 2 * ((int)lane % LPR);
    auto eoff = [](int row, int e) -> uint32_t {
      const uint32_t lin = (uint32_t)((e / C::ATOM_E) * C::Q_ATOM + row * C::SWZ + (e % C::ATOM_E) * 2);
      return lin ^ (((lin >> 7) & ((1u << C::SWZ_B) - 1)) << 4);
    };
    const uint32_t q0 = smem_u32(sQ), q1 = smem_u32(sQ1);
    int run = -1, run_d = 0;
    for (int j = 0; j < nt; ++j) {
      const int4 c0 = chunks[2 * j], c1 = chunks[2 * j + 1];
      if (c0.w < 0 && c1.w < 0) continue;
      const int d = (c0.w >= 0 ? c0.y : c1.y) >> 8;
      if (run >= 0 && d == run_d) continue;
      // the rotation's table entries load while the queries land / the previous run's MMAs drain
      const int ad = d < 0 ? -d : d;
      const float2 c = __ldg(reinterpret_cast<const float2*>(a.cos_tab + (long)ad * a.tab_ld + f0));
      float2 sn = __ldg(reinterpret_cast<const float2*>(a.sin_tab + (long)ad * a.tab_ld + f0));
      if (run < 0) mbar_wait(q_full, 0);
      else mbar_wait(q1_free, run & 1);      // the MMAs on the previous image's rotation are complete
      ++run;
      run_d = d;
      if (d < 0) sn = make_float2(-sn.x, -sn.y);
      const float2 nsn = make_float2(-sn.x, -sn.y);
      for (int k0 = 0; k0 < STEPS; k0 += B) {
        uint32_t lo[B], hi[B];
#pragma unroll
        for (int k = 0; k < B; ++k) {
          const int row = (k0 + k) * PA_ROT_WARPS * RPW + wr * RPW + (int)lane / LPR;
          lo[k] = lds32(q0 + eoff(row, f0));
          hi[k] = lds32(q0 + eoff(row, f0 + HALF));
        }
#pragma unroll
        for (int k = 0; k < B; ++k) {
          const float2 av = make_float2(bf16_lo(lo[k]), bf16_hi(lo[k]));
          const float2 bv = make_float2(bf16_lo(hi[k]), bf16_hi(hi[k]));
          const float2 ro = ffma2(bv, sn, fmul2(av, c));      // a cos + b sin
          const float2 rh = ffma2(av, nsn, fmul2(bv, c));     // b cos - a sin
          lo[k] = pack_bf16(ro.x, ro.y);
          hi[k] = pack_bf16(rh.x, rh.y);
        }
#pragma unroll
        for (int k = 0; k < B; ++k) {
          const int row = (k0 + k) * PA_ROT_WARPS * RPW + wr * RPW + (int)lane / LPR;
          sts32(q1 + eoff(row, f0), lo[k]);
          sts32(q1 + eoff(row, f0 + HALF), hi[k]);
        }
      }
      fence_proxy_async_smem();      // generic-proxy writes -> visible to the tensor core's reads
      mbar_arrive(q1_ready);
    }
  } else {
    // ---------------- softmax: warp w -> TMEM lane quadrant w & 3, chunk half hh
    const int hh = (warp - 2) >> 2;
    const int quad = warp & 3;
    const int r = quad * 32 + lane;
    const bool q_valid = r < nq;
    const int qp = q_valid ? a.qpos[q_row0 + r] : -1;
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    const uint32_t tO = tmem + C::o_col(hh) + lane_off;
    const float NEG_INF = -INFINITY;
    float m_run = NEG_INF, l_run = 0.f;
    for (int j = 0; j < nt; ++j) {
      const int4 ch = chunks[2 * j + hh];
      const uint32_t tS = tmem + C::s_col(j & 1) + lane_off + hh * CW;
      float s[CW];
      mbar_wait(&s_full[j & 1], (j >> 1) & 1);
      tc_fence_after();
      if (warp == 2 && lane == 0 && j < 16) PA_TRACE(2 + j);
#pragma unroll
      for (int c = 0; c < CW / 32; ++c) tmem_ld32(tS + 32 * c, s + 32 * c);
      tmem_wait_ld();
      // column c is key position ch.x + c, valid for c < len and position <= the query's
      const int lim = min(qp - ch.x, (ch.y & 0xff) - 1);
      if (lim < CW - 1) {
#pragma unroll
        for (int i = 0; i < CW; ++i) s[i] = (i <= lim) ? s[i] : NEG_INF;
      }
      float mx4[4] = {NEG_INF, NEG_INF, NEG_INF, NEG_INF};
#pragma unroll
      for (int i = 0; i < CW; i += 2) mx4[(i >> 1) & 3] = fmax3(mx4[(i >> 1) & 3], s[i], s[i + 1]);
      const float pmax = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3]));
      const float tmax = pmax * a.scale_log2;
      const float m_new = fmaxf(m_run, tmax);
      const bool need = m_new > m_run + 8.0f;          // lazy rescale: only when the max grows by > 2^8
      const bool has_o = m_run != NEG_INF;
      const bool resc = __any_sync(0xffffffffu, need && has_o);
      // P(j) goes over S buffer j & 1, whose previous P (PV(j-2)) is complete: S(j) was issued after
      // it.  O is touched only when some row rescales, and then PV(j-1) must be complete first;
      // otherwise PV(j-1)'s phase is still observed below, before P(j) is published (every o_done
      // phase gets a waiter before the next one can complete -- compute-sanitizer synccheck)
      if (j > 0 && resc) {
        mbar_wait(o_done, (j - 1) & 1);
        tc_fence_after();
      }
      if (resc) {
        const float sc = (need && has_o) ? fast_exp2(m_run - m_new) : 1.0f;
#pragma unroll
        for (int c = 0; c < HD / 16; ++c) {
          float o[16];
          tmem_ld16(tO + c * 16, o);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 16; ++i) o[i] *= sc;
          tmem_st16(tO + c * 16, o);
        }
        tmem_wait_st();
      }
      if (need) {
        l_run = has_o ? l_run * fast_exp2(m_run - m_new) : 0.f;
        m_run = m_new;
      }
      const bool any = m_run != NEG_INF;
      const float nm = any ? -m_run : NEG_INF;       // all-masked row: every p = exp2(-inf) = 0
      float ls4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int i = 0; i < CW / 2; ++i) {               // P packed in place into s[0, CW/2)
        const float p0 = fast_exp2(fmaf(s[2 * i], a.scale_log2, nm));
        const float p1 = fast_exp2(fmaf(s[2 * i + 1], a.scale_log2, nm));
        ls4[i & 3] += p0 + p1;
        s[i] = __uint_as_float(pack_bf16(p0, p1));
      }
      l_run += (ls4[0] + ls4[1]) + (ls4[2] + ls4[3]);
      if (j > 0 && !resc) mbar_wait(o_done, (j - 1) & 1);   // PV(j-1): issued a softmax ago, done
      tmem_st32f(tS, s);                               // P over this half's own S columns
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(&p_full[j & 1]);
    }
    if (nt > 0) {    // o_done has completed nt - 1 or nt phases here
      mbar_wait(o_done, (nt - 1) & 1);
      tc_fence_after();
    }
    if (warp == 2 && lane == 0) PA_TRACE(50);
    // merge the two halves' (max, sum): M = max, w_h = 2^(m_h - M), L = w0 l0 + w1 l1
    xm[hh * 128 + r] = m_run;
    xm[256 + hh * 128 + r] = l_run;
    asm volatile("bar.sync 1, 256;" ::: "memory");
    const float m_o = xm[(1 - hh) * 128 + r], l_o = xm[256 + (1 - hh) * 128 + r];
    const float M = fmaxf(m_run, m_o);
    const float w_own = m_run == NEG_INF ? 0.f : fast_exp2(m_run - M);
    const float w_oth = m_o == NEG_INF ? 0.f : fast_exp2(m_o - M);
    l_run = w_own * l_run + w_oth * l_o;
    m_run = M;
    const int qrow = q_row0 + r;
    // OC O columns (chunk c of this thread's OW) of the row: w_own O_own + w_oth O_other
    auto load_o = [&](int c, float* o) {
      float o2[OC];
      tmem_ld_n<OC>(tmem + C::o_col(hh) + lane_off + hh * OW + c * OC, o);
      tmem_ld_n<OC>(tmem + C::o_col(1 - hh) + lane_off + hh * OW + c * OC, o2);
      tmem_wait_ld();
#pragma unroll
      for (int i = 0; i < OC; ++i) o[i] = w_own * o[i] + w_oth * o2[i];
    };
    if (group < 0) {
      const float inv = (l_run > 0.f) ? 1.0f / l_run : 0.f;
      const int orow_i = q_valid ? a.rowof[qrow] : 0;
      __nv_bfloat16* obase = reinterpret_cast<__nv_bfloat16*>(a.out);
#pragma unroll
      for (int c = 0; c < OW / OC; ++c) {
        float o[OC];
        if (nt > 0) {
          load_o(c, o);
        } else {
#pragma unroll
          for (int i = 0; i < OC; ++i) o[i] = 0.f;
        }
        if (q_valid) {
#pragma unroll
          for (int g8 = 0; g8 < OC / 8; ++g8) {
            uint32_t pkk[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) pkk[q] = pack_bf16(o[8 * g8 + 2 * q] * inv, o[8 * g8 + 2 * q + 1] * inv);
            const int col = head * HD + hh * OW + c * OC + 8 * g8;
            const long off = a.pk_rows > 0 ? packed_off(orow_i, col, a.pk_rows, a.pk_kb) : (long)orow_i * a.ldo + col;
            *reinterpret_cast<uint4*>(obase + off) = make_uint4(pkk[0], pkk[1], pkk[2], pkk[3]);
          }
        }
      }
    } else {
      // Split partial: once every MMA of the CTA is complete the K/V ring is free; stage the tile's
      // fp32 O rows there (row-major, float4 slot c4 at c4 ^ (row & 7): bank-conflict free, same
      // layout in ws_o) and write them with one bulk copy.
      const long prow0 = ((long)group * 8 + part) * 256;
      if (nt > 0) mbar_wait(all_done, 0);
      tc_fence_after();
      float4* stg = reinterpret_cast<float4*>(sK) + r * (HD / 4);
#pragma unroll
      for (int c = 0; c < OW / OC; ++c) {
        float o[OC];
        if (nt > 0) {
          load_o(c, o);
        } else {
#pragma unroll
          for (int i = 0; i < OC; ++i) o[i] = 0.f;
        }
#pragma unroll
        for (int q = 0; q < OC / 4; ++q) {
          const int c4 = (hh * OW + c * OC) / 4 + q;
          stg[c4 ^ (r & 7) % (HD / 4)] = make_float4(o[4 * q], o[4 * q + 1], o[4 * q + 2], o[4 * q + 3]);
        }
      }
      fence_proxy_async_smem();
      asm volatile("bar.sync 1, 256;" ::: "memory");
      if (quad == 0 && lane == 0 && hh == 0 && nq > 0)
        bulk_store_wait(a.ws_o + prow0 * HD, sK, (uint32_t)(nq * HD * 4));
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
  if (threadIdx.x == 0) PA_TRACE(51);
  if (group < 0) return;
  // ---------------- parallel merge of the nsplit partials (all CTAs of the group co-resident).
  // This CTA merges rows [r_lo, r_hi) of the group: pass 1 turns each row's (m, l) per split into
  // normalised weights (smem, in the K/V ring, free once this CTA's partial is written); pass 2 is
  // one thread per (row, float4 of the head) with every split's load independent.
  if (threadIdx.x == 0) {
    atomicAdd(&a.counters[group], 1);
    volatile int* cnt = a.counters + group;
    while (*cnt < nsplit) __nanosleep(32);
  }
  __syncthreads();
  __threadfence();
  if (threadIdx.x == 0) PA_TRACE(52);
  const int r_lo = nq * part / nsplit, r_hi = nq * (part + 1) / nsplit;
  const int nr = max(0, r_hi - r_lo);
  float2* s_ml = reinterpret_cast<float2*>(sK);                 // [nr][8]
  float* s_w = reinterpret_cast<float*>(s_ml + 256 * 8);        // [nr][8] weight / L
  int* s_orow = reinterpret_cast<int*>(s_w + 256 * 8);          // [nr]
  const long gbase = (long)group * 8 * 256;
  for (int t = threadIdx.x; t < nr * 8; t += PA_THREADS) {
    const int rr = t >> 3, s2 = t & 7;
    s_ml[t] = s2 < nsplit ? __ldcg(reinterpret_cast<const float2*>(a.ws_ml) + gbase + s2 * 256 + r_lo + rr)
                          : make_float2(-INFINITY, 0.f);
  }
  for (int rr = threadIdx.x; rr < nr; rr += PA_THREADS) s_orow[rr] = a.rowof[q_row0 + r_lo + rr];
  __syncthreads();
  for (int rr = threadIdx.x; rr < nr; rr += PA_THREADS) {
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
  for (int t = threadIdx.x; t < nr * C4; t += PA_THREADS) {
    const int rr = t / C4, c4 = t % C4;
    const int row = r_lo + rr;
    const float4* src = reinterpret_cast<const float4*>(a.ws_o) + (gbase + row) * C4 + ((c4 ^ (row & 7)) % C4);
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
  if (threadIdx.x == 0) PA_TRACE(53);
  if (threadIdx.x == 0) {
    // the last CTA of the group to finish merging re-zeroes both counters for the next launch
    if (atomicAdd(&a.counters[a.ws_slots + group], 1) == nsplit - 1) {
      a.counters[group] = 0;
      a.counters[a.ws_slots + group] = 0;
    }
  }
}

template <int HD>
static cudaError_t launch_paged_hd(const vlc_attn_paged_args& a, cudaStream_t stream) {
  using C = PaCfg<HD>;
  CUtensorMap mq, mkc, mvc, mpk, mpv;
  // Q: {atom elems, rows, atoms} box {ATOM_E, 128, N_ATOMS}
  cudaError_t e = make_tmap_3d(&mq, a.q, C::ATOM_E, a.q_rows_cap, a.kv / C::ATOM_E, (uint64_t)a.kv * 2,
                               (uint64_t)C::SWZ, C::ATOM_E, 128, C::N_ATOMS, C::SWZ);
  if (e != cudaSuccess) return e;
  // request K / V: {elems, rows, atoms, layer} box {ATOM_E, 64, 1, 1}
  const uint64_t dims[4] = {(uint64_t)C::ATOM_E, (uint64_t)a.kv_rows_cap, (uint64_t)(a.kv / C::ATOM_E),
                            (uint64_t)a.layers_cap};
  const uint64_t strides[3] = {(uint64_t)a.kv * 2, (uint64_t)C::SWZ, (uint64_t)a.kv * 2 * a.kv_rows_cap};
  const uint32_t box[4] = {(uint32_t)C::ATOM_E, (uint32_t)PA_CHUNK, 1, 1};
  if ((e = make_tmap_4d(&mkc, a.kc, dims, strides, box, C::SWZ)) != cudaSuccess) return e;
  if ((e = make_tmap_4d(&mvc, a.vc, dims, strides, box, C::SWZ)) != cudaSuccess) return e;
  // store pools: {elems, pool rows, atoms} box {ATOM_E, 64, 1}; without a pool the maps alias the
  // request buffers (never read: no chunk refers to the store)
  const void* pk = a.pool_k ? a.pool_k : a.kc;
  const void* pv = a.pool_v ? a.pool_v : a.vc;
  const uint64_t prow = a.pool_k ? (uint64_t)a.pool_rows : (uint64_t)a.kv_rows_cap;
  if ((e = make_tmap_3d(&mpk, pk, C::ATOM_E, prow, a.kv / C::ATOM_E, (uint64_t)a.kv * 2, (uint64_t)C::SWZ,
                        C::ATOM_E, PA_CHUNK, 1, C::SWZ)) != cudaSuccess)
    return e;
  if ((e = make_tmap_3d(&mpv, pv, C::ATOM_E, prow, a.kv / C::ATOM_E, (uint64_t)a.kv * 2, (uint64_t)C::SWZ,
                        C::ATOM_E, PA_CHUNK, 1, C::SWZ)) != cudaSuccess)
    return e;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attn_paged_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, PA_SMEM_MAX);
    attr = true;
  }
  return launch_chain(attn_paged_kernel<HD>, dim3(a.n_items), dim3(PA_THREADS), C::SMEM, stream, a.ws_slots > 0,
                      mq, mkc, mvc, mpk, mpv, a);
}

cudaError_t launch_attention_paged(const vlc_attn_paged_args& a, cudaStream_t stream) {
  if (a.n_items <= 0) return cudaSuccess;
  switch (a.head_dim) {
    case 16: return launch_paged_hd<16>(a, stream);
    case 32: return launch_paged_hd<32>(a, stream);
    case 64: return launch_paged_hd<64>(a, stream);
    case 128: return launch_paged_hd<128>(a, stream);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace vlc
