// Weight-streaming tcgen05 GEMM for the recomputed rows of the reuse prefill.
//
//   acc[f, j] = sum_k W[f, k] * X[j, k]          (swap-AB: weights on UMMA M)
//
// W (the layer weight, [n_out, k]) and X (the c computed tokens, [rows, k]) are both in the
// PACKED operand layout of include/vlcache.h, so each pipeline stage is two contiguous
// cp.async.bulk copies (32 KB of weights, n_tile*256 B of activations): TMA tensor boxes cost
// ~3 cycles per 128 B row per SM, bulk copies ~190 ns per op (tools/tma_probe.py).  A CTA owns a
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
#include <type_traits>

#include "vlc_internal.h"
#include "vlc_gemm_epi.cuh"

namespace vlc {

constexpr int GEMM_EPI_WARPS = 8;                  // two groups of 4 (one warp per TMEM lane quadrant)
constexpr int GEMM_THREADS = 64 + 32 * GEMM_EPI_WARPS;
constexpr int GEMM_BM = 128;
constexpr int GEMM_BK = 128;   // one stage = two 64-element (128 B) swizzle atoms along K
constexpr int GEMM_ATOM_K = 64;

// ------------------------------------------------------------------ stream-K schedule
struct SkSched {
  long long U;   // total work units = tiles * KB
  int G;         // CTAs (all co-resident: cooperative launch)
  int KB;        // k-blocks per tile
  int m_tiles;
  int red;       // RESID split partials reduced with red.add (1) or through the ordered fix-up (0)
  unsigned long long* dbg;   // phase timestamps (experiments; nullptr)
  int xh;        // decoupled: activation slots hold one 64-k atom (half a k-block) instead of a k-block
  int sw, sx;    // > 0: decoupled rings (one tile per CTA, H = 1): sw weight stages fed by warp 0 with
                 // no dependence on the previous kernel, sx activation stages fed by warp 2; the
                 // epilogue staging aliases the weight ring (free once the accumulator is complete)
  __device__ __forceinline__ long long u0(int g) const { return U * g / G; }
  __device__ __forceinline__ int cta_of(long long u) const {
    int g = (int)((u * G) / U);
    while (g + 1 < G && u0(g + 1) <= u) ++g;
    while (g > 0 && u0(g) > u) --g;
    return g;
  }
};

constexpr int SK_MAX_PART = 8;  // participants per split tile

static unsigned long long* h_dbg = nullptr;  // phase timestamps (experiments only; kernel parameter sk.dbg)
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define DBG(slot) do { if (sk.dbg) sk.dbg[blockIdx.x * 8 + (slot)] = gtimer(); } while (0)

// H = 1: 128 weight rows per tile, 128-wide k-blocks (two swizzle atoms), double-buffered TMEM
//        accumulator.
// H = 2: 256 weight rows per tile (two M=128 UMMAs sharing each activation k-block), 64-wide
//        k-blocks: the activation bytes per weight byte halve, which keeps the L2 traffic of
//        c ~ 240-token GEMMs under the LTS cap.  Single accumulator of 2 x n_tile columns.
// The A (weight) bytes of a stage are 32 KB in both cases.
// decoupled rings: the QKV_ROPE token tile's staged positions / destination rows + their barrier
constexpr int ROPE_STAGE_BYTES = 4096 + 64;
template <int KIND, int H>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    gemm_bf16_tc(const uint8_t* __restrict__ wp, const uint8_t* __restrict__ xp, GemmEpi epi, SkSched sk,
                 int n_tile, int stages, float* ws, int* counters) {
  constexpr int BM = GEMM_BM * H;
  constexpr int BK = GEMM_BK / H;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int a_bytes = BM * BK * 2;          // 32 KB
  const int b_bytes = n_tile * BK * 2;
  const bool dec = H == 1 && sk.sw > 0;
  const int wst = dec ? sk.sw : stages, xst = dec ? sk.sx : stages;   // weight / activation ring depth
  const int x_unit = (dec && sk.xh) ? b_bytes / 2 : b_bytes;          // activation slot bytes
  uint8_t* sa = smem;
  uint8_t* sb = smem + wst * a_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(sb + xst * x_unit);    // [wst] (coupled: both operands)
  uint64_t* empty = full + wst;
  uint64_t* xfull = empty + wst;                                       // [xst] decoupled only
  uint64_t* xempty = xfull + (dec ? xst : 0);
  uint64_t* acc_full = xempty + (dec ? xst : 0);   // [2]
  uint64_t* acc_empty = acc_full + 2;    // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  float* stage_all = dec ? reinterpret_cast<float*>(smem)   // [2][32][128] fp32
                         : reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(acc_empty) + 64);
  // decoupled rings, QKV_ROPE: the token tile's positions and destination rows ([512] + [512] int32, 4 KB)
  int* s_rope = reinterpret_cast<int*>(reinterpret_cast<uint8_t*>(acc_empty) + 64);
  uint64_t* rope_bar = reinterpret_cast<uint64_t*>(s_rope + 1024);

  const uint32_t warp = warp_id(), lane = lane_id();
  const int g = blockIdx.x;
  const long long u_begin = sk.u0(g), u_end = sk.u0(g + 1);
  const int t_first = (int)(u_begin / sk.KB);
  const int t_last = (u_end > u_begin) ? (int)((u_end - 1) / sk.KB) : t_first - 1;
  const int kb128 = H == 1 ? sk.KB : sk.KB / 2;   // 128-wide blocks per packed row tile
  // decoupled mode: every CTA owns exactly one k-range [dkb0, dkb0 + dnkb) of one tile
  const int dkb0 = (int)(u_begin - (long long)t_first * sk.KB), dnkb = (int)(u_end - u_begin);

  if (warp == 0 && lane == 0) {
    DBG(0);
    for (int s = 0; s < wst; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    if (dec)
      for (int s = 0; s < xst; ++s) {
        mbar_init(&xfull[s], 1);
        mbar_init(&xempty[s], 1);
      }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&acc_full[s], 1);
      mbar_init(&acc_empty[s], 32 * GEMM_EPI_WARPS);
    }
    if (dec) mbar_init(rope_bar, 32 * (GEMM_EPI_WARPS - 1));
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // source of the weight half h of k-block kb of weight tile mt (PACKED layout, include/vlcache.h)
  auto a_src = [&](int mt, int kb, int h) -> const uint8_t* {
    if (H == 1) return wp + ((long)mt * kb128 + kb) * 32768;
    return wp + ((((long)(2 * mt + h) * kb128 + (kb >> 1)) * 2 + (kb & 1)) << 14);
  };
  auto b_src = [&](int tt, int kb) -> const uint8_t* {
    if (H == 1) return xp + ((long)tt * kb128 + kb) * b_bytes;
    return xp + (((long)tt * kb128 + (kb >> 1)) * 2 + (kb & 1)) * (long)b_bytes;
  };

  if (dec && warp == 0) {
    // decoupled: weight ring only; weights never depend on the previous kernel (no pdl_wait), so
    // the ring fills while the predecessor drains and stays wst deep ahead of the MMA
    if (lane == 0) {
      DBG(1);
      const uint64_t pol_w = policy_evict_first();
      const int mt = t_first % sk.m_tiles;
      for (int i = 0; i < dnkb; ++i) {
        const int st = i % wst;
        if (i >= wst) mbar_wait(&empty[st], ((i / wst) & 1) ^ 1);
        mbar_expect_tx(&full[st], a_bytes);
        bulk_load(sa + st * a_bytes, a_src(mt, dkb0 + i, 0), a_bytes, &full[st], pol_w);
      }
      DBG(2);
    }
  } else if (dec && warp == 1) {
    if (lane == 0) {
      // N chunks: <= 256 tokens per UMMA; a wide tile (257..512) is two halves into adjacent columns
      const int nw0 = n_tile > 256 ? ((n_tile / 2 + 15) & ~15) : n_tile, nw1 = n_tile - nw0;
      const uint32_t idesc = make_idesc_bf16(GEMM_BM, nw0, 0, 0);
      const uint32_t idesc1 = make_idesc_bf16(GEMM_BM, nw1 > 0 ? nw1 : 16, 0, 0);
      mbar_wait(&acc_empty[0], 1);
      tc_fence_after();
      const int xper = sk.xh ? 2 : 1;   // activation slots per k-block
      long long c0 = 0;
      if (sk.dbg) { asm volatile("mov.u64 %0, %%clock64;" : "=l"(c0)); DBG(5); }
      // the narrow loop keeps the code of a single N chunk; wide tiles issue both chunks per K step
      auto mainloop = [&](auto wide_tag) {
        constexpr bool WIDE = decltype(wide_tag)::value;
        for (int kb = 0; kb < dnkb; ++kb) {   // kb: index within this CTA's single k-range
          const int ws_ = kb % wst;
          mbar_wait(&full[ws_], (kb / wst) & 1);
          const uint32_t a_addr = smem_u32(sa + ws_ * a_bytes);
#pragma unroll
          for (int hx = 0; hx < 2; ++hx) {
            if (hx >= xper) break;
            const int u = kb * xper + hx, xs = u % xst;
            mbar_wait(&xfull[xs], (u / xst) & 1);
            tc_fence_after();
            const uint32_t b_addr = smem_u32(sb + xs * x_unit);
#pragma unroll
            for (int k = 0; k < GEMM_BK / 16; ++k) {
              const int at = k >> 2;
              if (xper == 2 && at != hx) continue;   // half slots: atom hx of the k-block only
              const uint64_t ad = make_sdesc(a_addr + at * (GEMM_BM * 128) + (k & 3) * 32, 16, 1024, 128);
              const uint32_t b0 = b_addr + (xper == 2 ? 0 : at * (n_tile * 128)) + (k & 3) * 32;
              tc_mma_f16(tmem, ad, make_sdesc(b0, 16, 1024, 128), idesc, (kb > 0 || k > 0) ? 1u : 0u);
              if constexpr (WIDE)   // tokens nw0 .. n_tile: rows nw0.. of the same activation block
                tc_mma_f16(tmem + nw0, ad, make_sdesc(b0 + nw0 * 128, 16, 1024, 128), idesc1,
                           (kb > 0 || k > 0) ? 1u : 0u);
            }
            tc_commit(&xempty[xs]);
          }
          tc_commit(&empty[ws_]);
        }
      };
      if (nw1 > 0) mainloop(std::true_type{});
      else mainloop(std::false_type{});
      tc_commit(&acc_full[0]);
      if (sk.dbg) {   // mainloop SM cycles next to globaltimer slots 5 / 6: the SM clock under load
        mbar_wait(&acc_full[0], 0);
        long long c1;
        asm volatile("mov.u64 %0, %%clock64;" : "=l"(c1));
        DBG(6);
        sk.dbg[(160 + blockIdx.x) * 8] = (unsigned long long)(c1 - c0);   // buffers >= 320 x 8 entries
      }
    }
    __syncwarp();
  } else if (warp == 0) {
    if (lane == 0) {
      DBG(1);
      const uint64_t pol_w = policy_evict_first();
      const uint64_t pol_x = policy_evict_last();
      // The weights do not depend on the previous kernel: fill the first ring pass with weight
      // copies before waiting on it (programmatic dependent launch), activations after.
      int pre = 0;
      for (int t = t_first; t <= t_last && pre < stages; ++t) {
        const long long tb = (long long)t * sk.KB;
        const int kb_lo = (int)(max(u_begin, tb) - tb), kb_hi = (int)(min(u_end, tb + sk.KB) - tb);
        const int mt = t % sk.m_tiles;
        for (int kb = kb_lo; kb < kb_hi && pre < stages; ++kb, ++pre) {
          mbar_expect_tx(&full[pre], a_bytes + b_bytes);
#pragma unroll
          for (int h = 0; h < H; ++h)
            bulk_load(sa + pre * a_bytes + h * (a_bytes / H), a_src(mt, kb, h), a_bytes / H, &full[pre], pol_w);
        }
      }
      pdl_wait();
      int stage = 0, u = 0;
      uint32_t phase = 0;
      for (int t = t_first; t <= t_last; ++t) {
        const long long tb = (long long)t * sk.KB;
        const int kb_lo = (int)(max(u_begin, tb) - tb), kb_hi = (int)(min(u_end, tb + sk.KB) - tb);
        const int mt = t % sk.m_tiles, tt = t / sk.m_tiles;
        for (int kb = kb_lo; kb < kb_hi; ++kb, ++u) {
          if (u >= pre) {
            mbar_wait(&empty[stage], phase ^ 1);
            mbar_expect_tx(&full[stage], a_bytes + b_bytes);
#pragma unroll
            for (int h = 0; h < H; ++h)
              bulk_load(sa + stage * a_bytes + h * (a_bytes / H), a_src(mt, kb, h), a_bytes / H, &full[stage],
                        pol_w);
          }
          bulk_load(sb + stage * b_bytes, b_src(tt, kb), b_bytes, &full[stage], pol_x);
          if (++stage == stages) { stage = 0; phase ^= 1; }
        }
      }
      DBG(2);
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
        const int slot = H == 1 ? (seg & 1) : 0;
        const uint32_t acc_phase = H == 1 ? (((seg >> 1) & 1) ^ 1) : ((seg & 1) ^ 1);
        mbar_wait(&acc_empty[slot], acc_phase);
        tc_fence_after();
        const uint32_t d = tmem + slot * 256;
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(sa + stage * a_bytes);
          const uint32_t b_addr = smem_u32(sb + stage * b_bytes);
          if (H == 1) {
#pragma unroll
            for (int k = 0; k < GEMM_BK / 16; ++k) {
              const int at = k >> 2;
              const uint64_t ad = make_sdesc(a_addr + at * (GEMM_BM * 128) + (k & 3) * 32, 16, 1024, 128);
              const uint64_t bd = make_sdesc(b_addr + at * (n_tile * 128) + (k & 3) * 32, 16, 1024, 128);
              tc_mma_f16(d, ad, bd, idesc, (kb > 0 || k > 0) ? 1u : 0u);
            }
          } else {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const uint64_t bd = make_sdesc(b_addr + k * 32, 16, 1024, 128);
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const uint64_t ad = make_sdesc(a_addr + h * 16384 + k * 32, 16, 1024, 128);
                tc_mma_f16(d + h * 256, ad, bd, idesc, (kb > 0 || k > 0) ? 1u : 0u);
              }
            }
          }
          tc_commit(&empty[stage]);
          if (++stage == stages) { stage = 0; phase ^= 1; }
        }
        tc_commit(&acc_full[slot]);
      }
    }
    __syncwarp();
  } else {
    pdl_wait();                     // outputs / residual rows belong to the previous kernels
    if (threadIdx.x == 64) pdl_trigger();
    if (dec && warp == 2) {
      // decoupled: the activation ring (the previous kernel's output), xst deep ahead of the MMA
      if (lane == 0) {
        const uint64_t pol_x = policy_evict_last();
        const int tt = t_first / sk.m_tiles;
        const int xper = sk.xh ? 2 : 1;
        for (int u = 0; u < dnkb * xper; ++u) {
          const int st = u % xst;
          if (u >= xst) mbar_wait(&xempty[st], ((u / xst) & 1) ^ 1);
          mbar_expect_tx(&xfull[st], x_unit);
          const int kbu = dkb0 + (xper == 2 ? (u >> 1) : u);
          const uint8_t* src = xper == 2 ? b_src(tt, kbu) + (u & 1) * (n_tile * 128) : b_src(tt, kbu);
          bulk_load(sb + st * x_unit, src, x_unit, &xfull[st], pol_x);
        }
      }
      __syncwarp();
    }
    // ---------------- epilogue warps 2..9 (quad = TMEM lane quadrant).  H == 1: group eg = 0/1
    // takes alternate 32-column chunks; H == 2: group eg drains weight half eg.
    // TMEM (thread = weight row) -> smem stage [32 tokens][128 rows] -> token-major float4
    // groups written coalesced (write_group), or raw partial rows for split tiles.
    const int quad = warp & 3;
    const int eg = (warp - 2) >> 2;
    const int row = quad * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    float* stage_buf = stage_all + eg * 32 * 128;
    const int bar_id = 1 + eg;
    const bool leader = (threadIdx.x == 64);
    int seg = 0;
    for (int t = t_first; t <= t_last; ++t, ++seg) {
      const long long tb = (long long)t * sk.KB;
      const int gf = sk.cta_of(tb), gl = sk.cta_of(tb + sk.KB - 1);
      const int m0 = (t % sk.m_tiles) * BM, tok0 = (t / sk.m_tiles) * n_tile;
      const int slot = H == 1 ? (seg & 1) : 0;
      const bool split_t = gf != gl && !(KIND == EPI_RESID && sk.red);
      if constexpr (KIND == EPI_QKV_ROPE && H == 1) {
        if (!split_t) {
          // metadata + RoPE tables of chunk c+1 load while chunk c is stored; chunk 0's before the
          // accumulator is ready (all independent of it)
          const int nch = (n_tile + 31) / 32;
          // decoupled rings (one tile per CTA): the tile's positions / destination rows go to shared memory
          // while the mainloop runs -- warps 3..9 stage them (warp 2 is feeding the activation ring), every
          // epilogue warp waits on rope_bar
          const int* s_pos = nullptr;
          const int* s_dr = nullptr;
          if (dec) {
            if (warp != 2) {
              const int sec = m0 / epi.seg;
              for (int i = threadIdx.x - 96; i < n_tile; i += 32 * (GEMM_EPI_WARPS - 1)) {
                const int j = tok0 + i;
                const bool ok = j < epi.m_tokens;
                s_rope[i] = ok && sec != 2 ? __ldg(epi.pos + j) : 0;
                s_rope[512 + i] = !ok ? 0 : sec == 0 ? (epi.map1 ? __ldg(epi.map1 + j) : j) : __ldg(epi.map2 + j);
              }
              mbar_arrive(rope_bar);
            }
            mbar_wait(rope_bar, 0);
            s_pos = s_rope - tok0;
            s_dr = s_rope + 512 - tok0;
          }
          // eight features per lane (head_dim % 8 == 0, validated by vlc_gemm_bf16): lanes 0-15 / 16-31 take
          // two tokens per step, each rotated half one 8-byte store (vlc_gemm_epi.cuh)
          const int Fl = m0 + 8 * (lane & 15), bl = quad + 4 * (lane >> 4);
          const float* sbl = stage_buf + 8 * (lane & 15);
          RopeMeta8 ma, mb;   // two register-resident sets, roles alternate (no copies, no local memory)
          if (eg < nch)
            rope8_prefetch(epi, Fl, tok0 + eg * 32, bl, min(32, epi.m_tokens - tok0 - eg * 32), ma, s_pos, s_dr);
          mbar_wait(&acc_full[slot], (seg >> 1) & 1);
          tc_fence_after();
          if (leader) DBG(3);
          const uint32_t d = tmem + slot * 256 + lane_off;
          auto step = [&](int ci, const RopeMeta8& cur, RopeMeta8& nxt) {
            const int c = ci * 32;
            float v[32];
            tmem_ld32(d + c, v);
            tmem_wait_ld();
#pragma unroll
            for (int jj = 0; jj < 32; ++jj) stage_buf[jj * 128 + row] = v[jj];
            asm volatile("bar.sync %0, 128;" ::"r"(bar_id) : "memory");
            if (ci + 2 < nch)     // the chunk after next's tables load while this chunk is stored
              rope8_prefetch(epi, Fl, tok0 + c + 64, bl, min(32, epi.m_tokens - tok0 - c - 64), nxt, s_pos, s_dr);
            rope8_store(epi, Fl, tok0 + c, bl, min(32, epi.m_tokens - tok0 - c), cur, sbl);
            asm volatile("bar.sync %0, 128;" ::"r"(bar_id) : "memory");
          };
          for (int ci = eg; ci < nch; ci += 4) {
            step(ci, ma, mb);
            if (ci + 2 < nch) step(ci + 2, mb, ma);
          }
          tc_fence_before();
          mbar_arrive(&acc_empty[slot]);
          continue;
        }
      }
      mbar_wait(&acc_full[slot], H == 1 ? ((seg >> 1) & 1) : (seg & 1));
      tc_fence_after();
      if (leader) DBG(3);
      const uint32_t d = tmem + slot * 256 + (H == 2 ? eg * 256 : 0) + lane_off;
      const int hoff = H == 2 ? eg * 128 : 0;                 // weight-row offset of this group
      const bool split = gf != gl && !(KIND == EPI_RESID && sk.red);   // RESID partials: red.add in L2
      float* part = split ? ws + (2L * g + (t == t_first ? 0 : 1)) * (long)n_tile * BM : nullptr;
      const int nch = (n_tile + 31) / 32;
      for (int ci = (H == 1 ? eg : 0); ci < nch; ci += (H == 1 ? 2 : 1)) {
        const int c = ci * 32;
        float v[32];
        tmem_ld32(d + c, v);
        tmem_wait_ld();
#pragma unroll
        for (int jj = 0; jj < 32; ++jj) stage_buf[jj * 128 + row] = v[jj];
        asm volatile("bar.sync %0, 128;" ::"r"(bar_id) : "memory");
        const int jmax = min(32, n_tile - c);
        if (split) {
          for (int jj = quad; jj < jmax; jj += 4)
            __stcg(reinterpret_cast<float4*>(part + (long)(c + jj) * BM + hoff) + lane,
                   *reinterpret_cast<const float4*>(stage_buf + jj * 128 + 4 * lane));
        } else {
          const int jv = min(jmax, epi.m_tokens - tok0 - c);
          bool done = false;
          if constexpr (KIND == EPI_SWIGLU && H == 1) {   // packed SwiGLU: four outputs per lane (one store)
            done = swiglu8_packed(epi, m0 + 8 * (lane & 15), tok0 + c, quad + 4 * (lane >> 4), jv,
                                  stage_buf + 8 * (lane & 15));
          }
          if (!done) write_chunk<KIND>(epi, m0 + hoff + 4 * lane, tok0 + c, quad, jv, stage_buf + 4 * lane);
        }
        asm volatile("bar.sync %0, 128;" ::"r"(bar_id) : "memory");
      }
      tc_fence_before();
      mbar_arrive(&acc_empty[slot]);   // this thread's TMEM reads of the accumulator are done
      if (split) {
        __threadfence();
        asm volatile("bar.sync 3, 256;" ::: "memory");
        if (leader) atomicAdd(&counters[2 * gf], 1);
      }
    }
    if (leader) DBG(4);
    // ---- parallel fixup of the split tiles this CTA touched: participant p of nseg owns a
    // contiguous token range of the tile; partials are token-major rows of BM fp32, in the
    // partial slot (2 per CTA: first / last tile of its unit range) of each participant.
    const int ew = warp - 2;   // 0..7
    for (int t = t_first; t <= t_last; ++t) {
      const long long tb = (long long)t * sk.KB;
      const int gf = sk.cta_of(tb), gl = sk.cta_of(tb + sk.KB - 1);
      if (gf == gl || (KIND == EPI_RESID && sk.red)) continue;
      const int nseg = gl - gf + 1, p = g - gf;
      if (leader) {
        volatile int* cnt = counters + 2 * gf;
        while (*cnt < nseg) __nanosleep(32);
      }
      asm volatile("bar.sync 3, 256;" ::: "memory");
      __threadfence();
      if (leader) DBG(5);
      const int m0 = (t % sk.m_tiles) * BM, tok0 = (t / sk.m_tiles) * n_tile;
      const int j_lo = n_tile * p / nseg, j_hi = min(n_tile * (p + 1) / nseg, epi.m_tokens - tok0);
      const long pstride = (long)n_tile * BM;
      const float* bases[SK_MAX_PART];
#pragma unroll
      for (int s2 = 0; s2 < SK_MAX_PART; ++s2) {
        const int gp = gf + (s2 < nseg ? s2 : 0);
        bases[s2] = ws + (2L * gp + ((int)(sk.u0(gp) / sk.KB) == t ? 0 : 1)) * pstride;
      }
      for (int jt = j_lo + ew; jt < j_hi; jt += GEMM_EPI_WARPS) {
#pragma unroll
        for (int hf = 0; hf < H; ++hf) {
          float4 x[SK_MAX_PART];
#pragma unroll
          for (int s2 = 0; s2 < SK_MAX_PART; ++s2)
            if (s2 < nseg) x[s2] = __ldcg(reinterpret_cast<const float4*>(bases[s2] + (long)jt * BM + hf * 128) + lane);
          float4 acc = x[0];
#pragma unroll
          for (int s2 = 1; s2 < SK_MAX_PART; ++s2)
            if (s2 < nseg) { acc.x += x[s2].x; acc.y += x[s2].y; acc.z += x[s2].z; acc.w += x[s2].w; }
          write_group<KIND>(epi, m0 + hf * 128 + 4 * lane, tok0 + jt, acc);
        }
      }
      asm volatile("bar.sync 3, 256;" ::: "memory");
      if (leader) {
        if (atomicAdd(&counters[2 * gf + 1], 1) == nseg - 1) {
          counters[2 * gf] = 0;
          counters[2 * gf + 1] = 0;
        }
      }
    }
  }
  if (threadIdx.x == 64) DBG(6);
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
  if (threadIdx.x == 0) DBG(7);
}

int g_stage_override = 0;
void set_debug_buffer(unsigned long long* p) { h_dbg = p; }
unsigned long long* debug_buffer() { return h_dbg; }

int g_coop = 1;
int g_pdl = 1;

int g_pair = 0;           // tuning key 10: CTA-pair stream-K GEMM (multi-wave) when the token tile >= this (0 = off: measured)
int g_unsplit_min = 64;   // tuning key 9: tile count from which each tile gets its own CTA (no split-K)
int g_wide = 1;   // tuning key 7: 0 auto, 1 never use 256-row tiles (default: measured slower), 2 always
int g_aligned_split = 2;   // tuning key 17: tile-aligned split-K instead of stream-K when it fills >= 70% of SMs
                           // (1: split count divides the k-blocks, 2: any split count -- 140 CTAs on C3)
int g_dec_min_tile = 16;   // tuning key 20: smallest token tile that uses the decoupled rings
int g_decoupled = 1;       // tuning key 18: decoupled weight / activation rings for single-k-range CTAs
                           // (1: automatic activation depth, v >= 2: v stages, v >= 10: v-10 half-k-block
                           // stages, 0: off)

static int gemm_pick_stages(int n_tile, int H) {
  if (g_stage_override > 0) return g_stage_override;
  const int per = GEMM_BM * GEMM_BK * 2 + n_tile * (GEMM_BK / H) * 2;
  int s = (222 * 1024 - 32 * 1024) / per;
  if (s > 8) s = 8;
  if (s < 2) s = 2;
  return s;
}

static int gemm_smem_bytes(int n_tile, int stages, int H) {
  // pipeline stages + barriers (64 B reserved) + two 16 KB epilogue staging tiles
  return 1024 + stages * (GEMM_BM * GEMM_BK * 2 + n_tile * (GEMM_BK / H) * 2) + (2 * stages + 2) * 8 + 64 +
         2 * 32 * 128 * 4;
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

// Token (row) tile of a GEMM's packed activations: <= 256 rows per UMMA N, except that a one-wave GEMM
// (<= #SMs weight tiles) keeps 257..512 tokens in ONE wide tile -- two N chunks into one 512-column TMEM
// accumulator -- rather than two token tiles (which would double the CTAs past one wave: C3 at 6%
// recompute, c = 276 rows, ran at 1.9x the TTFT of 5%).
int gemm_row_tile(int n_pad, int m_tokens) {
  const int t = ((m_tokens + 15) / 16) * 16;
  if (m_tokens > 256 && m_tokens <= 512 && n_pad > 0 && n_pad / 128 <= num_sms()) return t;
  if (m_tokens >= 256) return 256;
  return t < 16 ? 16 : t;
}

// ws must hold G * 2 * BM * n_tile floats; counters 2 * G ints (zero).
cudaError_t launch_gemm(const void* W, int n_pad, int k_pad, const void* X, int x_rows_cap,
                        int m_tokens, const GemmEpi& epi, int max_ctas, float* ws, size_t ws_bytes,
                        int* counters, cudaStream_t stream) {
  if (m_tokens <= 0) return cudaSuccess;
  const int n_tile = gemm_row_tile(n_pad, m_tokens);
  const bool wide = n_tile > 256;   // one wide token tile: one k-range of one weight tile per CTA, decoupled rings
  // Multi-wave GEMMs (the LM head) with token tiles >= pair_min (key 10; default 0 = off): the CTA-pair
  // stream-K kernel (vlc_gemm_pair.cu).  Alone it is faster on the head (c = 236: 282 -> 258 us,
  // profiles/r2_gemm_pair_streamk.txt), but inside the prefill graph the single-CTA head gives the lower
  // TTFT (C3: 3.81 -> 3.77 ms, three A/B rounds, tools/ab_ttft.py VLC_TUNING=10:160 vs default): the
  // cluster launch starts later behind the last layer.  The one-wave projections stay on the single-CTA
  // kernel as well: under stream-K over all 74 pairs they are
  // L2-throughput bound like it (146 vs 219 MB through L2 but ~8 vs ~10 TB/s) and pay the exposed
  // last-segment epilogue on every SM (QKV 31.2 -> 32.9 us, gate/up 32.4 -> 38.3 us at c = 236).
  //  g_pair < 0: force the pair kernel from n_tile >= -g_pair (tests); 0: off
  const int pair_min = g_pair < 0 ? -g_pair : g_pair;
  const long long tiles128 = (long long)(n_pad / 128) * ((m_tokens + n_tile - 1) / n_tile);
  if (g_pair != 0 && n_tile >= pair_min && (g_pair < 0 || tiles128 >= 2LL * num_sms()) &&
      !(epi.kind == EPI_RESID && epi.deterministic)) {
    const cudaError_t e = launch_gemm_pair(W, n_pad, k_pad, X, x_rows_cap, m_tokens, epi,
                                           max_ctas > 0 ? max_ctas / 2 : 0, ws, ws_bytes, counters, stream);
    if (e != cudaErrorNotSupported) return e;
  }
  const bool wide_ok = n_pad % 256 == 0 && !wide;
  const int H = (g_wide == 2 && wide_ok) || (g_wide == 0 && wide_ok && n_tile >= 96) ? 2 : 1;
  const int BM = GEMM_BM * H, BK = GEMM_BK / H;
  const int KB = k_pad / BK;
  const int m_tiles = n_pad / BM;
  const int tok_tiles = (m_tokens + n_tile - 1) / n_tile;
  if (x_rows_cap < tok_tiles * n_tile) return cudaErrorInvalidValue;
  const long long U = (long long)m_tiles * tok_tiles * KB;
  int G = num_sms();
  if (max_ctas > 0 && max_ctas < G) G = max_ctas;
  // automatic schedule: enough weight tiles -> one CTA per tile (no split-K fixup); few tiles
  // (the d x d projections) -> stream-K over every SM
  const long long tiles = (long long)m_tiles * tok_tiles;
  if (max_ctas == 0 && tiles >= g_unsplit_min && tiles <= G) G = (int)tiles;
  // split tiles reduce through the workspace with <= 8 participants, except RESID (red.add into
  // the residual, any number of participants; >= 2 k-blocks per CTA)
  const bool red = epi.kind == EPI_RESID && !epi.deterministic;
  const int min_units = red ? 2 : (KB + 5) / 6;
  // Tile-aligned split-K when it keeps >= 70% of the SMs: every CTA then owns exactly one k-range
  // of one tile (one epilogue, no CTA waiting on a second tile's partial) -- measured on the C3
  // O / down projections: 148 stream-K CTAs 16.4 / 21.8 us, 112 aligned CTAs 14.0 / 19.9 us.
  // (g_aligned_split == 2: the split count need not divide the k-blocks -- G = tiles * s still puts
  // every CTA boundary of a tile on a tile boundary, ranges of floor / ceil(KB / s) k-blocks; only for
  // token tiles >= 160: at c = 112 the extra CTAs cost more than they bring, 3.64 -> 3.85 ms TTFT)
  if (max_ctas == 0 && g_aligned_split && tiles < G) {
    int best = 0;
    for (int sp = 2; sp <= KB / min_units; ++sp)
      if ((KB % sp == 0 || (g_aligned_split == 2 && n_tile >= 160)) && tiles * sp <= G) best = sp;
    if (best > 0 && (tiles * best * 10 >= 7LL * G || wide)) G = (int)(tiles * best);
  }
  if (wide) {
    // a single accumulator of n_tile columns: every CTA owns exactly one k-range of one weight tile
    if (tiles > num_sms()) return cudaErrorInvalidValue;
    if ((long long)G < tiles || G % tiles != 0 || G > num_sms()) G = (int)tiles;
  }
  if (!wide && (long long)G * min_units > U) G = (int)(U / min_units);
  if (G < 1) G = 1;
  const size_t need = (size_t)G * 2 * BM * n_tile * sizeof(float);
  if (!red && (need > ws_bytes || counters == nullptr)) {
    if (U / KB <= num_sms()) G = (int)(U / KB);   // no workspace: one CTA per tile, never split
    else return cudaErrorInvalidValue;
  }
  const int stages = gemm_pick_stages(n_tile, H);
  SkSched sk{U, G, KB, m_tiles, red ? 1 : 0, h_dbg, 0, 0, 0};
  // decoupled weight / activation rings for the one-tile-per-CTA schedule: the weight ring
  // (HBM-latency bound) gets every byte the activation ring (L2, 2 stages) leaves
  // (measured: QKV / gate-up at c = 236: 31.5 / 32.0 -> 29.9 / 29.6 us; slower at c = 112, where the
  // coupled ring already holds 3 stages -> only for token tiles >= 160)
  // (also for tile-aligned split-K: G a multiple of the tile count -> one k-range of one tile per CTA)
  if ((g_decoupled || wide) && H == 1 && n_tile >= g_dec_min_tile && G >= (int)tiles && G % (int)tiles == 0 &&
      tiles * KB == U && (U / G >= 2 || wide)) {
    const int a_b = GEMM_BM * GEMM_BK * 2, b_b = n_tile * GEMM_BK * 2;
    const int budget = 232448 - 1024 - 512 - ROPE_STAGE_BYTES;   // align, barriers, QKV_ROPE token metadata
    // key 18 value v: v in [2, 9] activation k-block stages; v >= 10: (v - 10) half-k-block stages
    // wide tiles: half-k-block activation slots when whole ones would leave < 2 weight stages
    const int xh = g_decoupled >= 10 || (wide && budget - 2 * b_b < 2 * a_b) ? 1 : 0;
    // g_decoupled == 1: floor(100 KB / activation stage) >= 2 activation stages -- measured best on C3:
    // 2 stages of 61 KB at c = 236, 3 of 28 KB at c = 112 (TTFT at r = 2%: 3.57 -> 3.49 ms)
    const int sx_auto = 100 * 1024 / b_b < 2 ? 2 : 100 * 1024 / b_b;
    const int sx = xh ? (g_decoupled - 10 >= 2 ? g_decoupled - 10 : 2)
                      : (g_decoupled >= 2 && !wide ? g_decoupled : sx_auto);
    const int xu = xh ? b_b / 2 : b_b;
    const int sw = (budget - sx * xu) / a_b;
    if (sw >= 2 && sw * a_b >= 2 * 32 * 128 * 4) { sk.sw = sw > 8 ? 8 : sw; sk.sx = sx; sk.xh = xh; }
  }
  if (wide && sk.sw <= 0) return cudaErrorInvalidValue;   // wide tiles run only on the decoupled rings
  const int smem = sk.sw > 0 ? 1024 + sk.sw * GEMM_BM * GEMM_BK * 2 + sk.sx * n_tile * GEMM_BK * (sk.xh ? 1 : 2) +
                                   (2 * sk.sw + 2 * sk.sx + 4) * 8 + 64 + ROPE_STAGE_BYTES
                             : gemm_smem_bytes(n_tile, stages, H);
  const uint8_t* wpp = reinterpret_cast<const uint8_t*>(W);
  const uint8_t* xpp = reinterpret_cast<const uint8_t*>(X);
  const int grid = G;
#define VLC_GEMM_KIND(K)                                                                              \
  case K: {                                                                                           \
    static bool attr = false;                                                                         \
    if (!attr) {                                                                                      \
      cudaFuncSetAttribute(gemm_bf16_tc<K, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);  \
      cudaFuncSetAttribute(gemm_bf16_tc<K, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);  \
      attr = true;                                                                                    \
    }                                                                                                 \
    if (H == 2)                                                                                       \
      return launch_chain(gemm_bf16_tc<K, 2>, dim3(grid), dim3(GEMM_THREADS), smem, stream, g_coop != 0, wpp,    \
                          xpp, epi, sk, n_tile, stages, ws, counters);                            \
    return launch_chain(gemm_bf16_tc<K, 1>, dim3(grid), dim3(GEMM_THREADS), smem, stream, g_coop != 0, wpp, xpp, \
                        epi, sk, n_tile, stages, ws, counters);                                   \
  }
  switch (epi.kind) {
    VLC_GEMM_KIND(EPI_F32)
    VLC_GEMM_KIND(EPI_RESID)
    VLC_GEMM_KIND(EPI_BF16)
    VLC_GEMM_KIND(EPI_BIAS_ADD)
    VLC_GEMM_KIND(EPI_SWIGLU)
    VLC_GEMM_KIND(EPI_QKV_PLAIN)
    VLC_GEMM_KIND(EPI_QKV_ROPE)
    default:
      return cudaErrorInvalidValue;
  }
#undef VLC_GEMM_KIND
}

// ------------------------------------------------------------------ operand packing
__global__ void pack_operand_kernel(const __nv_bfloat16* __restrict__ src, int rows, int cols, int ld,
                                    __nv_bfloat16* __restrict__ dst, int R, int KB) {
  const int row = blockIdx.x;
  if (row >= rows) return;
  for (int c8 = threadIdx.x * 8; c8 < cols; c8 += blockDim.x * 8) {
    if (c8 + 8 <= cols && (ld & 7) == 0) {
      *reinterpret_cast<uint4*>(dst + packed_off(row, c8, R, KB)) =
          *reinterpret_cast<const uint4*>(src + (long)row * ld + c8);
    } else {
      for (int k = c8; k < c8 + 8 && k < cols; ++k) dst[packed_off(row, k, R, KB)] = src[(long)row * ld + k];
    }
  }
}

cudaError_t launch_pack(const void* src, int rows, int cols, int ld, void* dst, int R, int KB, cudaStream_t s) {
  if (rows <= 0) return cudaSuccess;
  pack_operand_kernel<<<rows, 128, 0, s>>>(reinterpret_cast<const __nv_bfloat16*>(src), rows, cols, ld,
                                           reinterpret_cast<__nv_bfloat16*>(dst), R, KB);
  return cudaGetLastError();
}

}  // namespace vlc
