// Gather + RoPE re-rotation + scatter of cached pre-RoPE K and copy of V (engine.py:153-155 +
// engine.py:180), one RELOC_TOK-token block of one (layer, image) descriptor per call, for the
// kv_relocate kernel (vlc_misc.cu).
#pragma once
#include "vlc_internal.h"

namespace vlc {

constexpr int RELOC_TOK = 8;
constexpr int RELOC_THREADS = 256;

struct RelocArgs {
  const __nv_bfloat16* kpool;
  const __nv_bfloat16* vpool;
  int page_tokens;
  const int* page_table;
  int kv, hd;
  __nv_bfloat16* kc;
  __nv_bfloat16* vc;
  int kv_rows_cap;
  const int* descs;         // int32 [n][8] = {layer, page_tab_off, tok0, ntok, dst_row0, pos0, 0, 0}
  const int2* blocks;       // int32 [n_blocks][2] = {desc, token offset}
  int n_blocks;
  const float* cos_tab;
  const float* sin_tab;
  int tab_ld;
};

__device__ __forceinline__ uint4 ldg_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ void rotate8(const uint4& a, const uint4& b, const float* c, const float* s, uint4& oa,
                                        uint4& ob) {
  const uint32_t* pa = &a.x;
  const uint32_t* pb = &b.x;
  uint32_t* qa = &oa.x;
  uint32_t* qb = &ob.x;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float a0 = bf16_lo(pa[i]), a1 = bf16_hi(pa[i]);
    const float b0 = bf16_lo(pb[i]), b1 = bf16_hi(pb[i]);
    const float c0 = c[2 * i], c1 = c[2 * i + 1], s0 = s[2 * i], s1 = s[2 * i + 1];
    qa[i] = pack_bf16(a0 * c0 - b0 * s0, a1 * c1 - b1 * s1);
    qb[i] = pack_bf16(b0 * c0 + a0 * s0, b1 * c1 + a1 * s1);
  }
}

// Block `b` with threads tid < RELOC_THREADS.  K: thread (token, frequency chunk of 8, head
// group) rotates 8 pairs per head with 128-bit loads of both halves, cos/sin for the token's
// position loaded once and reused across heads.  V: straight 128-bit copy.
__device__ __forceinline__ void relocate_block(const RelocArgs& r, int b, int tid) {
  const int2 blk = r.blocks[b];
  const int* dsc = r.descs + blk.x * 8;
  const int layer = dsc[0], pt_off = dsc[1], tok0 = dsc[2], ntok = dsc[3];
  const int dst0 = dsc[4], pos0 = dsc[5];
  const int t_begin = blk.y;
  const int t_count = min(RELOC_TOK, ntok - t_begin);
  const int kv = r.kv, hd = r.hd;
  const int heads = kv / hd;
  const int fchunks = hd / 16;
  const long layer_off = (long)layer * r.kv_rows_cap;
  const int group_threads = fchunks * RELOC_TOK;
  const int n_groups = RELOC_THREADS / group_threads;
  if (tid < n_groups * group_threads) {
    const int fc = tid % fchunks;
    const int tk = (tid / fchunks) % RELOC_TOK;
    const int hg = tid / group_threads;
    if (tk < t_count) {
      const int t = tok0 + t_begin + tk;
      const long src_row = (long)r.page_table[pt_off + t / r.page_tokens] * r.page_tokens + (t % r.page_tokens);
      const long dst_row = layer_off + dst0 + t_begin + tk;
      const int pos = pos0 + t_begin + tk;
      float c[8], s[8];
      const float4* cp = reinterpret_cast<const float4*>(r.cos_tab + (long)pos * r.tab_ld + fc * 8);
      const float4* sp = reinterpret_cast<const float4*>(r.sin_tab + (long)pos * r.tab_ld + fc * 8);
      *reinterpret_cast<float4*>(c) = __ldg(cp);
      *reinterpret_cast<float4*>(c + 4) = __ldg(cp + 1);
      *reinterpret_cast<float4*>(s) = __ldg(sp);
      *reinterpret_cast<float4*>(s + 4) = __ldg(sp + 1);
      const __nv_bfloat16* srow = r.kpool + src_row * kv;
      __nv_bfloat16* drow = r.kc + dst_row * kv;
      const int half = hd >> 1;
#pragma unroll 4
      for (int h = hg; h < heads; h += n_groups) {
        const int ea = h * hd + fc * 8;
        const uint4 a = ldg_stream(reinterpret_cast<const uint4*>(srow + ea));
        const uint4 bb = ldg_stream(reinterpret_cast<const uint4*>(srow + ea + half));
        uint4 oa, ob;
        rotate8(a, bb, c, s, oa, ob);
        *reinterpret_cast<uint4*>(drow + ea) = oa;
        *reinterpret_cast<uint4*>(drow + ea + half) = ob;
      }
    }
  }
  if (r.vc == nullptr) return;   // K only (the store's rotated-at-origin copy)
  const int vec_per_row = kv / 8;
  const int total = t_count * vec_per_row;
#pragma unroll 4
  for (int i = tid; i < total; i += RELOC_THREADS) {
    const int tk = i / vec_per_row, vi = i - tk * vec_per_row;
    const int t = tok0 + t_begin + tk;
    const long src_row = (long)r.page_table[pt_off + t / r.page_tokens] * r.page_tokens + (t % r.page_tokens);
    const long dst_row = layer_off + dst0 + t_begin + tk;
    const uint4 v = ldg_stream(reinterpret_cast<const uint4*>(r.vpool + src_row * kv) + vi);
    reinterpret_cast<uint4*>(r.vc + dst_row * kv)[vi] = v;
  }
}

}  // namespace vlc
