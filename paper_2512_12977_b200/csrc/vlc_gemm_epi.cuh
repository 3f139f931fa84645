// Fused GEMM epilogues shared by the single-CTA and CTA-pair tcgen05 GEMMs (vlc_gemm.cu,
// vlc_gemm_pair.cu): one call writes the final values of 4 consecutive device features of one
// token (write_group) or of the up-to-8 tokens a warp owns in a 32-token chunk (write_chunk).
#pragma once
#include "vlc_internal.h"

namespace vlc {

// silu(g) = g sigmoid(g) = g (1 + tanh(g / 2)) / 2: one MUFU op (tanh.approx, ~2^-11 relative) instead of
// two (ex2 + rcp) -- the SwiGLU epilogue is MUFU-paced (gate/up 31.25 -> 30.3 us at C3)
__device__ __forceinline__ float silu_f(float g) {
  float t;
  asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(0.5f * g));
  return 0.5f * g * (1.0f + t);
}

__device__ __forceinline__ uint2 pack4_bf16(float a, float b, float c, float d) {
  return make_uint2(pack_bf16(a, b), pack_bf16(c, d));
}

// Final values of 4 consecutive DEVICE features [F, F+4) of token j (token-major group).
// Device feature order: q/k rows permuted so RoPE pairs are adjacent (F, F+1), gate/up
// interleaved (gate f at 2f, up f at 2f+1); see model.py DeviceWeights.
template <int KIND>
__device__ __forceinline__ void write_group(const GemmEpi& e, int F, int j, float4 v) {
  if (F >= e.n_valid) return;
  const bool full4 = F + 4 <= e.n_valid;
  switch (KIND) {
    case EPI_F32: {
      const long r = e.map1 ? __ldg(e.map1 + j) : j;
      float* o = reinterpret_cast<float*>(e.out) + r * e.ldo + F;
      if (full4 && (e.ldo & 3) == 0) {
        *reinterpret_cast<float4*>(o) = v;
      } else {
        const float vv[4] = {v.x, v.y, v.z, v.w};
        for (int i = 0; i < 4 && F + i < e.n_valid; ++i) o[i] = vv[i];
      }
      break;
    }
    case EPI_RESID: {   // x += acc as an L2 vector reduction: split-K partials need no fixup
      float* o = reinterpret_cast<float*>(e.out) + (long)j * e.ldo + F;
      asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(o), "f"(v.x), "f"(v.y), "f"(v.z),
                   "f"(v.w)
                   : "memory");
      break;
    }
    case EPI_BF16: {
      const long off = e.pk_rows > 0 ? packed_off(j, F, e.pk_rows, e.pk_kb) : (long)j * e.ldo + F;
      *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(e.out) + off) = pack4_bf16(v.x, v.y, v.z, v.w);
      break;
    }
    case EPI_BIAS_ADD: {
      float4 b = e.bias ? __ldg(reinterpret_cast<const float4*>(e.bias + F)) : make_float4(0.f, 0.f, 0.f, 0.f);
      float4 a = e.add ? __ldg(reinterpret_cast<const float4*>(e.add + (long)j * e.ld_add + F))
                       : make_float4(0.f, 0.f, 0.f, 0.f);
      *reinterpret_cast<float4*>(reinterpret_cast<float*>(e.out) + (long)j * e.ldo + F) =
          make_float4((v.x + b.x) + a.x, (v.y + b.y) + a.y, (v.z + b.z) + a.z, (v.w + b.w) + a.w);
      break;
    }
    case EPI_SWIGLU: {
      const long off = e.pk_rows > 0 ? packed_off(j, F >> 1, e.pk_rows, e.pk_kb) : (long)j * e.ldo + (F >> 1);
      *reinterpret_cast<uint32_t*>(reinterpret_cast<__nv_bfloat16*>(e.out) + off) =
          pack_bf16(silu_f(v.x) * v.y, silu_f(v.z) * v.w);
      break;
    }
    case EPI_QKV_PLAIN: {
      const int sec = F / e.seg, r = F - sec * e.seg;
      void* dst = sec == 0 ? e.out : sec == 1 ? e.out2 : e.out3;
      const int ld = sec == 0 ? e.ldo : sec == 1 ? e.ld2 : e.ld3;
      *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(dst) + (long)j * ld + r) = pack4_bf16(v.x, v.y, v.z, v.w);
      break;
    }
    case EPI_QKV_ROPE: {
      const int sec = F / e.seg, r = F - sec * e.seg;
      if (sec == 2) {
        const long kr = __ldg(e.map2 + j);
        *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(e.out3) + kr * e.ld3 + r) =
            pack4_bf16(v.x, v.y, v.z, v.w);
        break;
      }
      const int half = e.hd >> 1;
      const int head = r / e.hd, t = (r - head * e.hd) >> 1;   // pairs (t, t+half), (t+1, t+1+half)
      const long tab = (long)__ldg(e.pos + j) * e.tab_ld + t;
      const float2 c = __ldg(reinterpret_cast<const float2*>(e.cos_tab + tab));
      const float2 sn = __ldg(reinterpret_cast<const float2*>(e.sin_tab + tab));
      const uint32_t lo = pack_bf16(v.x * c.x - v.y * sn.x, v.z * c.y - v.w * sn.y);
      const uint32_t hi = pack_bf16(v.y * c.x + v.x * sn.x, v.w * c.y + v.z * sn.y);
      const int fa = head * e.hd + t;
      if (sec == 0) {
        const long qr = e.map1 ? __ldg(e.map1 + j) : j;
        __nv_bfloat16* q = reinterpret_cast<__nv_bfloat16*>(e.out) + qr * e.ldo;
        *reinterpret_cast<uint32_t*>(q + fa) = lo;
        *reinterpret_cast<uint32_t*>(q + fa + half) = hi;
      } else {
        const long kr = __ldg(e.map2 + j);
        __nv_bfloat16* k = reinterpret_cast<__nv_bfloat16*>(e.out2) + kr * e.ld2;
        *reinterpret_cast<uint32_t*>(k + fa) = lo;
        *reinterpret_cast<uint32_t*>(k + fa + half) = hi;
        if (e.out4) {
          __nv_bfloat16* kp = reinterpret_cast<__nv_bfloat16*>(e.out4) + (long)j * e.ld4;
          *reinterpret_cast<uint32_t*>(kp + fa) = pack_bf16(v.x, v.z);
          *reinterpret_cast<uint32_t*>(kp + fa + half) = pack_bf16(v.y, v.w);
        }
      }
      break;
    }
    default:
      break;
  }
}

// QKV_ROPE epilogue split in two: the per-token metadata and RoPE table entries of a 32-token chunk
// (rope8_prefetch: independent of the accumulator, so the GEMM issues the next chunk's -- and, before the
// accumulator is ready, the first chunk's -- while it stores the current one) and the rotation + stores
// (rope8_store).  s_pos / s_dr: the tile's per-token positions and destination rows staged in shared
// memory (indexed by token), so a chunk's RoPE-table loads are one global round trip; NULL: global.
// Eight features per lane (F multiple of 8: RoPE pairs t .. t+3 of one head, t a multiple of 4): lanes
// 0-15 and 16-31 cover the 128 rows for two tokens at a time, tokens jj = b + 8q (q < 4) of the chunk with
// b = quad + 4 (lane / 16).  Each rotated half (4 bf16) is one 8-byte store and a V row segment one 16-byte
// store -- half the store instructions of the 4-feature mapping.  Needs head_dim % 8 == 0.
struct RopeMeta8 {
  int dr[4];
  float4 c[4], s[4];   // cos / sin of pairs t .. t+3 for each token
};
__device__ __forceinline__ void rope8_prefetch(const GemmEpi& e, int F, int j0, int b, int jv, RopeMeta8& m,
                                               const int* s_pos, const int* s_dr) {
  if (F >= e.n_valid) return;
  const int sec = F / e.seg, r = F - sec * e.seg;
  const int t = (r - (r / e.hd) * e.hd) >> 1;
  int p[4];
  if (s_pos) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int jj = b + 8 * q;
      if (jj < jv) p[q] = s_pos[j0 + jj], m.dr[q] = s_dr[j0 + jj];
    }
  } else {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int jj = b + 8 * q, j = j0 + jj;
      if (jj < jv) {
        if (sec != 2) p[q] = __ldg(e.pos + j);
        m.dr[q] = sec == 0 ? (e.map1 ? __ldg(e.map1 + j) : j) : __ldg(e.map2 + j);
      }
    }
  }
  if (sec == 2) return;
  if (e.cs_tab) {   // interleaved (cos t, cos t+1, sin t, sin t+1): two 16-byte loads per token
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (b + 8 * q < jv) {
        const float4* cs = reinterpret_cast<const float4*>(e.cs_tab + (long)p[q] * e.hd + 2 * t);
        const float4 u0 = __ldg(cs), u1 = __ldg(cs + 1);
        m.c[q] = make_float4(u0.x, u0.y, u1.x, u1.y);
        m.s[q] = make_float4(u0.z, u0.w, u1.z, u1.w);
      }
    }
    return;
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    if (b + 8 * q < jv) {
      const long tab = (long)p[q] * e.tab_ld + t;
      m.c[q] = __ldg(reinterpret_cast<const float4*>(e.cos_tab + tab));
      m.s[q] = __ldg(reinterpret_cast<const float4*>(e.sin_tab + tab));
    }
  }
}
__device__ __forceinline__ void rope8_store(const GemmEpi& e, int F, int j0, int b, int jv, const RopeMeta8& m,
                                            const float* sb) {
  if (F >= e.n_valid) return;
  const int sec = F / e.seg, r = F - sec * e.seg;
  if (sec == 2) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int jj = b + 8 * q;
      if (jj < jv) {
        const float4 x0 = *reinterpret_cast<const float4*>(sb + jj * 128);
        const float4 x1 = *reinterpret_cast<const float4*>(sb + jj * 128 + 4);
        const uint2 a = pack4_bf16(x0.x, x0.y, x0.z, x0.w), c = pack4_bf16(x1.x, x1.y, x1.z, x1.w);
        *reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(e.out3) + (long)m.dr[q] * e.ld3 + r) =
            make_uint4(a.x, a.y, c.x, c.y);
      }
    }
    return;
  }
  const int half = e.hd >> 1;
  const int head = r / e.hd, t = (r - head * e.hd) >> 1;   // pairs (t + i, t + i + half), i < 4
  const int fa = head * e.hd + t;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int jj = b + 8 * q;
    if (jj >= jv) continue;
    const float4 c = m.c[q], sn = m.s[q];
    const float4 x0 = *reinterpret_cast<const float4*>(sb + jj * 128);        // (t, t+h, t+1, t+1+h)
    const float4 x1 = *reinterpret_cast<const float4*>(sb + jj * 128 + 4);    // (t+2, t+2+h, t+3, t+3+h)
    const uint2 lo = pack4_bf16(x0.x * c.x - x0.y * sn.x, x0.z * c.y - x0.w * sn.y, x1.x * c.z - x1.y * sn.z,
                                x1.z * c.w - x1.w * sn.w);
    const uint2 hi = pack4_bf16(x0.y * c.x + x0.x * sn.x, x0.w * c.y + x0.z * sn.y, x1.y * c.z + x1.x * sn.z,
                                x1.w * c.w + x1.z * sn.w);
    __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(sec == 0 ? e.out : e.out2) +
                       (long)m.dr[q] * (sec == 0 ? e.ldo : e.ld2);
    *reinterpret_cast<uint2*>(o + fa) = lo;
    *reinterpret_cast<uint2*>(o + fa + half) = hi;
    if (sec == 1 && e.out4) {
      __nv_bfloat16* kp = reinterpret_cast<__nv_bfloat16*>(e.out4) + (long)(j0 + jj) * e.ld4;
      *reinterpret_cast<uint2*>(kp + fa) = pack4_bf16(x0.x, x0.z, x1.x, x1.z);
      *reinterpret_cast<uint2*>(kp + fa + half) = pack4_bf16(x0.y, x0.w, x1.y, x1.w);
    }
  }
}

// SwiGLU into the PACKED layout with eight features (four outputs) per lane, lanes 0-15 / 16-31 on two
// tokens per step (b = quad + 4 (lane / 16), tokens jj = b + 8q): one 8-byte store per lane per token --
// half the store instructions of write_chunk's four-feature mapping.  Returns false (caller falls back)
// unless the output is packed, the 8 features are valid and the chunk sits inside one row tile.
__device__ __forceinline__ bool swiglu8_packed(const GemmEpi& e, int F, int j0, int b, int jv, const float* sb) {
  const int R = e.pk_rows;
  if (R <= 0 || F + 8 > e.n_valid) return false;
  const int rt = j0 / R, r0 = j0 - rt * R;
  if (r0 + 32 > R) return false;
  const int k = F >> 1;                                     // outputs k .. k+3 (k % 4 == 0)
  const long base = ((((long)rt * e.pk_kb + (k >> 7)) * 2 + ((k >> 6) & 1)) * R) * 64 + (k & 7);
  const int c = (k >> 3) & 7;
  __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(e.out);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int jj = b + 8 * q;
    if (jj >= jv) continue;
    const int r = r0 + jj;
    const float4 x0 = *reinterpret_cast<const float4*>(sb + jj * 128);       // (g k, u k, g k+1, u k+1)
    const float4 x1 = *reinterpret_cast<const float4*>(sb + jj * 128 + 4);   // (g k+2, u k+2, ...)
    *reinterpret_cast<uint2*>(o + base + (long)r * 64 + ((c ^ (r & 7)) << 3)) =
        pack4_bf16(silu_f(x0.x) * x0.y, silu_f(x0.z) * x0.w, silu_f(x1.x) * x1.y, silu_f(x1.z) * x1.w);
  }
  return true;
}

// The up-to-8 tokens jj = quad + 4q (q < 8, jj < jv) of one 32-token chunk, features [F, F+4):
// loads of per-token metadata / RoPE tables are issued for all tokens before any store, so the
// epilogue is not a chain of dependent global-load latencies.  sb = stage + 4*lane (token stride
// 128 floats).
template <int KIND>
__device__ __forceinline__ void write_chunk(const GemmEpi& e, int F, int j0, int quad, int jv, const float* sb) {
  if constexpr (KIND == EPI_QKV_ROPE) {
    if (F >= e.n_valid) return;
    const int sec = F / e.seg, r = F - sec * e.seg;
    float4 v[8];
    int p[8];
    long dr[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int jj = quad + 4 * q;
      if (jj < jv) {
        const int j = j0 + jj;
        v[q] = *reinterpret_cast<const float4*>(sb + jj * 128);
        p[q] = __ldg(e.pos + j);
        dr[q] = sec == 0 ? (e.map1 ? __ldg(e.map1 + j) : j) : __ldg(e.map2 + j);
      }
    }
    if (sec == 2) {
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (quad + 4 * q < jv)
          *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(e.out3) + dr[q] * e.ld3 + r) =
              pack4_bf16(v[q].x, v[q].y, v[q].z, v[q].w);
      return;
    }
    const int half = e.hd >> 1;
    const int head = r / e.hd, t = (r - head * e.hd) >> 1;   // pairs (t, t+half), (t+1, t+1+half)
    const int fa = head * e.hd + t;
    float2 cq[8], sq[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      if (quad + 4 * q < jv) {
        const long tab = (long)p[q] * e.tab_ld + t;
        cq[q] = __ldg(reinterpret_cast<const float2*>(e.cos_tab + tab));
        sq[q] = __ldg(reinterpret_cast<const float2*>(e.sin_tab + tab));
      }
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      if (quad + 4 * q >= jv) continue;
      const float2 c = cq[q], sn = sq[q];
      const float4 x = v[q];
      const uint32_t lo = pack_bf16(x.x * c.x - x.y * sn.x, x.z * c.y - x.w * sn.y);
      const uint32_t hi = pack_bf16(x.y * c.x + x.x * sn.x, x.w * c.y + x.z * sn.y);
      __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(sec == 0 ? e.out : e.out2) + dr[q] * (sec == 0 ? e.ldo : e.ld2);
      *reinterpret_cast<uint32_t*>(o + fa) = lo;
      *reinterpret_cast<uint32_t*>(o + fa + half) = hi;
      if (sec == 1 && e.out4) {
        __nv_bfloat16* kp = reinterpret_cast<__nv_bfloat16*>(e.out4) + (long)(j0 + quad + 4 * q) * e.ld4;
        *reinterpret_cast<uint32_t*>(kp + fa) = pack_bf16(x.x, x.z);
        *reinterpret_cast<uint32_t*>(kp + fa + half) = pack_bf16(x.y, x.w);
      }
    }
  } else {
    if constexpr (KIND == EPI_BF16 || KIND == EPI_SWIGLU) {
      // PACKED output, chunk inside one row tile: one division per chunk instead of one per token
      // (packed_off's row / R) -- the packed store path was ~3.5 us of the gate/up epilogue
      const int R = e.pk_rows;
      if (R > 0 && F < e.n_valid && F + 4 <= e.n_valid) {
        const int rt = j0 / R, r0 = j0 - rt * R;
        if (r0 + 32 <= R) {
          const int k = KIND == EPI_SWIGLU ? (F >> 1) : F;
          const long base = ((((long)rt * e.pk_kb + (k >> 7)) * 2 + ((k >> 6) & 1)) * R) * 64 + (k & 7);
          const int c = (k >> 3) & 7;
          __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(e.out);
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int jj = quad + 4 * q;
            if (jj >= jv) continue;
            const int r = r0 + jj;
            const long off = base + (long)r * 64 + ((c ^ (r & 7)) << 3);
            const float4 v = *reinterpret_cast<const float4*>(sb + jj * 128);
            if constexpr (KIND == EPI_SWIGLU)
              *reinterpret_cast<uint32_t*>(o + off) = pack_bf16(silu_f(v.x) * v.y, silu_f(v.z) * v.w);
            else
              *reinterpret_cast<uint2*>(o + off) = pack4_bf16(v.x, v.y, v.z, v.w);
          }
          return;
        }
      }
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int jj = quad + 4 * q;
      if (jj < jv) write_group<KIND>(e, F, j0 + jj, *reinterpret_cast<const float4*>(sb + jj * 128));
    }
  }
}


}  // namespace vlc
