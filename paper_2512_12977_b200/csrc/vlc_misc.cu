// Bandwidth kernels of the reuse prefill: embedding assembly, RMSNorm, the
// fused KV gather + RoPE re-rotation + scatter (kv_relocate), store page writes
// and image patchify.
#include "vlc_internal.h"
#include "vlc_reloc.cuh"

namespace vlc {

// ------------------------------------------------------------------ embed (K1)
__global__ void embed_assemble_kernel(float* __restrict__ x, int ldx,
                                      const __nv_bfloat16* __restrict__ embed, int d,
                                      const float* __restrict__ enc_a,
                                      const float* __restrict__ enc_b,
                                      const int2* __restrict__ src, int rows) {
  pdl_wait();
  pdl_trigger();
  const int r = blockIdx.x;
  if (r >= rows) return;
  const int2 s = src[r];
  float* dst = x + (long)r * ldx;
  if ((d & 3) == 0 && (ldx & 3) == 0) {
    // 128-bit loads / stores, all of a thread's loads issued before its stores
    constexpr int U = 4;
    const int d4 = d >> 2;
    float4* o = reinterpret_cast<float4*>(dst);
    for (int i0 = threadIdx.x; i0 < d4; i0 += U * blockDim.x) {
      float4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = i0 + u * blockDim.x;
        v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (i >= d4 || (s.x == 0 && s.y < 0)) continue;   // negative text id: zero embedding (model.py:349-353)
        if (s.x == 0) {
          const uint2 e = __ldg(reinterpret_cast<const uint2*>(embed + (long)s.y * d) + i);
          v[u] = make_float4(bf16_lo(e.x), bf16_hi(e.x), bf16_lo(e.y), bf16_hi(e.y));
        } else {
          v[u] = __ldg(reinterpret_cast<const float4*>((s.x == 1 ? enc_a : enc_b) + (long)s.y * d) + i);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (i0 + u * blockDim.x < d4) o[i0 + u * blockDim.x] = v[u];
    }
    return;
  }
  if (s.x == 0 && s.y < 0) {          // negative text id: zero embedding (model.py:349-353)
    for (int i = threadIdx.x; i < d; i += blockDim.x) dst[i] = 0.f;
  } else if (s.x == 0) {
    const __nv_bfloat16* e = embed + (long)s.y * d;
    for (int i = threadIdx.x; i < d; i += blockDim.x) dst[i] = __bfloat162float(e[i]);
  } else {
    const float* e = (s.x == 1 ? enc_a : enc_b) + (long)s.y * d;
    for (int i = threadIdx.x; i < d; i += blockDim.x) dst[i] = e[i];
  }
}

// ------------------------------------------------------------------ rmsnorm (K4)
// One 128-thread block per row, the row held in registers as float4 (VPT per thread), so x
// is read once; cross-warp sum through shared memory.
// With `add` (head-parallel attention): x[row] += add[row] first (the all-reduced O projection),
// written back, then normalised.
template <bool OUT_F32, int VPT>
__global__ void __launch_bounds__(128) rmsnorm_kernel(float* __restrict__ x, int ldx,
                                                      const float* __restrict__ g, void* __restrict__ out,
                                                      int ldo, int rows, int d,
                                                      const int* __restrict__ row_map, float eps,
                                                      int pk_rows, int pk_kb, const float* __restrict__ add,
                                                      int ld_add) {
  const int n4 = d >> 2;
  // gamma does not depend on the previous kernel: load it before griddepcontrol.wait, so only the
  // residual row's load + reduction + store stay on the critical path
  float4 gg[VPT];
  const float4* g4 = reinterpret_cast<const float4*>(g);
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const int i = threadIdx.x + 128 * k;
    gg[k] = i < n4 ? __ldg(g4 + i) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  pdl_wait();
  pdl_trigger();
  const int r = blockIdx.x;
  const int sr = row_map ? __ldg(row_map + r) : r;
  float4* xr = reinterpret_cast<float4*>(x + (long)sr * ldx);
  float4 v[VPT];
  float acc = 0.f;
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const int i = threadIdx.x + 128 * k;
    v[k] = i < n4 ? xr[i] : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  if (add) {
    const float4* ar = reinterpret_cast<const float4*>(add + (long)sr * ld_add);
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
      const int i = threadIdx.x + 128 * k;
      if (i < n4) {
        const float4 a = ar[i];
        v[k] = make_float4(v[k].x + a.x, v[k].y + a.y, v[k].z + a.z, v[k].w + a.w);
        xr[i] = v[k];
      }
    }
  }
#pragma unroll
  for (int k = 0; k < VPT; ++k) acc += v[k].x * v[k].x + v[k].y * v[k].y + v[k].z * v[k].z + v[k].w * v[k].w;
#pragma unroll
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  __shared__ float red[4];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  // one reciprocal per row, then multiplies (the reference divides, model.py:257-259; the product differs by
  // <= 1 fp32 ulp before the bf16 rounding of the output)
  const float inv = 1.0f / sqrtf((red[0] + red[1] + red[2] + red[3]) / (float)d + eps);
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const int i = threadIdx.x + 128 * k;
    if (i >= n4) break;
    const float4 y = make_float4((v[k].x * inv) * gg[k].x, (v[k].y * inv) * gg[k].y,
                                 (v[k].z * inv) * gg[k].z, (v[k].w * inv) * gg[k].w);
    if (OUT_F32) {
      reinterpret_cast<float4*>(reinterpret_cast<float*>(out) + (long)r * ldo)[i] = y;
    } else {
      uint2 pk = make_uint2(pack_bf16(y.x, y.y), pack_bf16(y.z, y.w));
      const long off = pk_rows > 0 ? packed_off(r, 4 * i, pk_rows, pk_kb) : (long)r * ldo + 4 * i;
      *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(out) + off) = pk;
    }
  }
}

// Generic fallback (any d): block per row.
template <bool OUT_F32>
__global__ void rmsnorm_generic(float* __restrict__ x, int ldx, const float* __restrict__ g,
                                void* __restrict__ out, int ldo, int rows, int d,
                                const int* __restrict__ row_map, float eps, int pk_rows, int pk_kb,
                                const float* __restrict__ add, int ld_add) {
  pdl_wait();
  pdl_trigger();
  const int r = blockIdx.x;
  const int sr = row_map ? row_map[r] : r;
  float* xr = x + (long)sr * ldx;
  if (add) {
    for (int i = threadIdx.x; i < d; i += blockDim.x) xr[i] += add[(long)sr * ld_add + i];
    __syncthreads();
  }
  float acc = 0.f;
  for (int i = threadIdx.x; i < d; i += blockDim.x) acc += xr[i] * xr[i];
  __shared__ float red[32];
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  const float denom = sqrtf(red[0] / (float)d + eps);
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    const float y = (xr[i] / denom) * g[i];
    if (OUT_F32) reinterpret_cast<float*>(out)[(long)r * ldo + i] = y;
    else reinterpret_cast<__nv_bfloat16*>(out)[pk_rows > 0 ? packed_off(r, i, pk_rows, pk_kb) : (long)r * ldo + i] =
        __float2bfloat16_rn(y);
  }
}

// ------------------------------------------------------------------ kv_relocate (K2+K3)
// One CTA per RELOC_TOK-token block (vlc_reloc.cuh).
__global__ void __launch_bounds__(RELOC_THREADS) kv_relocate_kernel(RelocArgs r) {
  pdl_wait();
  pdl_trigger();
  relocate_block(r, blockIdx.x, threadIdx.x);
}

cudaError_t launch_relocate(const RelocArgs& r, cudaStream_t stream) {
  if (r.n_blocks <= 0) return cudaSuccess;
  return launch_chain(kv_relocate_kernel, dim3(r.n_blocks), dim3(RELOC_THREADS), 0, stream, false, r);
}

// ------------------------------------------------------------------ store pages
template <bool SRC_F32>
__global__ void store_pages_kernel(const void* __restrict__ src, int layers, int tokens, int kv,
                                   const int* __restrict__ page_table, int pages_per_layer,
                                   __nv_bfloat16* __restrict__ pool, int page_tokens) {
  const long row = blockIdx.x;  // layer * tokens + t
  const int layer = (int)(row / tokens), t = (int)(row % tokens);
  const long dst = (long)page_table[layer * pages_per_layer + t / page_tokens] * page_tokens + t % page_tokens;
  __nv_bfloat16* d = pool + dst * kv;
  if (SRC_F32) {
    const float* s = reinterpret_cast<const float*>(src) + row * kv;
    for (int i = threadIdx.x; i < kv; i += blockDim.x) d[i] = __float2bfloat16_rn(s[i]);
  } else {
    const __nv_bfloat16* s = reinterpret_cast<const __nv_bfloat16*>(src) + row * kv;
    for (int i = threadIdx.x; i < kv; i += blockDim.x) d[i] = s[i];
  }
}

// ------------------------------------------------------------------ row gather (merged KV)
__global__ void __launch_bounds__(256) gather_rows_kernel(uint4* __restrict__ dst, const int* __restrict__ drow,
                                                          const uint4* __restrict__ src, const int* __restrict__ srow,
                                                          int n, int row16) {
  for (long r = blockIdx.x; r < n; r += gridDim.x) {
    const uint4* s = src + (long)__ldg(srow + r) * row16;
    uint4* d = dst + (long)__ldg(drow + r) * row16;
    for (int i = threadIdx.x; i < row16; i += blockDim.x) d[i] = __ldcs(s + i);
  }
}

// ------------------------------------------------------------------ patchify
__global__ void patchify_kernel(const float* __restrict__ px, int side, int p,
                                __nv_bfloat16* __restrict__ out, int row0, int pk_rows, int pk_kb) {
  const int t = blockIdx.x;  // patch index, row-major over the patch grid
  const int per_row = side / p;
  const int ty = t / per_row, tx = t % per_row;
  for (int e = threadIdx.x; e < p * p; e += blockDim.x) {
    const int py = e / p, pxx = e % p;
    out[packed_off(row0 + t, e, pk_rows, pk_kb)] = __float2bfloat16_rn(px[(long)(ty * p + py) * side + tx * p + pxx]);
  }
}

}  // namespace vlc

using namespace vlc;

extern "C" {

int vlc_embed_assemble_impl(float* x, int ldx, const void* embed_bf16, int d, const float* enc_a,
                            const float* enc_b, const int* src, int rows, cudaStream_t stream) {
  if (rows <= 0) return 0;
  return (int)launch_chain(embed_assemble_kernel, dim3(rows), dim3(256), 0, stream, false, x, ldx,
                           reinterpret_cast<const __nv_bfloat16*>(embed_bf16), d, enc_a, enc_b,
                           reinterpret_cast<const int2*>(src), rows);
}

int vlc_rmsnorm_impl(float* x, int ldx, const float* gamma, void* out, int ldo, int out_f32,
                     int rows, int d, const int* row_map, float eps, int pk_rows, int pk_kb, cudaStream_t stream,
                     const float* add, int ld_add) {
  if (rows <= 0) return 0;
  const bool vec = (d % 4 == 0) && (ldx % 4 == 0) && (pk_rows > 0 || ldo % 4 == 0) && d <= 128 * 4 * 16 &&
                   (add == nullptr || ld_add % 4 == 0);
  const unsigned blocks = rows;
  cudaError_t e = cudaSuccess;
#define VLC_RMS(VPT)                                                                                   \
  e = launch_chain(out_f32 ? rmsnorm_kernel<true, VPT> : rmsnorm_kernel<false, VPT>, dim3(blocks), dim3(128), 0, \
                   stream, false, x, ldx, gamma, out, ldo, rows, d, row_map, eps, pk_rows, pk_kb, add, ld_add);
  if (vec) {
    const int vpt = (d / 4 + 127) / 128;
    if (vpt <= 1) { VLC_RMS(1) }
    else if (vpt <= 2) { VLC_RMS(2) }
    else if (vpt <= 4) { VLC_RMS(4) }
    else if (vpt <= 8) { VLC_RMS(8) }
    else { VLC_RMS(16) }
  } else {
    e = launch_chain(out_f32 ? rmsnorm_generic<true> : rmsnorm_generic<false>, dim3(rows), dim3(256), 0, stream,
                     false, x, ldx, gamma, out, ldo, rows, d, row_map, eps, pk_rows, pk_kb, add, ld_add);
  }
#undef VLC_RMS
  return (int)e;
}

int vlc_kv_relocate_impl(const void* kpool, const void* vpool, int page_tokens, const int* page_table,
                         int kv, int head_dim, void* kc, void* vc, int kv_rows_cap, const int* descs,
                         const int* blocks, int n_blocks, const float* cos_tab, const float* sin_tab,
                         int tab_ld, cudaStream_t stream) {
  if (n_blocks <= 0) return 0;
  RelocArgs r{reinterpret_cast<const __nv_bfloat16*>(kpool), reinterpret_cast<const __nv_bfloat16*>(vpool),
              page_tokens, page_table, kv, head_dim, reinterpret_cast<__nv_bfloat16*>(kc),
              reinterpret_cast<__nv_bfloat16*>(vc), kv_rows_cap, descs, reinterpret_cast<const int2*>(blocks),
              n_blocks, cos_tab, sin_tab, tab_ld};
  return (int)launch_relocate(r, stream);
}

int vlc_store_write_pages_impl(const void* src, int src_f32, int layers, int tokens, int kv,
                               const int* page_table, int pages_per_layer, void* pool, int page_tokens,
                               cudaStream_t stream) {
  const long rows = (long)layers * tokens;
  if (rows <= 0) return 0;
  if (src_f32)
    store_pages_kernel<true><<<(unsigned)rows, 256, 0, stream>>>(src, layers, tokens, kv, page_table,
                                                                 pages_per_layer,
                                                                 reinterpret_cast<__nv_bfloat16*>(pool),
                                                                 page_tokens);
  else
    store_pages_kernel<false><<<(unsigned)rows, 256, 0, stream>>>(src, layers, tokens, kv, page_table,
                                                                  pages_per_layer,
                                                                  reinterpret_cast<__nv_bfloat16*>(pool),
                                                                  page_tokens);
  return (int)cudaGetLastError();
}

int vlc_gather_rows_impl(void* dst, const int* dst_rows, const void* src, const int* src_rows, int n, int row_bytes,
                         cudaStream_t stream) {
  if (n <= 0) return 0;
  const int blocks = n < 148 * 16 ? n : 148 * 16;
  gather_rows_kernel<<<blocks, 256, 0, stream>>>(reinterpret_cast<uint4*>(dst), dst_rows,
                                                 reinterpret_cast<const uint4*>(src), src_rows, n, row_bytes / 16);
  return (int)cudaGetLastError();
}

int vlc_patchify_impl(const float* pixels, int side, int patch, void* out, int row0, int pk_rows, int pk_kb,
                      cudaStream_t stream) {
  const int T = (side / patch) * (side / patch);
  patchify_kernel<<<T, 64, 0, stream>>>(pixels, side, patch, reinterpret_cast<__nv_bfloat16*>(out), row0, pk_rows,
                                        pk_kb);
  return (int)cudaGetLastError();
}

}  // extern "C"
