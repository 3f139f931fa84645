// extern "C" surface of libvlcache.so (see include/vlcache.h): argument checks,
// status codes, thread-local error text and TMA descriptor construction.
#include <cstdio>
#include <cstring>
#include <mutex>

#include "vlc_internal.h"
#include "vlc_reloc.cuh"

namespace vlc {

static thread_local char g_err[512] = "";

static int fail(int code, const char* msg) {
  std::snprintf(g_err, sizeof(g_err), "%s", msg);
  return code;
}
static int cuda_status(cudaError_t e, const char* where) {
  if (e == cudaSuccess) return VLC_OK;
  std::snprintf(g_err, sizeof(g_err), "%s: %s", where, cudaGetErrorString(e));
  return VLC_ERR_CUDA;
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                  CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                  CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

static CUtensorMapSwizzle swz(int bytes) {
  return bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
         : bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
         : bytes == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                       : CU_TENSOR_MAP_SWIZZLE_NONE;
}

cudaError_t make_tmap_2d(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer,
                         uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer,
                         int swizzle_bytes) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return cudaErrorNotSupported;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {row_stride_bytes};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, swz(swizzle_bytes), CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

cudaError_t make_tmap_3d(CUtensorMap* map, const void* base, uint64_t d0, uint64_t d1, uint64_t d2,
                         uint64_t stride1_bytes, uint64_t stride2_bytes, uint32_t b0, uint32_t b1,
                         uint32_t b2, int swizzle_bytes) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return cudaErrorNotSupported;
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {stride1_bytes, stride2_bytes};
  cuuint32_t box[3] = {b0, b1, b2};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, swz(swizzle_bytes), CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

cudaError_t make_tmap_4d(CUtensorMap* map, const void* base, const uint64_t* dims, const uint64_t* strides_bytes,
                         const uint32_t* box, int swizzle_bytes) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return cudaErrorNotSupported;
  cuuint64_t d[4] = {dims[0], dims[1], dims[2], dims[3]};
  cuuint64_t st[3] = {strides_bytes[0], strides_bytes[1], strides_bytes[2]};
  cuuint32_t b[4] = {box[0], box[1], box[2], box[3]};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), d, st, b, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, swz(swizzle_bytes), CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

}  // namespace vlc

using namespace vlc;

extern "C" {

int vlc_embed_assemble_impl(float*, int, const void*, int, const float*, const float*, const int*, int, cudaStream_t);
int vlc_rmsnorm_impl(float*, int, const float*, void*, int, int, int, int, const int*, float, int, int,
                     cudaStream_t, const float*, int);
int vlc_kv_relocate_impl(const void*, const void*, int, const int*, int, int, void*, void*, int, const int*,
                         const int*, int, const float*, const float*, int, cudaStream_t);
int vlc_store_write_pages_impl(const void*, int, int, int, int, const int*, int, void*, int, cudaStream_t);
int vlc_patchify_impl(const float*, int, int, void*, int, int, int, cudaStream_t);
int vlc_gather_rows_impl(void*, const int*, const void*, const int*, int, int, cudaStream_t);

const char* vlc_last_error(void) { return g_err; }

int vlc_copy_h2d_async(void* device_dst, const void* host_src, size_t bytes, cudaStream_t stream) {
  if (bytes == 0) return VLC_OK;
  if (!device_dst || !host_src) return fail(VLC_ERR_INVALID, "copy_h2d: null pointer");
  return cuda_status(cudaMemcpyAsync(device_dst, host_src, bytes, cudaMemcpyHostToDevice, stream), "copy_h2d");
}

// Process-wide schedule / variant switches (experiments and tests; defaults = measured best,
// INTEGRATION.md lists them).
int vlc_set_tuning(int key, int value) {
  switch (key) {
    case 1: vlc::g_stage_override = value; return VLC_OK;        // GEMM pipeline stages (0 = auto)
    case 2: vlc::g_coop = value; return VLC_OK;                  // cooperative launch when PDL is off
    case 6: vlc::g_pdl = value; return VLC_OK;                   // programmatic dependent launch
    case 7: vlc::g_wide = value; return VLC_OK;                  // 256-row GEMM tiles
    case 9: vlc::g_unsplit_min = value; return VLC_OK;           // one-CTA-per-tile threshold
    case 10: vlc::g_pair = value; return VLC_OK;                 // CTA-pair GEMM threshold
    case 17: vlc::g_aligned_split = value; return VLC_OK;        // tile-aligned split-K
    case 18: vlc::g_decoupled = value; return VLC_OK;            // decoupled weight / activation rings
    case 20: vlc::g_dec_min_tile = value; return VLC_OK;         // smallest token tile using key 18
    default: return fail(VLC_ERR_INVALID, "set_tuning: unknown key");
  }
}
/* Experiments only: device buffer receiving per-CTA phase timestamps of the GEMM (NULL = off). */
int vlc_set_debug_buffer(void* p) {
  vlc::set_debug_buffer(reinterpret_cast<unsigned long long*>(p));
  return VLC_OK;
}
int vlc_version(void) { return 100; }

int vlc_embed_assemble(float* x, int ldx, const void* embed_bf16, int d, const float* enc_a, const float* enc_b,
                       const int* src, int rows, cudaStream_t stream) {
  if (rows < 0 || d <= 0 || ldx < d || !x || !src) return fail(VLC_ERR_INVALID, "embed_assemble: bad args");
  return cuda_status((cudaError_t)vlc_embed_assemble_impl(x, ldx, embed_bf16, d, enc_a, enc_b, src, rows, stream),
                     "embed_assemble");
}

int vlc_rmsnorm(const float* x, int ldx, const float* gamma, void* out, int ldo, int out_f32, int rows, int d,
                const int* row_map, float eps, int pk_rows, int pk_kb, cudaStream_t stream) {
  if (rows < 0 || d <= 0 || ldx < d || (pk_rows <= 0 && ldo < d) || !x || !gamma || !out)
    return fail(VLC_ERR_INVALID, "rmsnorm: bad args");
  if (pk_rows > 0 && (out_f32 || pk_rows % 8 || pk_kb * 128 < d))
    return fail(VLC_ERR_INVALID, "rmsnorm: packed output needs bf16, pk_rows % 8 == 0, pk_kb*128 >= d");
  return cuda_status((cudaError_t)vlc_rmsnorm_impl(const_cast<float*>(x), ldx, gamma, out, ldo, out_f32, rows, d,
                                                   row_map, eps, pk_rows, pk_kb, stream, nullptr, 0),
                     "rmsnorm");
}

int vlc_add_rmsnorm(float* x, int ldx, const float* add, int ld_add, const float* gamma, void* out, int ldo,
                    int rows, int d, float eps, int pk_rows, int pk_kb, cudaStream_t stream) {
  if (rows < 0 || d <= 0 || ldx < d || ld_add < d || (pk_rows <= 0 && ldo < d) || !x || !add || !gamma || !out)
    return fail(VLC_ERR_INVALID, "add_rmsnorm: bad args");
  if (pk_rows > 0 && (pk_rows % 8 || pk_kb * 128 < d))
    return fail(VLC_ERR_INVALID, "add_rmsnorm: packed output needs pk_rows % 8 == 0, pk_kb*128 >= d");
  return cuda_status((cudaError_t)vlc_rmsnorm_impl(x, ldx, gamma, out, ldo, 0, rows, d, nullptr, eps, pk_rows, pk_kb,
                                                   stream, add, ld_add),
                     "add_rmsnorm");
}

int vlc_kv_relocate(const void* kpool, const void* vpool, int page_tokens, const int* page_table, int kv,
                    int head_dim, void* kc, void* vc, int kv_rows_cap, const int* descs, const int* blocks,
                    int n_blocks, const float* cos_tab, const float* sin_tab, int tab_ld, cudaStream_t stream) {
  if (n_blocks < 0 || page_tokens <= 0 || head_dim < 16 || head_dim % 16 || kv % head_dim || kv_rows_cap <= 0)
    return fail(VLC_ERR_UNSUPPORTED, "kv_relocate: head_dim must be a multiple of 16 dividing kv");
  if (tab_ld != head_dim / 2) return fail(VLC_ERR_INVALID, "kv_relocate: tab_ld must be head_dim/2");
  if (n_blocks > 0 && (!kpool || !kc || !page_table || !descs || !blocks || !cos_tab || !sin_tab ||
                       (vc != nullptr && vpool == nullptr)))
    return fail(VLC_ERR_INVALID, "kv_relocate: null pointer");
  return cuda_status((cudaError_t)vlc_kv_relocate_impl(kpool, vpool, page_tokens, page_table, kv, head_dim, kc, vc,
                                                       kv_rows_cap, descs, blocks, n_blocks, cos_tab, sin_tab,
                                                       tab_ld, stream),
                     "kv_relocate");
}

int vlc_store_write_pages(const void* src, int src_f32, int layers, int tokens, int kv, const int* page_table,
                          int pages_per_layer, void* pool, int page_tokens, cudaStream_t stream) {
  if (!src || !pool || !page_table || layers <= 0 || tokens <= 0 || kv <= 0 || page_tokens <= 0)
    return fail(VLC_ERR_INVALID, "store_write_pages: bad args");
  return cuda_status((cudaError_t)vlc_store_write_pages_impl(src, src_f32, layers, tokens, kv, page_table,
                                                             pages_per_layer, pool, page_tokens, stream),
                     "store_write_pages");
}

int vlc_gemm_row_tile(int n_pad, int m_tokens) { return gemm_row_tile(n_pad, m_tokens); }

int vlc_pack_operand(const void* src, int rows, int cols, int ld, void* dst, int R, int KB, cudaStream_t stream) {
  if (!src || !dst || rows < 0 || cols <= 0 || ld < cols || R <= 0 || R % 8 || KB * 128 < cols)
    return fail(VLC_ERR_INVALID, "pack_operand: bad args");
  return cuda_status(launch_pack(src, rows, cols, ld, dst, R, KB, stream), "pack_operand");
}

int vlc_gemm_bf16(const void* w, int n_pad, int k_pad, const void* x, int x_rows_cap, int m_tokens,
                  const vlc_epilogue* epi, int max_ctas, float* ws, size_t ws_bytes, int* counters,
                  cudaStream_t stream) {
  if (!w || !x || !epi) return fail(VLC_ERR_INVALID, "gemm: null pointer");
  if (n_pad % 128 || k_pad % 128 || n_pad <= 0 || k_pad <= 0)
    return fail(VLC_ERR_UNSUPPORTED, "gemm: n_pad and k_pad must be multiples of 128");
  const int rt = gemm_row_tile(n_pad, m_tokens);
  if (m_tokens > 0 && x_rows_cap < (m_tokens + rt - 1) / rt * rt)
    return fail(VLC_ERR_INVALID, "gemm: x_rows_cap must cover whole row tiles of the packed activations");
  if ((epi->kind == VLC_EPI_BF16 || epi->kind == VLC_EPI_SWIGLU) && epi->pk_rows > 0 && epi->pk_rows % 8)
    return fail(VLC_ERR_INVALID, "gemm: packed epilogue output needs pk_rows % 8 == 0");
  if (epi->m_tokens != m_tokens) return fail(VLC_ERR_INVALID, "gemm: epilogue m_tokens mismatch");
  if (epi->kind == VLC_EPI_QKV_ROPE && (!epi->map2 || !epi->pos || !epi->cos_tab || epi->hd % 2))
    return fail(VLC_ERR_INVALID, "gemm: QKV_ROPE needs map2/pos/tables");
  if (epi->kind == VLC_EPI_QKV_ROPE && epi->hd % 8)   // the epilogue rotates 4 pairs per lane
    return fail(VLC_ERR_UNSUPPORTED, "gemm: QKV_ROPE needs head_dim % 8 == 0");
  return cuda_status(launch_gemm(w, n_pad, k_pad, x, x_rows_cap, m_tokens, *epi, max_ctas, ws, ws_bytes, counters,
                                 stream),
                     "gemm_bf16");
}

int vlc_attn_paged(const vlc_attn_paged_args* a, cudaStream_t stream) {
  if (!a || !a->q || !a->kc || !a->vc || !a->items || !a->chunks || !a->qpos || !a->rowof || !a->out)
    return fail(VLC_ERR_INVALID, "attn_paged: null pointer");
  if (a->head_dim != 16 && a->head_dim != 32 && a->head_dim != 64 && a->head_dim != 128)
    return fail(VLC_ERR_UNSUPPORTED, "attn_paged: head_dim must be 16/32/64/128");
  if (a->kv != a->heads * a->head_dim) return fail(VLC_ERR_INVALID, "attn_paged: kv != heads*head_dim");
  if (a->pool_k && (!a->pool_v || !a->page_table || a->page_rows <= 0 || !a->cos_tab || !a->sin_tab ||
                    a->tab_ld != a->head_dim / 2))
    return fail(VLC_ERR_INVALID, "attn_paged: store chunks need pools, page table and RoPE tables");
  // split groups merge in-kernel: every CTA of the launch must be resident at once
  if (a->ws_slots > 0 && (!a->counters || !a->ws_o || !a->ws_ml || a->n_items > 148))
    return fail(VLC_ERR_INVALID, "attn_paged: split groups need counters / workspaces and <= 148 items");
  return cuda_status(launch_attention_paged(*a, stream), "attn_paged");
}

int vlc_gather_rows(void* dst, const int* dst_rows, const void* src, const int* src_rows, int n, int row_bytes,
                    cudaStream_t stream) {
  if (n < 0 || (n > 0 && (!dst || !dst_rows || !src || !src_rows)) || row_bytes <= 0 || row_bytes % 16 ||
      (reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) % 16)
    return fail(VLC_ERR_INVALID, "gather_rows: bad args");
  return cuda_status((cudaError_t)vlc_gather_rows_impl(dst, dst_rows, src, src_rows, n, row_bytes, stream),
                     "gather_rows");
}

int vlc_patchify(const float* pixels, int side, int patch, void* out, int row0, int pk_rows, int pk_kb,
                 cudaStream_t stream) {
  if (!pixels || !out || patch <= 0 || side % patch || pk_rows <= 0 || pk_rows % 8 || pk_kb * 128 < patch * patch)
    return fail(VLC_ERR_INVALID, "patchify: bad args");
  return cuda_status((cudaError_t)vlc_patchify_impl(pixels, side, patch, out, row0, pk_rows, pk_kb, stream),
                     "patchify");
}

}  // extern "C"
