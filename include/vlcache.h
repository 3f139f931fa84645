/*
 * vlcache.h -- C ABI of the B200 (sm_100a) VLCache cache-reuse prefill kernels.
 *
 * The reference (`kvreuse` 0.1.0, /root/reference/pkg/src/kvreuse) is a pure
 * Python/NumPy package with no FFI: its plugin boundary is the Python API
 * (`prefill_with_reuse`, `CacheStore`, `plan_greedy`, ...; __init__.py:3-16).
 * The drop-in keeps that Python API (package `paper_2512_12977_b200`) and moves
 * every NumPy op of the hot path behind this C ABI; each entry point names the
 * reference lines it replaces.  The Python binding is ctypes
 * (paper_2512_12977_b200/_native.py); see INTEGRATION.md.
 *
 * Conventions: every function returns 0 (VLC_OK) or a VLC_ERR_* status and never
 * throws; vlc_last_error() gives a thread-local message.  All tensor arguments
 * are caller-owned DEVICE pointers; nothing synchronises the host; every call is
 * stream-ordered on `stream` and re-entrant across streams.  Dtypes: "bf16" =
 * IEEE bfloat16 stored as uint16, "f32" = float.
 */
#ifndef VLCACHE_H
#define VLCACHE_H

#include <stddef.h>
#include <stdint.h>
#include <cuda_runtime.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VLC_OK 0
#define VLC_ERR_INVALID 1     /* bad argument (maps to InputError)           */
#define VLC_ERR_UNSUPPORTED 2 /* shape the kernels do not handle             */
#define VLC_ERR_CUDA 3        /* CUDA runtime / driver failure               */

/* PACKED OPERAND LAYOUT (inputs of vlc_gemm_bf16).  A bf16 matrix [rows][K] is stored as
 * row tiles of R rows x 128-wide K blocks; block (rt, kb) is contiguous: two 64-column atoms,
 * each R rows x 128 B, and inside an atom the 16-byte chunk c of row r sits at chunk c^(r&7)
 * (the SWIZZLE_128B image UMMA expects).  Element (row, k), KB = ceil(K/128):
 *   ((((rt*KB + kb)*2 + atom)*R + r)*64 + ((c ^ (r&7)) << 3) + e),
 *   rt = row/R, r = row%R, kb = k>>7, atom = (k>>6)&1, c = (k>>3)&7, e = k&7.
 * Weights use R = 128; activations use R = vlc_gemm_row_tile(n_pad, m_tokens) of the consuming GEMM.
 * One (rt, kb) block is one cp.async.bulk copy, which is what lets a CTA stream at HBM speed. */
/* <= 256 tokens per row tile, except a one-wave GEMM (n_pad / 128 <= #SMs) keeps 257..512 tokens in one
 * wide tile (two UMMA N chunks into one TMEM accumulator). */
int vlc_gemm_row_tile(int n_pad, int m_tokens);
/* Row-major bf16 [rows][cols] (leading dimension ld) -> packed (R, KB); padding is untouched. */
int vlc_pack_operand(const void* src, int rows, int cols, int ld, void* dst, int R, int KB,
                     cudaStream_t stream);

/* GEMM epilogue kinds (vlc_gemm_bf16). */
#define VLC_EPI_F32 0       /* out[map1?map1[j]:j][f] = acc            (engine.py:187 logits)   */
#define VLC_EPI_RESID 1     /* out[j][f] += acc, fp32 residual          (engine.py:183, 185)     */
#define VLC_EPI_BF16 2      /* out[j][f] = bf16(acc)                                              */
#define VLC_EPI_BIAS_ADD 3  /* out[j][f] = acc + bias[f] + add[j][f]    (model.py:316)           */
#define VLC_EPI_SWIGLU 4    /* rows interleaved gate/up: out[j][f/2] = silu(g)*u (model.py:262)  */
#define VLC_EPI_QKV_PLAIN 5 /* q/k/v sections -> out/out2/out3          (model.py:318)           */
#define VLC_EPI_QKV_ROPE 6  /* q rot -> out[map1[j]], k -> out4[j] (pre-RoPE) and rot -> out2
                               [map2[j]], v -> out3[map2[j]]            (engine.py:176-180);
                               head_dim % 8 == 0, else VLC_ERR_UNSUPPORTED                         */

typedef struct vlc_epilogue {
  int kind;
  int n_valid;   /* valid weight rows (output features)            */
  int m_tokens;  /* valid token rows                                */
  void* out;  int ldo;
  void* out2; int ld2;
  void* out3; int ld3;
  void* out4; int ld4;
  const int* map1;   /* token -> destination row of `out` (NULL = identity) */
  const int* map2;   /* token -> KV-cache row                                 */
  const int* pos;    /* token -> absolute position in its request           */
  const float* cos_tab; /* [positions][tab_ld] f32 RoPE tables (model.py:129-134) */
  const float* sin_tab;
  int tab_ld;
  int hd;            /* head_dim                                             */
  int seg;           /* features per q / k / v section (= kv_dim)            */
  const float* bias;
  const float* add;  int ld_add;
  int pk_rows;       /* > 0: BF16 / SWIGLU output written PACKED (row tile pk_rows, pk_kb blocks) */
  int pk_kb;
  /* RESID: split-K partials reduced in a fixed order through `ws` (bitwise reproducible runs)
   * instead of red.add in arrival order (faster).  0 = red.add.                               */
  int deterministic;
  /* QKV_ROPE, optional: the RoPE tables interleaved, rows of head_dim floats (cos t, cos t+1, sin t,
   * sin t+1 for even t) -- one 16-byte load per token instead of two (NULL: cos_tab / sin_tab). */
  const float* cs_tab;
} vlc_epilogue;

/* Paged attention (vlc_attn_paged; model.py:274-291, engine.py:179-182): the recomputed queries of
 * one layer over all keys of their request.  The keys are a list of 64-key CHUNKS (contiguous
 * positions) per (request, layer): chunks int32[n][4] = {pos0, len <= 64 | D << 8, a, b}
 *   b <  0: request rows a .. a+63 of kc / vc (K already rotated: text / recomputed tokens);
 *   b >= 0: store rows page_table[a] * page_rows + b .. +63 of pool_k / pool_v (cached image tokens,
 *           K rotated at the position it was cached at, pos - D): the kernel multiplies them against its
 *           queries rotated by -D (fp32 tables, row |D|), since q . R(D) k_cached = (R(-D) q) . k_cached.
 * A 128-key tile = two consecutive chunks (lists padded to an even length with len = 0 chunks); its
 * store chunks share one D.
 * items int32[n][8] = {q_row0, n_q <= 128, head, chunk0, tile_begin, tile_end, group,
 * (part << 8) | nsplit}: queries q_row0 .. (position-sorted, positions qpos, output rows rowof)
 * over tiles [tile_begin, tile_end) of the chunk list starting at chunk0.  group < 0 writes
 * normalised rows; otherwise the nsplit CTAs of a group merge their fp32 partials (ws_o >= groups*8*256*hd
 * floats, ws_ml >= groups*8*256*2) in-kernel -- every CTA must be co-resident (n_items <= #SMs),
 * counters >= 2*ws_slots ints, zero, left zero. */
typedef struct vlc_attn_paged_args {
  const void* q; int q_rows_cap;                 /* bf16 [q_rows_cap][kv] rotated queries        */
  const void* kc; const void* vc;                /* bf16 [layers][kv_rows_cap][kv] request K / V */
  int layers_cap; int kv_rows_cap; int layer;
  const void* pool_k; const void* pool_v;        /* bf16 [pool_rows][kv] store pages (or NULL)   */
  int pool_rows; const int* page_table; int page_rows;
  const float* cos_tab; const float* sin_tab; int tab_ld;   /* fp32 [pos][head_dim/2]           */
  int kv; int heads; int head_dim;
  const int* chunks;
  const int* items; int n_items;
  const int* qpos;                               /* [q] position within request                  */
  const int* rowof;                              /* [q] output row                               */
  void* out; int ldo;                            /* bf16 [rows][ldo], PACKED when pk_rows > 0    */
  int pk_rows; int pk_kb;
  float* ws_o; float* ws_ml; int ws_slots;
  int* counters;
  float scale_log2;                              /* log2(e) / sqrt(head_dim)                     */
  unsigned long long* trace;                     /* NULL, or [n_items][64] globaltimer stamps    */
} vlc_attn_paged_args;

const char* vlc_last_error(void);
int vlc_version(void);
/* Asynchronous host -> device copy on `stream` (the per-call metadata upload of the host runtime:
 * a direct cudaMemcpyAsync without a framework dispatch).  host should be pinned.            */
int vlc_copy_h2d_async(void* device_dst, const void* host_src, size_t bytes, cudaStream_t stream);

/* Schedule overrides for experiments and tests ONLY (process-global, not re-entrant; nothing in
   the drop-in calls it): key 1 = GEMM pipeline stages (0 = automatic); other keys see vlc_capi.cu. */
int vlc_set_tuning(int key, int value);
int vlc_set_debug_buffer(void* device_ptr);

/* Layer-0 hidden rows of the computed set (model.py:339-359, engine.py:167).
 * src int32[rows][2] = {kind, index}: kind 0 -> bf16 embed row `index` (text token id),
 * kind 1 -> fp32 row `index` of enc_a (encoder-cache pool), kind 2 -> row of enc_b
 * (freshly encoded images of a cache miss). */
int vlc_embed_assemble(float* x, int ldx, const void* embed_bf16, int d, const float* enc_a,
                       const float* enc_b, const int* src, int rows, cudaStream_t stream);


/* RMSNorm eps (model.py:257-259) of rows (optionally gathered via row_map) -> bf16 or f32;
 * bf16 output is PACKED when pk_rows > 0 (then ldo is ignored). */
int vlc_rmsnorm(const float* x, int ldx, const float* gamma, void* out, int ldo, int out_f32,
                int rows, int d, const int* row_map, float eps, int pk_rows, int pk_kb,
                cudaStream_t stream);

/* Head-parallel attention: x[r] += add[r] (the all-reduced O projection),
 * written back, then RMSNorm of x[r] -> bf16 (PACKED when pk_rows > 0).  Replaces the residual add
 * of engine.py:183 + the MLP norm of engine.py:184 on each rank. */
int vlc_add_rmsnorm(float* x, int ldx, const float* add, int ld_add, const float* gamma, void* out, int ldo,
                    int rows, int d, float eps, int pk_rows, int pk_kb, cudaStream_t stream);

/* Fused gather + RoPE re-rotation + scatter of cached pre-RoPE K and copy of V from
 * the paged store into the request KV cache (engine.py:153-155 + engine.py:180).
 * descs int32[n][8] = {layer, page_tab_off, tok0, ntok, dst_row0, pos0, 0, 0};
 * blocks int32[n_blocks][2] = {desc, token offset}; kc/vc bf16 [layers][kv_rows_cap][kv].
 * vpool / vc NULL: K only (the store builds its rotated-at-origin K pages with it). */
int vlc_kv_relocate(const void* kpool, const void* vpool, int page_tokens, const int* page_table,
                    int kv, int head_dim, void* kc, void* vc, int kv_rows_cap, const int* descs,
                    const int* blocks, int n_blocks, const float* cos_tab, const float* sin_tab,
                    int tab_ld, cudaStream_t stream);

/* Row gather: dst row dst_rows[r] = src row src_rows[r] for r < n (rows of row_bytes bytes, a multiple
 * of 16; 16-byte aligned buffers).  Assembles ReuseResult.kv, the merged pre-RoPE K / V [L, n, kv] of
 * a request (engine.py:153-155, 177-178), from the QKV epilogue's computed rows and the store pages. */
int vlc_gather_rows(void* dst, const int* dst_rows, const void* src, const int* src_rows, int n, int row_bytes,
                    cudaStream_t stream);

/* Store write (store.py:140-147 put_kv): src [layers][T][kv] (f32 or bf16) -> bf16 pages. */
int vlc_store_write_pages(const void* src, int src_f32, int layers, int tokens, int kv,
                          const int* page_table, int pages_per_layer, void* pool,
                          int page_tokens, cudaStream_t stream);

/* Fused-epilogue tcgen05 GEMM: acc[f][j] = sum_k W[f][k] X[j][k]; W PACKED (R = 128) with
 * n_pad rows, X PACKED with R = vlc_gemm_row_tile(n_pad, m_tokens) and >= ceil(m/R)*R rows (x_rows_cap),
 * both with K = k_pad (% 128 == 0).  n_pad % 128 == 0.
 * Stream-K schedule over (128-row weight tile x token tile x 64-wide k-block) units on
 * max_ctas co-resident CTAs (0 = one per SM); tiles shared by several CTAs are reduced in
 * parallel through `ws` (>= ctas*8*128*256 floats) with `counters` (>= 2*ctas ints, zeroed
 * once; the kernel leaves them zeroed).  Token tiles >= 32 run the CTA-pair (cta_group::2)
 * stream-K schedule over 256-row tiles x 128-wide k-blocks on every SM pair: its split tiles
 * exchange fp32 partials through ws (2 * 74 * 128 * 256 floats) and per-tile flags in
 * counters[12288 .. 12288 + 2 * tiles) -- pass counters of >= 16384 ints (<= 2048 tiles; else
 * whole-tile pairs only).  Replaces engine.py:176-178, 183-185, 187. */
int vlc_gemm_bf16(const void* w, int n_pad, int k_pad, const void* x, int x_rows_cap,
                  int m_tokens, const vlc_epilogue* epi, int max_ctas, float* ws, size_t ws_bytes,
                  int* counters, cudaStream_t stream);

int vlc_attn_paged(const vlc_attn_paged_args* args, cudaStream_t stream);

/* Patchify (model.py:312-314): pixels f32 [side][side] -> bf16 patches, PACKED with row tile
 * pk_rows (patch rows start at row `row0`), K = patch^2 (kb blocks pk_kb). */
int vlc_patchify(const float* pixels, int side, int patch, void* out, int row0, int pk_rows,
                 int pk_kb, cudaStream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* VLCACHE_H */
