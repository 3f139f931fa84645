// Internal declarations shared by the VLCache sm_100a kernels and the C-ABI layer.
#pragma once
#include <cstddef>
#include <cstdint>
#include <utility>

#include "../../include/vlcache.h"
#include "vlc_ptx.cuh"

namespace vlc {

enum EpiKind {
  EPI_F32 = VLC_EPI_F32,
  EPI_RESID = VLC_EPI_RESID,
  EPI_BF16 = VLC_EPI_BF16,
  EPI_BIAS_ADD = VLC_EPI_BIAS_ADD,
  EPI_SWIGLU = VLC_EPI_SWIGLU,
  EPI_QKV_PLAIN = VLC_EPI_QKV_PLAIN,
  EPI_QKV_ROPE = VLC_EPI_QKV_ROPE,
};

using GemmEpi = vlc_epilogue;

extern int g_stage_override;  // experiment knob (vlc_set_tuning key 1)
extern int g_coop;            // key 2: cooperative launch of the stream-K GEMM
extern int g_pair;            // key 10: CTA-pair GEMM threshold on the token tile (0 = off)
extern int g_unsplit_min;     // key 9: tiles >= this (and <= #SMs) -> one CTA per tile
extern int g_wide;            // key 7: 256-row GEMM tiles (0 auto, 1 never, 2 always)
extern int g_aligned_split;   // key 17: tile-aligned split-K for the multi-CTA-per-tile schedule
extern int g_decoupled;       // key 18: decoupled weight / activation rings in the one-tile GEMM schedule
extern int g_dec_min_tile;    // key 20: smallest token tile using the decoupled rings
extern int g_pdl;             // key 6: programmatic dependent launch of the chain kernels (default 1)
void set_debug_buffer(unsigned long long* p);
unsigned long long* debug_buffer();

// Launch with programmatic stream serialization (g_pdl) and optionally cooperative residency
// (only when PDL is off: the kernels that rely on co-residency size their grids to <= #SMs).
template <typename... KArgs, typename... Args>
cudaError_t launch_chain(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                         bool coop, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  int n = 0;
  if (g_pdl) {
    at[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  } else if (coop) {
    at[n].id = cudaLaunchAttributeCooperative;
    at[n].val.cooperative = 1;
    ++n;
  }
  cfg.attrs = at;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}


// tensor maps (driver entry point resolved through the runtime, no -lcuda)
cudaError_t make_tmap_2d(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer,
                         uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer,
                         int swizzle_bytes);
cudaError_t make_tmap_3d(CUtensorMap* map, const void* base, uint64_t d0, uint64_t d1, uint64_t d2,
                         uint64_t stride1_bytes, uint64_t stride2_bytes, uint32_t b0, uint32_t b1,
                         uint32_t b2, int swizzle_bytes);

cudaError_t make_tmap_4d(CUtensorMap* map, const void* base, const uint64_t* dims, const uint64_t* strides_bytes,
                         const uint32_t* box, int swizzle_bytes);

struct RelocArgs;   // vlc_reloc.cuh
cudaError_t launch_relocate(const RelocArgs& r, cudaStream_t stream);
cudaError_t launch_gemm(const void* W, int n_pad, int k_pad, const void* X, int x_rows_cap,
                        int m_tokens, const GemmEpi& epi, int max_ctas, float* ws, size_t ws_bytes,
                        int* counters, cudaStream_t stream);
int gemm_row_tile(int n_pad, int m_tokens);
cudaError_t launch_gemm_pair(const void* W, int n_pad, int k_pad, const void* X, int x_rows_cap, int m_tokens,
                             const GemmEpi& epi, int max_pairs, float* ws, size_t ws_bytes, int* counters,
                             cudaStream_t stream);
cudaError_t launch_pack(const void* src, int rows, int cols, int ld, void* dst, int R, int KB, cudaStream_t s);

cudaError_t launch_attention_paged(const vlc_attn_paged_args& a, cudaStream_t stream);

}  // namespace vlc
