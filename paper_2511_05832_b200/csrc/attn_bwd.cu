// K7-K9: block-sparse attention backward (placeholder until the tcgen05 kernel lands).
#include "common.cuh"

extern "C" size_t hla_attn_bwd_workspace(int32_t batch, int32_t heads, int32_t n, int32_t head_dim) {
  return (size_t)batch * heads * n * head_dim * 4 + (size_t)batch * heads * n * 4 + 256;
}

extern "C" hla_status hla_attn_bwd(const hla_pattern_desc*, const hla_block_mask*, int32_t, int32_t, int32_t, float,
                                   const void*, const void*, const void*, const void*, const float*, const void*,
                                   void*, void*, void*, void*, size_t, int64_t*, cudaStream_t) {
  hla::set_error("backward not built yet");
  return HLA_ERR_UNSUPPORTED;
}
