// mmk_attention.cu — C-ABI entry of K5 (non-causal variable-length multi-head self-attention).
//
// Replaces the attention share of the modelled `encode_latency` (reference
// pkg/src/lmmsim/profiles.py:136-145).  Images never attend to each other, so
// every image is an independent sequence.  The kernel is the tcgen05/TMEM flash attention in
// mmk_attention_tc.cu.  (The first version of this file held a register-tiled mma.sync
// flash attention; on B200 it reached 255-292 TF/s on the Mllama shapes versus 690-850 TF/s
// for the tcgen05 kernel — profiles/r01_attention.md — and was removed.)
#include "sm100_common.cuh"
#include "mmk_internal.h"

namespace mmk {
template <int HD>
int launch_attn_tc(const void* qkv, void* out, const int32_t* cu, int n_seq, int max_s, int heads, float scale,
                   int64_t total_rows, void* workspace, cudaStream_t stream);
}

using namespace mmk;

extern "C" int64_t mmk_attention_workspace_size(void) { return 16; }

extern "C" int mmk_attention_varlen_bf16(const void* qkv, void* out, const int32_t* cu_seqlens, int32_t n_seq,
                                         int32_t max_seqlen, int32_t total_tokens, int32_t heads, int32_t head_dim,
                                         float scale, void* workspace, cudaStream_t stream) {
  if (n_seq < 0 || heads <= 0 || max_seqlen < 0 || total_tokens < 0)
    return set_error(MMK_ERR_ARG, "attention: bad shape");
  if (head_dim != 64 && head_dim != 80 && head_dim != 128)
    return set_error(MMK_ERR_UNSUPPORTED, "attention: head_dim %d not in {64, 80, 128}", head_dim);
  if (n_seq == 0 || max_seqlen == 0 || total_tokens == 0) return MMK_OK;
  if (workspace == nullptr) return set_error(MMK_ERR_ARG, "attention: workspace is NULL");
  if (head_dim == 64)
    return launch_attn_tc<64>(qkv, out, cu_seqlens, n_seq, max_seqlen, heads, scale, total_tokens, workspace, stream);
  if (head_dim == 128)
    return launch_attn_tc<128>(qkv, out, cu_seqlens, n_seq, max_seqlen, heads, scale, total_tokens, workspace, stream);
  return launch_attn_tc<80>(qkv, out, cu_seqlens, n_seq, max_seqlen, heads, scale, total_tokens, workspace, stream);
}
