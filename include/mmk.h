/*
 * mmk.h — C ABI of the B200 (sm_100a) image path: preprocess -> encode -> pack/handoff.
 *
 * This is the drop-in boundary for the image path of a ModServe-style server.  The
 * reference (arXiv 2502.00937, `lmmsim`, mounted read-only at /root/reference) models that
 * path with three stand-ins that the functions below replace with real execution:
 *
 *   reference symbol (file:line)                                   replaced by
 *   ------------------------------------------------------------   -----------------------------
 *   core.tile_count / image_tokens      core.py:58-74              mmk_tile_plan   (K0, bit-exact)
 *   Request.total_image_tokens/tiles    core.py:110-120            mmk_tile_plan   (int64 offsets)
 *   LatencyProfile.preprocess_latency   profiles.py:128-134        mmk_preprocess  (K1)
 *   LatencyProfile.encode_latency       profiles.py:136-145        mmk_gemm_bf16(_ln) / mmk_layernorm
 *                                                                  / mmk_attention_varlen_bf16 /
 *                                                                  mmk_embed_* (K2-K8)
 *   shard join + handoff                engine.py:730-752, :563-579 mmk_pack_mllama_peer (K9+K10 fused:
 *                                                                  pack straight into the LLM GPU's
 *                                                                  memory over NVLink) or mmk_pack_*
 *                                                                  + NCCL P2P (host side)
 *
 * Conventions (all functions):
 *   - return int status: MMK_OK, MMK_ERR_ARG (-> SpecError), MMK_ERR_UNSUPPORTED
 *     (-> ProfileError), MMK_ERR_CUDA (-> RuntimeError); mmk_last_error() has the message.
 *   - every pointer is a DEVICE pointer unless noted; the caller owns all memory; nothing
 *     here allocates device memory or synchronises; the stream is the last argument.
 *   - stateless and re-entrant (per-thread error string), safe on distinct streams.
 */
#ifndef MMK_H_
#define MMK_H_

#include <stdint.h>
#include <cuda_runtime_api.h>

#ifdef __cplusplus
extern "C" {
#endif

enum mmk_status { MMK_OK = 0, MMK_ERR_ARG = 1, MMK_ERR_UNSUPPORTED = 2, MMK_ERR_CUDA = 3 };

/* GEMM epilogues (mmk_gemm_bf16). */
enum mmk_epilogue {
  MMK_EPI_BF16 = 0,           /* out bf16 = acc + bias                              */
  MMK_EPI_BF16_GELU = 1,      /* out bf16 = gelu_erf(acc + bias)     (Mllama FC1)   */
  MMK_EPI_BF16_QUICKGELU = 2, /* out bf16 = quick_gelu(acc + bias)   (CLIP FC1)     */
  MMK_EPI_F32 = 3,            /* out f32  = acc + bias               (patch embed)  */
  MMK_EPI_RESID_F32 = 4,      /* out f32 += gate * (acc + bias); aux bf16 = out     */
  MMK_EPI_BF16_GELU_TANH = 5  /* out bf16 = gelu_tanh(acc + bias)    (SigLIP FC1)   */
};

const char* mmk_version(void);
const char* mmk_last_error(void);

/*
 * K0 — tile plan + ragged offsets.  Replaces core.tile_count (core.py:58-69),
 * core.image_tokens (core.py:72-74) and Request.total_tiles / total_image_tokens
 * (core.py:110-120) for n images at once, and adds the pixel geometry of each image.
 *   in : w[n], h[n] (int32 pixels, >= 1), tile edge T, tokens/tile, cap, thumbnail flag
 *   out: tiles[n]; tile_off[n+1], tok_off[n+1] (int64 exclusive prefix sums);
 *        geom[n*4] = {rows, cols, resized_w, resized_h} of the tile canvas
 *        (resize_mode 0: Mllama canvas fit; 1: CLIP shortest-side resize, crop later);
 *        ar_id[n] (optional) = 1 + index of (rows, cols) in the enumeration of all (a, b) with
 *        a*b <= cap, a outer (transformers Mllama supported_aspect_ratios; 0 = no image);
 *        bad[1] (int32) = number of images with w<1 or h<1 (their tiles are 0).
 * Two launches: a thread per image (count, canvas, aspect-ratio id), then one CTA scanning the
 * counts into the int64 offsets; n <= 65536.
 */
int mmk_tile_plan(const int32_t* w, const int32_t* h, int32_t n, int32_t tile_px,
                  int32_t tokens_per_tile, int32_t max_tiles, int32_t thumbnail,
                  int32_t resize_mode, int32_t* tiles,
                  int64_t* tile_off, int64_t* tok_off, int32_t* geom, int32_t* ar_id,
                  int32_t* bad, cudaStream_t stream);

/* Per-tile (image index, slot inside the image) from tile_off[n+1]; outputs sized total_tiles. */
int mmk_tile_index(const int64_t* tile_off, int32_t n, int32_t* tile_image, int32_t* tile_slot,
                   cudaStream_t stream);

/* Attention sequence offsets of the varlen attention (one sequence per image):
 * cu_seqlens[i] = tile_off[i] * seq_per_tile for i in [0, n] (int32; seq_per_tile = patches per
 * tile + class token); tile_off NULL: cu_seqlens[i] = i * seq_per_tile (one sequence per tile, n =
 * tiles).  Total sequence rows must stay below 2^31. */
int mmk_seq_offsets(const int64_t* tile_off, int32_t n, int32_t seq_per_tile, int32_t* cu_seqlens,
                    cudaStream_t stream);

/*
 * K1 — fused uint8 HWC -> resize (bilinear, fp32) -> pad -> normalize -> tile -> patchify.
 *   src       : concatenated uint8 RGB images; src_off[n] byte offsets; src_chw = 0: HWC
 *               (interleaved, host decoders), 1: CHW planes (GPU JPEG decode output)
 *   w, h      : source dims; tile_off[n+1], geom[n*4] from mmk_tile_plan
 *   mode      : 0 = canvas fit + zero pad (Mllama), 1 = shortest-side resize + centre crop (CLIP)
 *   scale3[3], shift3[3]: normalisation out = (v * (1/255) - mean) * (1/std) as two fp32 ops:
 *               out = v * scale3[c] + shift3[c] evaluated as round(round(v*s)+b)
 *   patches   : bf16 [total_tiles * (T/p)^2, k_pad], patch vector order (c, py, px) like
 *               nn.Conv2d weight flattening; columns [3*p*p, k_pad) are zero-filled.
 */
int mmk_preprocess(const uint8_t* src, const int64_t* src_off, int32_t src_chw, const int32_t* w,
                   const int32_t* h, const int64_t* tile_off, const int32_t* geom, int32_t n,
                   int32_t total_tiles, int32_t tile_px, int32_t patch_px, int32_t k_pad,
                   int32_t mode, int32_t thumbnail, const float* scale3, const float* shift3,
                   void* patches, cudaStream_t stream);

/*
 * K2/K4/K6/K7/K8 — D[M,N] = A[M,K] . B[N,K]^T on tcgen05 tensor cores (bf16 in, fp32 acc),
 * with the fused epilogue `epilogue` (enum mmk_epilogue).  lda/ldb/ldo/ld_aux in elements.
 * bias: f32 [N] (16-byte aligned) or NULL.  gate: residual scale (RESID_F32 only).  aux: optional bf16 copy of
 * the updated residual (intermediate-layer capture for K9), RESID_F32 only.
 */
int mmk_gemm_bf16(const void* a, int64_t lda, const void* b, int64_t ldb, int32_t m, int32_t n,
                  int32_t k, int32_t epilogue, const float* bias, void* out, int64_t ldo,
                  float gate, void* aux, int64_t ld_aux, cudaStream_t stream);

/*
 * The same GEMM with a LayerNorm folded into the residual GEMM before it and the GEMM after it
 * (no separate LayerNorm pass over the residual stream):
 *   producer  (RESID_F32): ln_stats_out f32 [m][n/32][2] = (mean, M2) of each 32-column chunk of
 *             the updated residual row; `aux` receives the bf16 copy of the row.
 *   finalize  mmk_ln_stats_finalize: stats -> ln_mr f32 [m][2] = (mean, 1/sqrt(var + eps)).
 *   consumer  (bf16 epilogues): a = that bf16 copy, b = W * gamma (gamma along K), ln_c1 f32 [n] =
 *             row sums of b, bias = beta . W^T + b:  out = act(rstd * (acc - mean * c1) + bias).
 * Pointers 16-byte aligned; NULL where unused.
 */
int mmk_gemm_bf16_ln(const void* a, int64_t lda, const void* b, int64_t ldb, int32_t m, int32_t n,
                     int32_t k, int32_t epilogue, const float* bias, void* out, int64_t ldo,
                     float gate, void* aux, int64_t ld_aux, float* ln_stats_out, const float* ln_mr,
                     const float* ln_c1, cudaStream_t stream);
int mmk_ln_stats_finalize(const float* stats, int32_t rows, int32_t d, float eps, int32_t rms, float* mr,
                          cudaStream_t stream);  /* rms != 0: RMSNorm, mr = (0, 1/sqrt(mean(x^2) + eps)) */

/* InternViT QK-norm: RMSNorm (weights q_w / k_w, f32 [d]) over each row's whole query columns
 * [0, d) and key columns [d, 2d) of the bf16 [Q | K | V] matrix (row pitch ld), in place. */
int mmk_qk_rmsnorm(void* qkv, int32_t rows, int32_t d, int64_t ld, const float* q_w, const float* k_w,
                   float eps, cudaStream_t stream);

/* InternVL pixel shuffle (downsample 0.5) into the prefill layout: each tile's side x side patch grid
 * (fp32 rows, `drop` leading class tokens skipped) -> (side/2)^2 bf16 rows of 4 d columns,
 * [f(2y,2x) | f(2y,2x+1) | f(2y+1,2x) | f(2y+1,2x+1)] (transformers InternVLModel.pixel_shuffle). */
int mmk_pack_pixel_shuffle(const float* src, int32_t tiles, int32_t side, int32_t tokens_per_tile,
                           int32_t drop, int32_t d, void* out, cudaStream_t stream);

/*
 * K3 — row LayerNorm: y_bf16 = LN(x_f32) * gamma + beta (+ optional per-tile additive term);
 *   beta NULL: RMSNorm, y = x / sqrt(mean(x^2) + eps) * gamma (InternViT).
 *   x f32 [rows, d]; y bf16 [rows, d] (or f32 when y_f32 != 0, may alias x).
 *   tile_add (optional, f32 [n_tables, slots, d]) :
 *       y += tile_add[image_table[tile_image[tile]], tile_slot[tile]],  tile = row / rows_per_tile
 *   (tile_image/tile_slot int32 [n_tiles], image_table int32 [n_images]).
 */
int mmk_layernorm(const float* x, void* y, int32_t y_f32, int32_t rows, int32_t d,
                  const float* gamma, const float* beta, float eps, const float* tile_add,
                  const int32_t* tile_image, const int32_t* image_table, const int32_t* tile_slot,
                  int32_t rows_per_tile, int32_t slots, cudaStream_t stream);

/* Row LayerNorm of bf16 rows of any width (multiple of 8), bf16 out (may alias x): the InternVL
 * projector's LayerNorm(4 d) over pixel-shuffled tokens on the LLM side. */
int mmk_layernorm_bf16(const void* x, void* y, int32_t rows, int32_t d, const float* gamma, const float* beta,
                       float eps, cudaStream_t stream);

/*
 * K5 — non-causal variable-length multi-head self-attention (one sequence per image).
 *   qkv bf16 [T, 3*H*hd] = [Q | K | V] (head h at column h*hd inside each block)
 *   out bf16 [T, H*hd]; cu_seqlens int32 [n_seq+1] (device); total_tokens = T = cu_seqlens[n_seq]
 *   (host copy, bounds the TMA tensor maps); hd in {64, 80, 128}; scale = hd^-0.5 typically.
 *   workspace: device memory of mmk_attention_workspace_size() bytes, overwritten (the persistent
 *   kernel's work-item counter, reset on `stream`); not to be shared by concurrent calls.
 */
int64_t mmk_attention_workspace_size(void);
int mmk_attention_varlen_bf16(const void* qkv, void* out, const int32_t* cu_seqlens, int32_t n_seq,
                              int32_t max_seqlen, int32_t total_tokens, int32_t heads,
                              int32_t head_dim, float scale, void* workspace, cudaStream_t stream);

/*
 * Embedding assembly (feeds K3 of layer 0): patch-embed output + class token + positional
 * terms, then LayerNorm (`layernorm_pre`), written to the fp32 residual stream.
 *   patch_out f32 [total_tiles*P, d]   (P = patches per tile; token 0 of a tile is CLS)
 *   tile_image/tile_slot int32 [total_tiles], image_ar int32 [n_images] (aspect-ratio id)
 *   cls f32[d]; pos f32[P+1, d]; pos_scale: pos multiplier ((1 - tanh g) for Mllama, 1 for CLIP)
 *   tile_pos (optional) f32 [n_ar, slots, P+1, d] scaled by tile_pos_scale (tanh g)
 *   pre_tile (optional) f32 [n_ar, slots, d] added to patch tokens only, scaled by pre_scale.
 *   resid f32 [total_tiles*(P+1), d] = LN(x; gamma, beta, eps)
 */
int mmk_embed_tokens(const float* patch_out, const int32_t* tile_image, const int32_t* tile_slot,
                     const int32_t* image_ar, int32_t total_tiles, int32_t patches_per_tile,
                     int32_t d, const float* cls, const float* pos, float pos_scale,
                     const float* tile_pos, float tile_pos_scale, const float* pre_tile,
                     float pre_scale, int32_t slots, const float* gamma, const float* beta,
                     float eps, float* resid, cudaStream_t stream);

/*
 * K9 — ragged pack into the LLM-prefill buffer.
 * Mllama: out bf16 [T, d*(1+n_inter)] = [final_f32 -> bf16 | interleaved intermediates]
 *   where column d + c*n_inter + j = inter[j][t][c]  (HF torch.stack(..., dim=-1) order).
 */
int mmk_pack_mllama(const float* final_resid, const void* inter, int32_t n_inter, int32_t rows,
                    int32_t d, void* out, cudaStream_t stream);
/*
 * K9 + K10 fused: the same layout as mmk_pack_mllama, for an `out` that may live in another GPU's
 * memory (a CUDA peer / symmetric-memory mapping of the LLM-backend GPU's receive buffer —
 * replaces the pack + NCCL send of the shard handoff, engine.py:563-579 / :730-752).  Each CTA
 * assembles whole output rows in shared memory and moves each row with one bulk copy, so the
 * NVLink fabric sees contiguous full-line writes.  out: 16-byte aligned.  The writes are complete
 * when the stream reaches the end of this call (signal the receiver after it, e.g. with an event).
 */
int mmk_pack_mllama_peer(const float* final_resid, const void* inter, int32_t n_inter, int32_t rows,
                         int32_t d, void* out, cudaStream_t stream);
/*
 * CLIP/LLaVA: drop the first `drop` tokens of every tile: out bf16 [tiles*(P-drop), d] from
 * src (bf16 or f32 when src_f32 != 0) [tiles*P, d].
 */
int mmk_pack_drop_cls(const void* src, int32_t src_f32, int32_t tiles, int32_t tokens_per_tile,
                      int32_t drop, int32_t d, void* out, cudaStream_t stream);

/* Element count checksum helper for end-to-end runs: out[0] = sum(float(x)) over n bf16. */
int mmk_checksum_bf16(const void* x, int64_t n, float* out, cudaStream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* MMK_H_ */
