/* Plain-C use of the libmmk C ABI (include/mmk.h): tile plan + preprocess of two images on the
 * device, no Python or PyTorch involved.  Build: make -C examples; run: examples/c_abi_demo.
 * Prints the token offsets (reference Request.total_image_tokens prefix sums, core.py:110-120)
 * and a checksum of the bf16 patch matrix; exits non-zero on any libmmk or CUDA error. */
#include <stdio.h>
#include <stdlib.h>
#include <stdint.h>
#include <cuda_runtime_api.h>
#include "mmk.h"

#define CHECK_MMK(x)                                                                     \
  do {                                                                                   \
    int rc_ = (x);                                                                       \
    if (rc_ != MMK_OK) {                                                                 \
      fprintf(stderr, "%s failed (%d): %s\n", #x, rc_, mmk_last_error());               \
      return 1;                                                                          \
    }                                                                                    \
  } while (0)
#define CHECK_CUDA(x)                                                                    \
  do {                                                                                   \
    cudaError_t e_ = (x);                                                                \
    if (e_ != cudaSuccess) {                                                             \
      fprintf(stderr, "%s failed: %s\n", #x, cudaGetErrorString(e_));                   \
      return 1;                                                                          \
    }                                                                                    \
  } while (0)

int main(void) {
  /* Llama-3.2-11B-Vision tiling (model_presets.json): 560 px tiles, 1601 tokens/tile, cap 4 */
  const int32_t n = 2, T = 560, tok = 1601, cap = 4, patch = 14, k_pad = 592;
  const int32_t w[2] = {1000, 560}, h[2] = {500, 1200};
  const int64_t src_off[2] = {0, 1000LL * 500 * 3};
  const size_t src_bytes = (size_t)1000 * 500 * 3 + (size_t)560 * 1200 * 3;
  printf("%s\n", mmk_version());

  int32_t *d_w, *d_h, *d_tiles, *d_geom, *d_ar, *d_bad;
  int64_t *d_tile_off, *d_tok_off, *d_src_off;
  uint8_t* d_src;
  float *d_scale, *d_shift;
  CHECK_CUDA(cudaMalloc((void**)&d_w, sizeof w));
  CHECK_CUDA(cudaMalloc((void**)&d_h, sizeof h));
  CHECK_CUDA(cudaMalloc((void**)&d_tiles, n * sizeof(int32_t)));
  CHECK_CUDA(cudaMalloc((void**)&d_geom, 4 * n * sizeof(int32_t)));
  CHECK_CUDA(cudaMalloc((void**)&d_ar, n * sizeof(int32_t)));
  CHECK_CUDA(cudaMalloc((void**)&d_bad, sizeof(int32_t)));
  CHECK_CUDA(cudaMalloc((void**)&d_tile_off, (n + 1) * sizeof(int64_t)));
  CHECK_CUDA(cudaMalloc((void**)&d_tok_off, (n + 1) * sizeof(int64_t)));
  CHECK_CUDA(cudaMalloc((void**)&d_src_off, sizeof src_off));
  CHECK_CUDA(cudaMalloc((void**)&d_src, src_bytes));
  CHECK_CUDA(cudaMalloc((void**)&d_scale, 3 * sizeof(float)));
  CHECK_CUDA(cudaMalloc((void**)&d_shift, 3 * sizeof(float)));

  uint8_t* src = (uint8_t*)malloc(src_bytes);
  for (size_t i = 0; i < src_bytes; ++i) src[i] = (uint8_t)((i * 2654435761u) >> 24);
  const float scale[3] = {1.f / (255.f * 0.26862954f), 1.f / (255.f * 0.26130258f), 1.f / (255.f * 0.27577711f)};
  const float shift[3] = {-0.48145466f / 0.26862954f, -0.4578275f / 0.26130258f, -0.40821073f / 0.27577711f};
  CHECK_CUDA(cudaMemcpy(d_w, w, sizeof w, cudaMemcpyHostToDevice));
  CHECK_CUDA(cudaMemcpy(d_h, h, sizeof h, cudaMemcpyHostToDevice));
  CHECK_CUDA(cudaMemcpy(d_src_off, src_off, sizeof src_off, cudaMemcpyHostToDevice));
  CHECK_CUDA(cudaMemcpy(d_src, src, src_bytes, cudaMemcpyHostToDevice));
  CHECK_CUDA(cudaMemcpy(d_scale, scale, sizeof scale, cudaMemcpyHostToDevice));
  CHECK_CUDA(cudaMemcpy(d_shift, shift, sizeof shift, cudaMemcpyHostToDevice));

  CHECK_MMK(mmk_tile_plan(d_w, d_h, n, T, tok, cap, 0, 0, d_tiles, d_tile_off, d_tok_off, d_geom, d_ar, d_bad, 0));
  int64_t tile_off[3], tok_off[3];
  CHECK_CUDA(cudaMemcpy(tile_off, d_tile_off, sizeof tile_off, cudaMemcpyDeviceToHost));
  CHECK_CUDA(cudaMemcpy(tok_off, d_tok_off, sizeof tok_off, cudaMemcpyDeviceToHost));
  printf("tok_off %lld %lld %lld\n", (long long)tok_off[0], (long long)tok_off[1], (long long)tok_off[2]);

  const int32_t total_tiles = (int32_t)tile_off[n];
  const size_t patches = (size_t)total_tiles * (T / patch) * (T / patch);
  uint16_t* d_patches;
  CHECK_CUDA(cudaMalloc((void**)&d_patches, patches * k_pad * sizeof(uint16_t)));
  CHECK_MMK(mmk_preprocess(d_src, d_src_off, 0, d_w, d_h, d_tile_off, d_geom, n, total_tiles, T, patch, k_pad, 0, 0,
                           d_scale, d_shift, d_patches, 0));
  uint16_t* hp = (uint16_t*)malloc(patches * k_pad * sizeof(uint16_t));
  CHECK_CUDA(cudaMemcpy(hp, d_patches, patches * k_pad * sizeof(uint16_t), cudaMemcpyDeviceToHost));
  uint64_t sum = 0;
  for (size_t i = 0; i < patches * k_pad; ++i) sum = sum * 1000003u + hp[i];
  printf("tiles %d patches %zu checksum %016llx\n", total_tiles, patches, (unsigned long long)sum);

  /* argument errors come back as status codes with a message, never as crashes */
  if (mmk_tile_plan(d_w, d_h, -1, T, tok, cap, 0, 0, d_tiles, d_tile_off, d_tok_off, d_geom, d_ar, d_bad, 0) !=
      MMK_ERR_ARG) {
    fprintf(stderr, "expected MMK_ERR_ARG\n");
    return 1;
  }
  printf("bad-arg status ok: %s\n", mmk_last_error());
  free(src);
  free(hp);
  return 0;
}
