// mmk_preprocess.cu — K1: fused uint8 HWC -> bilinear resize -> pad/crop -> normalize ->
// tile -> patchify, written straight into the bf16 patch matrix the patch-embed GEMM reads.
//
// Replaces the modelled CPU lane `LatencyProfile.preprocess_latency` (reference
// pkg/src/lmmsim/profiles.py:128-134, driven from engine.py:639-657).  The reference has no
// pixel arithmetic; the geometry and arithmetic here are the builder's definition
// (DESIGN.md §3), restated op-for-op in oracle/preprocess.py so results are bit-identical:
// every fp32 operation is an explicit round-to-nearest intrinsic (no FMA contraction).
//
// Grid: one CTA per (tile, patch-row).  Each thread produces 8 consecutive bf16 of a patch
// row and stores them as one 16-byte vector, so the dominant HBM stream (the bf16 patch
// matrix) is written fully coalesced; the uint8 source is read through L1 (each source pixel
// is touched by <= 4 neighbouring outputs).
#include "sm100_common.cuh"
#include "mmk_internal.h"

namespace mmk {

struct PrepImage {
  int img, slot, tiles, w, h, rows, cols, nw, nh;
  int64_t off;
};

template <bool CHW>
MMK_DEV float bilinear_u8(const uint8_t* __restrict__ img, int w, int h, int c, float sclx, float scly, int X,
                          int Y) {
  float sx = __fsub_rn(__fmul_rn(__fadd_rn(static_cast<float>(X), 0.5f), sclx), 0.5f);
  float sy = __fsub_rn(__fmul_rn(__fadd_rn(static_cast<float>(Y), 0.5f), scly), 0.5f);
  sx = fmaxf(sx, 0.f);
  sy = fmaxf(sy, 0.f);
  int x0 = static_cast<int>(floorf(sx)), y0 = static_cast<int>(floorf(sy));
  x0 = min(x0, w - 1);
  y0 = min(y0, h - 1);
  const int x1 = min(x0 + 1, w - 1), y1 = min(y0 + 1, h - 1);
  const float fx = __fsub_rn(sx, static_cast<float>(x0));
  const float fy = __fsub_rn(sy, static_cast<float>(y0));
  auto px = [&](int y, int x) -> float {
    if constexpr (CHW) return img[(static_cast<int64_t>(c) * h + y) * w + x];
    else return img[(static_cast<int64_t>(y) * w + x) * 3 + c];
  };
  const float p00 = px(y0, x0), p01 = px(y0, x1), p10 = px(y1, x0), p11 = px(y1, x1);
  const float gx = __fsub_rn(1.f, fx), gy = __fsub_rn(1.f, fy);
  const float top = __fadd_rn(__fmul_rn(gx, p00), __fmul_rn(fx, p01));
  const float bot = __fadd_rn(__fmul_rn(gx, p10), __fmul_rn(fx, p11));
  return __fadd_rn(__fmul_rn(gy, top), __fmul_rn(fy, bot));
}

template <bool CHW>
__global__ void __launch_bounds__(256)
preprocess_kernel(const uint8_t* __restrict__ src, const int64_t* __restrict__ src_off, const int32_t* __restrict__ w,
                  const int32_t* __restrict__ h, const int64_t* __restrict__ tile_off,
                  const int32_t* __restrict__ geom, int n, int T, int p, int k_pad, int mode, int thumb,
                  const float* __restrict__ scale3, const float* __restrict__ shift3,
                  __nv_bfloat16* __restrict__ patches) {
  griddep_wait();  // PDL: inputs come from the preceding kernel
  griddep_launch_dependents();
  __shared__ PrepImage meta;
  __shared__ float s_scale[3], s_shift[3];
  const int per_side = T / p;
  const int g = blockIdx.x / per_side;   // global tile
  const int pr = blockIdx.x % per_side;  // patch row inside the tile
  if (threadIdx.x == 0) {
    int lo = 0, hi = n - 1;  // last image with tile_off[i] <= g
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (tile_off[mid] <= g) lo = mid; else hi = mid - 1;
    }
    meta.img = lo;
    meta.slot = static_cast<int>(g - tile_off[lo]);
    meta.tiles = static_cast<int>(tile_off[lo + 1] - tile_off[lo]);
    meta.w = w[lo];
    meta.h = h[lo];
    meta.rows = geom[4 * lo + 0];
    meta.cols = geom[4 * lo + 1];
    meta.nw = geom[4 * lo + 2];
    meta.nh = geom[4 * lo + 3];
    meta.off = src_off[lo];
  }
  if (threadIdx.x < 3) {
    s_scale[threadIdx.x] = scale3[threadIdx.x];
    s_shift[threadIdx.x] = shift3[threadIdx.x];
  }
  __syncthreads();
  const PrepImage m = meta;
  const uint8_t* img = src + m.off;
  const bool is_thumb = thumb && m.tiles > 1 && m.slot == m.tiles - 1;
  int ox = 0, oy = 0, rw = m.nw, rh = m.nh;  // canvas origin of this tile, resize target
  bool crop = false;
  if (is_thumb) {
    rw = T; rh = T;
  } else if (mode == 0) {
    ox = (m.slot % m.cols) * T;
    oy = (m.slot / m.cols) * T;
  } else {
    ox = (m.nw - T) / 2;
    oy = (m.nh - T) / 2;
    crop = true;
  }
  const float sclx = __fdiv_rn(static_cast<float>(m.w), static_cast<float>(rw));
  const float scly = __fdiv_rn(static_cast<float>(m.h), static_cast<float>(rh));
  const int pp = p * p;
  const int kreal = 3 * pp;
  const int total = per_side * k_pad;  // outputs of this CTA
  __nv_bfloat16* out = patches + (static_cast<int64_t>(g) * per_side * per_side + static_cast<int64_t>(pr) * per_side) * k_pad;
  for (int base = threadIdx.x * 8; base < total; base += 256 * 8) {
    uint32_t packed[4];
#pragma unroll
    for (int e = 0; e < 8; e += 2) {
      float v2[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int idx = base + e + u;
        const int pc = idx / k_pad;      // patch column inside the patch row
        const int col = idx - pc * k_pad;
        float val = 0.f;
        if (col < kreal) {
          const int c = col / pp;
          const int rem = col - c * pp;
          const int iy = rem / p, ix = rem - iy * p;
          const int X = ox + pc * p + ix;
          const int Y = oy + pr * p + iy;
          float v = 0.f;  // padding pixel value (before normalisation), as HF Mllama pads with 0
          if (is_thumb || crop || (X < m.nw && Y < m.nh)) v = bilinear_u8<CHW>(img, m.w, m.h, c, sclx, scly, X, Y);
          val = __fadd_rn(__fmul_rn(v, s_scale[c]), s_shift[c]);
        }
        v2[u] = val;
      }
      packed[e / 2] = pack_bf16x2(v2[0], v2[1]);
    }
    st_global_v4(out + base, packed[0], packed[1], packed[2], packed[3]);
  }
}

}  // namespace mmk

using namespace mmk;

extern "C" int mmk_preprocess(const uint8_t* src, const int64_t* src_off, int32_t src_chw, const int32_t* w,
                              const int32_t* h,
                              const int64_t* tile_off, const int32_t* geom, int32_t n, int32_t total_tiles,
                              int32_t tile_px, int32_t patch_px, int32_t k_pad, int32_t mode, int32_t thumbnail,
                              const float* scale3, const float* shift3, void* patches, cudaStream_t stream) {
  if (n < 0 || total_tiles < 0) return set_error(MMK_ERR_ARG, "preprocess: negative sizes");
  if (patch_px < 1 || tile_px % patch_px != 0) return set_error(MMK_ERR_ARG, "preprocess: tile_px %% patch_px != 0");
  if (k_pad < 3 * patch_px * patch_px || k_pad % 8 != 0) return set_error(MMK_ERR_ARG, "preprocess: bad k_pad");
  if (mode != 0 && mode != 1) return set_error(MMK_ERR_ARG, "preprocess: mode must be 0 or 1");
  if (reinterpret_cast<uintptr_t>(patches) & 15) return set_error(MMK_ERR_ARG, "preprocess: patches not 16B aligned");
  if (n == 0 || total_tiles == 0) return MMK_OK;
  const int blocks = total_tiles * (tile_px / patch_px);
  if (src_chw)
    (void)launch_kernel(preprocess_kernel<true>, dim3(blocks), dim3(256), 0, stream, 1, total_tiles <= 64, src, src_off, w, h, tile_off, geom, n, tile_px, patch_px, k_pad,
                                                        mode, thumbnail, scale3, shift3,
                                                        reinterpret_cast<__nv_bfloat16*>(patches));
  else
    (void)launch_kernel(preprocess_kernel<false>, dim3(blocks), dim3(256), 0, stream, 1, total_tiles <= 64, src, src_off, w, h, tile_off, geom, n, tile_px, patch_px,
                                                         k_pad, mode, thumbnail, scale3, shift3,
                                                         reinterpret_cast<__nv_bfloat16*>(patches));
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? MMK_OK : set_cuda_error(e, "preprocess: launch");
}
