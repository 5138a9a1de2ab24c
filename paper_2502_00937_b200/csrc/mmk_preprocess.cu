// mmk_preprocess.cu — K1: fused uint8 HWC -> bilinear resize -> pad/crop -> normalize ->
// tile -> patchify, written straight into the bf16 patch matrix the patch-embed GEMM reads.
//
// Replaces the modelled CPU lane `LatencyProfile.preprocess_latency` (reference
// pkg/src/lmmsim/profiles.py:128-134, driven from engine.py:639-657).  The reference has no
// pixel arithmetic; the geometry and arithmetic here are the builder's definition
// (DESIGN.md §3), restated op-for-op in oracle/preprocess.py so results are bit-identical:
// every fp32 operation is an explicit round-to-nearest intrinsic (no FMA contraction).
//
// Grid: one CTA per (tile, patch-row) band of p pixel rows.  Each thread resamples whole
// pixels (the bilinear weights are shared by the three channels), writes the normalised bf16
// values into the band's patch vectors in shared memory, and the band — a contiguous
// per_side * k_pad run of the patch matrix — leaves with 16-byte stores, a warp covering 512
// contiguous bytes.  The uint8 source is read through L1 (each source pixel feeds <= 4 outputs
// per channel when upsampling).
#include "sm100_common.cuh"
#include "mmk_internal.h"

namespace mmk {

constexpr int kMaxPatch = 64;  // patch edge limit of the band kernel

// Exact uint8 -> fp32 on the FMA pipe: 2^23 + b has b in its low mantissa bits (the I2F
// conversion runs on the quarter-rate XU pipe and was this kernel's limiter).
MMK_DEV float u8_to_f32(uint32_t b) { return __fsub_rn(__uint_as_float(0x4B000000u | b), 8388608.f); }

struct PrepImage {
  int img, slot, tiles, w, h, rows, cols, nw, nh;
  int64_t off;
};

#ifndef MMK_PREP_MINB
#define MMK_PREP_MINB 2
#endif
#ifndef MMK_PREP_UNROLL
#define MMK_PREP_UNROLL 2
#endif
constexpr int kPrepUnroll = MMK_PREP_UNROLL;  // band rows in flight per thread
template <bool CHW>
__global__ void __launch_bounds__(512, MMK_PREP_MINB)
preprocess_kernel(const uint8_t* __restrict__ src, const int64_t* __restrict__ src_off, const int32_t* __restrict__ w,
                  const int32_t* __restrict__ h, const int64_t* __restrict__ tile_off,
                  const int32_t* __restrict__ geom, int n, int T, int p, int k_pad, int mode, int thumb,
                  const float* __restrict__ scale3, const float* __restrict__ shift3,
                  __nv_bfloat16* __restrict__ patches, int parts) {
  extern __shared__ __align__(16) uint8_t prep_smem[];
  __nv_bfloat16* band = reinterpret_cast<__nv_bfloat16*>(prep_smem);  // [per_side][k_pad]
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
  const float sc0 = s_scale[0], sc1 = s_scale[1], sc2 = s_scale[2];
  const float sh0 = s_shift[0], sh1 = s_shift[1], sh2 = s_shift[2];
  // 1) resample the band's p x T pixels.  The row-side bilinear terms depend only on the band
  //    row: computed once into shared memory.  Each thread owns fixed columns (the column-side
  //    terms and the patch coordinates are hoisted out of the row loop) and produces all three
  //    channels of each pixel; a warp covers 32 consecutive columns of one row.
  __shared__ int64_t s_r0[kMaxPatch], s_r1[kMaxPatch];  // byte offsets of source rows y0, y1
  __shared__ float s_fy[kMaxPatch], s_gy[kMaxPatch];
  if (threadIdx.x < p) {
    const int Y = oy + pr * p + threadIdx.x;
    float sy = __fsub_rn(__fmul_rn(__fadd_rn(static_cast<float>(Y), 0.5f), scly), 0.5f);
    sy = fmaxf(sy, 0.f);
    int y0 = static_cast<int>(floorf(sy));
    y0 = min(y0, m.h - 1);
    const int y1 = min(y0 + 1, m.h - 1);
    const float fy = __fsub_rn(sy, static_cast<float>(y0));
    const int64_t row_bytes = CHW ? m.w : 3ll * m.w;
    s_r0[threadIdx.x] = y0 * row_bytes;
    s_r1[threadIdx.x] = y1 * row_bytes;
    s_fy[threadIdx.x] = fy;
    s_gy[threadIdx.x] = __fsub_rn(1.f, fy);
  }
  __syncthreads();
  const int64_t plane = CHW ? static_cast<int64_t>(m.h) * m.w : 1;  // channel stride
#ifndef MMK_PREP_NO_PREFETCH
  {  // pull the band's source rows into L2 up front (bulk prefetch), so the per-pixel byte loads
     // below hit L2 instead of each waiting on HBM
    const auto col_of = [&](int X) {
      float sx = __fsub_rn(__fmul_rn(__fadd_rn(static_cast<float>(X), 0.5f), sclx), 0.5f);
      return min(static_cast<int>(floorf(fmaxf(sx, 0.f))), m.w - 1);
    };
    const int xa = col_of(ox), xb = min(col_of(ox + T - 1) + 1, m.w - 1);
    const int64_t rb = CHW ? m.w : 3ll * m.w;
    const int ya = static_cast<int>(s_r0[0] / rb), yb = static_cast<int>(s_r1[p - 1] / rb);
    const int nrows = (yb - ya + 1) * (CHW ? 3 : 1);
    for (int r = threadIdx.x; r < nrows; r += blockDim.x) {
      const int c = CHW ? r / (yb - ya + 1) : 0;
      const int y = ya + r - c * (yb - ya + 1);
      const uint8_t* lo = img + c * plane + y * rb + (CHW ? xa : 3 * xa);
      const uint8_t* hi = img + c * plane + y * rb + (CHW ? xb + 1 : 3 * (xb + 1));
      const uintptr_t a0 = reinterpret_cast<uintptr_t>(lo) & ~uintptr_t(15);
      const uintptr_t end = reinterpret_cast<uintptr_t>(img + 3ll * m.w * m.h) & ~uintptr_t(15);  // stay inside
      const uintptr_t a1 = min((reinterpret_cast<uintptr_t>(hi) + 15) & ~uintptr_t(15), end);
      if (a1 > a0)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a0), "r"(static_cast<uint32_t>(a1 - a0)) : "memory");
    }
  }
#endif
  const int row_lim = (is_thumb || crop) ? p : min(p, m.nh - (oy + pr * p));  // rows inside the resized image
  // the band is processed in `parts` column ranges of whole patches, sized so that one thread per
  // column covers a part in one pass (blockDim = the part's columns rounded up to a warp)
  const int pc_per = (per_side + parts - 1) / parts;
  for (int pc0 = 0; pc0 < per_side; pc0 += pc_per) {
    const int pc1 = min(per_side, pc0 + pc_per);
    if (pc0 > 0) __syncthreads();  // the previous part's copy-out has read the buffer
    for (int xl = pc0 * p + threadIdx.x; xl < pc1 * p; xl += blockDim.x) {
      const int pc = xl / p, ix = xl - pc * p;
      const int X = ox + xl;
      const bool col_in = is_thumb || crop || X < m.nw;
      // same operation sequence as the oracle's bilinear sample (bit-identical), column side
      float sx = __fsub_rn(__fmul_rn(__fadd_rn(static_cast<float>(X), 0.5f), sclx), 0.5f);
      sx = fmaxf(sx, 0.f);
      int x0 = static_cast<int>(floorf(sx));
      x0 = min(x0, m.w - 1);
      const int x1 = min(x0 + 1, m.w - 1);
      const float fx = __fsub_rn(sx, static_cast<float>(x0));
      const float gx = __fsub_rn(1.f, fx);
      const int cx0 = CHW ? x0 : 3 * x0, cx1 = CHW ? x1 : 3 * x1;  // byte offsets inside a row
      __nv_bfloat16* o = band + (pc - pc0) * k_pad + ix;  // patch vector order (c, py, px)
#pragma unroll kPrepUnroll
      for (int iy = 0; iy < p; ++iy, o += p) {
        float v[3] = {0.f, 0.f, 0.f};  // padding pixel value (before normalisation): 0, as HF Mllama
        if (col_in && iy < row_lim) {
          const uint8_t* a = img + s_r0[iy];
          const uint8_t* b = img + s_r1[iy];
          const float fy = s_fy[iy], gy = s_gy[iy];
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            const int64_t co = c * plane;
            const float p00 = u8_to_f32(__ldg(a + co + cx0)), p01 = u8_to_f32(__ldg(a + co + cx1));
            const float p10 = u8_to_f32(__ldg(b + co + cx0)), p11 = u8_to_f32(__ldg(b + co + cx1));
            const float top = __fadd_rn(__fmul_rn(gx, p00), __fmul_rn(fx, p01));
            const float bot = __fadd_rn(__fmul_rn(gx, p10), __fmul_rn(fx, p11));
            v[c] = __fadd_rn(__fmul_rn(gy, top), __fmul_rn(fy, bot));
          }
        }
        o[0] = __float2bfloat16_rn(__fadd_rn(__fmul_rn(v[0], sc0), sh0));
        o[pp] = __float2bfloat16_rn(__fadd_rn(__fmul_rn(v[1], sc1), sh1));
        o[2 * pp] = __float2bfloat16_rn(__fadd_rn(__fmul_rn(v[2], sc2), sh2));
      }
    }
    // 2) zero the K padding of every patch vector of the part
    const int padw = k_pad - kreal;
    for (int q = threadIdx.x; q < (pc1 - pc0) * padw; q += blockDim.x) {
      const int pc = q / padw;
      band[pc * k_pad + kreal + (q - pc * padw)] = __float2bfloat16_rn(0.f);
    }
    __syncthreads();
    // 3) the part is one contiguous run of the patch matrix: stream it out
    const uint4* sv = reinterpret_cast<const uint4*>(band);
    uint4* dv = reinterpret_cast<uint4*>(patches + ((static_cast<int64_t>(g) * per_side + pr) * per_side + pc0) * k_pad);
    const int nvec = (pc1 - pc0) * k_pad / 8;
    for (int i = threadIdx.x; i < nvec; i += blockDim.x) dv[i] = sv[i];
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
  if (patch_px > kMaxPatch) return set_error(MMK_ERR_UNSUPPORTED, "preprocess: patch_px %d > %d", patch_px, kMaxPatch);
  if (k_pad < 3 * patch_px * patch_px || k_pad % 8 != 0) return set_error(MMK_ERR_ARG, "preprocess: bad k_pad");
  if (mode != 0 && mode != 1) return set_error(MMK_ERR_ARG, "preprocess: mode must be 0 or 1");
  if (reinterpret_cast<uintptr_t>(patches) & 15) return set_error(MMK_ERR_ARG, "preprocess: patches not 16B aligned");
  if (n == 0 || total_tiles == 0) return MMK_OK;
  const int blocks = total_tiles * (tile_px / patch_px);
  const int per_side = tile_px / patch_px;
  int parts = 1;  // column parts per band: one thread per column of a part, at most 512 threads
  while ((per_side + parts - 1) / parts * patch_px > 512) ++parts;
  const int cols = (per_side + parts - 1) / parts * patch_px;
  const int threads = (cols + 31) / 32 * 32;
  const int smem = (per_side + parts - 1) / parts * k_pad * 2;
  if (smem > 200 * 1024) return set_error(MMK_ERR_UNSUPPORTED, "preprocess: patch row band of %d bytes", smem);
  auto* out = reinterpret_cast<__nv_bfloat16*>(patches);
  auto go = [&](auto kern) -> cudaError_t {
    if (smem > 48 * 1024) {
      const cudaError_t a = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      if (a != cudaSuccess) return a;
    }
    return launch_kernel(kern, dim3(blocks), dim3(threads), smem, stream, 1, total_tiles <= 64, src, src_off, w, h,
                         tile_off, geom, n, tile_px, patch_px, k_pad, mode, thumbnail, scale3, shift3, out, parts);
  };
  const cudaError_t le = src_chw ? go(preprocess_kernel<true>) : go(preprocess_kernel<false>);
  if (le != cudaSuccess) return set_cuda_error(le, "preprocess: launch");
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? MMK_OK : set_cuda_error(e, "preprocess: launch");
}
