// mmk_norm.cu — HBM-bound row kernels of the encoder:
//   K3  LayerNorm over the fp32 residual stream -> bf16 GEMM operand (optionally + per-tile
//       additive embedding: Mllama layernorm_post + post_tile_positional_embedding)
//   embedding assembly (class token, gated position / tile-position embeddings, layernorm_pre)
//   K9  ragged pack of final + intermediate hidden states into the LLM-prefill buffer
// One warp per row, float4 loads, statistics in fp32 (two-pass mean / variance in registers).
#include "sm100_common.cuh"
#include "mmk_internal.h"

namespace mmk {

MMK_DEV float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Normalise the VEC float4 of this lane (columns lane*4 + j*128) in place.
template <int VEC>
MMK_DEV void ln_inplace(float4 (&x)[VEC], int d, const float* __restrict__ gamma, const float* __restrict__ beta,
                        float eps, int lane) {
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < VEC; ++j) s += (x[j].x + x[j].y) + (x[j].z + x[j].w);
  const float mean = warp_sum(s) / d;
  float q = 0.f;
#pragma unroll
  for (int j = 0; j < VEC; ++j) {
    const float a = x[j].x - mean, b = x[j].y - mean, c = x[j].z - mean, e = x[j].w - mean;
    q += (a * a + b * b) + (c * c + e * e);
  }
  const float rstd = rsqrtf(warp_sum(q) / d + eps);
#pragma unroll
  for (int j = 0; j < VEC; ++j) {
    const int col = lane * 4 + j * 128;
    const float4 g = __ldg(reinterpret_cast<const float4*>(gamma + col));
    const float4 b = __ldg(reinterpret_cast<const float4*>(beta + col));
    x[j].x = (x[j].x - mean) * rstd * g.x + b.x;
    x[j].y = (x[j].y - mean) * rstd * g.y + b.y;
    x[j].z = (x[j].z - mean) * rstd * g.z + b.z;
    x[j].w = (x[j].w - mean) * rstd * g.w + b.w;
  }
}

// RMSNorm of the VEC float4 of this lane in place: x * rsqrt(mean(x^2) + eps) * gamma (InternViT).
template <int VEC>
MMK_DEV void rms_inplace(float4 (&x)[VEC], int d, const float* __restrict__ gamma, float eps, int lane) {
  float q = 0.f;
#pragma unroll
  for (int j = 0; j < VEC; ++j) q += (x[j].x * x[j].x + x[j].y * x[j].y) + (x[j].z * x[j].z + x[j].w * x[j].w);
  const float rstd = rsqrtf(warp_sum(q) / d + eps);
#pragma unroll
  for (int j = 0; j < VEC; ++j) {
    const float4 g = __ldg(reinterpret_cast<const float4*>(gamma + lane * 4 + j * 128));
    x[j].x = x[j].x * rstd * g.x;
    x[j].y = x[j].y * rstd * g.y;
    x[j].z = x[j].z * rstd * g.z;
    x[j].w = x[j].w * rstd * g.w;
  }
}

template <int VEC>
MMK_DEV void store_row(void* y, int y_f32, int64_t row, int d, const float4 (&x)[VEC], int lane) {
#pragma unroll
  for (int j = 0; j < VEC; ++j) {
    const int col = lane * 4 + j * 128;
    if (y_f32) {
      *reinterpret_cast<float4*>(reinterpret_cast<float*>(y) + row * d + col) = x[j];
    } else {
      uint2 v;
      v.x = pack_bf16x2(x[j].x, x[j].y);
      v.y = pack_bf16x2(x[j].z, x[j].w);
      *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(y) + row * d + col) = v;
    }
  }
}

template <int VEC>
__global__ void __launch_bounds__(256)
layernorm_kernel(const float* __restrict__ x, void* y, int y_f32, int rows, int d, const float* __restrict__ gamma,
                 const float* __restrict__ beta, float eps, const float* __restrict__ tile_add,
                 const int32_t* __restrict__ tile_image, const int32_t* __restrict__ image_table,
                 const int32_t* __restrict__ tile_slot, int rows_per_tile, int slots) {
  griddep_wait();  // PDL: inputs come from the preceding kernel
  griddep_launch_dependents();
  const int lane = threadIdx.x & 31;
  const int64_t row = static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  if (row >= rows) return;
  float4 v[VEC];
#pragma unroll
  for (int j = 0; j < VEC; ++j) v[j] = *reinterpret_cast<const float4*>(x + row * d + lane * 4 + j * 128);
  if (beta != nullptr) ln_inplace<VEC>(v, d, gamma, beta, eps, lane);
  else rms_inplace<VEC>(v, d, gamma, eps, lane);  // no beta: RMSNorm
  if (tile_add != nullptr) {
    const int64_t tile = row / rows_per_tile;
    const float* add = tile_add + (static_cast<int64_t>(image_table[tile_image[tile]]) * slots + tile_slot[tile]) * d;
#pragma unroll
    for (int j = 0; j < VEC; ++j) {
      const float4 a = __ldg(reinterpret_cast<const float4*>(add + lane * 4 + j * 128));
      v[j].x += a.x; v[j].y += a.y; v[j].z += a.z; v[j].w += a.w;
    }
  }
  store_row<VEC>(y, y_f32, row, d, v, lane);
}

#ifndef MMK_EMBED_MINB
#define MMK_EMBED_MINB 4  // 64 registers: 4 CTAs per SM (the unbounded 134-register build ran 1 CTA per SM, 2.9x slower)
#endif
template <int VEC>
__global__ void __launch_bounds__(256, MMK_EMBED_MINB)
embed_kernel(const float* __restrict__ patch_out, const int32_t* __restrict__ tile_image,
             const int32_t* __restrict__ tile_slot, const int32_t* __restrict__ image_ar, int total_tiles, int P, int d,
             const float* __restrict__ cls, const float* __restrict__ pos, float pos_scale,
             const float* __restrict__ tile_pos, float tile_pos_scale, const float* __restrict__ pre_tile,
             float pre_scale, int slots, const float* __restrict__ gamma, const float* __restrict__ beta, float eps,
             float* __restrict__ resid) {
  griddep_wait();  // PDL: inputs come from the preceding kernel
  griddep_launch_dependents();
  const int lane = threadIdx.x & 31;
  const int64_t row = static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  const int C = cls != nullptr ? 1 : 0;  // SigLIP-style encoders have no class token
  const int S = P + C;                   // tokens per tile
  const int64_t rows = static_cast<int64_t>(total_tiles) * S;
  if (row >= rows) return;
  const int g = static_cast<int>(row / S);
  const int p = static_cast<int>(row - static_cast<int64_t>(g) * S);
  const int ar = image_ar ? image_ar[tile_image[g]] : 0;
  const int slot = tile_slot ? tile_slot[g] : 0;
  float4 v[VEC];
#pragma unroll
  for (int j = 0; j < VEC; ++j) {
    const int col = lane * 4 + j * 128;
    float4 a;
    if (C && p == 0) {
      a = __ldg(reinterpret_cast<const float4*>(cls + col));
    } else {
      a = *reinterpret_cast<const float4*>(patch_out + (static_cast<int64_t>(g) * P + (p - C)) * d + col);
      if (pre_tile != nullptr) {
        const float4 t = __ldg(reinterpret_cast<const float4*>(pre_tile + (static_cast<int64_t>(ar) * slots + slot) * d + col));
        a.x += pre_scale * t.x; a.y += pre_scale * t.y; a.z += pre_scale * t.z; a.w += pre_scale * t.w;
      }
    }
    const float4 ps = __ldg(reinterpret_cast<const float4*>(pos + static_cast<int64_t>(p) * d + col));
    a.x += pos_scale * ps.x; a.y += pos_scale * ps.y; a.z += pos_scale * ps.z; a.w += pos_scale * ps.w;
    if (tile_pos != nullptr) {
      const float4 t = __ldg(reinterpret_cast<const float4*>(
          tile_pos + ((static_cast<int64_t>(ar) * slots + slot) * S + p) * d + col));
      a.x += tile_pos_scale * t.x; a.y += tile_pos_scale * t.y; a.z += tile_pos_scale * t.z; a.w += tile_pos_scale * t.w;
    }
    v[j] = a;
  }
  if (gamma != nullptr) ln_inplace<VEC>(v, d, gamma, beta, eps, lane);  // no LN_pre: SigLIP
  store_row<VEC>(resid, 1, row, d, v, lane);
}

// One CTA per token row: final fp32 -> bf16 columns [0, d); intermediates interleaved
// (column d + c*n_inter + j = inter[j][row][c]) staged through shared memory so that both
// the gather and the 16-byte stores are coalesced.
// One thread per (token row, group of 8 columns): the 8 final-hidden values (fp32 -> bf16) and,
// for each of the NI intermediate layers, 8 bf16 values loaded as one 16-byte vector, interleaved
// in registers into the 8*NI contiguous output values (column d + c*NI + j) and written as NI
// 16-byte stores — no shared memory, coalesced along the row.
template <int NI>
__global__ void __launch_bounds__(256)
pack_mllama_kernel(const float* __restrict__ fin, const __nv_bfloat16* __restrict__ inter, int rows, int d,
                   __nv_bfloat16* __restrict__ out) {
  griddep_wait();  // PDL: inputs come from the preceding kernel
  griddep_launch_dependents();
  const int groups = d / 8;
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= static_cast<int64_t>(rows) * groups) return;
  const int64_t row = idx / groups;
  const int c = static_cast<int>(idx - row * groups) * 8;
  const int64_t ldo = static_cast<int64_t>(d) * (1 + NI);
  __nv_bfloat16* o = out + row * ldo;
  const float4 a = __ldg(reinterpret_cast<const float4*>(fin + row * d + c));
  const float4 b = __ldg(reinterpret_cast<const float4*>(fin + row * d + c + 4));
  st_global_v4(o + c, pack_bf16x2(a.x, a.y), pack_bf16x2(a.z, a.w), pack_bf16x2(b.x, b.y), pack_bf16x2(b.z, b.w));
  if constexpr (NI > 0) {
    uint16_t v[NI][8];
#pragma unroll
    for (int j = 0; j < NI; ++j) {
      const uint4 q = __ldg(reinterpret_cast<const uint4*>(inter + (static_cast<int64_t>(j) * rows + row) * d + c));
      const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        v[j][2 * k] = static_cast<uint16_t>(w[k] & 0xFFFFu);
        v[j][2 * k + 1] = static_cast<uint16_t>(w[k] >> 16);
      }
    }
    // output element e (0 .. 8*NI) of this group = column c + e / NI, layer e % NI
    uint32_t ow[4 * NI];
#pragma unroll
    for (int e = 0; e < 8 * NI; e += 2)
      ow[e / 2] = static_cast<uint32_t>(v[e % NI][e / NI]) | (static_cast<uint32_t>(v[(e + 1) % NI][(e + 1) / NI]) << 16);
    __nv_bfloat16* oi = o + d + static_cast<int64_t>(c) * NI;
#pragma unroll
    for (int k = 0; k < NI; ++k) st_global_v4(oi + 8 * k, ow[4 * k], ow[4 * k + 1], ow[4 * k + 2], ow[4 * k + 3]);
  }
}

// K9 + K10 fused: the same packing, written to a destination that may live in another GPU's
// memory (NVLink peer mapping / symmetric memory).  Each CTA assembles whole output rows in shared
// memory and moves them out as one contiguous span per row — `BULK`: one cp.async.bulk copy per
// row, issued by one thread; else 16-byte stores with a warp covering 512 contiguous bytes — so
// the fabric sees full-line writes instead of the 80-byte-strided stores of the direct kernel.
// Rows are double-buffered: row i+1 is assembled while row i drains.
template <int NI, bool BULK>
__global__ void __launch_bounds__(256)
pack_mllama_staged_kernel(const float* __restrict__ fin, const __nv_bfloat16* __restrict__ inter, int rows, int d,
                          __nv_bfloat16* __restrict__ out) {
  extern __shared__ __align__(128) uint8_t pk_smem[];
  griddep_wait();
  griddep_launch_dependents();
  const int groups = d / 8;
  const int64_t ldo = static_cast<int64_t>(d) * (1 + NI);
  const int row_bytes = static_cast<int>(ldo * 2);
  const int row_vec = row_bytes / 16;
  int buf = 0;
  for (int64_t row = blockIdx.x; row < rows; row += gridDim.x, buf ^= 1) {
    uint8_t* sm = pk_smem + buf * row_bytes;
    if constexpr (BULK) {  // the copy that last read this buffer (two rows ago) has drained
      if (threadIdx.x == 0) tma_store_wait_read<1>();
      __syncthreads();
    }
    for (int g = threadIdx.x; g < groups; g += blockDim.x) {
      const int c = g * 8;
      const float4 a = __ldg(reinterpret_cast<const float4*>(fin + row * d + c));
      const float4 b = __ldg(reinterpret_cast<const float4*>(fin + row * d + c + 4));
      *reinterpret_cast<uint4*>(sm + c * 2) =
          make_uint4(pack_bf16x2(a.x, a.y), pack_bf16x2(a.z, a.w), pack_bf16x2(b.x, b.y), pack_bf16x2(b.z, b.w));
      if constexpr (NI > 0) {
        uint16_t v[NI][8];
#pragma unroll
        for (int j = 0; j < NI; ++j) {
          const uint4 q = __ldg(reinterpret_cast<const uint4*>(inter + (static_cast<int64_t>(j) * rows + row) * d + c));
          const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            v[j][2 * k] = static_cast<uint16_t>(w[k] & 0xFFFFu);
            v[j][2 * k + 1] = static_cast<uint16_t>(w[k] >> 16);
          }
        }
        uint32_t ow[4 * NI];
#pragma unroll
        for (int e = 0; e < 8 * NI; e += 2)
          ow[e / 2] = static_cast<uint32_t>(v[e % NI][e / NI]) | (static_cast<uint32_t>(v[(e + 1) % NI][(e + 1) / NI]) << 16);
        uint4* si = reinterpret_cast<uint4*>(sm + (d + c * NI) * 2);
#pragma unroll
        for (int k = 0; k < NI; ++k) si[k] = make_uint4(ow[4 * k], ow[4 * k + 1], ow[4 * k + 2], ow[4 * k + 3]);
      }
    }
    if constexpr (BULK) {
      fence_proxy_async();  // generic-proxy smem writes -> visible to the bulk copy
      __syncthreads();
      if (threadIdx.x == 0) {
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out + row * ldo),
                     "r"(smem_u32(sm)), "r"(row_bytes)
                     : "memory");
        tma_store_commit();
      }
    } else {
      __syncthreads();
      const uint4* src = reinterpret_cast<const uint4*>(sm);
      uint4* dst = reinterpret_cast<uint4*>(out + row * ldo);
      for (int i = threadIdx.x; i < row_vec; i += blockDim.x) dst[i] = src[i];
      // the next row assembles into the other buffer; this one is rewritten two rows on, after the
      // __syncthreads that precedes that row's copy-out
    }
  }
  if constexpr (BULK) {
    if (threadIdx.x == 0) tma_store_wait<0>();  // writes complete before the kernel retires
  }
}

__global__ void __launch_bounds__(256)
pack_drop_kernel(const void* __restrict__ src, int src_f32, int64_t out_rows, int tokens_per_tile, int drop, int d,
                 __nv_bfloat16* __restrict__ out) {
  griddep_wait();  // PDL: inputs come from the preceding kernel
  griddep_launch_dependents();
  const int keep = tokens_per_tile - drop;
  const int64_t orow = static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  if (orow >= out_rows) return;
  const int lane = threadIdx.x & 31;
  const int64_t tile = orow / keep;
  const int64_t srow = tile * tokens_per_tile + drop + (orow - tile * keep);
  for (int c = lane * 8; c < d; c += 256) {
    if (src_f32) {
      const float* s = reinterpret_cast<const float*>(src) + srow * d + c;
      const float4 a = *reinterpret_cast<const float4*>(s);
      const float4 b = *reinterpret_cast<const float4*>(s + 4);
      st_global_v4(out + orow * d + c, pack_bf16x2(a.x, a.y), pack_bf16x2(a.z, a.w), pack_bf16x2(b.x, b.y),
                   pack_bf16x2(b.z, b.w));
    } else {
      *reinterpret_cast<uint4*>(out + orow * d + c) =
          *reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(src) + srow * d + c);
    }
  }
}

__global__ void checksum_kernel(const __nv_bfloat16* __restrict__ x, int64_t n, float* out) {
  griddep_wait();  // PDL: inputs come from the preceding kernel
  griddep_launch_dependents();
  float s = 0.f;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    s += __bfloat162float(x[i]);
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, s);
}


static int grid_rows(int64_t rows) { return static_cast<int>((rows + 7) / 8); }

// Folded LayerNorm: the producer GEMM's per-32-column (mean, M2) of a row -> (mu, rstd), merged
// with Chan's formula.  A warp per row: the lanes read the row's chunk statistics coalesced (up to
// 2 chunks per lane, merged in registers), then a shuffle tree merges the lanes.
MMK_DEV void chan_merge(float& n, float& mean, float& m2, float nb, float meanb, float m2b) {
  const float nn = n + nb;
  if (nb == 0.f) return;
  if (n == 0.f) { n = nb; mean = meanb; m2 = m2b; return; }
  const float delta = meanb - mean;
  const float f = nb / nn;
  mean = fmaf(delta, f, mean);
  m2 = m2 + m2b + delta * delta * n * f;
  n = nn;
}

__global__ void ln_stats_finalize_kernel(const float2* __restrict__ stats, int rows, int parts, float inv_d, float eps,
                                         int rms, float2* __restrict__ mr) {
  griddep_wait();  // PDL: the statistics come from the preceding GEMM
  griddep_launch_dependents();
  const int lane = threadIdx.x & 31;
  const int64_t row = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= rows) return;
  const float2* s = stats + row * parts;
  float n = 0.f, mean = 0.f, m2 = 0.f;
  for (int i = lane; i < parts; i += 32) {
    const float2 b = s[i];
    chan_merge(n, mean, m2, 32.f, b.x, b.y);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float nb = __shfl_xor_sync(0xffffffffu, n, o), mb = __shfl_xor_sync(0xffffffffu, mean, o),
                m2b = __shfl_xor_sync(0xffffffffu, m2, o);
    chan_merge(n, mean, m2, nb, mb, m2b);
  }
  if (lane == 0) {
    if (rms)  // RMSNorm: no centring, mean(x^2) = M2 / n + mean^2
      mr[row] = make_float2(0.f, rsqrtf(fmaf(m2, inv_d, fmaf(mean, mean, eps))));
    else
      mr[row] = make_float2(mean, rsqrtf(fmaf(m2, inv_d, eps)));
  }
}

// Thread-per-row form (the chunk count even, as for every preset width: 24 / 32 / 36 / 40 / 100):
// a row's chunk statistics are 16-byte loads of one contiguous run (a warp covers 32 adjacent rows'
// runs, whole sectors), and equal-size chunks merge without divisions or shuffles:
//   mean = avg(mean_i),  M2 = sum(M2_i) + 32 * sum((mean_i - mean)^2)
// (the warp-per-row Chan merge above ran at ~1 TB/s: 5 shuffle rounds with a division each).
__global__ void __launch_bounds__(256)
ln_stats_finalize_rows_kernel(const float4* __restrict__ stats, int rows, int parts, float inv_d, float eps, int rms,
                              float2* __restrict__ mr) {
  griddep_wait();  // PDL: the statistics come from the preceding GEMM
  griddep_launch_dependents();
  const int64_t row = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (row >= rows) return;
  const int half = parts >> 1;  // float4 = two chunks (mean, M2, mean, M2)
  const float4* s = stats + row * half;
  float sm = 0.f, sq = 0.f;
#pragma unroll 4
  for (int i = 0; i < half; ++i) {
    const float4 v = __ldg(s + i);
    sm += v.x + v.z;
    sq += v.y + v.w;
  }
  const float mean = sm / static_cast<float>(parts);
  float dev = 0.f;
#pragma unroll 4
  for (int i = 0; i < half; ++i) {
    const float4 v = __ldg(s + i);
    const float a = v.x - mean, b = v.z - mean;
    dev = fmaf(a, a, fmaf(b, b, dev));
  }
  const float m2 = fmaf(32.f, dev, sq);
  mr[row] = rms ? make_float2(0.f, rsqrtf(fmaf(m2, inv_d, fmaf(mean, mean, eps))))
                : make_float2(mean, rsqrtf(fmaf(m2, inv_d, eps)));
}

// QK-norm (InternViT use_qk_norm): RMSNorm over the whole query and the whole key projection of a
// token (all heads, d columns each), in place on the bf16 [Q | K | V] rows; a warp per (row, Q or K).
// The warp's d columns are loaded once into registers (all NCH 16-byte loads in flight together:
// the loop form with a second read ran at 1.9 TB/s), reduced, scaled and stored.
template <int NCH>
__global__ void __launch_bounds__(256)
qk_rmsnorm_kernel(__nv_bfloat16* __restrict__ qkv, int rows, int d, int64_t ld, const float* __restrict__ q_w,
                  const float* __restrict__ k_w, float eps) {
  griddep_wait();
  griddep_launch_dependents();
  const int lane = threadIdx.x & 31;
  const int64_t item = static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  if (item >= 2ll * rows) return;
  const int64_t row = item >> 1;
  const int which = static_cast<int>(item & 1);  // 0: Q, 1: K
  __nv_bfloat16* p = qkv + row * ld + which * d;
  const float* w = which ? k_w : q_w;
  uint4 u[NCH];
#pragma unroll
  for (int j = 0; j < NCH; ++j) {
    const int c = lane * 8 + j * 256;
    u[j] = c < d ? *reinterpret_cast<const uint4*>(p + c) : make_uint4(0u, 0u, 0u, 0u);
  }
  float q = 0.f;
#pragma unroll
  for (int j = 0; j < NCH; ++j) {
    const uint32_t wv[4] = {u[j].x, u[j].y, u[j].z, u[j].w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&wv[i]));
      q = fmaf(f.x, f.x, fmaf(f.y, f.y, q));
    }
  }
  const float rstd = rsqrtf(warp_sum(q) / d + eps);
#pragma unroll
  for (int j = 0; j < NCH; ++j) {
    const int c = lane * 8 + j * 256;
    if (c >= d) break;
    uint32_t wv[4] = {u[j].x, u[j].y, u[j].z, u[j].w};
    const float4 w0 = __ldg(reinterpret_cast<const float4*>(w + c)), w1 = __ldg(reinterpret_cast<const float4*>(w + c + 4));
    const float ww[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&wv[i]));
      wv[i] = pack_bf16x2(f.x * rstd * ww[2 * i], f.y * rstd * ww[2 * i + 1]);
    }
    *reinterpret_cast<uint4*>(p + c) = make_uint4(wv[0], wv[1], wv[2], wv[3]);
  }
}

// InternVL pixel shuffle (downsample 0.5) of each tile's patch grid, CLS dropped: output token
// (yj, xk) of a tile = [f(2yj, 2xk) | f(2yj, 2xk+1) | f(2yj+1, 2xk) | f(2yj+1, 2xk+1)] (4 d columns;
// transformers InternVLModel.pixel_shuffle order).  A thread per (output row, 8 columns).
__global__ void __launch_bounds__(256)
pack_pixel_shuffle_kernel(const float* __restrict__ src, int64_t out_rows, int side, int tokens_per_tile, int drop,
                          int d, __nv_bfloat16* __restrict__ out) {
  griddep_wait();
  griddep_launch_dependents();
  const int groups = 4 * d / 8;
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= out_rows * groups) return;
  const int64_t orow = idx / groups;
  const int c8 = static_cast<int>(idx - orow * groups) * 8;
  const int half = side / 2;
  const int64_t tile = orow / (half * half);
  const int t = static_cast<int>(orow - tile * half * half);
  const int yj = t / half, xk = t - yj * half;
  const int q = c8 / d, c = c8 - q * d;
  const int y = 2 * yj + (q >> 1), x = 2 * xk + (q & 1);
  const float* s = src + (tile * tokens_per_tile + drop + y * side + x) * static_cast<int64_t>(d) + c;
  const float4 a = *reinterpret_cast<const float4*>(s), b = *reinterpret_cast<const float4*>(s + 4);
  st_global_v4(out + orow * (4ll * d) + c8, pack_bf16x2(a.x, a.y), pack_bf16x2(a.z, a.w), pack_bf16x2(b.x, b.y),
               pack_bf16x2(b.z, b.w));
}

// Wide-row LayerNorm on bf16 rows (the InternVL projector's LayerNorm(4 d) over pixel-shuffled
// tokens, 12800 columns): a CTA per row; the row (<= 32 KB) is read from L1/L2 three times.
__global__ void __launch_bounds__(256)
layernorm_bf16_kernel(const __nv_bfloat16* __restrict__ x, __nv_bfloat16* __restrict__ y, int d,
                      const float* __restrict__ gamma, const float* __restrict__ beta, float eps) {
  griddep_wait();
  griddep_launch_dependents();
  __shared__ float red[8];
  const int64_t row = blockIdx.x;
  const __nv_bfloat16* xr = x + row * d;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  auto block_sum = [&](float v) {
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    float t = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) t += red[i];
    return t;
  };
  float s = 0.f;
  for (int c = threadIdx.x * 8; c < d; c += 2048) {
    const uint4 u = *reinterpret_cast<const uint4*>(xr + c);
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[i]));
      s += f.x + f.y;
    }
  }
  const float mean = block_sum(s) / d;
  float q = 0.f;
  for (int c = threadIdx.x * 8; c < d; c += 2048) {
    const uint4 u = *reinterpret_cast<const uint4*>(xr + c);
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[i]));
      q = fmaf(f.x - mean, f.x - mean, fmaf(f.y - mean, f.y - mean, q));
    }
  }
  const float rstd = rsqrtf(block_sum(q) / d + eps);
  for (int c = threadIdx.x * 8; c < d; c += 2048) {
    const uint4 u = *reinterpret_cast<const uint4*>(xr + c);
    uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[i]));
      const int k = c + 2 * i;
      w[i] = pack_bf16x2(fmaf((f.x - mean) * rstd, __ldg(gamma + k), __ldg(beta + k)),
                         fmaf((f.y - mean) * rstd, __ldg(gamma + k + 1), __ldg(beta + k + 1)));
    }
    *reinterpret_cast<uint4*>(y + row * d + c) = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

}  // namespace mmk

using namespace mmk;

extern "C" int mmk_layernorm_bf16(const void* x, void* y, int32_t rows, int32_t d, const float* gamma,
                                  const float* beta, float eps, cudaStream_t stream) {
  if (rows < 0 || d <= 0 || d % 8 != 0 || gamma == nullptr || beta == nullptr)
    return set_error(MMK_ERR_ARG, "layernorm_bf16: rows >= 0, d a multiple of 8, gamma and beta required");
  if (rows == 0) return MMK_OK;
  (void)launch_kernel(layernorm_bf16_kernel, dim3(static_cast<unsigned>(rows)), dim3(256), 0, stream, 1,
                      rows <= kSmallRows, reinterpret_cast<const __nv_bfloat16*>(x),
                      reinterpret_cast<__nv_bfloat16*>(y), d, gamma, beta, eps);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? MMK_OK : set_cuda_error(e, "layernorm_bf16: launch");
}

#define MMK_LN_CASE(V)                                                                                       \
  case V:                                                                                                    \
    (void)launch_kernel(layernorm_kernel<V>, dim3(grid_rows(rows)), dim3(256), 0, stream, 1, rows <= kSmallRows, x, y, y_f32, rows, d, gamma, beta, eps, tile_add, \
                                                             tile_image, image_table, tile_slot, rows_per_tile, \
                                                             slots);                                            \
    break;

extern "C" int mmk_layernorm(const float* x, void* y, int32_t y_f32, int32_t rows, int32_t d, const float* gamma,
                             const float* beta, float eps, const float* tile_add, const int32_t* tile_image,
                             const int32_t* image_table, const int32_t* tile_slot, int32_t rows_per_tile,
                             int32_t slots, cudaStream_t stream) {
  if (rows < 0 || d <= 0) return set_error(MMK_ERR_ARG, "layernorm: bad shape");
  if (rows == 0) return MMK_OK;
  if (tile_add && (rows_per_tile <= 0 || !tile_image || !image_table || !tile_slot))
    return set_error(MMK_ERR_ARG, "layernorm: tile_add needs tile_image/image_table/tile_slot/rows_per_tile");
  switch (d / 128 * (d % 128 == 0)) {
    MMK_LN_CASE(4)
    MMK_LN_CASE(6)
    MMK_LN_CASE(9)
    MMK_LN_CASE(8)
    MMK_LN_CASE(10)
    MMK_LN_CASE(12)
    MMK_LN_CASE(16)
    MMK_LN_CASE(25)
    default: return set_error(MMK_ERR_UNSUPPORTED, "layernorm: d=%d unsupported", d);
  }
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? MMK_OK : set_cuda_error(e, "layernorm: launch");
}

#define MMK_EMB_CASE(V)                                                                                   \
  case V:                                                                                                 \
    (void)launch_kernel(embed_kernel<V>, dim3(grid_rows(rows)), dim3(256), 0, stream, 1, rows <= kSmallRows, patch_out, tile_image, tile_slot, image_ar,      \
                                                         total_tiles, patches_per_tile, d, cls, pos,       \
                                                         pos_scale, tile_pos, tile_pos_scale, pre_tile,    \
                                                         pre_scale, slots, gamma, beta, eps, resid);       \
    break;

extern "C" int mmk_embed_tokens(const float* patch_out, const int32_t* tile_image, const int32_t* tile_slot,
                                const int32_t* image_ar, int32_t total_tiles, int32_t patches_per_tile, int32_t d,
                                const float* cls, const float* pos, float pos_scale, const float* tile_pos,
                                float tile_pos_scale, const float* pre_tile, float pre_scale, int32_t slots,
                                const float* gamma, const float* beta, float eps, float* resid,
                                cudaStream_t stream) {
  if (total_tiles < 0 || patches_per_tile <= 0 || d <= 0) return set_error(MMK_ERR_ARG, "embed: bad shape");
  if ((tile_pos || pre_tile) && (!tile_image || !tile_slot || !image_ar))
    return set_error(MMK_ERR_ARG, "embed: tile embeddings need tile_image/tile_slot/image_ar");
  const int64_t rows = static_cast<int64_t>(total_tiles) * (patches_per_tile + (cls != nullptr ? 1 : 0));
  if (rows == 0) return MMK_OK;
  switch (d / 128 * (d % 128 == 0)) {
    MMK_EMB_CASE(4)
    MMK_EMB_CASE(9)
    MMK_EMB_CASE(6)
    MMK_EMB_CASE(8)
    MMK_EMB_CASE(10)
    MMK_EMB_CASE(12)
    MMK_EMB_CASE(16)
    MMK_EMB_CASE(25)
    default: return set_error(MMK_ERR_UNSUPPORTED, "embed: d=%d unsupported", d);
  }
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? MMK_OK : set_cuda_error(e, "embed: launch");
}

extern "C" int mmk_pack_mllama(const float* final_resid, const void* inter, int32_t n_inter, int32_t rows, int32_t d,
                               void* out, cudaStream_t stream) {
  if (rows < 0 || d <= 0 || n_inter < 0 || d % 8 != 0) return set_error(MMK_ERR_ARG, "pack_mllama: bad shape");
  if (n_inter > 8) return set_error(MMK_ERR_UNSUPPORTED, "pack_mllama: n_inter=%d > 8", n_inter);
  if (rows == 0) return MMK_OK;
  const int64_t items = static_cast<int64_t>(rows) * (d / 8);
  const dim3 grid(static_cast<unsigned>((items + 255) / 256));
  const auto* in = reinterpret_cast<const __nv_bfloat16*>(inter);
  auto* o = reinterpret_cast<__nv_bfloat16*>(out);
  const bool small = rows <= kSmallRows;
  switch (n_inter) {
#define MMK_PACK_CASE(N) \
  case N: (void)launch_kernel(pack_mllama_kernel<N>, grid, dim3(256), 0, stream, 1, small, final_resid, in, rows, d, o); break;
    MMK_PACK_CASE(0) MMK_PACK_CASE(1) MMK_PACK_CASE(2) MMK_PACK_CASE(3) MMK_PACK_CASE(4)
    MMK_PACK_CASE(5) MMK_PACK_CASE(6) MMK_PACK_CASE(7) MMK_PACK_CASE(8)
#undef MMK_PACK_CASE
  }
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? MMK_OK : set_cuda_error(e, "pack_mllama: launch");
}

extern "C" int mmk_pack_mllama_peer(const float* final_resid, const void* inter, int32_t n_inter, int32_t rows,
                                    int32_t d, void* out, cudaStream_t stream) {
  if (rows < 0 || d <= 0 || n_inter < 0 || d % 8 != 0) return set_error(MMK_ERR_ARG, "pack_mllama_peer: bad shape");
  if (n_inter > 8) return set_error(MMK_ERR_UNSUPPORTED, "pack_mllama_peer: n_inter=%d > 8", n_inter);
  if (reinterpret_cast<uintptr_t>(out) % 16 != 0) return set_error(MMK_ERR_ARG, "pack_mllama_peer: out not 16-byte aligned");
  if (rows == 0) return MMK_OK;
  static const int mode = [] {
    const char* e = getenv("MMK_PACK_PEER_BULK");
    return e ? atoi(e) : 1;
  }();
  const int smem = 2 * d * (1 + n_inter) * 2;
  if (smem > 200 * 1024) return set_error(MMK_ERR_UNSUPPORTED, "pack_mllama_peer: row of %d bytes", smem / 2);
  const dim3 grid(static_cast<unsigned>(rows < 4 * num_sms() ? rows : 4 * num_sms()));
  const auto* in = reinterpret_cast<const __nv_bfloat16*>(inter);
  auto* o = reinterpret_cast<__nv_bfloat16*>(out);
  cudaError_t e = cudaSuccess;
  auto go = [&](auto kern) {
    if (smem > 48 * 1024) e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e == cudaSuccess) e = launch_kernel(kern, grid, dim3(256), smem, stream, 1, false, final_resid, in, rows, d, o);
  };
  switch (n_inter) {
#define MMK_PACK_CASE(N) \
  case N: if (mode) go(pack_mllama_staged_kernel<N, true>); else go(pack_mllama_staged_kernel<N, false>); break;
    MMK_PACK_CASE(0) MMK_PACK_CASE(1) MMK_PACK_CASE(2) MMK_PACK_CASE(3) MMK_PACK_CASE(4)
    MMK_PACK_CASE(5) MMK_PACK_CASE(6) MMK_PACK_CASE(7) MMK_PACK_CASE(8)
#undef MMK_PACK_CASE
  }
  if (e == cudaSuccess) e = cudaGetLastError();
  return e == cudaSuccess ? MMK_OK : set_cuda_error(e, "pack_mllama_peer: launch");
}

extern "C" int mmk_pack_drop_cls(const void* src, int32_t src_f32, int32_t tiles, int32_t tokens_per_tile,
                                 int32_t drop, int32_t d, void* out, cudaStream_t stream) {
  if (tiles < 0 || tokens_per_tile <= drop || drop < 0 || d % 8 != 0) return set_error(MMK_ERR_ARG, "pack_drop: bad shape");
  const int64_t out_rows = static_cast<int64_t>(tiles) * (tokens_per_tile - drop);
  if (out_rows == 0) return MMK_OK;
  (void)launch_kernel(pack_drop_kernel, dim3(grid_rows(out_rows)), dim3(256), 0, stream, 1, out_rows <= kSmallRows, src, src_f32, out_rows, tokens_per_tile, drop, d,
                                                            reinterpret_cast<__nv_bfloat16*>(out));
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? MMK_OK : set_cuda_error(e, "pack_drop: launch");
}

extern "C" int mmk_checksum_bf16(const void* x, int64_t n, float* out, cudaStream_t stream) {
  if (n < 0) return set_error(MMK_ERR_ARG, "checksum: n < 0");
  cudaError_t e = cudaMemsetAsync(out, 0, sizeof(float), stream);
  if (e != cudaSuccess) return set_cuda_error(e, "checksum: memset");
  if (n == 0) return MMK_OK;
  (void)launch_kernel(checksum_kernel, dim3(4 * num_sms()), dim3(256), 0, stream, 1, n <= 1024 * kSmallRows, reinterpret_cast<const __nv_bfloat16*>(x), n, out);
  e = cudaGetLastError();
  return e == cudaSuccess ? MMK_OK : set_cuda_error(e, "checksum: launch");
}

extern "C" int mmk_ln_stats_finalize(const float* stats, int32_t rows, int32_t d, float eps, int32_t rms, float* mr,
                                     cudaStream_t stream) {
  if (rows < 0 || d < 32 || d % 32 != 0) return set_error(MMK_ERR_ARG, "ln_stats_finalize: rows < 0 or d %% 32 != 0");
  if (rows == 0) return MMK_OK;
  if ((d / 32) % 2 == 0 && (reinterpret_cast<uintptr_t>(stats) & 15) == 0) {
    (void)launch_kernel(ln_stats_finalize_rows_kernel, dim3((rows + 255) / 256), dim3(256), 0, stream, 1,
                        rows <= kSmallRows, reinterpret_cast<const float4*>(stats), rows, d / 32,
                        1.f / static_cast<float>(d), eps, rms, reinterpret_cast<float2*>(mr));
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? MMK_OK : set_cuda_error(e, "ln_stats_finalize: launch");
  }
  (void)launch_kernel(ln_stats_finalize_kernel, dim3((rows + 7) / 8), dim3(256), 0, stream, 1, rows <= kSmallRows,
                      reinterpret_cast<const float2*>(stats), rows, d / 32, 1.f / static_cast<float>(d), eps, rms,
                      reinterpret_cast<float2*>(mr));
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? MMK_OK : set_cuda_error(e, "ln_stats_finalize: launch");
}

extern "C" int mmk_qk_rmsnorm(void* qkv, int32_t rows, int32_t d, int64_t ld, const float* q_w, const float* k_w,
                              float eps, cudaStream_t stream) {
  if (rows < 0 || d <= 0 || d % 8 != 0 || ld < 3ll * d || ld % 8 != 0)
    return set_error(MMK_ERR_ARG, "qk_rmsnorm: bad shape (d multiple of 8, ld >= 3 d)");
  if (rows == 0) return MMK_OK;
  if (d > 16 * 256) return set_error(MMK_ERR_UNSUPPORTED, "qk_rmsnorm: d=%d > 4096", d);
  const int nch = (d + 255) / 256;
  auto kern = nch <= 4 ? qk_rmsnorm_kernel<4> : nch <= 8 ? qk_rmsnorm_kernel<8> : nch <= 13 ? qk_rmsnorm_kernel<13>
                                                                                             : qk_rmsnorm_kernel<16>;
  (void)launch_kernel(kern, dim3(grid_rows(2ll * rows)), dim3(256), 0, stream, 1, rows <= kSmallRows,
                      reinterpret_cast<__nv_bfloat16*>(qkv), rows, d, static_cast<int64_t>(ld), q_w, k_w, eps);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? MMK_OK : set_cuda_error(e, "qk_rmsnorm: launch");
}

extern "C" int mmk_pack_pixel_shuffle(const float* src, int32_t tiles, int32_t side, int32_t tokens_per_tile,
                                      int32_t drop, int32_t d, void* out, cudaStream_t stream) {
  if (tiles < 0 || side < 2 || side % 2 || tokens_per_tile != side * side + drop || d % 8 != 0)
    return set_error(MMK_ERR_ARG, "pack_pixel_shuffle: bad shape");
  const int64_t out_rows = static_cast<int64_t>(tiles) * (side / 2) * (side / 2);
  if (out_rows == 0) return MMK_OK;
  const int64_t items = out_rows * (4ll * d / 8);
  (void)launch_kernel(pack_pixel_shuffle_kernel, dim3(static_cast<unsigned>((items + 255) / 256)), dim3(256), 0, stream,
                      1, out_rows <= kSmallRows, src, out_rows, side, tokens_per_tile, drop, d,
                      reinterpret_cast<__nv_bfloat16*>(out));
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? MMK_OK : set_cuda_error(e, "pack_pixel_shuffle: launch");
}
