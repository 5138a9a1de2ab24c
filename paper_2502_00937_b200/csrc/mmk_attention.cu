// mmk_attention.cu — K5: non-causal variable-length multi-head self-attention over the
// tokens of each image (one sequence per image: Mllama n_tiles*1601 tokens, CLIP 577).
//
// Replaces the attention share of the modelled `encode_latency` (reference
// pkg/src/lmmsim/profiles.py:136-145).  Images never attend to each other,
// so sequences are independent: grid = (q-block, sequence, head).
//
// This file holds the register-tiled flash-attention kernel (online softmax, exp2, bf16
// mma.sync.m16n8k16 with fp32 accumulation, cp.async double-buffered K/V tiles).
#include "sm100_common.cuh"
#include <cstdlib>
#include "mmk_internal.h"

namespace mmk {

constexpr int kAttnBQ = 128;   // query rows per CTA (8 warps x 16 rows)
constexpr int kAttnBKV = 64;   // keys per iteration
constexpr int kAttnThreads = 256;

MMK_DEV void cp_async16(void* smem, const void* gmem, bool valid) {
  const int n = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(smem)), "l"(gmem), "r"(n)
               : "memory");
}
MMK_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
MMK_DEV void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
MMK_DEV void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
MMK_DEV void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
MMK_DEV void mma_bf16_16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

template <int HD>
__global__ void __launch_bounds__(kAttnThreads, 2)
attn_fwd_mma(const __nv_bfloat16* __restrict__ qkv, __nv_bfloat16* __restrict__ out,
             const int32_t* __restrict__ cu_seqlens, int heads, float scale_log2) {
  constexpr int LDS = HD + 8;  // padded smem row (elements): conflict-free ldmatrix
  constexpr int KSTEPS = HD / 16;
  constexpr int NT_S = kAttnBKV / 8;  // S n-tiles per warp
  constexpr int NT_O = HD / 8;        // O n-tiles per warp
  constexpr int CHUNKS = HD / 8;      // 16-byte chunks per row
  extern __shared__ __align__(16) uint8_t smem_raw[];
  __nv_bfloat16* sQ = reinterpret_cast<__nv_bfloat16*>(smem_raw);
  __nv_bfloat16* sK = sQ + kAttnBQ * LDS;          // [2][BKV][LDS]
  __nv_bfloat16* sV = sK + 2 * kAttnBKV * LDS;     // [2][BKV][LDS]

  const int seq = blockIdx.y;
  const int head = blockIdx.z;
  const int s_begin = cu_seqlens[seq];
  const int len = cu_seqlens[seq + 1] - s_begin;
  const int q0 = blockIdx.x * kAttnBQ;
  if (q0 >= len) return;

  const int64_t ld = 3LL * heads * HD;
  const __nv_bfloat16* gQ = qkv + static_cast<int64_t>(s_begin) * ld + head * HD;
  const __nv_bfloat16* gK = gQ + heads * HD;
  const __nv_bfloat16* gV = gK + heads * HD;

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;

  // Q tile
  for (int i = tid; i < kAttnBQ * CHUNKS; i += kAttnThreads) {
    const int r = i / CHUNKS, c = i % CHUNKS;
    const int qr = q0 + r;
    cp_async16(sQ + r * LDS + c * 8, gQ + static_cast<int64_t>(qr < len ? qr : 0) * ld + c * 8, qr < len);
  }
  auto load_kv = [&](int buf, int k0) {
    for (int i = tid; i < kAttnBKV * CHUNKS; i += kAttnThreads) {
      const int r = i / CHUNKS, c = i % CHUNKS;
      const int kr = k0 + r;
      const bool ok = kr < len;
      const int64_t off = static_cast<int64_t>(ok ? kr : 0) * ld + c * 8;
      cp_async16(sK + (buf * kAttnBKV + r) * LDS + c * 8, gK + off, ok);
      cp_async16(sV + (buf * kAttnBKV + r) * LDS + c * 8, gV + off, ok);
    }
  };
  load_kv(0, 0);
  cp_async_commit();

  const int n_kv = (len + kAttnBKV - 1) / kAttnBKV;
  float o[NT_O][4];
#pragma unroll
  for (int j = 0; j < NT_O; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
  float m_r[2] = {-INFINITY, -INFINITY}, l_r[2] = {0.f, 0.f};
  uint32_t qf[KSTEPS][4];

  for (int it = 0; it < n_kv; ++it) {
    if (it + 1 < n_kv) load_kv((it + 1) & 1, (it + 1) * kAttnBKV);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    if (it == 0) {
      const uint32_t qbase = smem_u32(sQ + (warp * 16 + (lane & 15)) * LDS + (lane >> 4) * 8);
#pragma unroll
      for (int s = 0; s < KSTEPS; ++s) ldsm_x4(qbase + s * 32, qf[s][0], qf[s][1], qf[s][2], qf[s][3]);
    }
    const int buf = it & 1;
    // S = Q K^T  (16 x 64 per warp)
    float sc[NT_S][4];
#pragma unroll
    for (int j = 0; j < NT_S; ++j) sc[j][0] = sc[j][1] = sc[j][2] = sc[j][3] = 0.f;
    const __nv_bfloat16* kb = sK + buf * kAttnBKV * LDS;
#pragma unroll
    for (int s = 0; s < KSTEPS; ++s) {
#pragma unroll
      for (int j = 0; j < NT_S; j += 2) {
        const int nrow = 8 * (j + (lane >> 4)) + (lane & 7);
        const int kcol = 16 * s + ((lane >> 3) & 1) * 8;
        uint32_t b0, b1, b2, b3;
        ldsm_x4(smem_u32(kb + nrow * LDS + kcol), b0, b1, b2, b3);
        mma_bf16_16816(sc[j], qf[s], b0, b1);
        mma_bf16_16816(sc[j + 1], qf[s], b2, b3);
      }
    }
    // mask keys past the sequence end
    const int k0 = it * kAttnBKV;
    if (k0 + kAttnBKV > len) {
#pragma unroll
      for (int j = 0; j < NT_S; ++j) {
        const int c = k0 + 8 * j + 2 * (lane & 3);
        if (c >= len) { sc[j][0] = -INFINITY; sc[j][2] = -INFINITY; }
        if (c + 1 >= len) { sc[j][1] = -INFINITY; sc[j][3] = -INFINITY; }
      }
    }
    // online softmax (rows g and g+8 of the warp's 16)
    float mx[2] = {m_r[0], m_r[1]};
#pragma unroll
    for (int j = 0; j < NT_S; ++j) {
      mx[0] = fmaxf(mx[0], fmaxf(sc[j][0], sc[j][1]) * scale_log2);
      mx[1] = fmaxf(mx[1], fmaxf(sc[j][2], sc[j][3]) * scale_log2);
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 1));
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 2));
    }
    float corr[2], rs[2] = {0.f, 0.f};
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      corr[r] = exp2f(m_r[r] - mx[r]);
      m_r[r] = mx[r];
    }
    uint32_t pf[NT_S / 2][4];
#pragma unroll
    for (int j = 0; j < NT_S; ++j) {
      const float p0 = exp2f(sc[j][0] * scale_log2 - mx[0]);
      const float p1 = exp2f(sc[j][1] * scale_log2 - mx[0]);
      const float p2 = exp2f(sc[j][2] * scale_log2 - mx[1]);
      const float p3 = exp2f(sc[j][3] * scale_log2 - mx[1]);
      rs[0] += p0 + p1;
      rs[1] += p2 + p3;
      pf[j >> 1][(j & 1) * 2 + 0] = pack_bf16x2(p0, p1);
      pf[j >> 1][(j & 1) * 2 + 1] = pack_bf16x2(p2, p3);
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) l_r[r] = l_r[r] * corr[r] + rs[r];
#pragma unroll
    for (int j = 0; j < NT_O; ++j) {
      o[j][0] *= corr[0]; o[j][1] *= corr[0];
      o[j][2] *= corr[1]; o[j][3] *= corr[1];
    }
    // O += P V
    const __nv_bfloat16* vb = sV + buf * kAttnBKV * LDS;
#pragma unroll
    for (int s = 0; s < kAttnBKV / 16; ++s) {
      // A fragment layout: {row g k-lo, row g+8 k-lo, row g k-hi, row g+8 k-hi}
      const uint32_t a[4] = {pf[s][0], pf[s][1], pf[s][2], pf[s][3]};
#pragma unroll
      for (int j = 0; j < NT_O; j += 2) {
        const int krow = 16 * s + (lane & 7) + ((lane >> 3) & 1) * 8;
        const int ncol = 8 * (j + (lane >> 4));
        uint32_t b0, b1, b2, b3;
        ldsm_x4_t(smem_u32(vb + krow * LDS + ncol), b0, b1, b2, b3);
        mma_bf16_16816(o[j], a, b0, b1);
        mma_bf16_16816(o[j + 1], a, b2, b3);
      }
    }
    __syncthreads();
  }
  // finalize
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    l_r[r] += __shfl_xor_sync(0xffffffffu, l_r[r], 1);
    l_r[r] += __shfl_xor_sync(0xffffffffu, l_r[r], 2);
  }
  const float inv0 = 1.f / l_r[0], inv1 = 1.f / l_r[1];
  const int row0 = q0 + warp * 16 + (lane >> 2);
  const int64_t ldo = static_cast<int64_t>(heads) * HD;
  __nv_bfloat16* go = out + static_cast<int64_t>(s_begin) * ldo + head * HD + 2 * (lane & 3);
#pragma unroll
  for (int j = 0; j < NT_O; ++j) {
    if (row0 < len)
      *reinterpret_cast<uint32_t*>(go + static_cast<int64_t>(row0) * ldo + 8 * j) =
          pack_bf16x2(o[j][0] * inv0, o[j][1] * inv0);
    if (row0 + 8 < len)
      *reinterpret_cast<uint32_t*>(go + static_cast<int64_t>(row0 + 8) * ldo + 8 * j) =
          pack_bf16x2(o[j][2] * inv1, o[j][3] * inv1);
  }
}

template <int HD>
static int launch_attn_mma(const void* qkv, void* out, const int32_t* cu, int n_seq, int max_s, int heads,
                           float scale, cudaStream_t stream) {
  constexpr int LDS = HD + 8;
  const int smem = (kAttnBQ + 4 * kAttnBKV) * LDS * 2;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(attn_fwd_mma<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return set_cuda_error(e, "attention: cudaFuncSetAttribute");
    attr = true;
  }
  dim3 grid((max_s + kAttnBQ - 1) / kAttnBQ, n_seq, heads);
  attn_fwd_mma<HD><<<grid, kAttnThreads, smem, stream>>>(
      reinterpret_cast<const __nv_bfloat16*>(qkv), reinterpret_cast<__nv_bfloat16*>(out), cu, heads,
      scale * 1.4426950408889634f);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? MMK_OK : set_cuda_error(e, "attention: launch");
}

}  // namespace mmk

using namespace mmk;

namespace mmk {
template <int HD>
int launch_attn_tc(const void* qkv, void* out, const int32_t* cu, int n_seq, int max_s, int heads, float scale,
                   int64_t total_rows, cudaStream_t stream);
}

extern "C" int mmk_attention_varlen_bf16(const void* qkv, void* out, const int32_t* cu_seqlens, int32_t n_seq,
                                         int32_t max_seqlen, int32_t total_tokens, int32_t heads, int32_t head_dim,
                                         float scale, cudaStream_t stream) {
  if (n_seq < 0 || heads <= 0 || max_seqlen < 0 || total_tokens < 0)
    return set_error(MMK_ERR_ARG, "attention: bad shape");
  if (head_dim != 64 && head_dim != 80)
    return set_error(MMK_ERR_UNSUPPORTED, "attention: head_dim %d not in {64, 80}", head_dim);
  if (n_seq == 0 || max_seqlen == 0 || total_tokens == 0) return MMK_OK;
  if (n_seq > 65535 || heads > 65535) return set_error(MMK_ERR_UNSUPPORTED, "attention: too many sequences/heads");
  static const bool legacy = getenv("MMK_ATTN_LEGACY") != nullptr;  // A/B against the mma.sync baseline
  if (legacy) {
    if (head_dim == 64) return launch_attn_mma<64>(qkv, out, cu_seqlens, n_seq, max_seqlen, heads, scale, stream);
    return launch_attn_mma<80>(qkv, out, cu_seqlens, n_seq, max_seqlen, heads, scale, stream);
  }
  if (head_dim == 64)
    return launch_attn_tc<64>(qkv, out, cu_seqlens, n_seq, max_seqlen, heads, scale, total_tokens, stream);
  return launch_attn_tc<80>(qkv, out, cu_seqlens, n_seq, max_seqlen, heads, scale, total_tokens, stream);
}
