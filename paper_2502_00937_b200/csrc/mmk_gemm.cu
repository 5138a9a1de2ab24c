// mmk_gemm.cu — persistent, warp-specialised tcgen05 GEMM with fused epilogues.
//
//   D[M, N] = A[M, K] · B[N, K]^T      A, B bf16 K-major (activations · nn.Linear weights)
//
// Replaces the modelled `LatencyProfile.encode_latency` (reference
// pkg/src/lmmsim/profiles.py:136-145) with the encoder's real dense contractions:
// patch-embed (K2), QKV (K4), O-proj + residual (K6), FC1 + GELU (K7), FC2 + residual (K8).
//
// Two kernels share the structure (persistent over output tiles, warp-specialised):
//   warp 0      TMA producer: A/B k-blocks -> STAGES-deep smem ring (128B swizzle)
//   warp 1      MMA issuer:   one elected thread issues tcgen05.mma into TMEM
//   warp 2      TMEM allocator (double-buffered fp32 accumulator)
//   warps 4..11 epilogue:     tcgen05.ld -> bias / activation / gated residual -> global
// Epilogue of tile i overlaps the MMAs of tile i+1 via the two accumulator buffers.
//   gemm_bf16_tcgen05      one CTA per SM, 128 x BN tiles, M=128 MMAs (small or odd-N problems)
//   gemm_bf16_tcgen05_2sm  CTA pairs (clusters of 2, one TPC): 256 x 256 tiles with
//                          tcgen05.mma.cta_group::2 (M=256), each CTA loading its 128 rows of A
//                          and half of B, completions counted on the leader CTA's barriers;
//                          bf16 outputs leave through 128B-swizzled smem + TMA stores, the fp32
//                          residual streams through a 2-slot TMA ring per epilogue warp.
#include "sm100_common.cuh"
#include <cstdlib>
#include "mmk_internal.h"

namespace mmk {

constexpr int kGemmBM = 128;
constexpr int kGemmBK = 64;
constexpr int kGemmThreads = 384;  // 4 control warps + 8 epilogue warps

template <int BN, int STAGES>
struct GemmSmem {
  static constexpr int kABytes = kGemmBM * kGemmBK * 2;
  static constexpr int kBBytes = BN * kGemmBK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kBarOffset = STAGES * kStageBytes;
  static constexpr int kTotal = kBarOffset + 256 + 1024;  // + barriers + alignment slack
};

// GELU(x) = x/2 (1 + erf(x / sqrt 2)), erf by Abramowitz-Stegun 7.1.26 (|error| < 1.5e-7, far
// below the bf16 output rounding): one MUFU reciprocal, one MUFU exp2, 9 FMA-pipe ops.
MMK_DEV float gelu_erf(float x) {
  const float z = fabsf(x) * 0.70710678118654752f;
  float t;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(t) : "f"(fmaf(0.3275911f, z, 1.0f)));
  float p = fmaf(1.061405429f, t, -1.453152027f);
  p = fmaf(p, t, 1.421413741f);
  p = fmaf(p, t, -0.284496736f);
  p = fmaf(p, t, 0.254829592f);
  p *= t;
  float e;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(-z * z * 1.4426950408889634f));
  const float erf_abs = fmaf(-p, e, 1.0f);
  return 0.5f * x * (1.0f + copysignf(erf_abs, x));
}
// x * sigmoid(1.702 x) with one MUFU ex2 and one MUFU rcp (an IEEE division here cost ~2x the
// epilogue time); x -> -inf gives x * rcp(inf) = -0, x -> +inf gives x * rcp(1) = x
MMK_DEV float quick_gelu(float x) {
  float e, r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(-2.4554669595930157f * x));  // 2^(-1.702 log2(e) x)
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(1.0f + e));
  return x * r;
}

// tanh-approximated GELU (gelu_pytorch_tanh, SigLIP): 0.5 x (1 + tanh(sqrt(2/pi) (x + 0.044715 x^3)))
// with tanh as 1 - 2 / (1 + e^{2u}) (one MUFU ex2, one MUFU rcp); saturates cleanly at +-inf.
MMK_DEV float gelu_tanh(float x) {
  const float u = 0.7978845608028654f * fmaf(0.044715f * x, x * x, x);
  float e, r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(2.8853900817779268f * u));  // e^{2u} = 2^{2u log2 e}
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(1.0f + e));
  return 0.5f * x * (2.0f - 2.0f * r);  // 1 + tanh(u) = 2 - 2 / (1 + e^{2u})
}

// Paired forms (FFMA2 / FMUL2 on the FMA pipe, half the issue slots; same math as above).
MMK_DEV float2 gelu_erf2(float2 x) {
  const float2 z = __fmul2_rn(make_float2(fabsf(x.x), fabsf(x.y)), make_float2(0.70710678118654752f, 0.70710678118654752f));
  const float2 den = __ffma2_rn(make_float2(0.3275911f, 0.3275911f), z, make_float2(1.0f, 1.0f));
  float2 t;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(t.x) : "f"(den.x));
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(t.y) : "f"(den.y));
  float2 p = __ffma2_rn(make_float2(1.061405429f, 1.061405429f), t, make_float2(-1.453152027f, -1.453152027f));
  p = __ffma2_rn(p, t, make_float2(1.421413741f, 1.421413741f));
  p = __ffma2_rn(p, t, make_float2(-0.284496736f, -0.284496736f));
  p = __ffma2_rn(p, t, make_float2(0.254829592f, 0.254829592f));
  p = __fmul2_rn(p, t);
  const float2 arg = __fmul2_rn(__fmul2_rn(z, z), make_float2(-1.4426950408889634f, -1.4426950408889634f));
  float2 e;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e.x) : "f"(arg.x));
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e.y) : "f"(arg.y));
  const float2 erf_abs = __ffma2_rn(make_float2(-p.x, -p.y), e, make_float2(1.0f, 1.0f));
  const float2 one_p = make_float2(1.0f + copysignf(erf_abs.x, x.x), 1.0f + copysignf(erf_abs.y, x.y));
  return __fmul2_rn(__fmul2_rn(make_float2(0.5f, 0.5f), x), one_p);
}

template <int EPI>
MMK_DEV float2 apply_act2(float2 v) {
  if constexpr (EPI == MMK_EPI_BF16_GELU) return gelu_erf2(v);
  else if constexpr (EPI == MMK_EPI_BF16_QUICKGELU) return make_float2(quick_gelu(v.x), quick_gelu(v.y));
  else if constexpr (EPI == MMK_EPI_BF16_GELU_TANH) return make_float2(gelu_tanh(v.x), gelu_tanh(v.y));
  else return v;
}

template <int EPI>
MMK_DEV float apply_act(float v) {
  if constexpr (EPI == MMK_EPI_BF16_GELU) return gelu_erf(v);
  else if constexpr (EPI == MMK_EPI_BF16_QUICKGELU) return quick_gelu(v);
  else if constexpr (EPI == MMK_EPI_BF16_GELU_TANH) return gelu_tanh(v);
  else return v;
}

// LayerNorm folded into the GEMMs around it (the LN between a residual update and the GEMM that
// consumes the normalised rows):
//   producer (RESID_F32): besides the fp32 residual, the bf16 copy of the new row goes to `aux`
//     and each 32-column chunk's (mean, M2) to stats_out[row][col / 32] (exact two-pass inside
//     the chunk; mmk_ln_stats_finalize merges the chunks, Chan's formula, into (mu, rstd)).
//   consumer (bf16 epilogues): A = that bf16 copy, B = W (x) gamma; out = act(rstd * (acc - mu *
//     c1[n]) + bias[n]) with c1[n] = sum_k W'[n,k] and bias = beta W^T + b (host-prepared).
struct LnFold {
  float2* stats_out;   // producer: [M][N/32] (mean, M2) per 32-column chunk, or null
  const float2* mr;    // consumer: [M] (mu, rstd), or null
  const float* c1;     // consumer: [N]
};

MMK_DEV void chunk_stats(const float (&v)[32], float2* dst) {
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 32; ++i) s += v[i];
  const float mean = s * (1.f / 32.f);
  float m2 = 0.f;
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    const float d = v[i] - mean;
    m2 = fmaf(d, d, m2);
  }
  *dst = make_float2(mean, m2);
}

// Tile order of the persistent CTA-pair kernel: group_m = 1 is N-major (the ~74 clusters in
// flight share ~1.5 A blocks, each streams its own weight tile); group_m > 1 walks down group_m M
// blocks before moving to the next N tile, so in-flight clusters share ~group_m A blocks and
// ~74/group_m weight tiles.  With InternViT's 61-82 MB weights the N-major order re-streamed them
// from DRAM for every M block (7-15x the algorithmic bytes, ncu); grouping by 16 is +0.7 % there
// and -1.5 % on Mllama's 3-13 MB weights (same box, alternating), hence the host's choice by
// weight size.
MMK_DEV void grouped_tile(int tile, int n_tiles_m, int n_tiles_n, int group_m, int& mb, int& nb) {
  const int per_group = group_m * n_tiles_n;
  const int first_m = (tile / per_group) * group_m;
  const int gm = min(group_m, n_tiles_m - first_m);
  const int local = tile - (tile / per_group) * per_group;
  mb = first_m + local % gm;
  nb = local / gm;
}

// Fused epilogue for 32 consecutive accumulator columns of one output row (thread-owned row).
template <int EPI>
MMK_DEV void epilogue_chunk(const uint32_t (&r)[32], int row, int col, const float* __restrict__ bias, void* out,
                            int64_t ldo, float gate, __nv_bfloat16* __restrict__ aux, int64_t ld_aux,
                            const LnFold& lf, float2 mr, int n_total) {
  float v[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
  if (lf.c1 != nullptr) {  // folded LayerNorm: rstd * (acc - mu * c1) + bias
#pragma unroll
    for (int i = 0; i < 32; i += 4) {
      const float4 c4 = __ldg(reinterpret_cast<const float4*>(lf.c1 + col + i));
      const float4 b4 = __ldg(reinterpret_cast<const float4*>(bias + col + i));
      v[i] = fmaf(mr.y, fmaf(-mr.x, c4.x, v[i]), b4.x);
      v[i + 1] = fmaf(mr.y, fmaf(-mr.x, c4.y, v[i + 1]), b4.y);
      v[i + 2] = fmaf(mr.y, fmaf(-mr.x, c4.z, v[i + 2]), b4.z);
      v[i + 3] = fmaf(mr.y, fmaf(-mr.x, c4.w, v[i + 3]), b4.w);
    }
  } else if (bias != nullptr) {
#pragma unroll
    for (int i = 0; i < 32; i += 4) {
      const float4 b4 = __ldg(reinterpret_cast<const float4*>(bias + col + i));
      v[i] += b4.x; v[i + 1] += b4.y; v[i + 2] += b4.z; v[i + 3] += b4.w;
    }
  }
  if constexpr (EPI == MMK_EPI_F32) {
    float* o = reinterpret_cast<float*>(out) + static_cast<int64_t>(row) * ldo + col;
#pragma unroll
    for (int i = 0; i < 32; i += 4)
      *reinterpret_cast<float4*>(o + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
  } else if constexpr (EPI == MMK_EPI_RESID_F32) {
    float* o = reinterpret_cast<float*>(out) + static_cast<int64_t>(row) * ldo + col;
#pragma unroll
    for (int i = 0; i < 32; i += 4) {
      float4 rr = *reinterpret_cast<const float4*>(o + i);
      rr.x = fmaf(gate, v[i], rr.x);
      rr.y = fmaf(gate, v[i + 1], rr.y);
      rr.z = fmaf(gate, v[i + 2], rr.z);
      rr.w = fmaf(gate, v[i + 3], rr.w);
      v[i] = rr.x; v[i + 1] = rr.y; v[i + 2] = rr.z; v[i + 3] = rr.w;
      *reinterpret_cast<float4*>(o + i) = rr;
    }
    if (aux != nullptr) {
      __nv_bfloat16* ao = aux + static_cast<int64_t>(row) * ld_aux + col;
#pragma unroll
      for (int i = 0; i < 32; i += 8)
        st_global_v4(ao + i, pack_bf16x2(v[i], v[i + 1]), pack_bf16x2(v[i + 2], v[i + 3]),
                     pack_bf16x2(v[i + 4], v[i + 5]), pack_bf16x2(v[i + 6], v[i + 7]));
    }
    if (lf.stats_out != nullptr) chunk_stats(v, lf.stats_out + static_cast<int64_t>(row) * (n_total / 32) + col / 32);
  } else {
    __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(out) + static_cast<int64_t>(row) * ldo + col;
#pragma unroll
    for (int i = 0; i < 32; i += 8)
      st_global_v4(o + i, pack_bf16x2(apply_act<EPI>(v[i]), apply_act<EPI>(v[i + 1])),
                   pack_bf16x2(apply_act<EPI>(v[i + 2]), apply_act<EPI>(v[i + 3])),
                   pack_bf16x2(apply_act<EPI>(v[i + 4]), apply_act<EPI>(v[i + 5])),
                   pack_bf16x2(apply_act<EPI>(v[i + 6]), apply_act<EPI>(v[i + 7])));
  }
}

template <int BN, int STAGES, int EPI>
__global__ void __launch_bounds__(kGemmThreads, 1)
gemm_bf16_tcgen05(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b,
                  int M, int N, int K, const float* __restrict__ bias, void* __restrict__ out,
                  int64_t ldo, float gate, __nv_bfloat16* __restrict__ aux, int64_t ld_aux, LnFold lf) {
  using S = GemmSmem<BN, STAGES>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + S::kBarOffset);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* tfull_bar = empty_bar + STAGES;  // [2]
  uint64_t* tempty_bar = tfull_bar + 2;      // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const uint32_t warp = warp_id_uniform();
  const uint32_t lane = lane_id();
  const int n_tiles_n = (N + BN - 1) / BN;
  const int n_tiles_m = (M + kGemmBM - 1) / kGemmBM;
  const int n_tiles = n_tiles_m * n_tiles_n;
  const int num_kb = (K + kGemmBK - 1) / kGemmBK;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmap_a);
    tma_prefetch_desc(&tmap_b);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull_bar[b], 1);
      mbar_init(&tempty_bar[b], 8);  // one arrive per epilogue warp
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<2 * BN>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  griddep_wait();  // setup above overlaps the previous kernel's tail (PDL)
  griddep_launch_dependents();

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (warp-uniform)
    const uint64_t pol_b = l2_policy_evict_last();  // weights: re-read by every M tile
    int stage = 0;
    uint32_t phase = 0;
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
      const int m0 = (tile / n_tiles_n) * kGemmBM;
      const int n0 = (tile % n_tiles_n) * BN;
      for (int kb = 0; kb < num_kb; ++kb) {
        mbar_wait(&empty_bar[stage], phase ^ 1);
        uint8_t* sa = smem + stage * S::kStageBytes;
        uint8_t* sb = sa + S::kABytes;
        if (elect_one()) {
          mbar_arrive_expect_tx(&full_bar[stage], S::kStageBytes);
          tma_load_2d(&tmap_a, &full_bar[stage], sa, kb * kGemmBK, m0);
          tma_load_2d_hint(&tmap_b, &full_bar[stage], sb, kb * kGemmBK, n0, pol_b);
        }
        __syncwarp();
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (warp-uniform,
    // one elected lane issues: descriptors stay in uniform registers)
    constexpr uint32_t idesc = umma_idesc_bf16_f32(kGemmBM, BN);
    const uint32_t smem_base = smem_u32(smem);
    int stage = 0;
    uint32_t phase = 0;
    int t = 0;
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++t) {
      const int acc = t & 1;
      const uint32_t acc_phase = (t >> 1) & 1;
      mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * BN;
      for (int kb = 0; kb < num_kb; ++kb) {
        mbar_wait(&full_bar[stage], phase);
        tc_fence_after();
        const uint32_t a_addr = smem_base + stage * S::kStageBytes;
        const uint64_t adesc = umma_desc_sw128_kmajor(a_addr);
        const uint64_t bdesc = umma_desc_sw128_kmajor(a_addr + S::kABytes);
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < kGemmBK / 16; ++k) {
            // +32 bytes per K=16 step inside the 128-byte swizzle row (desc unit = 16 B)
            umma_bf16_ss(d_tmem, adesc + 2 * k, bdesc + 2 * k, idesc, (kb | k) != 0);
          }
          umma_commit(&empty_bar[stage]);  // frees the smem slot when these MMAs retire
        }
        __syncwarp();
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      if (elect_one()) umma_commit(&tfull_bar[acc]);  // accumulator ready for the epilogue
      __syncwarp();
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue
    const uint32_t q = warp & 3;              // TMEM lane quarter this warp may access
    const uint32_t half = (warp - 4) >> 2;    // column half of the BN tile
    constexpr int kColsPerWarp = BN / 2;
    int t = 0;
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++t) {
      const int acc = t & 1;
      const uint32_t acc_phase = (t >> 1) & 1;
      const int m0 = (tile / n_tiles_n) * kGemmBM;
      const int n0 = (tile % n_tiles_n) * BN;
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const int row = m0 + q * 32 + lane;
      const bool row_ok = row < M;
      const float2 mr = lf.mr != nullptr ? lf.mr[row_ok ? row : M - 1] : make_float2(0.f, 1.f);
#pragma unroll 1
      for (int c = 0; c < kColsPerWarp / 32; ++c) {
        const int col_in_tile = half * kColsPerWarp + c * 32;
        const int col = n0 + col_in_tile;
        uint32_t r[32];
        tmem_ld_32x32b_x32(tmem_base + ((q * 32u) << 16) + acc * BN + col_in_tile, r);
        tmem_ld_wait();
        if (!row_ok || col >= N) continue;
        epilogue_chunk<EPI>(r, row, col, bias, out, ldo, gate, aux, ld_aux, lf, mr, N);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty_bar[acc]);
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc<2 * BN>(tmem_base);
}

// ------------------------------------------------------------------ CTA-pair variant
// cta_group::2: a cluster of 2 CTAs (one per SM of a TPC) computes a 256 x BN2 tile with
// tcgen05.mma M=256.  Each CTA stages its own 128 rows of A and its own BN2/2 rows of B per
// k-block (half the shared-memory traffic of the single-CTA kernel per SM); the leader CTA issues
// the MMAs, which read both CTAs' smem and write both CTAs' TMEM (128 lanes x BN2 cols each).
// Barriers: `full` lives in the leader (TMA completions of both CTAs counted there), `empty` and
// `tfull` are multicast by the leader's tcgen05.commit to both CTAs, `tempty` lives in the leader
// and counts the epilogue warps of both CTAs.
constexpr int kGemm2BN = 256;
template <int STAGES>
struct Gemm2Smem {
  static constexpr int kABytes = 128 * kGemmBK * 2;             // this CTA's 128 rows of A
  static constexpr int kBBytes = (kGemm2BN / 2) * kGemmBK * 2;  // this CTA's half of B
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kEpiOffset = STAGES * kStageBytes;
  // 8 warps x 2 x [32 rows][128 B]: bf16 output staging, or the residual ring (2 fp32 chunks of
  // [32 rows][32 cols] per warp; 3- and 4-slot rings with 4 / 3 mainloop stages measured slower)
  static constexpr int kEpiBytes = 8 * 2 * 4096;
  static constexpr int kBarOffset = kEpiOffset + kEpiBytes;
  static constexpr int kTotal = kBarOffset + 512 + 1024;
};

// bf16 epilogue through shared memory + TMA store: 32 rows x 64 cols per warp per step, staged in
// a 128B-swizzled [32][128 B] buffer (conflict-free 16-byte st.shared), written by one bulk
// tensor store; two buffers per warp so the store of one chunk overlaps the next chunk.
template <int EPI>
MMK_DEV void epilogue_bf16_tma(const uint32_t (&r0)[32], const uint32_t (&r1)[32], int col, int row0, uint32_t lane,
                               const float* __restrict__ bias, uint8_t* buf, const CUtensorMap* tmap_out,
                               const float* __restrict__ c1 = nullptr, float2 mr = make_float2(0.f, 1.f)) {
  uint32_t w[32];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const uint32_t (&r)[32] = h ? r1 : r0;
#pragma unroll
    for (int i = 0; i < 32; i += 4) {
      float2 a = make_float2(__uint_as_float(r[i]), __uint_as_float(r[i + 1]));
      float2 b = make_float2(__uint_as_float(r[i + 2]), __uint_as_float(r[i + 3]));
      if (c1 != nullptr) {  // folded LayerNorm: rstd * (acc - mu * c1) + bias
        const float4 c4 = __ldg(reinterpret_cast<const float4*>(c1 + col + 32 * h + i));
        const float4 b4 = __ldg(reinterpret_cast<const float4*>(bias + col + 32 * h + i));
        const float2 nmu = make_float2(-mr.x, -mr.x), rs = make_float2(mr.y, mr.y);
        a = __ffma2_rn(rs, __ffma2_rn(nmu, make_float2(c4.x, c4.y), a), make_float2(b4.x, b4.y));
        b = __ffma2_rn(rs, __ffma2_rn(nmu, make_float2(c4.z, c4.w), b), make_float2(b4.z, b4.w));
      } else if (bias != nullptr) {  // one 16-byte broadcast load per 4 columns
        const float4 b4 = __ldg(reinterpret_cast<const float4*>(bias + col + 32 * h + i));
        a = __fadd2_rn(a, make_float2(b4.x, b4.y));
        b = __fadd2_rn(b, make_float2(b4.z, b4.w));
      }
      a = apply_act2<EPI>(a);
      b = apply_act2<EPI>(b);
      w[16 * h + i / 2] = pack_bf16x2(a.x, a.y);
      w[16 * h + i / 2 + 1] = pack_bf16x2(b.x, b.y);
    }
  }
  if (lane == 0) tma_store_wait_read<1>();  // this buffer's previous store has been read out
  __syncwarp();
#pragma unroll
  for (int j = 0; j < 8; ++j) {  // 16-byte chunk j = columns 8j..8j+7 of this row
    const uint32_t dst = smem_u32(buf + lane * 128 + ((j ^ (lane & 7)) << 4));
    asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(dst), "r"(w[4 * j]), "r"(w[4 * j + 1]),
                 "r"(w[4 * j + 2]), "r"(w[4 * j + 3])
                 : "memory");
  }
  fence_proxy_async();
  __syncwarp();
  if (lane == 0) {
    tma_store_2d(tmap_out, buf, col, row0);
    tma_store_commit();
  }
}

template <int STAGES, int EPI, bool RES_TMA = false>
__global__ void __launch_bounds__(kGemmThreads, 1)
gemm_bf16_tcgen05_2sm(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b,
                      const __grid_constant__ CUtensorMap tmap_out, int M, int N, int K, const float* __restrict__ bias, void* __restrict__ out, int64_t ldo,
                      float gate, __nv_bfloat16* __restrict__ aux, int64_t ld_aux, LnFold lf, int group_m) {
  using S = Gemm2Smem<STAGES>;
  constexpr int BN = kGemm2BN;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + S::kBarOffset);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* tfull_bar = empty_bar + STAGES;  // [2]
  uint64_t* tempty_bar = tfull_bar + 2;      // [2]
  uint64_t* res_bar = tempty_bar + 2;        // [8 warps][2 slots] residual TMA loads (RES_TMA)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(res_bar + 32);

  const uint32_t warp = warp_id_uniform();
  const uint32_t lane = lane_id();
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  // N % 64 == 0: the last N tile may be partial (InternViT d 3200, SigLIP 1152): B rows past N
  // load as zeros (TMA out-of-bounds fill), stores past N are clipped by the output map or skipped
  const int n_tiles_n = (N + BN - 1) / BN;
  const int n_tiles_m = (M + 255) / 256;
  const int n_tiles = n_tiles_m * n_tiles_n;
  const int num_kb = (K + kGemmBK - 1) / kGemmBK;
  const int first = static_cast<int>(cluster_id_x()), step = static_cast<int>(n_clusters_x());

  if (warp == 0 && elect_one()) {
    tma_prefetch_desc(&tmap_a);
    tma_prefetch_desc(&tmap_b);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull_bar[b], 1);
      mbar_init(&tempty_bar[b], 16);  // 8 epilogue warps x 2 CTAs
    }
    if (RES_TMA) {
      tma_prefetch_desc(&tmap_out);
      for (int i = 0; i < 16; ++i) mbar_init(&res_bar[i], 1);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc_2sm<2 * BN>(tmem_slot);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  griddep_wait();  // setup above overlaps the previous kernel's tail (PDL)
  griddep_launch_dependents();

  if (warp == 0) {
    // ------------------------------------------------ TMA producer (both CTAs)
    // A tiles are re-read by the N/256 clusters working on the same M block (normal policy);
    // weights are re-read by every M block (keep in L2)
    const uint64_t pol_a = l2_policy_evict_normal();
    const uint64_t pol_b = l2_policy_evict_last();
    int stage = 0;
    uint32_t phase = 0;
    for (int tile = first; tile < n_tiles; tile += step) {
      int mb, nb;
      grouped_tile(tile, n_tiles_m, n_tiles_n, group_m, mb, nb);
      const int m0 = mb * 256 + rank * 128;
      const int n0 = nb * BN + rank * (BN / 2);
      for (int kb = 0; kb < num_kb; ++kb) {
        mbar_wait(&empty_bar[stage], phase ^ 1);
        uint8_t* sa = smem + stage * S::kStageBytes;
        uint8_t* sb = sa + S::kABytes;
        const uint32_t fb = mapa_shared(smem_u32(&full_bar[stage]), 0);  // leader's barrier
        if (elect_one()) {
          if (leader) mbar_arrive_expect_tx(&full_bar[stage], 2 * S::kStageBytes);
          tma_load_2d_2sm(&tmap_a, fb, sa, kb * kGemmBK, m0, pol_a);
          tma_load_2d_2sm(&tmap_b, fb, sb, kb * kGemmBK, n0, pol_b);
        }
        __syncwarp();
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer (leader CTA only)
    if (leader) {
      constexpr uint32_t idesc = umma_idesc_bf16_f32(256, BN);
      const uint32_t smem_base = smem_u32(smem);
      int stage = 0;
      uint32_t phase = 0;
      int t = 0;
      for (int tile = first; tile < n_tiles; tile += step, ++t) {
        const int acc = t & 1;
        const uint32_t acc_phase = (t >> 1) & 1;
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint32_t a_addr = smem_base + stage * S::kStageBytes;
          const uint64_t adesc = umma_desc_sw128_kmajor(a_addr);
          const uint64_t bdesc = umma_desc_sw128_kmajor(a_addr + S::kABytes);
          if (elect_one()) {
#pragma unroll
            for (int k = 0; k < kGemmBK / 16; ++k)
              umma_bf16_ss_2sm(d_tmem, adesc + 2 * k, bdesc + 2 * k, idesc, (kb | k) != 0);
            umma_commit_2sm(&empty_bar[stage], 0x3);
          }
          __syncwarp();
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        if (elect_one()) umma_commit_2sm(&tfull_bar[acc], 0x3);
        __syncwarp();
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------ epilogue (both CTAs, own 128 rows)
    constexpr bool kTmaStore = EPI == MMK_EPI_BF16 || EPI == MMK_EPI_BF16_GELU || EPI == MMK_EPI_BF16_QUICKGELU ||
                               EPI == MMK_EPI_BF16_GELU_TANH;
    const uint32_t q = warp & 3;
    const uint32_t half = (warp - 4) >> 2;
    constexpr int kColsPerWarp = BN / 2;
    const uint32_t tempty_leader0 = mapa_shared(smem_u32(&tempty_bar[0]), 0);
    uint8_t* ebuf = smem + S::kEpiOffset + (warp - 4) * 2 * 4096;
    int sb = 0;
    int t = 0;
    for (int tile = first; tile < n_tiles; tile += step, ++t) {
      const int acc = t & 1;
      const uint32_t acc_phase = (t >> 1) & 1;
      int mb, nb;
      grouped_tile(tile, n_tiles_m, n_tiles_n, group_m, mb, nb);
      const int m0 = mb * 256 + rank * 128;
      const int n0 = nb * BN;
      if constexpr (RES_TMA) {
        // residual chunks 0 and 1 of this tile into the warp's two slots (chunks 2, 3 follow as
        // the slots drain); issued before waiting for the accumulator so they overlap the MMAs
        if (lane == 0) {
          tma_store_wait_read<0>();  // the previous tile's stores have left both slots
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            mbar_arrive_expect_tx(&res_bar[(warp - 4) * 2 + c], 4096);
            tma_load_2d(&tmap_out, &res_bar[(warp - 4) * 2 + c], ebuf + c * 4096,
                        n0 + half * kColsPerWarp + c * 32, m0 + static_cast<int>(q) * 32);
          }
        }
        __syncwarp();
      }
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const uint32_t tm_row = tmem_base + ((q * 32u) << 16) + acc * BN;
      if constexpr (kTmaStore) {
        const int mrow = m0 + static_cast<int>(q) * 32 + static_cast<int>(lane);
        const float2 mr = lf.mr != nullptr ? lf.mr[mrow < M ? mrow : M - 1] : make_float2(0.f, 1.f);
#pragma unroll 1
        for (int c = 0; c < kColsPerWarp / 64; ++c) {
          const int col_in_tile = half * kColsPerWarp + c * 64;
          uint32_t r0[32], r1[32];
          tmem_ld_32x32b_x32(tm_row + col_in_tile, r0);
          tmem_ld_32x32b_x32(tm_row + col_in_tile + 32, r1);
          tmem_ld_wait();
          if (c == kColsPerWarp / 64 - 1) {  // accumulator fully read: release it early
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_remote(tempty_leader0 + acc * 8);
          }
          if (n0 + col_in_tile >= N) continue;  // past a partial last N tile (no store, same buffer next)
          epilogue_bf16_tma<EPI>(r0, r1, n0 + col_in_tile, m0 + static_cast<int>(q) * 32, lane, bias,
                                 ebuf + sb * 4096, &tmap_out, lf.c1, mr);
          sb ^= 1;
        }
      } else if constexpr (RES_TMA) {
        // fp32 residual read-modify-write through shared memory: 32x32 fp32 chunks of the warp's
        // residual slice stream through two slots (chunks 0, 1 TMA-loaded while the tile's MMAs
        // run), updated in place (128B-swizzled rows, conflict-free 16-byte accesses) and
        // TMA-stored back; a slot is refilled with chunk c+2 once the store of chunk c has read it.
        const int row = m0 + q * 32 + lane;
        const bool row_ok = row < M;
#pragma unroll 1
        for (int c = 0; c < kColsPerWarp / 32; ++c) {
          const int col_in_tile = half * kColsPerWarp + c * 32;
          const int col = n0 + col_in_tile;
          uint32_t r[32];
          tmem_ld_32x32b_x32(tm_row + col_in_tile, r);
          tmem_ld_wait();
          if (c == kColsPerWarp / 32 - 1) {  // accumulator fully read: release it early
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_remote(tempty_leader0 + acc * 8);
          }
          const int slot = c & 1;
          mbar_wait(&res_bar[(warp - 4) * 2 + slot], (2 * t + (c >> 1)) & 1);  // two uses per slot per tile
          uint8_t* rowp = ebuf + slot * 4096 + lane * 128;
          const bool col_ok = col < N;  // chunks past a partial last N tile: zeros in, store clipped
          float v[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
          if (bias != nullptr && col_ok) {
#pragma unroll
            for (int i = 0; i < 32; i += 4) {
              const float4 b4 = __ldg(reinterpret_cast<const float4*>(bias + col + i));
              v[i] += b4.x; v[i + 1] += b4.y; v[i + 2] += b4.z; v[i + 3] += b4.w;
            }
          }
#pragma unroll
          for (int j = 0; j < 8; ++j) {  // 16-byte chunk j = columns 4j..4j+3 of this row
            float4* p4 = reinterpret_cast<float4*>(rowp + ((j ^ (lane & 7)) << 4));
            float4 rr = *p4;
            rr.x = fmaf(gate, v[4 * j], rr.x);
            rr.y = fmaf(gate, v[4 * j + 1], rr.y);
            rr.z = fmaf(gate, v[4 * j + 2], rr.z);
            rr.w = fmaf(gate, v[4 * j + 3], rr.w);
            *p4 = rr;
            v[4 * j] = rr.x; v[4 * j + 1] = rr.y; v[4 * j + 2] = rr.z; v[4 * j + 3] = rr.w;
          }
          if (lf.stats_out != nullptr && row_ok && col_ok)
            chunk_stats(v, lf.stats_out + static_cast<int64_t>(row) * (N / 32) + col / 32);
          fence_proxy_async();
          __syncwarp();
          if (aux != nullptr && col_ok) {
            // bf16 copy of the updated 32x32 chunk, read back from the slot transposed so that a
            // warp store covers 8 whole 64-byte row segments (a row per lane would scatter each
            // store over 32 rows): lane = 4 r + cc writes columns 8cc..8cc+7 of row 8k + r
            const int rr0 = static_cast<int>(lane >> 2), cc = static_cast<int>(lane & 3);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              const int rr = 8 * kk + rr0;
              const uint8_t* src = ebuf + slot * 4096 + rr * 128;
              const float4 lo = *reinterpret_cast<const float4*>(src + (((2 * cc) ^ (rr & 7)) << 4));
              const float4 hi = *reinterpret_cast<const float4*>(src + (((2 * cc + 1) ^ (rr & 7)) << 4));
              const int grow = m0 + static_cast<int>(q) * 32 + rr;
              if (grow < M)
                st_global_v4(aux + static_cast<int64_t>(grow) * ld_aux + col + 8 * cc, pack_bf16x2(lo.x, lo.y),
                             pack_bf16x2(lo.z, lo.w), pack_bf16x2(hi.x, hi.y), pack_bf16x2(hi.z, hi.w));
            }
            __syncwarp();  // the slot may be refilled after this
          }
          if (lane == 0) {
            tma_store_2d(&tmap_out, ebuf + slot * 4096, col, m0 + static_cast<int>(q) * 32);
            tma_store_commit();
            if (c + 2 < kColsPerWarp / 32) {
              tma_store_wait_read<0>();  // chunk c has left the slot
              mbar_arrive_expect_tx(&res_bar[(warp - 4) * 2 + slot], 4096);
              tma_load_2d(&tmap_out, &res_bar[(warp - 4) * 2 + slot], ebuf + slot * 4096, col + 64,
                          m0 + static_cast<int>(q) * 32);
            }
          }
          __syncwarp();
        }
      } else if constexpr (EPI == MMK_EPI_F32) {
        // fp32 output (patch embedding) through the same two 32x32 fp32 slots: rows staged
        // 128B-swizzled, TMA-stored (rows >= M clipped by the map) — a thread-per-row float4
        // store would scatter every warp store over 32 rows
#pragma unroll 1
        for (int c = 0; c < kColsPerWarp / 32; ++c) {
          const int col_in_tile = half * kColsPerWarp + c * 32;
          const int col = n0 + col_in_tile;
          uint32_t r[32];
          tmem_ld_32x32b_x32(tm_row + col_in_tile, r);
          tmem_ld_wait();
          if (c == kColsPerWarp / 32 - 1) {  // accumulator fully read: release it early
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_remote(tempty_leader0 + acc * 8);
          }
          const int slot = c & 1;
          if (lane == 0) tma_store_wait_read<1>();  // the store that last used this slot has read it
          __syncwarp();
          uint8_t* rowp = ebuf + slot * 4096 + lane * 128;
          float v[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
          if (bias != nullptr && col < N) {
#pragma unroll
            for (int i = 0; i < 32; i += 4) {
              const float4 b4 = __ldg(reinterpret_cast<const float4*>(bias + col + i));
              v[i] += b4.x; v[i + 1] += b4.y; v[i + 2] += b4.z; v[i + 3] += b4.w;
            }
          }
#pragma unroll
          for (int j = 0; j < 8; ++j)
            *reinterpret_cast<float4*>(rowp + ((j ^ (lane & 7)) << 4)) =
                make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
          fence_proxy_async();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&tmap_out, ebuf + slot * 4096, col, m0 + static_cast<int>(q) * 32);
            tma_store_commit();
          }
          __syncwarp();
        }
      } else {
        const int row = m0 + q * 32 + lane;
        const bool row_ok = row < M;
#pragma unroll 1
        for (int c = 0; c < kColsPerWarp / 32; ++c) {
          const int col_in_tile = half * kColsPerWarp + c * 32;
          const int col = n0 + col_in_tile;
          uint32_t r[32];
          tmem_ld_32x32b_x32(tm_row + col_in_tile, r);
          tmem_ld_wait();
          if (!row_ok || col >= N) continue;
          epilogue_chunk<EPI>(r, row, col, bias, out, ldo, gate, aux, ld_aux, lf,
                              lf.mr != nullptr ? lf.mr[row] : make_float2(0.f, 1.f), N);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_remote(tempty_leader0 + acc * 8);
      }
    }
    if constexpr (kTmaStore || RES_TMA || EPI == MMK_EPI_F32) {
      if (lane == 0) tma_store_wait<0>();
      __syncwarp();
    }
  }

  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  if (warp == 2) tmem_dealloc_2sm<2 * BN>(tmem_base);
}

// ------------------------------------------------------------------ host side
template <int BN, int STAGES, int EPI>
static int launch_gemm(const CUtensorMap& ta, const CUtensorMap& tb, int M, int N, int K,
                       const float* bias, void* out, int64_t ldo, float gate, __nv_bfloat16* aux,
                       int64_t ld_aux, const LnFold& lf, cudaStream_t stream) {
  using S = GemmSmem<BN, STAGES>;
  auto kern = gemm_bf16_tcgen05<BN, STAGES, EPI>;
  static std::atomic<uint64_t> attr_done{0};  // per template instance
  if (int rc = ensure_smem_attr(reinterpret_cast<const void*>(kern), S::kTotal, attr_done, "gemm: cudaFuncSetAttribute"))
    return rc;
  const int tiles = ((M + kGemmBM - 1) / kGemmBM) * ((N + BN - 1) / BN);
  const int grid = tiles < num_sms() ? tiles : num_sms();
  cudaError_t e = launch_kernel(kern, dim3(grid), dim3(kGemmThreads), S::kTotal, stream, 1, tiles <= 2 * num_sms(), ta, tb, M, N, K, bias,
                                out, ldo, gate, aux, ld_aux, lf);
  if (e != cudaSuccess) return set_cuda_error(e, "gemm: launch");
  return MMK_OK;
}

template <int BN, int STAGES>
static int dispatch_epi(int epi, const CUtensorMap& ta, const CUtensorMap& tb, int M, int N, int K,
                        const float* bias, void* out, int64_t ldo, float gate, __nv_bfloat16* aux,
                        int64_t ld_aux, const LnFold& lf, cudaStream_t s) {
  switch (epi) {
    case MMK_EPI_BF16: return launch_gemm<BN, STAGES, MMK_EPI_BF16>(ta, tb, M, N, K, bias, out, ldo, gate, aux, ld_aux, lf, s);
    case MMK_EPI_BF16_GELU: return launch_gemm<BN, STAGES, MMK_EPI_BF16_GELU>(ta, tb, M, N, K, bias, out, ldo, gate, aux, ld_aux, lf, s);
    case MMK_EPI_BF16_QUICKGELU: return launch_gemm<BN, STAGES, MMK_EPI_BF16_QUICKGELU>(ta, tb, M, N, K, bias, out, ldo, gate, aux, ld_aux, lf, s);
    case MMK_EPI_BF16_GELU_TANH: return launch_gemm<BN, STAGES, MMK_EPI_BF16_GELU_TANH>(ta, tb, M, N, K, bias, out, ldo, gate, aux, ld_aux, lf, s);
    case MMK_EPI_F32: return launch_gemm<BN, STAGES, MMK_EPI_F32>(ta, tb, M, N, K, bias, out, ldo, gate, aux, ld_aux, lf, s);
    case MMK_EPI_RESID_F32: return launch_gemm<BN, STAGES, MMK_EPI_RESID_F32>(ta, tb, M, N, K, bias, out, ldo, gate, aux, ld_aux, lf, s);
    default: return set_error(MMK_ERR_ARG, "gemm: unknown epilogue %d", epi);
  }
}


template <int STAGES, int EPI, bool RES_TMA = false>
static int launch_gemm_2sm(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& to, int M, int N, int K,
                           const float* bias,
                           void* out, int64_t ldo, float gate, __nv_bfloat16* aux, int64_t ld_aux,
                           const LnFold& lf, int group_m, cudaStream_t stream) {
  using S = Gemm2Smem<STAGES>;
  auto kern = gemm_bf16_tcgen05_2sm<STAGES, EPI, RES_TMA>;
  static std::atomic<uint64_t> attr_done{0};  // per template instance
  if (int rc = ensure_smem_attr(reinterpret_cast<const void*>(kern), S::kTotal, attr_done, "gemm2: cudaFuncSetAttribute"))
    return rc;
  const int tiles = ((M + 255) / 256) * ((N + kGemm2BN - 1) / kGemm2BN);
  const int pairs_max = num_sms() / 2;
  const int pairs = tiles < pairs_max ? tiles : pairs_max;
  cudaError_t e = launch_kernel(kern, dim3(2 * pairs), dim3(kGemmThreads), S::kTotal, stream, 2, tiles <= num_sms(), ta, tb, to, M, N, K,
                                bias, out, ldo, gate, aux, ld_aux, lf, group_m);
  if (e != cudaSuccess) return set_cuda_error(e, "gemm2: launch");
  return MMK_OK;
}

template <int STAGES>
static int dispatch_epi_2sm(int epi, const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& to, int M,
                            int N, int K, const float* bias, void* out, int64_t ldo, float gate,
                            __nv_bfloat16* aux, int64_t ld_aux, const LnFold& lf, int g, cudaStream_t s) {
  switch (epi) {
    case MMK_EPI_BF16: return launch_gemm_2sm<STAGES, MMK_EPI_BF16>(ta, tb, to, M, N, K, bias, out, ldo, gate, aux, ld_aux, lf, g, s);
    case MMK_EPI_BF16_GELU: return launch_gemm_2sm<STAGES, MMK_EPI_BF16_GELU>(ta, tb, to, M, N, K, bias, out, ldo, gate, aux, ld_aux, lf, g, s);
    case MMK_EPI_BF16_QUICKGELU: return launch_gemm_2sm<STAGES, MMK_EPI_BF16_QUICKGELU>(ta, tb, to, M, N, K, bias, out, ldo, gate, aux, ld_aux, lf, g, s);
    case MMK_EPI_BF16_GELU_TANH: return launch_gemm_2sm<STAGES, MMK_EPI_BF16_GELU_TANH>(ta, tb, to, M, N, K, bias, out, ldo, gate, aux, ld_aux, lf, g, s);
    case MMK_EPI_F32: return launch_gemm_2sm<STAGES, MMK_EPI_F32>(ta, tb, to, M, N, K, bias, out, ldo, gate, aux, ld_aux, lf, g, s);
    case MMK_EPI_RESID_F32:
      // the fp32 residual streams through shared memory by TMA (O-proj 0.420 -> 0.365 ms, FC2
      // 1.165 -> 1.137 ms versus a direct read-modify-write from the epilogue registers)
      return launch_gemm_2sm<STAGES, MMK_EPI_RESID_F32, true>(ta, tb, to, M, N, K, bias, out, ldo, gate, aux, ld_aux, lf, g, s);
    default: return set_error(MMK_ERR_ARG, "gemm: unknown epilogue %d", epi);
  }
}
}  // namespace mmk

using namespace mmk;

extern "C" int mmk_gemm_bf16_ln(const void* a, int64_t lda, const void* b, int64_t ldb, int32_t m,
                                int32_t n, int32_t k, int32_t epilogue, const float* bias, void* out,
                                int64_t ldo, float gate, void* aux, int64_t ld_aux, float* ln_stats_out,
                                const float* ln_mr, const float* ln_c1, cudaStream_t stream) {
  if (m < 0 || n <= 0 || k <= 0) return set_error(MMK_ERR_ARG, "gemm: bad shape m=%d n=%d k=%d", m, n, k);
  if (m == 0) return MMK_OK;
  if (n % 32 != 0) return set_error(MMK_ERR_UNSUPPORTED, "gemm: N=%d must be a multiple of 32", n);
  if (lda % 8 != 0 || ldb % 8 != 0 || lda < k || ldb < k)
    return set_error(MMK_ERR_ARG, "gemm: lda/ldb must be >= K and multiples of 8 elements");
  if ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b) | reinterpret_cast<uintptr_t>(out) |
       reinterpret_cast<uintptr_t>(bias)) & 15)
    return set_error(MMK_ERR_ARG, "gemm: pointers (a, b, out, bias) must be 16-byte aligned");
  const bool f32_out = epilogue == MMK_EPI_F32 || epilogue == MMK_EPI_RESID_F32;
  if (ldo % (f32_out ? 4 : 8) != 0) return set_error(MMK_ERR_ARG, "gemm: ldo misaligned");
  if (aux != nullptr && (epilogue != MMK_EPI_RESID_F32 || ld_aux % 8 != 0))
    return set_error(MMK_ERR_ARG, "gemm: aux output only with RESID_F32 and 16B-aligned rows");
  if (ln_stats_out != nullptr && epilogue != MMK_EPI_RESID_F32)
    return set_error(MMK_ERR_ARG, "gemm: LN statistics only from a RESID_F32 epilogue");
  if ((ln_mr != nullptr) != (ln_c1 != nullptr) ||
      (ln_mr != nullptr && (epilogue == MMK_EPI_F32 || epilogue == MMK_EPI_RESID_F32 || bias == nullptr)))
    return set_error(MMK_ERR_ARG, "gemm: a folded LayerNorm needs mr, c1 and bias with a bf16 epilogue");
  if ((reinterpret_cast<uintptr_t>(ln_c1) | reinterpret_cast<uintptr_t>(ln_mr) |
       reinterpret_cast<uintptr_t>(ln_stats_out)) & 15)
    return set_error(MMK_ERR_ARG, "gemm: LN pointers must be 16-byte aligned");
  const LnFold lf{reinterpret_cast<float2*>(ln_stats_out), reinterpret_cast<const float2*>(ln_mr), ln_c1};
  // Kernel choice: CTA pairs (M=256 x N=256 tiles; N a multiple of 64, the last N tile possibly
  // partial) when there are enough tiles to occupy the pairs; otherwise the single-CTA kernel
  // with BN 256 or 128.
  static const bool no_2sm = getenv("MMK_GEMM_NO_2SM") != nullptr;  // A/B switch for profiling
  const int tiles2 = ((m + 255) / 256) * ((n + 255) / 256);
  if (!no_2sm && n % 64 == 0 && tiles2 >= num_sms() / 2) {
    CUtensorMap ta, tb;
    int rc = make_tmap_2d_bf16(&ta, a, k, m, lda, kGemmBK, 128, true);
    if (rc) return rc;
    rc = make_tmap_2d_bf16(&tb, b, k, n, ldb, kGemmBK, 128, true);
    if (rc) return rc;
    CUtensorMap to = tb;  // output map: bf16 [32 rows][64 cols] or fp32 residual [32 rows][32 cols], 128B swizzle
    if (!f32_out) {
      rc = make_tmap_2d_bf16(&to, out, n, m, ldo, 64, 32, true);
      if (rc) return rc;
    } else {  // fp32 output / residual: [32 rows][32 cols] boxes
      const uint64_t dims[2] = {static_cast<uint64_t>(n), static_cast<uint64_t>(m)};
      const uint64_t strides[1] = {static_cast<uint64_t>(ldo) * 4};
      const uint32_t box[2] = {32, 32};
      rc = make_tmap(&to, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, out, 2, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B);
      if (rc) return rc;
    }
    // grouped tile order only for large weight matrices (see grouped_tile)
    static const int group_env = getenv("MMK_GEMM_GROUP_M") ? atoi(getenv("MMK_GEMM_GROUP_M")) : 0;
    const int group_m = group_env > 0 ? group_env : (static_cast<int64_t>(n) * k * 2 > (32ll << 20) ? 16 : 1);
    return dispatch_epi_2sm<5>(epilogue, ta, tb, to, m, n, k, bias, out, ldo, gate,
                               reinterpret_cast<__nv_bfloat16*>(aux), ld_aux, lf, group_m, stream);
  }
  const int tiles256 = ((m + kGemmBM - 1) / kGemmBM) * ((n + 255) / 256);
  const bool use128 = (n % 256 != 0) || tiles256 < num_sms();
  CUtensorMap ta, tb;
  int rc = make_tmap_2d_bf16(&ta, a, k, m, lda, kGemmBK, kGemmBM, /*swizzle128=*/true);
  if (rc) return rc;
  rc = make_tmap_2d_bf16(&tb, b, k, n, ldb, kGemmBK, use128 ? 128 : 256, true);
  if (rc) return rc;
  if (use128)
    return dispatch_epi<128, 6>(epilogue, ta, tb, m, n, k, bias, out, ldo, gate,
                                reinterpret_cast<__nv_bfloat16*>(aux), ld_aux, lf, stream);
  return dispatch_epi<256, 4>(epilogue, ta, tb, m, n, k, bias, out, ldo, gate,
                              reinterpret_cast<__nv_bfloat16*>(aux), ld_aux, lf, stream);
}

extern "C" int mmk_gemm_bf16(const void* a, int64_t lda, const void* b, int64_t ldb, int32_t m,
                             int32_t n, int32_t k, int32_t epilogue, const float* bias, void* out,
                             int64_t ldo, float gate, void* aux, int64_t ld_aux, cudaStream_t stream) {
  return mmk_gemm_bf16_ln(a, lda, b, ldb, m, n, k, epilogue, bias, out, ldo, gate, aux, ld_aux, nullptr, nullptr,
                          nullptr, stream);
}
