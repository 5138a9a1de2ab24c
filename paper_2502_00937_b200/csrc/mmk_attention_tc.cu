// mmk_attention_tc.cu — K5 on 5th-generation tensor cores: varlen non-causal flash attention
// with S = Q K^T and O = P V accumulated in TMEM (tcgen05.mma), Q/K/V tiles staged by TMA.
//
// CTA = NQ 128-row query tiles of one (sequence, head), KV tiles of BKV keys; warp roles:
//   warps 4t..4t+3   softmax warpgroup t (query tile t, TMEM lanes 0-127 = rows)
//   warp 4*NQ        TMA producer (Q once; K/V tiles into a STAGES-deep ring)
//   warps 4*NQ+1..   MMA issuer of query tile t (warp-uniform, one elected lane); the first
//                    also allocates TMEM
// TMEM (512 columns): S_t at [t*BKV, (t+1)*BKV), O_t after them (hd columns each).  A softmax
// warpgroup releases its S buffer as soon as the scores are in registers (s_free), so the MMA
// warp issues S_t(j+1) = Q_t K(j+1)^T while the exponentials of tile j are still being
// computed; P (bf16 pairs) is written back to TMEM and read from there as the A operand of the
// PV MMA.  One MMA-issuer warp per query tile issues S_t(j) then PV_t(j-1).
// Online softmax in base 2 with a lazily updated running max (rescale O only when the row max
// grows by more than 2^8), so O is rarely touched.
//
// Two launch forms share the per-tile steps: a persistent kernel pulling (query block, head,
// image) work items from a global counter (launches with more than two waves of items), and one
// item per CTA (smaller launches); see attn_fwd_tc_persistent.  The softmax is speculative (the
// row max of an item's first KV tile is reused for the rest) with a gated exact pass behind it.
//
// head_dim 80 = 64 + 16: Q/K use a 128B-swizzled K-major block (4 MMA k-steps) plus a
// 32B-swizzled block (1 k-step); V is the MN-major B operand, split into N=64 (128B swizzle)
// and N=16 (32B swizzle) MMAs.  head_dim 64 uses the first block only.
#include "sm100_common.cuh"
#include <cstdlib>
#include "mmk_internal.h"

namespace mmk {

#ifdef MMK_ATTN_TRACE
// Debug build only (make trace): clock64 timestamps of CTA (0,0,0): [role][kv tile][event]
__device__ long long g_attn_trace[3][64][8];
#define TR(role, j, ev) \
  if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && (j) < 64) g_attn_trace[role][j][ev] = clock64();
#else
#define TR(role, j, ev)
#endif

// Pairs out of every 8 whose exp2 runs as an FMA-pipe polynomial (the rest on MUFU): 2 for the
// exact softmax, 1 for the speculative one, whose missing max pass leaves less FMA/ALU work to
// interleave with MUFU (measured, profiles/r01_attention.md).
#ifndef MMK_POLY8
#define MMK_POLY8 2
#endif
#ifndef MMK_POLY8_SPEC
#define MMK_POLY8_SPEC 1
#endif

constexpr int kTcBQ = 128;
constexpr float kRescaleThreshold = 8.0f;  // log2 units

// Row sums of P on the tensor core (hd 80): one more TS-MMA per 16-key step, O_t(:, HD) += P_t x ones,
// so the softmax warps drop their FADD2 sums and l is exactly the sum of the bf16 P the PV used.
#ifndef MMK_ATTN_LSUM
#define MMK_ATTN_LSUM 0
#endif
// Split softmax (needs LSUM): two warps per TMEM lane quarter, each owning half of a KV tile's
// keys, so every SM sub-partition runs twice as many softmax warps; with the tensor-core row sums
// and the speculative max the halves only meet at an item's first tile (row max via shared memory).
#ifndef MMK_ATTN_SPLIT
#define MMK_ATTN_SPLIT 0
#endif

// K/V ring depth for hd 128 (64-key tiles of 32 KB): 3 fits beside the persistent kernel's two Q
// slots once its longest-first schedule table is capped at 96 sequences (TcPersistLayout)
#ifndef MMK_ATTN_HD128_STAGES
#define MMK_ATTN_HD128_STAGES 3
#endif

template <int HD, int BKV, int NQ>
struct TcAttnCfg {
  static constexpr bool kLSum = MMK_ATTN_LSUM && HD == 80;   // l accumulated by the tensor core
  static constexpr int kOCols = HD + (kLSum ? 16 : 0);       // O_t columns (+ the l block)
  static constexpr bool kRem = (HD % 64) != 0;               // has a 16-wide remainder block
  static constexpr int kBlocks = HD / 64;                    // 64-column main blocks (2 for hd 128)
  static constexpr int kQBlock = kTcBQ * 64 * 2;             // one main block of Q: 128 rows x 64 cols
  static constexpr int kQMain = kBlocks * kQBlock;
  static constexpr int kQBytes = kQMain + (kRem ? kTcBQ * 16 * 2 : 0);
  static constexpr int kKVBlock = BKV * 64 * 2;              // one main block of K or V: BKV rows x 64 cols
  static constexpr int kKVMain = kBlocks * kKVBlock;
  static constexpr int kKVBytes = kKVMain + (kRem ? BKV * 16 * 2 : 0);
  static constexpr int STAGES = HD > 80 ? MMK_ATTN_HD128_STAGES : 4;
  static constexpr int kQOff = 0;
  static constexpr int kKVOff = NQ * kQBytes;
  static constexpr int kStageBytes = 2 * kKVBytes;           // K then V
  static constexpr int kOnesOff = kKVOff + STAGES * kStageBytes;  // 16 keys x 32 B of ones (kLSum)
  static constexpr int kBarOff = kOnesOff + (kLSum ? 512 : 0);
  static constexpr int kSmem = kBarOff + 256 + 1024;
  static constexpr bool kSplit = MMK_ATTN_SPLIT && kLSum;
  static constexpr int kHalves = kSplit ? 2 : 1;
  static constexpr int kSoftmaxWarps = 4 * NQ * kHalves;
  static constexpr int kThreads = 32 * (kSoftmaxWarps + 1 + NQ);  // softmax warps, TMA warp, NQ MMA warps
  static constexpr int kOBase = NQ * BKV;                    // TMEM column of O_0 (O_t: + t*kOCols)
  // P_t (bf16 pairs) in its own columns when S + O + P fit 512, else aliased onto S_t (then S_t(j+1)
  // is issued only after PV_t(j) has retired, instead of as soon as S_t(j) is in registers)
  static constexpr int kPStrideSep = (BKV / 2 + 31) / 32 * 32;
  static constexpr bool kAlias = (kOBase + NQ * kOCols + 31) / 32 * 32 + (NQ - 1) * kPStrideSep + BKV / 2 > 512;
  static constexpr int kPBase = kAlias ? 0 : (kOBase + NQ * kOCols + 31) / 32 * 32;  // P_t: + t*kPStride
  static constexpr int kPStride = kAlias ? BKV : kPStrideSep;
  static_assert(kPBase + (NQ - 1) * kPStride + BKV / 2 <= 512, "TMEM overflow: S + O + P > 512 columns");
  static_assert(BKV % 16 == 0, "key tile");
  static_assert(kSmem <= 232448, "shared memory overflow");
};

MMK_DEV float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

MMK_DEV bool warp_any(bool p) { return __any_sync(0xffffffffu, p); }

// Register dependency fence: values written by an asynchronous tcgen05.ld are only read after
// the tcgen05.wait::ld that precedes this (the compiler may not hoist their uses above it).
template <int N>
MMK_DEV void reg_fence(uint32_t* r) {
#pragma unroll
  for (int i = 0; i < N; ++i) asm volatile("" : "+r"(r[i]));
}

MMK_DEV float fmax3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

// 2^x for a pair on the FMA pipe: round-to-nearest split x = n + f (magic-number trick),
// degree-3 polynomial for 2^f on [-0.5, 0.5] (max rel err 1.0e-4, far below bf16's 2^-8), and
// the exponent added in the integer domain.  x is clamped at -126 (masked -inf -> ~0).
// (x > 127 wraps the exponent: the speculative softmax tracks the largest polynomial input and
// sends such rows to the exact pass.)
MMK_DEV float2 exp2_poly2(float2 x) {
  constexpr float kMagic = 12582912.f;  // 1.5 * 2^23
  x.x = fmaxf(x.x, -126.f);
  x.y = fmaxf(x.y, -126.f);
  const float2 t = __fadd2_rn(x, make_float2(kMagic, kMagic));
  const float2 rn = __fadd2_rn(t, make_float2(-kMagic, -kMagic));
  const float2 f = __ffma2_rn(rn, make_float2(-1.f, -1.f), x);
  float2 q = __ffma2_rn(f, make_float2(0.05592203564723278f, 0.05592203564723278f),
                        make_float2(0.24264008283277078f, 0.24264008283277078f));
  q = __ffma2_rn(q, f, make_float2(0.6931210339915522f, 0.6931210339915522f));
  q = __ffma2_rn(q, f, make_float2(0.9999244814555215f, 0.9999244814555215f));
  float2 e;
  // exponent added in the integer domain (LEA on the ALU pipe, not IMAD on the FMA pipe)
  e.x = __uint_as_float(__float_as_uint(q.x) + __funnelshift_l(0u, __float_as_uint(t.x), 23));
  e.y = __uint_as_float(__float_as_uint(q.y) + __funnelshift_l(0u, __float_as_uint(t.y), 23));
  return e;
}


// ---------------------------------------------------------------------------- per-tile steps
// (shared by the one-item-per-CTA kernel and the persistent kernel)

// S_t = Q_t K^T for one KV tile (one elected lane issues; Q and K K-major in smem).
template <int HD, int BKV, int NQ>
MMK_DEV void issue_s(uint32_t s_tm, uint32_t q_addr, uint32_t k_addr) {
  using C = TcAttnCfg<HD, BKV, NQ>;
  constexpr uint32_t idesc_s = umma_idesc_bf16_f32(kTcBQ, BKV);
#pragma unroll
  for (int b = 0; b < C::kBlocks; ++b) {
    const uint64_t qd = umma_desc_sw128_kmajor(q_addr + b * C::kQBlock);
    const uint64_t kd = umma_desc_sw128_kmajor(k_addr + b * C::kKVBlock);
#pragma unroll
    for (int k = 0; k < 4; ++k) umma_bf16_ss(s_tm, qd + 2 * k, kd + 2 * k, idesc_s, (b | k) > 0);
  }
#ifndef MMK_ATTN_XP_NOSREM  // timing experiment only (make xp): S without its remainder k-step
  if (C::kRem)
    umma_bf16_ss(s_tm, umma_desc_sw32_kmajor(q_addr + C::kQMain), umma_desc_sw32_kmajor(k_addr + C::kKVMain),
                 idesc_s, 1u);
#endif
}

// O_t (+)= P_t V for one KV tile: P_t from TMEM (bf16 pairs, 8 columns per 16 keys) as the A
// operand, V the MN-major B operand (8-row K groups at 128 B main / 32 B remainder per row).
// The constant B operand of the row-sum MMA: 16 keys x 16 columns, MN-major, 32-byte rows.  Both
// 16-byte halves of a row are (1, 0, ..., 0), so whatever the 32B swizzle does to a row's halves,
// columns 0 and 8 of the result hold the row sum of P.
MMK_DEV void init_ones_tile(uint8_t* p) {
  uint32_t* w = reinterpret_cast<uint32_t*>(p);
  for (int i = 0; i < 128; ++i) w[i] = (i & 3) == 0 ? 0x3F80u : 0u;  // bf16 1.0 in the low half of word 0 of each 16 B
}

template <int HD, int BKV, int NQ>
MMK_DEV void issue_pv(uint32_t o_tm, uint32_t p_tm, uint32_t v_addr, bool first, uint32_t ones_addr = 0) {
  using C = TcAttnCfg<HD, BKV, NQ>;
  constexpr uint32_t idesc_pv_main = umma_idesc_bf16_f32(kTcBQ, 64) | (1u << 16);  // B (V) MN-major
  constexpr uint32_t idesc_pv_rem = umma_idesc_bf16_f32(kTcBQ, 16) | (1u << 16);
  constexpr uint32_t kVStepMain = (16 * 128) >> 4, kVStepRem = (16 * 32) >> 4;  // desc units per k-step
  const uint64_t vd_rem = umma_desc_sw32_kmajor(v_addr + C::kKVMain);  // MN-major, SBO 256
#pragma unroll
  for (int k = 0; k < BKV / 16; ++k) {
    const uint32_t acc = (!first || k > 0) ? 1u : 0u;
#pragma unroll
    for (int b = 0; b < C::kBlocks; ++b)  // V block b -> O columns [64 b, 64 b + 64); MN-major, SBO 1024
      umma_bf16_ts(o_tm + 64 * b, p_tm + 8 * k, umma_desc_sw128_kmajor(v_addr + b * C::kKVBlock) + kVStepMain * k,
                   idesc_pv_main, acc);
    if (C::kRem) umma_bf16_ts(o_tm + 64 * C::kBlocks, p_tm + 8 * k, vd_rem + kVStepRem * k, idesc_pv_rem, acc);
    if constexpr (C::kLSum) umma_bf16_ts(o_tm + HD, p_tm + 8 * k, umma_desc_sw32_kmajor(ones_addr), idesc_pv_rem, acc);
  }
}

// One KV tile of the online softmax for this thread's query row (its TMEM lane): S_t -> registers
// (then S_t is released to the MMA warp), row max with a lazily updated running max (O_t is
// rescaled in TMEM only when the max grows by more than 2^8), exponentials -> P_t in TMEM, row
// sum.  `g` is the tile's index in query tile t's barrier sequence; `first` marks the first KV tile
// of a work item (no PV of this item precedes it); `valid` = keys of the tile inside the sequence.
//
// SPEC (speculative max): only an item's first tile computes a row max; every later tile reuses
// it without a max pass or rescale.  P = 2^(x - m) may then exceed 1 by any factor — harmless in
// bf16 P / fp32 O and l up to ~2^100 — and a row whose scores outgrow the first tile's by more
// than that ends with l > 2^100 or inf; the caller flags it and the launch is redone exactly.
template <int HD, int BKV, int NQ, bool SPEC = false>
MMK_DEV void softmax_tile(uint32_t s_tm, uint32_t o_tm, uint32_t p_tm, uint64_t* s_full, uint64_t* s_free,
                          uint64_t* pv_done, uint64_t* p_full, uint32_t g, bool first, int valid, float scale_log2,
                          float& m_used, float& l, uint32_t lane, bool trace, int t, int j) {
  (void)trace; (void)t; (void)j;
  if (trace) { TR(t, j, 0) }
  mbar_wait(s_full, g & 1);
  if (trace) { TR(t, j, 1) }
  tc_fence_after();
  uint32_t r[BKV];
  // Speculative non-first, non-last tiles need no row max, so the exponentials of the first 32
  // keys start while the other 80 are still in flight from TMEM (S is released after them).
  const bool pipelined = SPEC && !first && valid >= BKV;  // warp-uniform
  auto release_s = [&]() {
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(s_free);  // TMEM S_t may now be overwritten by the next S_t
  };
  tmem_ld_32x32b_x32(s_tm, *reinterpret_cast<uint32_t(*)[32]>(&r[0]));
  if (pipelined) {
    tmem_ld_wait();
    reg_fence<32>(r);
  }
#pragma unroll
  for (int c = 1; c < BKV / 32; ++c) {
    uint32_t (&rc)[32] = *reinterpret_cast<uint32_t(*)[32]>(&r[32 * c]);
    tmem_ld_32x32b_x32(s_tm + 32 * c, rc);
  }
  if constexpr (BKV % 32 != 0) {
    uint32_t (&rc)[16] = *reinterpret_cast<uint32_t(*)[16]>(&r[BKV - 16]);
    tmem_ld_32x32b_x16(s_tm + BKV - 16, rc);
  }
  if (!pipelined) {
    tmem_ld_wait();
    reg_fence<BKV>(r);
    release_s();
  }
  if (trace) { TR(t, j, 2) }
  if (valid < BKV) {                   // last tile only (uniform branch)
#pragma unroll
    for (int i = 0; i < BKV; ++i)
      if (i >= valid) r[i] = __float_as_uint(-INFINITY);
  }
  float m_new = m_used, corr = 1.f;
  if (!SPEC || first) {
    float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
    for (int i = 0; i < BKV; i += 8)
#pragma unroll
      for (int u = 0; u < 4; ++u) m4[u] = fmax3(m4[u], __uint_as_float(r[i + 2 * u]), __uint_as_float(r[i + 2 * u + 1]));
    const float mx = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3])) * scale_log2;
    if (mx > m_used + kRescaleThreshold) {
      m_new = mx;
      corr = fast_exp2(m_used - m_new);  // 0 on the first tile
    }
  }
  if (!SPEC && !first && warp_any(corr != 1.f)) {
    // rescale O_t once the previous PV_t has retired
    mbar_wait(pv_done, (g - 1) & 1);
    tc_fence_after();
    uint32_t o[16];
#pragma unroll
    for (int c = 0; c < TcAttnCfg<HD, BKV, NQ>::kOCols / 16; ++c) {  // with kLSum also rescales l
      tmem_ld_32x32b_x16(o_tm + 16 * c, o);
      tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 16; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * corr);
      tmem_st_32x32b_x16(o_tm + 16 * c, o);
    }
    tmem_st_wait();
  }
  m_used = m_new;
  // p = 2^(s*scale - m): MMK_POLY8(_SPEC) of every 8 pairs on the FMA pipe (polynomial), the rest on MUFU
  const float2 sc2 = make_float2(scale_log2, scale_log2);
  const float2 nm2 = make_float2(-m_new, -m_new);
  float2 sa = make_float2(0.f, 0.f), sb = make_float2(0.f, 0.f);
  float pm = -INFINITY;  // SPEC: largest polynomial input (the polynomial is valid up to 127)
  uint32_t p[BKV / 2];
  auto exp_pair = [&](int i) {
    const float2 x = __ffma2_rn(make_float2(__uint_as_float(r[2 * i]), __uint_as_float(r[2 * i + 1])), sc2, nm2);
    float2 e;
#ifdef MMK_ATTN_XP_NOEXP  // timing experiment only (make xp): no exponential
    if (true) {
      e = x;
    } else
#endif
    if ((i & 7) < (SPEC ? MMK_POLY8_SPEC : MMK_POLY8)) {
      if constexpr (SPEC) pm = fmax3(pm, x.x, x.y);
      e = exp2_poly2(x);
    } else {
      e.x = fast_exp2(x.x);
      e.y = fast_exp2(x.y);
    }
    if constexpr (!TcAttnCfg<HD, BKV, NQ>::kLSum) {
      if (i & 1) sb = __fadd2_rn(sb, e); else sa = __fadd2_rn(sa, e);
    }
    p[i] = pack_bf16x2(e.x, e.y);
  };
  if (pipelined) {
#pragma unroll
    for (int i = 0; i < 16; ++i) exp_pair(i);
    tmem_ld_wait();
    reg_fence<BKV>(r);
    release_s();
#pragma unroll
    for (int i = 16; i < BKV / 2; ++i) exp_pair(i);
  } else if (valid >= BKV) {
#pragma unroll
    for (int i = 0; i < BKV / 2; ++i) exp_pair(i);
  } else {
    // last tile of the sequence: 16-key groups entirely past its end get P = 0 without any
    // exponential (uniform branch per group)
#pragma unroll
    for (int g16 = 0; g16 < BKV / 16; ++g16) {
      if (16 * g16 < valid) {
#pragma unroll
        for (int k = 0; k < 8; ++k) exp_pair(8 * g16 + k);
      } else {
#pragma unroll
        for (int k = 0; k < 8; ++k) p[8 * g16 + k] = 0u;
      }
    }
  }
  if constexpr (TcAttnCfg<HD, BKV, NQ>::kLSum) {
    // l lives in O_t(:, HD) (tensor-core row sum); the register l only carries the wrap flag
    if constexpr (SPEC) {
      if (pm > 126.f) l = INFINITY;  // wrapped polynomial: route the row to the exact pass
    }
  } else {
    float sum = (sa.x + sa.y) + (sb.x + sb.y);
    if constexpr (SPEC) {
      if (pm > 126.f) sum = INFINITY;  // wrapped polynomial: route the row to the exact pass
    }
    l = l * corr + sum;
  }
  if (trace) { TR(t, j, 3) }
  // P_t -> TMEM (the previous PV_t must have finished reading the buffer; at the first tile of an
  // item the previous item's last PV retired before its output was read)
  if (!first) mbar_wait(pv_done, (g - 1) & 1);
  if (trace) { TR(t, j, 4) }
  tc_fence_after();
#pragma unroll
  for (int c = 0; c < BKV / 64; ++c)
    tmem_st_32x32b_x32(p_tm + 32 * c, *reinterpret_cast<const uint32_t(*)[32]>(&p[32 * c]));
  if constexpr ((BKV / 2) % 32 >= 16)
    tmem_st_32x32b_x16(p_tm + (BKV / 64) * 32, *reinterpret_cast<const uint32_t(*)[16]>(&p[(BKV / 64) * 32]));
  if constexpr ((BKV / 2) % 16 == 8)
    tmem_st_32x32b_x8(p_tm + BKV / 2 - 8, *reinterpret_cast<const uint32_t(*)[8]>(&p[BKV / 2 - 8]));
  tmem_st_wait();
  tc_fence_before();  // orders the O rescale / P (tcgen05.st) before the arrive
  __syncwarp();
  if (lane == 0) mbar_arrive(p_full);
  if (trace) { TR(t, j, 5) }
}

// Speculative softmax: a row whose l left the safe range (scores outgrew the first tile's max by
// more than ~2^100) marks the launch for the exact pass.
constexpr float kSpecLimit = 1.2676506e30f;  // 2^100
MMK_DEV void flag_overflow(float l, int* flag) {
  if (!(l <= kSpecLimit)) *reinterpret_cast<volatile int*>(flag) = 1;  // also catches inf / NaN
}

// Split form of softmax_tile (C::kSplit): this warp owns keys [h*KH, (h+1)*KH) of the tile for its
// 32 rows; the partner warp (same rows, other half) meets it only where a row max is computed
// (an item's first tile with SPEC, every tile without), through `red` [2][32] in shared memory and
// a 64-thread named barrier.  l is summed by the tensor core (kLSum); half 0 rescales O.
template <int HD, int BKV, int NQ, bool SPEC>
MMK_DEV void softmax_tile_split(uint32_t s_tm, uint32_t o_tm, uint32_t p_tm, uint64_t* s_full, uint64_t* s_free,
                                uint64_t* pv_done, uint64_t* p_full, uint32_t g, bool first, int valid,
                                float scale_log2, float& m_used, float& l, uint32_t lane, int h, float* red,
                                uint32_t bar_id) {
  constexpr int KH = BKV / 2;
  static_assert(KH % 16 == 0 && KH <= 64, "half tile");
  mbar_wait(s_full, g & 1);
  tc_fence_after();
  uint32_t r[KH];
  const uint32_t sc = s_tm + h * KH;
  tmem_ld_32x32b_x32(sc, *reinterpret_cast<uint32_t(*)[32]>(&r[0]));
  if constexpr (KH > 32) tmem_ld_32x32b_x16(sc + 32, *reinterpret_cast<uint32_t(*)[16]>(&r[32]));
  tmem_ld_wait();
  reg_fence<KH>(r);
  tc_fence_before();
  __syncwarp();
  if (lane == 0) mbar_arrive(s_free);
  const int vh = valid - h * KH;  // keys of this half inside the sequence
  if (vh < KH) {
#pragma unroll
    for (int i = 0; i < KH; ++i)
      if (i >= vh) r[i] = __float_as_uint(-INFINITY);
  }
  float m_new = m_used, corr = 1.f;
  if (!SPEC || first) {
    float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
    for (int i = 0; i < KH; i += 8)
#pragma unroll
      for (int u = 0; u < 4; ++u) m4[u] = fmax3(m4[u], __uint_as_float(r[i + 2 * u]), __uint_as_float(r[i + 2 * u + 1]));
    float mx = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
    red[h * 32 + lane] = mx;
    named_bar_sync(bar_id, 64);
    mx = fmaxf(mx, red[(h ^ 1) * 32 + lane]) * scale_log2;
    named_bar_sync(bar_id, 64);  // both read before the next exchange overwrites
    if (mx > m_used + kRescaleThreshold) {
      m_new = mx;
      corr = fast_exp2(m_used - m_new);
    }
  }
  if (!SPEC && !first && h == 0 && warp_any(corr != 1.f)) {
    mbar_wait(pv_done, (g - 1) & 1);
    tc_fence_after();
    uint32_t o[16];
#pragma unroll
    for (int c = 0; c < TcAttnCfg<HD, BKV, NQ>::kOCols / 16; ++c) {
      tmem_ld_32x32b_x16(o_tm + 16 * c, o);
      tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 16; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * corr);
      tmem_st_32x32b_x16(o_tm + 16 * c, o);
    }
    tmem_st_wait();
  }
  m_used = m_new;
  const float2 sc2 = make_float2(scale_log2, scale_log2);
  const float2 nm2 = make_float2(-m_new, -m_new);
  float pm = -INFINITY;
  uint32_t p[KH / 2];
#pragma unroll
  for (int i = 0; i < KH / 2; ++i) {
    float2 e;
    if (vh <= 2 * i) {  // pairs past the sequence end (last tile, uniform)
      e = make_float2(0.f, 0.f);
    } else {
      const float2 x = __ffma2_rn(make_float2(__uint_as_float(r[2 * i]), __uint_as_float(r[2 * i + 1])), sc2, nm2);
      if ((i & 7) < (SPEC ? MMK_POLY8_SPEC : MMK_POLY8)) {
        if constexpr (SPEC) pm = fmax3(pm, x.x, x.y);
        e = exp2_poly2(x);
      } else {
        e.x = fast_exp2(x.x);
        e.y = fast_exp2(x.y);
      }
    }
    p[i] = pack_bf16x2(e.x, e.y);
  }
  if constexpr (SPEC) {
    if (pm > 126.f) l = INFINITY;
  }
  if (!first) mbar_wait(pv_done, (g - 1) & 1);
  tc_fence_after();
  const uint32_t pc = p_tm + h * (KH / 2);
  if constexpr (KH / 2 == 32) {
    tmem_st_32x32b_x32(pc, *reinterpret_cast<const uint32_t(*)[32]>(&p[0]));
  } else {
    static_assert(KH / 2 == 24 || KH / 2 == 16 || KH / 2 == 8, "P half");
    if constexpr (KH / 2 >= 16) tmem_st_32x32b_x16(pc, *reinterpret_cast<const uint32_t(*)[16]>(&p[0]));
    if constexpr (KH / 2 == 24 || KH / 2 == 8)
      tmem_st_32x32b_x8(pc + (KH / 2 >= 16 ? 16 : 0), *reinterpret_cast<const uint32_t(*)[8]>(&p[KH / 2 >= 16 ? 16 : 0]));
  }
  tmem_st_wait();
  tc_fence_before();
  __syncwarp();
  if (lane == 0) mbar_arrive(p_full);
}

// The row's softmax denominator: with kLSum the tensor core's sum in O_t(:, HD) (the register l
// only carries the speculative pass's wrap flag, +inf), else the register sum.
template <int HD, int BKV, int NQ>
MMK_DEV float final_l(uint32_t o_tm, float l) {
  if constexpr (TcAttnCfg<HD, BKV, NQ>::kLSum) {
    uint32_t r[4];
    tmem_ld_32x32b_x4(o_tm + HD, r);
    tmem_ld_wait();
    return l == INFINITY ? INFINITY : __uint_as_float(r[0]);
  } else {
    return l;
  }
}

// O_t / l -> bf16 output row (16 columns per TMEM load, two 16-byte stores).
template <int HD>
MMK_DEV void store_o(uint32_t o_tm, float l, __nv_bfloat16* go, bool row_ok) {
  const float inv = 1.f / l;
#pragma unroll
  for (int c = 0; c < HD / 16; ++c) {
    uint32_t o[16];
    tmem_ld_32x32b_x16(o_tm + 16 * c, o);
    tmem_ld_wait();
    if (row_ok) {
      uint32_t w[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) w[i] = pack_bf16x2(__uint_as_float(o[2 * i]) * inv, __uint_as_float(o[2 * i + 1]) * inv);
      st_global_v4(go + 16 * c, w[0], w[1], w[2], w[3]);
      st_global_v4(go + 16 * c + 8, w[4], w[5], w[6], w[7]);
    }
  }
}

template <int HD, int BKV, int NQ, bool SPEC>
__global__ void __maxnreg__(MMK_ATTN_SPLIT && HD == 80 ? 96 : (NQ == 2 ? 168 : 128))
attn_fwd_tc(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_q_rem,
            const __grid_constant__ CUtensorMap tm_kv, const __grid_constant__ CUtensorMap tm_kv_rem,
            __nv_bfloat16* __restrict__ out, const int32_t* __restrict__ cu_seqlens, int heads, float scale_log2,
            int* __restrict__ overflow_flag) {
  using C = TcAttnCfg<HD, BKV, NQ>;
  constexpr int kTmaWarp = C::kSoftmaxWarps, kMmaWarp = C::kSoftmaxWarps + 1;  // MMA warp of tile t: kMmaWarp + t
  __shared__ float s_red[C::kSplit ? 4 * NQ * 64 : 1];  // split softmax: row-max exchange
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kBarOff);
  uint64_t* q_full = bars + 0;
  uint64_t* k_full = bars + 1;                 // [STAGES]
  uint64_t* v_full = k_full + C::STAGES;       // [STAGES]
  uint64_t* kv_empty = v_full + C::STAGES;     // [STAGES]
  uint64_t* s_full = kv_empty + C::STAGES;     // [NQ] MMA -> softmax: S_t ready
  uint64_t* s_free = s_full + NQ;              // [NQ] softmax -> MMA: S_t consumed
  uint64_t* p_full = s_free + NQ;              // [NQ] softmax -> MMA: P_t in smem (+ O_t rescaled)
  uint64_t* pv_done = p_full + NQ;             // [NQ] MMA -> softmax: PV_t retired
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pv_done + NQ);

  griddep_wait();  // cu_seqlens / QKV come from the preceding kernels (PDL)
  const int head = blockIdx.y, seq = blockIdx.z;  // heads of one image adjacent: K/V lines shared in L2
  const int s_begin = cu_seqlens[seq];
  const int len = cu_seqlens[seq + 1] - s_begin;
  const int q0 = blockIdx.x * NQ * kTcBQ;
  if (q0 >= len) return;
  const int n_qt = min(NQ, (len - q0 + kTcBQ - 1) / kTcBQ);
  const int nkv = (len + BKV - 1) / BKV;
  const int d_model = heads * HD;
  const int col_q = head * HD, col_k = d_model + head * HD, col_v = 2 * d_model + head * HD;

  const uint32_t warp = warp_id_uniform();
  const uint32_t lane = lane_id();

  if (warp == kTmaWarp && lane == 0) {
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_kv);
    if (C::kRem) {
      tma_prefetch_desc(&tm_q_rem);
      tma_prefetch_desc(&tm_kv_rem);
    }
    mbar_init(q_full, 1);
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&v_full[s], 1);
      mbar_init(&kv_empty[s], n_qt);  // released by every tile's MMA warp
    }
    for (int t = 0; t < NQ; ++t) {
      mbar_init(&s_full[t], 1);
      mbar_init(&s_free[t], 4 * C::kHalves);  // one arrive per softmax warp
      mbar_init(&p_full[t], 4 * C::kHalves);
      mbar_init(&pv_done[t], 1);
    }
    fence_barrier_init();
  }
  if (warp == kMmaWarp) tmem_alloc<512>(tmem_slot);
  if (C::kLSum && warp == kTmaWarp) {
    if (lane == 0) init_ones_tile(smem + C::kOnesOff);
    fence_proxy_async();  // generic-proxy writes read by the MMA (async proxy)
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  griddep_launch_dependents();

  auto tile_ptr = [&](int off) { return smem + off; };

  if (warp == kTmaWarp) {
    // ---------------------------------------------------------------- TMA producer
    if (elect_one()) {
      mbar_arrive_expect_tx(q_full, n_qt * C::kQBytes);
      for (int t = 0; t < n_qt; ++t) {
        uint8_t* q = tile_ptr(C::kQOff + t * C::kQBytes);
        for (int b = 0; b < C::kBlocks; ++b)
          tma_load_2d(&tm_q, q_full, q + b * C::kQBlock, col_q + 64 * b, s_begin + q0 + t * kTcBQ);
        if (C::kRem) tma_load_2d(&tm_q_rem, q_full, q + C::kQMain, col_q + 64 * C::kBlocks, s_begin + q0 + t * kTcBQ);
      }
      for (int j = 0; j < nkv; ++j) {
        const int st = j % C::STAGES;
        const uint32_t ph = (j / C::STAGES) & 1;
        mbar_wait(&kv_empty[st], ph ^ 1);
        uint8_t* kt = tile_ptr(C::kKVOff + st * C::kStageBytes);
        uint8_t* vt = kt + C::kKVBytes;
        const int row = s_begin + j * BKV;
        mbar_arrive_expect_tx(&k_full[st], C::kKVBytes);
        for (int b = 0; b < C::kBlocks; ++b) tma_load_2d(&tm_kv, &k_full[st], kt + b * C::kKVBlock, col_k + 64 * b, row);
        if (C::kRem) tma_load_2d(&tm_kv_rem, &k_full[st], kt + C::kKVMain, col_k + 64 * C::kBlocks, row);
        mbar_arrive_expect_tx(&v_full[st], C::kKVBytes);
        for (int b = 0; b < C::kBlocks; ++b) tma_load_2d(&tm_kv, &v_full[st], vt + b * C::kKVBlock, col_v + 64 * b, row);
        if (C::kRem) tma_load_2d(&tm_kv_rem, &v_full[st], vt + C::kKVMain, col_v + 64 * C::kBlocks, row);
      }
    }
  } else if (warp > kTmaWarp) {
    // ---------------------------------------------------------------- MMA issuers
    // One warp per query tile, so one tile's S never queues behind the other tile's PV in an
    // issue order; the whole warp runs the schedule (descriptors stay in uniform registers) and
    // one elected lane issues.  Per KV tile j: S_t(j) once softmax_t released S_t(j-1), then
    // PV_t(j-1) once P_t(j-1) is written.
    const int t = static_cast<int>(warp) - kMmaWarp;
    if (t < n_qt) {
      const uint32_t s_tm = tmem + t * BKV;
      const uint32_t o_tm = tmem + C::kOBase + t * C::kOCols;
      const uint32_t p_tm = tmem + C::kPBase + t * C::kPStride;
      const uint32_t q_addr = smem_u32(tile_ptr(C::kQOff + t * C::kQBytes));
      mbar_wait(q_full, 0);
      // Tile t > 0 starts once tile 0's first P is written: the two softmax warpgroups then run
      // their exponential phases offset instead of in lockstep, so one warpgroup's S-load / P-store
      // gaps are filled by the other's MUFU work (attention +2 % in-step, r01_attention.md).
      if (t > 0 && nkv > 1) mbar_wait(&p_full[0], 0);
      tc_fence_after();
      auto do_s = [&](int j) {
        const int st = j % C::STAGES;
        mbar_wait(&k_full[st], (j / C::STAGES) & 1);
        if (j > 0) {
          if constexpr (C::kAlias) mbar_wait(&pv_done[t], (j - 1) & 1);  // PV_t(j-1) has read P_t = S_t
          else mbar_wait(&s_free[t], (j - 1) & 1);                        // softmax has S_t(j-1) in registers
        }
        tc_fence_after();
        if (t < 2) { TR(2, j, 0) }
        const uint32_t k_addr = smem_u32(tile_ptr(C::kKVOff + st * C::kStageBytes));
        if (elect_one()) {
          issue_s<HD, BKV, NQ>(s_tm, q_addr, k_addr);
          umma_commit(&s_full[t]);
        }
        __syncwarp();
        if (t < 2) { TR(2, j, 1 + t) }
      };
      for (int j = 0; j <= nkv; ++j) {
        const int pst = (j - 1 + C::STAGES) % C::STAGES;
        if (!C::kAlias && j < nkv) do_s(j);
        if (j > 0) {
          mbar_wait(&v_full[pst], ((j - 1) / C::STAGES) & 1);
          mbar_wait(&p_full[t], (j - 1) & 1);
          tc_fence_after();
          if (t < 2) { TR(2, j - 1, 3 + t) }
          const uint32_t v_addr = smem_u32(tile_ptr(C::kKVOff + pst * C::kStageBytes + C::kKVBytes));
          if (elect_one()) {
            issue_pv<HD, BKV, NQ>(o_tm, p_tm, v_addr, j == 1, smem_u32(smem + C::kOnesOff));
            umma_commit(&pv_done[t]);
            umma_commit(&kv_empty[pst]);  // this tile is done with K(j-1), V(j-1)
          }
          __syncwarp();
          if (t < 2) { TR(2, j - 1, 5 + t) }
        }
        if (C::kAlias && j < nkv) do_s(j);
      }
    }
  } else {
    // ---------------------------------------------------------------- softmax warpgroups
    const int t = warp / (4 * C::kHalves);   // query tile
    const int h = (warp >> 2) % C::kHalves;  // key half (split softmax)
    const uint32_t q4 = warp & 3;            // lane quarter
    const uint32_t lane_base = (q4 * 32u) << 16;
    const uint32_t s_tm = tmem + t * BKV + lane_base;
    const uint32_t o_tm = tmem + C::kOBase + t * C::kOCols + lane_base;
    const int row = q0 + t * kTcBQ + q4 * 32 + lane;  // query row within the sequence
    if (t < n_qt) {
      const uint32_t p_tm = tmem + C::kPBase + t * C::kPStride + lane_base;
      float m_used = -INFINITY, l = 0.f;
      for (int j = 0; j < nkv; ++j) {
        if constexpr (C::kSplit)
          softmax_tile_split<HD, BKV, NQ, SPEC>(s_tm, o_tm, p_tm, &s_full[t], &s_free[t], &pv_done[t], &p_full[t], j,
                                                j == 0, len - j * BKV, scale_log2, m_used, l, lane, h,
                                                s_red + (t * 4 + q4) * 64, 1 + t * 4 + q4);
        else
          softmax_tile<HD, BKV, NQ, SPEC>(s_tm, o_tm, p_tm, &s_full[t], &s_free[t], &pv_done[t], &p_full[t], j, j == 0,
                                          len - j * BKV, scale_log2, m_used, l, lane, q4 == 0 && lane == 0 && t < 2, t,
                                          j);
      }
      mbar_wait(&pv_done[t], (nkv - 1) & 1);
      tc_fence_after();
      if (h == 0) {
        l = final_l<HD, BKV, NQ>(o_tm, l);
        if constexpr (SPEC) flag_overflow(l, overflow_flag);
        store_o<HD>(o_tm, l, out + static_cast<int64_t>(s_begin + row) * d_model + head * HD, row < len);
      } else if constexpr (SPEC) {
        flag_overflow(l, overflow_flag);  // the other half's wrap flag (its l is 0 or inf)
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == kMmaWarp) tmem_dealloc<512>(tmem);
}


// ---------------------------------------------------------------------------- persistent form
// One CTA per SM takes work items — (query block of NQ*128 rows, head, sequence), query block
// fastest, the heads of one image adjacent — from a global counter, so ragged batches balance
// dynamically.  With n_seq <= kMaxSched the sequences are visited longest first (LPT order: the
// last items to start are the cheapest, which shortens the tail) and only non-empty query blocks
// are items; the TMA warp of every CTA builds the same order (a rank sort over the lengths) and
// the per-sequence item prefix in shared memory at start-up.  The TMA warp fetches and decodes each item and hands it to the other warps
// through a 4-deep shared-memory ring; every role therefore walks the same item sequence, and the
// next item's Q (double-buffered) and first K/V tiles load, and its first S = Q K^T runs, while
// the previous item's last softmax, PV and output store are in flight.  Barrier phases run on
// counters that continue across items: `kv` (K/V ring), `qi` (Q slot), `g` (KV tiles seen by
// query tile t), `oi` (items in which tile t was active), `k` (item ring).  An `o_free` handshake
// keeps the next item's first PV (which overwrites O_t) behind the previous item's output read.
struct AttnItem {
  int s_begin, len, q0, head, n_qt, nkv;  // len < 0: no more items
};

template <int HD, int BKV, int NQ>
struct TcPersistLayout {
  using C = TcAttnCfg<HD, BKV, NQ>;
  // sequences the longest-first schedule can sort (more: natural order); hd 128 trades table
  // space for a third K/V stage (InternViT's per-tile sequences are all 1025 tokens long anyway)
  static constexpr int kMaxSched = HD > 80 ? 96 : 256;
  static constexpr int kQSlotBytes = NQ * C::kQBytes;
  static constexpr int kQOff = 0;                          // two Q slots
  static constexpr int kKVOff = 2 * kQSlotBytes;
  static constexpr int kOnesOff = kKVOff + C::STAGES * C::kStageBytes;  // row-sum B operand (kLSum)
  static constexpr int kBarOff = kOnesOff + (C::kLSum ? 512 : 0);
  // longest-first schedule (n_seq <= kMaxSched): lengths, sorted order, item prefix
  static constexpr int kSchedOff = kBarOff + 512;
  static constexpr int kSchedBytes = (3 * kMaxSched + 1) * 4;
  static constexpr int kSmem = kSchedOff + kSchedBytes + 1024;
  static_assert((12 + 3 * C::STAGES + 5 * NQ) * 8 + 4 * sizeof(AttnItem) + 4 <= 512, "barrier area");
  static_assert(kSmem <= 232448, "shared memory overflow");
};

// `gate`: when non-null the launch is the exact redo of a speculative pass and exits at once
// unless that pass flagged an overflow.
template <int HD, int BKV, int NQ, bool SPEC>
__global__ void __maxnreg__(MMK_ATTN_SPLIT && HD == 80 ? 96 : (NQ == 2 ? 168 : 128))
attn_fwd_tc_persistent(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_q_rem,
                       const __grid_constant__ CUtensorMap tm_kv, const __grid_constant__ CUtensorMap tm_kv_rem,
                       __nv_bfloat16* __restrict__ out, const int32_t* __restrict__ cu_seqlens, int n_seq,
                       int heads, int qblocks, float scale_log2, int* __restrict__ item_counter,
                       int* __restrict__ overflow_flag, const int* __restrict__ gate, bool lpt) {
  if (gate != nullptr) {  // the flag is written by the speculative pass just before (PDL)
    griddep_wait();
    if (*reinterpret_cast<const volatile int*>(gate) == 0) return;
  }
  using C = TcAttnCfg<HD, BKV, NQ>;
  using Lay = TcPersistLayout<HD, BKV, NQ>;
  constexpr int kTmaWarp = C::kSoftmaxWarps, kMmaWarp = C::kSoftmaxWarps + 1;  // MMA warp of tile t: kMmaWarp + t
  __shared__ float s_red[C::kSplit ? 4 * NQ * 64 : 1];  // split softmax: row-max exchange
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Lay::kBarOff);
  uint64_t* q_full = bars + 0;                 // [2] Q slot loaded
  uint64_t* q_empty = bars + 2;                // [2] every MMA warp is done with the Q slot
  uint64_t* k_full = bars + 4;                 // [STAGES]
  uint64_t* v_full = k_full + C::STAGES;       // [STAGES]
  uint64_t* kv_empty = v_full + C::STAGES;     // [STAGES]
  uint64_t* s_full = kv_empty + C::STAGES;     // [NQ]
  uint64_t* s_free = s_full + NQ;              // [NQ]
  uint64_t* p_full = s_free + NQ;              // [NQ]
  uint64_t* pv_done = p_full + NQ;             // [NQ]
  uint64_t* o_free = pv_done + NQ;             // [NQ] softmax -> MMA: O_t read out
  uint64_t* item_full = o_free + NQ;           // [4] work-item ring: item published
  uint64_t* item_empty = item_full + 4;        // [4] every consumer warp has copied it
  AttnItem* ring = reinterpret_cast<AttnItem*>(item_empty + 4);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ring + 4);

  int n_items = qblocks * heads * n_seq;
  const int d_model = heads * HD;
  constexpr int kMaxSched = Lay::kMaxSched;
  int* sch_len = reinterpret_cast<int*>(smem + Lay::kSchedOff);  // [kMaxSched]
  int* sch_order = sch_len + kMaxSched;                           // [kMaxSched] rank -> sequence
  int* sch_pre = sch_order + kMaxSched;                           // [kMaxSched + 1] items before rank
  const uint32_t warp = warp_id_uniform();
  const uint32_t lane = lane_id();

  if (warp == kTmaWarp && lane == 0) {
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_kv);
    if (C::kRem) {
      tma_prefetch_desc(&tm_q_rem);
      tma_prefetch_desc(&tm_kv_rem);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&q_full[b], 1);
      mbar_init(&q_empty[b], NQ);
    }
    for (int st = 0; st < C::STAGES; ++st) {
      mbar_init(&k_full[st], 1);
      mbar_init(&v_full[st], 1);
      mbar_init(&kv_empty[st], NQ);  // one release per query tile's MMA warp (inactive ones too)
    }
    for (int t = 0; t < NQ; ++t) {
      mbar_init(&s_full[t], 1);
      mbar_init(&s_free[t], 4 * C::kHalves);
      mbar_init(&p_full[t], 4 * C::kHalves);
      mbar_init(&pv_done[t], 1);
      mbar_init(&o_free[t], 4);
    }
    for (int i = 0; i < 4; ++i) {
      mbar_init(&item_full[i], 1);
      mbar_init(&item_empty[i], C::kSoftmaxWarps + NQ);  // MMA warps + softmax warps
    }
    fence_barrier_init();
  }
  if (warp == kMmaWarp) tmem_alloc<512>(tmem_slot);
  if (C::kLSum && warp == kTmaWarp) {
    if (lane == 0) init_ones_tile(smem + Lay::kOnesOff);
    fence_proxy_async();  // generic-proxy writes read by the MMA (async proxy)
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  griddep_wait();  // setup above overlaps the previous kernel's tail (PDL)
  griddep_launch_dependents();
  auto tile_ptr = [&](int off) { return smem + off; };
  // consumer side of the ring: copy item k, release its slot
  auto next_item = [&](uint32_t& k) -> AttnItem {
    const int slot = k & 3;
    mbar_wait(&item_full[slot], (k >> 2) & 1);
    const volatile AttnItem* e = ring + slot;
    // broadcast from lane 0 so the fields are provably warp-uniform (uniform registers, not the
    // vector registers the softmax loop needs)
    AttnItem it{__shfl_sync(0xffffffffu, e->s_begin, 0), __shfl_sync(0xffffffffu, e->len, 0),
                __shfl_sync(0xffffffffu, e->q0, 0), __shfl_sync(0xffffffffu, e->head, 0),
                __shfl_sync(0xffffffffu, e->n_qt, 0), __shfl_sync(0xffffffffu, e->nkv, 0)};
    __syncwarp();
    if (lane == 0) mbar_arrive(&item_empty[slot]);
    ++k;
    return it;
  };

  if (warp == kTmaWarp) {
    // ---------------------------------------------------------------- scheduler + TMA producer
    if (lpt) {
      for (int i = lane; i < n_seq; i += 32) sch_len[i] = __ldg(cu_seqlens + i + 1) - __ldg(cu_seqlens + i);
      __syncwarp();
      for (int i = lane; i < n_seq; i += 32) {  // rank = #longer + #equal with a lower index
        const int li = sch_len[i];
        int r = 0;
        for (int j = 0; j < n_seq; ++j) {
          const int lj = sch_len[j];
          r += (lj > li) | ((lj == li) & (j < i));
        }
        sch_order[r] = i;
      }
      __syncwarp();
      int carry = 0;
      if (lane == 0) sch_pre[0] = 0;
      for (int base = 0; base < n_seq; base += 32) {  // warp scan of the per-sequence item counts
        const int r = base + static_cast<int>(lane);
        int v = r < n_seq ? (sch_len[sch_order[r]] + NQ * kTcBQ - 1) / (NQ * kTcBQ) * heads : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int u = __shfl_up_sync(0xffffffffu, v, o);
          if (lane >= static_cast<uint32_t>(o)) v += u;
        }
        if (r < n_seq) sch_pre[r + 1] = carry + v;
        carry += __shfl_sync(0xffffffffu, v, 31);
      }
      __syncwarp();
      n_items = carry;
    }
    if (elect_one()) {
      uint32_t kv = 0, qi = 0;
      for (uint32_t k = 0;; ++k) {
        const int item = atomicAdd(item_counter, 1);
        AttnItem it{0, -1, 0, 0, 0, 0};
        if (item < n_items) {
          int qb, seq;
          if (lpt) {
            int lo = 0, hi = n_seq;  // largest lo with sch_pre[lo] <= item
            while (hi - lo > 1) {
              const int mid = (lo + hi) >> 1;
              if (sch_pre[mid] <= item) lo = mid; else hi = mid;
            }
            seq = sch_order[lo];
            const int local = item - sch_pre[lo];
            const int nqb = (sch_len[seq] + NQ * kTcBQ - 1) / (NQ * kTcBQ);
            qb = local % nqb;
            it.head = local / nqb;
          } else {
            qb = item % qblocks;
            const int rest = item / qblocks;
            it.head = rest % heads;
            seq = rest / heads;
          }
          it.s_begin = __ldg(cu_seqlens + seq);
          it.len = __ldg(cu_seqlens + seq + 1) - it.s_begin;
          it.q0 = qb * NQ * kTcBQ;
          it.n_qt = it.q0 < it.len ? min(NQ, (it.len - it.q0 + kTcBQ - 1) / kTcBQ) : 0;  // 0: empty item
          it.nkv = (it.len + BKV - 1) / BKV;
        }
        const int slot_i = k & 3;
        mbar_wait(&item_empty[slot_i], ((k >> 2) & 1) ^ 1);
        volatile AttnItem* e = ring + slot_i;
        e->s_begin = it.s_begin; e->len = it.len; e->q0 = it.q0; e->head = it.head; e->n_qt = it.n_qt; e->nkv = it.nkv;
        mbar_arrive(&item_full[slot_i]);  // release: the item is visible to the waiting warps
        if (it.len < 0) break;
        if (it.n_qt == 0) continue;
        const int col_q = it.head * HD, col_k = d_model + it.head * HD, col_v = 2 * d_model + it.head * HD;
        const int qs = qi & 1;
        mbar_wait(&q_empty[qs], ((qi >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&q_full[qs], it.n_qt * C::kQBytes);
        for (int t = 0; t < it.n_qt; ++t) {
          uint8_t* q = tile_ptr(Lay::kQOff + qs * Lay::kQSlotBytes + t * C::kQBytes);
          const int row = it.s_begin + it.q0 + t * kTcBQ;
          for (int b = 0; b < C::kBlocks; ++b) tma_load_2d(&tm_q, &q_full[qs], q + b * C::kQBlock, col_q + 64 * b, row);
          if (C::kRem) tma_load_2d(&tm_q_rem, &q_full[qs], q + C::kQMain, col_q + 64 * C::kBlocks, row);
        }
        ++qi;
        for (int j = 0; j < it.nkv; ++j, ++kv) {
          const int st = kv % C::STAGES;
          mbar_wait(&kv_empty[st], ((kv / C::STAGES) & 1) ^ 1);
          uint8_t* kt = tile_ptr(Lay::kKVOff + st * C::kStageBytes);
          uint8_t* vt = kt + C::kKVBytes;
          const int row = it.s_begin + j * BKV;
          mbar_arrive_expect_tx(&k_full[st], C::kKVBytes);
          for (int b = 0; b < C::kBlocks; ++b) tma_load_2d(&tm_kv, &k_full[st], kt + b * C::kKVBlock, col_k + 64 * b, row);
          if (C::kRem) tma_load_2d(&tm_kv_rem, &k_full[st], kt + C::kKVMain, col_k + 64 * C::kBlocks, row);
          mbar_arrive_expect_tx(&v_full[st], C::kKVBytes);
          for (int b = 0; b < C::kBlocks; ++b) tma_load_2d(&tm_kv, &v_full[st], vt + b * C::kKVBlock, col_v + 64 * b, row);
          if (C::kRem) tma_load_2d(&tm_kv_rem, &v_full[st], vt + C::kKVMain, col_v + 64 * C::kBlocks, row);
        }
      }
    }
  } else if (warp > kTmaWarp) {
    // ---------------------------------------------------------------- MMA issuers
    const int t = static_cast<int>(warp) - kMmaWarp;
    const uint32_t s_tm = tmem + t * BKV;
    const uint32_t o_tm = tmem + C::kOBase + t * C::kOCols;
    const uint32_t p_tm = tmem + C::kPBase + t * C::kPStride;
    uint32_t kv = 0, qi = 0, g = 0, oi = 0, k = 0;
    for (;;) {
      const AttnItem it = next_item(k);
      if (it.len < 0) break;
      if (it.n_qt == 0) continue;
      const int qs = qi & 1;
      const uint32_t q_phase = (qi >> 1) & 1;
      ++qi;
      if (t >= it.n_qt) {  // inactive in this item: keep the K/V ring and Q slot accounting
        for (int j = 0; j < it.nkv; ++j, ++kv) {
          const int st = kv % C::STAGES;
          mbar_wait(&k_full[st], (kv / C::STAGES) & 1);  // never run ahead of the ring's phase
          if (elect_one()) mbar_arrive(&kv_empty[st]);
          __syncwarp();
        }
        if (elect_one()) mbar_arrive(&q_empty[qs]);
        __syncwarp();
        continue;
      }
      const uint32_t q_addr = smem_u32(tile_ptr(Lay::kQOff + qs * Lay::kQSlotBytes + t * C::kQBytes));
      mbar_wait(&q_full[qs], q_phase);
      // staggered start (as in attn_fwd_tc): the offset set on the first item persists
      if (t > 0 && oi == 0 && it.nkv > 1) mbar_wait(&p_full[0], 0);
      tc_fence_after();
      auto do_s = [&](int j) {
        const uint32_t kvj = kv + j;
        const int st = kvj % C::STAGES;
        mbar_wait(&k_full[st], (kvj / C::STAGES) & 1);
        if (g + j > 0) {
          if constexpr (C::kAlias) mbar_wait(&pv_done[t], (g + j - 1) & 1);  // PV_t has read P_t = S_t
          else mbar_wait(&s_free[t], (g + j - 1) & 1);
        }
        tc_fence_after();
        const uint32_t k_addr = smem_u32(tile_ptr(Lay::kKVOff + st * C::kStageBytes));
        if (elect_one()) {
          issue_s<HD, BKV, NQ>(s_tm, q_addr, k_addr);
          umma_commit(&s_full[t]);
          if (j == it.nkv - 1) umma_commit(&q_empty[qs]);  // last read of this item's Q
        }
        __syncwarp();
      };
      for (int j = 0; j <= it.nkv; ++j) {
        if (!C::kAlias && j < it.nkv) do_s(j);
        if (j > 0) {
          const uint32_t kvp = kv + j - 1;
          const int pst = kvp % C::STAGES;
          mbar_wait(&v_full[pst], (kvp / C::STAGES) & 1);
          mbar_wait(&p_full[t], (g + j - 1) & 1);
          if (j == 1 && oi > 0) mbar_wait(&o_free[t], (oi - 1) & 1);  // previous item's O_t read out
          tc_fence_after();
          const uint32_t v_addr = smem_u32(tile_ptr(Lay::kKVOff + pst * C::kStageBytes + C::kKVBytes));
          if (elect_one()) {
            issue_pv<HD, BKV, NQ>(o_tm, p_tm, v_addr, j == 1, smem_u32(smem + Lay::kOnesOff));
            umma_commit(&pv_done[t]);
            umma_commit(&kv_empty[pst]);
          }
          __syncwarp();
        }
        if (C::kAlias && j < it.nkv) do_s(j);
      }
      kv += it.nkv;
      g += it.nkv;
      ++oi;
    }
  } else {
    // ---------------------------------------------------------------- softmax warpgroups
    const int t = warp / (4 * C::kHalves);
    const int h = (warp >> 2) % C::kHalves;
    const uint32_t q4 = warp & 3;
    const uint32_t lane_base = (q4 * 32u) << 16;
    const uint32_t s_tm = tmem + t * BKV + lane_base;
    const uint32_t o_tm = tmem + C::kOBase + t * C::kOCols + lane_base;
    const uint32_t p_tm = tmem + C::kPBase + t * C::kPStride + lane_base;
    uint32_t g = 0, k = 0;
    for (;;) {
      const AttnItem it = next_item(k);
      if (it.len < 0) break;
      if (t >= it.n_qt) continue;  // also skips empty items (n_qt == 0)
      float m_used = -INFINITY, l = 0.f;
      for (int j = 0; j < it.nkv; ++j) {
        if constexpr (C::kSplit)
          softmax_tile_split<HD, BKV, NQ, SPEC>(s_tm, o_tm, p_tm, &s_full[t], &s_free[t], &pv_done[t], &p_full[t],
                                                g + j, j == 0, it.len - j * BKV, scale_log2, m_used, l, lane, h,
                                                s_red + (t * 4 + q4) * 64, 1 + t * 4 + q4);
        else
          softmax_tile<HD, BKV, NQ, SPEC>(s_tm, o_tm, p_tm, &s_full[t], &s_free[t], &pv_done[t], &p_full[t], g + j,
                                          j == 0, it.len - j * BKV, scale_log2, m_used, l, lane, false, t, j);
      }
      g += it.nkv;
      mbar_wait(&pv_done[t], (g - 1) & 1);
      tc_fence_after();
      if (h == 0) {
        l = final_l<HD, BKV, NQ>(o_tm, l);
        if constexpr (SPEC) flag_overflow(l, overflow_flag);
        const int row = it.q0 + t * kTcBQ + q4 * 32 + lane;
        store_o<HD>(o_tm, l, out + static_cast<int64_t>(it.s_begin + row) * d_model + it.head * HD, row < it.len);
        tc_fence_before();  // O_t reads complete before the next item's first PV overwrites it
        __syncwarp();
        if (lane == 0) mbar_arrive(&o_free[t]);
      } else if constexpr (SPEC) {
        flag_overflow(l, overflow_flag);
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == kMmaWarp) tmem_dealloc<512>(tmem);
}

template <int HD, int BKV, int NQ, bool PERSIST, bool SPEC>
static int launch_attn_cfg(const void* qkv, void* out, const int32_t* cu, int n_seq, int max_s, int heads,
                           float scale, int64_t total_rows, void* workspace, cudaStream_t stream) {
  using C = TcAttnCfg<HD, BKV, NQ>;
  using Lay = TcPersistLayout<HD, BKV, NQ>;
  const uint64_t ld = 3ull * heads * HD;
  const uint64_t dims[2] = {ld, static_cast<uint64_t>(total_rows)};
  const uint64_t strides[1] = {ld * 2};
  CUtensorMap tq, tqr, tkv, tkvr;
  const uint32_t bq[2] = {64, kTcBQ}, bqr[2] = {16, kTcBQ}, bkv[2] = {64, BKV}, bkvr[2] = {16, BKV};
  int rc = make_tmap_bf16(&tq, qkv, 2, dims, strides, bq, CU_TENSOR_MAP_SWIZZLE_128B);
  if (!rc) rc = make_tmap_bf16(&tkv, qkv, 2, dims, strides, bkv, CU_TENSOR_MAP_SWIZZLE_128B);
  if (!rc && C::kRem) rc = make_tmap_bf16(&tqr, qkv, 2, dims, strides, bqr, CU_TENSOR_MAP_SWIZZLE_32B);
  if (!rc && C::kRem) rc = make_tmap_bf16(&tkvr, qkv, 2, dims, strides, bkvr, CU_TENSOR_MAP_SWIZZLE_32B);
  if (rc) return rc;
  if (!C::kRem) { tqr = tq; tkvr = tkv; }
  const float scale_log2 = scale * 1.4426950408889634f;
  const int qblocks = (max_s + NQ * kTcBQ - 1) / (NQ * kTcBQ);
  const int64_t n_items = static_cast<int64_t>(qblocks) * heads * n_seq;
  if (n_items >= INT32_MAX) return set_error(MMK_ERR_UNSUPPORTED, "attention_tc: too many work items");
  static const bool lpt_on = [] {
    const char* e = getenv("MMK_ATTN_LPT");
    return e ? atoi(e) != 0 : true;
  }();
  const bool lpt = lpt_on && n_seq <= TcPersistLayout<HD, BKV, NQ>::kMaxSched;
  const int persist_grid = static_cast<int>(n_items < num_sms() ? n_items : num_sms());  // one CTA per SM
  __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(out);
  // workspace: [0] work-item counter of the main pass, [1] overflow flag, [2] counter of the exact redo
  int* ws = reinterpret_cast<int*>(workspace);
  cudaError_t me = cudaMemsetAsync(ws, 0, 4 * sizeof(int), stream);
  if (me != cudaSuccess) return set_cuda_error(me, "attention_tc: workspace reset");
  if constexpr (PERSIST || SPEC) {
    static std::atomic<uint64_t> attr_p{0}, attr_x{0};
    rc = ensure_smem_attr(reinterpret_cast<const void*>(attn_fwd_tc_persistent<HD, BKV, NQ, SPEC>), Lay::kSmem,
                          attr_p, "attention_tc: cudaFuncSetAttribute");
    if (!rc && SPEC)
      rc = ensure_smem_attr(reinterpret_cast<const void*>(attn_fwd_tc_persistent<HD, BKV, NQ, false>), Lay::kSmem,
                            attr_x, "attention_tc: cudaFuncSetAttribute");
    if (rc) return rc;
  }
  if constexpr (PERSIST) {
    me = launch_kernel(attn_fwd_tc_persistent<HD, BKV, NQ, SPEC>, dim3(persist_grid), dim3(C::kThreads), Lay::kSmem,
                       stream, 1, false, tq, tqr, tkv, tkvr, o, cu, n_seq, heads, qblocks, scale_log2, ws, ws + 1,
                       static_cast<const int*>(nullptr), lpt);
    if (me != cudaSuccess) return set_cuda_error(me, "attention_tc: launch");
  } else {
    static std::atomic<uint64_t> attr_done{0};
    rc = ensure_smem_attr(reinterpret_cast<const void*>(attn_fwd_tc<HD, BKV, NQ, SPEC>), C::kSmem, attr_done,
                          "attention_tc: cudaFuncSetAttribute");
    if (rc) return rc;
    if (n_seq > 65535 || heads > 65535) return set_error(MMK_ERR_UNSUPPORTED, "attention: too many sequences/heads");
    me = launch_kernel(attn_fwd_tc<HD, BKV, NQ, SPEC>, dim3(qblocks, heads, n_seq), dim3(C::kThreads), C::kSmem,
                       stream, 1, true, tq, tqr, tkv, tkvr, o, cu, heads, scale_log2, ws + 1);
    if (me != cudaSuccess) return set_cuda_error(me, "attention_tc: launch");
  }
  if constexpr (SPEC) {
    // exact redo of the whole launch, gated on the overflow flag (all CTAs exit at once when clear)
    me = launch_kernel(attn_fwd_tc_persistent<HD, BKV, NQ, false>, dim3(persist_grid), dim3(C::kThreads),
                       Lay::kSmem, stream, 1, !PERSIST, tq, tqr, tkv, tkvr, o, cu, n_seq, heads, qblocks, scale_log2, ws + 2,
                       static_cast<int*>(nullptr), static_cast<const int*>(ws + 1), lpt);
    if (me != cudaSuccess) return set_cuda_error(me, "attention_tc: launch");
  }
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? MMK_OK : set_cuda_error(e, "attention_tc: launch");
}

// Tile configuration per head_dim (measured on B200, profiles/r01_attention.md).  Both keep P in
// TMEM (A operand of the PV MMA read from tensor memory), which needs S + O + P <= 512 columns:
//   hd 80: 2 query tiles, 112-key tiles:  S 2x112 + O 2x80 + P 2x56 (aligned)  = 504 columns
//   hd 64: 3 query tiles,  64-key tiles:  S 3x64  + O 3x64 + P 3x32           = 480 columns
//   Persistent when a launch has more than two waves of work items (each item's prologue and
//   epilogue overlap its neighbours: Mllama bench attention 800 -> 820 TF/s in-step, CLIP 577-token
//   sequences +20 %); a single partial wave is faster one item per CTA.  MMK_ATTN_PERSIST=0/1
//   overrides for A/B runs.
template <int HD>
int launch_attn_tc(const void* qkv, void* out, const int32_t* cu, int n_seq, int max_s, int heads, float scale,
                   int64_t total_rows, void* workspace, cudaStream_t stream) {
  static const int force = [] {
    const char* e = getenv("MMK_ATTN_PERSIST");
    return e ? atoi(e) : -1;
  }();
  static const bool spec = [] {
    const char* e = getenv("MMK_ATTN_SPEC");
    return e ? atoi(e) != 0 : true;
  }();
#ifndef MMK_ATTN_HD80_BKV
#define MMK_ATTN_HD80_BKV 112
#define MMK_ATTN_HD80_NQ 2
#endif
  // hd 128 (InternViT): 2 query tiles, 64-key tiles: S 2x64 + O 2x128 + P 2x32 = 448 columns
  constexpr int BKV = HD == 64 ? 64 : HD == 128 ? 64 : MMK_ATTN_HD80_BKV;
  constexpr int NQ = HD == 64 ? 3 : HD == 128 ? 2 : MMK_ATTN_HD80_NQ;
  const int64_t items = static_cast<int64_t>((max_s + NQ * kTcBQ - 1) / (NQ * kTcBQ)) * heads * n_seq;
  const bool persist = force == 1 || (force != 0 && items > 2 * num_sms());
  if (persist) {
    if (spec) return launch_attn_cfg<HD, BKV, NQ, true, true>(qkv, out, cu, n_seq, max_s, heads, scale, total_rows, workspace, stream);
    return launch_attn_cfg<HD, BKV, NQ, true, false>(qkv, out, cu, n_seq, max_s, heads, scale, total_rows, workspace, stream);
  }
  if (spec) return launch_attn_cfg<HD, BKV, NQ, false, true>(qkv, out, cu, n_seq, max_s, heads, scale, total_rows, workspace, stream);
  return launch_attn_cfg<HD, BKV, NQ, false, false>(qkv, out, cu, n_seq, max_s, heads, scale, total_rows, workspace, stream);
}

template int launch_attn_tc<64>(const void*, void*, const int32_t*, int, int, int, float, int64_t, void*, cudaStream_t);
template int launch_attn_tc<80>(const void*, void*, const int32_t*, int, int, int, float, int64_t, void*, cudaStream_t);
template int launch_attn_tc<128>(const void*, void*, const int32_t*, int, int, int, float, int64_t, void*, cudaStream_t);

}  // namespace mmk

#ifdef MMK_ATTN_TRACE
extern "C" int mmk_debug_attn_trace(long long* host_out) {
  return cudaMemcpyFromSymbol(host_out, mmk::g_attn_trace, sizeof(mmk::g_attn_trace)) == cudaSuccess ? 0 : 3;
}
#endif
