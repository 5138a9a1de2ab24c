// mmk_preprocess.cu — K1: fused uint8 HWC/CHW -> bilinear resize -> pad/crop -> normalize ->
// tile -> patchify, written straight into the bf16 patch matrix the patch-embed GEMM reads.
//
// Replaces the modelled CPU lane `LatencyProfile.preprocess_latency` (reference
// pkg/src/lmmsim/profiles.py:128-134, driven from engine.py:639-657).  The reference has no
// pixel arithmetic; the geometry is the builder's definition and the
// sampler is torch's bilinear (F.interpolate, align_corners=False, antialias=False) bit for bit:
//     src = max(fma(i + 0.5, in/out, -0.5), 0); i0 = min(floor(src), in-1); l1 = src - i0
//     row = fma(l0x, p[x0], l1x * p[x1]);  v = fma(l0y, row(y0), l1y * row(y1))
//     out = bf16_rn(fma(v, 1/(255 std), -mean/std))
// restated op for op in oracle/preprocess.c (bit-identical; pinned against torch and the HF
// processors in tests/test_k1_hf_pin.py).
//
// One CTA per (tile, patch-row band of p pixel rows, column part).  Design (HBM-bound byte work):
//  * the band's source rows are staged in shared memory once, with coalesced 16-byte loads of
//    each row's column span (only the rows the band's bilinear taps touch; chunked by rows when
//    the span is wide);
//  * separable resampling: each thread owns two adjacent output columns (fixed column taps) and
//    walks the band's rows keeping the horizontally interpolated values of the two source rows
//    it currently needs in registers, so a source row is interpolated once per column, not once
//    per output row that uses it;
//  * a source pixel's three channels are read as 32-bit shared-memory words and turned into
//    fp32 with byte permutes + the 2^23 magic (exact, FMA pipe); the two columns of a thread are
//    one f32x2 pair through every multiply/FMA (FMUL2/FFMA2);
//  * the normalised values land in the band's patch vectors in shared memory as bf16x2 (the two
//    columns are adjacent px of one patch row), and the band — one contiguous run of the patch
//    matrix — leaves with a single bulk asynchronous copy (cp.async.bulk shared -> global).
#include "sm100_common.cuh"
#include "mmk_internal.h"

namespace mmk {

constexpr int kMaxPatch = 64;          // patch edge limit
constexpr int kMaxSlots = 2 * kMaxPatch;
#ifndef MMK_PREP_STAGE_KB
#define MMK_PREP_STAGE_KB 24
#endif
#ifndef MMK_PREP_MAX_COLS
#define MMK_PREP_MAX_COLS 1024  // output columns per CTA (two per thread)
#endif
constexpr int kStageBytes = MMK_PREP_STAGE_KB * 1024;  // staged source rows per chunk (3 CTAs/SM with a 47 KB band)
constexpr int kPrepMaxThreads = 512;

struct PrepImage {
  int img, slot, tiles, w, h, rows, cols, nw, nh;
  int64_t off;
};

struct Tap {
  int i0, i1;
  float l0, l1;
};

// torch upsample_bilinear2d (align_corners=False) source tap of output index i.
MMK_DEV Tap bilinear_tap(int i, int in, float scale) {
  Tap t;
  float s = __fmaf_rn(__fadd_rn(static_cast<float>(i), 0.5f), scale, -0.5f);
  s = fmaxf(s, 0.f);
  t.i0 = min(static_cast<int>(floorf(s)), in - 1);
  t.i1 = min(t.i0 + 1, in - 1);
  t.l1 = __fsub_rn(s, static_cast<float>(t.i0));
  t.l0 = __fsub_rn(1.f, t.l1);
  return t;
}

MMK_DEV uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}
MMK_DEV uint32_t lds_u32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}
MMK_DEV uint32_t lds_u8(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}

constexpr uint32_t kMagic = 0x4B000000u;  // 2^23: (kMagic | b) as float == 2^23 + b exactly
// (magic_a, magic_b) -> exact (b_a, b_b) as fp32
MMK_DEV float2 u8pair_to_f32(uint32_t ma, uint32_t mb) {
  return __fadd2_rn(make_float2(__uint_as_float(ma), __uint_as_float(mb)), make_float2(-8388608.f, -8388608.f));
}

// Source pixels of one output column in a staged HWC row: the three channels of x0 (p0) and x1
// (p1) as magic words.  `base` = shared address of byte 0 of pixel x0; `sel1` gathers x1's bytes
// (x1 == x0 + 1: bytes 3..5; x1 == x0 at the right edge: bytes 0..2).
MMK_DEV void hwc_pixels(uint32_t base, uint32_t sel1, uint32_t (&p0)[3], uint32_t (&p1)[3]) {
  const uint32_t wa = base & ~3u, sh = (base & 3u) * 8u;
  const uint32_t w0 = lds_u32(wa), w1 = lds_u32(wa + 4), w2 = lds_u32(wa + 8);
  const uint32_t lo = __funnelshift_r(w0, w1, sh), hi = __funnelshift_r(w1, w2, sh);  // bytes 0..3, 4..7
  const uint32_t q1 = prmt(lo, hi, sel1);
  p0[0] = prmt(lo, kMagic, 0x7440); p0[1] = prmt(lo, kMagic, 0x7441); p0[2] = prmt(lo, kMagic, 0x7442);
  p1[0] = prmt(q1, kMagic, 0x7440); p1[1] = prmt(q1, kMagic, 0x7441); p1[2] = prmt(q1, kMagic, 0x7442);
}

#ifndef MMK_PREP_MAXNREG
#define MMK_PREP_MAXNREG 72  // 3 CTAs of 288 threads per SM (Mllama bands)
#endif
// P = patch edge (compile time for the presets' 14 and 16; 0 = runtime `p`)
template <bool CHW, int P>
__global__ void __maxnreg__(MMK_PREP_MAXNREG)
preprocess_kernel(const uint8_t* __restrict__ src, const int64_t* __restrict__ src_off, const int32_t* __restrict__ w,
                  const int32_t* __restrict__ h, const int64_t* __restrict__ tile_off,
                  const int32_t* __restrict__ geom, int n, int T, int p_rt, int k_pad, int mode, int thumb,
                  const float* __restrict__ scale3, const float* __restrict__ shift3,
                  __nv_bfloat16* __restrict__ patches, int parts, int band_bytes) {
  extern __shared__ __align__(128) uint8_t prep_smem[];
  __nv_bfloat16* band = reinterpret_cast<__nv_bfloat16*>(prep_smem);  // [patches of the part][k_pad]
  uint8_t* stage = prep_smem + band_bytes;                             // staged source rows
  __shared__ PrepImage meta;
  __shared__ float s_nrm[6];
  __shared__ int s_y0[kMaxPatch];
  __shared__ float4 s_rowtab[kMaxPatch];              // per band row: (slot of its lower source row, l0y, l1y, -)
  __shared__ int s_srow[kMaxSlots];                   // source row of each slot (ascending)
  __shared__ int s_rowoff[kMaxSlots * 3];             // per (chunk slot, plane): stage byte of pixel 0
  __shared__ int s_xa, s_rs, s_cap, s_nslot;
  __shared__ __align__(8) uint64_t s_bar;  // staging: bulk-copy completion
  griddep_wait();  // PDL: inputs come from the preceding kernel
  griddep_launch_dependents();

  const int p = P ? P : p_rt;
  const int per_side = T / p;
  const int pc_per = (per_side + parts - 1) / parts;  // patches per column part
  const int band_id = blockIdx.x / parts, part = blockIdx.x % parts;
  const int g = band_id / per_side;                   // global tile
  const int pr = band_id % per_side;                  // patch row inside the tile
  const int pc0 = part * pc_per, pc1 = min(per_side, pc0 + pc_per);
  const int tid = threadIdx.x;
  if (tid < 32) {
    // warp-parallel search for the last image with tile_off[i] <= g: each round narrows the
    // range 32x (one round for batches of <= 33 images)
    int lo = 0, hi = n;  // answer in [lo, hi)
    while (hi - lo > 1) {
      const int step = (hi - lo + 31) / 32;
      const int idx = lo + tid * step;
      const bool ok = idx < hi && tile_off[idx] <= g;
      const uint32_t bal = __ballot_sync(0xffffffffu, ok);
      const int k = 31 - __clz(bal);  // bal != 0: tile_off[lo] <= g
      lo = lo + k * step;
      hi = min(hi, lo + step);
    }
    if (tid == 0) {
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
  } else if (tid < 38) {
    const int c = tid - 32;
    s_nrm[c] = c < 3 ? scale3[c] : shift3[c - 3];
  } else if (tid == 38) {
    mbar_init(&s_bar, 1);
    fence_barrier_init();
  }
  __syncthreads();
  const PrepImage m = meta;
  const uint8_t* img = src + m.off;
  const bool is_thumb = thumb && m.tiles > 1 && m.slot == m.tiles - 1;
  int ox = 0, oy = 0, rw = m.nw, rh = m.nh;  // canvas origin of this tile, resize target
  bool clip = false;                         // Mllama canvas: pixels past the resized image are padding
  if (is_thumb) {
    rw = T; rh = T;
  } else if (mode == 0) {
    ox = (m.slot % m.cols) * T;
    oy = (m.slot / m.cols) * T;
    clip = true;
  } else {
    ox = (m.nw - T) / 2;
    oy = (m.nh - T) / 2;
  }
  const float sclx = __fdiv_rn(static_cast<float>(m.w), static_cast<float>(rw));
  const float scly = __fdiv_rn(static_cast<float>(m.h), static_cast<float>(rh));
  const int row_lim = clip ? max(0, min(p, m.nh - (oy + pr * p))) : p;  // band rows inside the image
  const int c_first = ox + pc0 * p;                                       // first canvas column of the part
  const int c_valid = clip ? max(0, min(pc1 * p, m.nw - ox) - pc0 * p) : (pc1 - pc0) * p;
  constexpr int planes = CHW ? 3 : 1;
  constexpr int bpp = CHW ? 1 : 3;  // bytes per pixel inside one staged plane row
  const int64_t plane = CHW ? static_cast<int64_t>(m.h) * m.w : 0;
  const int64_t row_bytes = CHW ? m.w : 3ll * m.w;

  // ---- 0) row taps of the band and its distinct source rows ("slots", ascending), column span
  //      of the part, staging plan.  Warp 0, lane = band row: a source row is new unless the
  //      previous band row already reads it; slot numbers are prefix counts of the new rows.
  // Rows are "virtual": a band row reads y0 and y0 + 1, and a virtual row v is the source row
  // min(v, h - 1) — at the bottom edge torch's clamped y1 == y0 reads the same pixels, and every
  // band row reads two consecutive slots (s1 - 1, s1).
  if (tid < 32) {
    Tap t{0, 0, 0.f, 0.f};
    if (tid < p) {
      t = bilinear_tap(oy + pr * p + tid, m.h, scly);
      s_y0[tid] = t.i0;
    }
    if (p <= 32) {
      const int y0 = t.i0, y1 = t.i0 + 1;
      const int y0p = __shfl_up_sync(0xffffffffu, y0, 1), y1p = y0p + 1;
      const bool valid = tid < row_lim;
      const bool f0 = valid && (tid == 0 || (y0 != y0p && y0 != y1p));
      const bool f1 = valid && (tid == 0 || y1 != y1p);
      const uint32_t b0 = __ballot_sync(0xffffffffu, f0), b1 = __ballot_sync(0xffffffffu, f1);
      const uint32_t lt = (1u << tid) - 1u;
      const int P0 = __popc(b0 & lt) + __popc(b1 & lt), P1 = P0 + f0;
      const int s1 = f1 ? P1 : P1 - 1;  // slot of y0 + 1 (slot of y0 = s1 - 1)
      if (f0) s_srow[P0] = min(y0, m.h - 1);
      if (f1) s_srow[P1] = min(y1, m.h - 1);
      if (valid) s_rowtab[tid] = make_float4(__int_as_float(s1), t.l0, t.l1, 0.f);
      if (tid == 0) s_nslot = __popc(b0) + __popc(b1);
    }
  } else if (tid == 32) {
    const int xa = c_valid > 0 ? bilinear_tap(c_first, m.w, sclx).i0 : 0;
    const int xb = c_valid > 0 ? bilinear_tap(c_first + c_valid - 1, m.w, sclx).i1 : 0;
    s_xa = xa;
    // bytes of one staged plane row: the span, its 16-byte misalignment, and 16 bytes of slack
    // for the 12-byte word window read at the last pixel
    const int rs = ((bpp * (xb - xa + 1) + 15 + 16) + 15) & ~15;
    s_rs = rs;
    s_cap = kStageBytes / (planes * rs);
  }
  if (p > 32) {  // generic patch sizes: the same plan, serially
    __syncthreads();
    if (tid == 0) {
      int ns = 0, last = -1;
      for (int iy = 0; iy < row_lim; ++iy) {
        const int y0 = s_y0[iy];
        const Tap t = bilinear_tap(oy + pr * p + iy, m.h, scly);
        for (int v = max(y0, last + 1); v <= y0 + 1; ++v) { s_srow[ns++] = min(v, m.h - 1); last = v; }
        s_rowtab[iy] = make_float4(__int_as_float(ns - 1), t.l0, t.l1, 0.f);  // last == y0 + 1
      }
      s_nslot = ns;
    }
  }

  // ---- the thread's two output columns (adjacent px of one patch row; p is even)
  const int xl = 2 * tid;                      // local column inside the part
  const int ncols = (pc1 - pc0) * p;
  const bool active = xl < ncols;
  Tap ta{0, 0, 0.f, 0.f}, tb{0, 0, 0.f, 0.f};
  __syncthreads();
  const int xa = s_xa;
  if (active) {
    if (xl < c_valid) ta = bilinear_tap(c_first + xl, m.w, sclx);
    else ta = Tap{xa, xa, 0.f, 0.f};           // padding column: weights 0 -> v = +0, as the oracle
    if (xl + 1 < c_valid) tb = bilinear_tap(c_first + xl + 1, m.w, sclx);
    else tb = Tap{xa, xa, 0.f, 0.f};
  }
  const float2 l0x = make_float2(ta.l0, tb.l0), l1x = make_float2(ta.l1, tb.l1);
  const uint32_t sel_a = ta.i1 > ta.i0 ? 0x0543u : 0x0210u, sel_b = tb.i1 > tb.i0 ? 0x0543u : 0x0210u;
  const int pp = p * p;
  const int pcl = xl / p, ix = xl - pcl * p;
  uint32_t* band32 = reinterpret_cast<uint32_t*>(band) + ((pcl * k_pad + ix) >> 1);  // (patch, c=0, py=0, px=ix)
  const float2 sc0 = make_float2(s_nrm[0], s_nrm[0]), sc1 = make_float2(s_nrm[1], s_nrm[1]),
               sc2 = make_float2(s_nrm[2], s_nrm[2]);
  const float2 sh0 = make_float2(s_nrm[3], s_nrm[3]), sh1 = make_float2(s_nrm[4], s_nrm[4]),
               sh2 = make_float2(s_nrm[5], s_nrm[5]);

  // zero the K padding of every patch vector of the part (the bulk copy moves whole vectors)
  const int kreal = 3 * pp, padw = k_pad - kreal;
  for (int q = tid; q < (pc1 - pc0) * padw; q += blockDim.x) {
    const int pc = q / padw;
    band[pc * k_pad + kreal + (q - pc * padw)] = __float2bfloat16_rn(0.f);
  }
  auto store_row = [&](int iy, float2 v0, float2 v1, float2 v2) {
    uint32_t* o = band32 + iy * (p >> 1);
    const float2 a = __ffma2_rn(v0, sc0, sh0), b = __ffma2_rn(v1, sc1, sh1), c = __ffma2_rn(v2, sc2, sh2);
    o[0] = pack_bf16x2(a.x, a.y);
    o[pp >> 1] = pack_bf16x2(b.x, b.y);
    o[pp] = pack_bf16x2(c.x, c.y);
  };
  const uint32_t stage_s = smem_u32(stage), rowoff_s = smem_u32(s_rowoff);
  const int nslot = s_nslot, rs = s_rs, cap = s_cap;
  // a source row span wider than half the staging buffer (> ~4300 px): read straight from global
  const bool direct = cap < 2;
  const int chunk = direct ? kMaxSlots : cap;

  // horizontal interpolation of the thread's two columns on one source row (chunk slot s, row y)
  auto hrow = [&](int s, int y, float2 (&H)[3]) {
    uint32_t a0[3], a1[3], b0[3], b1[3];
    if (direct) {
      const uint8_t* r = img + static_cast<int64_t>(y) * row_bytes;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const uint8_t* rc = r + c * plane + (CHW ? 0 : c);
        a0[c] = kMagic | __ldg(rc + bpp * ta.i0); a1[c] = kMagic | __ldg(rc + bpp * ta.i1);
        b0[c] = kMagic | __ldg(rc + bpp * tb.i0); b1[c] = kMagic | __ldg(rc + bpp * tb.i1);
      }
    } else if constexpr (!CHW) {
      int ro;
      asm volatile("ld.shared.u32 %0, [%1];" : "=r"(ro) : "r"(rowoff_s + 4u * s));
      const uint32_t rb = stage_s + ro;
      hwc_pixels(rb + 3u * ta.i0, sel_a, a0, a1);
      hwc_pixels(rb + 3u * tb.i0, sel_b, b0, b1);
    } else {
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const uint32_t rb = stage_s + s_rowoff[3 * s + c];
        a0[c] = kMagic | lds_u8(rb + ta.i0); a1[c] = kMagic | lds_u8(rb + ta.i1);
        b0[c] = kMagic | lds_u8(rb + tb.i0); b1[c] = kMagic | lds_u8(rb + tb.i1);
      }
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const float2 q0 = u8pair_to_f32(a0[c], b0[c]), q1 = u8pair_to_f32(a1[c], b1[c]);
      H[c] = __ffma2_rn(l0x, q0, __fmul2_rn(l1x, q1));
    }
  };

  // ---- 1..n) chunks of slots: stage their source rows, interpolate each slot once, emit the
  //      band rows whose lower source row it is
  float2 HA[3], HB[3];  // interpolated source rows of the even / odd slots
  int iy = 0;
  const uint32_t rowtab_s = smem_u32(s_rowtab), srow_s = smem_u32(s_srow);
  // band rows whose lower source row is slot sg (its upper row is slot sg - 1)
  auto emit = [&](int sg, const float2 (&Hu)[3], const float2 (&Hl)[3]) {
    for (; iy < row_lim; ++iy) {
      float4 rt;
      asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                   : "=f"(rt.x), "=f"(rt.y), "=f"(rt.z), "=f"(rt.w)
                   : "r"(rowtab_s + 16u * iy));
      if (__float_as_int(rt.x) != sg) break;
      const float2 l0y = make_float2(rt.y, rt.y), l1y = make_float2(rt.z, rt.z);
      store_row(iy, __ffma2_rn(l0y, Hu[0], __fmul2_rn(l1y, Hl[0])), __ffma2_rn(l0y, Hu[1], __fmul2_rn(l1y, Hl[1])),
                __ffma2_rn(l0y, Hu[2], __fmul2_rn(l1y, Hl[2])));
    }
  };
  const int nwarps = blockDim.x >> 5, wid = tid >> 5, lane = tid & 31;
  for (int sf = 0; sf < nslot; sf += chunk) {
    const int nsl = min(chunk, nslot - sf);
    if (!direct) {
      if (sf > 0) __syncthreads();  // the previous chunk's rows are no longer read
      // stage: chunk slot s, plane c -> stage + (s*planes + c)*rs, copied from the 16-byte aligned
      // address at or below the span start.  Warp 0 issues a bulk copy per row, a lane per row (the
      // TMA engine moves the bytes; completion counted on s_bar) for the whole 16-byte vectors inside
      // the image; the vector holding the image's last byte and any past it go by cp.async with zero
      // fill.  Reads stay inside [align16_down(image), image end): the aligned bytes before an
      // image share its allocation (allocations are >= 256-byte aligned).
      const uint8_t* img_end = img + (CHW ? 3 * plane : row_bytes * m.h);
      if (wid == 0) {  // warp 0: lane l owns rows l, l + 32, ...
        const int nrow = nsl * planes;
        auto row_src = [&](int r, const uint8_t*& span, const uint8_t*& gA) {
          const int s = CHW ? r / 3 : r, c = CHW ? r - 3 * s : 0;
          span = img + c * plane + static_cast<int64_t>(s_srow[sf + s]) * row_bytes + bpp * xa;
          gA = reinterpret_cast<const uint8_t*>(reinterpret_cast<uintptr_t>(span) & ~uintptr_t(15));
        };
        auto whole = [&](const uint8_t* gA) {  // bytes of whole vectors inside the image
          const int64_t left = img_end - gA;
          return left >= rs ? static_cast<uint32_t>(rs) : static_cast<uint32_t>(left > 0 ? left & ~int64_t(15) : 0);
        };
        uint32_t tx = 0;
        for (int r = lane; r < nrow; r += 32) {
          const uint8_t *span, *gA;
          row_src(r, span, gA);
          tx += whole(gA);
          s_rowoff[r] = r * rs + static_cast<int>(span - gA) - bpp * xa;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) tx += __shfl_xor_sync(0xffffffffu, tx, o);
        if (lane == 0) mbar_arrive_expect_tx(&s_bar, tx);
        __syncwarp();
        const uint32_t bar = smem_u32(&s_bar);
        for (int r = lane; r < nrow; r += 32) {
          const uint8_t *span, *gA;
          row_src(r, span, gA);
          const uint32_t full = whole(gA), dst = stage_s + r * rs;
          if (full)
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(dst), "l"(gA), "r"(full), "r"(bar) : "memory");
          for (uint32_t v = full; v < static_cast<uint32_t>(rs); v += 16) {
            const int64_t left = img_end - (gA + v);
            const uint32_t nb = left >= 16 ? 16u : (left > 0 ? static_cast<uint32_t>(left) : 0u);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst + v), "l"(nb ? gA + v : img),
                         "r"(nb)
                         : "memory");
          }
        }
        asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
      }
      mbar_wait(&s_bar, static_cast<uint32_t>(sf / chunk) & 1u);
      __syncthreads();
    }
    if (active) {
      for (int s = 0; s < nsl; ++s) {
        const int sg = sf + s;
        int y;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(y) : "r"(srow_s + 4u * sg));
        if (sg & 1) {
          hrow(s, y, HB);
          emit(sg, HA, HB);
        } else {
          hrow(s, y, HA);
          emit(sg, HB, HA);
        }
      }
    }
  }
  // rows past the resized image (Mllama canvas padding): v = 0 before normalisation
  if (active) {
    const float2 z = make_float2(0.f, 0.f);
    for (int r = row_lim; r < p; ++r) store_row(r, z, z, z);
  }
  // ---- out) the part is one contiguous run of the patch matrix: one bulk copy
  fence_proxy_async();
  __syncthreads();
  if (tid == 0) {
    __nv_bfloat16* dst = patches + ((static_cast<int64_t>(g) * per_side + pr) * per_side + pc0) * k_pad;
    const uint32_t bytes = static_cast<uint32_t>((pc1 - pc0) * k_pad * 2);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(band)),
                 "r"(bytes)
                 : "memory");
    tma_store_commit();
    tma_store_wait_read<0>();
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
  // the patch grid is floor(tile_px / patch_px) per side (SigLIP 384 / 14 -> 27, trailing pixels unused,
  // as a stride-p "valid" convolution)
  if (patch_px < 1 || tile_px < patch_px) return set_error(MMK_ERR_ARG, "preprocess: tile_px < patch_px");
  if (patch_px > kMaxPatch) return set_error(MMK_ERR_UNSUPPORTED, "preprocess: patch_px %d > %d", patch_px, kMaxPatch);
  if (patch_px % 2) return set_error(MMK_ERR_UNSUPPORTED, "preprocess: odd patch_px %d", patch_px);
  if (k_pad < 3 * patch_px * patch_px || k_pad % 8 != 0) return set_error(MMK_ERR_ARG, "preprocess: bad k_pad");
  if (mode != 0 && mode != 1) return set_error(MMK_ERR_ARG, "preprocess: mode must be 0 or 1");
  if (reinterpret_cast<uintptr_t>(patches) & 15) return set_error(MMK_ERR_ARG, "preprocess: patches not 16B aligned");
  if (n == 0 || total_tiles == 0) return MMK_OK;
  const int per_side = tile_px / patch_px;
  int parts = 1;  // column parts per band: two columns per thread, at most kPrepMaxThreads threads
  while ((per_side + parts - 1) / parts * patch_px > MMK_PREP_MAX_COLS) ++parts;
  const int pc_per = (per_side + parts - 1) / parts;
  const int threads = (pc_per * patch_px / 2 + 31) / 32 * 32;
  const int band_bytes = (pc_per * k_pad * 2 + 127) & ~127;
  const int smem = band_bytes + kStageBytes;
  if (smem > 200 * 1024) return set_error(MMK_ERR_UNSUPPORTED, "preprocess: patch row band of %d bytes", band_bytes);
  const int blocks = total_tiles * per_side * parts;
  auto* out = reinterpret_cast<__nv_bfloat16*>(patches);
  auto go = [&](auto kern) -> int {
    // max shared-memory carveout (3 Mllama bands per SM need 3 x 74 KB) + the dynamic size; set
    // on every call (two attribute writes, cheap next to the launch)
    cudaError_t a = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                         cudaSharedmemCarveoutMaxShared);
    if (a == cudaSuccess) a = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (a != cudaSuccess) return set_cuda_error(a, "preprocess: smem attribute");
    const cudaError_t le = launch_kernel(kern, dim3(blocks), dim3(threads), smem, stream, 1, total_tiles <= 64, src,
                                         src_off, w, h, tile_off, geom, n, tile_px, patch_px, k_pad, mode, thumbnail,
                                         scale3, shift3, out, parts, band_bytes);
    if (le != cudaSuccess) return set_cuda_error(le, "preprocess: launch");
    return MMK_OK;
  };
  int rc;
  if (src_chw) {
    rc = patch_px == 14 ? go(preprocess_kernel<true, 14>) : patch_px == 16 ? go(preprocess_kernel<true, 16>)
                                                                           : go(preprocess_kernel<true, 0>);
  } else {
    rc = patch_px == 14 ? go(preprocess_kernel<false, 14>) : patch_px == 16 ? go(preprocess_kernel<false, 16>)
                                                                            : go(preprocess_kernel<false, 0>);
  }
  if (rc != MMK_OK) return rc;
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? MMK_OK : set_cuda_error(e, "preprocess: launch");
}
