/*
 * oracle/preprocess.c — TEST INFRASTRUCTURE ONLY (never linked into the product).
 *
 * Plain-C restatement of K1 (paper_2502_00937_b200/csrc/mmk_preprocess.cu), the checker the
 * device kernel is compared with bit for bit.  Only tests/, __graft_entry__.smoke() and
 * bench.py's CPU legs load it (through oracle/preprocess.py).
 *
 * The reference has no pixel arithmetic ("only counts and latencies"); the geometry
 * is the builder's definition, aligned with transformers' Mllama / CLIP image
 * processors (canvas and resized size from oracle/tile_plan.c, which reproduces
 * get_image_size_fit_to_canvas / get_resize_output_image_size exactly — tests/test_k1_hf_pin.py).
 *
 * Sampling is torch.nn.functional.interpolate(mode="bilinear", align_corners=False,
 * antialias=False) EXACTLY, including its float32 rounding (pinned bit for bit in
 * tests/test_k1_hf_pin.py):
 *     scale = (float)in / (float)out
 *     src   = max(fmaf(i + 0.5f, scale, -0.5f), 0);  i0 = min(floor(src), in-1);
 *     i1    = min(i0 + 1, in-1);  l1 = src - i0;  l0 = 1 - l1
 *     row   = fmaf(l0x, p[i0], l1x * p[i1])            (per source row, per channel)
 *     v     = fmaf(l0y, row(y0), l1y * row(y1))
 * then normalisation as one FMA with float32 constants, out = fmaf(v, 1/(255 std), -mean/std),
 * and one round-to-nearest-even to bf16.  Padding pixels (Mllama canvas beyond the resized
 * image) are v = 0 before normalisation, as HF pads.
 * Compiled with -ffp-contract=off: every float operation is written out; fmaf is libm's
 * correctly rounded fused multiply-add.
 */
#include <math.h>
#include <stdint.h>

static uint16_t bf16_rn(float x) {
  union { float f; uint32_t u; } v;
  v.f = x;
  return (uint16_t)((v.u + 0x7FFFu + ((v.u >> 16) & 1u)) >> 16);
}

typedef struct { int i0, i1; float l0, l1; } Tap;

static Tap tap(int i, int in, int out) {
  Tap t;
  float scale = (float)in / (float)out;
  float src = fmaf((float)i + 0.5f, scale, -0.5f);
  int i0;
  if (src < 0.f) src = 0.f;
  i0 = (int)floorf(src);
  if (i0 > in - 1) i0 = in - 1;
  t.i0 = i0;
  t.i1 = i0 + 1 < in - 1 ? i0 + 1 : in - 1;
  t.l1 = src - (float)i0;
  t.l0 = 1.0f - t.l1;
  return t;
}

/* one channel value of the source image */
static float px(const uint8_t* img, int w, int h, int chw, int y, int x, int c) {
  return (float)(chw ? img[(int64_t)c * h * w + (int64_t)y * w + x] : img[((int64_t)y * w + x) * 3 + c]);
}

/* bilinear sample of channel c of img (w x h) resized to (rw x rh) at output pixel (X, Y) */
float oracle_bilinear(const uint8_t* img, int w, int h, int chw, int rw, int rh, int X, int Y, int c) {
  Tap tx = tap(X, w, rw), ty = tap(Y, h, rh);
  float top = fmaf(tx.l0, px(img, w, h, chw, ty.i0, tx.i0, c), tx.l1 * px(img, w, h, chw, ty.i0, tx.i1, c));
  float bot = fmaf(tx.l0, px(img, w, h, chw, ty.i1, tx.i0, c), tx.l1 * px(img, w, h, chw, ty.i1, tx.i1, c));
  return fmaf(ty.l0, top, ty.l1 * bot);
}

/* Whole batch, same arguments as the device ABI mmk_preprocess; out = bf16 bits
   [total_tiles * (T/p)^2, k_pad] (K padding zeroed). */
void oracle_preprocess(const uint8_t* src, const int64_t* src_off, int chw, const int32_t* w, const int32_t* h,
                       const int64_t* tile_off, const int32_t* geom, int n, int T, int p, int k_pad, int mode,
                       int thumb, const float* scale3, const float* shift3, uint16_t* out) {
  const int ps = T / p, pp = p * p;
  int i;
  for (i = 0; i < n; ++i) {
    const uint8_t* img = src + src_off[i];
    const int W = w[i], H = h[i], cols = geom[4 * i + 1], nw = geom[4 * i + 2], nh = geom[4 * i + 3];
    const int ntile = (int)(tile_off[i + 1] - tile_off[i]);
    int t;
    for (t = 0; t < ntile; ++t) {
      const int is_thumb = thumb && ntile > 1 && t == ntile - 1;
      int ox = 0, oy = 0, rw = nw, rh = nh, clip = 0, yy, xx;
      if (is_thumb) { rw = T; rh = T; }
      else if (mode == 0) { ox = (t % cols) * T; oy = (t / cols) * T; clip = 1; }
      else { ox = (nw - T) / 2; oy = (nh - T) / 2; }
      for (yy = 0; yy < ps * p; ++yy) {    /* the patch grid: floor(T / p) patches per side */
        for (xx = 0; xx < ps * p; ++xx) {
          const int X = ox + xx, Y = oy + yy;
          const int64_t patch = (tile_off[i] + t) * (int64_t)ps * ps + (yy / p) * ps + (xx / p);
          int c;
          for (c = 0; c < 3; ++c) {
            float v = 0.f;
            if (!clip || (X < nw && Y < nh)) v = oracle_bilinear(img, W, H, chw, rw, rh, X, Y, c);
            out[patch * k_pad + c * pp + (yy % p) * p + (xx % p)] = bf16_rn(fmaf(v, scale3[c], shift3[c]));
          }
        }
      }
      {
        int64_t q0 = (tile_off[i] + t) * (int64_t)ps * ps, q;
        for (q = q0; q < q0 + (int64_t)ps * ps; ++q) {
          int k;
          for (k = 3 * pp; k < k_pad; ++k) out[q * k_pad + k] = 0;
        }
      }
    }
  }
}

/* The whole image resized (float32 [rh][rw][3]), for the torch pin in tests/test_k1_hf_pin.py. */
void oracle_resize(const uint8_t* img, int w, int h, int chw, int rw, int rh, float* out) {
  int y, x, c;
  for (y = 0; y < rh; ++y)
    for (x = 0; x < rw; ++x)
      for (c = 0; c < 3; ++c) out[((int64_t)y * rw + x) * 3 + c] = oracle_bilinear(img, w, h, chw, rw, rh, x, y, c);
}
