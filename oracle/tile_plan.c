/*
 * oracle/tile_plan.c — TEST INFRASTRUCTURE ONLY (never linked into the product).
 *
 * Plain-C restatement of the image path's integer semantics, used as the checker for the
 * device kernel mmk_tile_plan (K0).  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg load it.
 *
 * Follows the reference:
 *   tile_count   /root/reference/pkg/src/lmmsim/core.py:58-69
 *                  grid = ceil(w/T)*ceil(h/T); +1 thumbnail if thumbnail_tile and grid>1;
 *                  min(cap); w<1 or h<1 -> SpecError (here: tiles 0, counted in *bad)
 *   image_tokens core.py:72-74 ; Request.total_tiles / total_image_tokens core.py:110-120
 * and the builder-defined canvas geometry of DESIGN.md §3 (rows x cols, resized size).
 * PINNED: tests/golden/tiling.json holds the reference's own tile_count / image_tokens for
 * ~4.7k dims x 9 specs; tests/test_oracle.py checks this file against it.
 */
#include <math.h>
#include <stdint.h>

static int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

/* min(cw/w, ch/h) as num/den */
static void fit(int64_t w, int64_t h, int64_t cw, int64_t ch, int64_t* num, int64_t* den) {
  if (cw * h <= ch * w) { *num = cw; *den = w; } else { *num = ch; *den = h; }
}

/* geom[5] = {tiles, rows, cols, new_w, new_h} */
void oracle_plan_one(int64_t w, int64_t h, int64_t T, int64_t cap, int thumb, int mode, int32_t* geom) {
  int64_t gw, gh, grid, tiles, main_tiles, rows, cols;
  geom[0] = geom[1] = geom[2] = geom[3] = geom[4] = 0;
  if (w < 1 || h < 1) return;
  gw = cdiv(w, T);
  gh = cdiv(h, T);
  grid = gw * gh;
  tiles = grid;
  if (thumb && grid > 1) tiles = grid + 1;
  if (tiles > cap) tiles = cap;
  main_tiles = (thumb && tiles > 1) ? tiles - 1 : tiles;
  if (main_tiles == grid) {
    rows = gh;
    cols = gw;
  } else {
    /* Mllama get_optimal_tiled_canvas criterion over r*c == main_tiles:
       smallest scale >= 1 if any, else largest scale < 1; ties keep the first (fewest rows). */
    int64_t r, best = -1, bn = 0, bd = 1;
    int best_up = 0;
    for (r = 1; r <= main_tiles; ++r) {
      int64_t c, n, d;
      int up, take;
      if (main_tiles % r) continue;
      c = main_tiles / r;
      fit(w, h, c * T, r * T, &n, &d);
      up = n >= d;
      if (best < 0) take = 1;
      else if (up != best_up) take = up;
      else if (up) take = n * bd < bn * d;
      else take = bn * d < n * bd;
      if (take) { best = r; bn = n; bd = d; best_up = up; }
    }
    rows = best;
    cols = main_tiles / best;
  }
  geom[0] = (int32_t)tiles;
  geom[1] = (int32_t)rows;
  geom[2] = (int32_t)cols;
  if (mode == 0) {
    /* transformers get_image_size_fit_to_canvas (image_processing_mllama.py:82-130) in double,
       as Python evaluates it: floor(dim * (target / dim_other)) */
    int64_t cw = cols * T, ch = rows * T;
    int64_t tw = w < T ? T : (w > cw ? cw : w);
    int64_t th = h < T ? T : (h > ch ? ch : h);
    double scale_h = (double)th / (double)h, scale_w = (double)tw / (double)w;
    int64_t nw, nh;
    if (scale_w < scale_h) {
      nw = tw;
      nh = (int64_t)floor((double)h * scale_w);
      if (nh < 1) nh = 1;
      if (nh > th) nh = th;
    } else {
      nh = th;
      nw = (int64_t)floor((double)w * scale_h);
      if (nw < 1) nw = 1;
      if (nw > tw) nw = tw;
    }
    geom[3] = (int32_t)nw;
    geom[4] = (int32_t)nh;
  } else {
    if (w <= h) { geom[3] = (int32_t)T; geom[4] = (int32_t)((T * h) / w); }
    else { geom[4] = (int32_t)T; geom[3] = (int32_t)((T * w) / h); }
  }
}

/* Batch version with exclusive prefix sums; mirrors the device ABI of mmk_tile_plan. */
int32_t oracle_tile_plan(const int32_t* w, const int32_t* h, int32_t n, int32_t T, int32_t tok, int32_t cap,
                         int32_t thumb, int32_t mode, int32_t* tiles, int64_t* tile_off, int64_t* tok_off,
                         int32_t* geom4) {
  int32_t i, bad = 0;
  int64_t run = 0;
  for (i = 0; i < n; ++i) {
    int32_t g[5];
    oracle_plan_one(w[i], h[i], T, cap, thumb, mode, g);
    tiles[i] = g[0];
    geom4[4 * i + 0] = g[1];
    geom4[4 * i + 1] = g[2];
    geom4[4 * i + 2] = g[3];
    geom4[4 * i + 3] = g[4];
    bad += g[0] == 0;
    tile_off[i] = run;
    tok_off[i] = run * tok;
    run += g[0];
  }
  tile_off[n] = run;
  tok_off[n] = run * tok;
  return bad;
}
