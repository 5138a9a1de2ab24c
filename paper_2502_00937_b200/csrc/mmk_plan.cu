// mmk_plan.cu — K0: per-image tile plan + ragged offset scan (bit-exact integer work).
//
// Restates, for a whole batch at once on the GPU:
//   core.tile_count   (reference pkg/src/lmmsim/core.py:58-69):
//       grid = ceil(w/T) * ceil(h/T); +1 thumbnail if spec.thumbnail_tile and grid > 1;
//       min(cap); SpecError when w < 1 or h < 1   (here: tiles = 0 and `bad` is counted)
//   core.image_tokens (core.py:72-74): tiles * tokens_per_tile
//   Request.total_tiles / total_image_tokens (core.py:110-120): exclusive int64 prefix sums
// plus the builder-defined pixel geometry:
//   rows x cols tile canvas (ceil grid when it fits the cap, else the best r*c == tiles
//   arrangement by Mllama's scale criterion) and the resized image size (transformers'
//   get_image_size_fit_to_canvas in float64 as Python evaluates it, or CLIP's shortest-edge
//   resize, int(T * long / short), which integer division reproduces exactly at these sizes).
//
// Two launches: a thread per image for the plan (tile count, canvas, aspect-ratio id), then one
// CTA scanning the tile counts in coalesced 1024-image chunks (warp-shuffle + shared-memory scan,
// int64 carry between chunks).
#include "sm100_common.cuh"
#include "mmk_internal.h"

namespace mmk {

struct TileGeom {
  int32_t tiles, rows, cols, new_w, new_h;
};

__host__ __device__ inline int64_t ceil_div64(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Fraction a/b <  c/d  for positive denominators.
__host__ __device__ inline bool frac_lt(int64_t a, int64_t b, int64_t c, int64_t d) { return a * d < c * b; }

// scale of fitting (w,h) into canvas (cw,ch): min(cw/w, ch/h) as a fraction num/den.
__host__ __device__ inline void fit_scale(int64_t w, int64_t h, int64_t cw, int64_t ch, int64_t& num, int64_t& den) {
  if (cw * h <= ch * w) { num = cw; den = w; } else { num = ch; den = h; }
}

__host__ __device__ inline TileGeom plan_one(int64_t w, int64_t h, int64_t T, int64_t cap, bool thumb, int mode) {
  TileGeom g{0, 0, 0, 0, 0};
  if (w < 1 || h < 1) return g;
  const int64_t gw = ceil_div64(w, T), gh = ceil_div64(h, T);
  const int64_t grid = gw * gh;
  int64_t tiles = (thumb && grid > 1) ? grid + 1 : grid;
  if (tiles > cap) tiles = cap;
  g.tiles = static_cast<int32_t>(tiles);
  const int64_t main = (thumb && tiles > 1) ? tiles - 1 : tiles;
  int64_t rows, cols;
  if (main == grid) {
    rows = gh; cols = gw;
  } else {
    // grid exceeds the budget: choose r*c == main by Mllama's criterion (smallest upscale if
    // any candidate upscales, else the largest downscale); ties keep the fewest rows.
    int64_t best_r = -1, bn = 0, bd = 1;
    bool best_up = false;
    for (int64_t r = 1; r <= main; ++r) {
      if (main % r) continue;
      const int64_t c = main / r;
      int64_t n_, d_;
      fit_scale(w, h, c * T, r * T, n_, d_);
      const bool up = n_ >= d_;
      bool take;
      if (best_r < 0) take = true;
      else if (up != best_up) take = up;
      else if (up) take = frac_lt(n_, d_, bn, bd);
      else take = frac_lt(bn, bd, n_, d_);
      if (take) { best_r = r; bn = n_; bd = d_; best_up = up; }
    }
    rows = best_r; cols = main / best_r;
  }
  g.rows = static_cast<int32_t>(rows);
  g.cols = static_cast<int32_t>(cols);
  if (mode == 0) {
    // transformers' get_image_size_fit_to_canvas (image_processing_mllama.py:82-130), float64
    // exactly as Python evaluates it: target = clip(dim, T, canvas); scale = target / dim;
    // the other side = floor(dim * scale) (so 400x180 -> 560x251, not the rational 252).
    // Division and multiply are single correctly rounded IEEE double ops on host and device.
    const int64_t cw = cols * T, ch = rows * T;
    const int64_t tw = w < T ? T : (w > cw ? cw : w);
    const int64_t th = h < T ? T : (h > ch ? ch : h);
    const double scale_h = static_cast<double>(th) / static_cast<double>(h);
    const double scale_w = static_cast<double>(tw) / static_cast<double>(w);
    int64_t nw, nh;
    if (scale_w < scale_h) {
      nw = tw;
      nh = static_cast<int64_t>(floor(static_cast<double>(h) * scale_w)); if (nh < 1) nh = 1; if (nh > th) nh = th;
    } else {
      nh = th;
      nw = static_cast<int64_t>(floor(static_cast<double>(w) * scale_h)); if (nw < 1) nw = 1; if (nw > tw) nw = tw;
    }
    g.new_w = static_cast<int32_t>(nw);
    g.new_h = static_cast<int32_t>(nh);
  } else {
    // CLIP: shortest edge -> T, long edge = floor(T * long / short); centre crop happens in K1
    if (w <= h) { g.new_w = static_cast<int32_t>(T); g.new_h = static_cast<int32_t>((T * h) / w); }
    else { g.new_h = static_cast<int32_t>(T); g.new_w = static_cast<int32_t>((T * w) / h); }
  }
  return g;
}

constexpr int kMapThreads = 256;
constexpr int kScanThreads = 1024;

// K0a: one thread per image — tile count, canvas geometry, aspect-ratio id (fully parallel).
__global__ void __launch_bounds__(kMapThreads)
tile_plan_map_kernel(const int32_t* __restrict__ w, const int32_t* __restrict__ h, int n, int T, int cap, int thumb,
                     int mode, int32_t* __restrict__ tiles, int32_t* __restrict__ geom, int32_t* __restrict__ ar_id) {
  griddep_wait();  // PDL: inputs come from the preceding kernel
  griddep_launch_dependents();
  const int i = blockIdx.x * kMapThreads + threadIdx.x;
  if (i >= n) return;
  const TileGeom g = plan_one(w[i], h[i], T, cap, thumb != 0, mode);
  tiles[i] = g.tiles;
  if (geom) {
    geom[4 * i + 0] = g.rows; geom[4 * i + 1] = g.cols;
    geom[4 * i + 2] = g.new_w; geom[4 * i + 3] = g.new_h;
  }
  if (ar_id) {
    // index of (rows, cols) in [(a, b) for a in 1..cap for b in 1..cap if a*b <= cap], + 1
    int id = 0;
    if (g.tiles > 0) {
      id = g.cols;
      for (int a = 1; a < g.rows; ++a) id += cap / a;
    }
    ar_id[i] = id;
  }
}

// K0b: one CTA, coalesced 1024-image chunks: exclusive int64 prefix sums of the tile counts
// (Request.total_tiles / total_image_tokens offsets) and the count of rejected images.
__global__ void __launch_bounds__(kScanThreads)
tile_plan_scan_kernel(const int32_t* __restrict__ tiles, int n, int tok_per_tile, int64_t* __restrict__ tile_off,
                      int64_t* __restrict__ tok_off, int32_t* __restrict__ bad) {
  griddep_wait();  // PDL: inputs come from the preceding kernel
  griddep_launch_dependents();
  __shared__ int64_t warp_tot[32];
  __shared__ int32_t warp_bad[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int64_t carry = 0;
  int32_t nbad = 0;
  for (int base = 0; base < n; base += kScanThreads) {
    const int i = base + tid;
    const int64_t v = i < n ? tiles[i] : 0;
    nbad += (i < n && v == 0);
    int64_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t u = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += u;
    }
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      const int64_t t = warp_tot[lane];
      int64_t x = t;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t u = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += u;
      }
      warp_tot[lane] = x - t;  // exclusive offsets of the warps
    }
    __syncthreads();
    const int64_t excl = carry + warp_tot[warp] + incl - v;
    if (i < n) {
      tile_off[i] = excl;
      tok_off[i] = excl * tok_per_tile;
    }
    __syncthreads();
    if (tid == kScanThreads - 1) warp_tot[0] = excl + v - carry;  // this chunk's total
    __syncthreads();
    carry += warp_tot[0];
    __syncthreads();
  }
  for (int o = 16; o > 0; o >>= 1) nbad += __shfl_xor_sync(0xffffffffu, nbad, o);
  if (lane == 0) warp_bad[warp] = nbad;
  __syncthreads();
  if (tid == 0) {
    int32_t b = 0;
    for (int k = 0; k < kScanThreads / 32; ++k) b += warp_bad[k];
    if (bad) *bad = b;
    tile_off[n] = carry;
    tok_off[n] = carry * tok_per_tile;
  }
}

// Per-tile (image index, slot within image) for the embedding / tile-position kernels.
__global__ void tile_index_kernel(const int64_t* __restrict__ tile_off, int n, int32_t* __restrict__ tile_image,
                                  int32_t* __restrict__ tile_slot) {
  griddep_wait();  // PDL: inputs come from the preceding kernel
  griddep_launch_dependents();
  const int i = blockIdx.x * blockDim.y + threadIdx.y;
  if (i >= n) return;
  const int64_t a = tile_off[i], b = tile_off[i + 1];
  for (int64_t t = a + threadIdx.x; t < b; t += blockDim.x) {
    tile_image[t] = i;
    tile_slot[t] = static_cast<int32_t>(t - a);
  }
}

// int32 attention offsets cu_seqlens[i] = tile_off[i] * seq_per_tile (i <= n): the sequences of
// the varlen attention are whole images (Mllama: all tiles of an image attend to each other);
// tile_off == NULL gives one sequence per tile (CLIP-family encoders see each tile alone).
__global__ void seq_offsets_kernel(const int64_t* __restrict__ tile_off, int n, int seq_per_tile,
                                   int32_t* __restrict__ cu_seqlens) {
  griddep_wait();  // PDL: inputs come from the preceding kernel
  griddep_launch_dependents();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i <= n) cu_seqlens[i] = static_cast<int32_t>((tile_off ? tile_off[i] : i) * seq_per_tile);
}

}  // namespace mmk

using namespace mmk;

extern "C" int mmk_tile_plan(const int32_t* w, const int32_t* h, int32_t n, int32_t tile_px, int32_t tokens_per_tile,
                             int32_t max_tiles, int32_t thumbnail, int32_t resize_mode, int32_t* tiles,
                             int64_t* tile_off, int64_t* tok_off, int32_t* geom, int32_t* ar_id, int32_t* bad,
                             cudaStream_t stream) {
  if (n < 0 || n > 65536) return set_error(MMK_ERR_ARG, "tile_plan: n=%d outside [0, 65536]", n);
  if (tile_px < 1 || tokens_per_tile < 1 || max_tiles < 1)
    return set_error(MMK_ERR_ARG, "tile_plan: tile_edge_px, tokens_per_tile, max_tiles must be >= 1");
  if (resize_mode != 0 && resize_mode != 1) return set_error(MMK_ERR_ARG, "tile_plan: resize_mode must be 0 or 1");
  if (n > 0)
    (void)launch_kernel(tile_plan_map_kernel, dim3((n + kMapThreads - 1) / kMapThreads), dim3(kMapThreads), 0, stream, 1, n <= 4096, 
        w, h, n, tile_px, max_tiles, thumbnail, resize_mode, tiles, geom, ar_id);
  (void)launch_kernel(tile_plan_scan_kernel, dim3(1), dim3(kScanThreads), 0, stream, 1, n <= 4096, tiles, n, tokens_per_tile, tile_off, tok_off, bad);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? MMK_OK : set_cuda_error(e, "tile_plan: launch");
}

extern "C" int mmk_tile_index(const int64_t* tile_off, int32_t n, int32_t* tile_image, int32_t* tile_slot,
                              cudaStream_t stream) {
  if (n < 0) return set_error(MMK_ERR_ARG, "tile_index: n < 0");
  if (n == 0) return MMK_OK;
  dim3 block(32, 8);
  (void)launch_kernel(tile_index_kernel, dim3((n + 7) / 8), dim3(block), 0, stream, 1, n <= 4096, tile_off, n, tile_image, tile_slot);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? MMK_OK : set_cuda_error(e, "tile_index: launch");
}

extern "C" int mmk_seq_offsets(const int64_t* tile_off, int32_t n, int32_t seq_per_tile, int32_t* cu_seqlens,
                               cudaStream_t stream) {
  if (n < 0 || seq_per_tile < 1) return set_error(MMK_ERR_ARG, "seq_offsets: n < 0 or seq_per_tile < 1");
  (void)launch_kernel(seq_offsets_kernel, dim3(n / 256 + 1), dim3(256), 0, stream, 1, n <= 4096, tile_off, n,
                      seq_per_tile, cu_seqlens);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? MMK_OK : set_cuda_error(e, "seq_offsets: launch");
}
