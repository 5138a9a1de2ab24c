// FFMA2 / FADD2 / FFMA throughput (development only): 16 independent chains per thread,
// 8 warps per CTA, one CTA per SM.  Prints element-ops and warp-instructions per clock per SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define ITERS 2048
template <int OP>
__global__ void k(float* out, float seed) {
  float2 a[16];
  float b[32];
  for (int i = 0; i < 16; ++i) a[i] = make_float2(seed * i, seed * (i + 1));
  for (int i = 0; i < 32; ++i) b[i] = seed * i;
  const float2 m = make_float2(1.0001f, 0.9999f), c = make_float2(1e-4f, -1e-4f);
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if constexpr (OP == 0) a[i] = __ffma2_rn(a[i], m, c);
      if constexpr (OP == 1) a[i] = __fadd2_rn(a[i], c);
      if constexpr (OP == 2) { b[2 * i] = fmaf(b[2 * i], 1.0001f, 1e-4f); b[2 * i + 1] = fmaf(b[2 * i + 1], 0.9999f, -1e-4f); }
      if constexpr (OP == 3) { b[2 * i] = fmaxf(fmaxf(b[2 * i], b[2 * i + 1]), 0.5f); }
    }
  }
  float s = 0;
  for (int i = 0; i < 16; ++i) s += a[i].x + a[i].y;
  for (int i = 0; i < 32; ++i) s += b[i];
  if (s == 1234.5f) out[0] = s;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* o; cudaMalloc(&o, 4);
  const char* names[] = {"FFMA2 (x16 float2 chains)", "FADD2 (x16 float2 chains)", "FFMA  (x32 scalar chains)", "FMNMX (x16 chains)"};
  const int instr_per_iter[] = {16, 16, 32, 32};
  const int elems_per_instr[] = {2, 2, 1, 1};
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int op = 0; op < 4; ++op) {
    auto f = op == 0 ? k<0> : op == 1 ? k<1> : op == 2 ? k<2> : k<3>;
    for (int threads : {256, 512, 1024}) {
      f<<<sms, threads>>>(o, 1.f);
      cudaEventRecord(e0);
      f<<<sms, threads>>>(o, 1.f);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      const double winstr = double(sms) * (threads / 32) * ITERS * instr_per_iter[op];
      const double per_clk_sm = winstr / (ms * 1e-3) / sms / (clk * 1e3);
      printf("%-28s threads=%4d  %6.3f warp-instr/clk/SM  %7.1f element-ops/clk/SM (max-clock basis)\n", names[op],
             threads, per_clk_sm, per_clk_sm * 32 * elems_per_instr[op]);
    }
  }
  return 0;
}
