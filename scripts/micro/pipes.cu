// Pipe throughput microbenchmark (development only): per-SM rate of MUFU.EX2 (f32, f16x2, bf16x2),
// FFMA2, HFMA2, F2FP pack, FMNMX3.  One CTA per SM, 8 warps, 16 independent chains per thread.
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_bf16.h>
#define ITERS 4096
template <int OP>
__global__ void k(float* out, float seed) {
  float a[16];
  uint32_t h[16];
  for (int i = 0; i < 16; ++i) { a[i] = seed * (i + 1) * 1e-3f - 1.f; h[i] = 0x3c003c00u + i; }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if constexpr (OP == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
      if constexpr (OP == 1) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h[i]));
      if constexpr (OP == 2) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(h[i]));
      if constexpr (OP == 3) {
        uint64_t v = (uint64_t(__float_as_uint(a[i])) << 32) | __float_as_uint(a[(i + 1) & 15]);
        asm volatile("fma.rn.f32x2 %0, %0, %0, %0;" : "+l"(v));
        a[i] = __uint_as_float(uint32_t(v >> 32)); a[(i + 1) & 15] = __uint_as_float(uint32_t(v));
      }
      if constexpr (OP == 4) asm volatile("fma.rn.f16x2 %0, %0, %0, %0;" : "+r"(h[i]));
      if constexpr (OP == 5) {
        uint32_t r;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[i]), "f"(__uint_as_float(h[i])));
        h[i] = r;
      }
      if constexpr (OP == 6) asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(a[(i + 5) & 15]), "f"(a[(i + 7) & 15]));
      if constexpr (OP == 7) asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(a[i]));
    }
  }
  float s = 0;
  for (int i = 0; i < 16; ++i) s += a[i] + __uint_as_float(h[i]);
  if (s == 12345.f) out[0] = s;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* o; cudaMalloc(&o, 4);
  const char* names[] = {"MUFU ex2 f32", "ex2 f16x2 (2 elem)", "ex2 bf16x2 (2 elem)", "FFMA2 (2 elem)", "HFMA2 (2 elem)", "cvt bf16x2 pack", "FMNMX3", "FFMA"};
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int op = 0; op < 8; ++op) {
    auto f = op == 0 ? k<0> : op == 1 ? k<1> : op == 2 ? k<2> : op == 3 ? k<3> : op == 4 ? k<4> : op == 5 ? k<5> : op == 6 ? k<6> : k<7>;
    f<<<sms, 256>>>(o, 1.f);
    cudaEventRecord(e0);
    f<<<sms, 256>>>(o, 1.f);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double instr = double(sms) * 256 * ITERS * 16;  // thread-instructions
    printf("%-22s %8.3f ms  %7.2f thread-instr/clk/SM (at max clock %d MHz)\n", names[op], ms, instr / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
  }
  return 0;
}
