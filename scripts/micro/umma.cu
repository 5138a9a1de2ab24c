// tcgen05.mma issue/throughput microbenchmark (development only): cycles per M=128, K=16 bf16 MMA
// for several N, operands from shared memory (SS) or A from TMEM (TS), B K-major or MN-major.
// One CTA per SM, one elected thread issues R MMAs back to back into one accumulator, commit, wait.
#include <cstdio>
#include "../../paper_2502_00937_b200/csrc/sm100_common.cuh"
using namespace mmk;
constexpr int R = 512;
template <int N, bool TS, bool BMN>
__global__ void __launch_bounds__(128, 1) k(long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 65536 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc<512>(&slot);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (warp == 1) {
    const uint64_t ad = umma_desc_sw128_kmajor(smem_u32(smem));
    const uint64_t bd = umma_desc_sw128_kmajor(smem_u32(smem + 32768));
    uint32_t idesc = umma_idesc_bf16_f32(128, N) | (BMN ? (1u << 16) : 0u);
    long long t0 = clock64();
    if (elect_one()) {
      for (int r = 0; r < R; ++r) {
        if (TS) umma_bf16_ts(tmem, tmem + 256, bd, idesc, 1u);
        else umma_bf16_ss(tmem, ad, bd, idesc, 1u);
      }
      umma_commit(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (threadIdx.x == 32) out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc<512>(tmem);
}
template <int N, bool TS, bool BMN>
void run(long long* d, int sms) {
  auto f = k<N, TS, BMN>;
  cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  f<<<sms, 128, 70000>>>(d);
  f<<<sms, 128, 70000>>>(d);
  cudaDeviceSynchronize();
  long long h[256];
  cudaMemcpy(h, d, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < sms; ++i) avg += h[i];
  avg /= sms;
  const double ideal = 128.0 * N * 16 * 2 / 8192.0;
  printf("N=%3d %s B%s: %6.1f clk/MMA (ideal at 8192 flop/clk/SM: %5.1f)  err=%s\n", N, TS ? "TS" : "SS",
         BMN ? "-MN" : "-K ", avg / R, ideal, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* d; cudaMalloc(&d, sizeof(long long) * 256);
  run<16, false, false>(d, sms); run<32, false, false>(d, sms); run<64, false, false>(d, sms);
  run<80, false, false>(d, sms); run<112, false, false>(d, sms); run<128, false, false>(d, sms);
  run<256, false, false>(d, sms);
  run<16, true, true>(d, sms); run<32, true, true>(d, sms); run<64, true, true>(d, sms); run<80, true, true>(d, sms);
  run<128, true, true>(d, sms); run<256, true, true>(d, sms);
  run<112, true, false>(d, sms);
  return 0;
}
