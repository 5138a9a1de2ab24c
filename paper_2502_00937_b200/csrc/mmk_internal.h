// mmk_internal.h — shared host-side helpers of libmmk (error state, SM count, TMA maps).
#pragma once
#include <atomic>
#include <cstdint>
#include <utility>
#include <cuda.h>
#include <cuda_runtime.h>
#include "mmk.h"

namespace mmk {

int set_error(int code, const char* fmt, ...);
int set_cuda_error(cudaError_t e, const char* where);
int num_sms();

// 2-D bf16 tensor map over a row-major [rows, inner] matrix with row pitch `ld` elements,
// box = {box_inner, box_rows}; 128-byte swizzle (box_inner*2 must be 128) or none.
int make_tmap_2d_bf16(CUtensorMap* map, const void* base, uint64_t inner, uint64_t rows,
                      uint64_t ld, uint32_t box_inner, uint32_t box_rows, bool swizzle128);
// Generic encoder (rank <= 5), strides in bytes for dims 1..rank-1.
int make_tmap_bf16(CUtensorMap* map, const void* base, int rank, const uint64_t* dims,
                   const uint64_t* strides_bytes, const uint32_t* box, CUtensorMapSwizzle swz);
int make_tmap(CUtensorMap* map, CUtensorMapDataType dtype, const void* base, int rank, const uint64_t* dims,
              const uint64_t* strides_bytes, const uint32_t* box, CUtensorMapSwizzle swz);

// Raise a kernel's dynamic shared-memory limit once per device.  `done` is a per-kernel bit set
// of devices (a static at the call site); concurrent first calls may both set the attribute,
// which is idempotent.
inline int ensure_smem_attr(const void* kern, int bytes, std::atomic<uint64_t>& done, const char* what) {
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return MMK_OK;
  const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) return set_cuda_error(e, what);
  done.fetch_or(bit, std::memory_order_release);
  return MMK_OK;
}

// Kernel launch through cudaLaunchKernelEx: optional thread-block cluster (cluster_x > 1) and
// programmatic dependent launch (PDL; the kernels call griddep_wait() before touching data of
// the preceding kernel).  PDL pays off for small, launch-latency-bound problems (ViT-B batch 8:
// +2.5 %) and costs ~1.8 % on the large Mllama step, so callers pass `small` and PDL is used for
// those only; MMK_PDL=0 / 1 turns it off / on for every launch (A/B runs).
bool pdl_for(bool small);
constexpr int64_t kSmallRows = 32768;  // row-parallel kernels at or below this size count as small
template <typename... KArgs, typename... Args>
cudaError_t launch_kernel(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                          int cluster_x, bool small, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  unsigned na = 0;
  if (cluster_x > 1) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = cluster_x;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  if (pdl_for(small)) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

}  // namespace mmk
