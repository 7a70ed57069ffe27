// Internal helpers shared by the libzorse_b200 translation units (host side).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#define ZB_ERR_INVALID 1001
#define ZB_ERR_CUDA 1002
#define ZB_ERR_NCCL 1003
#define ZB_ERR_UNSUPPORTED 1004

namespace zb {
// Record an error message (thread-local) and return `code`.
int set_error(int code, const char* fmt, ...);
int set_cuda_error(cudaError_t e, const char* where);
// Number of SMs on the current device (cached per device).
int num_sms();
// cuTensorMapEncodeTiled resolved through the runtime's driver entry point.
int tensor_map_encode(CUtensorMap* m, CUtensorMapDataType dt, cuuint32_t rank, void* gaddr,
                      const cuuint64_t* dims, const cuuint64_t* strides, const cuuint32_t* box,
                      const cuuint32_t* estrides, CUtensorMapInterleave il,
                      CUtensorMapSwizzle sw, CUtensorMapL2promotion l2,
                      CUtensorMapFloatOOBfill oob);
// 2-D bf16 tensor map, 128-byte swizzle, box {box_inner, box_outer}.
int make_tmap_bf16_2d(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer,
                      uint64_t ld_elems, uint32_t box_inner, uint32_t box_outer);

// Programmatic dependent launch (PDL) on `stream`: the kernel may be scheduled while
// its predecessor drains (once every predecessor CTA executed griddep_launch()), and
// must call griddep_wait() (common.cuh pdl_enter) before touching global memory.
bool pdl_enabled();
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                         cudaStream_t stream, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}
}  // namespace zb
