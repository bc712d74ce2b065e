// Error / launch helpers shared by the library's translation units (abi.cu,
// abi_exact.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdlib>
#include <string>

#include "../../include/sss_b200.h"

namespace sss_abi {
// one error string per thread, shared by every translation unit of the library
inline std::string& err_ref() {
  static thread_local std::string s;
  return s;
}
#define g_err (::sss_abi::err_ref())

inline int fail(int code, const char* msg) {
  g_err = msg;
  return code;
}

inline int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    g_err = std::string(what) + ": " + cudaGetErrorString(e);
    return SSS_ECUDA;
  }
  return SSS_OK;
}

inline bool pow2(int v) { return v > 0 && (v & (v - 1)) == 0; }

inline int set_smem(const void* fn, size_t bytes) {
  if (bytes > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess) {
      g_err = std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e);
      return SSS_ECUDA;
    }
  }
  return SSS_OK;
}

inline int check_geom(int side, int levels) {
  if (!pow2(side) || side < 2) return fail(SSS_EINVAL, "side must be a power of two >= 2");
  if (levels < 1 || (1 << levels) > side || levels > 6)
    return fail(SSS_EINVAL, "levels must lie in [1, min(6, log2 side)]");
  return SSS_OK;
}

inline cudaStream_t S_(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Launch of a kernel of the frame's chain with programmatic stream
// serialization (see sss_common.cuh pdl_*): the kernel may start while its
// predecessor in the stream is still running and orders its own memory
// accesses with griddepcontrol.wait. SSS_PDL=0 turns the attribute off
// (plain stream order). Works eagerly and under stream capture (the edge
// becomes a programmatic dependency of the graph).
inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("SSS_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_chain(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                                cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}
}  // namespace sss_abi
using namespace sss_abi;
