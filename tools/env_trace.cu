// Phase timeline of k_env_project (CTA 0, %globaltimer): tools only.
#define SSS_ENV_TRACE 1
#include "../paper_2203_12339_b200/csrc/frame.cu"

extern "C" int env_trace(const double* faces, int s, int n_keep, uint32_t* idx, double* val,
                         unsigned long long* out) {
  const int s2 = s * s;
  const size_t smem = (size_t)12 * s2 * sizeof(double) + sizeof(sss::SelShared);
  cudaFuncSetAttribute(sss::k_env_project, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  unsigned long long zero[16] = {0};
  cudaMemcpyToSymbol(sss::g_env_trace, zero, sizeof(zero));
  sss::k_env_project<<<3, 1024, smem>>>(faces, s, n_keep, idx, val, nullptr);
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, sss::g_env_trace, sizeof(zero));
  return (int)cudaGetLastError();
}
