// Phase timeline of k_select_cluster (CTA 0, %globaltimer): tools only.
#define SSS_SELECT_TRACE 1
#include "../paper_2203_12339_b200/csrc/select_cluster.cu"

extern "C" int select_trace(const double* v, int nvec, int n_dom, int n_keep, const uint32_t* f2t,
                            double* x, uint32_t* mask, double* energy, unsigned long long* out) {
  const int chunk = (((n_dom + sss::kSelCluster - 1) / sss::kSelCluster) + 31) / 32 * 32;
  const size_t smem = ((sizeof(sss::ClusterSelShared) + 15) & ~size_t(15)) + chunk * sizeof(double);
  cudaFuncSetAttribute(sss::k_select_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (sss::kSelCluster > 8)
    cudaFuncSetAttribute(sss::k_select_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaMemset(mask, 0, (size_t)nvec * ((n_dom + 31) / 32) * 4);
  unsigned long long zero[32] = {0};
  cudaMemcpyToSymbol(sss::g_sel_trace, zero, sizeof(zero));
  sss::k_select_cluster<<<nvec * sss::kSelCluster, 1024, smem>>>(v, n_dom, n_keep, chunk, f2t, x,
                                                                  mask, energy, nullptr, nullptr);
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, sss::g_sel_trace, sizeof(zero));
  return (int)cudaGetLastError();
}
