// Bandwidth probes for the flat-stream transfer (tools only, not part of the
// product ABI): MODE 1 = stream without x gathers, MODE 2 = columns + gathers
// without operator values, plus a plain coalesced read-reduce of both arrays.
#include "../paper_2203_12339_b200/csrc/flat15.cu"

__global__ void k_read_reduce(const uint4* __restrict__ a, unsigned long long n4,
                              unsigned long long* out) {
  unsigned long long acc = 0;
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n4;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const uint4 v = __ldg(&a[i]);
    acc += v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345) atomicAdd(out, acc);
}

extern "C" int probe_flat(int mode, int ga, int n_rows, const void* pcols, const void* pvals, unsigned n4,
                          const void* heads, const void* hpre, const void* rowk, const void* wbeg,
                          int n_warps, const void* xp, const void* bits, double* vk) {
  auto bt = (const uint32_t*)bits;
  const size_t smem = bt ? (size_t)((n_rows + 31) / 32) * 4 : 0;
  const unsigned grid = n_warps / (sss::kV15Threads / 32);
  auto c4 = (const uint4*)pcols;
  auto v4 = (const float4*)pvals;
  auto h = (const uint32_t*)heads;
  auto hp = (const uint32_t*)hpre;
  auto rk = (const uint32_t*)rowk;
  auto wb = (const unsigned*)wbeg;
  auto x4 = (const double4*)xp;
#define PR(M, G) if (mode == M && ga == G) sss::k_transfer_flat<M, G><<<grid, sss::kV15Threads, smem>>>(n_rows, n4, c4, v4, h, hp, rk, wb, x4, bt, vk)
  PR(0, 1); PR(0, 2); PR(0, 3); PR(1, 2); PR(2, 1); PR(2, 2); PR(2, 3);
  return (int)cudaGetLastError();
}

extern "C" int probe_read(const void* a, unsigned long long n4, int grid, unsigned long long* out) {
  k_read_reduce<<<grid, 256>>>((const uint4*)a, n4, out);
  return (int)cudaGetLastError();
}
