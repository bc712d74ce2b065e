// Microbenchmark: HBM -> shared memory streaming with cp.async.bulk on B200.
// One CTA per SM (persistent), NSLOT-deep ring of SLOT-byte bulk copies,
// consumer warps touch every 16 B of each slot. Prints GB/s per config.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_bench tools/tma_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile("{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n"
               ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}

template <int NW>
__global__ void k_stream(const unsigned char* __restrict__ src, size_t per_cta, int slot, int nslot,
                         unsigned long long* sink, int lane0_poll) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + (size_t)nslot * slot);
  uint64_t* empty = full + nslot;
  const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < nslot; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], NW); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const unsigned char* base = src + (size_t)blockIdx.x * per_cta;
  const int nchunks = (int)(per_cta / slot);
  if (wid == NW) {
    if (lane == 0)
      for (int i = 0; i < nchunks; ++i) {
        const int s = i % nslot, use = i / nslot;
        if (use >= 1) mbar_wait(&empty[s], (use - 1) & 1);
        mbar_expect_tx(&full[s], slot);
        bulk_g2s(sm + (size_t)s * slot, base + (size_t)i * slot, slot, &full[s]);
      }
  } else {
    unsigned long long acc = 0;
    for (int i = 0; i < nchunks; ++i) {
      const int s = i % nslot;
      if (lane0_poll) {
        if (lane == 0) mbar_wait(&full[s], (i / nslot) & 1);
        __syncwarp();
      } else {
        mbar_wait(&full[s], (i / nslot) & 1);
      }
      const uint4* p = reinterpret_cast<const uint4*>(sm + (size_t)s * slot);
      for (int q = tid; q < slot / 16; q += NW * 32) acc += p[q].x;
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    if (acc == 0x1234567) sink[0] = acc;
  }
}

int main() {
  const size_t total = (size_t)4 << 30;  // 4 GiB
  unsigned char* d;
  unsigned long long* sink;
  cudaMalloc(&d, total);
  cudaMalloc(&sink, 8);
  cudaMemset(d, 1, total);
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int slots[] = {8192, 16384, 32768};
  const int nslots[] = {2, 4, 6};
  for (int lp = 0; lp < 2; ++lp)
    for (int si = 0; si < 3; ++si)
      for (int ni = 0; ni < 3; ++ni) {
        const int slot = slots[si], nslot = nslots[ni];
        const size_t smem = (size_t)slot * nslot + 2 * nslot * 8;
        if (smem > 220 * 1024) continue;
        const size_t per_cta = (total / nsm) / slot * slot;
        cudaFuncSetAttribute(k_stream<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_stream<16><<<nsm, 16 * 32 + 32, smem>>>(d, per_cta, slot, nslot, sink, lp);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a);
        for (int r = 0; r < 5; ++r) k_stream<16><<<nsm, 16 * 32 + 32, smem>>>(d, per_cta, slot, nslot, sink, lp);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double bytes = 5.0 * per_cta * nsm;
        printf("lane0_poll=%d slot=%6d nslot=%d  %8.1f GB/s  err=%s\n", lp, slot, nslot, bytes / (ms * 1e-3) / 1e9,
               cudaGetErrorString(cudaGetLastError()));
      }
  return 0;
}
