// Transfer v20: dense K-fused pairs, one lane per (row, column) pair.
//
// The K <= 8 operators share most of a row's columns (K-fill 0.37 on C3), so
// the layout stores every (row, column) pair once with its K values in one
// 32-byte slot (0 for absent terms). A lane owns a pair: the term index is the
// slot index, so the 24 accumulators (8 terms x 3 channels) are static
// registers, and ONE x gather serves all of the pair's terms. A pair whose
// column no channel keeps skips its 32-byte value sector and its gather, so
// the bytes read track the kept pairs. Rows are padded to 32 pairs (column =
// N marks padding) and cut into pieces: a warp iteration never straddles a
// row, lanes accumulate privately across the piece, and the 24 sums are
// reduced once per piece (transposed butterfly, v12_reduce24) and added into
// the zeroed v_k. Pipeline: columns two iterations ahead, values and x of the
// next iteration issued before the current one is consumed.
#include "sss_common.cuh"

namespace sss {

constexpr int kV20Threads = 256;

struct V20Pair {
  float4 v0, v1;   // terms 0..3, 4..7
  double x0, x1, x2;
};

__device__ __forceinline__ void v20_fetch(V20Pair& P, uint32_t c, int N, const uint32_t* sbits,
                                          const float4* __restrict__ vals4, unsigned p,
                                          const double4* __restrict__ xp) {
  const bool kept = c < (uint32_t)N && ((sbits[c >> 5] >> (c & 31u)) & 1u);
  if (kept) {
    P.v0 = __ldg(&vals4[2 * (size_t)p]);
    P.v1 = __ldg(&vals4[2 * (size_t)p + 1]);
    double x3;
    asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(P.x0), "=d"(P.x1), "=d"(P.x2), "=d"(x3) : "l"(xp + c));
  } else {
    P.v0 = P.v1 = make_float4(0.f, 0.f, 0.f, 0.f);
    P.x0 = P.x1 = P.x2 = 0.0;
  }
}

__device__ __forceinline__ void v20_accumulate(const V20Pair& P, double (&acc)[24]) {
  const float v[8] = {P.v0.x, P.v0.y, P.v0.z, P.v0.w, P.v1.x, P.v1.y, P.v1.z, P.v1.w};
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const double dv = (double)v[k];
    acc[3 * k + 0] = fma(dv, P.x0, acc[3 * k + 0]);
    acc[3 * k + 1] = fma(dv, P.x1, acc[3 * k + 1]);
    acc[3 * k + 2] = fma(dv, P.x2, acc[3 * k + 2]);
  }
}

template <int MINB>
__global__ void __launch_bounds__(kV20Threads, MINB) k_transfer_k8(
    int K, int N, const uint32_t* __restrict__ cols, const float4* __restrict__ vals4,
    const uint4* __restrict__ pieces, const unsigned* __restrict__ warp_begin,
    const double4* __restrict__ xp, const uint32_t* __restrict__ bits, double* __restrict__ vk) {
  extern __shared__ uint32_t v20_bits[];
  for (int q = threadIdx.x; q < ((N + 31) >> 5); q += blockDim.x) v20_bits[q] = bits[q];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const unsigned b = warp_begin[w], e = warp_begin[w + 1];
#pragma unroll 1
  for (unsigned pi = b; pi < e; ++pi) {
    const uint4 pc = __ldg(&pieces[pi]);
    const unsigned p0 = pc.x, nit = pc.y >> 5, row = pc.z;
    double acc[24];
#pragma unroll
    for (int t = 0; t < 24; ++t) acc[t] = 0.0;
    // pipeline: c1 / c2 = columns of iterations it+1 / it+2, A = data of it
    uint32_t c1 = nit > 1 ? __ldg(&cols[p0 + 32 + lane]) : (uint32_t)N;
    V20Pair A, B;
    v20_fetch(A, __ldg(&cols[p0 + lane]), N, v20_bits, vals4, p0 + lane, xp);
#pragma unroll 1
    for (unsigned it = 0; it < nit; ++it) {
      const uint32_t c2 = it + 2 < nit ? __ldg(&cols[p0 + (it + 2) * 32 + lane]) : (uint32_t)N;
      if (it + 1 < nit) v20_fetch(B, c1, N, v20_bits, vals4, p0 + (it + 1) * 32 + lane, xp);
      v20_accumulate(A, acc);
      A = B;
      c1 = c2;
    }
    double r[3];
    v12_reduce24(acc, lane, r);
    if ((lane & 3) == 0) {
      const int g = lane >> 2;
#pragma unroll
      for (int t = 0; t < 3; ++t) {
        const int f = 3 * g + t;  // = 3 k + c
        if (f < 3 * K && r[t] != 0.0) atomicAdd(&vk[(size_t)f * N + row], r[t]);
      }
    }
  }
}

}  // namespace sss
