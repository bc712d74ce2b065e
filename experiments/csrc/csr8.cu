// Transfer v8: persistent merge-path CSR SpMV over all (row, k) segments.
//
// The K per-term CSR operators are one stream of (row, k) segments. At layout
// time (runtime.csr8_schedule) the segments are ordered by (row, k) — rows of
// a tile are adjacent, so consecutive segments touch the same source region
// and their x gathers hit L1 — long segments are cut into pieces of at most
// kSplit entries, and the piece list is cut into W contiguous, entry-balanced
// ranges, one per warp of a persistent grid (W = #SM x warps per SM).
// A warp walks its pieces: coalesced 4-way-unrolled entry loads, packed-x
// gathers (one 32 B sector), fp64 accumulation, one warp reduction per piece,
// and a red.global.add.f64 of the three channel sums into v_k (zeroed before).
// The recombine + inverse Haar + shade epilogue is k_edit_finish.
#include "sss_common.cuh"

namespace sss {

constexpr int kV8Threads = 256;

struct V8Piece {
  unsigned start;  // first entry (global index into cols / vals)
  unsigned len;    // entries
  unsigned rowk;   // tile-major row * 16 + k
  unsigned pad;
};

__device__ __forceinline__ double4 ldx8(const double4* __restrict__ xp, uint32_t c) {
  const double2* q = reinterpret_cast<const double2*>(xp + c);
  const double2 a = __ldg(q);
  const double b = __ldg(reinterpret_cast<const double*>(q + 1));
  return make_double4(a.x, a.y, b, 0.0);
}

__global__ void __launch_bounds__(kV8Threads) k_transfer_csr8(
    int N, const uint32_t* __restrict__ cols, const float* __restrict__ vals,
    const V8Piece* __restrict__ pieces, const unsigned* __restrict__ warp_begin /* W + 1 */,
    const double4* __restrict__ xp, double* __restrict__ vk) {
  const int lane = threadIdx.x & 31;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const unsigned b = warp_begin[w], e_end = warp_begin[w + 1];
  for (unsigned base = b; base < e_end; base += 32) {
    // 32 descriptors at a time, one per lane; broadcast one by one
    V8Piece mine;
    if (base + lane < e_end) mine = pieces[base + lane];
    const int cnt = (int)min(32u, e_end - base);
    for (int j = 0; j < cnt; ++j) {
      const unsigned s = __shfl_sync(0xffffffffu, mine.start, j);
      const unsigned len = __shfl_sync(0xffffffffu, mine.len, j);
      const unsigned rowk = __shfl_sync(0xffffffffu, mine.rowk, j);
      const unsigned e = s + len;
      double a0 = 0.0, a1 = 0.0, a2 = 0.0;
      unsigned p = s + lane;
      for (; p + 96 < e; p += 128) {
        const uint32_t c0 = __ldg(&cols[p]), c1 = __ldg(&cols[p + 32]), c2 = __ldg(&cols[p + 64]),
                       c3 = __ldg(&cols[p + 96]);
        const float v0 = __ldg(&vals[p]), v1 = __ldg(&vals[p + 32]), v2 = __ldg(&vals[p + 64]),
                    v3 = __ldg(&vals[p + 96]);
        const double4 x0 = ldx8(xp, c0), x1 = ldx8(xp, c1), x2 = ldx8(xp, c2), x3 = ldx8(xp, c3);
        a0 = fma((double)v0, x0.x, a0); a1 = fma((double)v0, x0.y, a1); a2 = fma((double)v0, x0.z, a2);
        a0 = fma((double)v1, x1.x, a0); a1 = fma((double)v1, x1.y, a1); a2 = fma((double)v1, x1.z, a2);
        a0 = fma((double)v2, x2.x, a0); a1 = fma((double)v2, x2.y, a1); a2 = fma((double)v2, x2.z, a2);
        a0 = fma((double)v3, x3.x, a0); a1 = fma((double)v3, x3.y, a1); a2 = fma((double)v3, x3.z, a2);
      }
      for (; p < e; p += 32) {
        const uint32_t c = __ldg(&cols[p]);
        const double v = (double)__ldg(&vals[p]);
        const double4 xv = ldx8(xp, c);
        a0 = fma(v, xv.x, a0); a1 = fma(v, xv.y, a1); a2 = fma(v, xv.z, a2);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        a0 += __shfl_xor_sync(0xffffffffu, a0, o);
        a1 += __shfl_xor_sync(0xffffffffu, a1, o);
        a2 += __shfl_xor_sync(0xffffffffu, a2, o);
      }
      if (lane == 0) {
        const int row = (int)(rowk >> 4), k = (int)(rowk & 15u);
        double* vo = vk + (size_t)k * 3 * N;
        atomicAdd(&vo[row], a0);
        atomicAdd(&vo[N + row], a1);
        atomicAdd(&vo[2 * N + row], a2);
      }
    }
  }
}

}  // namespace sss
