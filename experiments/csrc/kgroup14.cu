// Transfer v14: K-packed pairs, one 8-lane group per pair, lane = term k.
//
// Layout: the v10 K-packed pairs (meta = column | k-mask << 24, the f32
// values of the terms present, k ascending), rows padded to a multiple of 32
// pairs (meta 0 = empty). A warp walks its rows 32 pairs at a time: one
// coalesced meta load per lane, a warp scan of the popcounts for the value
// offsets, then 8 sub-steps in which group g (lanes 8g .. 8g+7) takes pair
// 4s+g and lane k of the group handles term k:
//   * the k index of a lane is fixed, so its accumulator is 3 registers (no
//     per-lane k loop, no dynamic indexing);
//   * all lanes of a group gather the same packed x column (one L1 wavefront
//     per pair instead of one per term);
//   * a tile-major kept-column bitmap staged in shared memory skips the value
//     load, the gather and the FMAs of columns no channel keeps (their terms
//     are exact zeros), the row-driven form of the reference's csc_apply over
//     the kept columns (transfer.py:66-71).
// All 8 sub-steps issue their loads before any FMA. Rows are cut into pieces
// of <= split pairs (long coarse-receiver rows would otherwise serialize on
// one warp); piece end: the 4 groups' partial sums are combined with 2
// xor-shuffle steps and lanes k < K add the 3 channel sums into the zeroed
// v_k (red.global.add.f64).
#include "sss_common.cuh"

namespace sss {

constexpr int kV14Threads = 256;

struct V14Row {    // a piece of a row
  unsigned pair0;  // first pair (multiple of 32)
  unsigned npair;  // pairs, multiple of 32
  unsigned val0;   // first value of the piece
  unsigned row;    // tile-major row
};

__global__ void __launch_bounds__(kV14Threads) k_transfer_kgroup(
    int K, int N, const uint32_t* __restrict__ meta, const float* __restrict__ vals,
    const V14Row* __restrict__ rows, const unsigned* __restrict__ warp_begin,
    const double4* __restrict__ xp, const uint32_t* __restrict__ bits, double* __restrict__ vk) {
  extern __shared__ uint32_t sbits[];
  const int nw = (N + 31) >> 5;
  for (int i = threadIdx.x; i < nw; i += blockDim.x) sbits[i] = bits[i];
  __syncthreads();
  const int lane = threadIdx.x & 31, grp = lane >> 3, kl = lane & 7;
  const unsigned below = (1u << kl) - 1u;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const unsigned b = warp_begin[w], e = warp_begin[w + 1];
  for (unsigned ri = b; ri < e; ++ri) {
    const V14Row rw = rows[ri];
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    unsigned vbase = rw.val0;
    uint32_t m_next = rw.npair ? __ldg(&meta[rw.pair0 + lane]) : 0u;
    for (unsigned q = 0; q < rw.npair; q += 32) {
      const uint32_t m = m_next;
      if (q + 32 < rw.npair) m_next = __ldg(&meta[rw.pair0 + q + 32 + lane]);
      const unsigned cnt = __popc(m >> 24);
      unsigned incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const unsigned off = vbase + incl - cnt;
      vbase += __shfl_sync(0xffffffffu, incl, 31);
      float v[8];
      double x0[8], x1[8], x2[8];
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        const uint32_t ms = __shfl_sync(0xffffffffu, m, 4 * s + grp);
        const unsigned os = __shfl_sync(0xffffffffu, off, 4 * s + grp);
        const unsigned mask = ms >> 24, col = ms & 0xffffffu;
        const bool hit = ((mask >> kl) & 1u) && ((sbits[col >> 5] >> (col & 31u)) & 1u);
        v[s] = 0.0f;
        x0[s] = x1[s] = x2[s] = 0.0;
        if (hit) {
          v[s] = __ldg(&vals[os + __popc(mask & below)]);
          double x3;
          asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
                       : "=d"(x0[s]), "=d"(x1[s]), "=d"(x2[s]), "=d"(x3)
                       : "l"(xp + col));
        }
      }
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        const double dv = (double)v[s];
        a0 = fma(dv, x0[s], a0);
        a1 = fma(dv, x1[s], a1);
        a2 = fma(dv, x2[s], a2);
      }
    }
    a0 += __shfl_xor_sync(0xffffffffu, a0, 8);
    a1 += __shfl_xor_sync(0xffffffffu, a1, 8);
    a2 += __shfl_xor_sync(0xffffffffu, a2, 8);
    a0 += __shfl_xor_sync(0xffffffffu, a0, 16);
    a1 += __shfl_xor_sync(0xffffffffu, a1, 16);
    a2 += __shfl_xor_sync(0xffffffffu, a2, 16);
    if (lane < K) {  // long rows are split into pieces: add into the zeroed v_k
      double* vo = vk + (size_t)lane * 3 * N + rw.row;
      atomicAdd(vo, a0);
      atomicAdd(vo + N, a1);
      atomicAdd(vo + 2 * (size_t)N, a2);
    }
  }
}

}  // namespace sss
