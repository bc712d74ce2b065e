// Transfer v23 "pairgroup": one x gather per (row, column) pair, four lanes
// per pair.
//
// flat8 is bound by L1TEX wavefronts (80 % of peak at C3), 61 % of them its
// 28.8 M x gathers: one per stored coefficient whose column is kept. A (row,
// column) pair carries 2.7 of the K = 8 terms on average, so gathering per
// pair needs 2.7x fewer. v21 (lane per pair, all K terms in one lane) paid for
// it with an 8-term loop per lane and 24 accumulators. Here a pair is served
// by a group of four lanes (lane = 4 * pair + g): lane g owns terms g and
// g + 4, so it keeps 6 fp64 accumulators and loads at most two values; the
// four lanes of a pair gather the same x address in the same instruction, one
// wavefront per pair. A warp handles 8 pairs per step, rows in sequence
// (whole rows per warp, ~equal pair counts); at a row's end the partial sums
// are reduced over the 8 pair slots (3 xor-shuffle steps) and lanes 0..3
// write v_k directly: no atomics, no memset, deterministic.
//
// Layout (runtime.kpairs_layout): hdr[p] = column | term mask << 16, values
// pair-major (terms ascending inside a pair), per-row pair and value starts.
#include "sss_common.cuh"

namespace sss {

constexpr int kV23Threads = 256;

template <int K, int U = 4>
__global__ void __launch_bounds__(kV23Threads) k_transfer_pairgroup(
    int N, const uint32_t* __restrict__ pp, const uint32_t* __restrict__ vp,
    const uint32_t* __restrict__ hdr, const float* __restrict__ vals,
    const uint32_t* __restrict__ rbeg, const double4* __restrict__ xp,
    const uint32_t* __restrict__ bits, double* __restrict__ vk) {
  extern __shared__ uint32_t v23_bits[];
  for (int t = threadIdx.x; t < ((N + 31) >> 5); t += blockDim.x) v23_bits[t] = bits[t];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int p = lane >> 2, g = lane & 3;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t r0 = rbeg[w], r1 = rbeg[w + 1];
  const uint32_t below0 = (1u << g) - 1u, below1 = (1u << (g + 4)) - 1u;
#pragma unroll 1
  for (uint32_t r = r0; r < r1; ++r) {
    const uint32_t a = __ldg(pp + r), b = __ldg(pp + r + 1);
    uint32_t vb = __ldg(vp + r);
    double s00 = 0.0, s01 = 0.0, s02 = 0.0, s10 = 0.0, s11 = 0.0, s12 = 0.0;
    // U steps of 8 pairs per iteration: all headers, then all gathers and
    // value loads, then the FMAs, so one memory latency covers 8 U pairs
#pragma unroll 1
    for (uint32_t j = a; j < b; j += 8 * U) {
      uint32_t h[U], off[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t q = j + 8 * u + p;
        h[u] = q < b ? __ldg(hdr + q) : 0u;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t cnt = __popc((h[u] >> 16) & 0xffu);
        uint32_t inc = cnt;  // inclusive scan over the 8 pair slots (lane stride 4)
#pragma unroll
        for (int o = 4; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
          if (lane >= o) inc += y;
        }
        off[u] = vb + inc - cnt;
        vb += __shfl_sync(0xffffffffu, inc, 28);
      }
      double x0[U], x1[U], x2[U];
      float v0[U], v1[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t m = (h[u] >> 16) & 0xffu;
        const uint32_t c = h[u] & 0xffffu;
        const bool kept = m && ((v23_bits[c >> 5] >> (c & 31u)) & 1u);
        const bool t0 = kept && ((m >> g) & 1u);
        const bool t1 = K > 4 && kept && ((m >> (g + 4)) & 1u);
        x0[u] = x1[u] = x2[u] = 0.0;
        v0[u] = v1[u] = 0.0f;
        if (t0 || t1) {
          double x3;
          asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
                       : "=d"(x0[u]), "=d"(x1[u]), "=d"(x2[u]), "=d"(x3)
                       : "l"(xp + c));
          (void)x3;
        }
        if (t0) v0[u] = __ldg(vals + off[u] + __popc(m & below0));
        if (t1) v1[u] = __ldg(vals + off[u] + __popc(m & below1));
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const double a0 = (double)v0[u], a1 = (double)v1[u];
        s00 = fma(a0, x0[u], s00);
        s01 = fma(a0, x1[u], s01);
        s02 = fma(a0, x2[u], s02);
        if (K > 4) {
          s10 = fma(a1, x0[u], s10);
          s11 = fma(a1, x1[u], s11);
          s12 = fma(a1, x2[u], s12);
        }
      }
    }
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
      s00 += __shfl_xor_sync(0xffffffffu, s00, o);
      s01 += __shfl_xor_sync(0xffffffffu, s01, o);
      s02 += __shfl_xor_sync(0xffffffffu, s02, o);
      if (K > 4) {
        s10 += __shfl_xor_sync(0xffffffffu, s10, o);
        s11 += __shfl_xor_sync(0xffffffffu, s11, o);
        s12 += __shfl_xor_sync(0xffffffffu, s12, o);
      }
    }
    if (lane < 4) {  // lane g: terms g and g + 4
      if (g < K) {
        double* o0 = vk + (size_t)g * 3 * N + r;
        o0[0] = s00;
        o0[N] = s01;
        o0[2 * (size_t)N] = s02;
      }
      if (g + 4 < K) {
        double* o1 = vk + (size_t)(g + 4) * 3 * N + r;
        o1[0] = s10;
        o1[N] = s11;
        o1[2 * (size_t)N] = s12;
      }
    }
  }
}

}  // namespace sss
