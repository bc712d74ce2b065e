// Transfer v18: mask-sorted K-fused warp steps, streamed flat.
//
// Layout = v12's steps (a row's (row, column) pairs sorted by k-mask, 32 per
// step; per step 32 columns and, for each k of the step's OR-mask, 32 f32
// values in lane order). One x gather per PAIR serves all K terms (3x fewer
// gather instructions than per-term CSR on C3), and value loads are 128-byte
// coalesced rows, one per (step, k).
//
// v12 lost to latency (record -> column -> gather chained per step). Here:
//   * step records are held one per lane, 32 at a time (two batches in
//     flight), and broadcast with shuffles - no per-step record load;
//   * columns + values of step s+2 are requested while step s is consumed,
//     the x gathers of step s+1 are issued before it (three register slots
//     rotate; values are kept indexed by k, the running slot rank only enters
//     the load address, so no dynamic register indexing);
//   * the kept-column bitmap (shared memory) skips gathers of unkept columns.
// Row end (or warp-range end): transposed-butterfly reduction of the 24 sums
// and red.global.add.f64 into the zeroed v_k. Epilogue: k_edit_finish.
#include "sss_common.cuh"

namespace sss {

constexpr int kV18Threads = 128;

struct V18Slot {
  uint32_t col, info, row;
  float v[8];      // by k; only the terms of the step's mask are loaded
  double x0, x1, x2;
};

template <int DUMMY = 0>
__global__ void __launch_bounds__(kV18Threads, 4) k_transfer_kflat(
    int K, int N, const uint32_t* __restrict__ cols, const float* __restrict__ vals,
    const uint4* __restrict__ steps, const unsigned* __restrict__ warp_begin,
    const double4* __restrict__ xp, const uint32_t* __restrict__ bits, double* __restrict__ vk) {
  extern __shared__ uint32_t v18_bits[];
  if (bits) {
    for (int t = threadIdx.x; t < ((N + 31) >> 5); t += blockDim.x) v18_bits[t] = bits[t];
    __syncthreads();
  }
  const int lane = threadIdx.x & 31;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const unsigned s0 = warp_begin[w], s1 = warp_begin[w + 1];
  if (s0 >= s1) return;
  const unsigned ns = s1 - s0;

  unsigned base = 0;  // rA holds local steps [base, base + 32), rB the next 32
  uint4 rA = make_uint4(0u, 0u, 0u, 0u), rB = rA;
  if (lane < ns) rA = __ldg(&steps[s0 + lane]);
  if (lane + 32 < ns) rB = __ldg(&steps[s0 + 32 + lane]);

  auto load = [&](V18Slot& S, unsigned j) {  // warp-uniform j < ns, j < base + 64
    const bool inA = j < base + 32;
    const int src = (int)(j - base) - (inA ? 0 : 32);
    const uint32_t px = __shfl_sync(0xffffffffu, inA ? rA.x : rB.x, src);
    const uint32_t py = __shfl_sync(0xffffffffu, inA ? rA.y : rB.y, src);
    const uint32_t pz = __shfl_sync(0xffffffffu, inA ? rA.z : rB.z, src);
    const uint32_t pw = __shfl_sync(0xffffffffu, inA ? rA.w : rB.w, src);
    S.info = pw;
    S.row = pz;
    const unsigned mask = pw & 0xffu, cnt = (pw >> 8) & 0xffu;
    S.col = lane < (int)cnt ? __ldg(&cols[px + lane]) : 0u;
    const float* vp = vals + py + lane;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if ((mask >> k) & 1u) {
        S.v[k] = __ldg(vp);
        vp += 32;
      }
    }
  };
  auto gather = [&](V18Slot& S) {
    S.x0 = S.x1 = S.x2 = 0.0;
    const uint32_t c = S.col;
    const bool kept = bits ? ((v18_bits[c >> 5] >> (c & 31u)) & 1u) : true;
    if (kept && lane < (int)((S.info >> 8) & 0xffu)) {
      double x3;
      asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
                   : "=d"(S.x0), "=d"(S.x1), "=d"(S.x2), "=d"(x3)
                   : "l"(xp + c));
    }
  };

  double acc[24];
#pragma unroll
  for (int t = 0; t < 24; ++t) acc[t] = 0.0;
  // one step: consume C (x gathered), gather N (loaded), load F (free) <- j+2
  auto step = [&](unsigned j, V18Slot& C, V18Slot& Nx, V18Slot& F) {
    if (j + 2 < ns) load(F, j + 2);
    if (j + 1 < ns) gather(Nx);
    const unsigned mask = C.info & 0xffu;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if ((mask >> k) & 1u) {
        const double v = (double)C.v[k];
        acc[3 * k + 0] = fma(v, C.x0, acc[3 * k + 0]);
        acc[3 * k + 1] = fma(v, C.x1, acc[3 * k + 1]);
        acc[3 * k + 2] = fma(v, C.x2, acc[3 * k + 2]);
      }
    }
    if (((C.info >> 16) & 1u) || j + 1 == ns) {
      double r[3];
      v12_reduce24(acc, lane, r);
      if ((lane & 3) == 0) {
        const int g = lane >> 2;
#pragma unroll
        for (int t = 0; t < 3; ++t) {
          const int f = 3 * g + t;  // = 3 k + c
          if (f < 3 * K && r[t] != 0.0) atomicAdd(&vk[(size_t)f * N + C.row], r[t]);
        }
      }
#pragma unroll
      for (int t = 0; t < 24; ++t) acc[t] = 0.0;
    }
    if (j + 1 == base + 32) {  // next record batch
      rA = rB;
      base += 32;
      rB = make_uint4(0u, 0u, 0u, 0u);
      if (base + 32 + lane < ns) rB = __ldg(&steps[s0 + base + 32 + lane]);
    }
  };
  V18Slot S0, S1, S2;
  load(S0, 0);
  if (1 < ns) load(S1, 1);
  gather(S0);
  // unrolled by 3 so the slots change roles without register moves
#pragma unroll 1
  for (unsigned j = 0; j < ns; j += 3) {
    step(j, S0, S1, S2);
    if (j + 1 >= ns) break;
    step(j + 1, S1, S2, S0);
    if (j + 2 >= ns) break;
    step(j + 2, S2, S0, S1);
  }
}

}  // namespace sss
