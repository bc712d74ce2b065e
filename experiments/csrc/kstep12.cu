// Transfer v12: mask-sorted K-fused warp steps.
//
// The (row, column) pairs of the K operators (K-fill 0.37 on C3) are sorted,
// within a row, by (popcount, k-mask) and cut into 32-pair warp steps. A step
// stores its 32 columns and, for every k in the OR of its pairs' masks, 32
// f32 values in lane order (0 where a pair lacks k): one coalesced 128-byte
// load per (step, k), one 256-bit x gather per pair, and a k loop that is
// uniform across the warp (no per-lane mask bookkeeping). Mask sorting keeps
// the padding at ~1.7x the coefficients, so the stored bytes match the
// per-term CSR while the x gathers drop 3x.
//
// Steps are cut into cost-balanced contiguous per-warp ranges (persistent
// grid). acc[k][c] lives in registers; at a row end (or the end of the warp's
// range) the 24 sums are reduced across the warp with a transposed butterfly
// (27 double shuffles) and added into the zeroed v_k with red.global.add.f64.
// Epilogue: k_edit_finish.
#include "sss_common.cuh"

namespace sss {

constexpr int kV12Threads = 128;

struct V12Step {
  unsigned pair0;  // first column of the step in cols
  unsigned val0;   // first value (multiple of 32)
  unsigned row;    // tile-major row
  unsigned info;   // k-mask | count << 8 | row_end << 16
};

// 24 per-lane partial sums -> lane (g << 2), g = lane >> 2 in 0..7, holds the
// complete sums of a[3g .. 3g+2]; 12 + 6 + 3 + 3 + 3 shuffles.
__device__ __forceinline__ void v12_reduce24(const double (&a)[24], int lane, double (&r)[3]) {
  double b[12];
  const bool h4 = lane & 16;
#pragma unroll
  for (int i = 0; i < 12; ++i) {
    const double send = h4 ? a[i] : a[i + 12];
    const double keep = h4 ? a[i + 12] : a[i];
    b[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
  }
  double c[6];
  const bool h3 = lane & 8;
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    const double send = h3 ? b[i] : b[i + 6];
    const double keep = h3 ? b[i + 6] : b[i];
    c[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
  }
  const bool h2 = lane & 4;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const double send = h2 ? c[i] : c[i + 3];
    const double keep = h2 ? c[i + 3] : c[i];
    r[i] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
  }
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    r[i] += __shfl_xor_sync(0xffffffffu, r[i], 2);
    r[i] += __shfl_xor_sync(0xffffffffu, r[i], 1);
  }
}

__global__ void __launch_bounds__(kV12Threads) k_transfer_kstep(
    int K, int N, const uint32_t* __restrict__ cols, const float* __restrict__ vals,
    const uint4* __restrict__ steps, const unsigned* __restrict__ warp_begin,
    const double4* __restrict__ xp, double* __restrict__ vk) {
  const int lane = threadIdx.x & 31;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const unsigned s0 = warp_begin[w], s1 = warp_begin[w + 1];
  if (s0 >= s1) return;
  double acc[24];
#pragma unroll
  for (int i = 0; i < 24; ++i) acc[i] = 0.0;
  // one-step lookahead: the next step's record, column and x gather
  uint4 rec = __ldg(&steps[s0]);
  double x0 = 0.0, x1 = 0.0, x2 = 0.0;
  {
    const bool act = lane < (int)((rec.w >> 8) & 0xffu);
    if (act) {
      const uint32_t c = __ldg(&cols[rec.x + lane]);
      double x3;
      asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
                   : "=d"(x0), "=d"(x1), "=d"(x2), "=d"(x3) : "l"(xp + c));
    }
  }
  for (unsigned s = s0; s < s1; ++s) {
    const uint4 cur = rec;
    const double c0 = x0, c1 = x1, c2 = x2;
    if (s + 1 < s1) {
      rec = __ldg(&steps[s + 1]);
      const bool act = lane < (int)((rec.w >> 8) & 0xffu);
      x0 = x1 = x2 = 0.0;
      if (act) {
        const uint32_t c = __ldg(&cols[rec.x + lane]);
        double x3;
        asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
                     : "=d"(x0), "=d"(x1), "=d"(x2), "=d"(x3) : "l"(xp + c));
      }
    }
    const unsigned mask = cur.w & 0xffu;
    float v[8];
    unsigned j = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      v[k] = 0.0f;
      if ((mask >> k) & 1u) {
        v[k] = __ldg(&vals[cur.y + j * 32 + lane]);
        ++j;
      }
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if ((mask >> k) & 1u) {
        const double dv = (double)v[k];
        acc[3 * k + 0] = fma(dv, c0, acc[3 * k + 0]);
        acc[3 * k + 1] = fma(dv, c1, acc[3 * k + 1]);
        acc[3 * k + 2] = fma(dv, c2, acc[3 * k + 2]);
      }
    }
    if ((cur.w >> 16) & 1u || s + 1 == s1) {
      double r[3];
      v12_reduce24(acc, lane, r);
      if ((lane & 3) == 0) {
        const int g = lane >> 2;
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          const int f = 3 * g + i;  // = 3 k + c
          if (f < 3 * K) atomicAdd(&vk[(size_t)f * N + cur.z], r[i]);
        }
      }
#pragma unroll
      for (int i = 0; i < 24; ++i) acc[i] = 0.0;
    }
  }
}

}  // namespace sss
