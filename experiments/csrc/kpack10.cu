// Transfer v10: K-packed pair SpMV.
//
// The K = 8 PCA-term operators of a row share most of their column support
// (the same receiver sees the same source coefficients), so the layout stores
// each (row, column) pair ONCE: meta = column (24 bits) | k-mask (8 bits) << 24
// followed, in a parallel value stream, by the f32 values of the terms present
// (k ascending). One 256-bit gather of the packed x column serves every term
// of the pair (3x fewer L1 requests than per-term CSR on the C3 operator), and
// the stored bytes drop from 8 B per coefficient to 4 B per pair + 4 B per
// coefficient.
//
// Rows are padded to a multiple of 4 pairs (meta 0 = empty pair) so a lane
// takes 4 consecutive pairs with one 16-byte meta load; a warp step covers
// 128 pairs. Per step: meta -> popcounts -> warp scan; the 4 x gathers are
// issued first, then the warp's contiguous value run is copied (coalesced)
// into a per-warp shared-memory buffer and read back per lane, so value
// traffic costs ~S/32 L1 line requests instead of 8 scattered loads per pair.
//
// Pieces = runs of a row's pairs (long rows split), cut into cost-balanced
// contiguous per-warp ranges of a persistent grid; one warp reduction of the
// K*3 sums per piece, then red.global.add.f64 into v_k. Epilogue:
// k_edit_finish.
#include "sss_common.cuh"

namespace sss {

constexpr int kV10Threads = 256;
constexpr int kV10StepPairs = 128;                 // pairs per warp step
constexpr int kV10Buf = kV10StepPairs * 8;         // max values per step

struct V10Piece {
  unsigned pair0;  // first (padded) pair, multiple of 4
  unsigned npair;  // padded pairs, multiple of 4
  unsigned val0;   // first value of the first pair
  unsigned row;    // tile-major row
};

__device__ __forceinline__ void v10_gather(const double4* __restrict__ xp, uint32_t m, double& x0,
                                           double& x1, double& x2) {
  double x3;
  x0 = x1 = x2 = 0.0;
  if (m >> 24)
    asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(x0), "=d"(x1), "=d"(x2), "=d"(x3)
                 : "l"(xp + (m & 0xffffffu)));
}

template <int KMAX>
__device__ __forceinline__ void v10_pair(uint32_t m, const float* sv, unsigned& o, double x0,
                                         double x1, double x2, double (&acc)[KMAX][3]) {
  const unsigned mask = m >> 24;
#pragma unroll
  for (int k = 0; k < KMAX; ++k) {
    if ((mask >> k) & 1u) {
      const double v = (double)sv[o++];
      acc[k][0] = fma(v, x0, acc[k][0]);
      acc[k][1] = fma(v, x1, acc[k][1]);
      acc[k][2] = fma(v, x2, acc[k][2]);
    }
  }
}

template <int KMAX>
__global__ void __launch_bounds__(kV10Threads, 2) k_transfer_kpack(
    int K, int N, const uint4* __restrict__ meta4, const float* __restrict__ vals,
    const V10Piece* __restrict__ pieces, const unsigned* __restrict__ warp_begin,
    const double4* __restrict__ xp, double* __restrict__ vk) {
  __shared__ float s_val[kV10Threads / 32][kV10Buf];
  const int lane = threadIdx.x & 31;
  float* sv = s_val[threadIdx.x >> 5];
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const unsigned b = warp_begin[w], e_end = warp_begin[w + 1];
  for (unsigned pi = b; pi < e_end; ++pi) {
    const V10Piece pc = pieces[pi];
    double acc[KMAX][3];
#pragma unroll
    for (int k = 0; k < KMAX; ++k) acc[k][0] = acc[k][1] = acc[k][2] = 0.0;
    unsigned vbase = pc.val0;
    for (unsigned q = 0; q < pc.npair; q += kV10StepPairs) {
      const bool act = q + 4 * lane < pc.npair;
      uint4 m = make_uint4(0u, 0u, 0u, 0u);
      if (act) m = __ldg(&meta4[(pc.pair0 + q) / 4 + lane]);
      const unsigned c0 = __popc(m.x >> 24), c1 = __popc(m.y >> 24), c2 = __popc(m.z >> 24),
                     c3 = __popc(m.w >> 24);
      const unsigned cnt = c0 + c1 + c2 + c3;
      unsigned incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const unsigned S = __shfl_sync(0xffffffffu, incl, 31);
      // x gathers first (independent of the value copy)
      double xa0, xa1, xa2, xb0, xb1, xb2, xc0, xc1, xc2, xd0, xd1, xd2;
      v10_gather(xp, m.x, xa0, xa1, xa2);
      v10_gather(xp, m.y, xb0, xb1, xb2);
      v10_gather(xp, m.z, xc0, xc1, xc2);
      v10_gather(xp, m.w, xd0, xd1, xd2);
      // coalesced copy of this step's value run into the warp buffer
      for (unsigned s0 = 0; s0 < S; s0 += 256) {
        float r[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          const unsigned i = s0 + t * 32 + lane;
          r[t] = i < S ? __ldg(&vals[vbase + i]) : 0.0f;
        }
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          const unsigned i = s0 + t * 32 + lane;
          if (i < S) sv[i] = r[t];
        }
      }
      __syncwarp();
      unsigned o = incl - cnt;
      v10_pair<KMAX>(m.x, sv, o, xa0, xa1, xa2, acc);
      v10_pair<KMAX>(m.y, sv, o, xb0, xb1, xb2, acc);
      v10_pair<KMAX>(m.z, sv, o, xc0, xc1, xc2, acc);
      v10_pair<KMAX>(m.w, sv, o, xd0, xd1, xd2, acc);
      __syncwarp();
      vbase += S;
    }
    // warp reduction of the K x 3 sums
#pragma unroll
    for (int k = 0; k < KMAX; ++k) {
      if (k >= K) break;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        double a = acc[k][c];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
        if (lane == k * 3 + c) atomicAdd(&vk[((size_t)k * 3 + c) * N + pc.row], a);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Pipelined variant. A warp walks its steps (piece, q) with
//   * meta of step i+2 and values of step i+1 in flight as one cp.async group
//     (LDGSTS, no registers) into per-warp shared-memory rings,
//   * x gathers of step i+1 issued before step i is consumed,
// so each step exposes one memory latency instead of three dependent ones.
// ---------------------------------------------------------------------------
constexpr int kV11Threads = 128;

__device__ __forceinline__ void cp_async4(void* s, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(s)), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async8(void* s, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(s)), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async16(void* s, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(s)), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

template <int PPL>
struct V11Meta;
template <>
struct V11Meta<2> {
  using T = uint2;
  static __device__ __forceinline__ unsigned get(const T& m, int j) { return j == 0 ? m.x : m.y; }
};
template <>
struct V11Meta<4> {
  using T = uint4;
  static __device__ __forceinline__ unsigned get(const T& m, int j) {
    return j == 0 ? m.x : j == 1 ? m.y : j == 2 ? m.z : m.w;
  }
};

template <int KMAX, int PPL>
__global__ void __launch_bounds__(kV11Threads) k_transfer_kpack_pipe(
    int K, int N, const uint32_t* __restrict__ meta, const float* __restrict__ vals,
    const V10Piece* __restrict__ pieces, const unsigned* __restrict__ warp_begin,
    const double4* __restrict__ xp, double* __restrict__ vk) {
  constexpr int STEP = 32 * PPL;
  constexpr int WARPS = kV11Threads / 32;
  using MT = typename V11Meta<PPL>::T;
  __shared__ __align__(16) uint32_t s_meta[WARPS][3][STEP];
  __shared__ __align__(16) float s_val[WARPS][2][STEP * 8];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const unsigned b = warp_begin[w], e = warp_begin[w + 1];
  if (b >= e) return;

  // step cursors: piece index + pair offset + the piece descriptor
  unsigned pi0 = b, q0 = 0;
  V10Piece P0 = pieces[b];
  unsigned pi1 = pi0, q1 = q0 + STEP;
  V10Piece P1 = P0;
  if (q1 >= P1.npair) { ++pi1; q1 = 0; if (pi1 < e) P1 = pieces[pi1]; }
  unsigned pi2 = pi1, q2 = q1 + STEP;
  V10Piece P2 = P1;
  if (pi2 < e && q2 >= P2.npair) { ++pi2; q2 = 0; if (pi2 < e) P2 = pieces[pi2]; }

  auto issue_meta = [&](unsigned pi, unsigned q, const V10Piece& P, int slot) {
    if (pi < e && q + PPL * lane < P.npair) {
      if constexpr (PPL == 4)
        cp_async16(&s_meta[wl][slot][PPL * lane], meta + P.pair0 + q + PPL * lane);
      else
        cp_async8(&s_meta[wl][slot][PPL * lane], meta + P.pair0 + q + PPL * lane);
    }
  };
  auto read_meta = [&](unsigned pi, unsigned q, const V10Piece& P, int slot) {
    MT m;
    if constexpr (PPL == 4) m = make_uint4(0u, 0u, 0u, 0u); else m = make_uint2(0u, 0u);
    if (pi < e && q + PPL * lane < P.npair) m = *reinterpret_cast<const MT*>(&s_meta[wl][slot][PPL * lane]);
    return m;
  };
  auto scan = [&](const MT& m, unsigned& excl, unsigned& S) {
    unsigned cnt = 0;
#pragma unroll
    for (int j = 0; j < PPL; ++j) cnt += __popc(V11Meta<PPL>::get(m, j) >> 24);
    unsigned incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    S = __shfl_sync(0xffffffffu, incl, 31);
    excl = incl - cnt;
  };
  auto issue_vals = [&](unsigned vb, unsigned S, int slot) {
    for (unsigned i = lane; i < S; i += 32) cp_async4(&s_val[wl][slot][i], vals + vb + i);
  };

  // prologue: meta of steps 0 and 1, then values of step 0
  issue_meta(pi0, q0, P0, 0);
  issue_meta(pi1, q1, P1, 1);
  cp_async_commit();
  cp_async_wait_all();
  __syncwarp();
  MT m0 = read_meta(pi0, q0, P0, 0);
  unsigned ex0, S0;
  scan(m0, ex0, S0);
  unsigned vb0 = P0.val0;
  issue_vals(vb0, S0, 0);
  cp_async_commit();
  double x0[PPL][3];
#pragma unroll
  for (int j = 0; j < PPL; ++j) v10_gather(xp, V11Meta<PPL>::get(m0, j), x0[j][0], x0[j][1], x0[j][2]);

  double acc[KMAX][3];
#pragma unroll
  for (int k = 0; k < KMAX; ++k) acc[k][0] = acc[k][1] = acc[k][2] = 0.0;

  for (int i = 0;; ++i) {
    cp_async_wait_all();  // vals(i), meta(i+1)
    __syncwarp();
    // step i+1: scan, values + meta(i+2) in flight, gathers issued
    MT m1;
    unsigned ex1 = 0, S1 = 0, vb1 = 0;
    double x1[PPL][3];
    if (pi1 < e) {
      m1 = read_meta(pi1, q1, P1, (i + 1) % 3);
      scan(m1, ex1, S1);
      vb1 = (pi1 == pi0) ? vb0 + S0 : P1.val0;
      issue_vals(vb1, S1, (i + 1) & 1);
    }
    issue_meta(pi2, q2, P2, (i + 2) % 3);
    cp_async_commit();
    if (pi1 < e) {
#pragma unroll
      for (int j = 0; j < PPL; ++j)
        v10_gather(xp, V11Meta<PPL>::get(m1, j), x1[j][0], x1[j][1], x1[j][2]);
    }
    // consume step i
    {
      const float* sv = s_val[wl][i & 1];
      unsigned o = ex0;
#pragma unroll
      for (int j = 0; j < PPL; ++j) v10_pair<KMAX>(V11Meta<PPL>::get(m0, j), sv, o, x0[j][0], x0[j][1], x0[j][2], acc);
    }
    if (pi1 != pi0) {  // piece ends: reduce the K x 3 sums
#pragma unroll
      for (int k = 0; k < KMAX; ++k) {
        if (k < K) {
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            double a = acc[k][c];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
            if (lane == k * 3 + c) atomicAdd(&vk[((size_t)k * 3 + c) * N + P0.row], a);
          }
        }
        acc[k][0] = acc[k][1] = acc[k][2] = 0.0;
      }
    }
    __syncwarp();
    if (pi1 >= e) break;
    // rotate cursors
    pi0 = pi1; q0 = q1; P0 = P1; m0 = m1; ex0 = ex1; S0 = S1; vb0 = vb1;
#pragma unroll
    for (int j = 0; j < PPL; ++j) { x0[j][0] = x1[j][0]; x0[j][1] = x1[j][1]; x0[j][2] = x1[j][2]; }
    pi1 = pi2; q1 = q2; P1 = P2;
    if (pi2 < e) {
      q2 += STEP;
      if (q2 >= P2.npair) { ++pi2; q2 = 0; if (pi2 < e) P2 = pieces[pi2]; }
    }
  }
}

}  // namespace sss
