// Transfer v7: warp-per-(row, k) CSR SpMV with L1-resident x.
//
// A CTA owns G tiles (R rows); its R*K (row, k) segments are visited
// longest-first through a shared-memory work counter (dynamic LPT inside the
// CTA). A warp streams a segment's entries with coalesced loads (lane p takes
// entries p, p+32, ...), gathers x from a packed (N, 4) fp64 array — one
// 32-byte sector per entry, and because the operator has local support the
// columns a CTA touches repeat across its rows, so the gathers mostly hit L1
// (the kernel uses almost no shared memory, leaving L1 to x) — accumulates in
// fp64 registers and warp-reduces once per segment. v_k goes straight to
// global memory; after a CTA barrier the epilogue recombines from the (L2-hot)
// v_k, inverse-Haars the G tiles in one batch and shades.
#include "sss_common.cuh"

namespace sss {

constexpr int kV7Threads = 256;

// one 32-byte sector: {x0, x1} as a 16-byte read-only load + x2
__device__ __forceinline__ double4 ldx(const double4* __restrict__ xp, uint32_t c) {
  const double2* q = reinterpret_cast<const double2*>(xp + c);
  const double2 a = __ldg(q);
  const double b = __ldg(reinterpret_cast<const double*>(q + 1));
  return make_double4(a.x, a.y, b, 0.0);
}

__global__ void __launch_bounds__(kV7Threads) k_transfer_csr7(
    int K, int S, int L, int G, const uint64_t* __restrict__ rowptr,
    const uint32_t* __restrict__ cols, const float* __restrict__ vals,
    const unsigned short* __restrict__ order /* per CTA: R*K (row_local << 4 | k), longest first */,
    const double4* __restrict__ xp /* (N) {x0, x1, x2, 0}, tile-major columns */,
    const double* __restrict__ g, const float* __restrict__ positions,
    const float* __restrict__ normals, const double* __restrict__ cam,
    const double* __restrict__ material, double* __restrict__ vk, double* __restrict__ scatter,
    float* __restrict__ radiance, float* __restrict__ radiance_unclamped) {
  extern __shared__ double sm7[];
  __shared__ int counter;
  const int T = 1 << L, T2 = T * T, N = S * S;
  const int R = G * T2, tile0 = blockIdx.x * G, row0 = tile0 * T2;
  const int lane = threadIdx.x & 31;
  const int npairs = R * K;
  const unsigned short* ord = order + (size_t)blockIdx.x * npairs;
  if (threadIdx.x == 0) counter = 0;
  __syncthreads();
  while (true) {
    int idx = 0;
    if (lane == 0) idx = atomicAdd(&counter, 1);
    idx = __shfl_sync(0xffffffffu, idx, 0);
    if (idx >= npairs) break;
    const int pk = ord[idx];
    const int row = row0 + (pk >> 4), k = pk & 15;
    const uint64_t s = rowptr[(size_t)k * (N + 1) + row], e = rowptr[(size_t)k * (N + 1) + row + 1];
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    uint64_t p = s + lane;
    for (; p + 96 < e; p += 128) {  // 4 independent entries per lane in flight
      const uint32_t c0 = __ldg(&cols[p]), c1 = __ldg(&cols[p + 32]), c2 = __ldg(&cols[p + 64]),
                     c3 = __ldg(&cols[p + 96]);
      const float v0 = __ldg(&vals[p]), v1 = __ldg(&vals[p + 32]), v2 = __ldg(&vals[p + 64]),
                  v3 = __ldg(&vals[p + 96]);
      const double4 x0 = ldx(xp, c0), x1 = ldx(xp, c1), x2 = ldx(xp, c2), x3 = ldx(xp, c3);
      a0 = fma((double)v0, x0.x, a0); a1 = fma((double)v0, x0.y, a1); a2 = fma((double)v0, x0.z, a2);
      a0 = fma((double)v1, x1.x, a0); a1 = fma((double)v1, x1.y, a1); a2 = fma((double)v1, x1.z, a2);
      a0 = fma((double)v2, x2.x, a0); a1 = fma((double)v2, x2.y, a1); a2 = fma((double)v2, x2.z, a2);
      a0 = fma((double)v3, x3.x, a0); a1 = fma((double)v3, x3.y, a1); a2 = fma((double)v3, x3.z, a2);
    }
    for (; p < e; p += 32) {
      const uint32_t c = __ldg(&cols[p]);
      const double v = (double)__ldg(&vals[p]);
      const double4 xv = ldx(xp, c);
      a0 = fma(v, xv.x, a0); a1 = fma(v, xv.y, a1); a2 = fma(v, xv.z, a2);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a0 += __shfl_xor_sync(0xffffffffu, a0, o);
      a1 += __shfl_xor_sync(0xffffffffu, a1, o);
      a2 += __shfl_xor_sync(0xffffffffu, a2, o);
    }
    if (lane == 0) {
      double* vo = vk + (size_t)k * 3 * N;
      vo[row] = a0; vo[N + row] = a1; vo[2 * N + row] = a2;
    }
  }
  __syncthreads();  // this CTA's v_k rows are complete (own writes, visible to the CTA)
  double* summed = sm7;                       // G x 3 x T2
  double* tmp = summed + (size_t)G * 3 * T2;  // same
  for (int r = threadIdx.x; r < R; r += blockDim.x) {
    const int row = row0 + r;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
    for (int k = 0; k < K; ++k) {
      const double* vo = vk + (size_t)k * 3 * N;
      s0 += g[k] * vo[row];
      s1 += g[K + k] * vo[N + row];
      s2 += g[2 * K + k] * vo[2 * N + row];
    }
    const int tj = r / T2, e = r % T2;
    summed[(tj * 3 + 0) * T2 + e] = s0;
    summed[(tj * 3 + 1) * T2 + e] = s1;
    summed[(tj * 3 + 2) * T2 + e] = s2;
  }
  __syncthreads();
  multi_tile_epilogue(summed, tmp, T, tile0, G, S, positions, normals, cam, material, scatter,
                      radiance, radiance_unclamped);
}

// x (3, N) -> packed (N) {x0, x1, x2, 0}
__global__ void k_pack_x(const double* __restrict__ x, int N, double4* __restrict__ xp) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < N) xp[i] = make_double4(x[i], x[N + i], x[2 * N + i], 0.0);
}

}  // namespace sss
