// Transfer v19: receiver regions with the x working set in shared memory.
//
// The dipole operator is spatially local: the 64 rows of one 2^L receiver tile
// read ~8.3 K distinct columns on C3 (each x value ~8 times), of which ~4.6 K
// are kept in a frame. A persistent CTA takes one region at a time:
//   1. map: over the region's sorted union column list, a block scan of the
//      kept bits assigns compact shared-memory slots; kept x values (fp64, 3
//      channels) are gathered once, coalesced (sorted columns), into smem;
//      columns kept past the smem capacity fall back to global gathers;
//   2. stream: the warps split the region's 256-entry iterations of the flat8
//      stream (segments padded to 8, lane-interleaved, regions padded to whole
//      iterations) whose column fields hold region-local slots; x comes from
//      shared memory (LDS) instead of L1/L2 gathers; segment sums by the
//      head-flag segmented scan, tails add into the zeroed v_k.
// Unkept slots skip their loads and FMAs (exact zeros), like every variant.
#include "sss_common.cuh"  // V17Slot / v17_load / v15_gather1: flat15.cu, included first by abi.cu

namespace sss {

constexpr int kV19Threads = 768;
constexpr int kV19Warps = kV19Threads / 32;

// one stream iteration of a region: 8 entries per lane (region-local slots),
// x from the shared-memory tile, head-flag segmented scan, tails -> v_k
__device__ __forceinline__ void v19_consume(const V17Slot& S, const short* map, const double* xs,
                                            const uint32_t* __restrict__ ucols, int u0,
                                            const double4* __restrict__ xp, int lane,
                                            unsigned upto, int N,
                                            const uint32_t* __restrict__ rowk,
                                            double* __restrict__ vk) {
  double p0 = 0.0, p1 = 0.0, p2 = 0.0;
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const uint32_t sl = v17_col(S, e);
    const double v = (double)v17_val(S, e);
    const int m = map[sl];
    if (m >= 0) {
      p0 = fma(v, xs[3 * m], p0);
      p1 = fma(v, xs[3 * m + 1], p1);
      p2 = fma(v, xs[3 * m + 2], p2);
    } else if (m == -2) {
      double x[3];
      v15_gather1(xp, __ldg(&ucols[u0 + sl]), x);
      p0 = fma(v, x[0], p0);
      p1 = fma(v, x[1], p1);
      p2 = fma(v, x[2], p2);
    }
  }
  const unsigned hm = S.h & upto;
  const int sstart = hm ? 31 - __clz(hm) : -1;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double y0 = __shfl_up_sync(0xffffffffu, p0, o);
    const double y1 = __shfl_up_sync(0xffffffffu, p1, o);
    const double y2 = __shfl_up_sync(0xffffffffu, p2, o);
    if (lane >= o && lane - o >= sstart) {
      p0 += y0;
      p1 += y1;
      p2 += y2;
    }
  }
  const bool tail = (lane == 31) || ((S.h >> (lane + 1)) & 1u);
  if (tail && (p0 != 0.0 || p1 != 0.0 || p2 != 0.0)) {
    const unsigned rk = __ldg(&rowk[S.hp + __popc(hm) - 1u]);
    double* vo = vk + (size_t)(rk & 15u) * 3 * N + (rk >> 4);
    atomicAdd(vo, p0);
    atomicAdd(vo + N, p1);
    atomicAdd(vo + 2 * (size_t)N, p2);
  }
}

__global__ void __launch_bounds__(kV19Threads, 1) k_transfer_regional(
    int N, int n_regions, int xcap, const uint32_t* __restrict__ ucols,
    const int* __restrict__ uoff, const int* __restrict__ rit,
    const unsigned long long* __restrict__ C8, const unsigned long long* __restrict__ V8,
    unsigned n8, const uint32_t* __restrict__ H, const uint32_t* __restrict__ hpre,
    const uint32_t* __restrict__ rowk, const double4* __restrict__ xp,
    const uint32_t* __restrict__ bits, double* __restrict__ vk) {
  extern __shared__ __align__(16) uint8_t v19_smem[];
  const int nwb = (N + 31) >> 5;
  uint32_t* sbits = reinterpret_cast<uint32_t*>(v19_smem);                     // kept bitmap
  double* xs = reinterpret_cast<double*>(v19_smem + (((size_t)nwb * 4 + 15) & ~size_t(15)));
  short* map = reinterpret_cast<short*>(xs + (size_t)xcap * 3);               // slot -> x index
  __shared__ int wsum[kV19Warps];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int q = tid; q < nwb; q += kV19Threads) sbits[q] = bits[q];
  __syncthreads();
  const unsigned upto = (2u << lane) - 1u;

#pragma unroll 1
  for (int r = blockIdx.x; r < n_regions; r += gridDim.x) {
    const int u0 = uoff[r], nu = uoff[r + 1] - u0;
    // ---- 1a. kept flags (coalesced over the sorted union list)
    for (int s = tid; s < nu; s += kV19Threads) {
      const uint32_t c = __ldg(&ucols[u0 + s]);
      map[s] = (short)((sbits[c >> 5] >> (c & 31u)) & 1u);
    }
    __syncthreads();
    // ---- 1b. exclusive scan of the flags (chunked over shared memory)
    const int per = (nu + kV19Threads - 1) / kV19Threads;
    const int s0 = min(tid * per, nu), s1 = min(s0 + per, nu);
    int cnt = 0;
    for (int s = s0; s < s1; ++s) cnt += map[s];
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      const int w = lane < kV19Warps ? wsum[lane] : 0;
      int wi = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, wi, o);
        if (lane >= o) wi += y;
      }
      if (lane < kV19Warps) wsum[lane] = wi - w;
    }
    __syncthreads();
    int k = wsum[warp] + incl - cnt;
    for (int s = s0; s < s1; ++s) {
      if (map[s]) {
        map[s] = (short)(k < xcap ? k : -2);
        ++k;
      } else {
        map[s] = -1;
      }
    }
    __syncthreads();
    // ---- 1c. x tile: independent gathers (coalesced-ish: sorted columns)
    for (int s = tid; s < nu; s += kV19Threads) {
      const int m = map[s];
      if (m >= 0) {
        double x[3];
        v15_gather1(xp, __ldg(&ucols[u0 + s]), x);
        xs[3 * m] = x[0];
        xs[3 * m + 1] = x[1];
        xs[3 * m + 2] = x[2];
      }
    }
    __syncthreads();
    // ---- 2. stream the region's iterations: warp w takes w, w + W, ...,
    //         two iterations in flight
    const int it0 = rit[r], it1 = rit[r + 1];
#pragma unroll 1
    for (int i = it0 + warp; i < it1; i += 2 * kV19Warps) {
      V17Slot A, B;
      v17_load(A, (unsigned)i, lane, n8, C8, V8, H, hpre);
      const bool two = i + kV19Warps < it1;
      if (two) v17_load(B, (unsigned)(i + kV19Warps), lane, n8, C8, V8, H, hpre);
      v19_consume(A, map, xs, ucols, u0, xp, lane, upto, N, rowk, vk);
      if (two) v19_consume(B, map, xs, ucols, u0, xp, lane, upto, N, rowk, vk);
    }
    __syncthreads();  // map / xs reused by the next region
  }
}

}  // namespace sss
