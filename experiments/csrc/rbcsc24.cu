// Transfer v24 "rbcsc": row-block column-major transfer with exact fixed-point
// accumulation in shared memory.
//
// Every row-major variant (flat8 and its successors) gathers x once per
// stored coefficient whose column is kept: 28.8 M random 32-byte gathers per
// C3 frame, one L1TEX wavefront each, which is what bounds them (LSU
// wavefronts ~80 % of peak). Here the operator is stored per block of RB
// consecutive (tile-major) receiver rows in column-major order: for each
// (row block, column) a segment of entries (row in block | k << 7, f32
// value), described by (column, length, offset). Per frame a CTA owns one row
// block: its warps walk the block's segment descriptors 32 at a time, keep
// the segments whose column is in the frame's kept set (the per-frame
// union over channels), fetch that column's x once for the whole segment
// (2.5 M fetches per frame instead of 28.8 M) and stream only the kept
// segments' entries (only touched coefficients are read: 6 bytes each).
//
// The entries of a segment scatter into (row, k) outputs of the block; the
// CTA accumulates them in shared memory as 64-bit fixed-point integers, each
// kept as two 32-bit words updated with native 32-bit shared atomics (carry
// from the returned old low word): q = rn(v * x * S_kc), S_kc = 2^(61 - e),
// 2^e > B_kc = max_row sum |T_k| * max |x_c| (max |x_c| bounded by the square
// root of the kept energy of channel c). Integer sums are exact and order
// independent, so the result is deterministic; each product is rounded once
// to 2^-61 B_kc (the f32 operator values and the fp64 x enter exactly). At the
// end the CTA writes its block's v_k rows (every row, zeros included): no
// memset, no global atomics.
#include "sss_common.cuh"

namespace sss {

constexpr int kV24Threads = 256;
constexpr int kV24Warps = kV24Threads / 32;

template <int RB, int K>
__global__ void __launch_bounds__(kV24Threads) k_transfer_rbcsc(
    int N, const uint2* __restrict__ desc, const uint32_t* __restrict__ dptr,
    const uint16_t* __restrict__ rk, const float* __restrict__ vals,
    const double* __restrict__ rowabs, const double* __restrict__ energy,
    const double4* __restrict__ xp, const uint32_t* __restrict__ bits,
    double* __restrict__ vk) {
  constexpr int kSh = RB == 32 ? 5 : RB == 64 ? 6 : 7;  // row-in-block bits
  static_assert(RB == 32 || RB == 64 || RB == 128, "RB in {32, 64, 128}");
  // exact 64-bit fixed-point sums as two 32-bit halves: native shared-memory
  // ATOMS.ADD on the low word returns the old value, so the carry of every
  // single addition is known and added to the high word (64-bit shared
  // atomics compile to CAS loops on sm_100a)
  // (k, c) planes of RB + 1 words: entries of one segment share rows, so a
  // plain RB stride would put (row, k) and (row, k') in the same bank
  constexpr int PL = RB + 1;
  __shared__ uint32_t acc_lo[K * 3 * PL], acc_hi[K * 3 * PL];
  __shared__ double scale[K * 3], inv_scale[K * 3];
  __shared__ double xs[kV24Warps][32][3];
  __shared__ uint32_t sst[kV24Warps][33], soff[kV24Warps][32];
  __shared__ uint32_t smask[kV24Warps][32], wpre[kV24Warps][32];
  const int rb = blockIdx.x;
  for (int t = threadIdx.x; t < K * 3 * PL; t += blockDim.x) acc_lo[t] = acc_hi[t] = 0u;
  if (threadIdx.x < K * 3) {
    const int k = threadIdx.x / 3, c = threadIdx.x % 3;
    const double B = rowabs[k] * sqrt(fmax(energy[c * 2 + 1], 0.0));
    int e = 0;
    if (B > 0.0) frexp(B, &e);  // B < 2^e
    scale[threadIdx.x] = B > 0.0 ? ldexp(1.0, 61 - e) : 1.0;
    inv_scale[threadIdx.x] = B > 0.0 ? ldexp(1.0, e - 61) : 1.0;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint32_t d0 = dptr[rb], d1 = dptr[rb + 1];
  const unsigned lt = (1u << lane) - 1u;
#pragma unroll 1
  for (uint32_t d = d0 + wid * 32; d < d1; d += kV24Warps * 32) {
    const bool valid = d + lane < d1;
    const uint2 ds = valid ? __ldg(desc + d + lane) : make_uint2(0u, 0u);
    const uint32_t col = ds.x & 0xffffu, cnt = ds.x >> 16;
    const bool kept = valid && ((__ldg(bits + (col >> 5)) >> (col & 31u)) & 1u);
    const unsigned m = __ballot_sync(0xffffffffu, kept);
    if (!m) continue;
    // exclusive scan of the kept segments' lengths over the lanes
    uint32_t inc = kept ? cnt : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    const uint32_t total = __shfl_sync(0xffffffffu, inc, 31);
    const uint32_t start = inc - cnt;
    smask[wid][lane] = 0u;
    __syncwarp();
    if (kept) {
      const int s = __popc(m & lt);
      double x3;
      asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
                   : "=d"(xs[wid][s][0]), "=d"(xs[wid][s][1]), "=d"(xs[wid][s][2]), "=d"(x3)
                   : "l"(xp + col));
      (void)x3;
      sst[wid][s] = start;
      soff[wid][s] = ds.y;
      // segment-start bitmap over the first 1024 virtual entries
      if (start < 1024u) atomicOr(&smask[wid][start >> 5], 1u << (start & 31u));
    }
    const int nk = __popc(m);
    if (lane == 0) sst[wid][nk] = total;
    __syncwarp();
    {
      const uint32_t pc = __popc(smask[wid][lane]);
      uint32_t ps = pc;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, ps, o);
        if (lane >= o) ps += y;
      }
      wpre[wid][lane] = ps - pc;
    }
    __syncwarp();
#pragma unroll 1
    for (uint32_t e = lane; e < total; e += 32) {
      int sg;  // the segment of virtual entry e: starts at or below e, minus one
      if (e < 1024u) {
        const uint32_t wd = smask[wid][e >> 5];
        sg = (int)(wpre[wid][e >> 5] + __popc(wd & ((2u << (e & 31u)) - 1u))) - 1;
      } else {  // long batches: binary search over the (<= 32) starts
        int a0 = 0, a1 = nk - 1;
        while (a0 < a1) {
          const int mid = (a0 + a1 + 1) >> 1;
          if (sst[wid][mid] <= e) a0 = mid; else a1 = mid - 1;
        }
        sg = a0;
      }
      const uint32_t idx = soff[wid][sg] + (e - sst[wid][sg]);
      const uint32_t q = __ldcs(rk + idx);
      const double v = (double)__ldcs(vals + idx);
      const int r = q & (RB - 1), k = q >> kSh;
      // branch-free: every product does both word updates (zeros included)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double p = dmul(v, xs[wid][sg][c]);
        const unsigned long long uq =
            (unsigned long long)__double2ll_rn(dmul(p, scale[k * 3 + c]));
        const int a = (k * 3 + c) * PL + r;
        const uint32_t wlo = (uint32_t)uq, whi = (uint32_t)(uq >> 32);
        const uint32_t old = atomicAdd(acc_lo + a, wlo);
        atomicAdd(acc_hi + a, whi + (uint32_t)(old + wlo < old));  // + carry of the low word
      }
    }
    __syncwarp();
  }
  __syncthreads();
  for (int t = threadIdx.x; t < K * 3 * RB; t += blockDim.x) {
    const int kc = t / RB, r = t % RB, a = kc * PL + r;
    const long long q = (long long)(((unsigned long long)acc_hi[a] << 32) | acc_lo[a]);
    vk[(size_t)kc * N + (size_t)rb * RB + r] = dmul(__ll2double_rn(q), inv_scale[kc]);
  }
}

}  // namespace sss
