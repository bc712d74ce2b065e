// Transfer v9: persistent merge-path CSR SpMV, 4 pieces per warp in flight.
//
// Same schedule idea as v8 — (row, k)-ordered segment pieces cut into
// entry-balanced contiguous per-warp ranges, x gathered through L1 from a
// packed (N, 4) fp64 array — with two changes that multiply the bytes each
// warp keeps in flight:
//   * every (k, row) segment is padded to a multiple of 4 entries (col 0,
//     val 0) in a separate 16-byte aligned copy of the operator, so a lane
//     loads 4 columns + 4 values with two 16-byte loads;
//   * a warp is 4 groups of 8 lanes, group g streaming pieces g, g+4, ... of
//     the warp's range, 32 entries per group-step, 2 steps in flight.
// Group reduction (3 shuffle steps) per piece, red.global.add.f64 into v_k.
#include "sss_common.cuh"

namespace sss {

constexpr int kV9Threads = 256;

struct V9Piece {
  unsigned start;  // first entry (multiple of 4) in the padded arrays
  unsigned len4;   // entries, multiple of 4
  unsigned rowk;   // tile-major row * 16 + k
  unsigned pad;
};

// one 256-bit read-only load (LDG.E.ENL2.256 on sm_100a): the packed
// {x0, x1, x2, 0} of a column in a single L1 request
__device__ __forceinline__ void v9_acc(const double4* __restrict__ xp, uint32_t c, float v,
                                       double& a0, double& a1, double& a2) {
  double x0, x1, x2, x3;
  asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(x0), "=d"(x1), "=d"(x2), "=d"(x3)
               : "l"(xp + c));
  const double dv = (double)v;
  a0 = fma(dv, x0, a0);
  a1 = fma(dv, x1, a1);
  a2 = fma(dv, x2, a2);
}

__global__ void __launch_bounds__(kV9Threads) k_transfer_csr9(
    int N, const uint4* __restrict__ cols4, const float4* __restrict__ vals4,
    const V9Piece* __restrict__ pieces, const unsigned* __restrict__ warp_begin,
    const double4* __restrict__ xp, double* __restrict__ vk) {
  const int lane = threadIdx.x & 31, grp = lane >> 3, gl = lane & 7;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const unsigned b = warp_begin[w], e_end = warp_begin[w + 1];
  const unsigned gmask = 0xffu << (grp * 8);
  // group g takes pieces b + g, b + g + 4, ...; all groups iterate the same
  // number of rounds (inactive groups idle) so warp-synchronous shuffles are safe
  const unsigned rounds = (e_end - b + 3) / 4;
  for (unsigned r = 0; r < rounds; ++r) {
    const unsigned pi = b + r * 4 + grp;
    const bool act = pi < e_end;
    V9Piece pc = {0u, 0u, 0u, 0u};
    if (act) pc = pieces[pi];
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    const unsigned q0 = pc.start >> 2, qn = pc.len4 >> 2;  // in uint4 units
    unsigned q = gl;
    for (; q + 8 < qn; q += 16) {  // two 32-entry steps per group in flight
      const uint4 c0 = __ldg(&cols4[q0 + q]), c1 = __ldg(&cols4[q0 + q + 8]);
      const float4 v0 = __ldg(&vals4[q0 + q]), v1 = __ldg(&vals4[q0 + q + 8]);
      v9_acc(xp, c0.x, v0.x, a0, a1, a2); v9_acc(xp, c0.y, v0.y, a0, a1, a2);
      v9_acc(xp, c0.z, v0.z, a0, a1, a2); v9_acc(xp, c0.w, v0.w, a0, a1, a2);
      v9_acc(xp, c1.x, v1.x, a0, a1, a2); v9_acc(xp, c1.y, v1.y, a0, a1, a2);
      v9_acc(xp, c1.z, v1.z, a0, a1, a2); v9_acc(xp, c1.w, v1.w, a0, a1, a2);
    }
    if (q < qn) {
      const uint4 c0 = __ldg(&cols4[q0 + q]);
      const float4 v0 = __ldg(&vals4[q0 + q]);
      v9_acc(xp, c0.x, v0.x, a0, a1, a2); v9_acc(xp, c0.y, v0.y, a0, a1, a2);
      v9_acc(xp, c0.z, v0.z, a0, a1, a2); v9_acc(xp, c0.w, v0.w, a0, a1, a2);
    }
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) {
      a0 += __shfl_xor_sync(0xffffffffu, a0, o);
      a1 += __shfl_xor_sync(0xffffffffu, a1, o);
      a2 += __shfl_xor_sync(0xffffffffu, a2, o);
    }
    (void)gmask;
    if (act && gl == 0) {
      const int row = (int)(pc.rowk >> 4), k = (int)(pc.rowk & 15u);
      double* vo = vk + (size_t)k * 3 * N;
      atomicAdd(&vo[row], a0);
      atomicAdd(&vo[N + row], a1);
      atomicAdd(&vo[2 * N + row], a2);
    }
  }
}

// csr9 with selection skip: the packed x comes with a tile-major bitmap of
// the columns some channel keeps (x != 0); it is staged in shared memory and
// an entry whose column is not kept issues no gather and no FMA (its
// contribution is an exact zero, so v_k is unchanged bit for bit). The
// reference's csc_apply only visits kept columns (transfer.py:66-71); this is
// the row-major equivalent.
__device__ __forceinline__ void v9s_acc(const double4* __restrict__ xp, const uint32_t* sbits,
                                        uint32_t c, float v, double& a0, double& a1, double& a2) {
  if ((sbits[c >> 5] >> (c & 31u)) & 1u) v9_acc(xp, c, v, a0, a1, a2);
}

__global__ void __launch_bounds__(kV9Threads) k_transfer_csr9s(
    int N, const uint4* __restrict__ cols4, const float4* __restrict__ vals4,
    const V9Piece* __restrict__ pieces, const unsigned* __restrict__ warp_begin,
    const double4* __restrict__ xp, const uint32_t* __restrict__ bits, double* __restrict__ vk) {
  extern __shared__ uint32_t sbits[];
  const int nw = (N + 31) >> 5;
  for (int i = threadIdx.x; i < nw; i += blockDim.x) sbits[i] = bits[i];
  __syncthreads();
  const int lane = threadIdx.x & 31, grp = lane >> 3, gl = lane & 7;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const unsigned b = warp_begin[w], e_end = warp_begin[w + 1];
  const unsigned rounds = (e_end - b + 3) / 4;
  for (unsigned r = 0; r < rounds; ++r) {
    const unsigned pi = b + r * 4 + grp;
    const bool act = pi < e_end;
    V9Piece pc = {0u, 0u, 0u, 0u};
    if (act) pc = pieces[pi];
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    const unsigned q0 = pc.start >> 2, qn = pc.len4 >> 2;
    unsigned q = gl;
    for (; q + 8 < qn; q += 16) {
      const uint4 c0 = __ldg(&cols4[q0 + q]), c1 = __ldg(&cols4[q0 + q + 8]);
      const float4 v0 = __ldg(&vals4[q0 + q]), v1 = __ldg(&vals4[q0 + q + 8]);
      v9s_acc(xp, sbits, c0.x, v0.x, a0, a1, a2); v9s_acc(xp, sbits, c0.y, v0.y, a0, a1, a2);
      v9s_acc(xp, sbits, c0.z, v0.z, a0, a1, a2); v9s_acc(xp, sbits, c0.w, v0.w, a0, a1, a2);
      v9s_acc(xp, sbits, c1.x, v1.x, a0, a1, a2); v9s_acc(xp, sbits, c1.y, v1.y, a0, a1, a2);
      v9s_acc(xp, sbits, c1.z, v1.z, a0, a1, a2); v9s_acc(xp, sbits, c1.w, v1.w, a0, a1, a2);
    }
    if (q < qn) {
      const uint4 c0 = __ldg(&cols4[q0 + q]);
      const float4 v0 = __ldg(&vals4[q0 + q]);
      v9s_acc(xp, sbits, c0.x, v0.x, a0, a1, a2); v9s_acc(xp, sbits, c0.y, v0.y, a0, a1, a2);
      v9s_acc(xp, sbits, c0.z, v0.z, a0, a1, a2); v9s_acc(xp, sbits, c0.w, v0.w, a0, a1, a2);
    }
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) {
      a0 += __shfl_xor_sync(0xffffffffu, a0, o);
      a1 += __shfl_xor_sync(0xffffffffu, a1, o);
      a2 += __shfl_xor_sync(0xffffffffu, a2, o);
    }
    if (act && gl == 0) {
      const int row = (int)(pc.rowk >> 4), k = (int)(pc.rowk & 15u);
      double* vo = vk + (size_t)k * 3 * N;
      atomicAdd(&vo[row], a0);
      atomicAdd(&vo[N + row], a1);
      atomicAdd(&vo[2 * N + row], a2);
    }
  }
}

// packed x + kept-column bitmap (bit c of bits set iff any channel of x[:, c]
// is nonzero); n a multiple of 32
__global__ void k_pack_x_bits(const double* __restrict__ x, int N, double4* __restrict__ xp,
                              uint32_t* __restrict__ bits) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  double a = 0.0, b = 0.0, c = 0.0;
  if (i < N) {
    a = x[i]; b = x[N + i]; c = x[2 * N + i];
    xp[i] = make_double4(a, b, c, 0.0);
  }
  const unsigned m = __ballot_sync(0xffffffffu, i < N && (a != 0.0 || b != 0.0 || c != 0.0));
  if ((threadIdx.x & 31) == 0 && i < N) bits[i >> 5] = m;
}

// packed x in a permuted column order (xp[j] = x[:, perm[j]]) + the kept
// bitmap in that order: the flat8 layout's 2x2-tile-block column space
__global__ void k_pack_x_perm_bits(const double* __restrict__ x, int N,
                                   const int* __restrict__ perm, double4* __restrict__ xp,
                                   uint32_t* __restrict__ bits) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  double a = 0.0, b = 0.0, c = 0.0;
  if (j < N) {
    const int i = perm[j];
    a = x[i]; b = x[N + i]; c = x[2 * N + i];
    xp[j] = make_double4(a, b, c, 0.0);
  }
  const unsigned m = __ballot_sync(0xffffffffu, j < N && (a != 0.0 || b != 0.0 || c != 0.0));
  if ((threadIdx.x & 31) == 0 && j < N) bits[j >> 5] = m;
}

// packed fp32 x (N, 4) {x0, x1, x2, 0} + the kept-column bitmap
__global__ void k_pack_x_f32_bits(const double* __restrict__ x, int N, float4* __restrict__ xp,
                                  uint32_t* __restrict__ bits) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  double a = 0.0, b = 0.0, c = 0.0;
  if (i < N) {
    a = x[i]; b = x[N + i]; c = x[2 * N + i];
    xp[i] = make_float4((float)a, (float)b, (float)c, 0.0f);
  }
  const unsigned m = __ballot_sync(0xffffffffu, i < N && (a != 0.0 || b != 0.0 || c != 0.0));
  if ((threadIdx.x & 31) == 0 && i < N) bits[i >> 5] = m;
}

// padded copy of the canonical CSR: segment i (start s, len l) -> new start
// ps (multiple of 4), entries copied, padding (col 0, val 0)
__global__ void k_pad_segments(const uint64_t* __restrict__ seg_src, const uint32_t* __restrict__ seg_len,
                               const uint64_t* __restrict__ seg_dst, long long nseg,
                               const uint32_t* __restrict__ cols, const float* __restrict__ vals,
                               uint32_t* __restrict__ pcols, float* __restrict__ pvals) {
  const long long i = (long long)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (i >= nseg) return;
  const int lane = threadIdx.x & 31;
  const uint64_t s = seg_src[i], d = seg_dst[i];
  const uint32_t l = seg_len[i], l4 = (l + 3u) & ~3u;
  for (uint32_t j = lane; j < l4; j += 32) {
    pcols[d + j] = j < l ? cols[s + j] : 0u;
    pvals[d + j] = j < l ? vals[s + j] : 0.0f;
  }
}

}  // namespace sss
