// Transfer v22 "flat8c": the flat8 stream split into column partitions, with
// each CTA's partition of x resident in shared memory.
//
// flat8 is bound by its x gathers: 28.8 M 32-byte L2 gathers per C3 frame,
// one L1TEX wavefront per active lane and an L2 round trip (~1 us under
// load) in every lane's dependency chain. Here the operator's columns are cut
// into P partitions of CW = N / P consecutive tile-major ids; every (row, k)
// segment is split at partition boundaries (sub-segments padded to a multiple
// of 8 entries, column ids stored as 16-bit partition-local ids, so an entry
// is 6 bytes instead of 8), and the stream is ordered partition-major. A CTA
// serves one partition: it stages the partition's x (3 x CW fp64 planes) and
// kept bits in shared memory once, then its warps stream their equal ranges
// of the partition exactly like flat8 (8 entries per lane, head-flag
// segmented warp scan, tail lanes add into the zeroed v_k), with the x
// gathers served from shared memory.
#include "sss_common.cuh"

namespace sss {

constexpr int kV22Threads = 512;

struct V22Slot {
  uint4 c;                  // 8 u16 partition-local columns
  unsigned long long v[4];  // 8 f32 values
  uint32_t h, hp;
};

__device__ __forceinline__ void v22_load(V22Slot& S, unsigned i, int lane,
                                         const uint4* __restrict__ C16,
                                         const unsigned long long* __restrict__ V8,
                                         const uint32_t* __restrict__ H,
                                         const uint32_t* __restrict__ hpre) {
  const size_t q = (size_t)i * 32u + (unsigned)lane;
  S.c = __ldcs(C16 + q);
  asm volatile("ld.global.nc.L1::no_allocate.v4.u64 {%0,%1,%2,%3}, [%4];"
               : "=l"(S.v[0]), "=l"(S.v[1]), "=l"(S.v[2]), "=l"(S.v[3])
               : "l"(V8 + 4 * q));
  S.h = __ldg(&H[i]);
  S.hp = __ldg(&hpre[i]);
}

__device__ __forceinline__ uint32_t v22_col(const V22Slot& S, int e) {
  const uint32_t w = e < 2 ? S.c.x : e < 4 ? S.c.y : e < 6 ? S.c.z : S.c.w;
  return (w >> (16 * (e & 1))) & 0xffffu;
}
__device__ __forceinline__ float v22_val(const V22Slot& S, int e) {
  return __uint_as_float((uint32_t)(S.v[e >> 1] >> (32 * (e & 1))));
}

template <int CW>
__global__ void __launch_bounds__(kV22Threads, 2) k_transfer_flat8c(
    int N, const uint4* __restrict__ C16, const unsigned long long* __restrict__ V8,
    const uint32_t* __restrict__ H, const uint32_t* __restrict__ hpre,
    const uint32_t* __restrict__ rowk, const unsigned* __restrict__ warp_begin,
    const int* __restrict__ cta_part, const double4* __restrict__ xp,
    const uint32_t* __restrict__ bits, double* __restrict__ vk) {
  extern __shared__ double v22_sm[];
  double* xs = v22_sm;                                              // [3][CW]
  uint32_t* sb = reinterpret_cast<uint32_t*>(v22_sm + 3 * CW);     // [CW / 32]
  const int part = cta_part[blockIdx.x];
  const int c0 = part * CW;
  for (int t = threadIdx.x; t < CW; t += blockDim.x) {
    const double2* xq = reinterpret_cast<const double2*>(xp + c0 + t);
    const double2 a = __ldg(xq), b = __ldg(xq + 1);
    xs[t] = a.x;
    xs[CW + t] = a.y;
    xs[2 * CW + t] = b.x;
  }
  for (int t = threadIdx.x; t < CW / 32; t += blockDim.x) sb[t] = bits[c0 / 32 + t];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const unsigned i0 = warp_begin[w], i1 = warp_begin[w + 1];
  const unsigned upto = (2u << lane) - 1u;
#pragma unroll 1
  for (unsigned i = i0; i < i1; ++i) {
    V22Slot S;
    v22_load(S, i, lane, C16, V8, H, hpre);
    double p0 = 0.0, p1 = 0.0, p2 = 0.0;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const uint32_t c = v22_col(S, e);
      if ((sb[c >> 5] >> (c & 31u)) & 1u) {
        const double v = (double)v22_val(S, e);
        p0 = fma(v, xs[c], p0);
        p1 = fma(v, xs[CW + c], p1);
        p2 = fma(v, xs[2 * CW + c], p2);
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
}

}  // namespace sss
