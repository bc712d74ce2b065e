// Transfer v13: mask-sorted K-fused warp steps, TMA-streamed.
//
// Same warp steps as v12 (pairs of a row sorted by k-mask, 32 per step, one
// 256-bit x gather per pair, k loop uniform across the warp), but every step
// is ONE contiguous 16-byte aligned blob  [32 u32 columns | popc(mask) x 32
// f32 values]  and a warp's steps are consecutive in memory. Each warp keeps
// D steps in flight: lane 0 issues one cp.async.bulk per step into a per-warp
// D-slot shared-memory ring (mbarrier transaction count per slot), the warp
// consumes slot i while slots i+1 .. i+D-1 land. The x of step i+G is
// gathered (two 16-byte cp.async per lane, padded lanes read column 0 times a
// zero value) into a per-warp (G+1)-slot x ring while step i is consumed. Step records (blob offset, row,
// info) are read 32 at a time, one per lane, and broadcast with shuffles.
//
// Row ends / range ends: transposed-butterfly reduction of the 24 sums
// (v12_reduce24) and red.global.add.f64 into the zeroed v_k.
#include "sss_common.cuh"

namespace sss {

constexpr int kV13Threads = 128;
constexpr int kV13SlotBytes = 128 + 8 * 128;

__device__ __forceinline__ uint4 v13_shfl_rec(const uint4& r, int src) {
  uint4 o;
  o.x = __shfl_sync(0xffffffffu, r.x, src);
  o.y = __shfl_sync(0xffffffffu, r.y, src);
  o.z = __shfl_sync(0xffffffffu, r.z, src);
  o.w = 0u;
  return o;
}

__device__ __forceinline__ void v13_cp16(void* s, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(s)), "l"(g) : "memory");
}
__device__ __forceinline__ void v13_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void v13_wait_group() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// per-warp shared memory: D blob slots, G+1 x slots (32 lanes x 32 B), D mbarriers
template <int D, int G>
struct V13Smem {
  static constexpr size_t ring = (size_t)D * kV13SlotBytes;
  static constexpr size_t xr = (size_t)(G + 1) * 32 * 32;
  static constexpr size_t per_warp = ring + xr + D * 8;
};

template <int D, int G>
__global__ void __launch_bounds__(kV13Threads) k_transfer_kstream(
    int K, int N, const uint8_t* __restrict__ blob, const uint4* __restrict__ recs,
    const unsigned* __restrict__ warp_begin, const double4* __restrict__ xp,
    double* __restrict__ vk) {
  static_assert(D >= 2 && D <= 16 && G >= 1 && G < D, "ring depth");
  using SM = V13Smem<D, G>;
  extern __shared__ __align__(128) uint8_t v13_smem[];
  constexpr int WARPS = kV13Threads / 32;
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  uint8_t* ring = v13_smem + (size_t)wl * SM::per_warp;
  double* xring = reinterpret_cast<double*>(ring + SM::ring);
  uint64_t* bars = reinterpret_cast<uint64_t*>(ring + SM::ring + SM::xr);
  const int w = blockIdx.x * WARPS + wl;
  const unsigned s0 = warp_begin[w], s1 = warp_begin[w + 1];
  if (s0 >= s1) return;
  const unsigned ns = s1 - s0;
  if (lane == 0) {
#pragma unroll
    for (int d = 0; d < D; ++d) mbar_init(&bars[d], 1);
    fence_mbar_init();
  }
  __syncwarp();

  // record batches: rA holds local steps [base, base + 32), rB the next 32
  unsigned base = 0;
  uint4 rA = make_uint4(0u, 0u, 0u, 0u), rB = rA;
  if (lane < ns) rA = __ldg(&recs[s0 + lane]);
  if (lane + 32 < ns) rB = __ldg(&recs[s0 + 32 + lane]);
  auto rec_of = [&](unsigned i) {  // warp-uniform i in [base, base + 64)
    return (i < base + 32) ? v13_shfl_rec(rA, (int)(i - base)) : v13_shfl_rec(rB, (int)(i - base - 32));
  };
  auto issue = [&](unsigned i, const uint4& r) {  // lane 0
    const unsigned bytes = (1u + __popc(r.z & 0xffu)) * 128u;
    uint64_t* bar = &bars[i % D];
    mbar_expect_tx(bar, bytes);
    bulk_g2s(ring + (size_t)(i % D) * kV13SlotBytes, blob + (size_t)r.x * 16u, bytes, bar);
  };
  // x of step j -> x slot j % (G+1): wait for the blob, one 32-byte gather per
  // lane as two 16-byte cp.async (padded lanes carry column 0, value 0)
  auto gather = [&](unsigned j) {
    if (j < ns) {
#ifdef SSS_V13_HINT
      mbar_wait_warp(&bars[j % D], (j / D) & 1u);
#else
      mbar_wait_warp_spin(&bars[j % D], (j / D) & 1u);
#endif
      const uint32_t c = reinterpret_cast<const uint32_t*>(ring + (size_t)(j % D) * kV13SlotBytes)[lane];
      double* dst = xring + ((size_t)(j % (G + 1)) * 32 + lane) * 4;
      const double* src = reinterpret_cast<const double*>(xp + c);
      v13_cp16(dst, src);
      v13_cp16(dst + 2, src + 2);
    }
    v13_commit();
  };

  // prologue: D blobs in flight, x of steps 0 .. G-1 in flight
#pragma unroll 1
  for (unsigned i = 0; i < (unsigned)D && i < ns; ++i) {
    const uint4 r = rec_of(i);
    if (lane == 0) issue(i, r);
  }
#pragma unroll 1
  for (unsigned j = 0; j < (unsigned)G; ++j) gather(j);

  double acc[24];
#pragma unroll
  for (int t = 0; t < 24; ++t) acc[t] = 0.0;

#pragma unroll 1
  for (unsigned i = 0; i < ns; ++i) {
    const uint4 rc = rec_of(i);
    gather(i + G);
    v13_wait_group<G>();  // this lane's x of step i
    {
      const double* xs = xring + ((size_t)(i % (G + 1)) * 32 + lane) * 4;
      const double2 xa = *reinterpret_cast<const double2*>(xs);
      const double xc2 = xs[2];
      const float* sv = reinterpret_cast<const float*>(ring + (size_t)(i % D) * kV13SlotBytes + 128);
      const unsigned mask = rc.z & 0xffu;
      unsigned j = 0;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if ((mask >> k) & 1u) {
          const double dv = (double)sv[j * 32 + lane];
          ++j;
          acc[3 * k + 0] = fma(dv, xa.x, acc[3 * k + 0]);
          acc[3 * k + 1] = fma(dv, xa.y, acc[3 * k + 1]);
          acc[3 * k + 2] = fma(dv, xc2, acc[3 * k + 2]);
        }
      }
    }
    if (((rc.z >> 16) & 1u) || i + 1 == ns) {
      double r[3];
      v12_reduce24(acc, lane, r);
      if ((lane & 3) == 0) {
        const int g = lane >> 2;
#pragma unroll
        for (int t = 0; t < 3; ++t) {
          const int f = 3 * g + t;  // = 3 k + c
          if (f < 3 * K) atomicAdd(&vk[(size_t)f * N + rc.y], r[t]);
        }
      }
#pragma unroll
      for (int t = 0; t < 24; ++t) acc[t] = 0.0;
    }
    __syncwarp();
    // refill blob slot i % D with step i + D
    if (i + D < ns) {
      const uint4 r = rec_of(i + D);
      if (lane == 0) {
        fence_proxy_async();
        issue(i + D, r);
      }
    }
    if (i + 1 == base + 32) {  // rotate the record batches
      rA = rB;
      base += 32;
      rB = make_uint4(0u, 0u, 0u, 0u);
      if (base + 32 + lane < ns) rB = __ldg(&recs[s0 + base + 32 + lane]);
    }
  }
}

}  // namespace sss
