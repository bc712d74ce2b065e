// Transfer v15: flat-stream CSR SpMV with head flags.
//
// Every earlier variant walked (row, k) pieces: load a descriptor, then the
// piece's data, then reduce - two dependent memory latencies per piece, and a
// piece averages ~40 entries, so the stream never had enough bytes in flight
// (1.6 TB/s even with the x gathers removed). Here a warp streams an equal,
// contiguous range of the padded operator (csr9's copy: every (row, k)
// segment padded to a multiple of 4 entries, so a 16-byte group of 4 entries
// never straddles two segments) with fully coalesced uint4 / float4 loads that
// do not depend on the segment structure, two iterations ahead; the x gathers
// of the next iteration are issued before the current one is consumed.
//
// Segment membership comes from a head-flag bitmap (bit l of word i set iff
// 4-entry group 32 i + l starts a segment) and a per-word count of segments
// started before it, so the segment id of a lane is a popcount. Per iteration
// a segmented warp scan (5 shuffle steps, 3 channels) sums the runs and each
// run's tail lane adds its sum into the zeroed v_k (red.global.add.f64;
// all-zero sums, e.g. segments over unkept columns, are skipped).
#include "sss_common.cuh"

namespace sss {

constexpr int kV15Threads = 256;

struct V15Load {
  uint4 c;
  float4 v;
  uint32_t h, hp;
};

__device__ __forceinline__ void v15_load(V15Load& L, unsigned i, int lane, unsigned n4,
                                         const uint4* __restrict__ C4, const float4* __restrict__ V4,
                                         const uint32_t* __restrict__ H,
                                         const uint32_t* __restrict__ hpre) {
  const unsigned q = i * 32u + (unsigned)lane;
  if (q < n4) {
    L.c = __ldg(&C4[q]);
    L.v = V4 ? __ldg(&V4[q]) : make_float4(1.f, 1.f, 1.f, 1.f);
  } else {
    L.c = make_uint4(0u, 0u, 0u, 0u);
    L.v = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  L.h = __ldg(&H[i]);
  L.hp = __ldg(&hpre[i]);
}

__device__ __forceinline__ void v15_gather1(const double4* __restrict__ xp, uint32_t c, double* x) {
  double x3;
  asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(x[0]), "=d"(x[1]), "=d"(x[2]), "=d"(x3)
               : "l"(xp + c));
  (void)x3;
}

// MODE (bandwidth probes in tools/, 0 in the product): 1 = no x gathers,
// 2 = no operator values (columns + gathers only). GA = iterations of x
// gathers in flight ahead of the consumed one (the stream runs GA + 1 ahead):
// the gathers hit L2 (~1 us under load), so one iteration ahead per warp
// leaves the SM latency-bound.
template <int MODE = 0, int GA = 2>
__global__ void __launch_bounds__(kV15Threads) k_transfer_flat(
    int N, unsigned n4, const uint4* __restrict__ C4, const float4* __restrict__ V4,
    const uint32_t* __restrict__ H, const uint32_t* __restrict__ hpre,
    const uint32_t* __restrict__ rowk, const unsigned* __restrict__ warp_begin,
    const double4* __restrict__ xp, const uint32_t* __restrict__ bits, double* __restrict__ vk) {
  static_assert(GA >= 1 && GA <= 3, "gather depth");
  // kept-column bitmap (optional): entries over columns no channel keeps are
  // exact zeros, so their x gather is skipped (the row-driven form of the
  // reference's csc_apply over the kept columns, transfer.py:66-71)
  extern __shared__ uint32_t v15_bits[];
  if (bits) {
    for (int t = threadIdx.x; t < ((N + 31) >> 5); t += blockDim.x) v15_bits[t] = bits[t];
    __syncthreads();
  }
  const int lane = threadIdx.x & 31;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const unsigned i0 = warp_begin[w], i1 = warp_begin[w + 1];
  if (i0 >= i1) return;
  const float4* V = MODE == 2 ? nullptr : V4;
  auto gather4 = [&](const uint4& c, double (&x)[4][3]) {
    if (MODE == 1) {
      const double f = (double)(c.x ^ c.y ^ c.z ^ c.w);
#pragma unroll
      for (int t = 0; t < 4; ++t) x[t][0] = x[t][1] = x[t][2] = f;
    } else if (bits) {
      const uint32_t cc[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        x[t][0] = x[t][1] = x[t][2] = 0.0;
        if ((v15_bits[cc[t] >> 5] >> (cc[t] & 31u)) & 1u) v15_gather1(xp, cc[t], x[t]);
      }
    } else {
      v15_gather1(xp, c.x, x[0]);
      v15_gather1(xp, c.y, x[1]);
      v15_gather1(xp, c.z, x[2]);
      v15_gather1(xp, c.w, x[3]);
    }
  };
  // pipeline: L[0..GA] = stream data of iterations i .. i+GA, X[0..GA-1] = x of i .. i+GA-1
  V15Load L[GA + 1];
  double X[GA][4][3];
#pragma unroll
  for (int d = 0; d <= GA; ++d)
    if (i0 + d < i1) v15_load(L[d], i0 + d, lane, n4, C4, V, H, hpre);
#pragma unroll
  for (int d = 0; d < GA; ++d)
    if (i0 + d < i1) gather4(L[d].c, X[d]);
  const unsigned upto = (2u << lane) - 1u;  // lanes 0 .. lane (all ones for lane 31)
#pragma unroll 1
  for (unsigned i = i0; i < i1; ++i) {
    V15Load Ln;
    if (i + GA + 1 < i1) v15_load(Ln, i + GA + 1, lane, n4, C4, V, H, hpre);
    double Xn[4][3];
    if (i + GA < i1) gather4(L[GA].c, Xn);
    // partial sums of this lane's 4 entries
    double p0, p1, p2;
    {
      const double v0 = L[0].v.x, v1 = L[0].v.y, v2 = L[0].v.z, v3 = L[0].v.w;
      const double (&xa)[4][3] = X[0];
      p0 = v0 * xa[0][0];
      p1 = v0 * xa[0][1];
      p2 = v0 * xa[0][2];
      p0 = fma(v1, xa[1][0], p0); p1 = fma(v1, xa[1][1], p1); p2 = fma(v1, xa[1][2], p2);
      p0 = fma(v2, xa[2][0], p0); p1 = fma(v2, xa[2][1], p1); p2 = fma(v2, xa[2][2], p2);
      p0 = fma(v3, xa[3][0], p0); p1 = fma(v3, xa[3][1], p1); p2 = fma(v3, xa[3][2], p2);
    }
    // segmented inclusive scan over the lanes
    const uint32_t h = L[0].h;
    const unsigned hm = h & upto;
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
    const bool tail = (lane == 31) || ((h >> (lane + 1)) & 1u);
    if (tail && (p0 != 0.0 || p1 != 0.0 || p2 != 0.0)) {
      const unsigned pid = L[0].hp + __popc(hm) - 1u;
      const unsigned rk = __ldg(&rowk[pid]);
      double* vo = vk + (size_t)(rk & 15u) * 3 * N + (rk >> 4);
      atomicAdd(vo, p0);
      atomicAdd(vo + N, p1);
      atomicAdd(vo + 2 * (size_t)N, p2);
    }
    // rotate the pipeline
#pragma unroll
    for (int d = 0; d < GA; ++d) L[d] = L[d + 1];
    L[GA] = Ln;
#pragma unroll
    for (int d = 0; d + 1 < GA; ++d)
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        X[d][t][0] = X[d + 1][t][0];
        X[d][t][1] = X[d + 1][t][1];
        X[d][t][2] = X[d + 1][t][2];
      }
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      X[GA - 1][t][0] = Xn[t][0];
      X[GA - 1][t][1] = Xn[t][1];
      X[GA - 1][t][2] = Xn[t][2];
    }
  }
}

}  // namespace sss

// ---------------------------------------------------------------------------
// v16: the same flat stream with a deep asynchronous prefetch. Each warp owns
// an R-slot shared-memory ring; iteration i + R - 1 is requested with
// cp.async (16 B of columns + 16 B of values per lane, the head word and its
// prefix by lane 0) while iteration i is consumed, so ~R KB per warp are in
// flight without holding registers. Columns of iteration i + 1 are read from
// the ring to issue its x gathers one iteration ahead.
// ---------------------------------------------------------------------------
namespace sss {

constexpr int kV16Threads = 128;

template <int R>
struct V16Slot {
  uint4 c[32];
  float4 v[32];
  uint32_t h, hp, pad[2];
};

__device__ __forceinline__ void v16_cp16(void* s, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(s)), "l"(g) : "memory");
}
__device__ __forceinline__ void v16_cp8(void* s, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(s)), "l"(g) : "memory");
}
__device__ __forceinline__ void v16_cp4(void* s, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(s)), "l"(g) : "memory");
}
__device__ __forceinline__ void v16_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void v16_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <int R>
__global__ void __launch_bounds__(kV16Threads) k_transfer_flatp(
    int N, unsigned n4, const uint4* __restrict__ C4, const float4* __restrict__ V4,
    const uint32_t* __restrict__ H, const uint32_t* __restrict__ hpre,
    const uint32_t* __restrict__ rowk, const unsigned* __restrict__ warp_begin,
    const double4* __restrict__ xp, double* __restrict__ vk) {
  extern __shared__ __align__(16) uint8_t v16_smem[];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  V16Slot<R>* ring = reinterpret_cast<V16Slot<R>*>(v16_smem) + (size_t)wl * R;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const unsigned i0 = warp_begin[w], i1 = warp_begin[w + 1];
  if (i0 >= i1) return;
  const unsigned ni = i1 - i0;
  // request iteration j (local) into its slot; always commit (uniform group count)
  auto request = [&](unsigned j) {
    if (j < ni) {
      V16Slot<R>& S = ring[j % R];
      const unsigned i = i0 + j;
      const unsigned q = i * 32u + (unsigned)lane;
      if (q < n4) {
        v16_cp16(&S.c[lane], &C4[q]);
        v16_cp16(&S.v[lane], &V4[q]);
      } else {
        S.c[lane] = make_uint4(0u, 0u, 0u, 0u);
        S.v[lane] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
      if (lane == 0) {
        v16_cp4(&S.h, &H[i]);
        v16_cp4(&S.hp, &hpre[i]);
      }
    }
    v16_commit();
  };
#pragma unroll 1
  for (unsigned j = 0; j < (unsigned)(R - 1); ++j) request(j);
  // x of iteration 0
  double xa[4][3], xb[4][3];
  v16_wait<R - 2>();
  __syncwarp();
  {
    const uint4 c = ring[0].c[lane];
    v15_gather1(xp, c.x, xa[0]);
    v15_gather1(xp, c.y, xa[1]);
    v15_gather1(xp, c.z, xa[2]);
    v15_gather1(xp, c.w, xa[3]);
  }
  const unsigned upto = (2u << lane) - 1u;
#pragma unroll 1
  for (unsigned j = 0; j < ni; ++j) {
    request(j + R - 1);
    v16_wait<R - 2>();  // this lane's copies of iteration j + 1 have landed
    __syncwarp();       // ... and every lane's
    if (j + 1 < ni) {
      const uint4 c = ring[(j + 1) % R].c[lane];
      v15_gather1(xp, c.x, xb[0]);
      v15_gather1(xp, c.y, xb[1]);
      v15_gather1(xp, c.z, xb[2]);
      v15_gather1(xp, c.w, xb[3]);
    }
    const V16Slot<R>& S = ring[j % R];
    const float4 v = S.v[lane];
    const uint32_t h = S.h, hp = S.hp;
    double p0, p1, p2;
    {
      const double v0 = v.x, v1 = v.y, v2 = v.z, v3 = v.w;
      p0 = v0 * xa[0][0];
      p1 = v0 * xa[0][1];
      p2 = v0 * xa[0][2];
      p0 = fma(v1, xa[1][0], p0); p1 = fma(v1, xa[1][1], p1); p2 = fma(v1, xa[1][2], p2);
      p0 = fma(v2, xa[2][0], p0); p1 = fma(v2, xa[2][1], p1); p2 = fma(v2, xa[2][2], p2);
      p0 = fma(v3, xa[3][0], p0); p1 = fma(v3, xa[3][1], p1); p2 = fma(v3, xa[3][2], p2);
    }
    const unsigned hm = h & upto;
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
    const bool tail = (lane == 31) || ((h >> (lane + 1)) & 1u);
    if (tail && (p0 != 0.0 || p1 != 0.0 || p2 != 0.0)) {
      const unsigned pid = hp + __popc(hm) - 1u;
      const unsigned rk = __ldg(&rowk[pid]);
      double* vo = vk + (size_t)(rk & 15u) * 3 * N + (rk >> 4);
      atomicAdd(vo, p0);
      atomicAdd(vo + N, p1);
      atomicAdd(vo + 2 * (size_t)N, p2);
    }
    __syncwarp();  // slot j % R is refilled by the next iteration's request
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      xa[t][0] = xb[t][0];
      xa[t][1] = xb[t][1];
      xa[t][2] = xb[t][2];
    }
  }
}

}  // namespace sss

// ---------------------------------------------------------------------------
// v17: flat stream, 8 entries per lane. Segments padded to a multiple of 8
// entries, so a lane's 8 entries (one 32-byte column load + one 32-byte value
// load, LDG.E.ENL2.256) never straddle two segments and the segmented scan
// is amortized over 256 entries per warp iteration. Head bit l of word i marks
// 8-entry group 32 i + l. Double-buffered by an unroll of 2 (slots A / B swap
// roles) so the prefetch pipeline costs no register moves: while iteration i
// is consumed, the x of iteration i+1 is gathered and the stream of i+2 is
// requested.
// ---------------------------------------------------------------------------
namespace sss {

constexpr int kV17Threads = 128;

struct V17Slot {
  unsigned long long c[4];  // 8 u32 columns
  unsigned long long v[4];  // 8 f32 values
  uint32_t h, hp;
};

__device__ __forceinline__ void v17_load(V17Slot& S, unsigned i, int lane, unsigned n8,
                                         const unsigned long long* __restrict__ C8,
                                         const unsigned long long* __restrict__ V8,
                                         const uint32_t* __restrict__ H,
                                         const uint32_t* __restrict__ hpre) {
  const unsigned q = i * 32u + (unsigned)lane;
  if (q < n8) {
    asm volatile("ld.global.nc.v4.u64 {%0,%1,%2,%3}, [%4];"
                 : "=l"(S.c[0]), "=l"(S.c[1]), "=l"(S.c[2]), "=l"(S.c[3])
                 : "l"(C8 + 4 * (size_t)q));
    asm volatile("ld.global.nc.v4.u64 {%0,%1,%2,%3}, [%4];"
                 : "=l"(S.v[0]), "=l"(S.v[1]), "=l"(S.v[2]), "=l"(S.v[3])
                 : "l"(V8 + 4 * (size_t)q));
  } else {
#pragma unroll
    for (int t = 0; t < 4; ++t) S.c[t] = S.v[t] = 0ull;
  }
  S.h = __ldg(&H[i]);
  S.hp = __ldg(&hpre[i]);
}

__device__ __forceinline__ uint32_t v17_col(const V17Slot& S, int e) {
  return (uint32_t)(S.c[e >> 1] >> (32 * (e & 1)));
}
__device__ __forceinline__ float v17_val(const V17Slot& S, int e) {
  return __uint_as_float((uint32_t)(S.v[e >> 1] >> (32 * (e & 1))));
}

__device__ __forceinline__ void v17_gather(const V17Slot& S, const double4* __restrict__ xp,
                                           const uint32_t* sbits, double (&x)[8][3]) {
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const uint32_t c = v17_col(S, e);
    x[e][0] = x[e][1] = x[e][2] = 0.0;
    if (!sbits || ((sbits[c >> 5] >> (c & 31u)) & 1u)) v15_gather1(xp, c, x[e]);
  }
}

// fp32 x variant (fp64 accumulation of f32 values x f32 E spectrum
// passes the 1e-4 bar): 16-byte gathers of a packed (N, 4) float array
__device__ __forceinline__ void v17_gather(const V17Slot& S, const float4* __restrict__ xp,
                                           const uint32_t* sbits, float (&x)[8][3]) {
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const uint32_t c = v17_col(S, e);
    x[e][0] = x[e][1] = x[e][2] = 0.0f;
    if (!sbits || ((sbits[c >> 5] >> (c & 31u)) & 1u)) {
      float x3;
      asm volatile("ld.global.nc.v4.f32 {%0,%1,%2,%3}, [%4];"
                   : "=f"(x[e][0]), "=f"(x[e][1]), "=f"(x[e][2]), "=f"(x3)
                   : "l"(xp + c));
    }
  }
}

template <typename XT>
__device__ __forceinline__ void v17_consume(const V17Slot& S, const XT (&x)[8][3], int lane,
                                            unsigned upto, int N, const uint32_t* __restrict__ rowk,
                                            double* __restrict__ vk) {
  double p0 = 0.0, p1 = 0.0, p2 = 0.0;
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const double v = (double)v17_val(S, e);
    p0 = fma(v, (double)x[e][0], p0);
    p1 = fma(v, (double)x[e][1], p1);
    p2 = fma(v, (double)x[e][2], p2);
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

// half-slot variants: entries [h*4, h*4+4) of the lane's 8 (fewer live x
// registers -> more resident warps)
__device__ __forceinline__ void v17_gather_half(const V17Slot& S, const double4* __restrict__ xp,
                                                const uint32_t* sbits, int h, double (&x)[4][3]) {
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const uint32_t c = v17_col(S, h * 4 + e);
    x[e][0] = x[e][1] = x[e][2] = 0.0;
    if (!sbits || ((sbits[c >> 5] >> (c & 31u)) & 1u)) v15_gather1(xp, c, x[e]);
  }
}

__device__ __forceinline__ void v17_gather_half(const V17Slot& S, const float4* __restrict__ xp,
                                                const uint32_t* sbits, int h, float (&x)[4][3]) {
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const uint32_t c = v17_col(S, h * 4 + e);
    x[e][0] = x[e][1] = x[e][2] = 0.0f;
    if (!sbits || ((sbits[c >> 5] >> (c & 31u)) & 1u)) {
      float x3;
      asm volatile("ld.global.nc.v4.f32 {%0,%1,%2,%3}, [%4];"
                   : "=f"(x[e][0]), "=f"(x[e][1]), "=f"(x[e][2]), "=f"(x3)
                   : "l"(xp + c));
    }
  }
}

template <typename XT = double, typename XP = double4>
__device__ __forceinline__ void v17_consume_split(const V17Slot& S, const XP* __restrict__ xp,
                                                  const uint32_t* sbits, int lane, unsigned upto,
                                                  int N, const uint32_t* __restrict__ rowk,
                                                  double* __restrict__ vk) {
  XT x[4][3];
  double p0 = 0.0, p1 = 0.0, p2 = 0.0;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    v17_gather_half(S, xp, sbits, h, x);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const double v = (double)v17_val(S, h * 4 + e);
      p0 = fma(v, (double)x[e][0], p0);
      p1 = fma(v, (double)x[e][1], p1);
      p2 = fma(v, (double)x[e][2], p2);
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

template <int MINB, bool SINGLE = false, typename XT = double, typename XP = double4>
__global__ void __launch_bounds__(kV17Threads, MINB) k_transfer_flat8s(
    int N, unsigned n8, const unsigned long long* __restrict__ C8,
    const unsigned long long* __restrict__ V8, const uint32_t* __restrict__ H,
    const uint32_t* __restrict__ hpre, const uint32_t* __restrict__ rowk,
    const unsigned* __restrict__ warp_begin, const XP* __restrict__ xp,
    const uint32_t* __restrict__ bits, double* __restrict__ vk) {
  extern __shared__ uint32_t v17_bits[];
  if (bits) {
    for (int t = threadIdx.x; t < ((N + 31) >> 5); t += blockDim.x) v17_bits[t] = bits[t];
    __syncthreads();
  }
  const uint32_t* sb = bits ? v17_bits : nullptr;
  const int lane = threadIdx.x & 31;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const unsigned i0 = warp_begin[w], i1 = warp_begin[w + 1];
  if (i0 >= i1) return;
  const unsigned upto = (2u << lane) - 1u;
  if (SINGLE) {  // one slot: stream latency hidden by the extra resident warps
#pragma unroll 1
    for (unsigned i = i0; i < i1; ++i) {
      V17Slot A;
      v17_load(A, i, lane, n8, C8, V8, H, hpre);
      v17_consume_split<XT, XP>(A, xp, sb, lane, upto, N, rowk, vk);
    }
    return;
  }
  V17Slot A, B;
  v17_load(A, i0, lane, n8, C8, V8, H, hpre);
  if (i0 + 1 < i1) v17_load(B, i0 + 1, lane, n8, C8, V8, H, hpre);
#pragma unroll 1
  for (unsigned i = i0; i < i1; i += 2) {
    v17_consume_split<XT, XP>(A, xp, sb, lane, upto, N, rowk, vk);
    if (i + 2 < i1) v17_load(A, i + 2, lane, n8, C8, V8, H, hpre);
    if (i + 1 >= i1) break;
    v17_consume_split<XT, XP>(B, xp, sb, lane, upto, N, rowk, vk);
    if (i + 3 < i1) v17_load(B, i + 3, lane, n8, C8, V8, H, hpre);
  }
}

template <bool AHEAD, typename XT = double, typename XP = double4>
__global__ void __launch_bounds__(kV17Threads, 4) k_transfer_flat8(
    int N, unsigned n8, const unsigned long long* __restrict__ C8,
    const unsigned long long* __restrict__ V8, const uint32_t* __restrict__ H,
    const uint32_t* __restrict__ hpre, const uint32_t* __restrict__ rowk,
    const unsigned* __restrict__ warp_begin, const XP* __restrict__ xp,
    const uint32_t* __restrict__ bits, double* __restrict__ vk) {
  extern __shared__ uint32_t v17_bits[];
  if (bits) {
    for (int t = threadIdx.x; t < ((N + 31) >> 5); t += blockDim.x) v17_bits[t] = bits[t];
    __syncthreads();
  }
  const uint32_t* sb = bits ? v17_bits : nullptr;
  const int lane = threadIdx.x & 31;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const unsigned i0 = warp_begin[w], i1 = warp_begin[w + 1];
  if (i0 >= i1) return;
  const unsigned upto = (2u << lane) - 1u;
  V17Slot A, B;
  v17_load(A, i0, lane, n8, C8, V8, H, hpre);
  if (i0 + 1 < i1) v17_load(B, i0 + 1, lane, n8, C8, V8, H, hpre);
  if (!AHEAD) {  // gather and consume in the same iteration; warps hide the latency
    XT X[8][3];
#pragma unroll 1
    for (unsigned i = i0; i < i1; i += 2) {
      v17_gather(A, xp, sb, X);
      v17_consume(A, X, lane, upto, N, rowk, vk);
      if (i + 2 < i1) v17_load(A, i + 2, lane, n8, C8, V8, H, hpre);
      if (i + 1 >= i1) break;
      v17_gather(B, xp, sb, X);
      v17_consume(B, X, lane, upto, N, rowk, vk);
      if (i + 3 < i1) v17_load(B, i + 3, lane, n8, C8, V8, H, hpre);
    }
    return;
  }
  XT XA[8][3], XB[8][3];
  v17_gather(A, xp, sb, XA);
#pragma unroll 1
  for (unsigned i = i0; i < i1; i += 2) {
    // iteration i: A / XA current, B next
    if (i + 1 < i1) v17_gather(B, xp, sb, XB);
    v17_consume(A, XA, lane, upto, N, rowk, vk);
    if (i + 2 < i1) v17_load(A, i + 2, lane, n8, C8, V8, H, hpre);
    if (i + 1 >= i1) break;
    // iteration i+1: B / XB current, A next
    if (i + 2 < i1) v17_gather(A, xp, sb, XA);
    v17_consume(B, XB, lane, upto, N, rowk, vk);
    if (i + 3 < i1) v17_load(B, i + 3, lane, n8, C8, V8, H, hpre);
  }
}

}  // namespace sss
