// Transfer v25 "flat16": flat8 with 16 entries per lane.
//
// In flat8 (v17) the segmented warp scan that closes every 256-entry warp
// iteration (5 shuffle steps x 3 fp64 channels = 30 SHFL) costs 8.5 M of the
// kernel's 45.8 M L1 data-pipe wavefronts at C3 (the x gathers are 28.8 M).
// Sixteen entries per lane (segments padded to a multiple of 16 and
// lane-interleaved the same way) halve the iterations, so the scans, the head
// / prefix loads and the loop overhead halve, for ~3 % more padding entries.
// Gathers run in quarters of four entries (12 live fp64 x registers).
#include "sss_common.cuh"

namespace sss {

constexpr int kV25Threads = 128;

template <bool COL16>
struct V25Slot {
  unsigned long long c[COL16 ? 4 : 8];  // 16 u16 or u32 columns
  unsigned long long v[8];              // 16 f32 values
  uint32_t h, hp;
};

// group q = i * 32 + lane of G = E / 16 sub-slots; sub-slot j of the group is
// the 16 entries at (q * G + j) * 16
template <bool COL16>
__device__ __forceinline__ void v25_load(V25Slot<COL16>& S, size_t q, unsigned ngroups, int G,
                                         int j, const unsigned long long* __restrict__ C16,
                                         const unsigned long long* __restrict__ V16) {
  constexpr int NC = COL16 ? 4 : 8;
  if (q >= ngroups) {  // past the stream's last group (partial last word)
#pragma unroll
    for (int t = 0; t < NC; ++t) S.c[t] = 0ull;
#pragma unroll
    for (int t = 0; t < 8; ++t) S.v[t] = 0ull;
    return;
  }
  q = q * G + j;
#pragma unroll
  for (int h = 0; h < NC / 4; ++h)
    asm volatile("ld.global.nc.L1::no_allocate.v4.u64 {%0,%1,%2,%3}, [%4];"
                 : "=l"(S.c[4 * h]), "=l"(S.c[4 * h + 1]), "=l"(S.c[4 * h + 2]), "=l"(S.c[4 * h + 3])
                 : "l"(C16 + NC * q + 4 * h));
#pragma unroll
  for (int h = 0; h < 2; ++h)
    asm volatile("ld.global.nc.L1::no_allocate.v4.u64 {%0,%1,%2,%3}, [%4];"
                 : "=l"(S.v[4 * h]), "=l"(S.v[4 * h + 1]), "=l"(S.v[4 * h + 2]), "=l"(S.v[4 * h + 3])
                 : "l"(V16 + 8 * q + 4 * h));
}

template <bool COL16>
__device__ __forceinline__ uint32_t v25_col(const V25Slot<COL16>& S, int e) {
  if (COL16) return (uint32_t)(S.c[e >> 2] >> (16 * (e & 3))) & 0xffffu;
  return (uint32_t)(S.c[e >> 1] >> (32 * (e & 1)));
}
template <bool COL16>
__device__ __forceinline__ float v25_val(const V25Slot<COL16>& S, int e) {
  return __uint_as_float((uint32_t)(S.v[e >> 1] >> (32 * (e & 1))));
}

// COL16: 16-bit columns (n <= 65536; 6 bytes per entry instead of 8);
// padding entries then keep column 0 with value 0
template <int MINB, int E = 16, bool COL16 = false>
__global__ void __launch_bounds__(kV25Threads, MINB) k_transfer_flat16(
    int N, unsigned ngroups, const unsigned long long* __restrict__ C16,
    const unsigned long long* __restrict__ V16,
    const uint32_t* __restrict__ H, const uint32_t* __restrict__ hpre,
    const uint32_t* __restrict__ rowk, const unsigned* __restrict__ warp_begin,
    const double4* __restrict__ xp, const uint32_t* __restrict__ bits, double* __restrict__ vk,
    unsigned* __restrict__ work = nullptr, int chunk = 4, double* __restrict__ part = nullptr) {
  constexpr int G = E / 16;
  extern __shared__ uint32_t v25_bits[];
  // one word past the N columns: padding entries carry column N, never kept
  for (int t = threadIdx.x; t <= (N >> 5); t += blockDim.x) v25_bits[t] = bits[t];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const unsigned upto = (2u << lane) - 1u;
  const unsigned nwords_all = warp_begin[(gridDim.x * blockDim.x) >> 5];
  auto word = [&](unsigned i) {
    V25Slot<COL16> S;
    S.h = __ldg(&H[i]);
    S.hp = __ldg(&hpre[i]);
    double p0 = 0.0, p1 = 0.0, p2 = 0.0;
#pragma unroll 1
    for (int j = 0; j < G; ++j) {
      v25_load<COL16>(S, (size_t)i * 32u + (unsigned)lane, ngroups, G, j, C16, V16);
#pragma unroll
      for (int qd = 0; qd < 4; ++qd) {
        double x[4][3];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const uint32_t c = v25_col<COL16>(S, qd * 4 + e);
          x[e][0] = x[e][1] = x[e][2] = 0.0;
          // padding entries (value 0, column 0 with u16 columns) may gather
          // x[0]: all such lanes of an instruction share that one address
          if ((v25_bits[c >> 5] >> (c & 31u)) & 1u) v15_gather1(xp, c, x[e]);
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const double v = (double)v25_val<COL16>(S, qd * 4 + e);
          p0 = fma(v, x[e][0], p0);
          p1 = fma(v, x[e][1], p1);
          p2 = fma(v, x[e][2], p2);
        }
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
    if (part) {
      // Deterministic sums: a (row, term) segment that starts and ends inside
      // this word is stored directly (v_k is zeroed, nobody else writes it);
      // a segment continuing the previous word's row (no head at or before
      // the lane) leaves its sum in the word's slot 0, one running into the
      // next word (lane 31, next word's lane 0 is no head) in slot 1, and
      // k_flat16_merge adds the pieces of every spanning row in word order
      const bool cont = hm == 0u;
      const bool open = lane == 31 && i + 1u < nwords_all && !(__ldg(&H[i + 1u]) & 1u);
      if (tail && (cont || open)) {
        double* q = part + ((size_t)i * 2 + (cont ? 0 : 1)) * 3;
        q[0] = p0; q[1] = p1; q[2] = p2;
      } else if (tail && (p0 != 0.0 || p1 != 0.0 || p2 != 0.0)) {
        const unsigned rk = __ldg(&rowk[S.hp + __popc(hm) - 1u]);
        double* vo = vk + (size_t)(rk & 15u) * 3 * N + (rk >> 4);
        vo[0] = p0;
        vo[N] = p1;
        vo[2 * (size_t)N] = p2;
      }
    } else if (tail && (p0 != 0.0 || p1 != 0.0 || p2 != 0.0)) {
      const unsigned rk = __ldg(&rowk[S.hp + __popc(hm) - 1u]);
      double* vo = vk + (size_t)(rk & 15u) * 3 * N + (rk >> 4);
      atomicAdd(vo, p0);
      atomicAdd(vo + N, p1);
      atomicAdd(vo + 2 * (size_t)N, p2);
    }
  };
  if (!work) {  // static equal word ranges
    const unsigned i0 = warp_begin[w], i1 = warp_begin[w + 1];
#pragma unroll 1
    for (unsigned i = i0; i < i1; ++i) word(i);
    return;
  }
  // dynamic: warps claim chunks of words from a zeroed counter (the equal
  // static ranges differ in gather count: SM busy times spread by +-10 %)
  const unsigned nwords = nwords_all;
#pragma unroll 1
  for (;;) {
    unsigned c = 0;
    if (lane == 0) c = atomicAdd(work, 1u);
    c = __shfl_sync(0xffffffffu, c, 0);
    const unsigned i0 = c * (unsigned)chunk;
    if (i0 >= nwords) break;
    const unsigned i1 = min(i0 + (unsigned)chunk, nwords);
#pragma unroll 1
    for (unsigned i = i0; i < i1; ++i) word(i);
  }
}

// The second pass of the deterministic form: one thread per word that CLOSES a
// row spanning several words (it continues the previous word, and the row ends
// in it: a head further on, or the next word starts fresh, or the stream ends). The row's pieces are the open last segment
// of the word it began in (slot 1), the whole of every headless word in
// between (slot 0) and this word's leading segment (slot 0), added in word
// order - a fixed order, so v_k is bitwise reproducible.
__global__ void k_flat16_merge(int N, unsigned nwords, const uint32_t* __restrict__ H,
                               const uint32_t* __restrict__ hpre,
                               const uint32_t* __restrict__ rowk,
                               const uint32_t* __restrict__ span_first,
                               const double* __restrict__ part, double* __restrict__ vk) {
  pdl_launch_dependents();
  pdl_wait();
  const unsigned b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b == 0u || b >= nwords) return;
  // every independent load first (the kernel is a chain of L2 round trips)
  const uint32_t h = __ldg(&H[b]);
  const uint32_t hn = b + 1u < nwords ? __ldg(&H[b + 1u]) : 1u;
  const unsigned a = __ldg(&span_first[b]);  // the word the row began in (layout.flat16_layout)
  const unsigned seg = __ldg(&hpre[b]) - 1u;
  const double* qb = part + (size_t)b * 2 * 3;
  const double b0 = qb[0], b1 = qb[1], b2 = qb[2];
  if (h & 1u) return;  // starts fresh: nothing continues into this word
  // a headless word whose row also runs into the next word is a through word
  if (h == 0u && !(hn & 1u)) return;
  const unsigned rk = __ldg(&rowk[seg]);
  const double* q = part + ((size_t)a * 2 + 1) * 3;
  double s0 = q[0], s1 = q[1], s2 = q[2];
  for (unsigned w0 = a + 1u; w0 < b; w0 += 4u) {  // the through words, four loads in flight, adds in order
    double t[4][3];
#pragma unroll
    for (unsigned u = 0; u < 4u; ++u) {
      const bool in = w0 + u < b;
      q = part + (size_t)(in ? w0 + u : b) * 2 * 3;
      t[u][0] = in ? q[0] : 0.0; t[u][1] = in ? q[1] : 0.0; t[u][2] = in ? q[2] : 0.0;
    }
#pragma unroll
    for (unsigned u = 0; u < 4u; ++u)
      if (w0 + u < b) { s0 += t[u][0]; s1 += t[u][1]; s2 += t[u][2]; }
  }
  s0 += b0; s1 += b1; s2 += b2;
  double* vo = vk + (size_t)(rk & 15u) * 3 * N + (rk >> 4);
  vo[0] = s0;
  vo[N] = s1;
  vo[2 * (size_t)N] = s2;
}

}  // namespace sss
