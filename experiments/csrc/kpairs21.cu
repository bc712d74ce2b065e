// Transfer v21 "kpairs": one x gather per (row, column) pair for all K terms.
//
// The flat8 stream gathers x once per stored coefficient: 28.8 M 32-byte
// gathers per C3 frame, one L1TEX wavefront each, which is what bounds it.
// A (row, column) pair carries on average 2.7 of the K = 8 terms (the same
// receiver/source pair survives the compression of several PCA terms), so
// gathering per pair cuts the gathers 2.7x. Layout (transfer.kpairs_layout):
//
//   hdr[p]   u32   column (low 16 bits, N <= 65536) | term mask << 16
//   vals[e]  f32   pair-major, terms ascending inside a pair: pair p's values
//                  are vals[vbase(p) .. vbase(p) + popc(mask))
//   chunk[q] uint4 {row, first pair, pair count (<= 32), vbase(first pair)}
//                  rows split into chunks of 32 pairs; every row has >= 1
//                  chunk (empty rows write zeros)
//   cbeg[w]        first chunk of warp w; warps own whole rows
//
// A warp walks its chunks with a two-deep software pipeline (descriptor and
// headers two chunks ahead, gathers and values one chunk ahead), lane j owns
// pair j of the chunk and keeps 8 x 3 fp64 accumulators. Unkept columns
// (kept bitmap in shared memory) skip both the gather and the value loads. At
// a row's last chunk the warp reduce-scatters the 24 accumulators (butterfly,
// 31 shuffles) so lane l < 3K holds term l / 3, channel l % 3, and writes
// v_k directly: no atomics, no memset, deterministic sums.
#include "sss_common.cuh"

namespace sss {

constexpr int kV21Threads = 256;

struct V21Stage {
  uint4 d;       // chunk descriptor
  uint32_t h;    // this lane's pair header (0 beyond the chunk)
};

struct V21Work {
  uint32_t row, last;
  uint32_t mask;     // term mask if the column is kept, else 0
  double x0, x1, x2;
  float v[8];
};

__device__ __forceinline__ void v21_fetch(V21Stage& S, uint32_t q, int lane,
                                          const uint4* __restrict__ chunks,
                                          const uint32_t* __restrict__ hdr) {
  S.d = __ldg(chunks + q);
  S.h = lane < (int)S.d.z ? __ldcs(hdr + S.d.y + lane) : 0u;
}

template <int K>
__device__ __forceinline__ void v21_issue(const V21Stage& S, int lane, uint32_t next_row,
                                          const uint32_t* sbits, const double4* __restrict__ xp,
                                          const float* __restrict__ vals, V21Work& W) {
  const uint32_t m = (S.h >> 16) & 0xffu;
  const uint32_t c = S.h & 0xffffu;
  // exclusive scan of the per-pair value counts -> this lane's value offset
  uint32_t cnt = __popc(m), inc = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  const uint32_t off = S.d.w + inc - cnt;
  const bool kept = m && ((sbits[c >> 5] >> (c & 31u)) & 1u);
  W.row = S.d.x;
  W.last = next_row != S.d.x;
  W.mask = kept ? m : 0u;
  W.x0 = W.x1 = W.x2 = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) W.v[k] = 0.0f;
  if (kept) {
    double x3;
    asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(W.x0), "=d"(W.x1), "=d"(W.x2), "=d"(x3)
                 : "l"(xp + c));
    (void)x3;
#pragma unroll
    for (int k = 0; k < K; ++k)
      if ((m >> k) & 1u) W.v[k] = __ldcs(vals + off + __popc(m & ((1u << k) - 1u)));
  }
}

// butterfly reduce-scatter of a[0..31] over the warp: afterwards lane l holds
// the warp total of a[l] in a[0]
__device__ __forceinline__ double v21_reduce_scatter(double (&a)[32], int lane) {
#pragma unroll
  for (int half = 16; half >= 1; half >>= 1) {
    const bool up = lane & half;
#pragma unroll
    for (int i = 0; i < half; ++i) {
      const double send = up ? a[i] : a[i + half];
      const double keep = up ? a[i + half] : a[i];
      a[i] = keep + __shfl_xor_sync(0xffffffffu, send, half);
    }
  }
  return a[0];
}

template <int K>
__device__ __forceinline__ void v21_consume(const V21Work& W, int lane, int N, double (&acc)[K][3],
                                            double* __restrict__ vk) {
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const double v = (double)W.v[k];
    acc[k][0] = fma(v, W.x0, acc[k][0]);
    acc[k][1] = fma(v, W.x1, acc[k][1]);
    acc[k][2] = fma(v, W.x2, acc[k][2]);
  }
  if (W.last) {  // warp-uniform: every lane of the chunk has the same row
    double a[32];
#pragma unroll
    for (int k = 0; k < K; ++k) {
#pragma unroll
      for (int c = 0; c < 3; ++c) a[k * 3 + c] = acc[k][c];
    }
#pragma unroll
    for (int i = 3 * K; i < 32; ++i) a[i] = 0.0;
    const double s = v21_reduce_scatter(a, lane);
    if (lane < 3 * K) vk[(size_t)lane * N + W.row] = s;  // (k * 3 + c) * N + row
#pragma unroll
    for (int k = 0; k < K; ++k) acc[k][0] = acc[k][1] = acc[k][2] = 0.0;
  }
}

template <int K>
__global__ void __launch_bounds__(kV21Threads) k_transfer_kpairs(
    int N, const uint4* __restrict__ chunks, const uint32_t* __restrict__ hdr,
    const float* __restrict__ vals, const uint32_t* __restrict__ cbeg,
    const double4* __restrict__ xp, const uint32_t* __restrict__ bits, double* __restrict__ vk) {
  extern __shared__ uint32_t v21_bits[];
  for (int t = threadIdx.x; t < ((N + 31) >> 5); t += blockDim.x) v21_bits[t] = bits[t];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t q0 = cbeg[w], q1 = cbeg[w + 1];
  if (q0 >= q1) return;
  double acc[K][3];
#pragma unroll
  for (int k = 0; k < K; ++k) acc[k][0] = acc[k][1] = acc[k][2] = 0.0;
  // pipeline: S* = fetched (descriptor + header), W* = issued (gathers + values)
  V21Stage SA, SB;
  V21Work WA, WB;
  v21_fetch(SA, q0, lane, chunks, hdr);
  if (q0 + 1 < q1) v21_fetch(SB, q0 + 1, lane, chunks, hdr);
  v21_issue<K>(SA, lane, q0 + 1 < q1 ? SB.d.x : 0xffffffffu, v21_bits, xp, vals, WA);
  if (q0 + 2 < q1) v21_fetch(SA, q0 + 2, lane, chunks, hdr);
#pragma unroll 1
  for (uint32_t q = q0; q < q1; q += 2) {
    // chunk q in WA; SB holds q + 1, SA holds q + 2
    if (q + 1 < q1) v21_issue<K>(SB, lane, q + 2 < q1 ? SA.d.x : 0xffffffffu, v21_bits, xp, vals, WB);
    if (q + 3 < q1) v21_fetch(SB, q + 3, lane, chunks, hdr);
    v21_consume<K>(WA, lane, N, acc, vk);
    if (q + 1 >= q1) break;
    // chunk q + 1 in WB; SA holds q + 2, SB holds q + 3
    if (q + 2 < q1) v21_issue<K>(SA, lane, q + 3 < q1 ? SB.d.x : 0xffffffffu, v21_bits, xp, vals, WA);
    if (q + 4 < q1) v21_fetch(SA, q + 4, lane, chunks, hdr);
    v21_consume<K>(WB, lane, N, acc, vk);
  }
}

}  // namespace sss
