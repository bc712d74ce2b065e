// Stage 2 of the frame: v_k[c] = T_k x_c for every PCA term k and channel c.
//
// Reference: TransferOperator.apply -> csc_apply (transfer.py:50-71,
// _kernels_nb.py:301-313), called K x 3 times per frame by _stage2_transfer
// (runtime.py:138-150). x_c is the kept w0 spectrum of channel c (zero where
// compress_top_n dropped the coefficient), T_k the compressed operator.
//
// k_transfer_kfr ("K-fused rows", the default). The frame is bound by the
// L1 data pipe, not by HBM: every kept operator coefficient needs x of its
// column, a gather that touches its own 128-byte line. 28.6 M coefficients
// of the C3 operator are kept per frame but they sit on only 10.2 M distinct
// (row, column) pairs (the K terms of one row share columns), so this kernel
// gathers x once per PAIR and applies it to all the pair's terms:
//   * the layout (layout.py:kfr_layout) cuts every receiver row into chunks
//     of <= 512 (column, term-mask) pairs; a warp owns 32 chunks (lane ==
//     chunk == one row, all K terms: 3K fp64 accumulators in registers, no
//     atomics, no cross-lane reduction, deterministic order);
//   * step s of a warp: every lane takes the s-th pair of its chunk. The
//     pairs' {col u16 | mask << 16} words of one step are stored compacted
//     (active lanes in lane order), the f32 values term-plane by term-plane
//     (plane k: the lanes whose mask has bit k, in lane order), so the lane
//     offsets are __popc of warp ballots: no per-step headers;
//   * the warp's stream (words + values) is staged through shared memory by
//     TMA bulk copies (cp.async.bulk, mbarrier transaction counts), two
//     batches of U steps in flight per warp: reading it costs one
//     conflict-free LDS per plane, and the L1 pipe is left to the x gathers;
//   * only lanes whose column is kept (kept-column bitmap in shared memory)
//     gather x (one 32-byte fp64 record) and touch their values;
//   * chunks of rows longer than 512 pairs write fp64 partial sums; the last
//     chunk to finish a row (atomic arrival count) sums them in chunk order.
// Products are f32 operator value x fp64 x, accumulated in fp64 (SURVEY §8d:
// fp32 accumulation fails the 1e-4 bar); the summation order is fixed by the
// layout, so every frame is bitwise reproducible.
#include "sss_common.cuh"

namespace sss {

// packed x (N, 4) fp64 {x0, x1, x2, 0} + kept-column bitmap (bit c set iff
// any channel of x[:, c] is nonzero); one word past N stays clear
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

// one 32-byte x record through the read-only path
__device__ __forceinline__ void gather_x(const double4* __restrict__ xp, uint32_t c, double& a,
                                         double& b, double& d) {
  double e;
  asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(a), "=d"(b), "=d"(d), "=d"(e) : "l"(xp + c));
  (void)e;
}

// the same through the L1-bypassing load the flat16 kernel uses
__device__ __forceinline__ void v15_gather1(const double4* __restrict__ xp, uint32_t c, double* x) {
  double x3;
  asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(x[0]), "=d"(x[1]), "=d"(x[2]), "=d"(x3)
               : "l"(xp + c));
  (void)x3;
}

constexpr int kKfrWarps = 4;  // warps per CTA (independent; each owns its smem ring)
constexpr int kKfrU = 4;      // steps per staged batch

template <int K>
struct KfrSmem {
  // one batch: <= U*32 words and <= U*32*K values, + 32 bytes of alignment
  // slack each (the bulk copies start and end on 16-byte boundaries)
  static constexpr int CMB = kKfrU * 32 * 4 + 32;
  static constexpr int VB = kKfrU * 32 * K * 4 + 32;
  static constexpr int SLOT = CMB + VB;
  static constexpr int WARP = 2 * SLOT + 16;  // two slots + two mbarriers
};

inline size_t kfr_smem_bytes(int K, int N) {
  const size_t bits = (((size_t)((N >> 5) + 1) * 4 + 127) / 128) * 128;
  const size_t slot = (size_t)(kKfrU * 32 * 4 + 32) + (size_t)(kKfrU * 32 * K * 4 + 32);
  return bits + (size_t)kKfrWarps * (2 * slot + 16);
}

// K = accumulator slots (>= the operator's term count Kr; mask bits >= Kr are
// never set)
template <int K, int MINB>
__global__ void __launch_bounds__(kKfrWarps * 32, MINB) k_transfer_kfr(
    int N, int Kr, unsigned n_items, unsigned n_partials, const uint2* __restrict__ items,
    const uint32_t* __restrict__ lane_len, const uint32_t* __restrict__ lane_dst,
    const uint2* __restrict__ boff, const uint32_t* __restrict__ cm, const float* __restrict__ vals,
    const double4* __restrict__ xp, const uint32_t* __restrict__ bits, double* __restrict__ vk,
    double* __restrict__ part, const uint32_t* __restrict__ part_row,
    const uint4* __restrict__ minfo, unsigned* __restrict__ mcount) {
  using SM = KfrSmem<K>;
  extern __shared__ __align__(128) unsigned char kfr_smem[];
  const int nbw = (N >> 5) + 1;
  const int bits_bytes = ((nbw * 4 + 127) / 128) * 128;
  uint32_t* sbits = reinterpret_cast<uint32_t*>(kfr_smem);
  for (int t = threadIdx.x; t < nbw; t += blockDim.x) sbits[t] = bits[t];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* wb = kfr_smem + bits_bytes + wid * SM::WARP;
  uint64_t* bar = reinterpret_cast<uint64_t*>(wb + 2 * SM::SLOT);
  if (lane == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const unsigned lt = (1u << lane) - 1u;
  unsigned seq = 0;  // batches consumed by this warp: slot seq & 1, parity (seq >> 1) & 1
  const unsigned nwarps = gridDim.x * kKfrWarps;

  auto issue = [&](unsigned b, unsigned slot) {
    if (lane == 0) {
      const uint2 o0 = __ldg(&boff[b]), o1 = __ldg(&boff[b + 1]);
      const unsigned ca = (o0.x * 4u) & ~15u, ce = (o1.x * 4u + 15u) & ~15u;
      const unsigned va = (o0.y * 4u) & ~15u, ve = (o1.y * 4u + 15u) & ~15u;
      unsigned char* s = wb + slot * SM::SLOT;
      fence_proxy_async();
      mbar_expect_tx(&bar[slot], (ce - ca) + (ve - va));
      bulk_g2s(s, reinterpret_cast<const unsigned char*>(cm) + ca, ce - ca, &bar[slot]);
      bulk_g2s(s + SM::CMB, reinterpret_cast<const unsigned char*>(vals) + va, ve - va, &bar[slot]);
    }
  };

  for (unsigned item = blockIdx.x * kKfrWarps + wid; item < n_items; item += nwarps) {
    const uint2 it = __ldg(&items[item]);
    const unsigned b0 = it.x, S = it.y, nb = (S + kKfrU - 1) / kKfrU;
    const unsigned len = __ldg(&lane_len[item * 32 + lane]);
    double acc[K][3];
#pragma unroll
    for (int k = 0; k < K; ++k) acc[k][0] = acc[k][1] = acc[k][2] = 0.0;
    if (nb) issue(b0, seq & 1u);
#pragma unroll 1
    for (unsigned b = 0; b < nb; ++b) {
      const unsigned slot = seq & 1u, par = (seq >> 1) & 1u;
      if (b + 1 < nb) issue(b0 + b + 1, slot ^ 1u);
      const uint2 o0 = __ldg(&boff[b0 + b]);
      mbar_wait_warp(&bar[slot], par);
      ++seq;
      const uint32_t* scm = reinterpret_cast<const uint32_t*>(wb + slot * SM::SLOT) + (o0.x & 3u);
      const float* sv = reinterpret_cast<const float*>(wb + slot * SM::SLOT + SM::CMB) + (o0.y & 3u);
      // phase A: this batch's pair words, kept test, x gathers (U in flight)
      uint32_t w[kKfrU];
      bool kp[kKfrU];
      double xa[kKfrU][3];
      unsigned co = 0;
#pragma unroll
      for (int t = 0; t < kKfrU; ++t) {
        const bool act = b * kKfrU + t < len;
        const unsigned am = __ballot_sync(0xffffffffu, act);
        w[t] = act ? scm[co + __popc(am & lt)] : 0u;
        co += __popc(am);
        const uint32_t c = w[t] & 0xffffu;
        kp[t] = act && ((sbits[c >> 5] >> (c & 31u)) & 1u);
        xa[t][0] = xa[t][1] = xa[t][2] = 0.0;
        if (kp[t]) gather_x(xp, c, xa[t][0], xa[t][1], xa[t][2]);
      }
      // phase B: term planes, fp64 accumulation in (step, term) order
      unsigned vo = 0;
#pragma unroll
      for (int t = 0; t < kKfrU; ++t) {
        const uint32_t m = w[t] >> 16;  // 0 on inactive lanes
#pragma unroll
        for (int k = 0; k < K; ++k) {
          const unsigned bk = __ballot_sync(0xffffffffu, (m >> k) & 1u);
          if (bk) {
            if (kp[t] && ((m >> k) & 1u)) {
              const double v = (double)sv[vo + __popc(bk & lt)];
              acc[k][0] = fma(v, xa[t][0], acc[k][0]);
              acc[k][1] = fma(v, xa[t][1], acc[k][1]);
              acc[k][2] = fma(v, xa[t][2], acc[k][2]);
            }
            vo += __popc(bk);
          }
        }
      }
      __syncwarp();  // every lane is done with this slot before it is refilled
    }
    const unsigned dst = __ldg(&lane_dst[item * 32 + lane]);
    if (dst == 0xffffffffu) continue;  // padding lane of the last item
    if (!(dst & 0x80000000u)) {
#pragma unroll
      for (int k = 0; k < K; ++k)
        if (k < Kr)
#pragma unroll
          for (int c = 0; c < 3; ++c) vk[((size_t)k * 3 + c) * N + dst] = acc[k][c];
      continue;
    }
    // one chunk of a long row: partial sums; the last arriving chunk of the
    // row adds all of them in chunk order (the sum order is fixed)
    const unsigned p = dst & 0x7fffffffu;
#pragma unroll
    for (int k = 0; k < K; ++k)
      if (k < Kr)
#pragma unroll
        for (int c = 0; c < 3; ++c) part[((size_t)k * 3 + c) * n_partials + p] = acc[k][c];
    __threadfence();
    const unsigned m = __ldg(&part_row[p]);
    const uint4 mi = __ldg(&minfo[m]);  // (row, first partial, count, -)
    const unsigned old = atomicAdd(&mcount[m], 1u);
    if (old == mi.z - 1u) {
      __threadfence();
#pragma unroll 1
      for (int j = 0; j < 3 * Kr; ++j) {
        double s = 0.0;
        for (unsigned i = 0; i < mi.z; ++i) s += __ldcg(&part[(size_t)j * n_partials + mi.y + i]);
        vk[(size_t)j * N + mi.x] = s;
      }
      mcount[m] = 0u;  // ready for the next frame
    }
  }
}

}  // namespace sss
