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
//     of a length chosen per operator (layout.kfr_auto_chunk: just under the
//     mean work per warp) of (column, term-mask) pairs; a warp owns 32 chunks (lane ==
//     chunk == one row, all K terms: 3K fp64 accumulators in registers, no
//     atomics, no cross-lane reduction, deterministic order);
//   * step s of a warp: every lane takes the s-th pair of its chunk. The
//     pairs' {col u16 | mask << 16 | value offset << 20} words of one step are
//     32 dense words (0 where the lane's chunk has ended), the f32 values of a
//     batch of U steps follow in (step, lane, term) order and every word
//     carries its lane's offset in that block: no per-step headers, no
//     running base between the steps of a batch;
//   * the warp's stream (words + values) is staged through shared memory by
//     TMA bulk copies (cp.async.bulk, mbarrier transaction counts), two
//     batches of U steps in flight per warp: reading it costs one
//     conflict-free LDS per plane, and the L1 pipe is left to the x gathers;
//   * only lanes whose column is kept (kept-column bitmap in shared memory)
//     gather x (one 32-byte fp64 record) and touch their values;
//   * chunks of rows longer than one chunk write fp64 partial sums; the last
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

// one 32-byte x record through the read-only path, predicated inside the
// instruction: the destination registers ARE the lane's x registers (a lane
// that skips keeps its last record), so no conditional moves sit between the
// load and its first use and the U gathers of a batch stay in flight together
__device__ __forceinline__ void gather_x_if(const double4* __restrict__ xp, uint32_t c, bool kept,
                                            double (&x)[4]) {
  asm("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %5, 0;\n\t"
      "@q ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];\n\t}"
      : "+d"(x[0]), "+d"(x[1]), "+d"(x[2]), "+d"(x[3])
      : "l"(xp + c), "r"((unsigned)kept));
}

// the same through the L1-bypassing load the flat16 kernel uses
__device__ __forceinline__ void v15_gather1(const double4* __restrict__ xp, uint32_t c, double* x) {
  double x3;
  asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(x[0]), "=d"(x[1]), "=d"(x[2]), "=d"(x3)
               : "l"(xp + c));
  (void)x3;
}

constexpr int kKfrWarps = 8;  // warps per CTA (independent; each owns its smem ring)
constexpr int kKfrG = 4;      // terms per group: a chunk accumulates G terms x 3 channels
static_assert(kKfrG == 4, "phase B's slot selects are written for groups of 4 terms");
constexpr int kKfrMaxBatches = 128;  // batches per item (chunk length <= 128 * steps per batch)

template <int U, int NS>  // steps per staged batch, ring slots per warp
struct KfrSmem {
  // one batch of the stream: U*32 pair words (dense per step), then <= U*32*G
  // values, padded to 16 bytes (one bulk copy per batch)
  static constexpr int WB = U * 32 * 4;
  static constexpr int VB = U * 32 * kKfrG * 4 + 16;  // + slack: lanes read 4 values unconditionally
  static constexpr int SLOT = (WB + VB + 15) / 16 * 16;
  static_assert(WB % 16 == 0, "word block must keep 16-byte alignment");
  // the item's batch offsets (<= kKfrMaxBatches + 1 u32)
  static constexpr int BOFF = (kKfrMaxBatches + 1) * 4;
  // NS slots + NS mbarriers + offsets, 128-byte aligned (bulk copies need 16)
  static constexpr int WARP = ((NS * SLOT + 8 * NS + BOFF) + 127) / 128 * 128;
};

constexpr int kKfrBitWords = 65536 / 32 + 1;  // kept-column bitmap, static shared

inline size_t kfr_smem_bytes(int N, size_t warp_bytes) {
  (void)N;
  return (size_t)kKfrWarps * warp_bytes;  // dynamic part (the bitmap is static)
}

// Pair word: col (bits 0-15) | term mask within the group (16-19) | offset of
// the lane's first value in the batch's value block (20-31); 0 = no pair.
template <int U, int NS, int MINB>
__global__ void __launch_bounds__(kKfrWarps * 32, MINB) k_transfer_kfr(
    int N, int Kr, unsigned n_items, unsigned n_partials, const uint2* __restrict__ items,
    const uint32_t* __restrict__ lane_len, const uint32_t* __restrict__ lane_dst,
    const uint32_t* __restrict__ boff, const unsigned char* __restrict__ stream,
    const double4* __restrict__ xp,
    const uint32_t* __restrict__ bits, double* __restrict__ vk, double* __restrict__ part,
    const uint32_t* __restrict__ part_row, const uint4* __restrict__ minfo,
    unsigned* __restrict__ mcount, unsigned* __restrict__ work) {
  using SM = KfrSmem<U, NS>;
  constexpr int G = kKfrG;
  extern __shared__ __align__(128) unsigned char kfr_smem[];
  __shared__ uint32_t sbits[kKfrBitWords];
  pdl_launch_dependents();
  const int nbw = (N >> 5) + 1;
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* wb = kfr_smem + wid * SM::WARP;
  uint64_t* bar = reinterpret_cast<uint64_t*>(wb + NS * SM::SLOT);
  uint32_t* sboff = reinterpret_cast<uint32_t*>(wb + NS * SM::SLOT + 8 * NS);
  if (lane == 0) {
#pragma unroll
    for (int j = 0; j < NS; ++j) mbar_init(&bar[j], 1);
    fence_mbar_init();
  }
  pdl_wait();  // x, the bitmap and the claim counters are the predecessor's
  for (int t = threadIdx.x; t < nbw; t += blockDim.x) sbits[t] = bits[t];
  __syncthreads();
  // batches consumed by this warp: slot seq % NS, parity (seq / NS) & 1; the
  // ring runs NS - 1 batches ahead of the consumer
  unsigned seq = 0;

  // batch b = stream bytes [boff[b], boff[b + 1]), 16-byte aligned. The slot
  // was last read by this warp (its loads completed before the __syncwarp
  // that ended that batch): no proxy fence is needed for the write-after-read
  auto issue = [&](unsigned b, unsigned slot) {  // b: batch of the current item
    if (lane == 0) {  // one TMA bulk copy, completion counted on the slot's mbarrier
      const unsigned a0 = sboff[b], a1 = sboff[b + 1];
      mbar_expect_tx(&bar[slot], a1 - a0);
      bulk_g2s(wb + slot * SM::SLOT, stream + a0, a1 - a0, &bar[slot]);
    }
  };

  for (;;) {
    // items are ordered longest first; warps claim them dynamically (the
    // counters are reset by the last CTA out, so graph replays work)
    unsigned item = 0;
    if (lane == 0) item = atomicAdd(&work[0], 1u);
    item = __shfl_sync(0xffffffffu, item, 0);
    if (item >= n_items) break;
    const uint2 it = __ldg(&items[item]);
    const unsigned b0 = it.x, S = it.y, nb = (S + U - 1) / U;
    // the item's batch offsets, staged once (the issuing lane reads them from
    // shared memory instead of an L2 round trip per batch)
    for (unsigned j = lane; j <= nb; j += 32) sboff[j] = __ldg(&boff[b0 + j]);
    __syncwarp();
    double acc[G][3];
#pragma unroll
    for (int k = 0; k < G; ++k) acc[k][0] = acc[k][1] = acc[k][2] = 0.0;
    // phase A of a batch: pair words (0 past the chunk's end), kept test, x
    // gathers (U in flight per lane). x of a skipped step keeps the last
    // gathered (finite) value, so an absent or unkept term's 0 * x adds
    // exactly nothing
    auto phaseA = [&](const unsigned char* slot_p, uint32_t (&w)[U], bool (&kp)[U],
                      double (&xa)[U][4]) {
      const uint32_t* sw = reinterpret_cast<const uint32_t*>(slot_p);
#pragma unroll
      for (int t = 0; t < U; ++t) {
        w[t] = sw[t * 32 + lane];
        const uint32_t c = w[t] & 0xffffu;
        // an empty slot (word 0: column 0, mask 0) may pass the test and gather
        // x[0]; its mask contributes no values, so nothing is added
        kp[t] = ((sbits[c >> 5] >> (c & 31u)) & 1u) != 0u;
        gather_x_if(xp, c, kp[t], xa[t]);
      }
    };
    // phase B: the lane's values (lane-major in the step block; the term of
    // each is the next set bit of the mask), fp64 accumulation in (step,
    // term) order
    auto phaseB = [&](const unsigned char* slot_p, const uint32_t (&w)[U], const bool (&kp)[U],
                      const double (&xa)[U][4]) {
      const float* sv = reinterpret_cast<const float*>(slot_p + SM::WB);
#pragma unroll
      for (int t = 0; t < U; ++t) {
        const uint32_t m = (w[t] >> 16) & 0xfu;
        const float* sl = sv + (w[t] >> 20);  // offset in the batch's value block
        const uint32_t mk = kp[t] ? m : 0u;
        float vf[G];  // one predicated load per present term
#pragma unroll
        for (int k = 0; k < G; ++k)
          vf[k] = ((mk >> k) & 1u) ? sl[__popc(m & ((1u << k) - 1u))] : 0.0f;
#pragma unroll
        for (int k = 0; k < G; ++k) {
          const double v = (double)vf[k];
          acc[k][0] = fma(v, xa[t][0], acc[k][0]);
          acc[k][1] = fma(v, xa[t][1], acc[k][1]);
          acc[k][2] = fma(v, xa[t][2], acc[k][2]);
        }
      }
    };
    auto slot_of = [&](unsigned q) { return wb + (q % NS) * SM::SLOT; };
    uint32_t w[U];
    bool kp[U];
    double xa[U][4];
#pragma unroll
    for (int t = 0; t < U; ++t) xa[t][0] = xa[t][1] = xa[t][2] = xa[t][3] = 0.0;
    const unsigned q0 = seq;  // ring position of batch 0 of this item
#pragma unroll
    for (int j = 0; j < NS; ++j)
      if ((unsigned)j < nb) issue(j, (q0 + j) % NS);
#pragma unroll 1
    for (unsigned b = 0; b < nb; ++b) {
      const unsigned q = q0 + b;
      mbar_wait_warp_spin(&bar[q % NS], (q / NS) & 1u);
      phaseA(slot_of(q), w, kp, xa);
      phaseB(slot_of(q), w, kp, xa);
      __syncwarp();  // every lane is done with this slot before it is refilled
      if (b + NS < nb) issue(b + NS, q % NS);
    }
    seq = q0 + nb;
    const unsigned dst = __ldg(&lane_dst[item * 32 + lane]);
    if (dst != 0xffffffffu && !(dst & 0x80000000u)) {  // a whole (row, term group)
      const unsigned row = dst & 0xffffu, k0 = (dst >> 16) * G;
#pragma unroll
      for (int k = 0; k < G; ++k)
        if (k0 + k < (unsigned)Kr)
#pragma unroll
          for (int c = 0; c < 3; ++c) vk[((size_t)(k0 + k) * 3 + c) * N + row] = acc[k][c];
    } else if (dst != 0xffffffffu) {
      // one chunk of a long (row, group): partial sums; the last arriving
      // chunk adds all of them in chunk order (the sum order is fixed)
      const unsigned p = dst & 0x7fffffffu;
#pragma unroll
      for (int k = 0; k < G; ++k)
#pragma unroll
        for (int c = 0; c < 3; ++c) part[((size_t)k * 3 + c) * n_partials + p] = acc[k][c];
      __threadfence();
      const unsigned m = __ldg(&part_row[p]);
      const uint4 mi = __ldg(&minfo[m]);  // (row, first partial, count, group)
      const unsigned old = atomicAdd(&mcount[m], 1u);
      if (old == mi.z - 1u) {
        __threadfence();
        // fixed order: i ascending per component. All G terms' partial sums of
        // four chunks are loaded together (one round trip for the usual rows
        // of <= 4 chunks instead of one per term; the adds stay in order)
        double sum[G][3];
#pragma unroll
        for (int k = 0; k < G; ++k) sum[k][0] = sum[k][1] = sum[k][2] = 0.0;
#pragma unroll 1
        for (unsigned i0 = 0; i0 < mi.z; i0 += 4) {
          double q[G][3][4];
#pragma unroll
          for (int k = 0; k < G; ++k)
#pragma unroll
            for (int c = 0; c < 3; ++c)
#pragma unroll
              for (int i = 0; i < 4; ++i)
                q[k][c][i] = (i0 + i < mi.z)
                                 ? __ldcg(&part[(size_t)(k * 3 + c) * n_partials + mi.y + i0 + i]) : 0.0;
#pragma unroll
          for (int k = 0; k < G; ++k)
#pragma unroll
            for (int c = 0; c < 3; ++c)
#pragma unroll
              for (int i = 0; i < 4; ++i)
                if (i0 + i < mi.z) sum[k][c] += q[k][c][i];
        }
#pragma unroll
        for (int k = 0; k < G; ++k)
          if (mi.w * G + k < (unsigned)Kr)
#pragma unroll
            for (int c = 0; c < 3; ++c) vk[((size_t)(mi.w * G + k) * 3 + c) * N + mi.x] = sum[k][c];
        mcount[m] = 0u;  // ready for the next frame
      }
    }
    __syncwarp();
  }
  // the last CTA out resets the claim counters for the next launch
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&work[1], 1u) == gridDim.x - 1u) {
      work[0] = 0u;
      work[1] = 0u;
      __threadfence();
    }
  }
}

}  // namespace sss
