// Frame layout v6: persistent, warp-specialized transfer kernel with
// per-item merge-path balancing.
//
// One CTA per unit (a contiguous range of tiles, ~one unit per SM). The
// unit's entries are grouped into items = (column band[, split]); inside an
// item they are sorted by (row, k, column), i.e. by "segment" (row, k). An
// entry is {u32 = (row_local << 4 | k) << 11 | band-local column, f32 val}.
//
// The transfer's work is spatially bursty: in a given column band only the
// rows near those source tiles have entries (local support of the
// diffusion kernel), so a static thread-per-row split is 60x imbalanced per
// item. Instead every item is split EVENLY across the 512 consumer threads
// (thread t takes entries [t n / 512, (t+1) n / 512)), each thread walks its
// contiguous slice accumulating the current segment in fp64 registers, and:
//   * segments that start and end inside the slice are added to the
//     unit's accumulator acc[row][k][c] in shared memory (exclusive);
//   * the slice's first / last partial segments are merged across lanes with
//     a warp-level affine scan (shuffles, no atomics) and across warps through
//     16 boundary records, then added once.
// Items are consumed by all warps together (two CTA barriers per item), so
// accumulator updates never race. A producer warp streams items through a
// cp.async.bulk ring and the x bands through a double buffer (mbarriers).
#include "sss_common.cuh"

namespace sss {

constexpr int kV6Warps = 16;
constexpr int kV6TPU = kV6Warps * 32;
constexpr int kV6Slots = 3;
constexpr int kV6XBufs = 2;
constexpr int kV6Threads = kV6TPU + 32;
constexpr int kV6ColBits = 11;  // band_width <= 2048

struct V6Item {
  unsigned long long off;  // byte offset of the item's entries in the stream (16-B aligned)
  unsigned n;              // entries
  unsigned short band;
  unsigned short pad;
};

struct V6Rec {  // warp boundary record
  int seg;
  int flag;  // head: 1 = the warp is one run end to end (head == tail)
  double v[3];
};

__device__ __forceinline__ void v6_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// named barrier over the 16 consumer warps only (the producer warp runs ahead)
__device__ __forceinline__ void consumer_sync() {
  asm volatile("bar.sync 1, %0;" ::"r"(kV6TPU) : "memory");
}

__device__ __forceinline__ void acc_flush(double* acc, int K, int seg, double a0, double a1,
                                          double a2) {
  const int idx = ((seg >> 4) * K + (seg & 15)) * 3;
  acc[idx] += a0;
  acc[idx + 1] += a1;
  acc[idx + 2] += a2;
}

__global__ void __launch_bounds__(kV6Threads, 1) k_transfer_v6(
    int K, int S, int L, int band_width, int slot_bytes,
    const int* __restrict__ unit_tile0, const int* __restrict__ unit_ntiles,
    const int* __restrict__ unit_item0, const int* __restrict__ unit_nitems,
    const V6Item* __restrict__ items, const unsigned char* __restrict__ stream,
    const double* __restrict__ x, const double* __restrict__ g,
    const float* __restrict__ positions, const float* __restrict__ normals,
    const double* __restrict__ cam, const double* __restrict__ material,
    double* __restrict__ vk, double* __restrict__ scatter, float* __restrict__ radiance,
    float* __restrict__ radiance_unclamped) {
  extern __shared__ __align__(128) unsigned char smraw[];
  const int T = 1 << L, T2 = T * T, N = S * S;
  const int unit = blockIdx.x;
  const int tile0 = unit_tile0[unit], ntiles = unit_ntiles[unit];
  const int R = ntiles * T2;
  const int row0 = tile0 * T2;
  const int nitems = unit_nitems[unit];

  unsigned char* ring = smraw;                                             // slots
  double* xsb = reinterpret_cast<double*>(ring + kV6Slots * slot_bytes);   // xbufs x 3 x bw
  double* acc = xsb + kV6XBufs * 3 * band_width;                           // R x K x 3
  V6Rec* head = reinterpret_cast<V6Rec*>(acc + (size_t)R * K * 3);         // kV6Warps
  V6Rec* tail = head + kV6Warps;                                           // kV6Warps
  uint64_t* bars = reinterpret_cast<uint64_t*>(tail + kV6Warps);
  uint64_t* full = bars;
  uint64_t* empty = full + kV6Slots;
  uint64_t* xfull = empty + kV6Slots;
  uint64_t* xempty = xfull + kV6XBufs;
  V6Item* uitems = reinterpret_cast<V6Item*>(xempty + kV6XBufs);
  const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;

  for (int i = tid; i < nitems; i += blockDim.x) uitems[i] = items[unit_item0[unit] + i];
  for (int i = tid; i < R * K * 3; i += blockDim.x) acc[i] = 0.0;
  if (tid == 0) {
    for (int s = 0; s < kV6Slots; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int j = 0; j < kV6XBufs; ++j) { mbar_init(&xfull[j], 1); mbar_init(&xempty[j], 1); }
    fence_mbar_init();
  }
  __syncthreads();

  if (wid == kV6Warps) {
    // ----------------------------- producer warp ------------------------------
    if (lane == 0) {
      int last_band = -1, bs = -1;
      for (int i = 0; i < nitems; ++i) {
        const V6Item it = uitems[i];
        if (it.band != last_band) {
          ++bs;
          const int j = bs % kV6XBufs, use = bs / kV6XBufs;
          if (use >= 1) mbar_wait(&xempty[j], (use - 1) & 1);
          const int c0 = it.band * band_width;
          const unsigned bytes = (unsigned)min(band_width, N - c0) * 8u;
          mbar_expect_tx(&xfull[j], 3u * bytes);
          for (int c = 0; c < 3; ++c)
            bulk_g2s(xsb + (j * 3 + c) * band_width, x + (size_t)c * N + c0, bytes, &xfull[j]);
          last_band = it.band;
        }
        const int s = i % kV6Slots, use = i / kV6Slots;
        if (use >= 1) mbar_wait(&empty[s], (use - 1) & 1);
        const unsigned bytes = ((it.n * 8u) + 15u) & ~15u;
        mbar_expect_tx(&full[s], bytes);
        bulk_g2s(ring + (size_t)s * slot_bytes, stream + it.off, bytes, &full[s]);
      }
    }
  } else {
    // ----------------------------- consumer warps -----------------------------
    int cur_bs = -1, cur_band = -1;
    const double* xs = xsb;
    for (int i = 0; i < nitems; ++i) {
      const V6Item it = uitems[i];
      if (it.band != cur_band) {
        ++cur_bs;
        cur_band = it.band;
        mbar_wait_warp(&xfull[cur_bs % kV6XBufs], (cur_bs / kV6XBufs) & 1);
        xs = xsb + (cur_bs % kV6XBufs) * 3 * band_width;
      }
      const int s = i % kV6Slots;
      mbar_wait_warp(&full[s], (i / kV6Slots) & 1);
      const uint2* ent = reinterpret_cast<const uint2*>(ring + (size_t)s * slot_bytes);
      const unsigned n = it.n;
      // even split of the item over the consumer threads
      unsigned lo, hi;
      if (n >= (unsigned)kV6TPU) {
        lo = (unsigned)(((unsigned long long)tid * n) / kV6TPU);
        hi = (unsigned)(((unsigned long long)(tid + 1) * n) / kV6TPU);
      } else {
        lo = min((unsigned)tid, n);
        hi = min((unsigned)tid + 1u, n);
      }
      const bool has = hi > lo;
      int fseg = -1, cur = -1;
      bool single = true;
      double f0 = 0.0, f1 = 0.0, f2 = 0.0;  // first segment partial
      double a0 = 0.0, a1 = 0.0, a2 = 0.0;  // current segment partial
      if (has) {
        cur = fseg = (int)(ent[lo].x >> kV6ColBits);
#pragma unroll 4
        for (unsigned p = lo; p < hi; ++p) {
          const uint2 e = ent[p];
          const int seg = (int)(e.x >> kV6ColBits);
          if (seg != cur) {
            if (single) { f0 = a0; f1 = a1; f2 = a2; single = false; }
            else acc_flush(acc, K, cur, a0, a1, a2);  // interior segment: exclusive
            a0 = a1 = a2 = 0.0;
            cur = seg;
          }
          const int col = (int)(e.x & ((1u << kV6ColBits) - 1u));
          const double v = (double)__uint_as_float(e.y);
          a0 = fma(v, xs[col], a0);
          a1 = fma(v, xs[band_width + col], a1);
          a2 = fma(v, xs[2 * band_width + col], a2);
        }
        if (single) { f0 = a0; f1 = a1; f2 = a2; }
      }
      // ---- warp-level merge of slice-boundary segments (affine scan)
      const int oseg = has ? cur : -2;                       // segment passed to the next lane
      const int prev_oseg = __shfl_up_sync(0xffffffffu, oseg, 1);
      const bool f = has && lane > 0 && fseg == prev_oseg;  // my first segment continues
      // O_l = alpha_l O_{l-1} + beta_l, alpha = single && f
      double b0 = single ? f0 : a0, b1 = single ? f1 : a1, b2 = single ? f2 : a2;
      int al = (has && single && f) ? 1 : 0;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int pa = __shfl_up_sync(0xffffffffu, al, d);
        const double p0 = __shfl_up_sync(0xffffffffu, b0, d);
        const double p1 = __shfl_up_sync(0xffffffffu, b1, d);
        const double p2 = __shfl_up_sync(0xffffffffu, b2, d);
        if (lane >= d) {
          if (al) { b0 += p0; b1 += p1; b2 += p2; }
          al = al & pa;
        }
      }
      // b = O_l ; carry into my first segment
      const double c0 = __shfl_up_sync(0xffffffffu, b0, 1);
      const double c1 = __shfl_up_sync(0xffffffffu, b1, 1);
      const double c2 = __shfl_up_sync(0xffffffffu, b2, 1);
      const double ft0 = f0 + (f ? c0 : 0.0), ft1 = f1 + (f ? c1 : 0.0), ft2 = f2 + (f ? c2 : 0.0);
      const bool next_f = __shfl_down_sync(0xffffffffu, f ? 1 : 0, 1) && lane < 31;
      // the run starting at lane 0 (may continue from the previous warp): find
      // its last lane r0 = first lane that is multi-segment or not continued
      const unsigned brk = __ballot_sync(0xffffffffu, !has || !single || !next_f);
      const int r0 = brk ? __ffs(brk) - 1 : 31;
      // flush decisions for my first segment
      if (has) {
        const bool ends_here = !single || !next_f;        // run containing my first seg ends here
        const bool in_head_run = lane <= r0;               // run reaches back to lane 0
        const bool tail_run = single && lane == 31;        // continues into the next warp
        if (ends_here && !in_head_run && !tail_run) {
          if (single) acc_flush(acc, K, fseg, b0, b1, b2);
          else acc_flush(acc, K, fseg, ft0, ft1, ft2);
        }
        // my last segment (multi-segment lanes) ends here unless the next
        // lane continues it; lane 31 hands it to the tail record
        if (!single && !next_f && lane < 31) acc_flush(acc, K, cur, a0, a1, a2);
      }
      {
        const int seg0 = __shfl_sync(0xffffffffu, fseg, 0);
        const int has0 = __shfl_sync(0xffffffffu, has ? 1 : 0, 0);
        if (lane == r0) {
          V6Rec& h = head[wid];
          h.seg = has0 ? seg0 : -1;
          h.flag = (r0 == 31 && single && has) ? 1 : 0;  // whole warp is one run
          const bool use_b = single;
          h.v[0] = use_b ? b0 : ft0;
          h.v[1] = use_b ? b1 : ft1;
          h.v[2] = use_b ? b2 : ft2;
          if (!has) { h.v[0] = h.v[1] = h.v[2] = 0.0; }
        }
        if (lane == 31) {
          V6Rec& tl = tail[wid];
          // the segment leaving the warp: lane 31's out segment, value O_31
          tl.seg = has ? oseg : -1;
          tl.v[0] = has ? b0 : 0.0;
          tl.v[1] = has ? b1 : 0.0;
          tl.v[2] = has ? b2 : 0.0;
          // multi-segment lane 31: its last segment partial is b (= a, alpha 0)
          tl.flag = (!single && has) ? 0 : 1;
        }
      }
      consumer_sync();  // all slices done, records visible
      if (wid == 0) {
        // cross-warp merge over 16 records (lanes 0..15): same affine scan
        const bool act = lane < kV6Warps;
        const int hs = act ? head[lane].seg : -3;
        const int ts = act ? tail[lane].seg : -4;
        const int through = act ? head[lane].flag : 0;
        const double hv0 = act ? head[lane].v[0] : 0.0, hv1 = act ? head[lane].v[1] : 0.0,
                     hv2 = act ? head[lane].v[2] : 0.0;
        const double tv0 = act ? tail[lane].v[0] : 0.0, tv1 = act ? tail[lane].v[1] : 0.0,
                     tv2 = act ? tail[lane].v[2] : 0.0;
        const int pts = __shfl_up_sync(0xffffffffu, ts, 1);
        const bool cf = act && lane > 0 && hs >= 0 && hs == pts;  // head continues prev tail
        // out_w = through ? (cf ? out_{w-1} : 0) + hv : tv
        double o0 = through ? hv0 : tv0, o1 = through ? hv1 : tv1, o2 = through ? hv2 : tv2;
        int al = (through && cf) ? 1 : 0;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const int pa = __shfl_up_sync(0xffffffffu, al, d);
          const double p0 = __shfl_up_sync(0xffffffffu, o0, d);
          const double p1 = __shfl_up_sync(0xffffffffu, o1, d);
          const double p2 = __shfl_up_sync(0xffffffffu, o2, d);
          if (lane >= d) {
            if (al) { o0 += p0; o1 += p1; o2 += p2; }
            al = al & pa;
          }
        }
        const double q0 = __shfl_up_sync(0xffffffffu, o0, 1);
        const double q1 = __shfl_up_sync(0xffffffffu, o1, 1);
        const double q2 = __shfl_up_sync(0xffffffffu, o2, 1);
        const bool next_cf = __shfl_down_sync(0xffffffffu, cf ? 1 : 0, 1) && lane + 1 < kV6Warps;
        if (act) {
          if (!through) {
            // head run of warp `lane` ends inside it: flush (with carry-in)
            if (hs >= 0)
              acc_flush(acc, K, hs, hv0 + (cf ? q0 : 0.0), hv1 + (cf ? q1 : 0.0),
                        hv2 + (cf ? q2 : 0.0));
            // tail: flushed here unless the next warp continues it
            if (ts >= 0 && !next_cf) acc_flush(acc, K, ts, tv0, tv1, tv2);
          } else {
            // through warp: the accumulated run leaves unless continued
            if (ts >= 0 && !next_cf) acc_flush(acc, K, ts, o0, o1, o2);
          }
        }
      }
      consumer_sync();  // cross-warp flushes done before the next item touches acc
      if (tid == 0) {
        v6_arrive(&empty[s]);
        // band buffer release once the next item moves to another band
        if (i + 1 == nitems || uitems[i + 1].band != cur_band) v6_arrive(&xempty[cur_bs % kV6XBufs]);
      }
    }
  }
  __syncthreads();

  // ------------------------------ epilogue (all threads) ----------------------
  double* summed = reinterpret_cast<double*>(smraw);     // ntiles x 3 x T2 (ring reused)
  double* tmp = summed + (size_t)ntiles * 3 * T2;
  for (int r = tid; r < R; r += blockDim.x) {
    const int row = row0 + r;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
    for (int k = 0; k < K; ++k) {
      const double* a = acc + (r * K + k) * 3;
      double* vo = vk + (size_t)k * 3 * N;
      vo[row] = a[0]; vo[N + row] = a[1]; vo[2 * N + row] = a[2];
      s0 += g[k] * a[0];
      s1 += g[K + k] * a[1];
      s2 += g[2 * K + k] * a[2];
    }
    const int tj = r / T2, e = r % T2;
    summed[(tj * 3 + 0) * T2 + e] = s0;
    summed[(tj * 3 + 1) * T2 + e] = s1;
    summed[(tj * 3 + 2) * T2 + e] = s2;
  }
  __syncthreads();
  multi_tile_epilogue(summed, tmp, T, tile0, ntiles, S, positions, normals, cam, material, scatter,
                      radiance, radiance_unclamped);
}

}  // namespace sss
