// Exact top-n selection of the irradiance spectrum with one 16-CTA thread-block
// cluster per channel (runtime.py:112-118 -> wavelets.compress_top_n,
// wavelets.py:128-136). Each CTA keeps its 1/16 slice of the channel resident
// in shared memory; every rank merges the per-digit histograms through
// distributed shared memory (DSMEM) itself, so the radix passes run on-chip on
// 16 SMs with one cluster barrier each; once <= 64 keys remain in the
// threshold bucket they are gathered cluster-wide and ranked exactly.
#include <cooperative_groups.h>

#include "select.cuh"

namespace sss {
namespace cg = cooperative_groups;

// phase timestamps for tools/select_trace (compiled only with SSS_SELECT_TRACE)
#ifdef SSS_SELECT_TRACE
__device__ unsigned long long g_sel_trace[32];
#define SEL_TRACE(i)                                                                  \
  do {                                                                                \
    if (blockIdx.x == 0 && threadIdx.x == 0) {                                        \
      unsigned long long t_;                                                          \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                          \
      g_sel_trace[i] = t_;                                                            \
    }                                                                                 \
  } while (0)
#else
#define SEL_TRACE(i) \
  do {               \
  } while (0)
#endif

// 16-CTA clusters (non-portable size, allowed on sm_100a): half the slice per
// CTA; measured 36 -> 32 us per 3 x 65536 select at C3 vs 8-CTA clusters
constexpr int kSelCluster = 16;

struct ClusterSelShared {
  unsigned hist[2][256];  // double-buffered by pass parity (see below)
  unsigned wtot[8];
  uint64_t wsum64[32];
  long long tie_cnt;
  double red[32];
  int scal_b;
  long long scal_need, scal_cnt;
  // early finish: candidates of the threshold bucket, gathered cluster-wide
  int ncand;
  int cnt_all[kSelCluster];
  uint64_t ckey[64];
  uint64_t gkey[64];
  unsigned char gsrc[64];
  uint64_t t_early;
  long long take_early, ties_early;
  int ties_below;
  double epart[kSelCluster][2];  // rank 0's copy receives every rank's energy sums
  uint32_t kbits[512];           // keep bits of the slice (chunk <= 16384)
};
static_assert(kSelCluster * 64 == 1024, "the candidate copy maps one thread per (rank, slot)");

// xp / bits (optional, 3 vectors = the frame's RGB spectrum): the packed
// (n_dom, 4) fp64 records {x0, x1, x2, 0} and the kept-column bitmap the
// transfer kernels read (sss_pack_x_bits' outputs, written here directly so
// the frame needs no packing launch). bits must be zero on entry; the fourth
// component of every record is never written (allocated zero).
__global__ void __cluster_dims__(kSelCluster, 1, 1) __launch_bounds__(1024)
    k_select_cluster(const double* __restrict__ ehat, int n_dom, int n_keep, int chunk,
                     const uint32_t* __restrict__ f2t, double* __restrict__ x,
                     uint32_t* __restrict__ mask, double* __restrict__ energy,
                     double* __restrict__ xp, uint32_t* __restrict__ bits) {
  extern __shared__ __align__(16) unsigned char dsm[];
  ClusterSelShared& sh = *reinterpret_cast<ClusterSelShared*>(dsm);
  double* v = reinterpret_cast<double*>(dsm + ((sizeof(ClusterSelShared) + 15) & ~size_t(15)));
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int c = blockIdx.x / kSelCluster;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wid = tid >> 5;
  const int lo = rank * chunk, hi = min(lo + chunk, n_dom), cnt_local = max(hi - lo, 0);
  pdl_launch_dependents();
  pdl_wait();
  SEL_TRACE(0);
  const double* src = ehat + (size_t)c * n_dom;
  for (int i = tid; i < cnt_local; i += nt) v[i] = src[lo + i];
  // output positions of this thread's first four elements, fetched now
  uint32_t tm4[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int i = tid + j * nt;
    tm4[j] = (f2t && i < cnt_local) ? __ldg(&f2t[lo + i]) : (uint32_t)(lo + i);
  }
  if (tid < 512) (&sh.hist[0][0])[tid] = 0u;
  const int n = min(n_keep, n_dom);
  __syncthreads();
  SEL_TRACE(1);

  uint64_t prefix = 0, pmask = 0;
  long long need = n;
  long long tie_total = 0;
  bool early = false;
  // 8-bit digits: the per-pass merge reads 16 x 256 remote counters (DSMEM
  // bandwidth, ~20 B/cycle/SM, made 11-bit digits cost 3.5 us per pass).
  constexpr int kPasses = 8;
  // Each pass: local histogram -> ONE cluster barrier -> every rank merges the
  // histograms through DSMEM and finds the bucket itself (deterministic, so
  // all ranks agree) - no second barrier and no serial rank-0 phase. The
  // histograms alternate between two buffers: buffer (p + 1) & 1 is cleared
  // after the pass p barrier, which every rank reaches only once it has
  // finished reading its peers' copy of that buffer (pass p - 1's merge).
  if (n > 0) {
    for (int p = 0; p < kPasses; ++p) {
      const int shf = 56 - 8 * p;
      unsigned* hist = sh.hist[p & 1];
      for (int i0 = 0; i0 < cnt_local; i0 += nt) {
        const int i = i0 + tid;
        unsigned bin = 0xffffffffu;
        if (i < cnt_local) {
          const uint64_t k = mkey(v[i]);
          if ((k & pmask) == prefix) bin = (unsigned)(k >> shf) & 255u;
        }
        if (p == 0) {
          // the top digit (high exponent bits) takes a handful of values: one
          // shared atomic per distinct digit of the warp, not one per lane
          const unsigned peers = __match_any_sync(0xffffffffu, bin);
          if (bin != 0xffffffffu && lane == __ffs(peers) - 1) atomicAdd(&hist[bin], __popc(peers));
        } else if (bin != 0xffffffffu) {
          atomicAdd(&hist[bin], 1u);
        }
      }
      SEL_TRACE(2 + 3 * p);
      cluster.sync();
      SEL_TRACE(3 + 3 * p);
      // threads 0..255: bin 255 - tid, counts merged over the ranks, scanned
      // from the top; threads 256..511 clear the other buffer meanwhile
      unsigned s = 0;
      if (tid < 256) {
        unsigned q[kSelCluster];
#pragma unroll
        for (int r = 0; r < kSelCluster; ++r) q[r] = cluster.map_shared_rank(hist, r)[255 - tid];
#pragma unroll
        for (int r = 0; r < kSelCluster; ++r) s += q[r];
      } else if (tid < 512) {
        sh.hist[(p + 1) & 1][tid - 256] = 0u;
      }
      unsigned incl = s;
      if (tid < 256) {
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        if (lane == 31) sh.wtot[wid] = incl;
      }
      if (tid == 0) sh.scal_b = -1;
      __syncthreads();
      if (tid < 256) {
        long long before = (long long)(incl - s);
        for (int w = 0; w < wid; ++w) before += sh.wtot[w];
        if (before < need && need <= before + (long long)s) {
          sh.scal_b = 255 - tid;
          sh.scal_need = need - before;
          sh.scal_cnt = s;
        }
      }
      __syncthreads();
      if (sh.scal_b < 0) {  // unreachable for consistent counts: everything down to bucket 0
        if (tid == 0) {
          long long above = 0;
          for (int w = 0; w < 8; ++w) above += sh.wtot[w];
          unsigned s0 = 0;
          for (int r = 0; r < kSelCluster; ++r) s0 += cluster.map_shared_rank(hist, r)[0];
          sh.scal_need = need - (above - (long long)s0);
          sh.scal_cnt = s0;
        }
        __syncthreads();
        if (tid == 0) sh.scal_b = 0;
        __syncthreads();
      }
      const int b = sh.scal_b;
      need = sh.scal_need;
      const long long cnt_bucket = sh.scal_cnt;
      tie_total = cnt_bucket;
      prefix |= (uint64_t)b << shf;
      pmask |= (uint64_t)255u << shf;
      SEL_TRACE(4 + 3 * p);
      if (p + 1 < kPasses && cnt_bucket <= 64) {
        // Few keys left in the threshold bucket (cluster-wide): gather them all
        // and finish exactly with a rank count instead of the remaining passes.
        if (tid == 0) sh.ncand = 0;
        __syncthreads();
        for (int i = tid; i < cnt_local; i += nt) {
          const uint64_t k = mkey(v[i]);
          if ((k & pmask) == prefix) sh.ckey[atomicAdd(&sh.ncand, 1)] = k;
        }
        cluster.sync();
        if (tid < kSelCluster) sh.cnt_all[tid] = cluster.map_shared_rank(&sh, tid)->ncand;
        __syncthreads();
        {  // thread (r, j) copies candidate j of rank r (all remote reads in flight at once)
          const int r = tid >> 6, j = tid & 63;
          if (j < sh.cnt_all[r]) {
            int off = 0;
            for (int q = 0; q < r; ++q) off += sh.cnt_all[q];
            sh.gkey[off + j] = cluster.map_shared_rank(&sh, r)->ckey[j];
            sh.gsrc[off + j] = (unsigned char)r;
          }
        }
        __syncthreads();
        int total = 0;
        for (int r = 0; r < kSelCluster; ++r) total += sh.cnt_all[r];
        if (tid < total) {
          const uint64_t kj = sh.gkey[tid];
          long long g = 0, e = 0;
          for (int q = 0; q < total; ++q) {
            const uint64_t kq = sh.gkey[q];
            g += kq > kj;
            e += kq == kj;
          }
          if (g < need && need <= g + e) {  // every equal key writes the same values
            sh.t_early = kj;
            sh.take_early = need - g;
            sh.ties_early = e;
          }
        }
        if (tid == 0) sh.ties_below = 0;
        __syncthreads();
        prefix = sh.t_early;
        need = sh.take_early;
        tie_total = sh.ties_early;
        pmask = ~0ULL;
        early = true;
        if (need != tie_total && tid < total && sh.gkey[tid] == prefix && (int)sh.gsrc[tid] < rank)
          atomicAdd(&sh.ties_below, 1);  // ties held by lower ranks (index order across the cluster)
        break;
      }
    }
  }
  const uint64_t t = n > 0 ? prefix : ~0ULL;
  const long long take = n > 0 ? need : 0;
  const int per = (cnt_local + nt - 1) / nt;
  const int a0 = min(tid * per, cnt_local), a1 = min(a0 + per, cnt_local);
  // ties in index order across the cluster - only when some but not all of
  // the keys equal to the threshold are kept (otherwise keep <=> key >= t)
  const bool all_ties = take == tie_total;
  long long tie_rank = 0;
  if (!all_ties) {
    long long my_ties = 0;
    for (int i = a0; i < a1; ++i) my_ties += (mkey(v[i]) == t);
    const uint64_t before_local = block_excl_scan_u64((uint64_t)my_ties, sh.wsum64);
    long long before_rank = 0;
    if (early) {
      __syncthreads();  // ties_below complete
      before_rank = sh.ties_below;
    } else {
      if (tid == nt - 1) sh.tie_cnt = (long long)(before_local + my_ties);
      cluster.sync();
      for (int r = 0; r < rank; ++r) before_rank += cluster.map_shared_rank(&sh, r)->tie_cnt;
    }
    tie_rank = before_rank + (long long)before_local;
  }
  SEL_TRACE(20);
  // decide in blocked index order (tie ranks), keep-bits into shared words
  // (4 threads x 8 elements per word, combined with shuffles), kept values in
  // place; then coalesced writes of x (scattered only through f2t) and mask
  double tot = 0.0, kept = 0.0;
  double* xo = x ? x + (size_t)c * n_dom : nullptr;
  unsigned bits8 = 0;
  for (int i = a0; i < a1; ++i) {
    const double e = v[i];
    const uint64_t k = mkey(e);
    bool keep = all_ties ? k >= t : k > t;
    if (!all_ties && k == t) { keep = tie_rank < take; ++tie_rank; }
    tot += e * e;
    if (keep) kept += e * e;
    bits8 |= (keep ? 1u : 0u) << (i - a0);
    v[i] = keep ? e : 0.0;
  }
  uint32_t* kbits = sh.kbits;
  if (per <= 32 && (per & (per - 1)) == 0 && cnt_local % 32 == 0) {
    // 32 / per adjacent lanes own the 32 elements of one word
    const int lpw = 32 / per;
    unsigned w = bits8 << ((lane & (lpw - 1)) * per);
    for (int o = 1; o < lpw; o <<= 1) w |= __shfl_xor_sync(0xffffffffu, w, o);
    if ((lane & (lpw - 1)) == 0 && a0 < cnt_local) kbits[a0 >> 5] = w;
    __syncthreads();
  } else {
    for (int q = tid; q * 32 < cnt_local; q += nt) kbits[q] = 0u;
    __syncthreads();
    for (int i = a0; i < a1; ++i)
      if ((bits8 >> (i - a0)) & 1u) atomicOr(&kbits[i >> 5], 1u << (i & 31));
    __syncthreads();
  }
  for (int i = tid, j = 0; i < cnt_local; i += nt, ++j) {
    const int gi = lo + i;
    const uint32_t tm = j < 4 ? tm4[j] : (f2t ? __ldg(&f2t[gi]) : (uint32_t)gi);
    const double val = v[i];
    if (xo) xo[tm] = val;
    if (xp) {
      xp[(size_t)tm * 4 + c] = val;
      if (val != 0.0) atomicOr(&bits[tm >> 5], 1u << (tm & 31u));
    }
  }
  if (mask) {
    uint32_t* mo = mask + (size_t)c * ((n_dom + 31) / 32);
    for (int q = tid; q * 32 < cnt_local; q += nt) mo[(lo >> 5) + q] = kbits[q];
  }
  SEL_TRACE(27);
  // both sums in one pass: warp shuffles, then warp 0 over the 32 warp sums
  for (int o = 16; o > 0; o >>= 1) {
    tot += __shfl_xor_sync(0xffffffffu, tot, o);
    kept += __shfl_xor_sync(0xffffffffu, kept, o);
  }
  double* red2 = reinterpret_cast<double*>(sh.wsum64);  // 32 u64: unused by now
  if (lane == 0) { sh.red[wid] = tot; red2[wid] = kept; }
  __syncthreads();
  if (wid == 0) {
    tot = lane < (nt >> 5) ? sh.red[lane] : 0.0;
    kept = lane < (nt >> 5) ? red2[lane] : 0.0;
    for (int o = 16; o > 0; o >>= 1) {
      tot += __shfl_xor_sync(0xffffffffu, tot, o);
      kept += __shfl_xor_sync(0xffffffffu, kept, o);
    }
    if (lane == 0) {  // every rank deposits its sums in rank 0's shared memory
      double* dst = cluster.map_shared_rank(&sh.epart[0][0], 0);
      dst[rank * 2 + 0] = tot;
      dst[rank * 2 + 1] = kept;
    }
  }
  // the one closing barrier: after it no CTA reads a peer's shared memory, so
  // every CTA may exit; rank 0 sums the deposits in rank order (deterministic)
  cluster.sync();
  if (rank == 0 && tid == 0 && energy) {
    double T = 0.0, Kp = 0.0;
    for (int r = 0; r < kSelCluster; ++r) {
      T += sh.epart[r][0];
      Kp += sh.epart[r][1];
    }
    energy[c * 2 + 0] = T;
    energy[c * 2 + 1] = fmin(Kp, T);
  }
  SEL_TRACE(28);
}

}  // namespace sss
