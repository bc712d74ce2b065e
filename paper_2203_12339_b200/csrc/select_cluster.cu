// Exact top-n selection of the irradiance spectrum with one 8-CTA thread-block
// cluster per channel (runtime.py:112-118 -> wavelets.compress_top_n,
// wavelets.py:128-136). Each CTA keeps its 1/8 slice of the channel resident
// in shared memory; the per-digit histograms are merged through distributed
// shared memory (DSMEM) by the cluster's rank-0 CTA, so all six radix passes
// run on-chip with 8 SMs instead of one.
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
  unsigned hist[2][2048];  // double-buffered by pass parity (see below)
  unsigned merged[2048];
  uint64_t wsum64[32];
  int dec_b[2];
  long long dec_need[2];
  long long dec_cnt[2];
  long long tie_cnt;
  double part_tot, part_kept;
  double red[32];
  long long redi[32];
  int scal_b;
  long long scal_need, scal_cnt;
  // early finish: candidates of the threshold bucket, gathered cluster-wide
  int ncand;
  uint64_t ckey[1024];
  uint64_t gkey[1024];
  uint64_t t_early;
  long long take_early;
};

__global__ void __cluster_dims__(kSelCluster, 1, 1) __launch_bounds__(1024)
    k_select_cluster(const double* __restrict__ ehat, int n_dom, int n_keep, int chunk,
                     const uint32_t* __restrict__ f2t, double* __restrict__ x,
                     uint32_t* __restrict__ mask, double* __restrict__ energy) {
  extern __shared__ __align__(16) unsigned char dsm[];
  ClusterSelShared& sh = *reinterpret_cast<ClusterSelShared*>(dsm);
  double* v = reinterpret_cast<double*>(dsm + ((sizeof(ClusterSelShared) + 15) & ~size_t(15)));
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int c = blockIdx.x / kSelCluster;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int lo = rank * chunk, hi = min(lo + chunk, n_dom), cnt_local = max(hi - lo, 0);
  SEL_TRACE(0);
  const double* src = ehat + (size_t)c * n_dom;
  for (int i = tid; i < cnt_local; i += nt) v[i] = src[lo + i];
  const int n = min(n_keep, n_dom);
  __syncthreads();
  SEL_TRACE(1);

  uint64_t prefix = 0, pmask = 0;
  long long need = n;
  // 8-bit digits: the per-pass merge reads 8 x 256 remote counters (DSMEM
  // bandwidth, ~20 B/cycle/SM, made 11-bit digits cost 3.5 us per pass)
  constexpr int kPasses = 8;
  const int digits[kPasses] = {56, 48, 40, 32, 24, 16, 8, 0};
  const int widths[kPasses] = {8, 8, 8, 8, 8, 8, 8, 8};
  // Each pass: local histogram -> ONE cluster barrier -> every rank merges the
  // 8 histograms through DSMEM and finds the bucket itself (deterministic, so
  // all ranks agree) - no second barrier and no serial rank-0 phase. The
  // histograms alternate between two buffers: buffer p & 1 is rewritten two
  // passes later, after the pass p+1 barrier, which every rank reaches only
  // once it has finished reading its peers' buffer p.
  if (n > 0) {
    for (int p = 0; p < kPasses; ++p) {
      const int shf = digits[p], nb = 1 << widths[p];
      unsigned* hist = sh.hist[p & 1];
      for (int b = tid; b < nb; b += nt) hist[b] = 0;
      __syncthreads();
      for (int i = tid; i < cnt_local; i += nt) {
        const uint64_t k = mkey(v[i]);
        if ((k & pmask) == prefix) atomicAdd(&hist[(k >> shf) & (nb - 1)], 1u);
      }
      SEL_TRACE(2 + 3 * p);
      cluster.sync();
      SEL_TRACE(3 + 3 * p);
      for (int b = tid; b < nb; b += nt) {
        unsigned s = 0;
#pragma unroll
        for (int r = 0; r < kSelCluster; ++r) s += cluster.map_shared_rank(hist, r)[b];
        sh.merged[b] = s;
      }
      __syncthreads();
      {
        const int per = (nb + nt - 1) / nt;
        const int top = nb - 1 - tid * per;
        uint64_t s = 0;
        for (int q = 0; q < per; ++q) {
          const int b = top - q;
          if (b < 0) break;
          s += sh.merged[b];
        }
        const uint64_t before = block_excl_scan_u64(s, sh.wsum64);
        if (tid == 0) sh.scal_b = -1;
        __syncthreads();
        if ((long long)before < need && need <= (long long)(before + s)) {
          uint64_t acc = before;
          for (int q = 0; q < per; ++q) {
            const int b = top - q;
            if ((long long)(acc + sh.merged[b]) >= need) {
              sh.scal_b = b;
              sh.scal_need = need - (long long)acc;
              sh.scal_cnt = sh.merged[b];
              break;
            }
            acc += sh.merged[b];
          }
        }
        __syncthreads();
        if (tid == 0 && sh.scal_b < 0) {  // unreachable for consistent counts: bucket 0
          uint64_t above = 0;
          for (int b = nb - 1; b > 0; --b) above += sh.merged[b];
          sh.scal_b = 0;
          sh.scal_need = need - (long long)above;
          sh.scal_cnt = sh.merged[0];
        }
        __syncthreads();
      }
      const int b = sh.scal_b;
      need = sh.scal_need;
      const long long cnt_bucket = sh.scal_cnt;
      prefix |= (uint64_t)b << shf;
      pmask |= (uint64_t)(nb - 1) << shf;
      __syncthreads();  // scal_* reused next pass
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
        int total = 0;
        for (int r = 0; r < kSelCluster; ++r) {
          ClusterSelShared* rs = cluster.map_shared_rank(&sh, r);
          const int nr = rs->ncand;
          for (int j = tid; j < nr; j += nt) sh.gkey[total + j] = rs->ckey[j];
          total += nr;
        }
        __syncthreads();
        for (int j = tid; j < total; j += nt) {
          const uint64_t kj = sh.gkey[j];
          long long g = 0, e = 0;
          for (int q = 0; q < total; ++q) {
            const uint64_t kq = sh.gkey[q];
            g += kq > kj;
            e += kq == kj;
          }
          if (g < need && need <= g + e) {  // every equal key writes the same values
            sh.t_early = kj;
            sh.take_early = need - g;
          }
        }
        __syncthreads();
        prefix = sh.t_early;
        need = sh.take_early;
        pmask = ~0ULL;
        break;
      }
    }
  }
  const uint64_t t = n > 0 ? prefix : ~0ULL;
  const long long take = n > 0 ? need : 0;
  // ties in index order across the cluster: count local ties, scan by rank
  const int per = (cnt_local + nt - 1) / nt;
  const int a0 = min(tid * per, cnt_local), a1 = min(a0 + per, cnt_local);
  long long my_ties = 0;
  for (int i = a0; i < a1; ++i) my_ties += (mkey(v[i]) == t);
  const uint64_t before_local = block_excl_scan_u64((uint64_t)my_ties, sh.wsum64);
  if (tid == nt - 1) sh.tie_cnt = (long long)(before_local + my_ties);
  cluster.sync();
  long long before_rank = 0;
  for (int r = 0; r < rank; ++r) before_rank += cluster.map_shared_rank(&sh, r)->tie_cnt;
  long long tie_rank = before_rank + (long long)before_local;
  SEL_TRACE(20);
  // decide in blocked index order (tie ranks), keep-bits into shared words
  // (4 threads x 8 elements per word, combined with shuffles), kept values in
  // place; then coalesced writes of x (scattered only through f2t) and mask
  double tot = 0.0, kept = 0.0;
  double* xo = x + (size_t)c * n_dom;
  unsigned bits8 = 0;
  for (int i = a0; i < a1; ++i) {
    const double e = v[i];
    const uint64_t k = mkey(e);
    bool keep = k > t;
    if (k == t) { keep = tie_rank < take; ++tie_rank; }
    tot += e * e;
    if (keep) kept += e * e;
    bits8 |= (keep ? 1u : 0u) << (i - a0);
    v[i] = keep ? e : 0.0;
  }
  uint32_t* kbits = reinterpret_cast<uint32_t*>(sh.merged);  // free after the passes
  if (per == 8) {
    // lanes 4j..4j+3 own the 32 elements of one word
    const int lane = tid & 31;
    unsigned w = bits8 << ((lane & 3) * 8);
    w |= __shfl_xor_sync(0xffffffffu, w, 1);
    w |= __shfl_xor_sync(0xffffffffu, w, 2);
    if ((lane & 3) == 0 && a0 < cnt_local) kbits[a0 >> 5] = w;
    __syncthreads();
  } else {
    for (int q = tid; q * 32 < cnt_local; q += nt) kbits[q] = 0u;
    __syncthreads();
    for (int i = a0; i < a1; ++i)
      if ((bits8 >> (i - a0)) & 1u) atomicOr(&kbits[i >> 5], 1u << (i & 31));
    __syncthreads();
  }
  for (int i = tid; i < cnt_local; i += nt) {
    const int gi = lo + i;
    xo[f2t ? __ldg(&f2t[gi]) : gi] = v[i];
  }
  if (mask) {
    uint32_t* mo = mask + (size_t)c * ((n_dom + 31) / 32);
    for (int q = tid; q * 32 < cnt_local; q += nt) mo[(lo >> 5) + q] = kbits[q];
  }
  SEL_TRACE(27);
  tot = block_sum_d(tot, sh.red);
  kept = block_sum_d(kept, sh.red);
  if (tid == 0) { sh.part_tot = tot; sh.part_kept = kept; }
  cluster.sync();
  if (rank == 0 && tid == 0 && energy) {
    double T = 0.0, Kp = 0.0;
    for (int r = 0; r < kSelCluster; ++r) {
      T += cluster.map_shared_rank(&sh, r)->part_tot;
      Kp += cluster.map_shared_rank(&sh, r)->part_kept;
    }
    energy[c * 2 + 0] = T;
    energy[c * 2 + 1] = fmin(Kp, T);
  }
  cluster.sync();  // keep every CTA's shared memory alive until rank 0 has read it
  SEL_TRACE(28);
}

}  // namespace sss
