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

constexpr int kSelCluster = 8;

struct ClusterSelShared {
  unsigned hist[2048];
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
  const double* src = ehat + (size_t)c * n_dom;
  for (int i = tid; i < cnt_local; i += nt) v[i] = src[lo + i];
  const int n = min(n_keep, n_dom);
  __syncthreads();

  uint64_t prefix = 0, pmask = 0;
  long long need = n;
  const int digits[6] = {53, 42, 31, 20, 9, 0};
  const int widths[6] = {11, 11, 11, 11, 11, 9};
  if (n > 0) {
    for (int p = 0; p < 6; ++p) {
      const int shf = digits[p], nb = 1 << widths[p];
      for (int b = tid; b < nb; b += nt) sh.hist[b] = 0;
      __syncthreads();
      for (int i = tid; i < cnt_local; i += nt) {
        const uint64_t k = mkey(v[i]);
        if ((k & pmask) == prefix) atomicAdd(&sh.hist[(k >> shf) & (nb - 1)], 1u);
      }
      cluster.sync();
      if (rank == 0) {
        for (int b = tid; b < nb; b += nt) {
          unsigned s = 0;
          for (int r = 0; r < kSelCluster; ++r) s += cluster.map_shared_rank(sh.hist, r)[b];
          sh.merged[b] = s;
        }
        __syncthreads();
        // find_bucket over the merged histogram (reuse the generic routine
        // through a SelShared-shaped view of the scratch)
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
          if (tid == 0) {
            if (sh.scal_b < 0) {  // unreachable (cannot happen for counts): bucket 0
              uint64_t above = 0;
              for (int b = nb - 1; b > 0; --b) above += sh.merged[b];
              sh.scal_b = 0;
              sh.scal_need = need - (long long)above;
              sh.scal_cnt = sh.merged[0];
            }
            sh.dec_b[p & 1] = sh.scal_b;
            sh.dec_need[p & 1] = sh.scal_need;
            sh.dec_cnt[p & 1] = sh.scal_cnt;
          }
        }
      }
      cluster.sync();
      ClusterSelShared* s0 = cluster.map_shared_rank(&sh, 0);
      const int b = s0->dec_b[p & 1];
      need = s0->dec_need[p & 1];
      prefix |= (uint64_t)b << shf;
      pmask |= (uint64_t)(nb - 1) << shf;
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
  double tot = 0.0, kept = 0.0;
  double* xo = x + (size_t)c * n_dom;
  for (int i = a0; i < a1; ++i) {
    const double e = v[i];
    const uint64_t k = mkey(e);
    bool keep = k > t;
    if (k == t) { keep = tie_rank < take; ++tie_rank; }
    tot += e * e;
    if (keep) kept += e * e;
    const int gi = lo + i;
    xo[f2t ? f2t[gi] : gi] = keep ? e : 0.0;
    v[i] = keep ? 1.0 : 0.0;  // reuse as the keep flag for the mask words
  }
  __syncthreads();
  if (mask) {
    uint32_t* mo = mask + (size_t)c * ((n_dom + 31) / 32);
    for (int w = tid; w * 32 < cnt_local; w += nt) {
      uint32_t word = 0;
      for (int bb = 0; bb < 32 && w * 32 + bb < cnt_local; ++bb)
        word |= (v[w * 32 + bb] != 0.0 ? 1u : 0u) << bb;
      mo[(lo >> 5) + w] = word;
    }
  }
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
}

}  // namespace sss
