// Per-frame relight / material-edit path on sm_100a.
//
//   (a) light projection + w0 Haar   k_sh_irradiance_haar / k_env_*      (runtime.py:109-136)
//       exact-n selection            k_select_topn                       (wavelets.py:128-136)
//   (c) material weights g_k         k_material_weights                  (basisgen.py:172-191)
//   (b) transfer                     transfer.cu                         (runtime.py:138-150)
//   (c) recombine + inverse Haar + Fresnel shade, relight and edit
//                                    k_edit_finish_multi                 (runtime.py:152-216)
//
// Numerics: E, its Haar and the selection are fp64 with the reference's exact
// operation order (no FMA), so kept index sets are bit-identical to the CPU
// reference; transfer sums accumulate fp64 over f32 operator values
// (fp64 accumulation is what makes the 1e-4 criterion hold).
#include "select.cuh"

namespace sss {

// ---------------------------------------------------------------------------
// exact top-n selection over a shared-memory or global array of doubles
// (|x| descending, ties -> lower index), as compress_top_n
// ---------------------------------------------------------------------------

__device__ __forceinline__ uint64_t mag_key(double v) {
  return (uint64_t)__double_as_longlong(v) & 0x7fffffffffffffffULL;
}

// Block-wide radix select. Finds the key K* of the n-th largest element and
// the number `take_eq` of elements equal to K* (lowest indices first) to keep.
// `vals` may live in global or shared memory; count n_el. Requires blockDim
// a multiple of 32 and <= 1024. hist: 2048 uint32 in shared memory.
struct SelectResult {
  uint64_t key;       // threshold key
  int take_eq;        // how many elements with key == threshold are kept
};

__device__ SelectResult block_radix_select(const double* vals, int n_el, int n,
                                           unsigned* hist, int* sh_scalar) {
  const int tid = threadIdx.x, nt = blockDim.x;
  uint64_t prefix = 0, prefix_mask = 0;
  int need = n;  // elements still to take among candidates matching prefix
  const int digits[6] = {53, 42, 31, 20, 9, 0};
  const int widths[6] = {11, 11, 11, 11, 11, 9};
  for (int p = 0; p < 6; ++p) {
    const int sh = digits[p], w = widths[p], nb = 1 << w;
    for (int b = tid; b < nb; b += nt) hist[b] = 0;
    __syncthreads();
    for (int i = tid; i < n_el; i += nt) {
      const uint64_t k = mag_key(vals[i]);
      if ((k & prefix_mask) == prefix) atomicAdd(&hist[(k >> sh) & (nb - 1)], 1u);
    }
    __syncthreads();
    if (tid == 0) {
      int acc = 0, b = nb - 1;
      for (; b > 0; --b) {
        if (acc + (int)hist[b] >= need) break;
        acc += hist[b];
      }
      sh_scalar[0] = b;
      sh_scalar[1] = need - acc;  // still needed inside bucket b
    }
    __syncthreads();
    const int b = sh_scalar[0];
    need = sh_scalar[1];
    prefix |= (uint64_t)b << sh;
    prefix_mask |= (uint64_t)(nb - 1) << sh;
    __syncthreads();
  }
  SelectResult r;
  r.key = prefix;
  r.take_eq = need;
  return r;
}

// Block-wide exclusive rank, in index order, of elements with key == thr.
// Each thread handles a contiguous chunk of indices so the rank is in index
// order. Returns through `keep(i)` callback semantics: writes the selection
// decision via the supplied functor.
template <class F>
__device__ void block_apply_selection(const double* vals, int n_el, SelectResult sel,
                                      int* warp_sums, F&& on_elem) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int chunk = (n_el + nt - 1) / nt;
  const int lo = min(tid * chunk, n_el), hi = min(lo + chunk, n_el);
  int cnt = 0;
  for (int i = lo; i < hi; ++i) cnt += (mag_key(vals[i]) == sel.key);
  // block exclusive scan of cnt
  const int lane = tid & 31, wid = tid >> 5, nw = nt >> 5;
  int incl = cnt;
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) warp_sums[wid] = incl;
  __syncthreads();
  if (tid == 0) {
    int a = 0;
    for (int w = 0; w < nw; ++w) { const int t = warp_sums[w]; warp_sums[w] = a; a += t; }
  }
  __syncthreads();
  int rank = warp_sums[wid] + incl - cnt;
  for (int i = lo; i < hi; ++i) {
    const uint64_t k = mag_key(vals[i]);
    bool keep = k > sel.key;
    if (k == sel.key) { keep = rank < sel.take_eq; ++rank; }
    on_elem(i, keep);
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// (a) SH light projection fused with the w0 Haar of E
// ---------------------------------------------------------------------------

// grid: one CTA per 2^L x 2^L tile; T_l: (nl, N) l-major float32 transfer;
// Lsh: (nl, 3) doubles. Writes ehat (3, N) in global Mallat order, E (N, 3).
__global__ void k_sh_irradiance_haar(const float* __restrict__ T_l, const double* __restrict__ Lsh,
                                     int nl, int S, int L, double* __restrict__ E_out,
                                     double* __restrict__ ehat) {
  extern __shared__ double sm[];
  const int T = 1 << L, T2 = T * T;
  double* a = sm;            // 3 * T2
  double* tmp = sm + 3 * T2; // T2
  const int tiles_per_row = S / T;
  const int tr = blockIdx.x / tiles_per_row, tc = blockIdx.x % tiles_per_row;
  const int N = S * S;
  for (int e = threadIdx.x; e < T2; e += blockDim.x) {
    const int i = (tr * T + e / T) * S + tc * T + e % T;
    double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0;
    for (int l = 0; l < nl; ++l) {
      const double t = (double)T_l[(size_t)l * N + i];
      acc0 = dadd(acc0, dmul(t, Lsh[l * 3 + 0]));
      acc1 = dadd(acc1, dmul(t, Lsh[l * 3 + 1]));
      acc2 = dadd(acc2, dmul(t, Lsh[l * 3 + 2]));
    }
    a[e] = acc0; a[T2 + e] = acc1; a[2 * T2 + e] = acc2;
    if (E_out) { E_out[i * 3 + 0] = acc0; E_out[i * 3 + 1] = acc1; E_out[i * 3 + 2] = acc2; }
  }
  __syncthreads();
  for (int c = 0; c < 3; ++c) tile_haar_fwd(a + c * T2, tmp, T, blockDim.x, threadIdx.x);
  for (int e = threadIdx.x; e < T2; e += blockDim.x) {
    int gr, gc;
    local_to_global(e / T, e % T, tr, tc, L, S, &gr, &gc);
    const int g = gr * S + gc;
    ehat[g] = a[e]; ehat[N + g] = a[T2 + e]; ehat[2 * N + g] = a[2 * T2 + e];
  }
}

// ---------------------------------------------------------------------------
// (a) environment light: per-face full Haar + top-n_keep per channel
// (project_environment, lighting.py:293-305), then E = W^{w2} L^{w2}
// ---------------------------------------------------------------------------

// grid: 3 CTAs (channels), faces (6, s, s, 3) doubles
#ifdef SSS_ENV_TRACE
__device__ unsigned long long g_env_trace[16];
#define ENV_TRACE(i)                                                         \
  do {                                                                       \
    if (blockIdx.x == 0 && threadIdx.x == 0) {                               \
      unsigned long long t_;                                                 \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                 \
      g_env_trace[i] = t_;                                                   \
    }                                                                        \
  } while (0)
#else
#define ENV_TRACE(i) \
  do {               \
  } while (0)
#endif

// batch_tile_haar_fwd for the cubemap faces with the small levels (s <= 8)
// done by one warp per face under __syncwarp: the same arithmetic, six block
// barriers fewer (the pass count, not the work, bounds this transform)
__device__ inline void env_faces_haar_fwd(double* a, double* tmp, int T, int B) {
  constexpr int kTail = 8;
  const int T2 = T * T, nt = blockDim.x, tid = threadIdx.x;
  int s = T;
  for (; s > kTail; s >>= 1) {
    const int h = s >> 1, lh = ilog2i(h), lsh = ilog2i(s * h);
    for (int q = tid; q < (B << lsh); q += nt) {
      const int b = q >> lsh, e = q & ((1 << lsh) - 1);
      const int i = e >> lh, j = e & (h - 1);
      const double* g = a + b * T2;
      double* o = tmp + b * T2;
      const double ev = g[i * T + 2 * j], od = g[i * T + 2 * j + 1];
      o[i * T + j] = dmul(dadd(ev, od), SSS_ISQRT2);
      o[i * T + h + j] = dmul(dsub(ev, od), SSS_ISQRT2);
    }
    __syncthreads();
    for (int q = tid; q < (B << lsh); q += nt) {
      const int b = q >> lsh, e = q & ((1 << lsh) - 1);
      const int i = e >> (lh + 1), j = e & (2 * h - 1);  // j (of s) fastest: no bank conflicts
      const double* g = tmp + b * T2;
      double* o = a + b * T2;
      const double ev = g[(2 * i) * T + j], od = g[(2 * i + 1) * T + j];
      o[i * T + j] = dmul(dadd(ev, od), SSS_ISQRT2);
      o[(h + i) * T + j] = dmul(dsub(ev, od), SSS_ISQRT2);
    }
    __syncthreads();
  }
  const int warp = tid >> 5, lane = tid & 31;
  if (warp < B) {
    double* g = a + warp * T2;
    double* o = tmp + warp * T2;
    for (; s >= 2; s >>= 1) {
      const int h = s >> 1;
      for (int q = lane; q < s * h; q += 32) {
        const int i = q / h, j = q % h;
        const double ev = g[i * T + 2 * j], od = g[i * T + 2 * j + 1];
        o[i * T + j] = dmul(dadd(ev, od), SSS_ISQRT2);
        o[i * T + h + j] = dmul(dsub(ev, od), SSS_ISQRT2);
      }
      __syncwarp();
      for (int q = lane; q < s * h; q += 32) {
        const int i = q / s, j = q % s;
        const double ev = o[(2 * i) * T + j], od = o[(2 * i + 1) * T + j];
        g[i * T + j] = dmul(dadd(ev, od), SSS_ISQRT2);
        g[(h + i) * T + j] = dmul(dsub(ev, od), SSS_ISQRT2);
      }
      __syncwarp();
    }
  }
  __syncthreads();
}

// Selection state of k_env_project (one CTA, keys in registers).
struct EnvSelShared {
  unsigned hist[256];
  int scal_b, ncand, wsum[32];
  long long scal_need, scal_cnt, take, ties;
  uint64_t ckey[64], thr;
  double red[32], red2[32];
};

// grid: one CTA of 1024 threads per channel. Per-face full-pyramid Haar of the
// 6 x s x s cubemap (lighting.py:293-305), then the exact top-n_keep by
// magnitude (ties -> lower id) with a most-significant-digit radix descent on
// keys held in registers (each thread owns kEnvPer consecutive ids, so the
// ordered compaction is one block scan): three 8-bit passes, then the <= 64
// keys left in the threshold bucket are ranked directly.
constexpr int kEnvPer = 6;  // ids per thread: 1024 x 6 = the 6 x 32 x 32 cubemap
__global__ void __launch_bounds__(1024) k_env_project(const double* __restrict__ faces, int s,
                                                      int n_keep, uint32_t* __restrict__ idx_out,
                                                      double* __restrict__ val_out,
                                                      double* __restrict__ energy) {
  extern __shared__ __align__(16) double sm[];
  const int c = blockIdx.x, s2 = s * s, D = 6 * s2;
  double* a = sm;             // D
  double* tmp = sm + D;       // D (the 6 faces transform as one batch)
  EnvSelShared& sh = *reinterpret_cast<EnvSelShared*>(tmp + D);
  pdl_launch_dependents();
  pdl_wait();
  ENV_TRACE(0);
  for (int e = threadIdx.x; e < D; e += blockDim.x) a[e] = faces[(size_t)e * 3 + c];
  __syncthreads();
  ENV_TRACE(1);
  env_faces_haar_fwd(a, tmp, s, 6);
  ENV_TRACE(2);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int n = min(n_keep, D);
  const int lo = min(tid * kEnvPer, D), cnt_own = min(kEnvPer, D - lo);
  double v[kEnvPer];
  uint64_t key[kEnvPer];
#pragma unroll
  for (int j = 0; j < kEnvPer; ++j) {
    v[j] = j < cnt_own ? a[lo + j] : 0.0;
    key[j] = mkey(v[j]);
  }
  uint64_t prefix = 0, pmask = 0;
  long long need = n, ties = 0;
  for (int p = 0; p < 8 && n > 0; ++p) {
    const int shf = 56 - 8 * p;
    if (tid < 256) sh.hist[tid] = 0u;
    if (tid == 0) { sh.scal_b = 0; sh.scal_need = need; sh.scal_cnt = 0; sh.ncand = 0; }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kEnvPer; ++j) {
      unsigned bin = 0xffffffffu;
      if (j < cnt_own && (key[j] & pmask) == prefix) bin = (unsigned)(key[j] >> shf) & 255u;
      if (p == 0) {  // the top digit takes a handful of values: aggregate per warp
        const unsigned peers = __match_any_sync(0xffffffffu, bin);
        if (bin != 0xffffffffu && lane == __ffs(peers) - 1) atomicAdd(&sh.hist[bin], __popc(peers));
      } else if (bin != 0xffffffffu) {
        atomicAdd(&sh.hist[bin], 1u);
      }
    }
    __syncthreads();
    if (wid == 0) {  // lane l: bins 255 - 8l .. 248 - 8l, scanned from the top
      unsigned h[8], ssum = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) { h[q] = sh.hist[255 - 8 * lane - q]; ssum += h[q]; }
      unsigned incl = ssum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      long long before = (long long)(incl - ssum);
      if (before < need && need <= before + (long long)ssum) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          if (before + (long long)h[q] >= need) {
            sh.scal_b = 255 - 8 * lane - q;
            sh.scal_need = need - before;
            sh.scal_cnt = h[q];
            break;
          }
          before += h[q];
        }
      }
    }
    __syncthreads();
    const int bsel = sh.scal_b;
    need = sh.scal_need;
    ties = sh.scal_cnt;
    prefix |= (uint64_t)bsel << shf;
    pmask |= (uint64_t)255u << shf;
    if (p < 7 && ties <= 64) {
#pragma unroll
      for (int j = 0; j < kEnvPer; ++j)
        if (j < cnt_own && (key[j] & pmask) == prefix) sh.ckey[atomicAdd(&sh.ncand, 1)] = key[j];
      __syncthreads();
      const int total = sh.ncand;
      if (tid < total) {
        const uint64_t kj = sh.ckey[tid];
        long long g = 0, e = 0;
        for (int q = 0; q < total; ++q) {
          g += sh.ckey[q] > kj;
          e += sh.ckey[q] == kj;
        }
        if (g < need && need <= g + e) {  // equal keys write equal values
          sh.thr = kj;
          sh.take = need - g;
          sh.ties = e;
        }
      }
      __syncthreads();
      prefix = sh.thr;
      need = sh.take;
      ties = sh.ties;
      break;
    }
  }
  ENV_TRACE(3);
  const uint64_t t = n > 0 ? prefix : ~0ULL;
  const long long take = n > 0 ? need : 0;
  const bool all_ties = take == ties;  // every key equal to the threshold is kept
  int tie_rank = 0;
  if (!all_ties) {  // some ties kept: the lowest ids first (block scan of the tie counts)
    int my = 0;
#pragma unroll
    for (int j = 0; j < kEnvPer; ++j) my += (j < cnt_own && key[j] == t);
    int incl = my;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    __syncthreads();
    if (lane == 31) sh.wsum[wid] = incl;
    __syncthreads();
    int base = 0;
    for (int w = 0; w < wid; ++w) base += sh.wsum[w];
    tie_rank = base + incl - my;
    __syncthreads();
  }
  unsigned kb = 0;
  int cnt = 0;
#pragma unroll
  for (int j = 0; j < kEnvPer; ++j) {
    if (j >= cnt_own) break;
    bool keep = all_ties ? key[j] >= t : key[j] > t;
    if (!all_ties && key[j] == t) { keep = tie_rank < take; ++tie_rank; }
    kb |= (keep ? 1u : 0u) << j;
    cnt += keep;
  }
  ENV_TRACE(4);
  // ordered compaction: exclusive block scan of the kept counts
  int incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) sh.wsum[wid] = incl;
  __syncthreads();
  int pos = incl - cnt;
  for (int w = 0; w < wid; ++w) pos += sh.wsum[w];
#pragma unroll
  for (int j = 0; j < kEnvPer; ++j)
    if ((kb >> j) & 1u) {
      idx_out[c * n_keep + pos] = (uint32_t)(lo + j);
      val_out[c * n_keep + pos] = v[j];
      ++pos;
    }
  for (int q = n + tid; q < n_keep; q += blockDim.x) {
    idx_out[c * n_keep + q] = 0xffffffffu;
    val_out[c * n_keep + q] = 0.0;
  }
  ENV_TRACE(5);
  if (energy) {
    double tot = 0.0, kept = 0.0;
#pragma unroll
    for (int j = 0; j < kEnvPer; ++j) {
      tot += v[j] * v[j];
      if ((kb >> j) & 1u) kept += v[j] * v[j];
    }
    for (int o = 16; o > 0; o >>= 1) {
      tot += __shfl_xor_sync(0xffffffffu, tot, o);
      kept += __shfl_xor_sync(0xffffffffu, kept, o);
    }
    __syncthreads();
    if (lane == 0) { sh.red[wid] = tot; sh.red2[wid] = kept; }
    __syncthreads();
    if (tid == 0) {
      double T = 0.0, Kp = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { T += sh.red[w]; Kp += sh.red2[w]; }
      energy[c * 2 + 0] = T;
      energy[c * 2 + 1] = fmin(Kp, T);
    }
  }
}

// one thread: ascending union of the three channels' kept w2 ids with the
// per-channel value (0 where the channel dropped the id)
__global__ void __launch_bounds__(1024) k_env_union(const uint32_t* __restrict__ idx,
                                                    const double* __restrict__ val, int n_keep, int D,
                                                    uint32_t* __restrict__ union_idx,
                                                    double* __restrict__ union_lc,
                                                    int* __restrict__ n_union) {
  // parallel: mark the kept ids of every channel in a D-long flag array, then
  // an index-order block scan compacts the ascending union (D <= 6144)
  __shared__ unsigned char flag[6144];
  __shared__ unsigned short pos[3][6144];
  __shared__ int wsum[32];
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int i = tid; i < D; i += nt) flag[i] = 0;
  __syncthreads();
  for (int e = tid; e < 3 * n_keep; e += nt) {
    const int c = e / n_keep, q = e % n_keep;
    const uint32_t id = idx[e];
    if (id < (uint32_t)D) {
      atomicOr(reinterpret_cast<unsigned*>(flag) + (id >> 2), 1u << (8 * (id & 3) + c));
      pos[c][id] = (unsigned short)q;
    }
  }
  __syncthreads();
  const int chunk = (D + nt - 1) / nt;
  const int lo = min(tid * chunk, D), hi = min(lo + chunk, D);
  int cnt = 0;
  for (int i = lo; i < hi; ++i) cnt += flag[i] != 0;
  const int lane = tid & 31, wid = tid >> 5, nw = nt >> 5;
  int incl = cnt;
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) wsum[wid] = incl;
  __syncthreads();
  if (tid == 0) {
    int a = 0;
    for (int w = 0; w < nw; ++w) { const int t = wsum[w]; wsum[w] = a; a += t; }
    *n_union = a;
  }
  __syncthreads();
  int m = wsum[wid] + incl - cnt;
  for (int i = lo; i < hi; ++i) {
    const unsigned f = flag[i];
    if (!f) continue;
    union_idx[m] = (uint32_t)i;
    for (int c = 0; c < 3; ++c)
      union_lc[m * 3 + c] = ((f >> c) & 1u) ? val[c * n_keep + pos[c][i]] : 0.0;
    ++m;
  }
}

// grid: one CTA per tile. W2: (D, N) float32 l-major (w2 coefficient major).
// E_i,c = sum over the ascending union of the three kept w2 id lists of
// W2[l, i] * L_c[l]   (zero where channel c dropped l), fp64 exact order.
__global__ void k_env_irradiance_haar(const float* __restrict__ W2, int D,
                                      const uint32_t* __restrict__ union_idx,
                                      const double* __restrict__ union_lc, const int* __restrict__ n_union,
                                      int n_keep, int S, int L, double* __restrict__ E_out,
                                      double* __restrict__ ehat) {
  extern __shared__ double sm[];
  const int T = 1 << L, T2 = T * T;
  double* a = sm;                  // 3*T2
  double* tmp = sm + 3 * T2;       // T2
  double* lc = tmp + T2;           // 3 * 3*n_keep
  int* ul = (int*)(lc + 9 * n_keep);   // union list (<= 3*n_keep)
  const int N = S * S;
  // union list + per-channel weights precomputed by k_env_union
  const int m = *n_union;
  for (int q = threadIdx.x; q < m; q += blockDim.x) {
    ul[q] = (int)union_idx[q];
    lc[q * 3] = union_lc[q * 3]; lc[q * 3 + 1] = union_lc[q * 3 + 1]; lc[q * 3 + 2] = union_lc[q * 3 + 2];
  }
  __syncthreads();

  const int tiles_per_row = S / T;
  const int tr = blockIdx.x / tiles_per_row, tc = blockIdx.x % tiles_per_row;
  for (int e = threadIdx.x; e < T2; e += blockDim.x) {
    const int i = (tr * T + e / T) * S + tc * T + e % T;
    double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0;
    constexpr int kPf = 8;  // independent loads in flight; the adds stay in l order
    for (int q0 = 0; q0 < m; q0 += kPf) {
      float wv[kPf];
#pragma unroll
      for (int u = 0; u < kPf; ++u)
        wv[u] = (q0 + u < m) ? __ldg(&W2[(size_t)ul[q0 + u] * N + i]) : 0.0f;
#pragma unroll
      for (int u = 0; u < kPf; ++u) {
        if (q0 + u >= m) break;
        const int q = q0 + u;
        const double w = (double)wv[u];
        const double l0 = lc[q * 3], l1 = lc[q * 3 + 1], l2 = lc[q * 3 + 2];
        if (l0 != 0.0) acc0 = dadd(acc0, dmul(w, l0));
        if (l1 != 0.0) acc1 = dadd(acc1, dmul(w, l1));
        if (l2 != 0.0) acc2 = dadd(acc2, dmul(w, l2));
      }
    }
    a[e] = acc0; a[T2 + e] = acc1; a[2 * T2 + e] = acc2;
    if (E_out) { E_out[i * 3 + 0] = acc0; E_out[i * 3 + 1] = acc1; E_out[i * 3 + 2] = acc2; }
  }
  __syncthreads();
  for (int c = 0; c < 3; ++c) tile_haar_fwd(a + c * T2, tmp, T, blockDim.x, threadIdx.x);
  for (int e = threadIdx.x; e < T2; e += blockDim.x) {
    int gr, gc;
    local_to_global(e / T, e % T, tr, tc, L, S, &gr, &gc);
    const int g = gr * S + gc;
    ehat[g] = a[e]; ehat[N + g] = a[T2 + e]; ehat[2 * N + g] = a[2 * T2 + e];
  }
}

// Multi-tile versions of the two light-projection kernels: TPB tiles per CTA,
// one thread per point (blockDim = TPB * 4^L), deeper load prefetch, one
// batched forward Haar for the 3 * TPB grids. Same arithmetic and summation
// order as above (bitwise-identical E and ehat).
__device__ __forceinline__ void scatter_ehat(const double* a, int T, int TPB, int tile0, int L,
                                             int S, double* __restrict__ ehat) {
  const int T2 = T * T, N = S * S, tpr = S / T;
  for (int q = threadIdx.x; q < TPB * T2; q += blockDim.x) {
    const int j = q / T2, e = q % T2;
    const int tile = tile0 + j;
    int gr, gc;
    local_to_global(e / T, e % T, tile / tpr, tile % tpr, L, S, &gr, &gc);
    const int g = gr * S + gc;
    ehat[g] = a[(j * 3 + 0) * T2 + e];
    ehat[N + g] = a[(j * 3 + 1) * T2 + e];
    ehat[2 * N + g] = a[(j * 3 + 2) * T2 + e];
  }
}

// union_idx != nullptr: the ascending union of the three channels' kept w2
// ids and their per-channel values come from k_env_union. union_idx ==
// nullptr: every CTA builds the same union itself from the per-channel kept
// lists sel_idx / sel_val (3 x n_keep, k_env_project's output): flags over the
// D ids, a word prefix, each kept id's rank = its union position (ascending),
// the value of a channel that dropped the id = 0 (k_env_union's rule).
__global__ void k_env_irradiance_multi(const float* __restrict__ W2,
                                       const uint32_t* __restrict__ union_idx,
                                       const double* __restrict__ union_lc,
                                       const int* __restrict__ n_union, int n_keep, int S, int L,
                                       int TPB, double* __restrict__ E_out,
                                       double* __restrict__ ehat,
                                       const uint32_t* __restrict__ sel_idx = nullptr,
                                       const double* __restrict__ sel_val = nullptr, int D = 0) {
  extern __shared__ double sm[];
  __shared__ int s_m;
  const int T = 1 << L, T2 = T * T, N = S * S, tpr = S / T;
  double* a = sm;                       // TPB * 3 * T2
  double* tmp = a + TPB * 3 * T2;       // TPB * 3 * T2
  double* lc = tmp + TPB * 3 * T2;      // 3 n_keep x 4 (l0, l1, l2, 0): one 16-B + one 8-B LDS
  int* ul = reinterpret_cast<int*>(lc + 12 * n_keep);
  if (union_idx) {
    const int mm = *n_union;
    for (int q = threadIdx.x; q < mm; q += blockDim.x) {
      ul[q] = (int)union_idx[q];
      lc[q * 4] = union_lc[q * 3]; lc[q * 4 + 1] = union_lc[q * 3 + 1];
      lc[q * 4 + 2] = union_lc[q * 3 + 2]; lc[q * 4 + 3] = 0.0;
    }
    if (threadIdx.x == 0) s_m = mm;
  } else {
    const int nw = (D + 31) >> 5;
    uint32_t* flag = reinterpret_cast<uint32_t*>(ul + 3 * n_keep);
    uint32_t* wpre = flag + nw;
    for (int w = threadIdx.x; w < nw; w += blockDim.x) flag[w] = 0u;
    for (int q = threadIdx.x; q < 12 * n_keep; q += blockDim.x) lc[q] = 0.0;
    __syncthreads();
    for (int e = threadIdx.x; e < 3 * n_keep; e += blockDim.x) {
      const uint32_t id = sel_idx[e];
      if (id < (uint32_t)D) atomicOr(&flag[id >> 5], 1u << (id & 31u));
    }
    __syncthreads();
    if (threadIdx.x < 32) {  // exclusive word prefix (<= 32 words per lane)
      const int lane = threadIdx.x, per = (nw + 31) >> 5;
      const int w0 = lane * per, w1 = min(w0 + per, nw);
      int cnt = 0;
      for (int w = w0; w < w1; ++w) cnt += __popc(flag[w]);
      int inc = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
      }
      int run = inc - cnt;
      for (int w = w0; w < w1; ++w) { wpre[w] = (uint32_t)run; run += __popc(flag[w]); }
      if (lane == 31) s_m = inc;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < 3 * n_keep; e += blockDim.x) {
      const uint32_t id = sel_idx[e];
      if (id >= (uint32_t)D) continue;
      const int c = e / n_keep;
      const int pos = (int)(wpre[id >> 5] + __popc(flag[id >> 5] & ((1u << (id & 31u)) - 1u)));
      ul[pos] = (int)id;
      lc[pos * 4 + c] = sel_val[e];
    }
  }
  __syncthreads();
  const int m = s_m;
  const int tile0 = blockIdx.x * TPB;
  for (int q = threadIdx.x; q < TPB * T2; q += blockDim.x) {
    // the CTA's TPB tiles are horizontally adjacent: consecutive threads walk
    // one image row across them, so a warp's W^{w2} loads are whole lines
    const int rr = q / (TPB * T), cc = q % (TPB * T);
    const int j = cc / T, e = rr * T + cc % T;
    const int tile = tile0 + j, tr = tile / tpr, tc = tile % tpr;
    const int i = (tr * T + e / T) * S + tc * T + e % T;
    double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0;
    // W^{w2} loads: one batch of kPf in flight while the previous batch is
    // summed (the order of the sum is fixed: ascending union position)
    constexpr int kPf = 32;
    float wv[kPf], wn[kPf];
#pragma unroll
    for (int u = 0; u < kPf; ++u) wn[u] = (u < m) ? __ldg(&W2[(size_t)ul[u] * N + i]) : 0.0f;
    for (int q0 = 0; q0 < m; q0 += kPf) {
#pragma unroll
      for (int u = 0; u < kPf; ++u) wv[u] = wn[u];
#pragma unroll
      for (int u = 0; u < kPf; ++u)
        wn[u] = (q0 + kPf + u < m) ? __ldg(&W2[(size_t)ul[q0 + kPf + u] * N + i]) : 0.0f;
      // a channel that dropped the id has l = 0: w * 0 adds an exact zero, so
      // the sums equal the per-channel ones of the reference (value-equal)
#pragma unroll
      for (int u = 0; u < kPf; ++u) {
        if (q0 + u >= m) break;
        const int qq = q0 + u;
        const double w = (double)wv[u];
        const double2 l01 = *reinterpret_cast<const double2*>(lc + qq * 4);
        const double l2 = lc[qq * 4 + 2];
        acc0 = dadd(acc0, dmul(w, l01.x));
        acc1 = dadd(acc1, dmul(w, l01.y));
        acc2 = dadd(acc2, dmul(w, l2));
      }
    }
    a[(j * 3 + 0) * T2 + e] = acc0;
    a[(j * 3 + 1) * T2 + e] = acc1;
    a[(j * 3 + 2) * T2 + e] = acc2;
    if (E_out) { E_out[i * 3 + 0] = acc0; E_out[i * 3 + 1] = acc1; E_out[i * 3 + 2] = acc2; }
  }
  __syncthreads();
  batch_tile_haar_fwd(a, tmp, T, 3 * TPB);
  scatter_ehat(a, T, TPB, tile0, L, S, ehat);
}

// The frame's environment irradiance, one thread per (point, channel): channel
// c sums W^{w2}[l, i] * L_c[l] over ITS OWN kept w2 ids in ascending order - the
// reference's per-channel sum (lighting.py:318-336 on the compress_top_n
// spectrum), and value-equal to the union form above, whose extra terms are
// exact zeros. Three times the threads of the per-point form (the sums are
// sequential, so threads are the only parallelism) for 128 instead of ~300
// terms each, and no union to build. The kept lists are staged as 32-bit row
// offsets (id * N < 2^32) and padded to a multiple of 8 with (row 0, L = 0),
// whose products add exact zeros after the last real term: the loop is
// branch-free, 8 loads in flight per thread. blockDim = 3 * TPB * 4^L.
__global__ void __launch_bounds__(768, 2) k_env_irradiance_chan(
    const float* __restrict__ W2, const uint32_t* __restrict__ sel_idx,
    const double* __restrict__ sel_val, int n_keep, int D, int S, int L, int TPB,
    double* __restrict__ E_out, double* __restrict__ ehat) {
  extern __shared__ __align__(16) double sm[];
  pdl_launch_dependents();
  const int T = 1 << L, T2 = T * T, N = S * S, tpr = S / T, P = TPB * T2;
  const int nk8 = (n_keep + 7) & ~7;
  double* a = sm;                   // TPB * 3 * T2
  double* tmp = a + 3 * P;          // TPB * 3 * T2
  double* lv = tmp + 3 * P;         // 3 nk8 kept values
  uint32_t* roff = reinterpret_cast<uint32_t*>(lv + 3 * nk8);  // 3 nk8 row offsets id * N
  pdl_wait();
  for (int e = threadIdx.x; e < 3 * nk8; e += blockDim.x) {
    const int c = e / nk8, q = e % nk8;
    const uint32_t id = q < n_keep ? sel_idx[c * n_keep + q] : 0xffffffffu;
    const bool ok = id < (uint32_t)D;
    roff[e] = ok ? id * (uint32_t)N : 0u;
    lv[e] = ok ? sel_val[c * n_keep + q] : 0.0;
  }
  __syncthreads();
  const int tile0 = blockIdx.x * TPB;
  const int lB = 31 - __clz(TPB), lP = lB + 2 * L, ltpr = 31 - __clz(tpr);
  for (int t = threadIdx.x; t < 3 * P; t += blockDim.x) {
    // the CTA's TPB tiles are horizontally adjacent: consecutive threads walk
    // one image row across them, so a warp's W^{w2} loads are whole lines
    // TPB, T, S are powers of two (the launcher enforces it): shifts, not divisions
    const int c = t >> lP, q = t & (P - 1);
    const int rr = q >> (lB + L), cc = q & ((TPB << L) - 1);
    const int j = cc >> L, e = (rr << L) + (cc & (T - 1));
    const int tile = tile0 + j, tr = tile >> ltpr, tc = tile & (tpr - 1);
    const uint32_t i = (uint32_t)((tr * T + rr) * S + tc * T + (cc & (T - 1)));
    const uint32_t* ro = roff + c * nk8;
    const double* lc = lv + c * nk8;
    double acc = 0.0;
#pragma unroll 2
    for (int q0 = 0; q0 < nk8; q0 += 8) {
      const uint4 r0 = *reinterpret_cast<const uint4*>(ro + q0);
      const uint4 r1 = *reinterpret_cast<const uint4*>(ro + q0 + 4);
      float w[8];
      w[0] = __ldg(W2 + (r0.x + i)); w[1] = __ldg(W2 + (r0.y + i));
      w[2] = __ldg(W2 + (r0.z + i)); w[3] = __ldg(W2 + (r0.w + i));
      w[4] = __ldg(W2 + (r1.x + i)); w[5] = __ldg(W2 + (r1.y + i));
      w[6] = __ldg(W2 + (r1.z + i)); w[7] = __ldg(W2 + (r1.w + i));
#pragma unroll
      for (int u = 0; u < 8; u += 2) {
        const double2 l = *reinterpret_cast<const double2*>(lc + q0 + u);
        acc = dadd(acc, dmul((double)w[u], l.x));
        acc = dadd(acc, dmul((double)w[u + 1], l.y));
      }
    }
    a[(j * 3 + c) * T2 + e] = acc;
    if (E_out) E_out[i * 3 + c] = acc;
  }
  __syncthreads();
  batch_tile_haar_fwd(a, tmp, T, 3 * TPB);
  scatter_ehat(a, T, TPB, tile0, L, S, ehat);
}

__global__ void k_sh_irradiance_multi(const float* __restrict__ T_l, const double* __restrict__ Lsh,
                                      int nl, int S, int L, int TPB, double* __restrict__ E_out,
                                      double* __restrict__ ehat) {
  extern __shared__ double sm[];
  const int T = 1 << L, T2 = T * T, N = S * S, tpr = S / T;
  double* a = sm;                  // TPB * 3 * T2
  double* tmp = a + TPB * 3 * T2;  // TPB * 3 * T2
  const int tile0 = blockIdx.x * TPB;
  for (int q = threadIdx.x; q < TPB * T2; q += blockDim.x) {
    const int j = q / T2, e = q % T2;
    const int tile = tile0 + j, tr = tile / tpr, tc = tile % tpr;
    const int i = (tr * T + e / T) * S + tc * T + e % T;
    double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0;
    for (int l = 0; l < nl; ++l) {
      const double t = (double)__ldg(&T_l[(size_t)l * N + i]);
      acc0 = dadd(acc0, dmul(t, Lsh[l * 3 + 0]));
      acc1 = dadd(acc1, dmul(t, Lsh[l * 3 + 1]));
      acc2 = dadd(acc2, dmul(t, Lsh[l * 3 + 2]));
    }
    a[(j * 3 + 0) * T2 + e] = acc0;
    a[(j * 3 + 1) * T2 + e] = acc1;
    a[(j * 3 + 2) * T2 + e] = acc2;
    if (E_out) { E_out[i * 3 + 0] = acc0; E_out[i * 3 + 1] = acc1; E_out[i * 3 + 2] = acc2; }
  }
  __syncthreads();
  batch_tile_haar_fwd(a, tmp, T, 3 * TPB);
  scatter_ehat(a, T, TPB, tile0, L, S, ehat);
}

// ---------------------------------------------------------------------------
// exact top-n of the irradiance spectrum per channel (runtime.py:112-118)
// grid: 3 CTAs x 1024 threads. x = ehat where kept, else 0.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) k_select_topn(const double* __restrict__ ehat, int n_dom, int n_keep,
                                                      const uint32_t* __restrict__ f2t,
                                                      double* __restrict__ x, uint32_t* __restrict__ mask,
                                                      double* __restrict__ energy) {
  extern __shared__ __align__(16) unsigned char dsm[];
  SelShared& sh = *reinterpret_cast<SelShared*>(dsm);
  const int c = blockIdx.x;
  const double* v = ehat + (size_t)c * n_dom;
  const int n = min(n_keep, n_dom);
  SelectResult sel;
  sel.key = ~0ULL;
  sel.take_eq = 0;
  if (n > 0) {
    uint64_t t;
    long long take, tiecnt;
    radix_cut<false>(v, n_dom, n, 0.0, sh, &t, &take, &tiecnt);
    sel.key = t;
    sel.take_eq = (int)take;
  }
  ENV_TRACE(3);
  double tot = 0.0, kept = 0.0;
  double* xo = x + (size_t)c * n_dom;
  uint32_t* mo = mask ? mask + (size_t)c * ((n_dom + 31) / 32) : nullptr;
  // x is written in the operator's column space: tile-major when f2t is given
  block_apply_selection(v, n_dom, sel, reinterpret_cast<int*>(sh.wsum), [&](int i, bool k) {
    const double e = v[i];
    tot += e * e;
    if (k) kept += e * e;
    xo[f2t ? f2t[i] : i] = k ? e : 0.0;
    if (mo && k) atomicOr(&mo[i >> 5], 1u << (i & 31));
  });
  tot = block_sum_d(tot, sh.red);
  kept = block_sum_d(kept, sh.red);
  if (threadIdx.x == 0 && energy) {
    energy[c * 2 + 0] = tot;
    energy[c * 2 + 1] = fmin(kept, tot);
  }
}

// ---------------------------------------------------------------------------
// (c) material weights g[c][k] = sum_j w_j b_k(r_j) R_d(r_j; sigma_c, eta)
// grid: 3 CTAs (channel) x 512 threads
// ---------------------------------------------------------------------------
__global__ void k_material_weights(const double* __restrict__ bw /* K x nr: bases * w */,
                                   const double* __restrict__ r_nodes, int K, int nr,
                                   const double* __restrict__ material /* sp[3], sa[3], eta */,
                                   double* __restrict__ g) {
  // all K dot products in one pass: per-thread partials for every k, one
  // warp reduction per k, one barrier (K <= 16)
  __shared__ double red[32][16];
  const int c = blockIdx.x;
  const Dipole d = derive_dipole(material[c], material[3 + c], material[6]);
  double part[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) part[k] = 0.0;
  for (int j = threadIdx.x; j < nr; j += blockDim.x) {
    const double rd = eval_rd(d, r_nodes[j]);
#pragma unroll
    for (int k = 0; k < 16; ++k)
      if (k < K) part[k] += bw[k * nr + j] * rd;
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    if (k >= K) break;
    double a = part[k];
    for (int o = 16; o > 0; o >>= 1) a += __shfl_down_sync(0xffffffffu, a, o);
    if (lane == 0) red[wid][k] = a;
  }
  __syncthreads();
  if (threadIdx.x < K) {
    double s = 0.0;
    for (int w = 0; w < nw; ++w) s += red[w][threadIdx.x];
    g[c * K + threadIdx.x] = s;
  }
}

// ---------------------------------------------------------------------------
// epilogue shared by relight and edit: summed (3, T2) in smem, tile local
// Mallat layout -> inverse Haar -> Fresnel exit shade -> radiance
// ---------------------------------------------------------------------------
__device__ void tile_epilogue(double* summed, double* tmp, int T, int tr, int tc, int S,
                              const float* __restrict__ positions, const float* __restrict__ normals,
                              const double* __restrict__ cam, const double* __restrict__ material,
                              double* __restrict__ scatter, float* __restrict__ radiance,
                              float* __restrict__ radiance_unclamped) {
  const int T2 = T * T;
  const double eta = material[6];
  for (int c = 0; c < 3; ++c) tile_haar_inv(summed + c * T2, tmp, T, blockDim.x, threadIdx.x);
  const double inv_pi = 1.0 / 3.141592653589793;
  for (int e = threadIdx.x; e < T2; e += blockDim.x) {
    const int i = (tr * T + e / T) * S + tc * T + e % T;
    const double px = positions[i * 3], py = positions[i * 3 + 1], pz = positions[i * 3 + 2];
    double vx = cam[0] - px, vy = cam[1] - py, vz = cam[2] - pz;
    const double inv = 1.0 / sqrt(vx * vx + vy * vy + vz * vz);
    vx *= inv; vy *= inv; vz *= inv;
    const double cs = (double)normals[i * 3] * vx + (double)normals[i * 3 + 1] * vy +
                      (double)normals[i * 3 + 2] * vz;
    const double f = fresnel_transmittance(eta, cs) * inv_pi;
    for (int c = 0; c < 3; ++c) {
      const double sc = summed[c * T2 + e];
      const double u = sc * f;
      if (scatter) scatter[i * 3 + c] = sc;
      radiance_unclamped[i * 3 + c] = (float)u;
      radiance[i * 3 + c] = (float)fmax(u, 0.0);
    }
  }
}

// the same epilogue for `ntiles` consecutive tiles (tile0..) at once:
// summed is [tile][c][T2]; one batched inverse Haar over all 3*ntiles grids
__device__ void multi_tile_epilogue(double* summed, double* tmp, int T, int tile0, int ntiles,
                                    int S, const float* __restrict__ positions,
                                    const float* __restrict__ normals,
                                    const double* __restrict__ cam,
                                    const double* __restrict__ material,
                                    double* __restrict__ scatter, float* __restrict__ radiance,
                                    float* __restrict__ radiance_unclamped,
                                    double* __restrict__ rad64 = nullptr) {
  const int T2 = T * T, tpr = S / T;
  const double eta = material[6];
  const size_t n3 = (size_t)3 * S * S;
  batch_tile_haar_inv(summed, tmp, T, 3 * ntiles);
  const double inv_pi = 1.0 / 3.141592653589793;
  for (int q = threadIdx.x; q < ntiles * T2; q += blockDim.x) {
    const int j = q / T2, e = q % T2;
    const int tile = tile0 + j, tr = tile / tpr, tc = tile % tpr;
    const int i = (tr * T + e / T) * S + tc * T + e % T;
    const double px = positions[i * 3], py = positions[i * 3 + 1], pz = positions[i * 3 + 2];
    double vx = cam[0] - px, vy = cam[1] - py, vz = cam[2] - pz;
    const double inv = 1.0 / sqrt(vx * vx + vy * vy + vz * vz);
    vx *= inv; vy *= inv; vz *= inv;
    const double cs = (double)normals[i * 3] * vx + (double)normals[i * 3 + 1] * vy +
                      (double)normals[i * 3 + 2] * vz;
    const double f = fresnel_transmittance(eta, cs) * inv_pi;
    for (int c = 0; c < 3; ++c) {
      const double sc = summed[(j * 3 + c) * T2 + e];
      const double u = sc * f;
      if (scatter) scatter[i * 3 + c] = sc;
      const float uf = (float)u, cf = (float)fmax(u, 0.0);
      radiance_unclamped[i * 3 + c] = uf;
      radiance[i * 3 + c] = cf;
      if (rad64) {  // the API's float64 FrameResult pair (k_widen_frame's output)
        rad64[i * 3 + c] = (double)cf;
        rad64[n3 + i * 3 + c] = (double)uf;
      }
    }
  }
}

// edit path: stages 3-5 against the cached v_k
__global__ void k_edit_finish(int K, int S, int L, const double* __restrict__ vk,
                              const double* __restrict__ g, const float* __restrict__ positions,
                              const float* __restrict__ normals, const double* __restrict__ cam,
                              const double* __restrict__ material, double* __restrict__ scatter,
                              float* __restrict__ radiance,
                              float* __restrict__ radiance_unclamped) {
  extern __shared__ double sm[];
  const int T = 1 << L, T2 = T * T, N = S * S;
  double* summed = sm;
  double* tmp = sm + 3 * T2;
  const int tile = blockIdx.x;
  const int tiles_per_row = S / T;
  const int tr = tile / tiles_per_row, tc = tile % tiles_per_row;
  for (int e = threadIdx.x; e < T2; e += blockDim.x) {
    const int row = tile * T2 + e;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
    for (int k = 0; k < K; ++k) {
      const double* vo = vk + (size_t)k * 3 * N;
      s0 += g[k] * vo[row];
      s1 += g[K + k] * vo[N + row];
      s2 += g[2 * K + k] * vo[2 * N + row];
    }
    summed[e] = s0; summed[T2 + e] = s1; summed[2 * T2 + e] = s2;
  }
  __syncthreads();
  tile_epilogue(summed, tmp, T, tr, tc, S, positions, normals, cam, material, scatter, radiance,
                radiance_unclamped);
}


// edit path, G consecutive tiles per CTA: recombine (coalesced v_k reads over
// G * T2 rows), one batched inverse Haar over the 3G tile grids, shade
__global__ void __launch_bounds__(256) k_edit_finish_multi(
    int K, int S, int L, int G, const double* __restrict__ vk, const double* __restrict__ g,
    const float* __restrict__ positions, const float* __restrict__ normals,
    const double* __restrict__ cam, const double* __restrict__ material,
    double* __restrict__ scatter, float* __restrict__ radiance,
    float* __restrict__ radiance_unclamped, double* __restrict__ rad64) {
  extern __shared__ double sm[];
  const int T = 1 << L, T2 = T * T, N = S * S;
  double* summed = sm;                        // G x 3 x T2
  double* tmp = sm + (size_t)G * 3 * T2;      // same
  const int tile0 = blockIdx.x * G;
  pdl_launch_dependents();
  pdl_wait();
  for (int q = threadIdx.x; q < G * T2; q += blockDim.x) {
    const int row = tile0 * T2 + q;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
    // eight terms' v_k loads in flight at once; the sums keep their k order
    for (int k0 = 0; k0 < K; k0 += 8) {
      double v[8][3];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const double* vo = vk + (size_t)(k0 + u) * 3 * N;
        const bool in = k0 + u < K;
        v[u][0] = in ? __ldcs(&vo[row]) : 0.0;
        v[u][1] = in ? __ldcs(&vo[N + row]) : 0.0;
        v[u][2] = in ? __ldcs(&vo[2 * N + row]) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (k0 + u >= K) break;
        s0 += g[k0 + u] * v[u][0];
        s1 += g[K + k0 + u] * v[u][1];
        s2 += g[2 * K + k0 + u] * v[u][2];
      }
    }
    const int j = q / T2, e = q % T2;
    summed[(j * 3 + 0) * T2 + e] = s0;
    summed[(j * 3 + 1) * T2 + e] = s1;
    summed[(j * 3 + 2) * T2 + e] = s2;
  }
  __syncthreads();
  multi_tile_epilogue(summed, tmp, T, tile0, G, S, positions, normals, cam, material, scatter,
                      radiance, radiance_unclamped, rad64);
}

// ---------------------------------------------------------------------------
// batch L-level Haar (haar2d_fwd_batch / haar2d_inv_batch restated with a
// level limit): grid = batch * tiles, CTA per 2^L tile (tile-local transform)
// fwd: in spatial (batch, S, S) -> out flat Mallat; inv: the reverse
// ---------------------------------------------------------------------------
__global__ void k_haar2d_batch(const double* __restrict__ in, double* __restrict__ out, int S,
                               int L, int inverse) {
  extern __shared__ double sm[];
  const int T = 1 << L, T2 = T * T;
  double* a = sm;
  double* tmp = sm + T2;
  const int tiles = (S / T) * (S / T);
  const int b = blockIdx.x / tiles, tile = blockIdx.x % tiles;
  const int tr = tile / (S / T), tc = tile % (S / T);
  const size_t base = (size_t)b * S * S;
  for (int e = threadIdx.x; e < T2; e += blockDim.x) {
    if (!inverse) {
      a[e] = in[base + (size_t)(tr * T + e / T) * S + tc * T + e % T];
    } else {
      int gr, gc;
      local_to_global(e / T, e % T, tr, tc, L, S, &gr, &gc);
      a[e] = in[base + (size_t)gr * S + gc];
    }
  }
  __syncthreads();
  if (!inverse) tile_haar_fwd(a, tmp, T, blockDim.x, threadIdx.x);
  else tile_haar_inv(a, tmp, T, blockDim.x, threadIdx.x);
  __syncthreads();  // `in` may alias `out`: every read above precedes every write
  for (int e = threadIdx.x; e < T2; e += blockDim.x) {
    if (inverse) {
      out[base + (size_t)(tr * T + e / T) * S + tc * T + e % T] = a[e];
    } else {
      int gr, gc;
      local_to_global(e / T, e % T, tr, tc, L, S, &gr, &gc);
      out[base + (size_t)gr * S + gc] = a[e];
    }
  }
}

// ---------------------------------------------------------------------------
// env transfer precompute: W = cos+ * d_omega (V = 1, eta = 1), per-face full
// Haar, float32 (D, N). grid: (ceil(N / P), 6 faces), P points per CTA
// ---------------------------------------------------------------------------
constexpr int kEnvP = 8;
__global__ void k_env_transfer(const float* __restrict__ normals, int n_points,
                               const double* __restrict__ dirs, const double* __restrict__ dom,
                               int s, float* __restrict__ W2) {
  extern __shared__ double sm[];
  const int s2 = s * s, f = blockIdx.y;
  double* a = sm;                 // kEnvP * s2
  double* tmp = sm + kEnvP * s2;  // s2
  const int i0 = blockIdx.x * kEnvP;
  for (int e = threadIdx.x; e < kEnvP * s2; e += blockDim.x) {
    const int p = e / s2, t = e % s2, i = i0 + p;
    double w = 0.0;
    if (i < n_points) {
      const double* dv = dirs + (size_t)(f * s2 + t) * 3;
      const double c = dadd(dadd(dmul((double)normals[i * 3], dv[0]),
                                 dmul((double)normals[i * 3 + 1], dv[1])),
                            dmul((double)normals[i * 3 + 2], dv[2]));
      const double cp = fmin(fmax(c, 0.0), 1.0);
      w = dmul(cp, dom[f * s2 + t]);
    }
    a[e] = w;
  }
  __syncthreads();
  for (int p = 0; p < kEnvP; ++p) tile_haar_fwd(a + p * s2, tmp, s, blockDim.x, threadIdx.x);
  const int N = n_points;
  for (int e = threadIdx.x; e < kEnvP * s2; e += blockDim.x) {
    const int t = e / kEnvP, p = e % kEnvP, i = i0 + p;
    if (i < n_points) W2[(size_t)(f * s2 + t) * N + i] = (float)a[p * s2 + t];
  }
}

}  // namespace sss
