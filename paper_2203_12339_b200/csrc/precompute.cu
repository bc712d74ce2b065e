// Offline pair pass + two-step wavelet compression on sm_100a (path d).
//
// Reference: precompute_compressed (transfer.py:350-361) = transfer_block
// (_kernels_nb.py:179-205) -> w0 Haar -> per-row top-n (step 1,
// transfer.py:216-230) -> per-k union (:233-246) -> dense union columns,
// w1 transform, per-column energy fraction (step 2, :249-333).
//
// B200 formulation (geometry image, L-level Haar on both axes, L <= 3):
//  * both transforms are tile-local, so one CTA per (receiver tile RT,
//    source tile ST) block computes the 4^L x 4^L pair block, Haars it along
//    sources (-> D, the step-1 rows) and, after the f32 rounding the
//    reference applies to step-2 columns (transfer.py:282-289), along
//    receivers (-> M, the step-2 columns). D and M for one k are
//    materialised in HBM (2 x N^2 doubles: 69 GB at 256^2, one k at a time);
//    the 180 GB part makes the reference's spill file and per-group row
//    re-evaluation unnecessary.
//  * step 1 / step 2 are exact radix selections (64-bit magnitude keys,
//    flat-index tie-break), the step-2 energy cut in 2^62 fixed point so the
//    per-bucket sums are exact integers (order independent).
//  * emission writes the frame layout directly: tile-major CSR per k.
// Lerp mode reproduces transfer_block bit for bit (fp64, reference operation
// order, no FMA); exact mode evaluates R_d per pair for every training
// material in fp32 and projects on the PCA bases.
#include "select.cuh"
#include "haar_tile.cuh"

namespace sss {

constexpr int kSelThreads = 1024;


// ---------------------------------------------------------------------------
// pair block: T[o][i] for a 4^L x 4^L (receiver tile, source tile) block,
// w0 Haar along sources -> D; f32 round; w1 Haar along receivers -> M.
// Layouts (tile-major on both axes, N = S*S):
//   D[o_tm * N + c_tm]   row-major (step-1 rows)
//   M[c_tm * N + r_tm]   column-major (step-2 columns)
// ---------------------------------------------------------------------------

struct PairParams {
  const float* pos;     // (N, 3)
  const float* area;    // (N,)
  const double* r_nodes;
  const double* bases;  // (K, nr)
  const double* slopes; // (K, nr-1)
  int nr, k, S;
  // exact mode
  const float* Pkm;     // (K, M) projection coefficients U/S
  const float* mat;     // (M, 4): sigma_tr, z_r, z_v, alpha'/(4 pi)
  int M;
  float r_max;
};

template <int L, bool EXACT>
__global__ void __launch_bounds__(128) k_pair_block(PairParams p, double* __restrict__ D,
                                                    double* __restrict__ Mout) {
  constexpr int T = 1 << L, T2 = T * T, LD = T2 + 1;
  extern __shared__ double smp[];
  double* blk = smp;                       // T2 x LD
  double* rn = blk + T2 * LD;              // nr
  double* bk = rn + p.nr;                  // nr
  double* sk = bk + p.nr;                  // nr - 1
  const int S = p.S, N = S * S, tpr = S / T;
  const int ST = blockIdx.x, RT = blockIdx.y;
  const int str = ST / tpr, stc = ST % tpr, rtr = RT / tpr, rtc = RT % tpr;
  // exact mode: the material table and this term's projection row in shared
  // memory (one LDS.128 + one LDS per material instead of five L1 loads)
  float4* mat4 = reinterpret_cast<float4*>(blk + T2 * LD);
  float* pk = reinterpret_cast<float*>(mat4 + (EXACT ? p.M : 0));
  if (!EXACT) {
    for (int j = threadIdx.x; j < p.nr; j += blockDim.x) {
      rn[j] = p.r_nodes[j];
      bk[j] = p.bases[(size_t)p.k * p.nr + j];
      if (j < p.nr - 1) sk[j] = p.slopes[(size_t)p.k * (p.nr - 1) + j];
    }
  } else {
    for (int m = threadIdx.x; m < p.M; m += blockDim.x) {
      mat4[m] = make_float4(p.mat[m * 4], p.mat[m * 4 + 1], p.mat[m * 4 + 2], p.mat[m * 4 + 3]);
      pk[m] = p.Pkm[p.k * p.M + m];
    }
  }
  __syncthreads();
  const double r_last = EXACT ? 0.0 : rn[p.nr - 1];
  for (int e = threadIdx.x; e < T2 * T2; e += blockDim.x) {
    const int o = e / T2, i = e % T2;
    const int oi = (rtr * T + o / T) * S + rtc * T + o % T;  // receiver point
    const int si = (str * T + i / T) * S + stc * T + i % T;  // source point
    if (!EXACT) {
      // transfer_block (_kernels_np.py:142-158): diff = receiver - source
      const double dx = dsub((double)p.pos[oi * 3], (double)p.pos[si * 3]);
      const double dy = dsub((double)p.pos[oi * 3 + 1], (double)p.pos[si * 3 + 1]);
      const double dz = dsub((double)p.pos[oi * 3 + 2], (double)p.pos[si * 3 + 2]);
      const double d = __dsqrt_rn(dadd(dadd(dmul(dx, dx), dmul(dy, dy)), dmul(dz, dz)));
      // j = bisect_right(r_nodes, d) - 1, clipped to [0, nr - 2]
      int lo = 0, hi = p.nr;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (rn[mid] <= d) lo = mid + 1; else hi = mid;
      }
      int j = lo - 1;
      j = j < 0 ? 0 : (j > p.nr - 2 ? p.nr - 2 : j);
      const double frac = dsub(d, rn[j]);
      const double a_eff = (d <= r_last) ? (double)p.area[si] : 0.0;
      blk[o * LD + i] = dmul(dadd(bk[j], dmul(sk[j], frac)), a_eff);
    } else {
      const float dx = p.pos[oi * 3] - p.pos[si * 3];
      const float dy = p.pos[oi * 3 + 1] - p.pos[si * 3 + 1];
      const float dz = p.pos[oi * 3 + 2] - p.pos[si * 3 + 2];
      const float r2 = dx * dx + dy * dy + dz * dz;
      const float d = sqrtf(r2);
      float acc = 0.0f;
      if (d <= p.r_max) {
        for (int m = 0; m < p.M; ++m) {
          const float4 mm = mat4[m];
          const float s = mm.x, zr = mm.y, zv = mm.z, c = mm.w;
          const float ir = rsqrtf(r2 + zr * zr), iv = rsqrtf(r2 + zv * zv);
          const float dr = (r2 + zr * zr) * ir, dv = (r2 + zv * zv) * iv;
          const float tr = zr * (s + ir) * __expf(-s * dr) * ir * ir;
          const float tv = zv * (s + iv) * __expf(-s * dv) * iv * iv;
          acc = fmaf(pk[m], c * (tr + tv), acc);
        }
      }
      blk[o * LD + i] = (double)(acc * p.area[si]);
    }
  }
  __syncthreads();
  // w0 Haar along sources (one receiver row per thread)
  if (threadIdx.x < T2) seq_haar_fwd<T>(blk + threadIdx.x * LD, 1);
  __syncthreads();
  // D rows: receiver o_tm = RT*T2 + o, columns c_tm = ST*T2 + c
  if (D) {
    for (int e = threadIdx.x; e < T2 * T2; e += blockDim.x) {
      const int o = e / T2, c = e % T2;
      D[(size_t)(RT * T2 + o) * N + ST * T2 + c] = blk[o * LD + c];
    }
  }
  if (!Mout) return;
  __syncthreads();
  // step-2 columns are gathered as float32 (transfer.py:282-289, :322)
  for (int e = threadIdx.x; e < T2 * T2; e += blockDim.x) {
    const int o = e / T2, c = e % T2;
    blk[o * LD + c] = (double)(float)blk[o * LD + c];
  }
  __syncthreads();
  // w1 Haar along receivers (one column per thread)
  if (threadIdx.x < T2) seq_haar_fwd<T>(blk + threadIdx.x, LD);
  __syncthreads();
  for (int e = threadIdx.x; e < T2 * T2; e += blockDim.x) {
    const int c = e / T2, r = e % T2;
    Mout[(size_t)(ST * T2 + c) * N + RT * T2 + r] = blk[r * LD + c];
  }
}

// step 1: one CTA per receiver row of D (tile-major), top-n with flat-index
// tie-break, OR the kept flat column ids into the per-k union bitmap
// rows (nullable): the CTA's row of D is rows[blockIdx.x]; row_bits (nullable):
// write the row's kept bitmap (flat ids, nw words per CTA) instead of OR-ing
// it into the union (the sampled-row parity hook)
__global__ void __launch_bounds__(kSelThreads) k_step1_select(const double* __restrict__ D, int N,
                                                              int n_keep,
                                                              const uint32_t* __restrict__ tm2flat,
                                                              uint32_t* __restrict__ union_bits,
                                                              const int* __restrict__ rows = nullptr,
                                                              uint32_t* __restrict__ row_bits = nullptr) {
  extern __shared__ __align__(16) unsigned char dsm[];
  SelShared& sh = *reinterpret_cast<SelShared*>(dsm);
  uint32_t* smb = reinterpret_cast<uint32_t*>(dsm + sizeof(SelShared));  // keep + tie bits
  const int nw = (N + 31) / 32;
  uint32_t* keep = smb;
  uint32_t* tie = smb + nw;
  const double* v = D + (size_t)(rows ? rows[blockIdx.x] : (int)blockIdx.x) * N;
  for (int w = threadIdx.x; w < 2 * nw; w += blockDim.x) smb[w] = 0;
  uint64_t t;
  long long take, tiecnt;
  radix_cut<false>(v, N, n_keep, 0.0, sh, &t, &take, &tiecnt);
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    const uint64_t k = mkey(v[i]);
    if (k > t) { const uint32_t f = tm2flat[i]; atomicOr(&keep[f >> 5], 1u << (f & 31)); }
    else if (k == t) { const uint32_t f = tm2flat[i]; atomicOr(&tie[f >> 5], 1u << (f & 31)); }
  }
  __syncthreads();
  int fmax = N;  // all ties kept
  if (take < tiecnt) fmax = kth_set_bit(tie, nw, take, sh);
  for (int w = threadIdx.x; w < nw; w += blockDim.x) {
    uint32_t tb = tie[w];
    if (fmax < N) {
      const int lo = w * 32;
      if (lo > fmax) tb = 0;
      else if (fmax - lo < 31) tb &= (2u << (fmax - lo)) - 1u;
    }
    const uint32_t kept = keep[w] | tb;
    if (row_bits) row_bits[(size_t)blockIdx.x * nw + w] = kept;
    else if (kept && (union_bits[w] & kept) != kept) atomicOr(&union_bits[w], kept);
  }
}

// step 2: one CTA per w0 column (flat id c); energy cut over the column of M
// (tile-major rows). Writes per-column threshold / tie bound / counts.
__global__ void __launch_bounds__(kSelThreads) k_step2_select(
    const double* __restrict__ M, int N, double fraction, const uint32_t* __restrict__ flat2tm,
    const uint32_t* __restrict__ tm2flat, const uint32_t* __restrict__ union_bits,
    uint64_t* __restrict__ col_t, uint32_t* __restrict__ col_fmax, uint32_t* __restrict__ col_cnt,
    double* __restrict__ col_energy /* (N, 2): kept, total */,
    uint32_t* __restrict__ col_nz /* may be null */) {
  extern __shared__ __align__(16) unsigned char dsm[];
  SelShared& sh = *reinterpret_cast<SelShared*>(dsm);
  uint32_t* smb = reinterpret_cast<uint32_t*>(dsm + sizeof(SelShared));  // tie bits
  const int c = blockIdx.x;  // flat column (fold: direction, identity map, no union)
  const int nw = (N + 31) / 32;
  const int ctm = flat2tm ? (int)flat2tm[c] : c;
  if (union_bits && !((union_bits[c >> 5] >> (c & 31)) & 1u)) {
    if (threadIdx.x == 0) {
      col_t[ctm] = ~0ULL; col_fmax[ctm] = 0; col_cnt[ctm] = 0;
      col_energy[ctm * 2] = 0.0; col_energy[ctm * 2 + 1] = 0.0;
    }
    return;
  }
  const double* v = M + (size_t)ctm * N;
  uint32_t* tie = smb;
  for (int w = threadIdx.x; w < nw; w += blockDim.x) tie[w] = 0;
  double tot = 0.0;
  long long nz = 0;
  for (int i = threadIdx.x; i < N; i += blockDim.x) { const double x = v[i]; tot += x * x; nz += (x != 0.0); }
  tot = block_sum_d(tot, sh.red);
  nz = block_sum_i(nz, sh.redi);
  uint64_t t = ~0ULL;
  long long take = 0, tiecnt = 0;
  if (fraction > 0.0 && tot > 0.0) {
    const double scale = 4611686018427387904.0 / tot;  // 2^62 / total
    const long long target = (long long)(fraction * 4611686018427387904.0);
    radix_cut<true>(v, N, target, scale, sh, &t, &take, &tiecnt);
  }
  // count kept (> t) and mark ties in flat order
  long long above = 0;
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    const uint64_t k = mkey(v[i]);
    if (k > t) ++above;
    else if (k == t && t != ~0ULL) { const uint32_t f = tm2flat[i]; atomicOr(&tie[f >> 5], 1u << (f & 31)); }
  }
  above = block_sum_i(above, sh.redi);
  __syncthreads();
  long long kept = above + take;
  int fmax = -1;
  if (take > 0) fmax = (take < tiecnt) ? kth_set_bit(tie, nw, take, sh) : N;
  if (kept > nz) {  // never keep zeros (wavelets.py:151)
    kept = nz;
    t = 0;
    fmax = -1;
  }
  // kept energy (compress_energy ledger)
  double ke = 0.0;
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    const double x = v[i];
    const uint64_t k = mkey(x);
    const bool kp = k > t || (k == t && fmax >= 0 && (int)tm2flat[i] <= fmax);
    if (kp) ke += x * x;
  }
  ke = block_sum_d(ke, sh.red);
  if (threadIdx.x == 0) {
    col_t[ctm] = t;
    col_fmax[ctm] = (uint32_t)(fmax < 0 ? 0xffffffffu : (uint32_t)fmax);
    col_cnt[ctm] = (uint32_t)kept;
    col_energy[ctm * 2] = fmin(ke, tot);
    col_energy[ctm * 2 + 1] = tot;
    if (col_nz) col_nz[ctm] = (uint32_t)nz;
  }
}

__device__ __forceinline__ bool kept_entry(uint64_t k, uint64_t t, uint32_t fmax, uint32_t flat_r) {
  return k > t || (k == t && fmax != 0xffffffffu && flat_r <= fmax);
}

// emission, pass A: per (receiver tile, column chunk) count kept entries per
// row. grid (chunks, tiles), T2 threads (one row each)
__global__ void k_emit_count(const double* __restrict__ M, int N, int T2, int chunk,
                             const uint64_t* __restrict__ col_t, const uint32_t* __restrict__ col_fmax,
                             const uint32_t* __restrict__ tm2flat, uint32_t* __restrict__ counts) {
  const int ch = blockIdx.x, RT = blockIdx.y, r = threadIdx.x;
  if (r >= T2) return;
  const int rtm = RT * T2 + r;
  const uint32_t fr = tm2flat[rtm];
  const int c0 = ch * chunk, c1 = min(c0 + chunk, N);
  unsigned cnt = 0;
  for (int c = c0; c < c1; ++c) {
    const uint64_t t = __ldg(&col_t[c]);
    if (t == ~0ULL) continue;
    const uint64_t k = mkey(M[(size_t)c * N + rtm]);
    cnt += kept_entry(k, t, __ldg(&col_fmax[c]), fr);
  }
  counts[(size_t)rtm * gridDim.x + ch] = cnt;
}

// pass B: write (flat col, f32 val) at the scanned offsets
__global__ void k_emit_write(const double* __restrict__ M, int N, int T2, int chunk,
                             const uint64_t* __restrict__ col_t, const uint32_t* __restrict__ col_fmax,
                             const uint32_t* __restrict__ tm2flat, const uint64_t* __restrict__ offs,
                             uint64_t base, uint32_t* __restrict__ cols, float* __restrict__ vals) {
  const int ch = blockIdx.x, RT = blockIdx.y, r = threadIdx.x;
  if (r >= T2) return;
  const int rtm = RT * T2 + r;
  const uint32_t fr = tm2flat[rtm];
  const int c0 = ch * chunk, c1 = min(c0 + chunk, N);
  uint64_t o = base + offs[(size_t)rtm * gridDim.x + ch];
  for (int c = c0; c < c1; ++c) {
    const uint64_t t = __ldg(&col_t[c]);
    if (t == ~0ULL) continue;
    const double x = M[(size_t)c * N + rtm];
    if (kept_entry(mkey(x), t, __ldg(&col_fmax[c]), fr)) {
      cols[o] = (uint32_t)c;  // tile-major w0 id (frame layout)
      vals[o] = (float)x;
      ++o;
    }
  }
}

// exclusive scan of u32 counts -> u64 offsets (3-kernel, 1024 per block)
__global__ void k_scan_blocks(const uint32_t* __restrict__ in, uint64_t* __restrict__ out, size_t n,
                              uint64_t* __restrict__ block_sums) {
  __shared__ uint64_t wsum[32];
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t x = i < n ? in[i] : 0;
  uint64_t incl = x;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) wsum[wid] = incl;
  __syncthreads();
  if (threadIdx.x < 32) {
    uint64_t s = threadIdx.x < (blockDim.x >> 5) ? wsum[threadIdx.x] : 0;
    uint64_t inc = s;
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(0xffffffffu, inc, o);
      if (threadIdx.x >= o) inc += y;
    }
    wsum[threadIdx.x] = inc - s;
    if (threadIdx.x == 31) block_sums[blockIdx.x] = inc;
  }
  __syncthreads();
  if (i < n) out[i] = wsum[wid] + incl - x;
}

__global__ void k_scan_sums(uint64_t* __restrict__ block_sums, int nb, uint64_t* __restrict__ total) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  uint64_t a = 0;
  for (int b = 0; b < nb; ++b) { const uint64_t t = block_sums[b]; block_sums[b] = a; a += t; }
  *total = a;
}

__global__ void k_scan_add(uint64_t* __restrict__ out, size_t n, const uint64_t* __restrict__ block_sums) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] += block_sums[blockIdx.x];
}

// rowptr (N+1) from the scanned (row, chunk) offsets
__global__ void k_rowptr(const uint64_t* __restrict__ offs, int nchunks, int N, uint64_t base,
                         const uint64_t* __restrict__ total, uint64_t* __restrict__ rowptr) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < N) rowptr[r] = base + offs[(size_t)r * nchunks];
  if (r == N) rowptr[N] = base + *total;
}

}  // namespace sss

namespace sss {
// per (k, row): offsets (relative to the row start) of the first entry whose
// tile-major column is >= b * band_width, b = 0..NB (frame layout v2)
__global__ void k_band_offsets(const uint64_t* __restrict__ rowptr, const uint32_t* __restrict__ cols,
                               int K, int N, int band_width, int NB, uint32_t* __restrict__ bandoff) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long long)K * N) return;
  const int k = (int)(i / N), r = (int)(i % N);
  const uint64_t s = rowptr[(size_t)k * (N + 1) + r], e = rowptr[(size_t)k * (N + 1) + r + 1];
  uint32_t* out = bandoff + (size_t)i * (NB + 1);
  for (int b = 0; b <= NB; ++b) {
    const uint32_t lim = (uint32_t)b * (uint32_t)band_width;
    uint64_t lo = s, hi = e;
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (cols[mid] < lim) lo = mid + 1; else hi = mid;
    }
    out[b] = (uint32_t)(lo - s);
  }
}

}  // namespace sss
