// Visibility precompute and ambient folding:
// precompute_visibility + fold_visibility (transfer.py:368-451) and the folded
// ambient term of the frame (runtime.py:146-149).
//
// Precompute, per scene:
//   k_visibility      V (D, N) u8: one thread per (direction, sample), a warp =
//                     32 neighbouring samples shooting parallel rays (coherent
//                     BVH paths); any-hit from direct.cu.
//   k_fold_weights    W = V F_t(eta, cos+) cos+ dw (visibility_weights,
//                     lighting.py:318-329) and the per-face full Haar over the
//                     direction axis (w2), written (D, N) fp64; the w0 Haar
//                     over samples then runs batched over the D images.
//   k_transpose_perm  (D, N flat) -> (N tile-major, D): v~ rows in the
//                     operator's column space, direction-contiguous.
//   k_fold_spmm       F_k = T_k v~ (the dense `dense @ v_tilde[cols]` of
//                     transfer.py:426): a warp per operator row, lanes over
//                     256 directions, fp64 FMA over the row's entries.
//   k_step2_select    compress_energy per direction column of F_k^T (the
//                     step-2 kernel with identity column map).
//   k_fold_emit       CSC per direction: kept rows ascending (flat ids), f32.
// Frame:
//   k_fold_apply      v_k += F_k L^{w2}: per CTA a block of 1024 flat rows,
//                     union coefficients in ascending order, each column's
//                     rows in order; the sums are the reference's serial
//                     csc_apply order (bitwise for the same stored values).
#include "sss_common.cuh"

namespace sss {

// ---- visibility (transfer.py:368-391): V[e][i] = n.d > 0 && !any_hit(far)
__global__ void __launch_bounds__(128) k_visibility(int N, const float* __restrict__ positions,
                                                    const float* __restrict__ normals,
                                                    const double* __restrict__ dirs,
                                                    double ray_offset, double far, BvhView B,
                                                    uint8_t* __restrict__ vis) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int e = blockIdx.y;
  if (i >= N) return;
  double p[3], n[3], o[3];
  load_point(i, positions, normals, ray_offset, p, n, o);
  const double d[3] = {dirs[3 * e], dirs[3 * e + 1], dirs[3 * e + 2]};
  const double cs = dot3(n, d);
  uint8_t v = 0;
  if (cs > 0.0) {
    Ray R;
    make_ray(R, o, d, far);
    v = any_hit(B, R) ? 0 : 1;
  }
  vis[(size_t)e * N + i] = v;
}

// ---- W = ((V F_t) cos+) dw, then per-face full Haar (transfer.py:405-411).
// grid (ceil(N / kFoldP), 6 faces); W2 (D, N) fp64.
constexpr int kFoldP = 8;

__global__ void __launch_bounds__(256) k_fold_weights(const float* __restrict__ normals, int N,
                                                      const double* __restrict__ dirs,
                                                      const double* __restrict__ dom, int s,
                                                      const uint8_t* __restrict__ vis, double eta,
                                                      double* __restrict__ W2) {
  extern __shared__ double fsm[];
  const int s2 = s * s, f = blockIdx.y;
  double* a = fsm;                  // kFoldP * s2
  double* tmp = fsm + kFoldP * s2;  // s2
  const int i0 = blockIdx.x * kFoldP;
  for (int e = threadIdx.x; e < kFoldP * s2; e += blockDim.x) {
    const int t = e / kFoldP, p = e % kFoldP, i = i0 + p;  // p fastest: 64-B vis / W2 runs
    double w = 0.0;
    if (i < N) {
      const int dd = f * s2 + t;
      if (vis[(size_t)dd * N + i]) {
        const double* dv = dirs + (size_t)dd * 3;
        const double c = dadd(dadd(dmul((double)normals[i * 3], dv[0]),
                                   dmul((double)normals[i * 3 + 1], dv[1])),
                              dmul((double)normals[i * 3 + 2], dv[2]));
        const double cp = fmin(fmax(c, 0.0), 1.0);
        w = dmul(dmul(ft_np(eta, cp), cp), dom[dd]);
      }
    }
    a[p * s2 + t] = w;
  }
  __syncthreads();
  for (int p = 0; p < kFoldP; ++p) tile_haar_fwd(a + p * s2, tmp, s, blockDim.x, threadIdx.x);
  for (int e = threadIdx.x; e < kFoldP * s2; e += blockDim.x) {
    const int t = e / kFoldP, p = e % kFoldP, i = i0 + p;
    if (i < N) W2[(size_t)(f * s2 + t) * N + i] = a[p * s2 + t];
  }
}

// ---- out (C, R) = in (R, C)^T with an optional column gather:
// out[j][r] = in[r][perm ? perm[j] : j]. block (32, 8), 32 x 32 tiles.
__global__ void __launch_bounds__(256) k_transpose_perm(const double* __restrict__ in, int R,
                                                        int C, const uint32_t* __restrict__ perm,
                                                        double* __restrict__ out) {
  __shared__ double t[32][33];
  const int j0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  for (int q = threadIdx.y; q < 32; q += 8) {
    const int r = r0 + q, j = j0 + threadIdx.x;
    t[q][threadIdx.x] = (r < R && j < C) ? in[(size_t)r * C + (perm ? perm[j] : j)] : 0.0;
  }
  __syncthreads();
  for (int q = threadIdx.y; q < 32; q += 8) {
    const int j = j0 + q, r = r0 + threadIdx.x;
    if (j < C && r < R) out[(size_t)j * R + r] = t[threadIdx.x][q];
  }
}

// ---- F (N, D) row-major = T_k (N x N, tile-major CSR, f32) x vt (N, D):
// a warp per row, lanes over a 256-direction chunk (8 per lane), entries
// four at a time so 32 gathers are in flight per lane.
constexpr int kSpmmWarps = 8;

__global__ void __launch_bounds__(32 * kSpmmWarps) k_fold_spmm(
    int N, int D, const long long* __restrict__ rowptr, const uint32_t* __restrict__ cols,
    const float* __restrict__ vals, const double* __restrict__ vt, double* __restrict__ F) {
  const int lane = threadIdx.x & 31;
  const int r = blockIdx.x * kSpmmWarps + (threadIdx.x >> 5);
  const int e0 = blockIdx.y * 256 + lane;
  if (r >= N) return;
  double acc[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) acc[q] = 0.0;
  const long long b = rowptr[r], e = rowptr[r + 1];
  const bool full = blockIdx.y * 256 + 256 <= D;
  long long j = b;
  for (; j + 4 <= e; j += 4) {
    uint32_t c[4];
    double v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      c[u] = __ldg(&cols[j + u]);
      v[u] = (double)__ldg(&vals[j + u]);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double* x = vt + (size_t)c[u] * D + e0;
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (full || e0 + 32 * q < D) acc[q] = fma(v[u], __ldg(&x[32 * q]), acc[q]);
    }
  }
  for (; j < e; ++j) {
    const uint32_t c = __ldg(&cols[j]);
    const double v = (double)__ldg(&vals[j]);
    const double* x = vt + (size_t)c * D + e0;
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (full || e0 + 32 * q < D) acc[q] = fma(v, __ldg(&x[32 * q]), acc[q]);
  }
#pragma unroll
  for (int q = 0; q < 8; ++q)
    if (full || e0 + 32 * q < D) F[(size_t)r * D + e0 + 32 * q] = acc[q];
}

// ---- emission: CSC per direction e of FT (D, N tm): kept rows in ascending
// flat order (wavelets.py:113-125 sorts the kept indices), values f32.
constexpr int kEmitThreads = 1024;

__global__ void __launch_bounds__(kEmitThreads) k_fold_emit(
    const double* __restrict__ FT, int N, const uint32_t* __restrict__ flat2tm,
    const uint64_t* __restrict__ col_t, const uint32_t* __restrict__ col_fmax,
    const uint32_t* __restrict__ col_cnt, const uint64_t* __restrict__ colptr,
    uint32_t* __restrict__ rows, float* __restrict__ vals) {
  __shared__ int wsum[kEmitThreads / 32];
  __shared__ int base;
  const int e = blockIdx.x;
  if (col_cnt[e] == 0) return;
  const uint64_t t = col_t[e];
  const int fmax = (int)col_fmax[e];
  const double* v = FT + (size_t)e * N;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) base = 0;
  __syncthreads();
  uint64_t out = colptr[e];
  for (int f0 = 0; f0 < N; f0 += kEmitThreads) {
    const int f = f0 + threadIdx.x;
    double x = 0.0;
    bool kp = false;
    if (f < N) {
      x = v[flat2tm[f]];
      const uint64_t k = mkey(x);
      kp = k > t || (k == t && fmax >= 0 && f <= fmax);
    }
    const unsigned bal = __ballot_sync(0xffffffffu, kp);
    if (lane == 0) wsum[warp] = __popc(bal);
    __syncthreads();
    if (warp == 0) {
      const int w = lane < kEmitThreads / 32 ? wsum[lane] : 0;
      int incl = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      if (lane < kEmitThreads / 32) wsum[lane] = incl - w;
    }
    __syncthreads();
    if (kp) {
      const uint64_t pos = out + base + wsum[warp] + __popc(bal & ((1u << lane) - 1u));
      rows[pos] = (uint32_t)f;
      vals[pos] = (float)x;
    }
    __syncthreads();
    if (threadIdx.x == kEmitThreads - 1) base += wsum[warp] + __popc(bal);
    __syncthreads();
  }
}

// ---- frame: v_k[c][tm(r)] += sum over union coefficients (ascending) of
// F_k[r][e] * L_c[e] (csc_apply order, _kernels_nb.py:301-313). grid
// (ceil(N / kFoldRows), K). colptr (K, D + 1) absolute; rows flat ids.
constexpr int kFoldRows = 1024;

__device__ __forceinline__ uint64_t lower_bound_u32(const uint32_t* a, uint64_t lo, uint64_t hi,
                                                    uint32_t key) {
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (a[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

__global__ void __launch_bounds__(256) k_fold_apply(
    int N, int D, const uint64_t* __restrict__ colptr, const uint32_t* __restrict__ rows,
    const float* __restrict__ vals, const uint32_t* __restrict__ union_idx,
    const double* __restrict__ union_lc, const int* __restrict__ n_union,
    const uint32_t* __restrict__ flat2tm, double* __restrict__ vk) {
  __shared__ double acc[3][kFoldRows];
  __shared__ uint64_t rng[2];
  const int k = blockIdx.y;
  const uint32_t r0 = blockIdx.x * kFoldRows;
  const uint32_t r1 = min((uint32_t)N, r0 + kFoldRows);
  for (int t = threadIdx.x; t < kFoldRows; t += blockDim.x)
    acc[0][t] = acc[1][t] = acc[2][t] = 0.0;
  const uint64_t* cp = colptr + (size_t)k * (D + 1);
  const int nu = *n_union;
  for (int u = 0; u < nu; ++u) {
    const uint32_t e = union_idx[u];
    __syncthreads();  // previous column's adds done before rng is rewritten
    if (threadIdx.x < 2) rng[threadIdx.x] = lower_bound_u32(rows, cp[e], cp[e + 1],
                                                            threadIdx.x ? r1 : r0);
    __syncthreads();
    const double l0 = union_lc[3 * u], l1 = union_lc[3 * u + 1], l2 = union_lc[3 * u + 2];
    for (uint64_t j = rng[0] + threadIdx.x; j < rng[1]; j += blockDim.x) {
      const int t = (int)(rows[j] - r0);
      const double v = (double)vals[j];
      acc[0][t] = dadd(acc[0][t], dmul(v, l0));
      acc[1][t] = dadd(acc[1][t], dmul(v, l1));
      acc[2][t] = dadd(acc[2][t], dmul(v, l2));
    }
  }
  __syncthreads();
  for (uint32_t r = r0 + threadIdx.x; r < r1; r += blockDim.x) {
    const uint32_t tm = flat2tm[r];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      double* o = vk + ((size_t)k * 3 + c) * N + tm;
      *o = dadd(*o, acc[c][r - r0]);
    }
  }
}

// ---- frame, row-major form: the same sums with one thread per (k, flat row)
// walking the row's entries in ascending direction order (the csc_apply
// order restricted to one row), the union's per-direction L_c gathered from
// a shared-memory table (zero for directions outside the union: adding
// v * 0 leaves a +0-started sum unchanged). No per-column barrier or search.
// Entries are ELL-interleaved per 32-row group (slot-major: entry s of lane
// j at gbase + 32 s + j, padded with (dir 0, val 0) to the group's longest
// row), so every warp load is one coalesced 128-B line.
// grid (N / 256, K), dynamic smem 24 * D bytes; N % 32 == 0.
__global__ void __launch_bounds__(256) k_fold_apply_rows(
    int N, int D, const uint64_t* __restrict__ gbase, const uint2* __restrict__ ent,
    const uint32_t* __restrict__ union_idx, const double* __restrict__ union_lc,
    const int* __restrict__ n_union, const uint32_t* __restrict__ flat2tm,
    double* __restrict__ vk) {
  extern __shared__ double tab[];  // [D][3]
  for (int t = threadIdx.x; t < 3 * D; t += blockDim.x) tab[t] = 0.0;
  __syncthreads();
  const int nu = *n_union;
  for (int u = threadIdx.x; u < nu; u += blockDim.x) {
    const uint32_t e = union_idx[u];
    tab[3 * e] = union_lc[3 * u];
    tab[3 * e + 1] = union_lc[3 * u + 1];
    tab[3 * e + 2] = union_lc[3 * u + 2];
  }
  __syncthreads();
  const int k = blockIdx.y;
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= N) return;
  const size_t g = (size_t)k * (N >> 5) + (r >> 5);
  const uint64_t b0 = gbase[g], b1 = gbase[g + 1];
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
  constexpr int U = 16;  // entries in flight per thread: the loads of a batch
                         // are independent, only the fp64 sums are serial
  constexpr int PF = 4;  // L2 prefetch distance in batches (the long, dense
                         // coarse rows are a serial chain: keep it fed from L2)
  const int lane = r & 31;
  for (uint64_t j = b0 + lane; j < b1; j += 32 * U) {
    {  // lane l prefetches line l of the batch PF ahead (32 lines = 32 * U entries)
      const uint64_t pj = (j - lane) + (uint64_t)PF * 32 * U + (uint64_t)lane * 16;
      if (pj < b1) asm volatile("prefetch.global.L2 [%0];" ::"l"(ent + pj));
    }
    uint2 x[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      x[u] = j + 32 * u < b1 ? __ldcs(ent + j + 32 * u) : make_uint2(0u, 0u);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const double v = (double)__uint_as_float(x[u].y);
      const double* t = tab + 3 * x[u].x;
      a0 = dadd(a0, dmul(v, t[0]));
      a1 = dadd(a1, dmul(v, t[1]));
      a2 = dadd(a2, dmul(v, t[2]));
    }
  }
  const uint32_t tm = flat2tm[r];
  double* o = vk + (size_t)k * 3 * N + tm;
  o[0] = dadd(o[0], a0);
  o[N] = dadd(o[N], a1);
  o[2 * (size_t)N] = dadd(o[2 * (size_t)N], a2);
}

}  // namespace sss
