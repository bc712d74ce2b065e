// Kernels behind the reference's kernel seam (`_accel.get_kernels()`,
// _accel.py:35-43): device twins of the hot loops in _kernels_nb.py with the
// same arithmetic, so the reference's own callers (wavelets.py, transfer.py,
// lighting.py, runtime.py) get bitwise-identical results from the GPU
// (paper_2203_12339_b200/kernels_b200.py binds them with numpy in / out).
//
//   k_wline<HAAR|CDF97, fwd|inv>  one level / axis of haar2d_* / cdf97_*_batch
//                                 (_kernels_nb.py:22-163): a line per group
//                                 of threads, staged in shared memory, the
//                                 lifting steps data-parallel along the line
//                                 (each step reads only the other parity)
//   k_csr_apply                   csc_apply (_kernels_nb.py:301-313) from a
//                                 row-major copy whose entries keep the
//                                 column order: each row's fp64 sum has the
//                                 reference's addition order
//   k_transfer_rows<T>            transfer_block (_kernels_nb.py:179-205)
//   k_bvh_any_hit                 bvh_any_hit (_kernels_nb.py:265-298) on the
//                                 reference's BVH arrays
// Everything is fp64 (or the caller's position dtype for the distance) with
// explicit round-to-nearest operations: no FMA contraction, like numba with
// fastmath off.
#include "sss_common.cuh"

namespace sss {

// CDF 9/7 lifting constants of _kernels_np.py:17-24, bit for bit (gamma and
// zeta are derived there in double; these are the resulting values)
constexpr double kCdfA = -0x1.960ce67635b8dp+0;
constexpr double kCdfB = -0x1.b2035c937d836p-5;
constexpr double kCdfG = 0x1.c40ceba55cf39p-1;
constexpr double kCdfD = 0x1.c626a904721eep-2;
constexpr double kCdfZ = 0x1.264c795071461p+0;
constexpr double kCdfIZ = 0x1.bd5edf975ce1cp-1;

enum { kWHaar = 0, kWCdf97 = 1 };

// lifting step on one parity of a line x[0..s): odd (i = 1, 3, ..): interior
// x[i] +-= c (x[i-1] + x[i+1]), boundary i = s-1: x[i] +-= (2c) x[s-2];
// even (i = 0, 2, ..): interior the same, boundary i = 0: x[0] +-= (2c) x[1]
template <bool ODD, bool SUB>
__device__ __forceinline__ void lift(double* x, int s, int t, int tpl, double c) {
  const double c2 = 2.0 * c;  // exact
  for (int idx = t; idx < (s >> 1); idx += tpl) {
    const int i = 2 * idx + (ODD ? 1 : 0);
    double d;
    if (ODD ? (i == s - 1) : (i == 0))
      d = dmul(c2, x[ODD ? s - 2 : 1]);
    else
      d = dmul(c, dadd(x[i - 1], x[i + 1]));
    x[i] = SUB ? dsub(x[i], d) : dadd(x[i], d);
  }
}

// One pass of a 2D transform level over nb blocks (full x full, row-major):
// lines of length s inside the top-left s x s sub-block, along rows (axis 0)
// or columns (axis 1). tpl threads per line, blockDim / tpl lines per CTA.
template <int KIND, bool INV>
__global__ void __launch_bounds__(256) k_wline(double* __restrict__ data, int nb, int full, int s,
                                               int axis, int tpl) {
  extern __shared__ double wl_smem[];
  const int lpc = blockDim.x / tpl;
  const int stride = s + 1;  // odd stride: column-line stores hit distinct banks
  double* buf = wl_smem;
  double* tmp = wl_smem + lpc * stride;
  const long long lines = (long long)nb * s;
  const long long l0 = (long long)blockIdx.x * lpc;
  auto addr = [&](int li, int k) -> long long {
    const long long line = l0 + li;
    if (line >= lines) return -1;
    const long long b = line / s, q = line % s;
    return b * full * (long long)full + (axis == 0 ? q * full + k : (long long)k * full + q);
  };
  for (int e = threadIdx.x; e < lpc * s; e += blockDim.x) {
    // rows: consecutive threads walk one line; columns: across lines
    const int li = axis == 0 ? e / s : e % lpc, k = axis == 0 ? e % s : e / lpc;
    const long long a = addr(li, k);
    if (a >= 0) buf[li * stride + k] = data[a];
  }
  __syncthreads();
  const int li = threadIdx.x / tpl, t = threadIdx.x % tpl, h = s >> 1;
  double* x = buf + li * stride;
  double* y = tmp + li * stride;
  if (KIND == kWHaar) {
    for (int j = t; j < h; j += tpl) {
      if (!INV) {
        const double ev = x[2 * j], od = x[2 * j + 1];
        y[j] = dmul(dadd(ev, od), SSS_ISQRT2);
        y[h + j] = dmul(dsub(ev, od), SSS_ISQRT2);
      } else {
        const double lo = x[j], hi = x[h + j];
        y[2 * j] = dmul(dadd(lo, hi), SSS_ISQRT2);
        y[2 * j + 1] = dmul(dsub(lo, hi), SSS_ISQRT2);
      }
    }
  } else if (!INV) {  // _cdf97_line_fwd (_kernels_nb.py:81-101)
    lift<true, false>(x, s, t, tpl, kCdfA);
    __syncthreads();
    lift<false, false>(x, s, t, tpl, kCdfB);
    __syncthreads();
    lift<true, false>(x, s, t, tpl, kCdfG);
    __syncthreads();
    lift<false, false>(x, s, t, tpl, kCdfD);
    __syncthreads();
    for (int j = t; j < h; j += tpl) {
      y[j] = dmul(x[2 * j], kCdfZ);
      y[h + j] = dmul(x[2 * j + 1], kCdfIZ);
    }
  } else {  // _cdf97_line_inv (_kernels_nb.py:104-121)
    for (int j = t; j < h; j += tpl) {
      y[2 * j] = dmul(x[j], kCdfIZ);
      y[2 * j + 1] = dmul(x[h + j], kCdfZ);
    }
    __syncthreads();
    lift<false, true>(y, s, t, tpl, kCdfD);
    __syncthreads();
    lift<true, true>(y, s, t, tpl, kCdfG);
    __syncthreads();
    lift<false, true>(y, s, t, tpl, kCdfB);
    __syncthreads();
    lift<true, true>(y, s, t, tpl, kCdfA);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < lpc * s; e += blockDim.x) {
    const int lj = axis == 0 ? e / s : e % lpc, k = axis == 0 ? e % s : e / lpc;
    const long long a = addr(lj, k);
    if (a >= 0) data[a] = tmp[lj * stride + k];
  }
}

// out[r] = sum over the row's entries, in stored (= ascending column) order,
// of vals[e] * xcol[cpos[e]] for the columns present in x (present bit set);
// rows with no present entry are 0.0, like np.zeros + skipped columns.
__global__ void k_csr_apply(int n_rows, const long long* __restrict__ rowptr,
                            const int* __restrict__ cpos, const double* __restrict__ vals,
                            const double* __restrict__ xcol, const unsigned char* __restrict__ present,
                            double* __restrict__ out) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_rows) return;
  double acc = 0.0;
  for (long long e = rowptr[r]; e < rowptr[r + 1]; ++e) {
    const int c = cpos[e];
    if (present[c]) acc = dadd(acc, dmul(vals[e], xcol[c]));
  }
  out[r] = acc;
}

template <typename T>
__device__ __forceinline__ T tadd(T a, T b);
template <>
__device__ __forceinline__ float tadd(float a, float b) { return __fadd_rn(a, b); }
template <>
__device__ __forceinline__ double tadd(double a, double b) { return __dadd_rn(a, b); }
template <typename T>
__device__ __forceinline__ T tsub(T a, T b);
template <>
__device__ __forceinline__ float tsub(float a, float b) { return __fsub_rn(a, b); }
template <>
__device__ __forceinline__ double tsub(double a, double b) { return __dsub_rn(a, b); }
template <typename T>
__device__ __forceinline__ T tmul(T a, T b);
template <>
__device__ __forceinline__ float tmul(float a, float b) { return __fmul_rn(a, b); }
template <>
__device__ __forceinline__ double tmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float tsqrt(float a) { return __fsqrt_rn(a); }
__device__ __forceinline__ double tsqrt(double a) { return __dsqrt_rn(a); }

// out (nblk, K, n): (bases[k, j] + slopes[k, j] * frac) * area_eff (bases (K,
// nr), slopes (K, nr - 1) per-segment differences), the
// distance in the positions' dtype T, everything after it in fp64
template <typename T>
__global__ void k_transfer_rows(int nblk, int n, int K, int nr, const T* __restrict__ bpos,
                                const T* __restrict__ pos, const double* __restrict__ areas,
                                const double* __restrict__ r_nodes, const double* __restrict__ bases,
                                const double* __restrict__ slopes, double* __restrict__ out) {
  const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= (long long)nblk * n) return;
  const int b = (int)(g / n), i = (int)(g % n);
  const T dx = tsub(bpos[3 * b], pos[3 * i]);
  const T dy = tsub(bpos[3 * b + 1], pos[3 * i + 1]);
  const T dz = tsub(bpos[3 * b + 2], pos[3 * i + 2]);
  const T dt = tsqrt(tadd(tadd(tmul(dx, dx), tmul(dy, dy)), tmul(dz, dz)));
  const double d = (double)dt;
  int lo = 0, hi = nr;  // _bisect_right(r_nodes, d)
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (r_nodes[mid] <= d) lo = mid + 1; else hi = mid;
  }
  int j = lo - 1;
  j = j < 0 ? 0 : (j > nr - 2 ? nr - 2 : j);
  const double frac = dsub(d, r_nodes[j]);
  const double ae = d <= r_nodes[nr - 1] ? areas[i] : 0.0;
  for (int k = 0; k < K; ++k)
    out[((long long)b * K + k) * n + i] =
        dmul(dadd(bases[k * nr + j], dmul(slopes[k * (nr - 1) + j], frac)), ae);
}

struct RefBvh {
  const double *nmin, *nmax;
  const int *left, *right, *start, *count;
  const double *v0, *e1, *e2;
};

__device__ bool ref_tri_hit(double ox, double oy, double oz, double dx, double dy, double dz,
                            double tmax, const RefBvh& B, int t) {
  const double e1x = B.e1[3 * t], e1y = B.e1[3 * t + 1], e1z = B.e1[3 * t + 2];
  const double e2x = B.e2[3 * t], e2y = B.e2[3 * t + 1], e2z = B.e2[3 * t + 2];
  const double pvx = dsub(dmul(dy, e2z), dmul(dz, e2y));
  const double pvy = dsub(dmul(dz, e2x), dmul(dx, e2z));
  const double pvz = dsub(dmul(dx, e2y), dmul(dy, e2x));
  const double det = dadd(dadd(dmul(e1x, pvx), dmul(e1y, pvy)), dmul(e1z, pvz));
  if (fabs(det) <= 1e-14) return false;
  const double inv = __ddiv_rn(1.0, det);
  const double tvx = dsub(ox, B.v0[3 * t]), tvy = dsub(oy, B.v0[3 * t + 1]),
               tvz = dsub(oz, B.v0[3 * t + 2]);
  const double u = dmul(dadd(dadd(dmul(tvx, pvx), dmul(tvy, pvy)), dmul(tvz, pvz)), inv);
  if (u < 0.0 || u > 1.0) return false;
  const double qvx = dsub(dmul(tvy, e1z), dmul(tvz, e1y));
  const double qvy = dsub(dmul(tvz, e1x), dmul(tvx, e1z));
  const double qvz = dsub(dmul(tvx, e1y), dmul(tvy, e1x));
  const double v = dmul(dadd(dadd(dmul(dx, qvx), dmul(dy, qvy)), dmul(dz, qvz)), inv);
  if (v < 0.0 || dadd(u, v) > 1.0) return false;
  const double tt = dmul(dadd(dadd(dmul(e2x, qvx), dmul(e2y, qvy)), dmul(e2z, qvz)), inv);
  return tt > 1e-9 && tt < tmax;
}

__device__ bool ref_box_hit(const double o[3], const double d[3], double tmax, const RefBvh& B,
                            int node) {
  double tn = 0.0, tf = tmax;
  for (int ax = 0; ax < 3; ++ax) {
    const double lo = B.nmin[3 * node + ax], hi = B.nmax[3 * node + ax];
    if (d[ax] == 0.0) {
      if (o[ax] < lo || o[ax] > hi) return false;
    } else {
      const double inv = __ddiv_rn(1.0, d[ax]);
      double ta = dmul(dsub(lo, o[ax]), inv), tb = dmul(dsub(hi, o[ax]), inv);
      if (ta > tb) { const double q = ta; ta = tb; tb = q; }
      if (ta > tn) tn = ta;
      if (tb < tf) tf = tb;
      if (tn > tf) return false;
    }
  }
  return tn <= tf;
}

// one thread per ray, depth-first with the reference's push order (left,
// right: right popped first); the stack holds 64 nodes as the reference's
__global__ void k_bvh_any_hit(int n_rays, const double* __restrict__ origins,
                              const double* __restrict__ dirs, const double* __restrict__ tmax,
                              RefBvh B, unsigned char* __restrict__ hit, int* __restrict__ overflow) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_rays) return;
  const double o[3] = {origins[3 * r], origins[3 * r + 1], origins[3 * r + 2]};
  const double d[3] = {dirs[3 * r], dirs[3 * r + 1], dirs[3 * r + 2]};
  const double tm = tmax[r];
  int stack[64];
  stack[0] = 0;
  int top = 1;
  bool found = false;
  while (top > 0 && !found) {
    const int node = stack[--top];
    if (!ref_box_hit(o, d, tm, B, node)) continue;
    const int cnt = B.count[node];
    if (cnt > 0) {
      const int st = B.start[node];
      for (int t = st; t < st + cnt; ++t)
        if (ref_tri_hit(o[0], o[1], o[2], d[0], d[1], d[2], tm, B, t)) { found = true; break; }
    } else {
      if (top + 2 > 64) { atomicExch(overflow, 1); break; }
      stack[top] = B.left[node];
      stack[top + 1] = B.right[node];
      top += 2;
    }
  }
  hit[r] = found ? 1 : 0;
}


// ---------------------------------------------------------------------------
// the frame of an arbitrary QuadtreeAtlas (api.Scene, runtime.py:109-216):
// per-sample values <-> (m, side, side) part grids, recombination, shade
// ---------------------------------------------------------------------------

// dst (nch, D) (caller-zeroed: PAD cells stay 0) [c, flat_cells[i]] = src (nch, N) [c, i]
// (scatter_to_grids, transfer.py:128-132)
__global__ void k_atlas_scatter(const double* __restrict__ src, int nch, int N,
                                const int* __restrict__ flat_cells, int D, double* __restrict__ dst) {
  const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= (long long)nch * N) return;
  const int c = (int)(g / N), i = (int)(g % N);
  dst[(long long)c * D + flat_cells[i]] = src[g];
}

// out (3, D) = sum_k g[c, k] (vk[k, c] (+ vk2[k, c])), k ascending (the
// einsum "ck,kcd->cd" of runtime.py:204 over v_k + the folded ambient term)
__global__ void k_atlas_recombine(int K, int D, const double* __restrict__ vk,
                                  const double* __restrict__ vk2, const double* __restrict__ g,
                                  double* __restrict__ out) {
  const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= 3LL * D) return;
  const int c = (int)(q / D);
  const long long d = q % D;
  double acc = 0.0;
  for (int k = 0; k < K; ++k) {
    double v = vk[((long long)k * 3 + c) * D + d];
    if (vk2) v = dadd(v, vk2[((long long)k * 3 + c) * D + d]);
    acc = dadd(acc, dmul(g[c * K + k], v));
  }
  out[q] = acc;
}

// gather_from_grids (transfer.py:135-137) + _shade (runtime.py:162-168):
// radiance (N, 3) f64 = max(u, 0), u = scatter * (F_t(eta, cos) / pi)
__global__ void k_atlas_shade(int N, int D, const double* __restrict__ grids,
                              const int* __restrict__ flat_cells, const double* __restrict__ pos,
                              const double* __restrict__ nrm, const double* __restrict__ cam,
                              const double* __restrict__ material, double* __restrict__ radiance,
                              double* __restrict__ unclamped) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  double v[3] = {dsub(cam[0], pos[3 * i]), dsub(cam[1], pos[3 * i + 1]),
                 dsub(cam[2], pos[3 * i + 2])};
  const double nv = __dsqrt_rn(dadd(dadd(dmul(v[0], v[0]), dmul(v[1], v[1])), dmul(v[2], v[2])));
  v[0] = __ddiv_rn(v[0], nv);
  v[1] = __ddiv_rn(v[1], nv);
  v[2] = __ddiv_rn(v[2], nv);
  double cs = dadd(dadd(dmul(nrm[3 * i], v[0]), dmul(nrm[3 * i + 1], v[1])), dmul(nrm[3 * i + 2], v[2]));
  cs = fmin(fmax(cs, 0.0), 1.0);
  const double f = __ddiv_rn(ft_np(material[6], cs), 3.141592653589793);
  const int cell = flat_cells[i];
  for (int c = 0; c < 3; ++c) {
    const double u = dmul(grids[(long long)c * D + cell], f);
    unclamped[3 * i + c] = u;
    radiance[3 * i + c] = fmax(u, 0.0);
  }
}


// compress_energy's cut (wavelets.py:139-153) for nvec vectors whose squared
// magnitudes are given in descending-|v| order, stored transposed: sqT[i *
// nvec + v] (coalesced across vectors). kept[v] = the reference's
// searchsorted(cumsum, fraction * total, "left") + 1 with the SEQUENTIAL
// cumulative sums numpy forms, capped at the vector's nonzero count; 0 when
// fraction == 0 or total == 0.
__global__ void k_energy_cut(const double* __restrict__ sqT, int nvec, int D, double fraction,
                             const int* __restrict__ nnz, int* __restrict__ kept) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= nvec) return;
  double total = 0.0;
  for (int i = 0; i < D; ++i) total = dadd(total, sqT[(long long)i * nvec + v]);
  int k = 0;
  if (fraction != 0.0 && total != 0.0) {
    const double t = dmul(fraction, total);
    double cum = 0.0;
    int first = D;
    for (int i = 0; i < D; ++i) {
      cum = dadd(cum, sqT[(long long)i * nvec + v]);
      if (cum >= t) { first = i; break; }
    }
    k = first + 1;
    if (k > nnz[v]) k = nnz[v];
  }
  kept[v] = k;
}

}  // namespace sss
