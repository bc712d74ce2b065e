// Shared device helpers for the sm_100a relight / material-edit path.
//
// Index spaces (geometry image = identity atlas):
//   * w0 / w1 "flat" index = r * S + c of the L-level Mallat layout of the
//     S x S grid (the reference's domain, transfer.py:122-151).
//   * tile-major index = tile * T^2 + (lr * T + lc), T = 2^L, where (lr, lc)
//     is the position inside the tile's own L-level (= full-pyramid) Mallat
//     layout. The L-level transform is tile-local, so a CTA that owns a tile
//     owns every coefficient it needs for the inverse (the fused epilogue).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define SSS_ISQRT2 0.7071067811865475  // 1/sqrt(2) as the reference rounds it

namespace sss {

// Programmatic dependent launch (the frame's kernel chain, abi_util.cuh
// launch_chain): a kernel lets its successor's CTAs be scheduled as soon as
// all of its own have started (pdl_launch_dependents, first statement), and
// touches global memory only after its predecessor has completed and flushed
// (pdl_wait). Launch latency, CTA scheduling and shared-memory set-up of
// kernel n + 1 overlap the tail of kernel n; without the launch attribute
// both are no-ops.
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// exact-order double arithmetic (no FMA contraction) so results are bitwise
// equal to the numpy reference (_kernels_np.py, no fused multiply-add)
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }

// local tile position (lr, lc) of an L-level tile (tile side T = 1 << L) ->
// global Mallat (row, col) of an S x S grid, tile (tr, tc)
__device__ __forceinline__ void local_to_global(int lr, int lc, int tr, int tc,
                                                int L, int S, int* gr, int* gc) {
  const int T = 1 << L;
  int hl = 1, hg = S >> L;
  for (int l = 1; l <= L; ++l) {
    const int h = T >> l;
    if (lr >= h || lc >= h) { hl = h; hg = S >> l; break; }
  }
  *gr = (lr >= hl) ? hg + tr * hl + (lr - hl) : tr * hl + lr;
  *gc = (lc >= hl) ? hg + tc * hl + (lc - hl) : tc * hl + lc;
}

// global Mallat (r, c) -> (tile id, local index lr*T+lc)
__device__ __forceinline__ void global_to_tile(int r, int c, int L, int S,
                                               int* tile, int* local) {
  const int T = 1 << L;
  int hg = S >> L, hl = 1;  // LL band by default
  for (int l = 1; l <= L; ++l) {
    const int h = S >> l;
    if (r >= h || c >= h) { hg = h; hl = T >> l; break; }
  }
  const int pr = (r >= hg) ? r - hg : r;
  const int pc = (c >= hg) ? c - hg : c;
  const int tr = pr / hl, tc = pc / hl;
  const int lr = (r >= hg ? hl : 0) + pr % hl;
  const int lc = (c >= hg ? hl : 0) + pc % hl;
  *tile = tr * (S / T) + tc;
  *local = lr * T + lc;
}

// In-place forward full-pyramid Haar of a T x T tile held in shared memory
// (row-major, stride T), following haar2d_fwd_batch (_kernels_np.py:53-62):
// per level rows then columns. Called by all threads of the block; uses
// `tmp` (T*T doubles) as scratch. Bitwise equal to the reference.
// Per level the row pass writes the level's s x s block into tmp and the
// column pass reads it back into a (two passes, two barriers; no copy-back),
// indices by shifts (all sizes are powers of two). The per-element
// arithmetic (dadd / dmul order) is the reference's, so results are bitwise
// those of haar2d_fwd_batch / haar2d_inv_batch.
__device__ __forceinline__ int ilog2i(int v) { return 31 - __clz(v); }

__device__ inline void tile_haar_fwd(double* a, double* tmp, int T, int nthreads, int tid) {
  for (int s = T; s >= 2; s >>= 1) {
    const int h = s >> 1, lh = ilog2i(h);
    for (int e = tid; e < s * h; e += nthreads) {  // rows a -> tmp
      const int i = e >> lh, j = e & (h - 1);
      const double ev = a[i * T + 2 * j], od = a[i * T + 2 * j + 1];
      tmp[i * T + j] = dmul(dadd(ev, od), SSS_ISQRT2);
      tmp[i * T + h + j] = dmul(dsub(ev, od), SSS_ISQRT2);
    }
    __syncthreads();
    for (int e = tid; e < s * h; e += nthreads) {  // columns tmp -> a
      const int i = e >> (lh + 1), j = e & (2 * h - 1);  // j (of s) fastest: no bank conflicts
      const double ev = tmp[(2 * i) * T + j], od = tmp[(2 * i + 1) * T + j];
      a[i * T + j] = dmul(dadd(ev, od), SSS_ISQRT2);
      a[(h + i) * T + j] = dmul(dsub(ev, od), SSS_ISQRT2);
    }
    __syncthreads();
  }
}

// In-place inverse (haar2d_inv_batch, _kernels_np.py:65-74): per level
// columns then rows, s = 2 .. T.
__device__ inline void tile_haar_inv(double* a, double* tmp, int T, int nthreads, int tid) {
  for (int s = 2; s <= T; s <<= 1) {
    const int h = s >> 1, lh = ilog2i(h);
    for (int e = tid; e < s * h; e += nthreads) {  // columns a -> tmp
      const int i = e >> (lh + 1), j = e & (2 * h - 1);  // j (of s) fastest: no bank conflicts
      const double lo = a[i * T + j], hi = a[(h + i) * T + j];
      tmp[(2 * i) * T + j] = dmul(dadd(lo, hi), SSS_ISQRT2);
      tmp[(2 * i + 1) * T + j] = dmul(dsub(lo, hi), SSS_ISQRT2);
    }
    __syncthreads();
    for (int e = tid; e < s * h; e += nthreads) {  // rows tmp -> a
      const int i = e >> lh, j = e & (h - 1);
      const double lo = tmp[i * T + j], hi = tmp[i * T + h + j];
      a[i * T + 2 * j] = dmul(dadd(lo, hi), SSS_ISQRT2);
      a[i * T + 2 * j + 1] = dmul(dsub(lo, hi), SSS_ISQRT2);
    }
    __syncthreads();
  }
}

// Batched in-place forward full-pyramid Haar over B independent T x T grids
// (grid b at a + b * T * T); same arithmetic as tile_haar_fwd. tmp: B * T * T.
__device__ inline void batch_tile_haar_fwd(double* a, double* tmp, int T, int B) {
  const int T2 = T * T, nt = blockDim.x, tid = threadIdx.x;
  for (int s = T; s >= 2; s >>= 1) {
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
}

// Batched in-place inverse over B independent T x T grids (grid b at
// a + b * T * T); same arithmetic as tile_haar_inv. tmp: B * T * T doubles.
__device__ inline void batch_tile_haar_inv(double* a, double* tmp, int T, int B) {
  const int T2 = T * T, nt = blockDim.x, tid = threadIdx.x;
  for (int s = 2; s <= T; s <<= 1) {
    const int h = s >> 1, lh = ilog2i(h), lsh = ilog2i(s * h);
    for (int q = tid; q < (B << lsh); q += nt) {
      const int b = q >> lsh, e = q & ((1 << lsh) - 1);
      const int i = e >> (lh + 1), j = e & (2 * h - 1);  // j (of s) fastest: no bank conflicts
      const double* g = a + b * T2;
      double* o = tmp + b * T2;
      const double lo = g[i * T + j], hi = g[(h + i) * T + j];
      o[(2 * i) * T + j] = dmul(dadd(lo, hi), SSS_ISQRT2);
      o[(2 * i + 1) * T + j] = dmul(dsub(lo, hi), SSS_ISQRT2);
    }
    __syncthreads();
    for (int q = tid; q < (B << lsh); q += nt) {
      const int b = q >> lsh, e = q & ((1 << lsh) - 1);
      const int i = e >> lh, j = e & (h - 1);
      const double* g = tmp + b * T2;
      double* o = a + b * T2;
      const double lo = g[i * T + j], hi = g[i * T + h + j];
      o[i * T + 2 * j] = dmul(dadd(lo, hi), SSS_ISQRT2);
      o[i * T + 2 * j + 1] = dmul(dsub(lo, hi), SSS_ISQRT2);
    }
    __syncthreads();
  }
}

// F_t(eta, cos) = 1 - F_r, dipole.py:135-152
__device__ __forceinline__ double fresnel_transmittance(double eta, double ci) {
  ci = fmin(fmax(ci, 0.0), 1.0);
  if (eta == 1.0) return 1.0;
  const double sin2_t = (1.0 - ci * ci) / (eta * eta);
  if (sin2_t >= 1.0) return 0.0;
  const double ct = sqrt(fmax(1.0 - sin2_t, 0.0));
  const double rs = (ci - eta * ct) / (ci + eta * ct + 1e-300);
  const double rp = (eta * ci - ct) / (eta * ci + ct + 1e-300);
  const double ft = 1.0 - 0.5 * (rs * rs + rp * rp);
  return fmin(fmax(ft, 0.0), 1.0);
}

// Jensen dipole R_d (dipole.py:100-132) for one channel
struct Dipole {
  double alpha_prime, sigma_tr, z_r, z_v;
};

__device__ __forceinline__ Dipole derive_dipole(double sp, double sa, double eta) {
  const double st = sp + sa;
  const double f = -1.440 / (eta * eta) + 0.710 / eta + 0.668 + 0.0636 * eta;
  const double a = (1.0 + f) / (1.0 - f);
  Dipole d;
  d.alpha_prime = sp / st;
  d.sigma_tr = sqrt(3.0 * sa * st);
  d.z_r = 1.0 / st;
  d.z_v = d.z_r * (1.0 + 4.0 * a / 3.0);
  return d;
}

__device__ __forceinline__ double eval_rd(const Dipole& d, double r) {
  const double dr = sqrt(r * r + d.z_r * d.z_r);
  const double dv = sqrt(r * r + d.z_v * d.z_v);
  const double s = d.sigma_tr;
  const double tr = d.z_r * (s + 1.0 / dr) * exp(-s * dr) / (dr * dr);
  const double tv = d.z_v * (s + 1.0 / dv) * exp(-s * dv) / (dv * dv);
  return d.alpha_prime / (4.0 * 3.141592653589793) * (tr + tv);
}

}  // namespace sss

// ---------------------------------------------------------------------------
// TMA bulk copies (cp.async.bulk, no tensor map) + mbarrier transaction
// tracking, sm_90+ / sm_100a
// ---------------------------------------------------------------------------
namespace sss {

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

// global -> shared bulk copy; bytes and both addresses 16-byte aligned
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// warp-level wait: only lane 0 polls the barrier (with a suspend-time hint),
// the other lanes park on __syncwarp, so 16+ waiting warps do not flood the
// SM's barrier unit that also signals TMA transaction completion
__device__ __forceinline__ void mbar_wait_warp(uint64_t* bar, unsigned parity) {
  if ((threadIdx.x & 31) == 0) {
    asm volatile(
        "{\n .reg .pred p;\n WAITW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, "
        "%2;\n @!p bra WAITW_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(0x10000u)
        : "memory");
  }
  __syncwarp();
}

// warp-level wait without a suspend-time hint (lane 0 spins on try_wait)
__device__ __forceinline__ void mbar_wait_warp_spin(uint64_t* bar, unsigned parity) {
  if ((threadIdx.x & 31) == 0) {
    asm volatile(
        "{\n .reg .pred p;\n WAITS_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n "
        "@!p bra WAITS_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
  }
  __syncwarp();
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra "
      "WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

}  // namespace sss
