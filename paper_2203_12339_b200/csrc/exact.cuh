// C5 exact pair pass (own translation unit: abi_exact.cu, see build.py).
#pragma once
#include "haar_tile.cuh"

namespace sss {

// ---------------------------------------------------------------------------
// C5 exact pair pass, K-fused and streamed by receiver-tile blocks:
// every (receiver, source) pair evaluates the training materials' fp32 R_d
// ONCE and projects them on all K terms in registers (b_k = sum_m P[k, m]
// R_d,m), x area, then the w0 Haar along sources per (row, k). D_block (K,
// nrt * T2, N) holds the step-1 rows of nrt receiver tiles for every term;
// nothing N^2-sized per term is materialised. One CTA per (source tile,
// receiver tile), RPP receiver rows per pass.
//
// The material loop is unrolled at compile time and every per-material
// constant (the projection row P[:, m] and the dipole constants) comes from
// the kernel's parameter bank, so the projection is FFMA reg x const + reg
// (the 2-register-read form that issues every cycle) and there are no
// shared-memory loads in the loop. Per material: 2 MUFU.RSQ + 2 MUFU.EX2.
// ---------------------------------------------------------------------------
constexpr int kExactMaxK = 16, kExactMaxM = 64;

struct ExactTables {
  // material pairs for the packed-FP32x2 loop: entry j = materials (2j, 2j+1)
  float2 pA[kExactMaxM / 2], pB[kExactMaxM / 2], pS[kExactMaxM / 2], ps[kExactMaxM / 2];
  float2 pCr[kExactMaxM / 2], pCv[kExactMaxM / 2];
  float2 pP[kExactMaxK * kExactMaxM / 2];  // pP[k * MM / 2 + j]
  float P[kExactMaxK * kExactMaxM];  // P[k * MM + m] = U/S projection (zero rows past K)
  // per material, with S = -sigma_tr log2(e), c = alpha' / (4 pi):
  float4 m0[kExactMaxM];  // {z_r^2, z_v^2, S, sigma_tr}
  float4 m1[kExactMaxM];  // {c z_r, c z_v, 0, 0}
};

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// packed FP32x2 (Blackwell FFMA2 / FMUL2 / FADD2): two fp32 lanes per 64-bit
// register pair, one issue slot
typedef unsigned long long f32x2_t;
__device__ __forceinline__ f32x2_t pk2(float lo, float hi) {
  f32x2_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ f32x2_t pk2(float2 v) { return pk2(v.x, v.y); }
__device__ __forceinline__ void upk2(f32x2_t r, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(r));
}
__device__ __forceinline__ f32x2_t add2(f32x2_t a, f32x2_t b) {
  f32x2_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f32x2_t mul2(f32x2_t a, f32x2_t b) {
  f32x2_t r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f32x2_t fma2(f32x2_t a, f32x2_t b, f32x2_t c) {
  f32x2_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}

__device__ __forceinline__ float rsqrt_approx(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <int L, int KT, int MM, bool X2 = false>
__global__ void __launch_bounds__(256) k_pair_rows_exact(const __grid_constant__ ExactTables tb,
                                                         const float* __restrict__ pos,
                                                         const float* __restrict__ area, int S,
                                                         float r_max, int rt0, int nrt,
                                                         double* __restrict__ D) {
  constexpr int T = 1 << L, T2 = T * T, LD = T2 + 1;
  constexpr int RPP = 1024 / T2 > 0 ? (1024 / T2 < 16 ? 1024 / T2 : 16) : 1;  // receiver rows per pass
  extern __shared__ double smx[];
  double* hrow = smx;  // (KT * RPP) x LD
  const int N = S * S, tpr = S / T;
  const int ST = blockIdx.x, RT = rt0 + blockIdx.y;
  const int str = ST / tpr, stc = ST % tpr, rtr = RT / tpr, rtc = RT % tpr;
  const size_t NR = (size_t)nrt * T2;
  for (int r0 = 0; r0 < T2; r0 += RPP) {
    for (int e = threadIdx.x; e < RPP * T2; e += blockDim.x) {
      const int o = r0 + e / T2, i = e % T2;
      const int oi = (rtr * T + o / T) * S + rtc * T + o % T;  // receiver point
      const int si = (str * T + i / T) * S + stc * T + i % T;  // source point
      const float dx = pos[oi * 3] - pos[si * 3];
      const float dy = pos[oi * 3 + 1] - pos[si * 3 + 1];
      const float dz = pos[oi * 3 + 2] - pos[si * 3 + 2];
      const float r2 = dx * dx + dy * dy + dz * dz;
      float acc[KT];
#pragma unroll
      for (int k = 0; k < KT; ++k) acc[k] = 0.0f;
      if (X2 && sqrtf(r2) <= r_max) {
        // two materials per step in packed FP32x2 (the 4 MUFU ops per
        // material stay scalar); per term even / odd materials accumulate
        // separately and are added at the end
        const f32x2_t r22 = pk2(r2, r2);
        f32x2_t acc2[KT];
#pragma unroll
        for (int k = 0; k < KT; ++k) acc2[k] = 0ull;
#pragma unroll
        for (int j = 0; j < MM / 2; ++j) {
          const f32x2_t ar2 = add2(r22, pk2(tb.pA[j])), av2 = add2(r22, pk2(tb.pB[j]));
          float ar0, ar1, av0, av1;
          upk2(ar2, ar0, ar1);
          upk2(av2, av0, av1);
          const f32x2_t ir2 = pk2(rsqrt_approx(ar0), rsqrt_approx(ar1));
          const f32x2_t iv2 = pk2(rsqrt_approx(av0), rsqrt_approx(av1));
          float xr0, xr1, xv0, xv1;
          upk2(mul2(mul2(ar2, pk2(tb.pS[j])), ir2), xr0, xr1);
          upk2(mul2(mul2(av2, pk2(tb.pS[j])), iv2), xv0, xv1);
          const f32x2_t er2 = pk2(ex2_approx(xr0), ex2_approx(xr1));
          const f32x2_t ev2 = pk2(ex2_approx(xv0), ex2_approx(xv1));
          const f32x2_t tr2 = mul2(mul2(mul2(mul2(add2(ir2, pk2(tb.ps[j])), pk2(tb.pCr[j])), er2), ir2), ir2);
          const f32x2_t tv2 = mul2(mul2(mul2(mul2(add2(iv2, pk2(tb.ps[j])), pk2(tb.pCv[j])), ev2), iv2), iv2);
          const f32x2_t rd2 = add2(tr2, tv2);
#pragma unroll
          for (int k = 0; k < KT; ++k) acc2[k] = fma2(pk2(tb.pP[k * (MM / 2) + j]), rd2, acc2[k]);
        }
#pragma unroll
        for (int k = 0; k < KT; ++k) {
          float lo, hi;
          upk2(acc2[k], lo, hi);
          acc[k] = lo + hi;
        }
      } else if (!X2 && sqrtf(r2) <= r_max) {
#pragma unroll
        for (int m = 0; m < MM; ++m) {
          // R_d = c z_r (s + 1/d_r) e^{-s d_r} / d_r^2 + (the same at z_v),
          // d^2 = r^2 + z^2: 1/d = rsqrt(d^2), s d = S d^2 / d (in log2 units)
          // one parameter-bank operand per instruction (no LDC into registers)
          const float4 a = tb.m0[m], b = tb.m1[m];
          const float ar = r2 + a.x, av = r2 + a.y;
          const float ir = rsqrt_approx(ar), iv = rsqrt_approx(av);
          const float er = ex2_approx((ar * a.z) * ir), ev = ex2_approx((av * a.z) * iv);
          const float tr = ((ir + a.w) * b.x) * er * (ir * ir);
          const float tv = ((iv + a.w) * b.y) * ev * (iv * iv);
          const float rd = tr + tv;
#pragma unroll
          for (int k = 0; k < KT; ++k) acc[k] = fmaf(tb.P[k * MM + m], rd, acc[k]);
        }
      }
      const float ar_ = area[si];
#pragma unroll
      for (int k = 0; k < KT; ++k) hrow[(k * RPP + (o - r0)) * LD + i] = (double)(acc[k] * ar_);
    }
    __syncthreads();
    // w0 Haar along sources: one (term, receiver row) per thread
    for (int j = threadIdx.x; j < KT * RPP; j += blockDim.x) seq_haar_fwd<T>(hrow + j * LD, 1);
    __syncthreads();
    for (int e = threadIdx.x; e < KT * RPP * T2; e += blockDim.x) {
      const int j = e / T2, c = e % T2, k = j / RPP, o = r0 + j % RPP;
      D[((size_t)k * NR + (size_t)(RT - rt0) * T2 + o) * N + (size_t)ST * T2 + c] = hrow[j * LD + c];
    }
    __syncthreads();
  }
}

}  // namespace sss
