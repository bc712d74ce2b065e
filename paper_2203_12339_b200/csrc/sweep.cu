// C4 batched material sweep (BASELINE configs[3]):
//   out[c][m][n] = max(0, F_t(eta_m, cos_n) / pi * sum_k B[c][n][k] G[c][m][k])
// for M materials at once against the cached per-term transfer output
// (B_k = w1^-1 v_k, shared by every material), bf16 inputs, fp32 accumulate.
// Reference semantics: runtime.py:202-216 (_finish: recombine, inverse, shade)
// evaluated for a batch of materials; project_material basisgen.py:172-191.
//
// k_sweep_umma: one CTA per (128-point tile, channel). The 128 x 16 B tile and
// the M x 16 G block are staged in shared memory in the canonical K-major
// no-swizzle UMMA layout (8-row x 16-byte core matrices), one elected thread
// issues a single tcgen05.mma.cta_group::1.kind::f16 (M=128, N=M, K=16) into a
// TMEM accumulator and commits it to an mbarrier; the 4 warps then read their
// 32-lane quarter with tcgen05.ld.32x32b and shade. F_t(eta, cos) is smooth in
// eta on [eta_lo, eta_hi]: each thread (one point) fits it with a cubic in
// eta from 4 exact Chebyshev-node evaluations, so the per-element shade is 3
// FMAs; outputs are per-material images, one coalesced 128-byte store per
// (warp, material). Bound: the HBM write of the fp32 output.
#include <cuda_bf16.h>

#include "sss_common.cuh"

namespace sss {

constexpr int kSweepTileM = 128;
constexpr int kSweepK = 16;  // PCA terms padded to the bf16 UMMA K

// byte offset of element (row, k) of a rows x 16 bf16 K-major operand in the
// canonical no-swizzle layout: core matrix (row / 8, k / 8) = 8 rows x 16 B,
// LBO (k-chunk stride) = 128 B, SBO (8-row-group stride) = 256 B
__device__ __forceinline__ uint32_t umma_kmajor_off(int row, int k) {
  return (uint32_t)((row >> 3) * 256 + (k >> 3) * 128 + (row & 7) * 16 + (k & 7) * 2);
}

__device__ __forceinline__ uint64_t umma_smem_desc(const void* base) {
  const uint64_t addr = smem_u32(base);
  uint64_t d = (addr >> 4) & 0x3fffull;   // start address, 16-byte units
  d |= (uint64_t)(128 >> 4) << 16;        // leading byte offset (K direction)
  d |= (uint64_t)(256 >> 4) << 32;        // stride byte offset (M/N direction)
  d |= 1ull << 46;                        // descriptor version (sm_100)
  return d;                               // layout type 0 = SWIZZLE_NONE, base offset 0
}

// instruction descriptor: D f32, A/B bf16, both K-major, M = 128, N = n
__host__ __device__ constexpr uint32_t umma_idesc_bf16(int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

__device__ __forceinline__ float ft_exit_f(float eta, float ci) {
  ci = fminf(fmaxf(ci, 0.0f), 1.0f);
  const float sin2_t = (1.0f - ci * ci) / (eta * eta);
  if (sin2_t >= 1.0f) return 0.0f;
  const float ct = sqrtf(fmaxf(1.0f - sin2_t, 0.0f));
  const float rs = __fdividef(ci - eta * ct, ci + eta * ct + 1e-30f);
  const float rp = __fdividef(eta * ci - ct, eta * ci + ct + 1e-30f);
  return fminf(fmaxf(1.0f - 0.5f * (rs * rs + rp * rp), 0.0f), 1.0f);
}

// SWEEP_M materials per MMA (N of the UMMA): multiple of 16, <= 256.
// THREADS = 128 or 256: warp w reads TMEM lane quarter w % 4 (a tile row per
// lane); with 256 threads the two warps of a quarter split the columns.
// NC > 0: the point count is the compile-time constant NC (the 256^2 sweep),
// so the per-material store offsets j * N become STG immediates (no 64-bit
// address arithmetic per element)
template <int SWEEP_M, int THREADS, int NC = 0>
__global__ void __launch_bounds__(THREADS) k_sweep_umma(
    int N_rt, int M_total, const __nv_bfloat16* __restrict__ Bq /* (3, N, 16) */,
    const __nv_bfloat16* __restrict__ Gq /* (3, M_total, 16) */,
    const float* __restrict__ eta /* (M_total) */, float eta_lo, float eta_hi,
    const float* __restrict__ positions, const float* __restrict__ normals,
    const double* __restrict__ cam, float* __restrict__ out /* (3, M_total, N) */) {
  static_assert(SWEEP_M % 16 == 0 && SWEEP_M <= 256, "UMMA N");
  const int N = NC > 0 ? NC : N_rt;
  constexpr int TMEM_COLS = SWEEP_M <= 32 ? 32 : SWEEP_M <= 64 ? 64 : SWEEP_M <= 128 ? 128 : 256;
  extern __shared__ __align__(1024) uint8_t sw_smem[];
  uint8_t* sA = sw_smem;                                   // 128 x 16 bf16 = 4 KB
  uint8_t* sB = sw_smem + kSweepTileM * kSweepK * 2;       // SWEEP_M x 16 bf16
  float* st = reinterpret_cast<float*>(sB + SWEEP_M * kSweepK * 2);  // SWEEP_M (eta -> t)
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int c = blockIdx.y;
  const int p0 = blockIdx.x * kSweepTileM;
  const int m0 = blockIdx.z * SWEEP_M;
  const int nm = min(SWEEP_M, M_total - m0);

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base)),
                 "n"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  // operands -> canonical layout (16-byte chunks: one k-chunk of one row)
  {
    const uint4* gA = reinterpret_cast<const uint4*>(Bq + ((size_t)c * N + p0) * kSweepK);
    for (int q = tid; q < kSweepTileM * 2; q += blockDim.x) {
      const int row = q >> 1, kc = q & 1;
      const uint4 v = (p0 + row < N) ? gA[q] : make_uint4(0u, 0u, 0u, 0u);
      *reinterpret_cast<uint4*>(sA + umma_kmajor_off(row, kc * 8)) = v;
    }
    const uint4* gB = reinterpret_cast<const uint4*>(Gq + ((size_t)c * M_total + m0) * kSweepK);
    for (int q = tid; q < SWEEP_M * 2; q += blockDim.x) {
      const int row = q >> 1, kc = q & 1;
      const uint4 v = row < nm ? gB[q] : make_uint4(0u, 0u, 0u, 0u);
      *reinterpret_cast<uint4*>(sB + umma_kmajor_off(row, kc * 8)) = v;
    }
    const float mid = 0.5f * (eta_lo + eta_hi), half = fmaxf(0.5f * (eta_hi - eta_lo), 1e-6f);
    for (int m = tid; m < SWEEP_M; m += blockDim.x)
      st[m] = m < nm ? (eta[m0 + m] - mid) / half : 0.0f;
  }
  // generic-proxy smem writes -> visible to the tensor core (async proxy)
  fence_proxy_async();
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  if (tid == 0) {
    const uint64_t da = umma_smem_desc(sA), db = umma_smem_desc(sB);
    const uint32_t idesc = umma_idesc_bf16(SWEEP_M);
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
        "l"(da), "l"(db), "r"(idesc), "r"(0));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(&bar))
                 : "memory");
  }
  // per-point Fresnel fit while the MMA runs: F(t) = a0 + a1 t + a2 t^2 + a3 t^3
  const int quarter = warp & 3, colhalf = warp >> 2;
  constexpr int NCOL = SWEEP_M / (THREADS / 128);  // columns read by this warp
  const int p = p0 + quarter * 32 + lane;  // TMEM lane = tile row
  float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
  if (p < N) {
    const double px = positions[p * 3], py = positions[p * 3 + 1], pz = positions[p * 3 + 2];
    double vx = cam[0] - px, vy = cam[1] - py, vz = cam[2] - pz;
    const double inv = 1.0 / sqrt(vx * vx + vy * vy + vz * vz);
    const float cs = (float)(((double)normals[p * 3] * vx + (double)normals[p * 3 + 1] * vy +
                              (double)normals[p * 3 + 2] * vz) * inv);
    const float mid = 0.5f * (eta_lo + eta_hi), half = fmaxf(0.5f * (eta_hi - eta_lo), 1e-6f);
    // Chebyshev nodes t_j = cos((2j+1) pi / 8), coefficients by the discrete cosine sum
    float f[4];
    const float tj[4] = {0.92387953f, 0.38268343f, -0.38268343f, -0.92387953f};
#pragma unroll
    for (int j = 0; j < 4; ++j) f[j] = ft_exit_f(mid + half * tj[j], cs);
    // DCT-II of the node values: cos(q (2j+1) pi / 8)
    constexpr float kC1 = 0.92387953f, kC2 = 0.70710678f, kC3 = 0.38268343f;
    float ch[4];
    ch[0] = 0.25f * (f[0] + f[1] + f[2] + f[3]);
    ch[1] = 0.5f * (kC1 * (f[0] - f[3]) + kC3 * (f[1] - f[2]));
    ch[2] = 0.5f * kC2 * (f[0] - f[1] - f[2] + f[3]);
    ch[3] = 0.5f * (kC3 * (f[0] - f[3]) - kC1 * (f[1] - f[2]));
    const float ip = 0.318309886f;  // 1 / pi
    a0 = (ch[0] - ch[2]) * ip;
    a1 = (ch[1] - 3.f * ch[3]) * ip;
    a2 = (2.f * ch[2]) * ip;
    a3 = (4.f * ch[3]) * ip;
  }
  mbar_wait(&bar, 0u);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  float* oc = out + (size_t)c * M_total * N;
#pragma unroll 1
  for (int j0 = colhalf * NCOL; j0 < (colhalf + 1) * NCOL; j0 += 32) {
    uint32_t r[32];
    const uint32_t taddr = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)j0;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
        "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
          "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
          "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    if (p < N) {
      float* o = oc + (size_t)(m0 + j0) * N + p;
      if (j0 + 32 <= nm) {  // full chunk: no per-element bounds checks
        const float4* t4 = reinterpret_cast<const float4*>(st + j0);
        // two materials per packed FP32x2 instruction (FFMA2 / FMUL2): the
        // cubic in t and the scale, then clamp and store per element
        unsigned long long A0, A1, A2, A3;
        asm("mov.b64 %0, {%1, %1};" : "=l"(A0) : "f"(a0));
        asm("mov.b64 %0, {%1, %1};" : "=l"(A1) : "f"(a1));
        asm("mov.b64 %0, {%1, %1};" : "=l"(A2) : "f"(a2));
        asm("mov.b64 %0, {%1, %1};" : "=l"(A3) : "f"(a3));
        const unsigned long long* t2 = reinterpret_cast<const unsigned long long*>(st + j0);
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const unsigned long long T = t2[q];
          unsigned long long f, v;
          asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(f) : "l"(A3), "l"(T), "l"(A2));
          asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(f) : "l"(f), "l"(T), "l"(A1));
          asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(f) : "l"(f), "l"(T), "l"(A0));
          unsigned long long rr;
          asm("mov.b64 %0, {%1, %2};" : "=l"(rr) : "r"(r[2 * q]), "r"(r[2 * q + 1]));
          asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(v) : "l"(f), "l"(rr));
          float v0, v1;
          asm("mov.b64 {%0, %1}, %2;" : "=f"(v0), "=f"(v1) : "l"(v));
          if (NC > 0) {
            __stcs(o + (size_t)(2 * q) * NC, fmaxf(v0, 0.0f));
            __stcs(o + (size_t)(2 * q + 1) * NC, fmaxf(v1, 0.0f));
          } else {
            __stcs(o, fmaxf(v0, 0.0f));
            o += N;
            __stcs(o, fmaxf(v1, 0.0f));
            o += N;
          }
        }
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          if (j0 + j < nm) {
            const float t = st[j0 + j];
            const float ft = fmaf(fmaf(fmaf(a3, t, a2), t, a1), t, a0);
            __stcs(o, fmaxf(ft * __uint_as_float(r[j]), 0.0f));
          }
          o += N;
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "n"(TMEM_COLS));
}

// B[c][n][k] = (w1^-1 v_k[c])[n] as bf16, k padded to 16: CTA per 2^L tile,
// one batched inverse Haar over the 3K tile grids of the cached v_k
__global__ void k_sweep_basis(int K, int S, int L, const double* __restrict__ vk /* (K,3,N) tm */,
                              __nv_bfloat16* __restrict__ Bq /* (3, N, 16) flat points */) {
  extern __shared__ double sb[];
  const int T = 1 << L, T2 = T * T, N = S * S, tpr = S / T;
  double* a = sb;               // 3K x T2
  double* tmp = sb + 3 * K * T2;
  const int tile = blockIdx.x, tr = tile / tpr, tc = tile % tpr;
  for (int q = threadIdx.x; q < 3 * K * T2; q += blockDim.x) {
    const int g = q / T2, e = q % T2;  // g = k * 3 + c
    a[q] = vk[(size_t)g * N + (size_t)tile * T2 + e];
  }
  __syncthreads();
  batch_tile_haar_inv(a, tmp, T, 3 * K);
  for (int q = threadIdx.x; q < 3 * T2 * kSweepK; q += blockDim.x) {
    const int k = q % kSweepK, e = (q / kSweepK) % T2, c = q / (kSweepK * T2);
    const int i = (tr * T + e / T) * S + tc * T + e % T;
    const double v = k < K ? a[(k * 3 + c) * T2 + e] : 0.0;
    Bq[((size_t)c * N + i) * kSweepK + k] = __double2bfloat16(v);
  }
}

// project_material for a batch of materials (basisgen.py:172-191): block
// (channel, material); materials (M, 7) = {sp[3], sa[3], eta}; writes the
// fp64 weights (M, 3, K) and the bf16 G operand (3, M, 16)
__global__ void k_material_weights_batch(const double* __restrict__ bw, const double* __restrict__ r_nodes,
                                         int K, int nr, int M, const double* __restrict__ materials,
                                         double* __restrict__ g64, __nv_bfloat16* __restrict__ Gq,
                                         float* __restrict__ eta_f) {
  __shared__ double red[32][16];
  const int c = blockIdx.x, m = blockIdx.y;
  const double* mat = materials + (size_t)m * 7;
  if (c == 0 && threadIdx.x == 0 && eta_f) eta_f[m] = (float)mat[6];
  const Dipole d = derive_dipole(mat[c], mat[3 + c], mat[6]);
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
  if (threadIdx.x < kSweepK) {
    double s = 0.0;
    if (threadIdx.x < K) {
      for (int w = 0; w < nw; ++w) s += red[w][threadIdx.x];
      if (g64) g64[((size_t)m * 3 + c) * K + threadIdx.x] = s;
    }
    Gq[((size_t)c * M + m) * kSweepK + threadIdx.x] = __double2bfloat16(s);
  }
}

}  // namespace sss
