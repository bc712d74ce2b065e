// Abandoned transfer layouts v1 (k_transfer_relight) and v2 (k_transfer_banded),
// moved out of csrc/frame.cu; not built.
#include "../../paper_2203_12339_b200/csrc/sss_common.cuh"
namespace sss {
// ---------------------------------------------------------------------------
// (b)+(c) fused transfer: CTA per tile, K loop, row-major CSR per k over
// tile-major rows; v_k cached for edits; epilogue recombines, inverts, shades
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_transfer_relight(
    int K, int S, int L, const uint64_t* __restrict__ rowptr /* K x (N+1) */,
    const uint32_t* __restrict__ cols, const float* __restrict__ vals,
    const double* __restrict__ x /* 3 x N, flat w0 */, const double* __restrict__ g /* 3 x K */,
    const float* __restrict__ positions, const float* __restrict__ normals,
    const double* __restrict__ cam, const double* __restrict__ material,
    double* __restrict__ vk /* K x 3 x N tile-major */,
    double* __restrict__ scatter, float* __restrict__ radiance, float* __restrict__ radiance_unclamped) {
  extern __shared__ double sm[];
  const int T = 1 << L, T2 = T * T, N = S * S;
  double* summed = sm;            // 3 * T2
  double* tmp = sm + 3 * T2;      // T2
  const int tile = blockIdx.x;
  const int tiles_per_row = S / T;
  const int tr = tile / tiles_per_row, tc = tile % tiles_per_row;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const double* x0 = x;
  const double* x1 = x + N;
  const double* x2 = x + 2 * N;
  for (int e = threadIdx.x; e < 3 * T2; e += blockDim.x) summed[e] = 0.0;
  __syncthreads();
  for (int k = 0; k < K; ++k) {
    const uint64_t* rp = rowptr + (size_t)k * (N + 1);
    const double g0 = g[k], g1 = g[K + k], g2 = g[2 * K + k];
    for (int lr = wid; lr < T2; lr += nw) {
      const int row = tile * T2 + lr;
      const uint64_t b = rp[row], e = rp[row + 1];
      double a0 = 0.0, a1 = 0.0, a2 = 0.0;
      for (uint64_t p = b + lane; p < e; p += 32) {
        const uint32_t col = __ldg(&cols[p]);
        const double v = (double)__ldg(&vals[p]);
        a0 = fma(v, __ldg(&x0[col]), a0);
        a1 = fma(v, __ldg(&x1[col]), a1);
        a2 = fma(v, __ldg(&x2[col]), a2);
      }
      for (int o = 16; o > 0; o >>= 1) {
        a0 += __shfl_xor_sync(0xffffffffu, a0, o);
        a1 += __shfl_xor_sync(0xffffffffu, a1, o);
        a2 += __shfl_xor_sync(0xffffffffu, a2, o);
      }
      if (lane == 0) {
        double* vo = vk + (size_t)k * 3 * N;
        vo[row] = a0; vo[N + row] = a1; vo[2 * N + row] = a2;
        summed[lr] += g0 * a0;
        summed[T2 + lr] += g1 * a1;
        summed[2 * T2 + lr] += g2 * a2;
      }
    }
  }
  __syncthreads();
  tile_epilogue(summed, tmp, T, tr, tc, S, positions, normals, cam, material, scatter, radiance,
                radiance_unclamped);
}

}  // namespace sss

namespace sss {

// ---------------------------------------------------------------------------
// (b)+(c) fused transfer, frame layout v2 ("banded"): a CTA owns a unit of
// G tiles (R = G * 4^L rows, one thread per row, rows visited longest-first
// so a warp's rows have similar lengths); the masked E spectrum x is staged
// in shared memory one column band at a time (band_width tile-major w0 ids,
// fp64, 3 channels) and every row's entries inside the band are streamed
// with register accumulation for all K terms (no atomics, no shuffles, no
// L2 gathers). Epilogue: v_k cache write, sum_k g_k v_k, per-tile inverse
// Haar + Fresnel shade.
// ---------------------------------------------------------------------------
template <int KMAX>
__global__ void __launch_bounds__(256) k_transfer_banded(
    int K, int S, int L, int G, const uint64_t* __restrict__ rowptr,
    const uint32_t* __restrict__ bandoff, int band_width, int NB,
    const int* __restrict__ rowperm, const uint32_t* __restrict__ cols,
    const float* __restrict__ vals, const double* __restrict__ x, const double* __restrict__ g,
    const float* __restrict__ positions, const float* __restrict__ normals,
    const double* __restrict__ cam, const double* __restrict__ material,
    double* __restrict__ vk, double* __restrict__ scatter, float* __restrict__ radiance,
    float* __restrict__ radiance_unclamped) {
  extern __shared__ double sm[];
  const int T = 1 << L, T2 = T * T, N = S * S;
  const int R = G * T2;
  double* xs = sm;                          // 3 * band_width
  double* summed = xs + 3 * band_width;     // G * 3 * T2
  double* tmp = summed + 3 * R;             // T2
  const int unit = blockIdx.x;
  const int t = threadIdx.x;
  const int row = rowperm[unit * R + t];
  const int lr = row - unit * R;
  double acc[KMAX][3];
  uint64_t base[KMAX];
#pragma unroll
  for (int k = 0; k < KMAX; ++k) {
    acc[k][0] = acc[k][1] = acc[k][2] = 0.0;
    base[k] = k < K ? rowptr[(size_t)k * (N + 1) + row] : 0;
  }
  for (int b = 0; b < NB; ++b) {
    const int c0 = b * band_width;
    const int bw = min(band_width, N - c0);
    __syncthreads();
    for (int j = t; j < bw; j += blockDim.x) {
      xs[j] = x[c0 + j];
      xs[band_width + j] = x[N + c0 + j];
      xs[2 * band_width + j] = x[2 * N + c0 + j];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < KMAX; ++k) {
      if (k >= K) break;
      const uint32_t* bo = bandoff + ((size_t)k * N + row) * (NB + 1) + b;
      const uint64_t p0 = base[k] + bo[0], p1 = base[k] + bo[1];
      double a0 = acc[k][0], a1 = acc[k][1], a2 = acc[k][2];
#pragma unroll 4
      for (uint64_t p = p0; p < p1; ++p) {
        const int col = (int)__ldg(&cols[p]) - c0;
        const double v = (double)__ldg(&vals[p]);
        a0 = fma(v, xs[col], a0);
        a1 = fma(v, xs[band_width + col], a1);
        a2 = fma(v, xs[2 * band_width + col], a2);
      }
      acc[k][0] = a0; acc[k][1] = a1; acc[k][2] = a2;
    }
  }
  double s0 = 0.0, s1 = 0.0, s2 = 0.0;
#pragma unroll
  for (int k = 0; k < KMAX; ++k) {
    if (k >= K) break;
    double* vo = vk + (size_t)k * 3 * N;
    vo[row] = acc[k][0]; vo[N + row] = acc[k][1]; vo[2 * N + row] = acc[k][2];
    s0 += g[k] * acc[k][0];
    s1 += g[K + k] * acc[k][1];
    s2 += g[2 * K + k] * acc[k][2];
  }
  const int tj = lr / T2, e = lr % T2;
  summed[(tj * 3 + 0) * T2 + e] = s0;
  summed[(tj * 3 + 1) * T2 + e] = s1;
  summed[(tj * 3 + 2) * T2 + e] = s2;
  __syncthreads();
  const int tiles_per_row = S / T;
  for (int j = 0; j < G; ++j) {
    const int tile = unit * G + j;
    tile_epilogue(summed + j * 3 * T2, tmp, T, tile / tiles_per_row, tile % tiles_per_row, S,
                  positions, normals, cam, material, scatter, radiance, radiance_unclamped);
  }
}

}  // namespace sss
