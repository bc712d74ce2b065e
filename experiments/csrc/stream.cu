// Frame layout v3 ("stream"): the transfer operator re-laid out so that each
// CTA streams one contiguous byte range with TMA bulk copies.
//
// A unit = unit_tiles tiles = R rows (one thread per row, rows in rowperm
// order). Its entries are stored item by item, item = (column band b, PCA
// term k), b-major; inside an item the rows' band segments follow rowperm
// order. Entry = {u32 column local to the band, f32 value} (8 B, the
// reference container's width). Items are padded to an even entry count so
// every item starts 16-byte aligned (cp.async.bulk granularity).
//
// k_transfer_stream: a double-buffered cp.async.bulk + mbarrier pipeline
// feeds CAP-entry chunks into shared memory while the threads accumulate
// sum_p val_p * x[c][col_p] for their row from shared memory (x band staged
// once per band, fp64) into registers for all K terms; the epilogue is the
// same recombine + inverse Haar + Fresnel shade as the other layouts.
#include "sss_common.cuh"

namespace sss {

constexpr int kStreamCap = 2048;  // entries per pipeline stage (16 KB)

// item sizes (padded to even): grid = nitems, block = R
__global__ void k_stream_sizes(const uint32_t* __restrict__ bandoff, const int* __restrict__ rowperm,
                               int K, int N, int NB, int R, uint32_t* __restrict__ item_len) {
  __shared__ unsigned red[32];
  const int it = blockIdx.x;
  const int k = it % K, b = (it / K) % NB, u = it / (K * NB);
  const int row = rowperm[u * R + threadIdx.x];
  const uint32_t* bo = bandoff + ((size_t)k * N + row) * (NB + 1) + b;
  unsigned c = bo[1] - bo[0];
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned s = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
    item_len[it] = (s + 1u) & ~1u;
  }
}

// row offsets inside each item + the entry copy: grid = nitems, block = R
__global__ void k_stream_fill(const uint64_t* __restrict__ rowptr, const uint32_t* __restrict__ cols,
                              const float* __restrict__ vals, const uint32_t* __restrict__ bandoff,
                              const int* __restrict__ rowperm, int K, int N, int NB, int R,
                              int band_width, const uint64_t* __restrict__ item_off,
                              uint32_t* __restrict__ rowoff, uint2* __restrict__ stream) {
  __shared__ unsigned wsum[32];
  const int it = blockIdx.x;
  const int k = it % K, b = (it / K) % NB, u = it / (K * NB);
  const int t = threadIdx.x;
  const int row = rowperm[u * R + t];
  const uint32_t* bo = bandoff + ((size_t)k * N + row) * (NB + 1) + b;
  const unsigned c = bo[1] - bo[0];
  // block exclusive scan (thread order = rowperm order)
  const int lane = t & 31, wid = t >> 5, nw = blockDim.x >> 5;
  unsigned incl = c;
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) wsum[wid] = incl;
  __syncthreads();
  if (t == 0) {
    unsigned a = 0;
    for (int w = 0; w < nw; ++w) { const unsigned x = wsum[w]; wsum[w] = a; a += x; }
  }
  __syncthreads();
  const unsigned pre = wsum[wid] + incl - c;
  rowoff[(size_t)it * (R + 1) + t] = pre;
  if (t == R - 1) rowoff[(size_t)it * (R + 1) + R] = pre + c;
  const uint64_t src = rowptr[(size_t)k * (N + 1) + row] + bo[0];
  uint2* dst = stream + item_off[it] + pre;
  const unsigned c0 = (unsigned)b * (unsigned)band_width;
  for (unsigned j = 0; j < c; ++j) {
    dst[j] = make_uint2(cols[src + j] - c0, __float_as_uint(vals[src + j]));
  }
  if (t == R - 1 && ((pre + c) & 1u)) dst[c] = make_uint2(0u, 0u);  // pad to even
}

// issue the next (item, chunk) of the unit into stage buffer `buf`
__device__ __forceinline__ void stream_issue(int buf, int& pq, int& pj, int NQ, size_t item0,
                                             const uint32_t* __restrict__ item_len,
                                             const uint64_t* __restrict__ item_off,
                                             const uint2* __restrict__ stream, uint2* stage,
                                             uint64_t* mbar) {
  while (pq < NQ && (unsigned)pj * kStreamCap >= item_len[item0 + pq]) { ++pq; pj = 0; }
  if (pq >= NQ) return;
  const unsigned len = item_len[item0 + pq];
  const unsigned n = min((unsigned)kStreamCap, len - (unsigned)pj * kStreamCap);
  const unsigned bytes = n * 8u;
  mbar_expect_tx(&mbar[buf], bytes);
  bulk_g2s(stage + buf * kStreamCap, stream + item_off[item0 + pq] + (size_t)pj * kStreamCap, bytes,
           &mbar[buf]);
  ++pj;
}

template <int KMAX>
__global__ void __launch_bounds__(256, 2) k_transfer_stream(
    int K, int S, int L, int G, int band_width, int NB, const uint64_t* __restrict__ item_off,
    const uint32_t* __restrict__ item_len, const uint32_t* __restrict__ rowoff,
    const uint2* __restrict__ stream, const int* __restrict__ rowperm,
    const double* __restrict__ x, const double* __restrict__ g,
    const float* __restrict__ positions, const float* __restrict__ normals,
    const double* __restrict__ cam, const double* __restrict__ material,
    double* __restrict__ vk, double* __restrict__ scatter, float* __restrict__ radiance,
    float* __restrict__ radiance_unclamped) {
  extern __shared__ __align__(16) unsigned char dsm_raw[];
  const int T = 1 << L, T2 = T * T, N = S * S;
  const int R = G * T2;
  uint2* stage = reinterpret_cast<uint2*>(dsm_raw);               // 2 * kStreamCap
  uint64_t* mbar = reinterpret_cast<uint64_t*>(stage + 2 * kStreamCap);  // 2
  double* xs = reinterpret_cast<double*>(mbar + 2);               // 3 * band_width
  double* summed = xs + 3 * band_width;                           // 3 * R
  double* tmp = summed + 3 * R;                                   // T2
  const int unit = blockIdx.x, t = threadIdx.x;
  const int NQ = NB * K;
  const size_t item0 = (size_t)unit * NQ;
  const int row = rowperm[unit * R + t];
  const int lr = row - unit * R;

  if (t == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();

  // producer cursor (thread 0 only): next (item, chunk) to issue
  int pq = 0, pj = 0;
  if (t == 0) {
    stream_issue(0, pq, pj, NQ, item0, item_len, item_off, stream, stage, mbar);
    stream_issue(1, pq, pj, NQ, item0, item_len, item_off, stream, stage, mbar);
  }

  double acc[KMAX][3];
#pragma unroll
  for (int k = 0; k < KMAX; ++k) acc[k][0] = acc[k][1] = acc[k][2] = 0.0;

  int band = -1;
  unsigned ci = 0;  // consumed chunk counter
  for (int q = 0; q < NQ; ++q) {
    const unsigned len = item_len[item0 + q];
    if (len == 0) continue;
    const int b = q / K, k = q % K;
    if (b != band) {
      __syncthreads();
      const int c0 = b * band_width, bw = min(band_width, N - c0);
      for (int j = t; j < bw; j += blockDim.x) {
        xs[j] = x[c0 + j];
        xs[band_width + j] = x[N + c0 + j];
        xs[2 * band_width + j] = x[2 * N + c0 + j];
      }
      band = b;
      __syncthreads();
    }
    const uint32_t* ro = rowoff + (item0 + q) * (size_t)(R + 1);
    const unsigned s0 = ro[t], s1 = ro[t + 1];
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    for (unsigned base = 0; base < len; base += kStreamCap, ++ci) {
      const int buf = ci & 1;
      mbar_wait(&mbar[buf], (ci >> 1) & 1u);
      const uint2* st = stage + buf * kStreamCap;
      const unsigned lo = max(s0, base), hi = min(s1, base + (unsigned)kStreamCap);
#pragma unroll 4
      for (unsigned p = lo; p < hi; ++p) {
        const uint2 e = st[p - base];
        const double v = (double)__uint_as_float(e.y);
        a0 = fma(v, xs[e.x], a0);
        a1 = fma(v, xs[band_width + e.x], a1);
        a2 = fma(v, xs[2 * band_width + e.x], a2);
      }
      __syncthreads();  // every thread is done with this buffer
      if (t == 0) {
        fence_proxy_async();
        stream_issue(buf, pq, pj, NQ, item0, item_len, item_off, stream, stage, mbar);
      }
    }
#pragma unroll
    for (int kk = 0; kk < KMAX; ++kk)
      if (kk == k) { acc[kk][0] += a0; acc[kk][1] += a1; acc[kk][2] += a2; }
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
