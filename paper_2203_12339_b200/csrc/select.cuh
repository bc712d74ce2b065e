// Exact block-wide radix selection (shared by the per-frame irradiance
// selection and the precompute's step-1 / step-2 cuts).
//
// Keys are the 63-bit magnitudes of doubles (sign cleared): unsigned order ==
// |x| order, so a most-significant-digit radix descent finds the exact
// threshold. compress_top_n (wavelets.py:128-136) keeps the n largest |x|
// with ties to the lower flat index; compress_energy (wavelets.py:139-153)
// keeps the shortest |x|-ordered prefix whose cumulative energy reaches
// fraction * total — done here in 2^62 fixed point so bucket sums are exact
// integers, independent of summation order.
#pragma once
#include "sss_common.cuh"

namespace sss {

constexpr int kCandCap = 4096;

__device__ __forceinline__ uint64_t mkey(double v) {
  return (uint64_t)__double_as_longlong(v) & 0x7fffffffffffffffULL;
}

struct SelShared {
  unsigned hist[2048];
  unsigned elo[2048];
  unsigned ehi[2048];
  uint64_t cand_key[kCandCap];
  uint32_t cand_pos[kCandCap];
  uint64_t wsum64[32];
  int ncand_store;
  int scal_b;
  long long scal_need;
  long long scal_cnt;
  double red[32];
  long long redi[32];
  unsigned wsum[32];
  int result;
};

__device__ __forceinline__ double block_sum_d(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    double s = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) red[0] = s;
  }
  __syncthreads();
  const double s = red[0];
  __syncthreads();
  return s;
}

__device__ __forceinline__ long long block_sum_i(long long v, long long* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    long long s = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0;
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) red[0] = s;
  }
  __syncthreads();
  const long long s = red[0];
  __syncthreads();
  return s;
}

// exclusive block scan of a per-thread u64 (thread order)
__device__ __forceinline__ uint64_t block_excl_scan_u64(uint64_t v, uint64_t* wsum) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  uint64_t incl = v;
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  __syncthreads();
  if (lane == 31) wsum[wid] = incl;
  __syncthreads();
  if (threadIdx.x < 32) {
    const uint64_t s = threadIdx.x < nw ? wsum[threadIdx.x] : 0;
    uint64_t inc = s;
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(0xffffffffu, inc, o);
      if ((int)threadIdx.x >= o) inc += y;
    }
    if (threadIdx.x < nw) wsum[threadIdx.x] = inc - s;
  }
  __syncthreads();
  const uint64_t r = wsum[wid] + incl - v;
  __syncthreads();
  return r;
}

__device__ __forceinline__ uint64_t fixq(double v, double scale) {
  return (uint64_t)(v * v * scale);
}

// Parallel "from the top" bucket search: the largest bucket b with
// S(>b) < need <= S(>=b); writes sh.scal_b / scal_need (need - S(>b)) /
// scal_cnt (count in b). Unreachable need -> b = 0.
template <bool ENERGY>
__device__ void find_bucket(SelShared& sh, int nb, long long need) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int per = (nb + nt - 1) / nt;
  const int hi = nb - 1 - tid * per;  // this thread's top bin
  uint64_t s = 0;
  for (int q = 0; q < per; ++q) {
    const int b = hi - q;
    if (b < 0) break;
    s += ENERGY ? (((uint64_t)sh.ehi[b] << 32) | sh.elo[b]) : (uint64_t)sh.hist[b];
  }
  const uint64_t before = block_excl_scan_u64(s, sh.wsum64);
  if (tid == 0) sh.scal_b = -1;
  __syncthreads();
  if ((long long)before < need && need <= (long long)(before + s)) {
    uint64_t acc = before;
    for (int q = 0; q < per; ++q) {
      const int b = hi - q;
      const uint64_t w = ENERGY ? (((uint64_t)sh.ehi[b] << 32) | sh.elo[b]) : (uint64_t)sh.hist[b];
      if ((long long)(acc + w) >= need) {
        sh.scal_b = b;
        sh.scal_need = need - (long long)acc;
        sh.scal_cnt = sh.hist[b];
        break;
      }
      acc += w;
    }
  }
  __syncthreads();
  if (sh.scal_b < 0) {  // unreachable (rounding): take everything down to bucket 0
    __syncthreads();
    if (tid == 0) {
      uint64_t above = 0;
      for (int b = nb - 1; b > 0; --b)
        above += ENERGY ? (((uint64_t)sh.ehi[b] << 32) | sh.elo[b]) : (uint64_t)sh.hist[b];
      sh.scal_b = 0;
      sh.scal_need = need - (long long)above;
      sh.scal_cnt = sh.hist[0];
    }
  }
  __syncthreads();
}

// Returns threshold key t, `take` (# elements with key == t to keep, lowest
// flat index first) and the tie count. For ENERGY, need_init is the 2^62
// fixed-point target and scale = 2^62 / total.
template <bool ENERGY>
__device__ void radix_cut(const double* __restrict__ v, int N, long long need_init, double scale,
                          SelShared& sh, uint64_t* t_out, long long* take_out, long long* tiecnt) {
  const int tid = threadIdx.x, nt = blockDim.x;
  // energy cuts keep 11-bit digits (their fixed-point bucket sums are part of
  // the bitwise contract); plain top-n uses 8-bit digits and finishes exactly
  // from the gathered keys once the threshold bucket holds <= 64 of them
  constexpr int kPasses = ENERGY ? 6 : 8;
  const int digits_e[6] = {53, 42, 31, 20, 9, 0};
  const int widths_e[6] = {11, 11, 11, 11, 11, 9};
  const int digits_p[8] = {56, 48, 40, 32, 24, 16, 8, 0};
  uint64_t prefix = 0, pmask = 0;
  long long need = need_init;
  long long ncand = N;
  bool in_smem = false;
  for (int p = 0; p < kPasses; ++p) {
    const int shf = ENERGY ? digits_e[p] : digits_p[p];
    const int nb = 1 << (ENERGY ? widths_e[p] : 8);
    for (int b = tid; b < nb; b += nt) {
      sh.hist[b] = 0;
      if (ENERGY) { sh.elo[b] = 0; sh.ehi[b] = 0; }
    }
    const bool gather = !in_smem && ncand <= kCandCap;
    if (tid == 0 && gather) sh.ncand_store = 0;
    __syncthreads();
    if (!in_smem) {
      for (int i = tid; i < N; i += nt) {
        const double x = v[i];
        const uint64_t k = mkey(x);
        if ((k & pmask) != prefix) continue;
        const int b = (int)((k >> shf) & (nb - 1));
        atomicAdd(&sh.hist[b], 1u);
        if (ENERGY) {
          const uint64_t q = fixq(x, scale);
          const unsigned lo = (unsigned)q;
          const unsigned old = atomicAdd(&sh.elo[b], lo);
          atomicAdd(&sh.ehi[b], (unsigned)(q >> 32) + ((unsigned)(old + lo) < old ? 1u : 0u));
        }
        if (gather) {
          const int s = atomicAdd(&sh.ncand_store, 1);
          sh.cand_key[s] = k;
          sh.cand_pos[s] = (uint32_t)i;
        }
      }
    } else {
      const int nc = sh.ncand_store;
      for (int s = tid; s < nc; s += nt) {
        const uint64_t k = sh.cand_key[s];
        if ((k & pmask) != prefix) continue;
        const int b = (int)((k >> shf) & (nb - 1));
        atomicAdd(&sh.hist[b], 1u);
        if (ENERGY) {
          const uint64_t q = fixq(__longlong_as_double((long long)k), scale);
          const unsigned lo = (unsigned)q;
          const unsigned old = atomicAdd(&sh.elo[b], lo);
          atomicAdd(&sh.ehi[b], (unsigned)(q >> 32) + ((unsigned)(old + lo) < old ? 1u : 0u));
        }
      }
    }
    __syncthreads();
    find_bucket<ENERGY>(sh, nb, need);
    const int b = sh.scal_b;
    need = sh.scal_need;
    ncand = sh.scal_cnt;
    prefix |= (uint64_t)b << shf;
    pmask |= (uint64_t)(nb - 1) << shf;
    if (gather) in_smem = true;
    __syncthreads();
    if (!ENERGY && p + 1 < kPasses && ncand <= 64) {
      uint64_t* ek = reinterpret_cast<uint64_t*>(sh.elo);  // 64 keys (unused without ENERGY)
      if (tid == 0) sh.result = 0;
      __syncthreads();
      if (in_smem) {
        const int nc = sh.ncand_store;
        for (int q = tid; q < nc; q += nt) {
          const uint64_t k = sh.cand_key[q];
          if ((k & pmask) == prefix) ek[atomicAdd(&sh.result, 1)] = k;
        }
      } else {
        for (int i = tid; i < N; i += nt) {
          const uint64_t k = mkey(v[i]);
          if ((k & pmask) == prefix) ek[atomicAdd(&sh.result, 1)] = k;
        }
      }
      __syncthreads();
      const int total = sh.result;
      if (tid < total) {
        const uint64_t kj = ek[tid];
        long long g = 0, e = 0;
        for (int q = 0; q < total; ++q) {
          g += ek[q] > kj;
          e += ek[q] == kj;
        }
        if (g < need && need <= g + e) {  // equal keys write equal values
          sh.scal_cnt = e;
          sh.scal_need = need - g;
          reinterpret_cast<uint64_t*>(sh.ehi)[0] = kj;
        }
      }
      __syncthreads();
      prefix = reinterpret_cast<uint64_t*>(sh.ehi)[0];
      need = sh.scal_need;
      ncand = sh.scal_cnt;
      __syncthreads();
      break;
    }
  }
  *t_out = prefix;
  *tiecnt = ncand;
  if (ENERGY) {
    const uint64_t qt = fixq(__longlong_as_double((long long)prefix), scale);
    long long take = qt == 0 ? ncand : (long long)((need + (long long)qt - 1) / (long long)qt);
    if (need <= 0) take = 0;
    *take_out = take < ncand ? take : ncand;
  } else {
    *take_out = need;
  }
}

// flat index of the `take`-th (1-based) set bit of a block-shared bitmap
__device__ int kth_set_bit(const uint32_t* bits, int nwords, long long take, SelShared& sh) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int per = (nwords + nt - 1) / nt;
  const int w0 = min(tid * per, nwords), w1 = min(w0 + per, nwords);
  unsigned cnt = 0;
  for (int w = w0; w < w1; ++w) cnt += __popc(bits[w]);
  const uint64_t before = block_excl_scan_u64(cnt, sh.wsum64);
  if (tid == 0) sh.result = -1;
  __syncthreads();
  if (take > (long long)before && take <= (long long)(before + cnt)) {
    long long r = take - (long long)before;
    for (int w = w0; w < w1; ++w) {
      const uint32_t x = bits[w];
      const int pc = __popc(x);
      if (r > pc) { r -= pc; continue; }
      for (int b = 0; b < 32; ++b)
        if ((x >> b) & 1u) { if (--r == 0) { sh.result = w * 32 + b; break; } }
      break;
    }
  }
  __syncthreads();
  const int res = sh.result;
  __syncthreads();
  return res;
}

}  // namespace sss
