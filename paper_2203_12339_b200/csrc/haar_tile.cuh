// Tile-local sequential Haar shared by the pair passes (precompute.cu,
// exact.cuh).
#pragma once
#include "sss_common.cuh"

namespace sss {

// sequential full-pyramid Haar of a T x T tile held at base[(a*T+b)*stride]
// (one thread), reference order: per level rows then columns
template <int T>
__device__ __forceinline__ void seq_haar_fwd(double* base, int stride) {
  double tmp[T];
#pragma unroll
  for (int s = T; s >= 2; s >>= 1) {
    const int h = s >> 1;
    for (int i = 0; i < s; ++i) {
#pragma unroll
      for (int j = 0; j < h; ++j) {
        const double e = base[(i * T + 2 * j) * stride], o = base[(i * T + 2 * j + 1) * stride];
        tmp[j] = dmul(dadd(e, o), SSS_ISQRT2);
        tmp[h + j] = dmul(dsub(e, o), SSS_ISQRT2);
      }
      for (int j = 0; j < s; ++j) base[(i * T + j) * stride] = tmp[j];
    }
    for (int j = 0; j < s; ++j) {
#pragma unroll
      for (int i = 0; i < h; ++i) {
        const double e = base[((2 * i) * T + j) * stride], o = base[((2 * i + 1) * T + j) * stride];
        tmp[i] = dmul(dadd(e, o), SSS_ISQRT2);
        tmp[h + i] = dmul(dsub(e, o), SSS_ISQRT2);
      }
      for (int i = 0; i < s; ++i) base[(i * T + j) * stride] = tmp[i];
    }
  }
}

}  // namespace sss
