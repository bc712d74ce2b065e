// extern "C" sss_pair_rows_exact (include/sss_b200.h): the C5 exact pair
// pass in its own translation unit so its 64-material unrolled instantiations
// compile in parallel with the rest of the library (build.py).
#include <cstdlib>
#include <cstring>

#include "abi_util.cuh"
#include "exact.cuh"

namespace {
constexpr int kNotMine = -1000;
}
// the instantiations live in three translation units (csrc/abi_exact_part.cu
// compiled with SSS_EXACT_PART = 0, 1, 2) so they compile in parallel
#define SSS_EXACT_PART_DECL(P)                                                                   \
  int sss_exact_part##P(int levels, int KT, int MM, const sss::ExactTables& tb, const float* pos, \
                        const float* area, int side, float r_max, int rt0, int nrt, double* D,   \
                        dim3 grid, size_t smem, cudaStream_t st);
SSS_EXACT_PART_DECL(0)
SSS_EXACT_PART_DECL(1)
SSS_EXACT_PART_DECL(2)

extern "C" {

int sss_pair_rows_exact(int levels, int side, const float* pos, const float* area, int K,
                        const float* Pkm, const float* mat, int n_mat, float r_max, int rt0,
                        int nrt, double* D, void* stream) {
  if (int r = check_geom(side, levels)) return r;
  if (levels > 3) return fail(SSS_EINVAL, "pair pass supports levels <= 3");
  if (!pos || !area || !Pkm || !mat || !D) return fail(SSS_EINVAL, "bad pair_rows pointers");
  if (K < 1 || K > 8) return fail(SSS_EINVAL, "K must lie in [1, 8]");
  if (n_mat < 1 || n_mat > sss::kExactMaxM) return fail(SSS_EINVAL, "n_mat must lie in [1, 64]");
  const int MM = n_mat <= 16 ? 16 : (n_mat <= 32 ? 32 : 64);
  const int T = 1 << levels, T2 = T * T, tiles = (side / T) * (side / T);
  if (rt0 < 0 || nrt <= 0 || rt0 + nrt > tiles) return fail(SSS_EINVAL, "receiver tile block out of range");
  const int KT = K <= 4 ? 4 : 8;
  // host tables -> the kernel's parameter bank (Pkm / mat are host arrays:
  // Pkm (K, n_mat) row-major, mat (n_mat, 4) {sigma_tr, z_r, z_v, c}); the
  // padded materials and terms have zero weight
  sss::ExactTables tb;
  std::memset(&tb, 0, sizeof(tb));
  for (int k = 0; k < K; ++k)
    for (int m = 0; m < n_mat; ++m) tb.P[k * MM + m] = Pkm[k * n_mat + m];
  for (int m = 0; m < MM; ++m) {
    const bool real = m < n_mat;
    const float s = real ? mat[m * 4] : 1.0f, zr = real ? mat[m * 4 + 1] : 1.0f,
                zv = real ? mat[m * 4 + 2] : 1.0f, c = real ? mat[m * 4 + 3] : 0.0f;
    tb.m0[m] = make_float4(zr * zr, zv * zv, -s * 1.4426950408889634f, s);
    tb.m1[m] = make_float4(c * zr, c * zv, 0.0f, 0.0f);
  }
  for (int j = 0; j < MM / 2; ++j) {  // the packed material pairs
    const float4 a = tb.m0[2 * j], b = tb.m0[2 * j + 1], c = tb.m1[2 * j], d = tb.m1[2 * j + 1];
    tb.pA[j] = make_float2(a.x, b.x);
    tb.pB[j] = make_float2(a.y, b.y);
    tb.pS[j] = make_float2(a.z, b.z);
    tb.ps[j] = make_float2(a.w, b.w);
    tb.pCr[j] = make_float2(c.x, d.x);
    tb.pCv[j] = make_float2(c.y, d.y);
    for (int k = 0; k < sss::kExactMaxK; ++k)
      tb.pP[k * (MM / 2) + j] = make_float2(tb.P[k * MM + 2 * j], tb.P[k * MM + 2 * j + 1]);
  }
  dim3 grid(tiles, nrt);
  const int rpp = 1024 / T2 > 0 ? (1024 / T2 < 16 ? 1024 / T2 : 16) : 1;
  const size_t smem = (size_t)KT * rpp * (T2 + 1) * sizeof(double);
  for (auto part : {sss_exact_part0, sss_exact_part1, sss_exact_part2}) {
    const int r = part(levels, KT, MM, tb, pos, area, side, r_max, rt0, nrt, D, grid, smem, S_(stream));
    if (r != kNotMine) return r;
  }
  return fail(SSS_EINVAL, "pair_rows: unsupported (levels, K, n_mat)");
}

}  // extern "C"
