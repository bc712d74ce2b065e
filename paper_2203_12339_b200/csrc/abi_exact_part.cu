// The C5 exact pair pass instantiations, one third per compilation
// (build.py compiles this file with -DSSS_EXACT_PART=0, 1, 2; dispatcher in
// abi_exact.cu). K <= 8 terms (BASELINE C5: K = 8; K = 12 / 16 at 64
// materials took ~3 min of ptxas each). Only the packed FP32x2 form is built (the scalar form
// measured 0.365 s vs 0.325 s at 256^2, profiles/r02_c5_kfused_ncu.json).
#include "abi_util.cuh"
#include "exact.cuh"

#ifndef SSS_EXACT_PART
#error "compile with -DSSS_EXACT_PART=0|1|2"
#endif

#define SSS_CAT2(a, b) a##b
#define SSS_CAT(a, b) SSS_CAT2(a, b)

int SSS_CAT(sss_exact_part, SSS_EXACT_PART)(int levels, int KT, int MM, const sss::ExactTables& tb,
                                              const float* pos, const float* area, int side,
                                              float r_max, int rt0, int nrt, double* D, dim3 grid,
                                              size_t smem, cudaStream_t st) {
#define SSS_PR(LV, KK, M_)                                                                   \
  if (levels == LV && KT == KK && MM == M_) {                                                \
    if (int r = set_smem((const void*)sss::k_pair_rows_exact<LV, KK, M_, true>, smem)) return r; \
    sss::k_pair_rows_exact<LV, KK, M_, true><<<grid, 256, smem, st>>>(tb, pos, area, side, r_max, \
                                                                      rt0, nrt, D);          \
    return check_launch("k_pair_rows_exact");                                                \
  }
#if SSS_EXACT_PART == 0
  SSS_PR(3, 8, 64) SSS_PR(3, 4, 16)
#elif SSS_EXACT_PART == 1
  SSS_PR(3, 8, 32) SSS_PR(3, 4, 64) SSS_PR(2, 8, 32)
#else
  SSS_PR(2, 8, 64) SSS_PR(2, 4, 16)
#endif
#undef SSS_PR
  return -1000;
}
