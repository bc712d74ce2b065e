// extern "C" entry points declared in include/sss_b200.h. One translation unit
// so every kernel is visible to its launcher; built into
// paper_2203_12339_b200/_sss_b200.so for sm_100a (see build.py).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "../../include/sss_b200.h"
#include "frame.cu"
#include "precompute.cu"
#include "stream.cu"
#include "select_cluster.cu"
#include "stream4.cu"
#include "stream6.cu"
#include "csr7.cu"
#include "csr8.cu"
#include "csr9.cu"
#include "kpack10.cu"
#include "kstep12.cu"
#include "kstream13.cu"
#include "kgroup14.cu"
#include "flat15.cu"
#include "kflat18.cu"
#include "sweep.cu"
#include "regional19.cu"
#include "k8_20.cu"
#include "direct.cu"
#include "fold.cu"
#include "raster.cu"
#include "kpairs21.cu"
#include "flat8c22.cu"
#include "kgroup23.cu"
#include "rbcsc24.cu"
#include "flat16_25.cu"
#include "align26.cu"

namespace {
thread_local std::string g_err;

int fail(int code, const char* msg) {
  g_err = msg;
  return code;
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    g_err = std::string(what) + ": " + cudaGetErrorString(e);
    return SSS_ECUDA;
  }
  return SSS_OK;
}

bool pow2(int v) { return v > 0 && (v & (v - 1)) == 0; }

int set_smem(const void* fn, size_t bytes) {
  if (bytes > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess) {
      g_err = std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e);
      return SSS_ECUDA;
    }
  }
  return SSS_OK;
}

int check_geom(int side, int levels) {
  if (!pow2(side) || side < 2) return fail(SSS_EINVAL, "side must be a power of two >= 2");
  if (levels < 1 || (1 << levels) > side || levels > 6)
    return fail(SSS_EINVAL, "levels must lie in [1, min(6, log2 side)]");
  return SSS_OK;
}

inline cudaStream_t S_(void* s) { return reinterpret_cast<cudaStream_t>(s); }
}  // namespace

extern "C" {

const char* sss_last_error(void) { return g_err.c_str(); }
int sss_version(void) { return 1; }

int sss_haar2d(const double* in, double* out, int batch, int side, int levels, int inverse,
               void* stream) {
  if (int r = check_geom(side, levels)) return r;
  if (batch < 0 || !in || !out) return fail(SSS_EINVAL, "bad batch or pointer");
  if (batch == 0) return SSS_OK;
  const int T = 1 << levels;
  const long long grid = (long long)batch * (side / T) * (side / T);
  if (grid > 2147483647LL) return fail(SSS_EINVAL, "grid too large");
  const size_t smem = 2 * (size_t)T * T * sizeof(double);
  if (int r = set_smem((const void*)sss::k_haar2d_batch, smem)) return r;
  sss::k_haar2d_batch<<<(unsigned)grid, 256, smem, S_(stream)>>>(in, out, side, levels, inverse);
  return check_launch("k_haar2d_batch");
}

int sss_select_topn(const double* v, int nvec, int n_dom, int n_keep, const uint32_t* f2t,
                    double* x_out, uint32_t* mask, double* energy, void* stream) {
  if (nvec < 0 || nvec > 65535 || n_dom <= 0 || n_keep < 0 || !v || !x_out)
    return fail(SSS_EINVAL, "bad select arguments");
  if (nvec == 0) return SSS_OK;
  if (mask) {
    cudaError_t e = cudaMemsetAsync(mask, 0, (size_t)nvec * ((n_dom + 31) / 32) * 4, S_(stream));
    if (e != cudaSuccess) return fail(SSS_ECUDA, cudaGetErrorString(e));
  }
  const int chunk = (((n_dom + sss::kSelCluster - 1) / sss::kSelCluster) + 31) / 32 * 32;
  if (chunk <= 16384 && n_dom >= 32 * sss::kSelCluster) {
    // one 8-CTA cluster per vector, slices resident in shared memory
    const size_t smem = ((sizeof(sss::ClusterSelShared) + 15) & ~size_t(15)) + chunk * sizeof(double);
    if (int r = set_smem((const void*)sss::k_select_cluster, smem)) return r;
    if (sss::kSelCluster > 8)
      cudaFuncSetAttribute((const void*)sss::k_select_cluster,
                           cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    sss::k_select_cluster<<<nvec * sss::kSelCluster, 1024, smem, S_(stream)>>>(
        v, n_dom, n_keep, chunk, f2t, x_out, mask, energy);
    return check_launch("k_select_cluster");
  }
  const size_t smem = sizeof(sss::SelShared);
  if (int r = set_smem((const void*)sss::k_select_topn, smem)) return r;
  sss::k_select_topn<<<nvec, 1024, smem, S_(stream)>>>(v, n_dom, n_keep, f2t, x_out, mask, energy);
  return check_launch("k_select_topn");
}

int sss_sh_irradiance(const float* T_l, const double* Lsh, int nl, int side, int levels,
                      double* E_out, double* ehat, void* stream) {
  if (int r = check_geom(side, levels)) return r;
  if (nl <= 0 || !T_l || !Lsh || !ehat) return fail(SSS_EINVAL, "bad SH arguments");
  const int T = 1 << levels, T2 = T * T, tiles = (side / T) * (side / T);
  int tpb = 256 / T2 < 1 ? 1 : 256 / T2;
  while (tpb > 1 && tiles % tpb) tpb >>= 1;
  const size_t smem = 6 * (size_t)tpb * T2 * sizeof(double);
  if (int r = set_smem((const void*)sss::k_sh_irradiance_multi, smem)) return r;
  sss::k_sh_irradiance_multi<<<tiles / tpb, tpb * T2 < 32 ? 32 : tpb * T2, smem, S_(stream)>>>(
      T_l, Lsh, nl, side, levels, tpb, E_out, ehat);
  return check_launch("k_sh_irradiance_multi");
}

int sss_env_project(const double* faces, int env_side, int n_keep, uint32_t* idx, double* val,
                    uint32_t* union_idx, double* union_lc, int* n_union, void* stream) {
  if (!pow2(env_side) || env_side > 32 || n_keep <= 0 || !faces || !idx || !val)
    return fail(SSS_EINVAL, "bad env_project arguments (env_side must be a power of two <= 32)");
  const int s2 = env_side * env_side;
  const size_t smem = (size_t)12 * s2 * sizeof(double) + sizeof(sss::SelShared);
  if (int r = set_smem((const void*)sss::k_env_project, smem)) return r;
  sss::k_env_project<<<3, 1024, smem, S_(stream)>>>(faces, env_side, n_keep, idx, val, nullptr);
  if (int r = check_launch("k_env_project")) return r;
  if (union_idx && union_lc && n_union) {
    sss::k_env_union<<<1, 1024, 0, S_(stream)>>>(idx, val, n_keep, 6 * s2, union_idx, union_lc,
                                                n_union);
    return check_launch("k_env_union");
  }
  return SSS_OK;
}

int sss_env_irradiance(const float* W2, int D, const uint32_t* union_idx, const double* union_lc,
                       const int* n_union, int n_keep, int side, int levels, double* E_out,
                       double* ehat, void* stream) {
  if (int r = check_geom(side, levels)) return r;
  if (!W2 || !union_idx || !union_lc || !n_union || !ehat || n_keep <= 0)
    return fail(SSS_EINVAL, "bad env_irradiance arguments");
  const int T = 1 << levels, T2 = T * T, tiles = (side / T) * (side / T);
  // one point per thread with a sequential (bitwise-pinned) sum: balance the
  // grid across the SMs with small CTAs (>= 64 threads)
  // TPB horizontally adjacent tiles per CTA (a warp then reads whole 128-B
  // lines of W^{w2}); SSS_ENV_TPB overrides for experiments
  const char* tpb_env = getenv("SSS_ENV_TPB");
  int tpb = tpb_env ? atoi(tpb_env) : (T * 4 <= side ? 4 : 1);
  if (tpb < 1 || (side / T) % tpb) tpb = 1;
  const size_t smem = 6 * (size_t)tpb * T2 * sizeof(double) + 12 * (size_t)n_keep * sizeof(double) +
                      3 * (size_t)n_keep * sizeof(int);
  if (int r = set_smem((const void*)sss::k_env_irradiance_multi, smem)) return r;
  (void)D;
  sss::k_env_irradiance_multi<<<tiles / tpb, tpb * T2 < 32 ? 32 : tpb * T2, smem, S_(stream)>>>(
      W2, union_idx, union_lc, n_union, n_keep, side, levels, tpb, E_out, ehat);
  return check_launch("k_env_irradiance_multi");
}

int sss_env_irradiance_sel(const float* W2, int D, const uint32_t* sel_idx, const double* sel_val,
                           int n_keep, int side, int levels, double* E_out, double* ehat,
                           void* stream) {
  if (int r = check_geom(side, levels)) return r;
  if (!W2 || !sel_idx || !sel_val || !ehat || n_keep <= 0 || D <= 0 || D > 6 * 32 * 32)
    return fail(SSS_EINVAL, "bad env_irradiance_sel arguments");
  const int T = 1 << levels, T2 = T * T;
  const char* tpb_env = getenv("SSS_ENV_TPB");
  int tpb = tpb_env ? atoi(tpb_env) : (T * 4 <= side ? 4 : 1);
  if (tpb < 1 || (side / T) % tpb) tpb = 1;
  const int tiles = (side / T) * (side / T);
  const size_t nw = (size_t)(D + 31) / 32;
  const size_t smem = 6 * (size_t)tpb * T2 * sizeof(double) + 12 * (size_t)n_keep * sizeof(double) +
                      3 * (size_t)n_keep * sizeof(int) + 2 * nw * sizeof(uint32_t);
  if (int r = set_smem((const void*)sss::k_env_irradiance_multi, smem)) return r;
  sss::k_env_irradiance_multi<<<tiles / tpb, tpb * T2 < 32 ? 32 : tpb * T2, smem, S_(stream)>>>(
      W2, nullptr, nullptr, nullptr, n_keep, side, levels, tpb, E_out, ehat, sel_idx, sel_val, D);
  return check_launch("k_env_irradiance_multi");
}

int sss_env_transfer(const float* normals, int n_points, const double* dirs, const double* dom,
                     int env_side, float* W2, void* stream) {
  if (!pow2(env_side) || env_side > 64 || n_points <= 0 || !normals || !dirs || !dom || !W2)
    return fail(SSS_EINVAL, "bad env_transfer arguments");
  const int s2 = env_side * env_side;
  const size_t smem = (size_t)(sss::kEnvP + 1) * s2 * sizeof(double);
  if (int r = set_smem((const void*)sss::k_env_transfer, smem)) return r;
  dim3 grid((n_points + sss::kEnvP - 1) / sss::kEnvP, 6);
  sss::k_env_transfer<<<grid, 256, smem, S_(stream)>>>(normals, n_points, dirs, dom, env_side, W2);
  return check_launch("k_env_transfer");
}

int sss_material_weights(const double* bw, const double* r_nodes, int K, int nr,
                         const double* material, double* g, void* stream) {
  if (K <= 0 || nr < 2 || !bw || !r_nodes || !material || !g)
    return fail(SSS_EINVAL, "bad material_weights arguments");
  sss::k_material_weights<<<3, 512, nr * sizeof(double), S_(stream)>>>(bw, r_nodes, K, nr,
                                                                       material, g);
  return check_launch("k_material_weights");
}

int sss_transfer_relight(int K, int side, int levels, int unit_tiles, const uint64_t* rowptr,
                         const uint32_t* bandoff, int band_width, int n_bands, const int* rowperm,
                         const uint32_t* cols, const float* vals, const double* x, const double* g,
                         const float* positions, const float* normals, const double* cam,
                         const double* material, double* vk, double* scatter, float* radiance,
                         float* radiance_unclamped, void* stream) {
  if (int r = check_geom(side, levels)) return r;
  if (K <= 0 || K > 16 || !rowptr || !bandoff || !rowperm || !x || !g || !positions || !normals ||
      !cam || !material || !vk || !radiance || !radiance_unclamped)
    return fail(SSS_EINVAL, "bad transfer_relight arguments");
  const int T = 1 << levels, T2 = T * T;
  const int tiles = (side / T) * (side / T);
  if (unit_tiles <= 0 || tiles % unit_tiles || unit_tiles * T2 > 256 || (unit_tiles * T2) % 32)
    return fail(SSS_EINVAL, "unit_tiles * 4^levels must be a multiple of 32 and <= 256");
  if (band_width <= 0 || n_bands != (side * side + band_width - 1) / band_width)
    return fail(SSS_EINVAL, "band_width / n_bands mismatch");
  const int R = unit_tiles * T2;
  const size_t smem = (3 * (size_t)band_width + 3 * (size_t)R + T2) * sizeof(double);
  const unsigned grid = tiles / unit_tiles;
#define SSS_TB(KM)                                                                              \
  {                                                                                             \
    if (int r = set_smem((const void*)sss::k_transfer_banded<KM>, smem)) return r;              \
    sss::k_transfer_banded<KM><<<grid, R, smem, S_(stream)>>>(                                  \
        K, side, levels, unit_tiles, rowptr, bandoff, band_width, n_bands, rowperm, cols, vals, \
        x, g, positions, normals, cam, material, vk, scatter, radiance, radiance_unclamped);    \
  }
  if (K <= 4) SSS_TB(4)
  else if (K <= 8) SSS_TB(8)
  else if (K <= 12) SSS_TB(12)
  else SSS_TB(16)
#undef SSS_TB
  return check_launch("k_transfer_banded");
}

int sss_stream_build(int pass, const uint64_t* rowptr, const uint32_t* cols, const float* vals,
                     const uint32_t* bandoff, const int* rowperm, int K, int n_rows, int n_bands,
                     int unit_rows, int band_width, uint32_t* item_len, uint64_t* item_off,
                     uint64_t* block_sums, uint64_t* total, uint32_t* rowoff, void* entries,
                     void* stream) {
  if (!bandoff || !rowperm || !item_len || !item_off || K <= 0 || n_rows <= 0 || n_bands <= 0 ||
      unit_rows <= 0 || unit_rows > 1024 || unit_rows % 32 || n_rows % unit_rows)
    return fail(SSS_EINVAL, "bad stream_build arguments");
  const long long nitems = (long long)(n_rows / unit_rows) * n_bands * K;
  if (nitems > 2147483647LL) return fail(SSS_EINVAL, "too many items");
  if (pass == 0) {
    if (!block_sums || !total) return fail(SSS_EINVAL, "stream_build pass 0 needs scan scratch");
    sss::k_stream_sizes<<<(unsigned)nitems, unit_rows, 0, S_(stream)>>>(bandoff, rowperm, K, n_rows,
                                                                        n_bands, unit_rows, item_len);
    if (int r = check_launch("k_stream_sizes")) return r;
    return sss_scan_u32(item_len, item_off, (size_t)nitems, block_sums, total, stream);
  }
  if (!rowptr || !cols || !vals || !rowoff || !entries) return fail(SSS_EINVAL, "stream_build fill");
  sss::k_stream_fill<<<(unsigned)nitems, unit_rows, 0, S_(stream)>>>(
      rowptr, cols, vals, bandoff, rowperm, K, n_rows, n_bands, unit_rows, band_width, item_off,
      rowoff, reinterpret_cast<uint2*>(entries));
  return check_launch("k_stream_fill");
}

int sss_transfer_stream(int K, int side, int levels, int unit_tiles, int band_width, int n_bands,
                        const uint64_t* item_off, const uint32_t* item_len, const uint32_t* rowoff,
                        const void* entries, const int* rowperm, const double* x, const double* g,
                        const float* positions, const float* normals, const double* cam,
                        const double* material, double* vk, double* scatter, float* radiance,
                        float* radiance_unclamped, void* stream) {
  if (int r = check_geom(side, levels)) return r;
  if (K <= 0 || K > 16 || !item_off || !item_len || !rowoff || !entries || !rowperm || !x || !g ||
      !positions || !normals || !cam || !material || !vk || !radiance || !radiance_unclamped)
    return fail(SSS_EINVAL, "bad transfer_stream arguments");
  if (reinterpret_cast<uintptr_t>(entries) % 16) return fail(SSS_EINVAL, "entries not 16B aligned");
  const int T = 1 << levels, T2 = T * T;
  const int tiles = (side / T) * (side / T);
  if (unit_tiles <= 0 || tiles % unit_tiles || unit_tiles * T2 > 256 || (unit_tiles * T2) % 32)
    return fail(SSS_EINVAL, "unit_tiles * 4^levels must be a multiple of 32 and <= 256");
  const int R = unit_tiles * T2;
  const size_t smem = 2 * sss::kStreamCap * sizeof(uint2) + 2 * sizeof(uint64_t) +
                      (3 * (size_t)band_width + 3 * (size_t)R + T2) * sizeof(double);
  const unsigned grid = tiles / unit_tiles;
#define SSS_TS(KM)                                                                                \
  {                                                                                               \
    if (int r = set_smem((const void*)sss::k_transfer_stream<KM>, smem)) return r;                \
    sss::k_transfer_stream<KM><<<grid, R, smem, S_(stream)>>>(                                    \
        K, side, levels, unit_tiles, band_width, n_bands, item_off, item_len, rowoff,             \
        reinterpret_cast<const uint2*>(entries), rowperm, x, g, positions, normals, cam, material, \
        vk, scatter, radiance, radiance_unclamped);                                               \
  }
  if (K <= 4) SSS_TS(4)
  else if (K <= 8) SSS_TS(8)
  else if (K <= 12) SSS_TS(12)
  else SSS_TS(16)
#undef SSS_TS
  return check_launch("k_transfer_stream");
}

int sss_transfer_v4(int K, int side, int levels, int band_width, int slot_bytes, int units,
                    int max_unit_items,
                    const int* unit_tile0, const int* unit_ntiles, const int* unit_item0,
                    const int* unit_nitems, const void* items, const void* stream_bytes,
                    const void* vrow_first, const double* x, const double* g,
                    const float* positions, const float* normals, const double* cam,
                    const double* material, double* vk, double* scatter, float* radiance,
                    float* radiance_unclamped, void* stream) {
  if (int r = check_geom(side, levels)) return r;
  if (K <= 0 || K > 16 || units <= 0 || !unit_tile0 || !unit_ntiles || !unit_item0 ||
      !unit_nitems || !items || !stream_bytes || !vrow_first || !x || !g || !positions ||
      !normals || !cam || !material || !vk || !radiance || !radiance_unclamped)
    return fail(SSS_EINVAL, "bad transfer_v4 arguments");
  if (slot_bytes % 16 || reinterpret_cast<uintptr_t>(stream_bytes) % 16 ||
      (band_width * 8) % 16)
    return fail(SSS_EINVAL, "transfer_v4: 16-byte alignment violated");
  const int T = 1 << levels, T2 = T * T;
  const size_t pipe = (size_t)sss::kV4Slots * slot_bytes +
                      3 * (size_t)sss::kV4XBufs * band_width * 8 +
                      (2 * sss::kV4Slots + 2 * sss::kV4XBufs) * 8 +
                      (size_t)max_unit_items * sizeof(sss::V4Item);
  // partial sums + summed [tile][c][T2] + the batched-Haar scratch of the same size
  const size_t epi = (size_t)sss::kV4TPU * K * 3 * 8 + 2 * (size_t)(sss::kV4TPU / T2 + 1) * 3 * T2 * 8;
  const size_t smem = pipe > epi ? pipe : epi;
  if (smem > 227 * 1024) return fail(SSS_EINVAL, "transfer_v4: shared memory budget exceeded");
#define SSS_T4(KM)                                                                               \
  {                                                                                              \
    if (int r = set_smem((const void*)sss::k_transfer_v4<KM>, smem)) return r;                   \
    sss::k_transfer_v4<KM><<<units, sss::kV4Threads, smem, S_(stream)>>>(                        \
        K, side, levels, band_width, slot_bytes, unit_tile0, unit_ntiles, unit_item0,            \
        unit_nitems, reinterpret_cast<const sss::V4Item*>(items),                                \
        reinterpret_cast<const unsigned char*>(stream_bytes),                                    \
        reinterpret_cast<const unsigned short*>(vrow_first), x, g, positions, normals, cam,      \
        material, vk, scatter, radiance, radiance_unclamped);                                    \
  }
  if (K <= 4) SSS_T4(4)
  else if (K <= 8) SSS_T4(8)
  else if (K <= 12) SSS_T4(12)
  else SSS_T4(16)
#undef SSS_T4
  return check_launch("k_transfer_v4");
}

int sss_transfer_v6(int K, int side, int levels, int band_width, int slot_bytes, int units,
                    int max_unit_items, int max_unit_rows, const int* unit_tile0,
                    const int* unit_ntiles, const int* unit_item0, const int* unit_nitems,
                    const void* items, const void* stream_bytes, const double* x, const double* g,
                    const float* positions, const float* normals, const double* cam,
                    const double* material, double* vk, double* scatter, float* radiance,
                    float* radiance_unclamped, void* stream) {
  if (int r = check_geom(side, levels)) return r;
  if (K <= 0 || K > 16 || units <= 0 || max_unit_rows <= 0 || max_unit_rows > 512 || !unit_tile0 ||
      !unit_ntiles || !unit_item0 || !unit_nitems || !items || !stream_bytes || !x || !g ||
      !positions || !normals || !cam || !material || !vk || !radiance || !radiance_unclamped)
    return fail(SSS_EINVAL, "bad transfer_v6 arguments");
  if (slot_bytes % 16 || reinterpret_cast<uintptr_t>(stream_bytes) % 16 || band_width > 2048 ||
      (band_width * 8) % 16)
    return fail(SSS_EINVAL, "transfer_v6: alignment / band width");
  const int T = 1 << levels, T2 = T * T;
  const size_t smem = (size_t)sss::kV6Slots * slot_bytes +
                      3 * (size_t)sss::kV6XBufs * band_width * 8 +
                      (size_t)max_unit_rows * K * 3 * 8 + 2 * sss::kV6Warps * sizeof(sss::V6Rec) +
                      (2 * sss::kV6Slots + 2 * sss::kV6XBufs) * 8 +
                      (size_t)max_unit_items * sizeof(sss::V6Item);
  const size_t epi = 2 * (size_t)(max_unit_rows / T2 + 1) * 3 * T2 * 8;
  if (smem > 227 * 1024 || epi > (size_t)sss::kV6Slots * slot_bytes)
    return fail(SSS_EINVAL, "transfer_v6: shared memory budget exceeded");
  if (int r = set_smem((const void*)sss::k_transfer_v6, smem)) return r;
  sss::k_transfer_v6<<<units, sss::kV6Threads, smem, S_(stream)>>>(
      K, side, levels, band_width, slot_bytes, unit_tile0, unit_ntiles, unit_item0, unit_nitems,
      reinterpret_cast<const sss::V6Item*>(items), reinterpret_cast<const unsigned char*>(stream_bytes),
      x, g, positions, normals, cam, material, vk, scatter, radiance, radiance_unclamped);
  return check_launch("k_transfer_v6");
}

int sss_pack_x(const double* x, int n, void* xp, void* stream) {
  if (!x || !xp || n <= 0) return fail(SSS_EINVAL, "bad pack_x arguments");
  if (reinterpret_cast<uintptr_t>(xp) % 32) return fail(SSS_EINVAL, "xp must be 32-byte aligned");
  sss::k_pack_x<<<(n + 255) / 256, 256, 0, S_(stream)>>>(x, n, reinterpret_cast<double4*>(xp));
  return check_launch("k_pack_x");
}

int sss_transfer_csr7(int K, int side, int levels, int unit_tiles, const uint64_t* rowptr,
                      const uint32_t* cols, const float* vals, const void* order, const void* xp,
                      const double* g, const float* positions, const float* normals,
                      const double* cam, const double* material, double* vk, double* scatter,
                      float* radiance, float* radiance_unclamped, void* stream) {
  if (int r = check_geom(side, levels)) return r;
  if (K <= 0 || K > 16 || !rowptr || !cols || !vals || !order || !xp || !g || !positions ||
      !normals || !cam || !material || !vk || !radiance || !radiance_unclamped)
    return fail(SSS_EINVAL, "bad transfer_csr7 arguments");
  const int T = 1 << levels, T2 = T * T, tiles = (side / T) * (side / T);
  if (unit_tiles <= 0 || tiles % unit_tiles || unit_tiles * T2 > 4096)
    return fail(SSS_EINVAL, "transfer_csr7: unit_tiles must divide the tile count (<= 4096 rows)");
  const size_t smem = 2 * (size_t)unit_tiles * 3 * T2 * sizeof(double);
  if (int r = set_smem((const void*)sss::k_transfer_csr7, smem)) return r;
  sss::k_transfer_csr7<<<tiles / unit_tiles, sss::kV7Threads, smem, S_(stream)>>>(
      K, side, levels, unit_tiles, rowptr, cols, vals,
      reinterpret_cast<const unsigned short*>(order), reinterpret_cast<const double4*>(xp), g,
      positions, normals, cam, material, vk, scatter, radiance, radiance_unclamped);
  return check_launch("k_transfer_csr7");
}

int sss_transfer_csr8(int K, int n_rows, const uint32_t* cols, const float* vals,
                      const void* pieces, const unsigned* warp_begin, int n_warps, const void* xp,
                      double* vk, void* stream) {
  if (K <= 0 || n_rows <= 0 || !cols || !vals || !pieces || !warp_begin || !xp || !vk ||
      n_warps <= 0 || n_warps % (sss::kV8Threads / 32))
    return fail(SSS_EINVAL, "bad transfer_csr8 arguments");
  cudaError_t e = cudaMemsetAsync(vk, 0, (size_t)K * 3 * n_rows * sizeof(double), S_(stream));
  if (e != cudaSuccess) return fail(SSS_ECUDA, cudaGetErrorString(e));
  sss::k_transfer_csr8<<<n_warps / (sss::kV8Threads / 32), sss::kV8Threads, 0, S_(stream)>>>(
      n_rows, cols, vals, reinterpret_cast<const sss::V8Piece*>(pieces), warp_begin,
      reinterpret_cast<const double4*>(xp), vk);
  return check_launch("k_transfer_csr8");
}

int sss_pad_segments(const uint64_t* seg_src, const uint32_t* seg_len, const uint64_t* seg_dst,
                     long long nseg, const uint32_t* cols, const float* vals, uint32_t* pcols,
                     float* pvals, void* stream) {
  if (!seg_src || !seg_len || !seg_dst || nseg < 0 || !cols || !vals || !pcols || !pvals)
    return fail(SSS_EINVAL, "bad pad_segments arguments");
  if (nseg == 0) return SSS_OK;
  sss::k_pad_segments<<<(unsigned)((nseg + 7) / 8), 256, 0, S_(stream)>>>(seg_src, seg_len, seg_dst,
                                                                          nseg, cols, vals, pcols,
                                                                          pvals);
  return check_launch("k_pad_segments");
}

int sss_transfer_csr9(int K, int n_rows, const uint32_t* pcols, const float* pvals,
                      const void* pieces, const unsigned* warp_begin, int n_warps, const void* xp,
                      double* vk, void* stream) {
  if (K <= 0 || n_rows <= 0 || !pcols || !pvals || !pieces || !warp_begin || !xp || !vk ||
      n_warps <= 0 || n_warps % (sss::kV9Threads / 32))
    return fail(SSS_EINVAL, "bad transfer_csr9 arguments");
  if (reinterpret_cast<uintptr_t>(pcols) % 16 || reinterpret_cast<uintptr_t>(pvals) % 16)
    return fail(SSS_EINVAL, "transfer_csr9: padded arrays must be 16-byte aligned");
  cudaError_t e = cudaMemsetAsync(vk, 0, (size_t)K * 3 * n_rows * sizeof(double), S_(stream));
  if (e != cudaSuccess) return fail(SSS_ECUDA, cudaGetErrorString(e));
  sss::k_transfer_csr9<<<n_warps / (sss::kV9Threads / 32), sss::kV9Threads, 0, S_(stream)>>>(
      n_rows, reinterpret_cast<const uint4*>(pcols), reinterpret_cast<const float4*>(pvals),
      reinterpret_cast<const sss::V9Piece*>(pieces), warp_begin,
      reinterpret_cast<const double4*>(xp), vk);
  return check_launch("k_transfer_csr9");
}

int sss_transfer_kpack(int K, int n_rows, const uint32_t* meta, const float* vals,
                       const void* pieces, const unsigned* warp_begin, int n_warps, const void* xp,
                       double* vk, void* stream) {
  if (K <= 0 || K > 8 || n_rows <= 0 || n_rows > (1 << 24) || !meta || !vals || !pieces ||
      !warp_begin || !xp || !vk || n_warps <= 0 || n_warps % (sss::kV10Threads / 32))
    return fail(SSS_EINVAL, "bad transfer_kpack arguments");
  if (reinterpret_cast<uintptr_t>(meta) % 16)
    return fail(SSS_EINVAL, "transfer_kpack: meta must be 16-byte aligned");
  cudaError_t e = cudaMemsetAsync(vk, 0, (size_t)K * 3 * n_rows * sizeof(double), S_(stream));
  if (e != cudaSuccess) return fail(SSS_ECUDA, cudaGetErrorString(e));
  const unsigned grid = n_warps / (sss::kV10Threads / 32);
  const auto* pc = reinterpret_cast<const sss::V10Piece*>(pieces);
  const auto* x4 = reinterpret_cast<const double4*>(xp);
  const auto* m4 = reinterpret_cast<const uint4*>(meta);
  if (K <= 4)
    sss::k_transfer_kpack<4><<<grid, sss::kV10Threads, 0, S_(stream)>>>(K, n_rows, m4, vals, pc,
                                                                       warp_begin, x4, vk);
  else
    sss::k_transfer_kpack<8><<<grid, sss::kV10Threads, 0, S_(stream)>>>(K, n_rows, m4, vals, pc,
                                                                       warp_begin, x4, vk);
  return check_launch("k_transfer_kpack");
}

int sss_transfer_kpack_pipe(int K, int n_rows, const uint32_t* meta, const float* vals,
                            const void* pieces, const unsigned* warp_begin, int n_warps,
                            int pairs_per_lane, const void* xp, double* vk, void* stream) {
  if (K <= 0 || K > 8 || n_rows <= 0 || n_rows > (1 << 24) || !meta || !vals || !pieces ||
      !warp_begin || !xp || !vk || n_warps <= 0 || n_warps % (sss::kV11Threads / 32) ||
      (pairs_per_lane != 2 && pairs_per_lane != 4))
    return fail(SSS_EINVAL, "bad transfer_kpack_pipe arguments");
  if (reinterpret_cast<uintptr_t>(meta) % 16)
    return fail(SSS_EINVAL, "transfer_kpack_pipe: meta must be 16-byte aligned");
  cudaError_t e = cudaMemsetAsync(vk, 0, (size_t)K * 3 * n_rows * sizeof(double), S_(stream));
  if (e != cudaSuccess) return fail(SSS_ECUDA, cudaGetErrorString(e));
  const unsigned grid = n_warps / (sss::kV11Threads / 32);
  const auto* pc = reinterpret_cast<const sss::V10Piece*>(pieces);
  const auto* x4 = reinterpret_cast<const double4*>(xp);
#define SSS_KP(KM, PP)                                                                     \
  sss::k_transfer_kpack_pipe<KM, PP><<<grid, sss::kV11Threads, 0, S_(stream)>>>(K, n_rows, meta, \
                                                                               vals, pc,   \
                                                                               warp_begin, \
                                                                               x4, vk)
  if (K <= 4) {
    if (pairs_per_lane == 4) SSS_KP(4, 4); else SSS_KP(4, 2);
  } else {
    if (pairs_per_lane == 4) SSS_KP(8, 4); else SSS_KP(8, 2);
  }
#undef SSS_KP
  return check_launch("k_transfer_kpack_pipe");
}

int sss_transfer_kstep(int K, int n_rows, const uint32_t* cols, const float* vals,
                       const void* steps, const unsigned* warp_begin, int n_warps, const void* xp,
                       double* vk, void* stream) {
  if (K <= 0 || K > 8 || n_rows <= 0 || !cols || !vals || !steps || !warp_begin || !xp || !vk ||
      n_warps <= 0 || n_warps % (sss::kV12Threads / 32))
    return fail(SSS_EINVAL, "bad transfer_kstep arguments");
  cudaError_t e = cudaMemsetAsync(vk, 0, (size_t)K * 3 * n_rows * sizeof(double), S_(stream));
  if (e != cudaSuccess) return fail(SSS_ECUDA, cudaGetErrorString(e));
  sss::k_transfer_kstep<<<n_warps / (sss::kV12Threads / 32), sss::kV12Threads, 0, S_(stream)>>>(
      K, n_rows, cols, vals, reinterpret_cast<const uint4*>(steps), warp_begin,
      reinterpret_cast<const double4*>(xp), vk);
  return check_launch("k_transfer_kstep");
}

int sss_transfer_kstream(int K, int n_rows, const void* blob, const void* recs,
                         const unsigned* warp_begin, int n_warps, int depth, const void* xp,
                         double* vk, void* stream) {
  if (K <= 0 || K > 8 || n_rows <= 0 || !blob || !recs || !warp_begin || !xp || !vk ||
      n_warps <= 0 || n_warps % (sss::kV13Threads / 32) || (depth != 4 && depth != 8 && depth != 12))
    return fail(SSS_EINVAL, "bad transfer_kstream arguments");
  if (reinterpret_cast<uintptr_t>(blob) % 16 || reinterpret_cast<uintptr_t>(recs) % 16 ||
      reinterpret_cast<uintptr_t>(xp) % 32)
    return fail(SSS_EINVAL, "transfer_kstream: blob/recs 16-byte and xp 32-byte aligned");
  cudaError_t e = cudaMemsetAsync(vk, 0, (size_t)K * 3 * n_rows * sizeof(double), S_(stream));
  if (e != cudaSuccess) return fail(SSS_ECUDA, cudaGetErrorString(e));
  const unsigned grid = n_warps / (sss::kV13Threads / 32);
  const auto* b8 = reinterpret_cast<const uint8_t*>(blob);
  const auto* r4 = reinterpret_cast<const uint4*>(recs);
  const auto* x4 = reinterpret_cast<const double4*>(xp);
#define SSS_KS(DD, GG)                                                                             \
  do {                                                                                             \
    const size_t smem = (sss::kV13Threads / 32) * sss::V13Smem<DD, GG>::per_warp;                  \
    const void* fn = (const void*)sss::k_transfer_kstream<DD, GG>;                                 \
    if (int r = set_smem(fn, smem)) return r;                                                      \
    cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100);                 \
    sss::k_transfer_kstream<DD, GG><<<grid, sss::kV13Threads, smem, S_(stream)>>>(                 \
        K, n_rows, b8, r4, warp_begin, x4, vk);                                                    \
  } while (0)
  if (depth == 4) SSS_KS(4, 2);
  else if (depth == 8) SSS_KS(8, 3);
  else SSS_KS(12, 4);
#undef SSS_KS
  return check_launch("k_transfer_kstream");
}

int sss_pack_x_bits(const double* x, int n, void* xp, uint32_t* bits, void* stream) {
  if (!x || !xp || !bits || n <= 0) return fail(SSS_EINVAL, "bad pack_x_bits arguments");
  if (reinterpret_cast<uintptr_t>(xp) % 32) return fail(SSS_EINVAL, "xp must be 32-byte aligned");
  sss::k_pack_x_bits<<<(n + 255) / 256, 256, 0, S_(stream)>>>(x, n, reinterpret_cast<double4*>(xp),
                                                             bits);
  return check_launch("k_pack_x_bits");
}

int sss_transfer_csr9s(int K, int n_rows, const uint32_t* pcols, const float* pvals,
                       const void* pieces, const unsigned* warp_begin, int n_warps, const void* xp,
                       const uint32_t* bits, double* vk, void* stream) {
  if (K <= 0 || n_rows <= 0 || !pcols || !pvals || !pieces || !warp_begin || !xp || !bits || !vk ||
      n_warps <= 0 || n_warps % (sss::kV9Threads / 32))
    return fail(SSS_EINVAL, "bad transfer_csr9s arguments");
  if (reinterpret_cast<uintptr_t>(pcols) % 16 || reinterpret_cast<uintptr_t>(pvals) % 16)
    return fail(SSS_EINVAL, "transfer_csr9s: padded arrays must be 16-byte aligned");
  const size_t smem = (size_t)((n_rows + 31) / 32) * 4;
  if (int r = set_smem((const void*)sss::k_transfer_csr9s, smem)) return r;
  cudaError_t e = cudaMemsetAsync(vk, 0, (size_t)K * 3 * n_rows * sizeof(double), S_(stream));
  if (e != cudaSuccess) return fail(SSS_ECUDA, cudaGetErrorString(e));
  sss::k_transfer_csr9s<<<n_warps / (sss::kV9Threads / 32), sss::kV9Threads, smem, S_(stream)>>>(
      n_rows, reinterpret_cast<const uint4*>(pcols), reinterpret_cast<const float4*>(pvals),
      reinterpret_cast<const sss::V9Piece*>(pieces), warp_begin,
      reinterpret_cast<const double4*>(xp), bits, vk);
  return check_launch("k_transfer_csr9s");
}

int sss_transfer_kgroup(int K, int n_rows, const uint32_t* meta, const float* vals,
                        const void* pieces, const unsigned* warp_begin, int n_warps, const void* xp,
                        const uint32_t* bits, double* vk, void* stream) {
  if (K <= 0 || K > 8 || n_rows <= 0 || n_rows > (1 << 24) || !meta || !vals || !pieces ||
      !warp_begin || !xp || !bits || !vk || n_warps <= 0 || n_warps % (sss::kV14Threads / 32))
    return fail(SSS_EINVAL, "bad transfer_kgroup arguments");
  if (reinterpret_cast<uintptr_t>(xp) % 32) return fail(SSS_EINVAL, "xp must be 32-byte aligned");
  const size_t smem = (size_t)((n_rows + 31) / 32) * 4;
  if (int r = set_smem((const void*)sss::k_transfer_kgroup, smem)) return r;
  cudaError_t e = cudaMemsetAsync(vk, 0, (size_t)K * 3 * n_rows * sizeof(double), S_(stream));
  if (e != cudaSuccess) return fail(SSS_ECUDA, cudaGetErrorString(e));
  sss::k_transfer_kgroup<<<n_warps / (sss::kV14Threads / 32), sss::kV14Threads, smem, S_(stream)>>>(
      K, n_rows, meta, vals, reinterpret_cast<const sss::V14Row*>(pieces), warp_begin,
      reinterpret_cast<const double4*>(xp), bits, vk);
  return check_launch("k_transfer_kgroup");
}

int sss_transfer_flat(int K, int n_rows, const uint32_t* pcols, const float* pvals,
                      unsigned long long n_entries, const uint32_t* heads,
                      const uint32_t* head_prefix, const uint32_t* seg_rowk,
                      const unsigned* warp_begin, int n_warps, const void* xp,
                      const uint32_t* bits, double* vk, void* stream) {
  if (K <= 0 || n_rows <= 0 || !pcols || !pvals || !heads || !head_prefix || !seg_rowk ||
      !warp_begin || !xp || !vk || n_warps <= 0 || n_warps % (sss::kV15Threads / 32) ||
      n_entries % 4 || n_entries / 4 >= (1ull << 32) - 64)
    return fail(SSS_EINVAL, "bad transfer_flat arguments");
  if (reinterpret_cast<uintptr_t>(pcols) % 16 || reinterpret_cast<uintptr_t>(pvals) % 16 ||
      reinterpret_cast<uintptr_t>(xp) % 32)
    return fail(SSS_EINVAL, "transfer_flat: pcols/pvals 16-byte, xp 32-byte aligned");
  cudaError_t e = cudaMemsetAsync(vk, 0, (size_t)K * 3 * n_rows * sizeof(double), S_(stream));
  if (e != cudaSuccess) return fail(SSS_ECUDA, cudaGetErrorString(e));
  const size_t smem = bits ? (size_t)((n_rows + 31) / 32) * 4 : 0;
  if (int r = set_smem((const void*)sss::k_transfer_flat<0>, smem)) return r;
  sss::k_transfer_flat<0><<<n_warps / (sss::kV15Threads / 32), sss::kV15Threads, smem,
                            S_(stream)>>>(
      n_rows, (unsigned)(n_entries / 4), reinterpret_cast<const uint4*>(pcols),
      reinterpret_cast<const float4*>(pvals), heads, head_prefix, seg_rowk, warp_begin,
      reinterpret_cast<const double4*>(xp), bits, vk);
  return check_launch("k_transfer_flat");
}

int sss_transfer_flatp(int K, int n_rows, const uint32_t* pcols, const float* pvals,
                       unsigned long long n_entries, const uint32_t* heads,
                       const uint32_t* head_prefix, const uint32_t* seg_rowk,
                       const unsigned* warp_begin, int n_warps, int depth, const void* xp,
                       double* vk, void* stream) {
  if (K <= 0 || n_rows <= 0 || !pcols || !pvals || !heads || !head_prefix || !seg_rowk ||
      !warp_begin || !xp || !vk || n_warps <= 0 || n_warps % (sss::kV16Threads / 32) ||
      n_entries % 4 || n_entries / 4 >= (1ull << 32) - 64 ||
      (depth != 4 && depth != 8 && depth != 12))
    return fail(SSS_EINVAL, "bad transfer_flatp arguments");
  if (reinterpret_cast<uintptr_t>(pcols) % 16 || reinterpret_cast<uintptr_t>(pvals) % 16 ||
      reinterpret_cast<uintptr_t>(xp) % 32)
    return fail(SSS_EINVAL, "transfer_flatp: pcols/pvals 16-byte, xp 32-byte aligned");
  cudaError_t e = cudaMemsetAsync(vk, 0, (size_t)K * 3 * n_rows * sizeof(double), S_(stream));
  if (e != cudaSuccess) return fail(SSS_ECUDA, cudaGetErrorString(e));
  const unsigned grid = n_warps / (sss::kV16Threads / 32);
  const auto* c4 = reinterpret_cast<const uint4*>(pcols);
  const auto* v4 = reinterpret_cast<const float4*>(pvals);
  const auto* x4 = reinterpret_cast<const double4*>(xp);
  const unsigned n4 = (unsigned)(n_entries / 4);
#define SSS_FP(RR)                                                                                \
  do {                                                                                            \
    const size_t smem = (size_t)(sss::kV16Threads / 32) * RR * sizeof(sss::V16Slot<RR>);          \
    const void* fn = (const void*)sss::k_transfer_flatp<RR>;                                      \
    if (int r = set_smem(fn, smem)) return r;                                                     \
    cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100);                \
    sss::k_transfer_flatp<RR><<<grid, sss::kV16Threads, smem, S_(stream)>>>(                      \
        n_rows, n4, c4, v4, heads, head_prefix, seg_rowk, warp_begin, x4, vk);                    \
  } while (0)
  if (depth == 4) SSS_FP(4);
  else if (depth == 8) SSS_FP(8);
  else SSS_FP(12);
#undef SSS_FP
  return check_launch("k_transfer_flatp");
}

int sss_pack_x_perm_bits(const double* x, int n, const int* perm, void* xp, uint32_t* bits,
                         void* stream) {
  if (!x || !perm || !xp || !bits || n <= 0) return fail(SSS_EINVAL, "bad pack_x_perm_bits arguments");
  if (reinterpret_cast<uintptr_t>(xp) % 32) return fail(SSS_EINVAL, "xp must be 32-byte aligned");
  sss::k_pack_x_perm_bits<<<(n + 255) / 256, 256, 0, S_(stream)>>>(
      x, n, perm, reinterpret_cast<double4*>(xp), bits);
  return check_launch("k_pack_x_perm_bits");
}

int sss_pack_x_f32_bits(const double* x, int n, void* xp, uint32_t* bits, void* stream) {
  if (!x || !xp || !bits || n <= 0) return fail(SSS_EINVAL, "bad pack_x_f32_bits arguments");
  if (reinterpret_cast<uintptr_t>(xp) % 16) return fail(SSS_EINVAL, "xp must be 16-byte aligned");
  sss::k_pack_x_f32_bits<<<(n + 255) / 256, 256, 0, S_(stream)>>>(x, n, reinterpret_cast<float4*>(xp),
                                                                 bits);
  return check_launch("k_pack_x_f32_bits");
}

int sss_transfer_flat8(int K, int n_rows, const uint32_t* pcols, const float* pvals,
                       unsigned long long n_entries, const uint32_t* heads,
                       const uint32_t* head_prefix, const uint32_t* seg_rowk,
                       const unsigned* warp_begin, int n_warps, const void* xp,
                       const uint32_t* bits, int variant, int x_f32, double* vk,
                       void* stream) {
  const int gather_ahead = variant;
  if (K <= 0 || n_rows <= 0 || !pcols || !pvals || !heads || !head_prefix || !seg_rowk ||
      !warp_begin || !xp || !vk || n_warps <= 0 || n_warps % (sss::kV17Threads / 32) ||
      n_entries % 8 || n_entries / 8 >= (1ull << 32) - 64)
    return fail(SSS_EINVAL, "bad transfer_flat8 arguments");
  if (reinterpret_cast<uintptr_t>(pcols) % 32 || reinterpret_cast<uintptr_t>(pvals) % 32 ||
      reinterpret_cast<uintptr_t>(xp) % 32)
    return fail(SSS_EINVAL, "transfer_flat8: pcols/pvals/xp must be 32-byte aligned");
  cudaError_t e = cudaMemsetAsync(vk, 0, (size_t)K * 3 * n_rows * sizeof(double), S_(stream));
  if (e != cudaSuccess) return fail(SSS_ECUDA, cudaGetErrorString(e));
  const size_t smem = bits ? (size_t)((n_rows + 31) / 32) * 4 : 0;
  const auto* c8 = reinterpret_cast<const unsigned long long*>(pcols);
  const auto* v8 = reinterpret_cast<const unsigned long long*>(pvals);
  const auto* x4 = reinterpret_cast<const double4*>(xp);
  const unsigned grid = n_warps / (sss::kV17Threads / 32);
  const unsigned n8 = (unsigned)(n_entries / 8);
  if (gather_ahead >= 4) {  // split-half variants with a register cap: 4 + min CTAs/SM - 4
    const int minb = gather_ahead;
#define SSS_F8S(MB)                                                                               \
    do {                                                                                          \
      if (int r = set_smem((const void*)sss::k_transfer_flat8s<MB>, smem)) return r;              \
      sss::k_transfer_flat8s<MB><<<grid, sss::kV17Threads, smem, S_(stream)>>>(                   \
          n_rows, n8, c8, v8, heads, head_prefix, seg_rowk, warp_begin, x4, bits, vk);            \
    } while (0)
#define SSS_F8S1(MB)                                                                              \
    do {                                                                                          \
      if (int r = set_smem((const void*)sss::k_transfer_flat8s<MB, true>, smem)) return r;        \
      sss::k_transfer_flat8s<MB, true><<<grid, sss::kV17Threads, smem, S_(stream)>>>(             \
          n_rows, n8, c8, v8, heads, head_prefix, seg_rowk, warp_begin, x4, bits, vk);            \
    } while (0)
    if (x_f32 && minb == 16) {
      const auto* xf = reinterpret_cast<const float4*>(xp);
      if (int r = set_smem((const void*)sss::k_transfer_flat8s<8, true, float, float4>, smem)) return r;
      sss::k_transfer_flat8s<8, true, float, float4><<<grid, sss::kV17Threads, smem, S_(stream)>>>(
          n_rows, n8, c8, v8, heads, head_prefix, seg_rowk, warp_begin, xf, bits, vk);
    } else if (minb == 14) SSS_F8S1(6);
    else if (minb == 16) SSS_F8S1(8);
    else if (minb == 18) SSS_F8S1(10);
    else if (minb == 4) SSS_F8S(4);
    else if (minb == 5) SSS_F8S(5);
    else if (minb == 7) SSS_F8S(7);
    else if (minb == 8) SSS_F8S(8);
    else SSS_F8S(6);
#undef SSS_F8S
#undef SSS_F8S1
  } else if (x_f32) {
    const auto* xf = reinterpret_cast<const float4*>(xp);
    if (int r = set_smem((const void*)sss::k_transfer_flat8<false, float, float4>, smem)) return r;
    sss::k_transfer_flat8<false, float, float4><<<grid, sss::kV17Threads, smem, S_(stream)>>>(
        n_rows, n8, c8, v8, heads, head_prefix, seg_rowk, warp_begin, xf, bits, vk);
  } else if (gather_ahead) {
    if (int r = set_smem((const void*)sss::k_transfer_flat8<true>, smem)) return r;
    sss::k_transfer_flat8<true><<<grid, sss::kV17Threads, smem, S_(stream)>>>(
        n_rows, n8, c8, v8, heads, head_prefix, seg_rowk, warp_begin, x4, bits, vk);
  } else {
    if (int r = set_smem((const void*)sss::k_transfer_flat8<false>, smem)) return r;
    sss::k_transfer_flat8<false><<<grid, sss::kV17Threads, smem, S_(stream)>>>(
        n_rows, n8, c8, v8, heads, head_prefix, seg_rowk, warp_begin, x4, bits, vk);
  }
  return check_launch("k_transfer_flat8");
}

int sss_transfer_kflat(int K, int n_rows, const uint32_t* cols, const float* vals,
                       const void* steps, const unsigned* warp_begin, int n_warps, const void* xp,
                       const uint32_t* bits, double* vk, void* stream) {
  if (K <= 0 || K > 8 || n_rows <= 0 || !cols || !vals || !steps || !warp_begin || !xp || !vk ||
      n_warps <= 0 || n_warps % (sss::kV18Threads / 32))
    return fail(SSS_EINVAL, "bad transfer_kflat arguments");
  if (reinterpret_cast<uintptr_t>(xp) % 32 || reinterpret_cast<uintptr_t>(steps) % 16)
    return fail(SSS_EINVAL, "transfer_kflat: xp 32-byte, steps 16-byte aligned");
  cudaError_t e = cudaMemsetAsync(vk, 0, (size_t)K * 3 * n_rows * sizeof(double), S_(stream));
  if (e != cudaSuccess) return fail(SSS_ECUDA, cudaGetErrorString(e));
  const size_t smem = bits ? (size_t)((n_rows + 31) / 32) * 4 : 0;
  if (int r = set_smem((const void*)sss::k_transfer_kflat<0>, smem)) return r;
  sss::k_transfer_kflat<0><<<n_warps / (sss::kV18Threads / 32), sss::kV18Threads, smem,
                             S_(stream)>>>(K, n_rows, cols, vals,
                                           reinterpret_cast<const uint4*>(steps), warp_begin,
                                           reinterpret_cast<const double4*>(xp), bits, vk);
  return check_launch("k_transfer_kflat");
}

int sss_sweep_basis(int K, int side, int levels, const double* vk, void* Bq, void* stream) {
  if (int r = check_geom(side, levels)) return r;
  if (K <= 0 || K > sss::kSweepK || !vk || !Bq) return fail(SSS_EINVAL, "bad sweep_basis arguments");
  const int T = 1 << levels, T2 = T * T, tiles = (side / T) * (side / T);
  const size_t smem = 2 * 3 * (size_t)K * T2 * sizeof(double);
  if (int r = set_smem((const void*)sss::k_sweep_basis, smem)) return r;
  sss::k_sweep_basis<<<tiles, 256, smem, S_(stream)>>>(K, side, levels, vk,
                                                     reinterpret_cast<__nv_bfloat16*>(Bq));
  return check_launch("k_sweep_basis");
}

int sss_material_weights_batch(const double* bw, const double* r_nodes, int K, int nr, int M,
                               const double* materials, double* g64, void* Gq, float* eta_f,
                               void* stream) {
  if (K <= 0 || K > sss::kSweepK || nr < 2 || M <= 0 || M > 65535 || !bw || !r_nodes ||
      !materials || !Gq)
    return fail(SSS_EINVAL, "bad material_weights_batch arguments");
  sss::k_material_weights_batch<<<dim3(3, M), 256, 0, S_(stream)>>>(
      bw, r_nodes, K, nr, M, materials, g64, reinterpret_cast<__nv_bfloat16*>(Gq), eta_f);
  return check_launch("k_material_weights_batch");
}

static int sweep_variant() {
  const char* e = getenv("SSS_SWEEP_VARIANT");
  return e ? atoi(e) : 0;
}

int sss_sweep_gemm(int n_points, int M, const void* Bq, const void* Gq, const float* eta,
                   float eta_lo, float eta_hi, const float* positions, const float* normals,
                   const double* cam, float* out, void* stream) {
  if (n_points <= 0 || M <= 0 || !Bq || !Gq || !eta || !positions || !normals || !cam || !out ||
      !(eta_hi >= eta_lo) || eta_lo <= 1.0f)
    return fail(SSS_EINVAL, "bad sweep_gemm arguments (eta must exceed 1)");
  if (reinterpret_cast<uintptr_t>(Bq) % 16 || reinterpret_cast<uintptr_t>(Gq) % 16)
    return fail(SSS_EINVAL, "sweep_gemm: Bq / Gq must be 16-byte aligned");
  // variant: materials per UMMA (N) and threads per CTA; the dynamic shared
  // memory request caps residency at what TMEM (512 columns / SM) allows
  const int variant = sweep_variant();
  const dim3 g1((n_points + sss::kSweepTileM - 1) / sss::kSweepTileM, 3, 1);
#define SSS_SW(TMN, THR, SMEMKB)                                                                   \
  do {                                                                                             \
    const size_t smem = (size_t)(SMEMKB) * 1024;                                                  \
    const void* fn = (const void*)sss::k_sweep_umma<TMN, THR>;                                     \
    if (int r = set_smem(fn, smem)) return r;                                                      \
    dim3 grid = g1;                                                                                \
    grid.z = (M + TMN - 1) / TMN;                                                                  \
    sss::k_sweep_umma<TMN, THR><<<grid, THR, smem, S_(stream)>>>(                                  \
        n_points, M, reinterpret_cast<const __nv_bfloat16*>(Bq),                                   \
        reinterpret_cast<const __nv_bfloat16*>(Gq), eta, eta_lo, eta_hi, positions, normals, cam,   \
        out);                                                                                      \
  } while (0)
  if (variant == 1) SSS_SW(256, 128, 80);
  else if (variant == 2) SSS_SW(256, 256, 80);
  else SSS_SW(128, 256, 52);
#undef SSS_SW
  return check_launch("k_sweep_umma");
}

int sss_transfer_regional(int K, int n_rows, const uint32_t* ucols, const int* uoff,
                          const int* rit, int n_regions, int umax, const uint32_t* pcols,
                          const float* pvals, unsigned long long n_entries,
                          const uint32_t* heads, const uint32_t* head_prefix,
                          const uint32_t* seg_rowk, const void* xp, const uint32_t* bits,
                          double* vk, void* stream) {
  if (K <= 0 || n_rows <= 0 || !ucols || !uoff || !rit || n_regions <= 0 || umax <= 0 ||
      umax >= 32768 || !pcols || !pvals || !heads || !head_prefix || !seg_rowk || !xp || !bits ||
      !vk || n_entries % 8)
    return fail(SSS_EINVAL, "bad transfer_regional arguments");
  if (reinterpret_cast<uintptr_t>(pcols) % 32 || reinterpret_cast<uintptr_t>(pvals) % 32 ||
      reinterpret_cast<uintptr_t>(xp) % 32)
    return fail(SSS_EINVAL, "transfer_regional: pcols/pvals/xp must be 32-byte aligned");
  int dev = 0, nsm = 148, smem_optin = 227 * 1024;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  const size_t bits_b = (((size_t)(n_rows + 31) / 32) * 4 + 15) & ~size_t(15);
  const size_t map_b = (size_t)umax * sizeof(short);
  const long long room = (long long)smem_optin - 1024 - (long long)bits_b - (long long)map_b;
  if (room < 24 * 256) return fail(SSS_EINVAL, "transfer_regional: not enough shared memory");
  const int xcap = (int)std::min<long long>(room / 24, 32767);
  const size_t smem = bits_b + (size_t)xcap * 24 + map_b;
  if (int r = set_smem((const void*)sss::k_transfer_regional, smem)) return r;
  cudaError_t e = cudaMemsetAsync(vk, 0, (size_t)K * 3 * n_rows * sizeof(double), S_(stream));
  if (e != cudaSuccess) return fail(SSS_ECUDA, cudaGetErrorString(e));
  const int grid = std::min(n_regions, nsm);
  sss::k_transfer_regional<<<grid, sss::kV19Threads, smem, S_(stream)>>>(
      n_rows, n_regions, xcap, ucols, uoff, rit, reinterpret_cast<const unsigned long long*>(pcols),
      reinterpret_cast<const unsigned long long*>(pvals), (unsigned)(n_entries / 8), heads,
      head_prefix, seg_rowk, reinterpret_cast<const double4*>(xp), bits, vk);
  return check_launch("k_transfer_regional");
}

int sss_transfer_k8(int K, int n_rows, const uint32_t* cols, const float* vals, const void* pieces,
                    const unsigned* warp_begin, int n_warps, int min_ctas, const void* xp,
                    const uint32_t* bits, double* vk, void* stream) {
  if (K <= 0 || K > 8 || n_rows <= 0 || !cols || !vals || !pieces || !warp_begin || !xp ||
      !bits || !vk || n_warps <= 0 || n_warps % (sss::kV20Threads / 32))
    return fail(SSS_EINVAL, "bad transfer_k8 arguments");
  if (reinterpret_cast<uintptr_t>(vals) % 16 || reinterpret_cast<uintptr_t>(xp) % 32 ||
      reinterpret_cast<uintptr_t>(pieces) % 16)
    return fail(SSS_EINVAL, "transfer_k8: vals / pieces 16-byte, xp 32-byte aligned");
  cudaError_t e = cudaMemsetAsync(vk, 0, (size_t)K * 3 * n_rows * sizeof(double), S_(stream));
  if (e != cudaSuccess) return fail(SSS_ECUDA, cudaGetErrorString(e));
  const size_t smem = (size_t)((n_rows + 31) / 32) * 4;
  const unsigned grid = n_warps / (sss::kV20Threads / 32);
  const auto* v4 = reinterpret_cast<const float4*>(vals);
  const auto* pc = reinterpret_cast<const uint4*>(pieces);
  const auto* x4 = reinterpret_cast<const double4*>(xp);
#define SSS_K8(MB)                                                                              \
  do {                                                                                          \
    if (int r = set_smem((const void*)sss::k_transfer_k8<MB>, smem)) return r;                  \
    sss::k_transfer_k8<MB><<<grid, sss::kV20Threads, smem, S_(stream)>>>(K, n_rows, cols, v4,   \
                                                                         pc, warp_begin, x4,    \
                                                                         bits, vk);             \
  } while (0)
  if (min_ctas >= 3) SSS_K8(3);
  else if (min_ctas == 2) SSS_K8(2);
  else SSS_K8(1);
#undef SSS_K8
  return check_launch("k_transfer_k8");
}

int sss_direct_irradiance(int n_points, const float* positions, const float* normals,
                          int n_lights, const int* kinds, const double* lights,
                          const double* material, double ray_offset, double bbox_diagonal,
                          const double* nodes, const double* tris, double* E, void* stream) {
  if (n_points <= 0 || n_lights < 0 || !positions || !normals || !material || !E || !nodes ||
      !tris || (n_lights > 0 && (!lights || !kinds)))
    return fail(SSS_EINVAL, "bad direct_irradiance arguments");
  for (int l = 0; l < n_lights; ++l)
    if (kinds[l] < 0 || kinds[l] > 2) return fail(SSS_EINVAL, "unknown light kind");
  cudaStream_t st = S_(stream);
  if (cudaMemsetAsync(E, 0, sizeof(double) * 3 * (size_t)n_points, st) != cudaSuccess)
    return fail(SSS_ECUDA, "memset E");
  const sss::BvhView B{reinterpret_cast<const double2*>(nodes),
                       reinterpret_cast<const double2*>(tris)};
  const char* sv = getenv("SSS_DIRECT_SPLIT");
  const int split = sv ? atoi(sv) : 3;
  for (int l = 0; l < n_lights; ++l) {
    const double* L = lights + 12 * (size_t)l;
    if (kinds[l] < 2) {
#define SSS_DS(K, S)                                                                        \
  do {                                                                                      \
    const int grid = (n_points + (sss::kDirectThreads >> S) - 1) / (sss::kDirectThreads >> S); \
    sss::k_direct_single<K, S><<<grid, sss::kDirectThreads, 0, st>>>(                       \
        n_points, positions, normals, L, material, ray_offset, bbox_diagonal, B, E);         \
  } while (0)
#define SSS_DSK(K)        \
  if (split <= 0) SSS_DS(K, 0); \
  else if (split == 1) SSS_DS(K, 1); \
  else if (split == 2) SSS_DS(K, 2); \
  else if (split == 3) SSS_DS(K, 3); \
  else SSS_DS(K, 4)
      if (kinds[l] == 0) { SSS_DSK(0); } else { SSS_DSK(1); }
#undef SSS_DSK
#undef SSS_DS
    } else {
      sss::k_direct_sphere<<<(n_points + sss::kSpherePts - 1) / sss::kSpherePts,
                             64 * sss::kSpherePts, 0, st>>>(n_points, positions, normals, L,
                                                            material, ray_offset, B, E);
    }
    const int rc = check_launch("k_direct_light");
    if (rc) return rc;
  }
  return SSS_OK;
}

int sss_visibility(int n_points, const float* positions, const float* normals, int n_dirs,
                   const double* dirs, double ray_offset, double far, const double* nodes,
                   const double* tris, uint8_t* vis, void* stream) {
  if (n_points <= 0 || n_dirs <= 0 || n_dirs > 65535 || !positions || !normals || !dirs ||
      !nodes || !tris || !vis)
    return fail(SSS_EINVAL, "bad visibility arguments");
  const sss::BvhView B{reinterpret_cast<const double2*>(nodes),
                       reinterpret_cast<const double2*>(tris)};
  dim3 grid((n_points + 127) / 128, n_dirs);
  sss::k_visibility<<<grid, 128, 0, S_(stream)>>>(n_points, positions, normals, dirs, ray_offset,
                                                  far, B, vis);
  return check_launch("k_visibility");
}

int sss_fold_weights(const float* normals, int n_points, const double* dirs, const double* dom,
                     int face_side, const uint8_t* vis, double eta, double* W2, void* stream) {
  if (!normals || !dirs || !dom || !vis || !W2 || n_points <= 0 || face_side <= 0 ||
      (face_side & (face_side - 1)))
    return fail(SSS_EINVAL, "bad fold_weights arguments");
  const int s2 = face_side * face_side;
  const size_t smem = sizeof(double) * (size_t)(sss::kFoldP + 1) * s2;
  if (int r = set_smem((const void*)sss::k_fold_weights, smem)) return r;
  dim3 grid((n_points + sss::kFoldP - 1) / sss::kFoldP, 6);
  sss::k_fold_weights<<<grid, 256, smem, S_(stream)>>>(normals, n_points, dirs, dom, face_side,
                                                      vis, eta, W2);
  return check_launch("k_fold_weights");
}

int sss_transpose_f64(const double* in, int rows, int cols, const uint32_t* col_perm, double* out,
                      void* stream) {
  if (!in || !out || rows <= 0 || cols <= 0 || (rows + 31) / 32 > 65535)
    return fail(SSS_EINVAL, "bad transpose arguments");
  dim3 grid((cols + 31) / 32, (rows + 31) / 32);
  sss::k_transpose_perm<<<grid, dim3(32, 8), 0, S_(stream)>>>(in, rows, cols, col_perm, out);
  return check_launch("k_transpose_perm");
}

int sss_fold_spmm(int n_rows, int n_dirs, const long long* rowptr, const uint32_t* cols,
                  const float* vals, const double* vt, double* F, void* stream) {
  if (n_rows <= 0 || n_dirs <= 0 || !rowptr || !cols || !vals || !vt || !F ||
      (n_dirs + 255) / 256 > 65535)
    return fail(SSS_EINVAL, "bad fold_spmm arguments");
  dim3 grid((n_rows + sss::kSpmmWarps - 1) / sss::kSpmmWarps, (n_dirs + 255) / 256);
  sss::k_fold_spmm<<<grid, 32 * sss::kSpmmWarps, 0, S_(stream)>>>(n_rows, n_dirs, rowptr, cols,
                                                                 vals, vt, F);
  return check_launch("k_fold_spmm");
}

int sss_fold_select(const double* FT, int n_rows, int n_dirs, double fraction,
                    const uint32_t* tm2flat, uint64_t* col_t, uint32_t* col_fmax,
                    uint32_t* col_cnt, double* col_energy, uint32_t* col_nz, void* stream) {
  if (!FT || !tm2flat || !col_t || !col_fmax || !col_cnt || !col_energy || n_rows <= 0 ||
      n_dirs <= 0 || !(fraction >= 0.0 && fraction <= 1.0))
    return fail(SSS_EINVAL, "bad fold_select arguments");
  const size_t smem = sizeof(sss::SelShared) + (size_t)((n_rows + 31) / 32) * 4;
  if (int r = set_smem((const void*)sss::k_step2_select, smem)) return r;
  sss::k_step2_select<<<n_dirs, sss::kSelThreads, smem, S_(stream)>>>(
      FT, n_rows, fraction, nullptr, tm2flat, nullptr, col_t, col_fmax, col_cnt, col_energy,
      col_nz);
  return check_launch("k_step2_select");
}

int sss_fold_emit(const double* FT, int n_rows, int n_dirs, const uint32_t* flat2tm,
                  const uint64_t* col_t, const uint32_t* col_fmax, const uint32_t* col_cnt,
                  const uint64_t* colptr, uint32_t* rows, float* vals, void* stream) {
  if (!FT || !flat2tm || !col_t || !col_fmax || !col_cnt || !colptr || !rows || !vals ||
      n_rows <= 0 || n_dirs <= 0)
    return fail(SSS_EINVAL, "bad fold_emit arguments");
  sss::k_fold_emit<<<n_dirs, sss::kEmitThreads, 0, S_(stream)>>>(FT, n_rows, flat2tm, col_t,
                                                                 col_fmax, col_cnt, colptr, rows,
                                                                 vals);
  return check_launch("k_fold_emit");
}

int sss_fold_apply(int K, int n_rows, int n_dirs, const uint64_t* colptr, const uint32_t* rows,
                   const float* vals, const uint32_t* union_idx, const double* union_lc,
                   const int* n_union, const uint32_t* flat2tm, double* vk, void* stream) {
  if (K <= 0 || n_rows <= 0 || n_dirs <= 0 || !colptr || !rows || !vals || !union_idx ||
      !union_lc || !n_union || !flat2tm || !vk)
    return fail(SSS_EINVAL, "bad fold_apply arguments");
  dim3 grid((n_rows + sss::kFoldRows - 1) / sss::kFoldRows, K);
  sss::k_fold_apply<<<grid, 256, 0, S_(stream)>>>(n_rows, n_dirs, colptr, rows, vals, union_idx,
                                                  union_lc, n_union, flat2tm, vk);
  return check_launch("k_fold_apply");
}

int sss_transfer_flat8c(int K, int n_rows, const void* cols16, const float* vals,
                        unsigned long long n_entries, const uint32_t* heads,
                        const uint32_t* head_prefix, const uint32_t* seg_rowk,
                        const unsigned* warp_begin, const int* cta_part, int n_ctas,
                        int part_width, const void* xp, const uint32_t* bits, double* vk,
                        void* stream) {
  if (K <= 0 || K > 16 || n_rows <= 0 || !cols16 || !vals || !heads || !head_prefix ||
      !seg_rowk || !warp_begin || !cta_part || !xp || !bits || !vk || n_ctas <= 0 ||
      n_entries % 256 || n_entries / 8 >= (1ull << 32) - 64)
    return fail(SSS_EINVAL, "bad transfer_flat8c arguments");
  if (reinterpret_cast<uintptr_t>(cols16) % 16 || reinterpret_cast<uintptr_t>(vals) % 32 ||
      reinterpret_cast<uintptr_t>(xp) % 32)
    return fail(SSS_EINVAL, "transfer_flat8c: cols16 16-B, vals / xp 32-B aligned");
  cudaError_t e = cudaMemsetAsync(vk, 0, (size_t)K * 3 * n_rows * sizeof(double), S_(stream));
  if (e != cudaSuccess) return fail(SSS_ECUDA, cudaGetErrorString(e));
  const auto* c16 = reinterpret_cast<const uint4*>(cols16);
  const auto* v8 = reinterpret_cast<const unsigned long long*>(vals);
  const auto* x4 = reinterpret_cast<const double4*>(xp);
#define SSS_V22(CWV)                                                                             \
  case CWV: {                                                                                    \
    const size_t smem = (size_t)3 * CWV * 8 + CWV / 8;                                           \
    if (int r = set_smem((const void*)sss::k_transfer_flat8c<CWV>, smem)) return r;             \
    sss::k_transfer_flat8c<CWV><<<n_ctas, sss::kV22Threads, smem, S_(stream)>>>(                 \
        n_rows, c16, v8, heads, head_prefix, seg_rowk, warp_begin, cta_part, x4, bits, vk);      \
    break;                                                                                       \
  }
  switch (part_width) {
    SSS_V22(1024) SSS_V22(2048) SSS_V22(4096)
    default:
      return fail(SSS_EINVAL, "transfer_flat8c: part_width must be 1024, 2048 or 4096");
  }
#undef SSS_V22
  return check_launch("k_transfer_flat8c");
}

int sss_transfer_flat16(int K, int n_rows, const void* pcols, const float* pvals,
                        unsigned long long n_entries, const uint32_t* heads,
                        const uint32_t* head_prefix, const uint32_t* seg_rowk,
                        const unsigned* warp_begin, int n_warps, int min_blocks,
                        int entries_per_lane, int col_bits, int zero_vk, const void* xp,
                        const uint32_t* bits, double* vk, uint32_t* work_counter, int chunk,
                        void* stream) {
  const int E = entries_per_lane;
  if ((col_bits != 16 && col_bits != 32) || (col_bits == 16 && (n_rows > 65536 || E != 16)))
    return fail(SSS_EINVAL, "transfer_flat16: col_bits 32, or 16 with n_rows <= 65536 and E 16");
  if (K <= 0 || K > 16 || n_rows <= 0 || !pcols || !pvals || !heads || !head_prefix ||
      !seg_rowk || !warp_begin || !xp || !bits || !vk || n_warps <= 0 || (E != 16 && E != 32) ||
      n_warps % (sss::kV25Threads / 32) || n_entries % E || n_entries / E >= (1ull << 32) - 64)
    return fail(SSS_EINVAL, "bad transfer_flat16 arguments");
  if (reinterpret_cast<uintptr_t>(pcols) % 32 || reinterpret_cast<uintptr_t>(pvals) % 32 ||
      reinterpret_cast<uintptr_t>(xp) % 32)
    return fail(SSS_EINVAL, "transfer_flat16: pcols/pvals/xp must be 32-byte aligned");
  if (zero_vk) {
    cudaError_t e = cudaMemsetAsync(vk, 0, (size_t)K * 3 * n_rows * sizeof(double), S_(stream));
    if (e == cudaSuccess && work_counter)
      e = cudaMemsetAsync(work_counter, 0, sizeof(uint32_t), S_(stream));
    if (e != cudaSuccess) return fail(SSS_ECUDA, cudaGetErrorString(e));
  }
  if (chunk < 1) chunk = 1;
  const size_t smem = (size_t)((n_rows >> 5) + 1) * 4;
  const auto* c16 = reinterpret_cast<const unsigned long long*>(pcols);
  const auto* v16 = reinterpret_cast<const unsigned long long*>(pvals);
  const auto* x4 = reinterpret_cast<const double4*>(xp);
  const unsigned grid = n_warps / (sss::kV25Threads / 32);
  const unsigned ng = (unsigned)(n_entries / E);
#define SSS_V25(MB, EE)                                                                          \
  if (min_blocks == MB && E == EE) {                                                             \
    if (int r = set_smem((const void*)sss::k_transfer_flat16<MB, EE>, smem)) return r;           \
    sss::k_transfer_flat16<MB, EE><<<grid, sss::kV25Threads, smem, S_(stream)>>>(                \
        n_rows, ng, c16, v16, heads, head_prefix, seg_rowk, warp_begin, x4, bits, vk,            \
        work_counter, chunk);                                                                    \
    return check_launch("k_transfer_flat16");                                                    \
  }
  if (col_bits == 16) {
    if (min_blocks != 8) return fail(SSS_EINVAL, "transfer_flat16: 16-bit columns use min_blocks 8");
    if (int r = set_smem((const void*)sss::k_transfer_flat16<8, 16, true>, smem)) return r;
    sss::k_transfer_flat16<8, 16, true><<<grid, sss::kV25Threads, smem, S_(stream)>>>(
        n_rows, ng, c16, v16, heads, head_prefix, seg_rowk, warp_begin, x4, bits, vk,
        work_counter, chunk);
    return check_launch("k_transfer_flat16");
  }
  SSS_V25(4, 16) SSS_V25(6, 16) SSS_V25(8, 16) SSS_V25(8, 32) SSS_V25(6, 32)
#undef SSS_V25
  return fail(SSS_EINVAL, "transfer_flat16: (min_blocks, entries_per_lane) in {4,6,8}x16, {6,8}x32");
}

int sss_flat_align(unsigned n_words, unsigned n_groups, const uint32_t* cols_in, const float* vals_in,
                   const uint32_t* heads, uint32_t sentinel, uint32_t* cols_out, float* vals_out,
                   void* stream) {
  if (!cols_in || !vals_in || !heads || !cols_out || !vals_out || cols_in == cols_out ||
      vals_in == vals_out)
    return fail(SSS_EINVAL, "bad flat_align arguments");
  if (n_words == 0) return SSS_OK;
  if (n_groups > 32ull * n_words || n_groups + 32 <= 32ull * n_words)
    return fail(SSS_EINVAL, "flat_align: n_groups must cover the last word");
  sss::k_flat_align<<<(n_words + 63) / 64, 64, 0, S_(stream)>>>(n_words, n_groups, cols_in, vals_in,
                                                                heads, sentinel, cols_out, vals_out);
  return check_launch("k_flat_align");
}

int sss_transfer_rbcsc(int K, int n_rows, int row_block, const void* desc,
                       const uint32_t* desc_ptr, const uint16_t* rowk, const float* vals,
                       const double* rowabs, const double* energy, const void* xp,
                       const uint32_t* bits, double* vk, void* stream) {
  if (K <= 0 || K > 8 || n_rows <= 0 || n_rows > 65536 || !desc || !desc_ptr || !rowk ||
      !vals || !rowabs || !energy || !xp || !bits || !vk || n_rows % row_block)
    return fail(SSS_EINVAL, "bad transfer_rbcsc arguments");
  if (reinterpret_cast<uintptr_t>(xp) % 32 || reinterpret_cast<uintptr_t>(desc) % 8)
    return fail(SSS_EINVAL, "transfer_rbcsc: xp 32-B, desc 8-B aligned");
  const unsigned grid = n_rows / row_block;
  const auto* d2 = reinterpret_cast<const uint2*>(desc);
  const auto* x4 = reinterpret_cast<const double4*>(xp);
#define SSS_V24(RBV, KK)                                                                         \
  if (row_block == RBV && K == KK) {                                                             \
    sss::k_transfer_rbcsc<RBV, KK><<<grid, sss::kV24Threads, 0, S_(stream)>>>(                   \
        n_rows, d2, desc_ptr, rowk, vals, rowabs, energy, x4, bits, vk);                         \
    return check_launch("k_transfer_rbcsc");                                                     \
  }
  SSS_V24(64, 8) SSS_V24(128, 8) SSS_V24(32, 8)
  SSS_V24(64, 4) SSS_V24(128, 4) SSS_V24(32, 4)
  SSS_V24(64, 1) SSS_V24(64, 2) SSS_V24(64, 3) SSS_V24(64, 5) SSS_V24(64, 6) SSS_V24(64, 7)
#undef SSS_V24
  return fail(SSS_EINVAL, "transfer_rbcsc: row_block in {32, 64, 128} for K in {4, 8}, 64 for "
                          "K <= 8");
}

int sss_transfer_pairgroup(int K, int n_rows, const uint32_t* pair_ptr, const uint32_t* val_ptr,
                           const uint32_t* hdr, const float* vals, const uint32_t* row_begin,
                           int n_warps, const void* xp, const uint32_t* bits, double* vk,
                           void* stream) {
  if (K <= 0 || K > 8 || n_rows <= 0 || n_rows > 65536 || !pair_ptr || !val_ptr || !hdr ||
      !vals || !row_begin || !xp || !bits || !vk || n_warps <= 0 ||
      n_warps % (sss::kV23Threads / 32))
    return fail(SSS_EINVAL, "bad transfer_pairgroup arguments");
  if (reinterpret_cast<uintptr_t>(xp) % 32) return fail(SSS_EINVAL, "xp must be 32-byte aligned");
  const size_t smem = (size_t)((n_rows + 31) / 32) * 4;
  const unsigned grid = n_warps / (sss::kV23Threads / 32);
  const auto* x4 = reinterpret_cast<const double4*>(xp);
#define SSS_V23(KK)                                                                              \
  case KK:                                                                                       \
    if (int r = set_smem((const void*)sss::k_transfer_pairgroup<KK>, smem)) return r;            \
    sss::k_transfer_pairgroup<KK><<<grid, sss::kV23Threads, smem, S_(stream)>>>(                 \
        n_rows, pair_ptr, val_ptr, hdr, vals, row_begin, x4, bits, vk);                          \
    break;
  switch (K) {
    SSS_V23(1) SSS_V23(2) SSS_V23(3) SSS_V23(4) SSS_V23(5) SSS_V23(6) SSS_V23(7) SSS_V23(8)
  }
#undef SSS_V23
  return check_launch("k_transfer_pairgroup");
}

int sss_transfer_kpairs(int K, int n_rows, const void* chunks, const uint32_t* hdr,
                        const float* vals, const uint32_t* chunk_begin, int n_warps,
                        const void* xp, const uint32_t* bits, double* vk, void* stream) {
  if (K <= 0 || K > 8 || n_rows <= 0 || n_rows > 65536 || !chunks || !hdr || !vals ||
      !chunk_begin || !xp || !bits || !vk || n_warps <= 0 || n_warps % (sss::kV21Threads / 32))
    return fail(SSS_EINVAL, "bad transfer_kpairs arguments");
  if (reinterpret_cast<uintptr_t>(chunks) % 16 || reinterpret_cast<uintptr_t>(xp) % 32)
    return fail(SSS_EINVAL, "transfer_kpairs: chunks must be 16-byte and xp 32-byte aligned");
  const size_t smem = (size_t)((n_rows + 31) / 32) * 4;
  const unsigned grid = n_warps / (sss::kV21Threads / 32);
  const auto* c4 = reinterpret_cast<const uint4*>(chunks);
  const auto* x4 = reinterpret_cast<const double4*>(xp);
#define SSS_V21(KK)                                                                              \
  case KK:                                                                                       \
    if (int r = set_smem((const void*)sss::k_transfer_kpairs<KK>, smem)) return r;               \
    sss::k_transfer_kpairs<KK><<<grid, sss::kV21Threads, smem, S_(stream)>>>(                    \
        n_rows, c4, hdr, vals, chunk_begin, x4, bits, vk);                                       \
    break;
  switch (K) {
    SSS_V21(1) SSS_V21(2) SSS_V21(3) SSS_V21(4) SSS_V21(5) SSS_V21(6) SSS_V21(7) SSS_V21(8)
  }
#undef SSS_V21
  return check_launch("k_transfer_kpairs");
}

int sss_fold_apply_rows(int K, int n_rows, int n_dirs, const uint64_t* gbase,
                        const uint32_t* entries, const uint32_t* union_idx,
                        const double* union_lc, const int* n_union, const uint32_t* flat2tm,
                        double* vk, void* stream) {
  if (n_rows % 32) return fail(SSS_EINVAL, "fold_apply_rows: n_rows must be a multiple of 32");
  if (K <= 0 || n_rows <= 0 || n_dirs <= 0 || !gbase || !entries || !union_idx ||
      !union_lc || !n_union || !flat2tm || !vk)
    return fail(SSS_EINVAL, "bad fold_apply_rows arguments");
  const size_t smem = (size_t)24 * n_dirs;
  if (smem > 200 * 1024) return fail(SSS_EINVAL, "fold_apply_rows: too many directions (use sss_fold_apply)");
  if (int r = set_smem((const void*)sss::k_fold_apply_rows, smem)) return r;
  dim3 grid((n_rows + 255) / 256, K);
  sss::k_fold_apply_rows<<<grid, 256, smem, S_(stream)>>>(n_rows, n_dirs, gbase,
                                                          reinterpret_cast<const uint2*>(entries),
                                                          union_idx, union_lc, n_union, flat2tm, vk);
  return check_launch("k_fold_apply_rows");
}

int sss_band_offsets(const uint64_t* rowptr, const uint32_t* cols, int K, int n_rows,
                     int band_width, int n_bands, uint32_t* bandoff, void* stream) {
  if (!rowptr || !bandoff || K <= 0 || n_rows <= 0 || band_width <= 0 || n_bands <= 0)
    return fail(SSS_EINVAL, "bad band_offsets arguments");
  const long long n = (long long)K * n_rows;
  sss::k_band_offsets<<<(unsigned)((n + 255) / 256), 256, 0, S_(stream)>>>(rowptr, cols, K, n_rows,
                                                                          band_width, n_bands, bandoff);
  return check_launch("k_band_offsets");
}

int sss_edit_finish(int K, int side, int levels, const double* vk, const double* g,
                    const float* positions, const float* normals, const double* cam,
                    const double* material, double* scatter, float* radiance,
                    float* radiance_unclamped, void* stream) {
  if (int r = check_geom(side, levels)) return r;
  if (K <= 0 || !vk || !g || !positions || !normals || !cam || !material || !radiance ||
      !radiance_unclamped)
    return fail(SSS_EINVAL, "bad edit_finish arguments");
  const int T = 1 << levels, T2 = T * T, tiles = (side / T) * (side / T);
  // tiles per CTA: one (1024 CTAs of 64 threads at C3) measured fastest
  // (13.9 vs 15.9 us for four); SSS_EDIT_G overrides for A/B
  const char* g_env = getenv("SSS_EDIT_G");
  int G = g_env ? atoi(g_env) : 1;
  if (G < 1 || G * T2 > 256) G = 1;
  while (G > 1 && tiles % G) G >>= 1;
  if (T2 <= 256) {
    const size_t smem = 6 * (size_t)G * T2 * sizeof(double);
    if (int r = set_smem((const void*)sss::k_edit_finish_multi, smem)) return r;
    sss::k_edit_finish_multi<<<tiles / G, G * T2 < 64 ? 64 : G * T2, smem, S_(stream)>>>(
        K, side, levels, G, vk, g, positions, normals, cam, material, scatter, radiance,
        radiance_unclamped);
    return check_launch("k_edit_finish_multi");
  }
  const size_t smem = 4 * (size_t)T * T * sizeof(double);
  if (int r = set_smem((const void*)sss::k_edit_finish, smem)) return r;
  sss::k_edit_finish<<<tiles, 128, smem, S_(stream)>>>(
      K, side, levels, vk, g, positions, normals, cam, material, scatter, radiance,
      radiance_unclamped);
  return check_launch("k_edit_finish");
}

// ---------------------------------------------------------------------------
// precompute (path d)
// ---------------------------------------------------------------------------

int sss_pair_block(int levels, int exact, int side, const float* pos, const float* area,
                   const double* r_nodes, const double* bases, const double* slopes, int nr, int k,
                   const float* Pkm, const float* mat, int n_mat, float r_max, double* D,
                   double* Mout, void* stream) {
  if (int r = check_geom(side, levels)) return r;
  if (levels > 3) return fail(SSS_EINVAL, "pair pass supports levels <= 3");
  if (!pos || !area || (!D && !Mout)) return fail(SSS_EINVAL, "bad pair_block pointers");
  if (!exact && (!r_nodes || !bases || !slopes || nr < 2))
    return fail(SSS_EINVAL, "lerp mode needs r_nodes / bases / slopes");
  if (exact && (!Pkm || !mat || n_mat <= 0)) return fail(SSS_EINVAL, "exact mode needs Pkm / mat");
  sss::PairParams p{pos, area, r_nodes, bases, slopes, nr, k, side, Pkm, mat, n_mat, r_max};
  const int T = 1 << levels, T2 = T * T;
  const int tiles = (side / T) * (side / T);
  dim3 grid(tiles, tiles);
  const size_t smem = ((size_t)T2 * (T2 + 1) + (exact ? 0 : 3 * (size_t)nr)) * sizeof(double) +
                      (exact ? (size_t)n_mat * 5 * sizeof(float) : 0);
  const void* fn = nullptr;
#define SSS_PAIR_CASE(LV)                                                                     \
  case LV:                                                                                    \
    fn = exact ? (const void*)sss::k_pair_block<LV, true> : (const void*)sss::k_pair_block<LV, false>; \
    if (int r = set_smem(fn, smem)) return r;                                                 \
    if (exact) sss::k_pair_block<LV, true><<<grid, 128, smem, S_(stream)>>>(p, D, Mout);      \
    else sss::k_pair_block<LV, false><<<grid, 128, smem, S_(stream)>>>(p, D, Mout);           \
    break;
  switch (levels) {
    SSS_PAIR_CASE(1)
    SSS_PAIR_CASE(2)
    SSS_PAIR_CASE(3)
    default: return fail(SSS_EINVAL, "levels");
  }
#undef SSS_PAIR_CASE
  return check_launch("k_pair_block");
}

int sss_step1_select(const double* D, int n_dom, int n_rows, int n_keep, const uint32_t* tm2flat,
                     uint32_t* union_bits, void* stream) {
  if (!D || !tm2flat || !union_bits || n_dom <= 0 || n_rows < 0 || n_keep < 1)
    return fail(SSS_EINVAL, "bad step1 arguments");
  if (n_rows == 0) return SSS_OK;
  const size_t smem = sizeof(sss::SelShared) + 2 * (size_t)((n_dom + 31) / 32) * 4;
  if (int r = set_smem((const void*)sss::k_step1_select, smem)) return r;
  sss::k_step1_select<<<n_rows, sss::kSelThreads, smem, S_(stream)>>>(D, n_dom, n_keep, tm2flat,
                                                                      union_bits);
  return check_launch("k_step1_select");
}

int sss_step2_select(const double* M, int n_dom, double fraction, const uint32_t* flat2tm,
                     const uint32_t* tm2flat, const uint32_t* union_bits, uint64_t* col_t,
                     uint32_t* col_fmax, uint32_t* col_cnt, double* col_energy, void* stream) {
  if (!M || !flat2tm || !tm2flat || !union_bits || !col_t || !col_fmax || !col_cnt || !col_energy ||
      n_dom <= 0 || !(fraction >= 0.0 && fraction <= 1.0))
    return fail(SSS_EINVAL, "bad step2 arguments");
  const size_t smem = sizeof(sss::SelShared) + (size_t)((n_dom + 31) / 32) * 4;
  if (int r = set_smem((const void*)sss::k_step2_select, smem)) return r;
  sss::k_step2_select<<<n_dom, sss::kSelThreads, smem, S_(stream)>>>(
      M, n_dom, fraction, flat2tm, tm2flat, union_bits, col_t, col_fmax, col_cnt, col_energy,
      nullptr);
  return check_launch("k_step2_select");
}

int sss_emit(int pass, const double* M, int n_dom, int tile_rows, int chunk, const uint64_t* col_t,
             const uint32_t* col_fmax, const uint32_t* tm2flat, uint32_t* counts,
             const uint64_t* offs, uint32_t* cols, float* vals, void* stream) {
  if (!M || !col_t || !col_fmax || !tm2flat || tile_rows <= 0 || tile_rows > 1024 || chunk <= 0 ||
      n_dom % tile_rows)
    return fail(SSS_EINVAL, "bad emit arguments");
  dim3 grid((n_dom + chunk - 1) / chunk, n_dom / tile_rows);
  const int thr = ((tile_rows + 31) / 32) * 32;
  if (pass == 0) {
    if (!counts) return fail(SSS_EINVAL, "emit count needs counts");
    sss::k_emit_count<<<grid, thr, 0, S_(stream)>>>(M, n_dom, tile_rows, chunk, col_t, col_fmax,
                                                   tm2flat, counts);
    return check_launch("k_emit_count");
  }
  if (!offs || !cols || !vals) return fail(SSS_EINVAL, "emit write needs offs / cols / vals");
  sss::k_emit_write<<<grid, thr, 0, S_(stream)>>>(M, n_dom, tile_rows, chunk, col_t, col_fmax,
                                                 tm2flat, offs, 0, cols, vals);
  return check_launch("k_emit_write");
}

int sss_scan_u32(const uint32_t* in, uint64_t* out, size_t n, uint64_t* block_sums,
                 uint64_t* total, void* stream) {
  if (!in || !out || !block_sums || !total) return fail(SSS_EINVAL, "bad scan arguments");
  const int nb = (int)((n + 1023) / 1024);
  if (nb == 0) return cudaMemsetAsync(total, 0, 8, S_(stream)) == cudaSuccess ? SSS_OK : SSS_ECUDA;
  sss::k_scan_blocks<<<nb, 1024, 0, S_(stream)>>>(in, out, n, block_sums);
  sss::k_scan_sums<<<1, 1, 0, S_(stream)>>>(block_sums, nb, total);
  sss::k_scan_add<<<nb, 1024, 0, S_(stream)>>>(out, n, block_sums);
  return check_launch("k_scan");
}

int sss_rowptr(const uint64_t* offs, int nchunks, int n_rows, uint64_t base, const uint64_t* total,
               uint64_t* rowptr, void* stream) {
  if (!offs || !total || !rowptr || nchunks <= 0 || n_rows <= 0)
    return fail(SSS_EINVAL, "bad rowptr arguments");
  sss::k_rowptr<<<(n_rows + 1 + 255) / 256, 256, 0, S_(stream)>>>(offs, nchunks, n_rows, base,
                                                                   total, rowptr);
  return check_launch("k_rowptr");
}

int sss_raster_fill(const int64_t* tris, int n_tris, const double* sx, const double* sy,
                    const double* zn, const double* iw, const double* colors, int height,
                    int width, double* zbuf, double* img, unsigned long long* key,
                    uint32_t* win, double exposure, uint8_t* srgb8, void* stream) {
  if (height < 1 || width < 1) return fail(SSS_EINVAL, "image dimensions must be positive");
  if ((long long)height * width > (1ll << 31) - 1) return fail(SSS_EINVAL, "image too large");
  if (n_tris < 0 || (n_tris > 0 && (!tris || !sx || !sy || !zn || !iw || !colors)) || !zbuf ||
      !img || !key || !win)
    return fail(SSS_EINVAL, "bad raster_fill arguments");
  const int n_pix = height * width;
  cudaStream_t s = S_(stream);
  sss::k_raster_init<<<(n_pix + 255) / 256, 256, 0, s>>>(zbuf, n_pix, key, win);
  if (n_tris > 0) {
    const int g = (n_tris + 255) / 256;
    sss::k_raster_tri<false><<<g, 256, 0, s>>>(tris, n_tris, sx, sy, zn, iw, zbuf, height, width,
                                               key, win);
    sss::k_raster_tri<true><<<g, 256, 0, s>>>(tris, n_tris, sx, sy, zn, iw, zbuf, height, width,
                                              key, win);
  }
  sss::k_raster_resolve<<<(n_pix + 255) / 256, 256, 0, s>>>(tris, sx, sy, zn, iw, colors, height,
                                                           width, win, zbuf, img, exposure, srgb8);
  return check_launch("k_raster");
}

int sss_raster_clear(int height, int width, double b0, double b1, double b2, double* zbuf,
                     double* img, void* stream) {
  if (height < 1 || width < 1 || !zbuf || !img) return fail(SSS_EINVAL, "bad raster_clear arguments");
  const int n_pix = height * width;
  sss::k_raster_clear<<<(n_pix + 255) / 256, 256, 0, S_(stream)>>>(n_pix, b0, b1, b2, zbuf, img);
  return check_launch("k_raster_clear");
}

int sss_project_vertices(const double* vertices, int n_vertices, const double* cam, double f,
                         double aspect, int width, int height, double* sx, double* sy,
                         double* zn, double* iw, void* stream) {
  if (n_vertices < 0 || width < 1 || height < 1 ||
      (n_vertices > 0 && (!vertices || !cam || !sx || !sy || !zn || !iw)))
    return fail(SSS_EINVAL, "bad project_vertices arguments");
  if (n_vertices == 0) return SSS_OK;
  sss::k_raster_project<<<(n_vertices + 255) / 256, 256, 0, S_(stream)>>>(
      vertices, n_vertices, cam, f, aspect, width, height, sx, sy, zn, iw);
  return check_launch("k_raster_project");
}

int sss_vertex_colors(const float* radiance, const int32_t* source_vertex, int n, double* colors,
                      void* stream) {
  if (n < 0 || (n > 0 && (!radiance || !colors))) return fail(SSS_EINVAL, "bad vertex_colors arguments");
  if (n == 0) return SSS_OK;
  sss::k_vertex_colors<<<(n + 255) / 256, 256, 0, S_(stream)>>>(radiance, source_vertex, n, colors);
  return check_launch("k_vertex_colors");
}

int sss_zero(void* ptr, unsigned long long bytes, void* stream) {
  if (!ptr && bytes) return fail(SSS_EINVAL, "bad zero arguments");
  cudaError_t e = cudaMemsetAsync(ptr, 0, bytes, S_(stream));
  if (e != cudaSuccess) return fail(SSS_ECUDA, cudaGetErrorString(e));
  return SSS_OK;
}

int sss_widen_frame(const float* radiance, const float* radiance_unclamped, long long n,
                    double* out, void* stream) {
  if (n < 0 || (n > 0 && (!radiance || !radiance_unclamped || !out)))
    return fail(SSS_EINVAL, "bad widen_frame arguments");
  if (n == 0) return SSS_OK;
  sss::k_widen_frame<<<(unsigned)((n + 255) / 256), 256, 0, S_(stream)>>>(radiance,
                                                                         radiance_unclamped, n, out);
  return check_launch("k_widen_frame");
}

int sss_encode_srgb8(const double* x, long long n, double exposure, uint8_t* out, void* stream) {
  if (n < 0 || (n > 0 && (!x || !out))) return fail(SSS_EINVAL, "bad encode_srgb8 arguments");
  if (n == 0) return SSS_OK;
  sss::k_encode_srgb8<<<(unsigned)((n + 255) / 256), 256, 0, S_(stream)>>>(x, n, exposure, out);
  return check_launch("k_encode_srgb8");
}

}  // extern "C"
