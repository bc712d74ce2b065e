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
#include "transfer.cu"
#include "flat16_25.cu"
#include "select_cluster.cu"
#include "sweep.cu"
#include "direct.cu"
#include "fold.cu"
#include "raster.cu"
#include "seam.cu"

#include "abi_util.cuh"

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

static int select_topn_impl(const double* v, int nvec, int n_dom, int n_keep, const uint32_t* f2t,
                            double* x_out, uint32_t* mask, double* energy, double* xp,
                            uint32_t* bits, void* stream) {
  if (nvec < 0 || nvec > 65535 || n_dom <= 0 || n_keep < 0 || !v || !x_out)
    return fail(SSS_EINVAL, "bad select arguments");
  if (nvec == 0) return SSS_OK;
  const int chunk = (((n_dom + sss::kSelCluster - 1) / sss::kSelCluster) + 31) / 32 * 32;
  if (chunk <= 16384 && n_dom >= 32 * sss::kSelCluster) {
    // one 16-CTA cluster per vector, slices resident in shared memory; the
    // kernel writes every mask word of its slices itself
    const size_t smem = ((sizeof(sss::ClusterSelShared) + 15) & ~size_t(15)) + chunk * sizeof(double);
    if (int r = set_smem((const void*)sss::k_select_cluster, smem)) return r;
    if (sss::kSelCluster > 8)
      cudaFuncSetAttribute((const void*)sss::k_select_cluster,
                           cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    launch_chain(sss::k_select_cluster, dim3(nvec * sss::kSelCluster), dim3(1024), smem, S_(stream), v,
                 n_dom, n_keep, chunk, f2t, x_out, mask, energy, xp, bits);
    return check_launch("k_select_cluster");
  }
  if (mask) {
    cudaError_t e = cudaMemsetAsync(mask, 0, (size_t)nvec * ((n_dom + 31) / 32) * 4, S_(stream));
    if (e != cudaSuccess) return fail(SSS_ECUDA, cudaGetErrorString(e));
  }
  const size_t smem = sizeof(sss::SelShared);
  if (int r = set_smem((const void*)sss::k_select_topn, smem)) return r;
  sss::k_select_topn<<<nvec, 1024, smem, S_(stream)>>>(v, n_dom, n_keep, f2t, x_out, mask, energy);
  if (int r = check_launch("k_select_topn")) return r;
  if (xp) {  // small domains: the block kernel, then the packing pass
    sss::k_pack_x_bits<<<(n_dom + 255) / 256, 256, 0, S_(stream)>>>(
        x_out, n_dom, reinterpret_cast<double4*>(xp), bits);
    return check_launch("k_pack_x_bits");
  }
  return SSS_OK;
}

int sss_select_topn(const double* v, int nvec, int n_dom, int n_keep, const uint32_t* f2t,
                    double* x_out, uint32_t* mask, double* energy, void* stream) {
  return select_topn_impl(v, nvec, n_dom, n_keep, f2t, x_out, mask, energy, nullptr, nullptr, stream);
}

int sss_select_topn_pack(const double* v, int n_dom, int n_keep, const uint32_t* f2t, double* x_out,
                         uint32_t* mask, double* energy, double* xp, uint32_t* bits, void* stream) {
  if (!xp || !bits) return fail(SSS_EINVAL, "bad select_pack arguments");
  return select_topn_impl(v, 3, n_dom, n_keep, f2t, x_out, mask, energy, xp, bits, stream);
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
  launch_chain(sss::k_env_project, dim3(3), dim3(1024), smem, S_(stream), faces, env_side, n_keep, idx,
               val, (double*)nullptr);
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
  while (tpb & (tpb - 1)) tpb &= tpb - 1;  // a power of two (the kernel's index math shifts)
  const size_t nk8 = ((size_t)n_keep + 7) & ~size_t(7);
  const size_t smem = 6 * (size_t)tpb * T2 * sizeof(double) + 3 * nk8 * (sizeof(double) + sizeof(uint32_t));
  const int threads = 3 * tpb * T2 > 768 ? 768 : 3 * tpb * T2;  // the kernel strides over (point, channel)
  if ((double)D * side * side >= 4294967296.0)
    return fail(SSS_EINVAL, "env_irradiance_sel: W^{w2} larger than 2^32 elements");
  if (int r = set_smem((const void*)sss::k_env_irradiance_chan, smem)) return r;
  launch_chain(sss::k_env_irradiance_chan, dim3(tiles / tpb), dim3(threads < 32 ? 32 : threads), smem,
               S_(stream), W2, sel_idx, sel_val, n_keep, D, side, levels, tpb, E_out, ehat);
  return check_launch("k_env_irradiance_chan");
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















int sss_pack_x_bits(const double* x, int n, void* xp, uint32_t* bits, void* stream) {
  if (!x || !xp || !bits || n <= 0) return fail(SSS_EINVAL, "bad pack_x_bits arguments");
  if (reinterpret_cast<uintptr_t>(xp) % 32) return fail(SSS_EINVAL, "xp must be 32-byte aligned");
  sss::k_pack_x_bits<<<(n + 255) / 256, 256, 0, S_(stream)>>>(x, n, reinterpret_cast<double4*>(xp),
                                                             bits);
  return check_launch("k_pack_x_bits");
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
    const void* fn = n_points == 65536 ? (const void*)sss::k_sweep_umma<TMN, THR, 65536>          \
                                       : (const void*)sss::k_sweep_umma<TMN, THR>;                 \
    if (int r = set_smem(fn, smem)) return r;                                                      \
    dim3 grid = g1;                                                                                \
    grid.z = (M + TMN - 1) / TMN;                                                                  \
    if (n_points == 65536)                                                                         \
      sss::k_sweep_umma<TMN, THR, 65536><<<grid, THR, smem, S_(stream)>>>(                         \
          n_points, M, reinterpret_cast<const __nv_bfloat16*>(Bq),                                 \
          reinterpret_cast<const __nv_bfloat16*>(Gq), eta, eta_lo, eta_hi, positions, normals,     \
          cam, out);                                                                               \
    else                                                                                           \
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



}  // extern "C"

namespace {
// positions / normals in PT (float: geometry images; double: the reference's
// SurfaceSamples, sss_direct_irradiance64)
template <typename PT>
int direct_irradiance(int n_points, const PT* positions, const PT* normals, int n_lights,
                      const int* kinds, const double* lights, const double* material,
                      double ray_offset, double bbox_diagonal, const double* nodes,
                      const double* tris, double* E, void* stream) {
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
  constexpr int S = 3;  // 8 threads share a ray (one subtree each)
  for (int l = 0; l < n_lights; ++l) {
    const double* L = lights + 12 * (size_t)l;
    if (kinds[l] < 2) {
      const int grid = (n_points + (sss::kDirectThreads >> S) - 1) / (sss::kDirectThreads >> S);
      if (kinds[l] == 0)
        sss::k_direct_single<0, S, PT><<<grid, sss::kDirectThreads, 0, st>>>(
            n_points, positions, normals, L, material, ray_offset, bbox_diagonal, B, E);
      else
        sss::k_direct_single<1, S, PT><<<grid, sss::kDirectThreads, 0, st>>>(
            n_points, positions, normals, L, material, ray_offset, bbox_diagonal, B, E);
    } else {
      sss::k_direct_sphere<PT><<<(n_points + sss::kSpherePts - 1) / sss::kSpherePts,
                                 64 * sss::kSpherePts, 0, st>>>(n_points, positions, normals, L,
                                                                material, ray_offset, B, E);
    }
    const int rc = check_launch("k_direct_light");
    if (rc) return rc;
  }
  return SSS_OK;
}
}  // namespace

extern "C" {

int sss_direct_irradiance(int n_points, const float* positions, const float* normals,
                          int n_lights, const int* kinds, const double* lights,
                          const double* material, double ray_offset, double bbox_diagonal,
                          const double* nodes, const double* tris, double* E, void* stream) {
  return direct_irradiance<float>(n_points, positions, normals, n_lights, kinds, lights, material,
                                  ray_offset, bbox_diagonal, nodes, tris, E, stream);
}

int sss_direct_irradiance64(int n_points, const double* positions, const double* normals,
                            int n_lights, const int* kinds, const double* lights,
                            const double* material, double ray_offset, double bbox_diagonal,
                            const double* nodes, const double* tris, double* E, void* stream) {
  return direct_irradiance<double>(n_points, positions, normals, n_lights, kinds, lights,
                                   material, ray_offset, bbox_diagonal, nodes, tris, E, stream);
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

// stage 2, K-fused rows (csrc/transfer.cu; layout built by layout.kfr_layout)
int sss_transfer_kfr(int K, int n_rows, unsigned n_items, unsigned n_partials, const void* items,
                     const uint32_t* lane_len, const uint32_t* lane_dst, const uint32_t* batch_off,
                     const void* stream_bytes, const void* xp, const uint32_t* bits,
                     double* vk, double* partials, const uint32_t* partial_row,
                     const void* multi_info, uint32_t* multi_count, uint32_t* work,
                     int steps_per_batch, int n_warps, int min_blocks, void* stream) {
  if ((steps_per_batch != 4 && steps_per_batch != 8) || K <= 0 || K > 4 * sss::kKfrG || n_rows <= 0 || n_rows > 65536 || !items || !lane_len ||
      !lane_dst || !batch_off || !stream_bytes || !xp || !bits || !vk || !work || n_warps <= 0 ||
      n_warps % sss::kKfrWarps)
    return fail(SSS_EINVAL, "bad transfer_kfr arguments");
  if (n_partials && (!partials || !partial_row || !multi_info || !multi_count))
    return fail(SSS_EINVAL, "transfer_kfr: partial buffers required");
  if (reinterpret_cast<uintptr_t>(stream_bytes) % 16 || reinterpret_cast<uintptr_t>(xp) % 32)
    return fail(SSS_EINVAL, "transfer_kfr: stream 16- and xp 32-byte aligned");
  if (n_items == 0) return SSS_OK;
  const int ns = 2;  // ring slots per warp (3 measured slower: less L1 for the x gathers)
  unsigned grid = (unsigned)(n_warps / sss::kKfrWarps);
  const unsigned need = (n_items + sss::kKfrWarps - 1) / sss::kKfrWarps;
  if (grid > need) grid = need;
#define SSS_KFR(UU, NS, MB)                                                                      \
  if (steps_per_batch == UU && ns == NS && min_blocks == MB) {                                   \
    const size_t smem = sss::kfr_smem_bytes(n_rows, sss::KfrSmem<UU, NS>::WARP);                 \
    auto fn = sss::k_transfer_kfr<UU, NS, MB>;                                                   \
    /* the static bitmap counts against the default 48 KB: always raise */                     \
    if (cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize,       \
                             (int)smem) != cudaSuccess)                                          \
      return fail(SSS_ECUDA, "transfer_kfr: shared memory attribute");                          \
    launch_chain(fn, dim3(grid), dim3(sss::kKfrWarps * 32), smem, S_(stream), n_rows, K, n_items,   \
                 n_partials, reinterpret_cast<const uint2*>(items), lane_len, lane_dst, batch_off, \
                 reinterpret_cast<const unsigned char*>(stream_bytes),                           \
                 reinterpret_cast<const double4*>(xp), bits, vk, partials, partial_row,          \
                 reinterpret_cast<const uint4*>(multi_info), multi_count, work);                 \
    return check_launch("k_transfer_kfr");                                                       \
  }
  SSS_KFR(4, 2, 3) SSS_KFR(8, 2, 2)
#undef SSS_KFR
  return fail(SSS_EINVAL, "transfer_kfr: (steps_per_batch, min_blocks) in {(4, 3), (8, 2)}");
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


int sss_transfer_flat16(int K, int n_rows, const void* pcols, const float* pvals,
                        unsigned long long n_entries, const uint32_t* heads,
                        const uint32_t* head_prefix, const uint32_t* seg_rowk,
                        const unsigned* warp_begin, int n_warps, int min_blocks,
                        int entries_per_lane, int col_bits, int zero_vk, const void* xp,
                        const uint32_t* bits, double* vk, uint32_t* work_counter, int chunk,
                        double* word_partials, const uint32_t* span_first, void* stream) {
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
  // word_partials (2 x 3 doubles per word of 32 lanes): the deterministic form,
  // plain stores + k_flat16_merge instead of fp64 atomics
  const unsigned nwords = (ng + 31u) / 32u;
  auto merge = [&]() -> int {
    if (!word_partials) return SSS_OK;
    if (!span_first) return fail(SSS_EINVAL, "transfer_flat16: word_partials needs span_first");
    launch_chain(sss::k_flat16_merge, dim3((nwords + 127u) / 128u), dim3(128), 0, S_(stream), n_rows,
                 nwords, heads, head_prefix, seg_rowk, span_first, (const double*)word_partials, vk);
    return check_launch("k_flat16_merge");
  };
#define SSS_V25(MB, EE)                                                                          \
  if (min_blocks == MB && E == EE) {                                                             \
    if (int r = set_smem((const void*)sss::k_transfer_flat16<MB, EE>, smem)) return r;           \
    sss::k_transfer_flat16<MB, EE><<<grid, sss::kV25Threads, smem, S_(stream)>>>(                \
        n_rows, ng, c16, v16, heads, head_prefix, seg_rowk, warp_begin, x4, bits, vk,            \
        work_counter, chunk, word_partials);                                                     \
    if (int r = check_launch("k_transfer_flat16")) return r;                                     \
    return merge();                                                                              \
  }
  if (col_bits == 16) {
    if (min_blocks != 8) return fail(SSS_EINVAL, "transfer_flat16: 16-bit columns use min_blocks 8");
    if (int r = set_smem((const void*)sss::k_transfer_flat16<8, 16, true>, smem)) return r;
    sss::k_transfer_flat16<8, 16, true><<<grid, sss::kV25Threads, smem, S_(stream)>>>(
        n_rows, ng, c16, v16, heads, head_prefix, seg_rowk, warp_begin, x4, bits, vk,
        work_counter, chunk, word_partials);
    if (int r = check_launch("k_transfer_flat16")) return r;
    return merge();
  }
  SSS_V25(4, 16) SSS_V25(6, 16) SSS_V25(8, 16) SSS_V25(8, 32) SSS_V25(6, 32)
#undef SSS_V25
  return fail(SSS_EINVAL, "transfer_flat16: (min_blocks, entries_per_lane) in {4,6,8}x16, {6,8}x32");
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


int sss_edit_finish(int K, int side, int levels, const double* vk, const double* g,
                    const float* positions, const float* normals, const double* cam,
                    const double* material, double* scatter, float* radiance,
                    float* radiance_unclamped, void* stream) {
  return sss_edit_finish_wide(K, side, levels, vk, g, positions, normals, cam, material, scatter,
                              radiance, radiance_unclamped, nullptr, stream);
}

int sss_edit_finish_wide(int K, int side, int levels, const double* vk, const double* g,
                         const float* positions, const float* normals, const double* cam,
                         const double* material, double* scatter, float* radiance,
                         float* radiance_unclamped, double* rad64, void* stream) {
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
    launch_chain(sss::k_edit_finish_multi, dim3(tiles / G), dim3(G * T2 < 64 ? 64 : G * T2), smem,
                 S_(stream), K, side, levels, G, vk, g, positions, normals, cam, material, scatter,
                 radiance, radiance_unclamped, rad64);
    return check_launch("k_edit_finish_multi");
  }
  if (rad64) return fail(SSS_EINVAL, "edit_finish_wide: tiles larger than 16 x 16 are not widened");
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

int sss_step1_rows(const double* D, int n_dom, const int* rows, int n_sel, int n_keep,
                   const uint32_t* tm2flat, uint32_t* row_bits, void* stream) {
  if (!D || !rows || !tm2flat || !row_bits || n_dom <= 0 || n_sel < 0 || n_keep < 1)
    return fail(SSS_EINVAL, "bad step1_rows arguments");
  if (n_sel == 0) return SSS_OK;
  const size_t smem = sizeof(sss::SelShared) + 2 * (size_t)((n_dom + 31) / 32) * 4;
  if (int r = set_smem((const void*)sss::k_step1_select, smem)) return r;
  sss::k_step1_select<<<n_sel, sss::kSelThreads, smem, S_(stream)>>>(D, n_dom, n_keep, tm2flat,
                                                                     nullptr, rows, row_bits);
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

// ---- kernel seam (_accel.get_kernels(), _kernels_nb.py) -------------------

int sss_wavelet2d(const double* in, double* out, int batch, int side, int levels, int kind,
                  int inverse, void* stream) {
  if (!pow2(side) || side < 2) return fail(SSS_EINVAL, "side must be a power of two >= 2");
  int full = 0;
  while ((1 << full) < side) ++full;
  if (levels <= 0) levels = full;
  if (levels > full) return fail(SSS_EINVAL, "levels exceeds log2 side");
  if (kind != 0 && kind != 1) return fail(SSS_EINVAL, "kind must be 0 (Haar) or 1 (CDF 9/7)");
  if (batch < 0 || (batch > 0 && (!in || !out))) return fail(SSS_EINVAL, "bad batch or pointer");
  if (batch == 0) return SSS_OK;
  if (in != out) {
    cudaError_t e = cudaMemcpyAsync(out, in, (size_t)batch * side * side * sizeof(double),
                                    cudaMemcpyDeviceToDevice, S_(stream));
    if (e != cudaSuccess) return fail(SSS_ECUDA, cudaGetErrorString(e));
  }
  // forward: s = side .. side >> (levels-1), rows then columns;
  // inverse: s ascending, columns then rows (_kernels_nb.py:22-77, 124-163)
  const int s_lo = side >> (levels - 1);
  for (int step = 0; step < levels; ++step) {
    const int s = inverse ? (s_lo << step) : (side >> step);
    const int tpl = std::min(std::max(s / 2, 1), 256);
    const int lpc = 256 / tpl;
    const size_t smem = 2 * (size_t)lpc * (s + 1) * sizeof(double);
    const long long lines = (long long)batch * s;
    const long long grid = (lines + lpc - 1) / lpc;
    if (grid > 2147483647LL) return fail(SSS_EINVAL, "batch too large");
    for (int pass = 0; pass < 2; ++pass) {
      const int axis = inverse ? 1 - pass : pass;
      const void* fn = kind == 0 ? (inverse ? (const void*)sss::k_wline<0, true>
                                            : (const void*)sss::k_wline<0, false>)
                                 : (inverse ? (const void*)sss::k_wline<1, true>
                                            : (const void*)sss::k_wline<1, false>);
      if (int r = set_smem(fn, smem)) return r;
      if (kind == 0) {
        if (inverse) sss::k_wline<0, true><<<(unsigned)grid, 256, smem, S_(stream)>>>(out, batch, side, s, axis, tpl);
        else sss::k_wline<0, false><<<(unsigned)grid, 256, smem, S_(stream)>>>(out, batch, side, s, axis, tpl);
      } else {
        if (inverse) sss::k_wline<1, true><<<(unsigned)grid, 256, smem, S_(stream)>>>(out, batch, side, s, axis, tpl);
        else sss::k_wline<1, false><<<(unsigned)grid, 256, smem, S_(stream)>>>(out, batch, side, s, axis, tpl);
      }
      if (int r = check_launch("k_wline")) return r;
    }
  }
  return SSS_OK;
}

int sss_csr_apply(int n_rows, const int64_t* rowptr, const int32_t* cpos, const double* vals,
                  const double* xcol, const uint8_t* present, double* out, void* stream) {
  if (n_rows < 0 || (n_rows > 0 && (!rowptr || !out || !xcol || !present)))
    return fail(SSS_EINVAL, "bad csr_apply arguments");
  if (n_rows == 0) return SSS_OK;
  sss::k_csr_apply<<<(n_rows + 127) / 128, 128, 0, S_(stream)>>>(
      n_rows, reinterpret_cast<const long long*>(rowptr), cpos, vals, xcol, present, out);
  return check_launch("k_csr_apply");
}

int sss_transfer_rows(int nblk, int n, int K, int nr, int f64pos, const void* block_pos,
                      const void* positions, const double* areas, const double* r_nodes,
                      const double* bases, const double* slopes, double* out, void* stream) {
  if (nblk < 0 || n < 0 || K < 1 || nr < 2 || !areas || !r_nodes || !bases || !slopes ||
      ((long long)nblk * n > 0 && (!block_pos || !positions || !out)))
    return fail(SSS_EINVAL, "bad transfer_rows arguments");
  const long long total = (long long)nblk * n;
  if (total == 0) return SSS_OK;
  const unsigned grid = (unsigned)((total + 255) / 256);
  if (f64pos)
    sss::k_transfer_rows<double><<<grid, 256, 0, S_(stream)>>>(
        nblk, n, K, nr, (const double*)block_pos, (const double*)positions, areas, r_nodes, bases,
        slopes, out);
  else
    sss::k_transfer_rows<float><<<grid, 256, 0, S_(stream)>>>(
        nblk, n, K, nr, (const float*)block_pos, (const float*)positions, areas, r_nodes, bases,
        slopes, out);
  return check_launch("k_transfer_rows");
}

int sss_bvh_any_hit(int n_rays, const double* origins, const double* dirs, const double* tmax,
                    int n_nodes, const double* node_min, const double* node_max,
                    const int32_t* node_left, const int32_t* node_right, const int32_t* node_start,
                    const int32_t* node_count, const double* v0, const double* e1, const double* e2,
                    uint8_t* hit, int32_t* overflow, void* stream) {
  if (n_rays < 0 || n_nodes < 0 || (n_rays > 0 && (!origins || !dirs || !tmax || !hit)))
    return fail(SSS_EINVAL, "bad bvh_any_hit arguments");
  if (n_rays == 0) return SSS_OK;
  if (n_nodes == 0) {  // empty BVH: nothing is hit (_kernels_nb.py:269-270)
    cudaError_t e = cudaMemsetAsync(hit, 0, (size_t)n_rays, S_(stream));
    return e == cudaSuccess ? SSS_OK : fail(SSS_ECUDA, cudaGetErrorString(e));
  }
  if (!overflow) return fail(SSS_EINVAL, "overflow flag required");
  sss::RefBvh B{node_min, node_max, node_left, node_right, node_start, node_count, v0, e1, e2};
  sss::k_bvh_any_hit<<<(n_rays + 127) / 128, 128, 0, S_(stream)>>>(n_rays, origins, dirs, tmax, B,
                                                                   hit, overflow);
  return check_launch("k_bvh_any_hit");
}

int sss_atlas_scatter(const double* src, int nch, int N, const int32_t* flat_cells, int D,
                      double* dst, void* stream) {
  if (nch < 1 || N < 0 || D < N || !dst || (N > 0 && (!src || !flat_cells)))
    return fail(SSS_EINVAL, "bad atlas_scatter arguments");
  cudaError_t e = cudaMemsetAsync(dst, 0, (size_t)nch * D * sizeof(double), S_(stream));
  if (e != cudaSuccess) return fail(SSS_ECUDA, cudaGetErrorString(e));
  if (N == 0) return SSS_OK;
  const long long t = (long long)nch * N;
  sss::k_atlas_scatter<<<(unsigned)((t + 255) / 256), 256, 0, S_(stream)>>>(src, nch, N, flat_cells,
                                                                          D, dst);
  return check_launch("k_atlas_scatter");
}

int sss_atlas_recombine(int K, int D, const double* vk, const double* vk2, const double* g,
                        double* out, void* stream) {
  if (K < 1 || D < 1 || !vk || !g || !out) return fail(SSS_EINVAL, "bad atlas_recombine arguments");
  const long long t = 3LL * D;
  sss::k_atlas_recombine<<<(unsigned)((t + 255) / 256), 256, 0, S_(stream)>>>(K, D, vk, vk2, g, out);
  return check_launch("k_atlas_recombine");
}

int sss_atlas_shade(int N, int D, const double* grids, const int32_t* flat_cells,
                    const double* positions, const double* normals, const double* cam,
                    const double* material, double* radiance, double* radiance_unclamped,
                    void* stream) {
  if (N < 0 || (N > 0 && (!grids || !flat_cells || !positions || !normals || !cam || !material ||
                          !radiance || !radiance_unclamped)))
    return fail(SSS_EINVAL, "bad atlas_shade arguments");
  if (N == 0) return SSS_OK;
  sss::k_atlas_shade<<<(N + 127) / 128, 128, 0, S_(stream)>>>(N, D, grids, flat_cells, positions,
                                                             normals, cam, material, radiance,
                                                             radiance_unclamped);
  return check_launch("k_atlas_shade");
}

int sss_energy_cut(const double* sqT, int nvec, int D, double fraction, const int32_t* nnz,
                   int32_t* kept, void* stream) {
  if (nvec < 0 || D < 0 || fraction < 0.0 || fraction > 1.0 ||
      (nvec > 0 && (!sqT || !nnz || !kept)))
    return fail(SSS_EINVAL, "bad energy_cut arguments");
  if (nvec == 0) return SSS_OK;
  sss::k_energy_cut<<<(nvec + 127) / 128, 128, 0, S_(stream)>>>(sqT, nvec, D, fraction, nnz, kept);
  return check_launch("k_energy_cut");
}

// ---- one API frame's stream work in one call (runtime.Scene relight / edit)

int sss_frame_replay(void* graph_exec, int n_h2d, void* const* h2d_dst, const void* const* h2d_src,
                     const unsigned long long* h2d_bytes, void* ev_start, void* ev_end,
                     const float* radiance, const float* radiance_unclamped, long long n3,
                     double* rad64, void* host_rad64, const void* energy, void* host_energy,
                     unsigned long long energy_bytes, void* stream) {
  if (!graph_exec || n_h2d < 0 || (n_h2d > 0 && (!h2d_dst || !h2d_src || !h2d_bytes)))
    return fail(SSS_EINVAL, "bad frame_replay arguments");
  cudaStream_t st = S_(stream);
  for (int i = 0; i < n_h2d; ++i) {
    const cudaError_t e = cudaMemcpyAsync(h2d_dst[i], h2d_src[i], (size_t)h2d_bytes[i],
                                          cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return fail(SSS_ECUDA, cudaGetErrorString(e));
  }
  if (ev_start && cudaEventRecord(reinterpret_cast<cudaEvent_t>(ev_start), st) != cudaSuccess)
    return fail(SSS_ECUDA, "frame_replay: event record");
  cudaError_t e = cudaGraphLaunch(reinterpret_cast<cudaGraphExec_t>(graph_exec), st);
  if (e != cudaSuccess) return fail(SSS_ECUDA, cudaGetErrorString(e));
  if (ev_end && cudaEventRecord(reinterpret_cast<cudaEvent_t>(ev_end), st) != cudaSuccess)
    return fail(SSS_ECUDA, "frame_replay: event record");
  if (rad64 && host_rad64) {  // the float64 FrameResult arrays, widened on the device, one D2H
    // radiance == NULL: the graph's epilogue already wrote rad64 (sss_edit_finish_wide)
    if (radiance)
      if (int r = sss_widen_frame(radiance, radiance_unclamped, n3, rad64, stream)) return r;
    e = cudaMemcpyAsync(host_rad64, rad64, (size_t)(2 * n3) * sizeof(double),
                        cudaMemcpyDeviceToHost, st);
    if (e != cudaSuccess) return fail(SSS_ECUDA, cudaGetErrorString(e));
  }
  if (energy && host_energy && energy_bytes) {
    e = cudaMemcpyAsync(host_energy, energy, (size_t)energy_bytes, cudaMemcpyDeviceToHost, st);
    if (e != cudaSuccess) return fail(SSS_ECUDA, cudaGetErrorString(e));
  }
  return SSS_OK;
}

}  // extern "C"
