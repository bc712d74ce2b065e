/*
 * sss_b200.h — C ABI of the B200-native relight / material-edit path.
 *
 * Drop-in boundary for the reference's kernel seam (`_accel.get_kernels()`,
 * /root/reference/pkg/src/sssrelight/_accel.py:35-43) and the runtime API it
 * feeds (Scene / precompute_compressed / project_material). Every entry point:
 *   - takes DEVICE pointers owned by the caller (caller-allocated outputs),
 *     explicit sizes and a cudaStream_t (passed as void*), allocates nothing;
 *   - is stateless and thread-safe per stream;
 *   - returns 0 on success, <0 on a bad argument (SSS_EINVAL) or a CUDA error
 *     (SSS_ECUDA); sss_last_error() returns the message for the calling thread.
 * Kernels never raise in the reference either; validation happens
 * before launch.
 *
 * Index spaces: "flat" = r * S + c of the L-level Mallat layout of the S x S
 * geometry image (the reference's w0 / w1 domains, transfer.py:122-151);
 * "tile-major" = tile * 4^L + local, tile-local L-level layout (the frame
 * operator's row order and the v_k cache order).
 */
#ifndef SSS_B200_H
#define SSS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SSS_OK 0
#define SSS_EINVAL -1
#define SSS_ECUDA -2

const char* sss_last_error(void);
int sss_version(void);

/* ---- wavelets: replaces _k.haar2d_fwd_batch / haar2d_inv_batch
 *      (_kernels_nb.py:22-77), level-limited (L = log2 side -> full pyramid).
 *      in/out: (batch, side, side) doubles, may alias. */
int sss_haar2d(const double* in, double* out, int batch, int side, int levels,
               int inverse, void* stream);

/* ---- exact top-n (replaces wavelets.compress_top_n, wavelets.py:128-136):
 *      for each of `nvec` vectors of length n_dom, keep the n_keep largest |v|
 *      (ties -> lower index). x_out = v where kept else 0; mask (nvec x
 *      ceil(n_dom/32) words, zeroed by the callee) marks kept ids; energy
 *      (nvec x 2: total, kept) may be NULL. nvec <= 65535. */
int sss_select_topn(const double* v, int nvec, int n_dom, int n_keep, double* x_out,
                    uint32_t* mask, double* energy, void* stream);

/* ---- (a) light projection. SH: E = T L (ambient_irradiance_dense analogue,
 *      lighting.py:332-336) fused with the w0 Haar (transfer.w0_forward,
 *      transfer.py:140-144). T_l: (nl, N) float32 l-major; Lsh (nl, 3).
 *      E_out (N, 3) may be NULL; ehat (3, N) flat. */
int sss_sh_irradiance(const float* T_l, const double* Lsh, int nl, int side, int levels,
                      double* E_out, double* ehat, void* stream);

/* ---- (a) environment light: project_environment (lighting.py:293-305):
 *      per-face full Haar of a (6, s, s, 3) cubemap, top-n_keep per channel.
 *      idx (3, n_keep) ascending w2 ids, val (3, n_keep); then the union of the
 *      three lists (union_idx (3 n_keep), union_lc (3 n_keep, 3), n_union). */
int sss_env_project(const double* faces, int env_side, int n_keep, uint32_t* idx,
                    double* val, uint32_t* union_idx, double* union_lc, int* n_union,
                    void* stream);

/* ---- (a) E = W^{w2}[:, union] L^{w2} (Parseval form of
 *      ambient_irradiance_dense(W, reconstruct_environment(...)),
 *      lighting.py:308-336) fused with the w0 Haar. W2: (D, N) float32. */
int sss_env_irradiance(const float* W2, int D, const uint32_t* union_idx,
                       const double* union_lc, const int* n_union, int n_keep, int side,
                       int levels, double* E_out, double* ehat, void* stream);

/* ---- env transfer precompute: W[i, d] = V F_t cos+ d_omega with V = 1,
 *      eta = 1 (visibility_weights, lighting.py:318-329), per-face full Haar
 *      (fold_visibility's w2, transfer.py:407-411), stored float32 (D, N).
 *      dirs (D, 3), dom (D) doubles (envmap.py:45-66 tables). */
int sss_env_transfer(const float* normals, int n_points, const double* dirs,
                     const double* dom, int env_side, float* W2, void* stream);

/* ---- (c) material weights s[c][k] (project_material, basisgen.py:172-191).
 *      bw = bases * trapezoid weights (K, nr); material = device doubles
 *      {sp[3], sa[3], eta} (device-resident so a captured CUDA graph replays
 *      edits). */
int sss_material_weights(const double* bw, const double* r_nodes, int K, int nr,
                         const double* material, double* g, void* stream);

/* ---- (b)+(c) relight: K-fused transfer (TransferOperator.apply x K x 3,
 *      transfer.py:66-71 / csc_apply _kernels_nb.py:301-313) with the
 *      recombine + inverse-Haar + Fresnel shade epilogue (runtime.py:155-216).
 *      Operator: tile-major CSR per k: rowptr (K, N+1) u64 absolute offsets
 *      into cols (u32 flat w0 ids) / vals (f32). x (3, N) = masked E spectrum.
 *      g (3, K). vk (K, 3, N) tile-major cache out. scatter (N, 3) may be NULL.
 *      radiance / radiance_unclamped (N, 3) float32. cam (3). */
int sss_transfer_relight(int K, int side, int levels, const uint64_t* rowptr,
                         const uint32_t* cols, const float* vals, const double* x,
                         const double* g, const float* positions, const float* normals,
                         const double* cam, const double* material, double* vk, double* scatter,
                         float* radiance, float* radiance_unclamped, void* stream);

/* ---- edit path: stages 3-5 against the cached vk (Scene.set_material,
 *      runtime.py:189-216). */
int sss_edit_finish(int K, int side, int levels, const double* vk, const double* g,
                    const float* positions, const float* normals, const double* cam,
                    const double* material, double* scatter, float* radiance,
                    float* radiance_unclamped, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SSS_B200_H */
