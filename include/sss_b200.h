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
 *      (nvec x 2: total, kept) may be NULL. nvec <= 65535. f2t (may be NULL)
 *      permutes x_out into the operator's tile-major column space. */
int sss_select_topn(const double* v, int nvec, int n_dom, int n_keep, const uint32_t* f2t,
                    double* x_out, uint32_t* mask, double* energy, void* stream);

/* The frame's form of the same selection (runtime.py:112-118: the three RGB
 * spectra of E): additionally writes what the transfer kernels read, the
 * packed (n_dom, 4) fp64 records {x_r, x_g, x_b, 0} (xp; the fourth component
 * is never written) and the kept-column bitmap (bits, n_dom/32 + 1 words, bit
 * set iff any channel kept a nonzero coefficient of the column) - the outputs
 * of sss_pack_x_bits, without a second launch. bits MUST be zero on entry. */
int sss_select_topn_pack(const double* v, int n_dom, int n_keep, const uint32_t* f2t,
                         double* x_out, uint32_t* mask, double* energy, double* xp,
                         uint32_t* bits, void* stream);

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

/* sss_env_irradiance_sel: sss_env_irradiance with the union built inside
 *   every CTA from sss_env_project's per-channel kept lists (sel_idx (3, n_keep)
 *   u32, 0xffffffff-padded; sel_val (3, n_keep) f64) instead of k_env_union's
 *   output: same E and spectrum bits, one launch less per frame. D = 6 s^2 <= 6144. */
int sss_env_irradiance_sel(const float* W2, int D, const uint32_t* sel_idx, const double* sel_val,
                           int n_keep, int side, int levels, double* E_out, double* ehat,
                           void* stream);

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

/* ---- C4 batched material sweep (BASELINE configs[3]; runtime.py:202-216 for
 * a batch of materials). B operand: Bq (3, N, 16) bf16 = w1^-1 of the cached
 * v_k (K <= 16 terms, zero padded), points in flat (spatial) order. */
int sss_sweep_basis(int K, int side, int levels, const double* vk, void* Bq, void* stream);

/* ---- project_material (basisgen.py:172-191) for M materials at once:
 * materials (M, 7) doubles {sp[3], sa[3], eta}; g64 (M, 3, K) fp64 (may be
 * NULL), Gq (3, M, 16) bf16 (the sweep's G operand), eta_f (M) float (may be
 * NULL). */
int sss_material_weights_batch(const double* bw, const double* r_nodes, int K, int nr, int M,
                               const double* materials, double* g64, void* Gq, float* eta_f,
                               void* stream);

/* ---- the sweep contraction (tcgen05 UMMA, bf16 in, fp32 accumulate in TMEM):
 * out (3, M, N) fp32 = max(0, F_t(eta_m, cos_n) / pi * sum_k Bq[c][n][k]
 * Gq[c][m][k]), cos_n from positions / normals / cam; F_t is evaluated through
 * a per-point cubic fit in eta over [eta_lo, eta_hi] (all eta_m inside, > 1). */
int sss_sweep_gemm(int n_points, int M, const void* Bq, const void* Gq, const float* eta,
                   float eta_lo, float eta_hi, const float* positions, const float* normals,
                   const double* cam, float* out, void* stream);

/* ---- (a) direct lights with shadow rays: irradiance_direct
 * (lighting.py:208-290) with BVH any-hit visibility (lighting.py:101-176,
 * _kernels_nb.py:208-298). lights: n_lights x 12 doubles {kind (0 point, 1
 * directional, 2 sphere), a[3] (position / unit direction light->scene /
 * center), b[3] (intensity / irradiance / radiance), radius, 0...};
 * kinds: the same n_lights kinds in HOST memory (they pick each light's
 * kernel at launch; a graph captured for one rig structure replays any values
 * of that structure). material[6] = eta (the incident Fresnel term); ray
 * origins offset ray_offset along the normal; the packed BVH of
 * shadows.BVH.packed(): nodes (M, 8) doubles {min[3], max[3], (i32 left,
 * i32 right), (i32 start, i32 count)}, tris (T, 10) doubles {v0[3], e1[3],
 * e2[3], 0} in leaf order. E: planar (3, N) doubles (zeroed, then one launch
 * per light adds its term in light order). */
int sss_direct_irradiance(int n_points, const float* positions, const float* normals,
                          int n_lights, const int* kinds, const double* lights,
                          const double* material, double ray_offset, double bbox_diagonal,
                          const double* nodes, const double* tris, double* E, void* stream);

/* sss_direct_irradiance64: the same with fp64 positions / normals (the
 *   reference's SurfaceSamples of an arbitrary mesh, api.Scene). */
int sss_direct_irradiance64(int n_points, const double* positions, const double* normals,
                            int n_lights, const int* kinds, const double* lights,
                            const double* material, double ray_offset, double bbox_diagonal,
                            const double* nodes, const double* tris, double* E, void* stream);

/* ---- visibility precompute + ambient folding (
 * transfer.py:368-451). D = 6 face_side^2 cubemap texel directions.
 *
 * sss_visibility: precompute_visibility (transfer.py:368-391): vis (D, N) u8
 *   = n.d > 0 and no hit within `far` (4 bbox diagonal + 1) from p + offset n;
 *   dirs (D, 3) doubles (envmap.face_directions); packed BVH as for
 *   sss_direct_irradiance. */
int sss_visibility(int n_points, const float* positions, const float* normals, int n_dirs,
                   const double* dirs, double ray_offset, double far, const double* nodes,
                   const double* tris, uint8_t* vis, void* stream);

/* sss_fold_weights: visibility_weights with the material eta
 *   (lighting.py:318-329) and the per-face full Haar over directions
 *   (transfer.py:407-411): W2 (D, N) fp64 (then the w0 Haar over samples with
 *   sss_haar2d, batch D). */
int sss_fold_weights(const float* normals, int n_points, const double* dirs, const double* dom,
                     int face_side, const uint8_t* vis, double eta, double* W2, void* stream);

/* out (cols, rows) = in (rows, cols)^T, optionally gathering input columns:
 * out[j][r] = in[r][col_perm ? col_perm[j] : j]. */
int sss_transpose_f64(const double* in, int rows, int cols, const uint32_t* col_perm, double* out,
                      void* stream);

/* sss_fold_spmm: F (n_rows, n_dirs) row-major = T_k v~ (transfer.py:426's
 *   dense @ v_tilde[cols]) for one operator of the frame layout (rowptr
 *   absolute int64, tile-major cols, f32 vals); vt (N tm, n_dirs). */
int sss_fold_spmm(int n_rows, int n_dirs, const long long* rowptr, const uint32_t* cols,
                  const float* vals, const double* vt, double* F, void* stream);

/* sss_fold_select: compress_energy(fraction) of every direction column of FT
 *   (n_dirs, n_rows tm) (transfer.py:427, wavelets.py:139-153): threshold
 *   key, tie bound (flat row), kept count, (kept, total) energy, nonzeros. */
int sss_fold_select(const double* FT, int n_rows, int n_dirs, double fraction,
                    const uint32_t* tm2flat, uint64_t* col_t, uint32_t* col_fmax,
                    uint32_t* col_cnt, double* col_energy, uint32_t* col_nz, void* stream);

/* sss_fold_emit: CSC of the kept entries per direction, rows ascending flat
 *   ids, vals f32; colptr (n_dirs + 1) = exclusive scan of col_cnt. */
int sss_fold_emit(const double* FT, int n_rows, int n_dirs, const uint32_t* flat2tm,
                  const uint64_t* col_t, const uint32_t* col_fmax, const uint32_t* col_cnt,
                  const uint64_t* colptr, uint32_t* rows, float* vals, void* stream);

/* sss_fold_apply: the folded ambient term of _stage2_transfer
 *   (runtime.py:146-149): vk[k][c][tm] += sum over the environment union
 *   (sss_env_project's union_idx / union_lc / n_union, ascending) of
 *   F_k[r][e] L_c[e], in the reference's serial csc_apply order. colptr
 *   (K, n_dirs + 1) absolute into rows / vals. */
int sss_fold_apply(int K, int n_rows, int n_dirs, const uint64_t* colptr, const uint32_t* rows,
                   const float* vals, const uint32_t* union_idx, const double* union_lc,
                   const int* n_union, const uint32_t* flat2tm, double* vk, void* stream);

/* ---- (b) scattering transfer, stage 2 of the frame: replaces the K x 3
 *      TransferOperator.apply -> _k.csc_apply calls of _stage2_transfer
 *      (runtime.py:138-150, transfer.py:50-71, _kernels_nb.py:301-313):
 *      vk (K, 3, n_rows) f64 tile-major = T_k x_c for every term k and channel c.
 *      xp (n_rows, 4) f64 and bits (n_rows / 32 + 1 words, last word clear) are
 *      sss_pack_x_bits's packing of the kept spectrum x (3, n_rows).
 *
 * sss_transfer_kfr ("K-fused rows", default): the operator as a stream of
 *   (column, term-mask) pairs per (receiver row, group of 4 terms) chunk
 *   (layout.kfr_layout): items (n_items x {first batch, steps}), lane_len /
 *   lane_dst (32 per item: chunk length; row | group << 16, 0x80000000 |
 *   partial slot, or 0xffffffff), batch_off (byte offset of every batch in
 *   stream_bytes + a sentinel, multiples of 16), stream_bytes (per batch of
 *   steps_per_batch (4 or 8) steps: 32 words per step {col | mask << 16 |
 *   value offset << 20, 0 = no pair}, then the f32 values lane-major per
 *   step, padded to 16 bytes), partials ((12, n_partials) f64 scratch),
 *   partial_row (multi-chunk index of each slot), multi_info ({row, first
 *   slot, count, group} per multi-chunk (row, group)), multi_count (zeroed
 *   u32 per multi-chunk (row, group); left zero on return), work (two zeroed
 *   u32: item claim and CTA exit counters; left zero on return). Writes every
 *   row of vk (no memset), bitwise reproducible. K <= 16, n_rows <= 65536.
 *   n_warps: warps launched (multiple of 8), min_blocks: CTAs of 256 threads
 *   per SM (3 for 4-step batches, 2 for 8-step batches). */
int sss_transfer_kfr(int K, int n_rows, unsigned n_items, unsigned n_partials, const void* items,
                     const uint32_t* lane_len, const uint32_t* lane_dst, const uint32_t* batch_off,
                     const void* stream_bytes, const void* xp, const uint32_t* bits,
                     double* vk, double* partials, const uint32_t* partial_row,
                     const void* multi_info, uint32_t* multi_count, uint32_t* work,
                     int steps_per_batch, int n_warps, int min_blocks, void* stream);

/* sss_pack_x_bits: xp (n, 4) f64 = {x0, x1, x2, 0} of the kept spectrum
 *   x (3, n) and the kept-column bitmap (bit c set iff any channel is kept). */
int sss_pack_x_bits(const double* x, int n, void* xp, uint32_t* bits, void* stream);

/* sss_transfer_flat16 (A/B alternative): the operator as a flat stream of
 *   (row, k) segments, each padded to a multiple of entries_per_lane (16 or 32)
 *   entries and lane-interleaved, head bits one per group, per-word head prefix
 *   and segment (row << 4 | k) ids (layout.flat16_layout). col_bits 32: u32
 *   columns, padding entries carry column n_rows / value 0 and the kept bitmap
 *   `bits` needs n_rows / 32 + 1 words with the bit of column n_rows clear.
 *   col_bits 16 (n_rows <= 65536, 16 entries per lane): u16 columns, padding
 *   keeps column 0 with value 0. min_blocks = CTAs of 128 threads per SM: 4, 6,
 *   8 for 16 entries, 6, 8 for 32, 8 for 16-bit columns. vk must be zero
 *   (zeroed here when zero_vk). word_partials != NULL (6 doubles per word of
 *   32 lanes, ceil(n_entries / entries_per_lane / 32) words): deterministic
 *   sums - segments inside one word are stored, the pieces of rows spanning
 *   words are added in word order by a second small launch (span_first: per
 *   word, the word in which the row running into it began = the last word
 *   before it that holds a head); NULL: fp64 atomics into vk (order not fixed).
 *   work_counter (u32, nullable): warps claim `chunk` words at a time from it;
 *   it must be zero at launch (zeroed here with vk when zero_vk). */
int sss_transfer_flat16(int K, int n_rows, const void* pcols, const float* pvals,
                        unsigned long long n_entries, const uint32_t* heads,
                        const uint32_t* head_prefix, const uint32_t* seg_rowk,
                        const unsigned* warp_begin, int n_warps, int min_blocks,
                        int entries_per_lane, int col_bits, int zero_vk, const void* xp,
                        const uint32_t* bits, double* vk, uint32_t* work_counter, int chunk,
                        double* word_partials, const uint32_t* span_first, void* stream);

/* sss_fold_apply_rows: the same v_k update as sss_fold_apply from a row-major
 *   copy of the folded operators, ELL-interleaved per 32-row group: group g =
 *   k * (n_rows / 32) + row / 32 owns [gbase[g], gbase[g + 1]) (absolute), entry
 *   s of the group's lane j at gbase[g] + 32 s + j, ascending by direction within
 *   a row, padded with (dir 0, val 0); entries = (dir u32, val f32 bits) pairs. One thread per
 *   (k, row), per-row sums in the csc_apply order, bitwise equal to
 *   sss_fold_apply. n_rows % 32 == 0; 24 * n_dirs <= 200 KB of shared memory. */
int sss_fold_apply_rows(int K, int n_rows, int n_dirs, const uint64_t* gbase,
                        const uint32_t* entries, const uint32_t* union_idx,
                        const double* union_lc, const int* n_union, const uint32_t* flat2tm,
                        double* vk, void* stream);

/* ---- edit path: stages 3-5 against the cached vk (Scene.set_material,
 *      runtime.py:189-216). */
int sss_edit_finish(int K, int side, int levels, const double* vk, const double* g,
                    const float* positions, const float* normals, const double* cam,
                    const double* material, double* scatter, float* radiance,
                    float* radiance_unclamped, void* stream);

/* The same, additionally writing the API's float64 FrameResult pair rad64
 * (2 x N x 3: radiance, then radiance_unclamped, the float32 results widened:
 * sss_widen_frame's output) so an API frame needs no widening launch. rad64
 * may be NULL (= sss_edit_finish). Tiles up to 16 x 16 (levels <= 4). */
int sss_edit_finish_wide(int K, int side, int levels, const double* vk, const double* g,
                         const float* positions, const float* normals, const double* cam,
                         const double* material, double* scatter, float* radiance,
                         float* radiance_unclamped, double* rad64, void* stream);

/* ================= precompute (path d): pair pass + two-step compression ====
 * replaces precompute_compressed (transfer.py:350-361) for a geometry image
 * with L-level Haar (L <= 3) on w0 and w1. N = side^2; "tm" = tile-major.  */

/* Pair block pass for PCA term k (transfer_block, _kernels_nb.py:179-205):
 *   exact = 0: lerp of the tabulated bases, fp64, bitwise the reference's;
 *   exact = 1: R_d evaluated per pair for each of n_mat training materials in
 *              fp32, projected with Pkm (K, n_mat) = U/S (mat (n_mat, 4):
 *              sigma_tr, z_r, z_v, alpha'/(4 pi)), masked at r_max.
 * Writes D (N, N) fp64 = w0 Haar of each receiver row (tm rows, tm columns)
 * and/or Mout (N, N) fp64 = w1 Haar of f32(D) along receivers, column-major
 * (column c_tm contiguous). Either may be NULL. */
int sss_pair_block(int levels, int exact, int side, const float* pos, const float* area,
                   const double* r_nodes, const double* bases, const double* slopes, int nr, int k,
                   const float* Pkm, const float* mat, int n_mat, float r_max, double* D,
                   double* Mout, void* stream);

/* sss_pair_rows_exact: the exact pair pass K-fused and streamed (BASELINE
 * C5): for receiver tiles [rt0, rt0 + nrt) against every source tile, each
 * pair's fp32 R_d at the n_mat training materials is evaluated once and
 * projected on all K terms, x area, w0 Haar along sources. Pkm (K, n_mat)
 * and mat (n_mat, 4) {sigma_tr, z_r, z_v, alpha'/(4 pi)} are HOST arrays
 * (copied into the kernel's parameter bank; n_mat <= 64, K <= 8). D (K,
 * nrt * 4^L, N) fp64 = the step-1 rows of the block for every term
 * (tile-major rows and columns). */
int sss_pair_rows_exact(int levels, int side, const float* pos, const float* area, int K,
                        const float* Pkm, const float* mat, int n_mat, float r_max, int rt0,
                        int nrt, double* D, void* stream);

/* Step 1 (run_step1 + step1_unions, transfer.py:216-246): per row of D keep
 * the n_keep largest |v| (flat-index tie-break) and OR the kept flat column
 * ids into union_bits (N/32 words, caller-zeroed). */
int sss_step1_select(const double* D, int n_dom, int n_rows, int n_keep, const uint32_t* tm2flat,
                     uint32_t* union_bits, void* stream);

/* sss_step1_rows: the same per-row top-n for the listed rows of D only (tile-
 * major row ids), each row's kept flat ids written as a bitmap (n_sel x
 * N/32 words): the sampled-row parity hook of step 1. */
int sss_step1_rows(const double* D, int n_dom, const int* rows, int n_sel, int n_keep,
                   const uint32_t* tm2flat, uint32_t* row_bits, void* stream);

/* Step 2 (_threshold_columns, transfer.py:303-333 with compress_energy): for
 * each union column, the energy-fraction cut. Per tm column: threshold key
 * col_t (~0 = column dropped), tie bound col_fmax (flat row), kept count,
 * energy (kept, total). */
int sss_step2_select(const double* M, int n_dom, double fraction, const uint32_t* flat2tm,
                     const uint32_t* tm2flat, const uint32_t* union_bits, uint64_t* col_t,
                     uint32_t* col_fmax, uint32_t* col_cnt, double* col_energy, void* stream);

/* Emission into the frame layout (tile-major CSR). pass 0: counts
 * (N rows x nchunks); pass 1: write cols (flat w0 ids) / vals (f32) at offs
 * (exclusive scan of counts, relative to this k's arrays). */
int sss_emit(int pass, const double* M, int n_dom, int tile_rows, int chunk, const uint64_t* col_t,
             const uint32_t* col_fmax, const uint32_t* tm2flat, uint32_t* counts,
             const uint64_t* offs, uint32_t* cols, float* vals, void* stream);

/* exclusive scan u32 -> u64 (block_sums: ceil(n/1024) scratch; total out) */
int sss_scan_u32(const uint32_t* in, uint64_t* out, size_t n, uint64_t* block_sums,
                 uint64_t* total, void* stream);

/* rowptr[r] = base + offs[r * nchunks], rowptr[n_rows] = base + *total */
int sss_rowptr(const uint64_t* offs, int nchunks, int n_rows, uint64_t base, const uint64_t* total,
               uint64_t* rowptr, void* stream);

/* ---- rasterisation ---------------------------------- */

/* sss_raster_fill: replaces raster_fill (_kernels_nb.py:316-359,
 *   _kernels_np.py:264-313), called by render_image (runtime.py:242-243).
 *   In place on zbuf (height, width) f64 and img (height, width, 3) f64, exactly
 *   the reference's sequential semantics (triangles in order, strict z-test,
 *   perspective-correct colour; bitwise). tris (n_tris, 3) i64; sx, sy, zn, iw
 *   (V,) f64; colors (V, 3) f64. Scratch: key (height*width) u64, win
 *   (height*width) u32. srgb8 (optional, height*width*3 u8) receives render_image's
 *   (linear_to_srgb(img * exposure) * 255 + 0.5) quantisation (runtime.py:245). */
int sss_raster_fill(const int64_t* tris, int n_tris, const double* sx, const double* sy,
                    const double* zn, const double* iw, const double* colors, int height,
                    int width, double* zbuf, double* img, unsigned long long* key,
                    uint32_t* win, double exposure, uint8_t* srgb8, void* stream);

/* sss_raster_clear: zbuf = +inf, img = background (runtime.py:239-241). */
int sss_raster_clear(int height, int width, double b0, double b1, double b2, double* zbuf,
                     double* img, void* stream);

/* sss_project_vertices: replaces _project_vertices (runtime.py:247-273).
 *   cam = {position, right, up, fwd} (12 f64, device; the frame is built on
 *   the host as runtime.py:248-256 does); f = 1/tan(fov/2), aspect = w/h.
 *   Dot products evaluated as (x r0 + y r1) + z r2. Outputs sx, sy, zn, iw (V,). */
int sss_project_vertices(const double* vertices, int n_vertices, const double* cam, double f,
                         double aspect, int width, int height, double* sx, double* sy,
                         double* zn, double* iw, void* stream);

/* sss_vertex_colors: colors[source_vertex[i]] = radiance[i] (f32 -> f64), the
 *   scatter of render_image (runtime.py:236-237) and of the service frame
 *   payload (service.py:176-177). source_vertex NULL = identity. colors is
 *   caller-zeroed (V, 3). */
int sss_vertex_colors(const float* radiance, const int32_t* source_vertex, int n, double* colors,
                      void* stream);

/* sss_zero: cudaMemsetAsync(ptr, 0, bytes) on the stream (v_k before an
 *   accumulating transfer, issued on a side stream that overlaps stage 1). */
int sss_zero(void* ptr, unsigned long long bytes, void* stream);

/* sss_widen_frame: out (2, n) f64 = (radiance, radiance_unclamped) widened
 *   from the frame's f32 device buffers: the FrameResult arrays (runtime.py:
 *   56-62, float64) leave the device ready to use (n = points * 3). */
int sss_widen_frame(const float* radiance, const float* radiance_unclamped, long long n,
                    double* out, void* stream);

/* sss_encode_srgb8: out[i] = uint8(linear_to_srgb(x[i] * exposure) * 255 + 0.5),
 *   the quantised frame payload of the service (service.py:181, envmap.py:74-76). */
int sss_encode_srgb8(const double* x, long long n, double exposure, uint8_t* out, void* stream);

/* ---- kernel seam: device twins of _kernels_nb (bound with numpy in / out
 *      by paper_2203_12339_b200/kernels_b200.py, the module a maintainer puts
 *      behind _accel.get_kernels(), _accel.py:35-43). Bitwise the reference's
 *      arithmetic (no FMA contraction). ------------------------------------ */

/* sss_wavelet2d: replaces haar2d_fwd_batch / haar2d_inv_batch (kind 0,
 *   _kernels_nb.py:22-77) and cdf97_fwd_batch / cdf97_inv_batch (kind 1,
 *   _kernels_nb.py:80-163, used by w1_inverse transfer.py:147-151 and
 *   _threshold_columns transfer.py:303-316). (batch, side, side) f64, any
 *   power-of-two side; levels <= 0 = the full pyramid (the reference's only
 *   mode), else the first `levels` levels. in may alias out. */
int sss_wavelet2d(const double* in, double* out, int batch, int side, int levels, int kind,
                  int inverse, void* stream);

/* sss_csr_apply: replaces csc_apply (_kernels_nb.py:301-313, called by
 *   TransferOperator.apply, transfer.py:66-71). The operator as a row-major
 *   copy whose entries keep ascending column order (rowptr (n_rows+1) i64,
 *   cpos = column position, vals f64); xcol (n_cols) the spectrum value per
 *   column position, present (n_cols) u8 = the column is in x_idx. out[r] =
 *   the reference's fp64 sum in its order; rows without entries are 0. */
int sss_csr_apply(int n_rows, const int64_t* rowptr, const int32_t* cpos, const double* vals,
                  const double* xcol, const uint8_t* present, double* out, void* stream);

/* sss_transfer_rows: replaces transfer_block (_kernels_nb.py:179-205):
 *   out (nblk, K, n) f64. block_pos (nblk, 3) and positions (n, 3) in one
 *   dtype (f64pos = 1: double, 0: float; the distance is evaluated in it as
 *   numba does), areas (n) f64, r_nodes (nr), bases (K, nr), slopes (K, nr-1) f64. */
int sss_transfer_rows(int nblk, int n, int K, int nr, int f64pos, const void* block_pos,
                      const void* positions, const double* areas, const double* r_nodes,
                      const double* bases, const double* slopes, double* out, void* stream);

/* sss_bvh_any_hit: replaces bvh_any_hit (_kernels_nb.py:265-298) on the
 *   reference's RayAccelerator arrays (lighting.py:101-170): node_min/max
 *   (n_nodes, 3) f64, left/right/start/count i32, v0/e1/e2 (T, 3) f64;
 *   origins/dirs (n_rays, 3), tmax (n_rays). hit (n_rays) u8. *overflow is
 *   set to 1 if a traversal needed more than the reference's 64-entry stack. */
int sss_bvh_any_hit(int n_rays, const double* origins, const double* dirs, const double* tmax,
                    int n_nodes, const double* node_min, const double* node_max,
                    const int32_t* node_left, const int32_t* node_right, const int32_t* node_start,
                    const int32_t* node_count, const double* v0, const double* e1, const double* e2,
                    uint8_t* hit, int32_t* overflow, void* stream);

/* ---- the frame of an arbitrary QuadtreeAtlas (api.Scene; runtime.py:109-216)
 *      D = part_count * grid_side^2 (the w0 / w1 domain), flat_cells (N) i32 =
 *      part * side^2 + cell (atlas_flat_cells, transfer.py:122-125). */

/* sss_atlas_scatter: scatter_to_grids (transfer.py:128-132): dst (nch, D)
 *   zeroed (PAD cells), then dst[c, flat_cells[i]] = src[c, i]. */
int sss_atlas_scatter(const double* src, int nch, int N, const int32_t* flat_cells, int D,
                      double* dst, void* stream);

/* sss_atlas_recombine: out (3, D) = sum_k g[c, k] (vk[k, c] + vk2[k, c])
 *   (runtime.py:204; vk2 = the folded ambient term, may be NULL). */
int sss_atlas_recombine(int K, int D, const double* vk, const double* vk2, const double* g,
                        double* out, void* stream);

/* sss_atlas_shade: gather_from_grids (transfer.py:135-137) of the inverse-9/7
 *   grids (3, D) + _shade (runtime.py:162-168): radiance / radiance_unclamped
 *   (N, 3) f64; cam (3) f64 device, material {sp[3], sa[3], eta}. */
int sss_atlas_shade(int N, int D, const double* grids, const int32_t* flat_cells,
                    const double* positions, const double* normals, const double* cam,
                    const double* material, double* radiance, double* radiance_unclamped,
                    void* stream);

/* sss_energy_cut: the kept count of compress_energy (wavelets.py:139-153)
 *   for nvec vectors: sqT (D, nvec) = squared coefficients in descending-|v|
 *   order (stable), transposed; the reference's sequential cumsum and
 *   searchsorted(.., fraction * total, "left") + 1, capped at nnz[v]. */
int sss_energy_cut(const double* sqT, int nvec, int D, double fraction, const int32_t* nnz,
                   int32_t* kept, void* stream);

/* sss_frame_replay: one API frame's stream work in a single call (the Python
 *   per-call overhead of the relight / edit frames): n_h2d host->device copies
 *   from pinned staging (the new light / material / camera), an event, the
 *   frame's CUDA graph (cudaGraphExec_t), an event, the float64 widening of
 *   the radiance (as sss_widen_frame; skipped when radiance is NULL: the
 *   graph's epilogue wrote rad64 itself, sss_edit_finish_wide) and its
 *   device->host copy into pinned memory, the kept-energy copy. Any part may
 *   be NULL / 0. */
int sss_frame_replay(void* graph_exec, int n_h2d, void* const* h2d_dst, const void* const* h2d_src,
                     const unsigned long long* h2d_bytes, void* ev_start, void* ev_end,
                     const float* radiance, const float* radiance_unclamped, long long n3,
                     double* rad64, void* host_rad64, const void* energy, void* host_energy,
                     unsigned long long energy_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SSS_B200_H */
