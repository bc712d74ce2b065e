// ABI entry points of the abandoned transfer variants (moved out of csrc/abi.cu; not built).

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

int sss_band_offsets(const uint64_t* rowptr, const uint32_t* cols, int K, int n_rows,
                     int band_width, int n_bands, uint32_t* bandoff, void* stream) {
  if (!rowptr || !bandoff || K <= 0 || n_rows <= 0 || band_width <= 0 || n_bands <= 0)
    return fail(SSS_EINVAL, "bad band_offsets arguments");
  const long long n = (long long)K * n_rows;
  sss::k_band_offsets<<<(unsigned)((n + 255) / 256), 256, 0, S_(stream)>>>(rowptr, cols, K, n_rows,
                                                                          band_width, n_bands, bandoff);
  return check_launch("k_band_offsets");
}
