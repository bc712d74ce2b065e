// Rasterisation of per-vertex radiance: render_image /
// raster_fill (reference runtime.py:230-273, _kernels_nb.py:316-359).
//
// The reference walks triangles in order with a strict z-test, so a pixel ends
// up with the colour of the LOWEST-index triangle among those reaching the
// minimum depth (later equal depths do not overwrite), and an initial zbuf
// value acts like a triangle with index -1. The GPU reproduces exactly that
// order-independent characterisation in three passes over the triangles /
// pixels, with no ordering races:
//   1. k_raster_tri<false>: atomicMin of an order-preserving u64 key of z
//   2. k_raster_tri<true> : among covering triangles with key(z) == min, atomicMin
//                       of the triangle index
//   3. k_raster_resolve: per pixel, the winner recomputes its barycentrics and
//                       writes colour and depth (optionally the sRGB u8 pixel)
// All arithmetic is fp64 with the reference's expression order and no FMA
// contraction, so img / zbuf are bitwise equal to raster_fill's.
#pragma once
#include <cstdint>

namespace sss {

__device__ __forceinline__ unsigned long long depth_key(double z) {
  unsigned long long b = (unsigned long long)__double_as_longlong(z);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

struct RasterTri {
  double x0, y0, x1, y1, x2, y2, area;
  int i0, i1, i2;
  int xmin, xmax, ymin, ymax;
};

// The reference's per-triangle prologue (_kernels_nb.py:319-334). Returns false
// for clipped, degenerate and off-screen triangles.
__device__ __forceinline__ bool raster_setup(const int64_t* __restrict__ tris, int t,
                                             const double* __restrict__ sx,
                                             const double* __restrict__ sy,
                                             const double* __restrict__ iw, int height, int width,
                                             RasterTri& r) {
  r.i0 = (int)tris[3 * (int64_t)t];
  r.i1 = (int)tris[3 * (int64_t)t + 1];
  r.i2 = (int)tris[3 * (int64_t)t + 2];
  if (iw[r.i0] <= 0.0 || iw[r.i1] <= 0.0 || iw[r.i2] <= 0.0) return false;
  r.x0 = sx[r.i0]; r.y0 = sy[r.i0];
  r.x1 = sx[r.i1]; r.y1 = sy[r.i1];
  r.x2 = sx[r.i2]; r.y2 = sy[r.i2];
  r.area = __dsub_rn(__dmul_rn(__dsub_rn(r.x1, r.x0), __dsub_rn(r.y2, r.y0)),
                     __dmul_rn(__dsub_rn(r.y1, r.y0), __dsub_rn(r.x2, r.x0)));
  if (r.area == 0.0) return false;
  // int(floor/ceil) then clamp, evaluated in double so huge coordinates
  // near the clip plane cannot overflow the int conversion
  const double fxmin = fmax(floor(fmin(r.x0, fmin(r.x1, r.x2))), 0.0);
  const double fxmax = fmin(ceil(fmax(r.x0, fmax(r.x1, r.x2))), (double)(width - 1));
  const double fymin = fmax(floor(fmin(r.y0, fmin(r.y1, r.y2))), 0.0);
  const double fymax = fmin(ceil(fmax(r.y0, fmax(r.y1, r.y2))), (double)(height - 1));
  if (!(fxmin <= fxmax) || !(fymin <= fymax)) return false;
  r.xmin = (int)fxmin; r.xmax = (int)fxmax;
  r.ymin = (int)fymin; r.ymax = (int)fymax;
  return true;
}

// Edge functions, coverage and barycentrics of one pixel centre
// (_kernels_nb.py:335-348). Returns false when the pixel is outside.
__device__ __forceinline__ bool raster_bary(const RasterTri& r, int px, int py, double& l0,
                                            double& l1, double& l2) {
  const double pxg = (double)px + 0.5, pyg = (double)py + 0.5;
  const double w0 = __dsub_rn(__dmul_rn(__dsub_rn(r.x2, r.x1), __dsub_rn(pyg, r.y1)),
                              __dmul_rn(__dsub_rn(r.y2, r.y1), __dsub_rn(pxg, r.x1)));
  const double w1 = __dsub_rn(__dmul_rn(__dsub_rn(r.x0, r.x2), __dsub_rn(pyg, r.y2)),
                              __dmul_rn(__dsub_rn(r.y0, r.y2), __dsub_rn(pxg, r.x2)));
  const double w2 = __dsub_rn(__dmul_rn(__dsub_rn(r.x1, r.x0), __dsub_rn(pyg, r.y0)),
                              __dmul_rn(__dsub_rn(r.y1, r.y0), __dsub_rn(pxg, r.x0)));
  if (r.area > 0.0) {
    if (w0 < 0.0 || w1 < 0.0 || w2 < 0.0) return false;
  } else {
    if (w0 > 0.0 || w1 > 0.0 || w2 > 0.0) return false;
  }
  l0 = __ddiv_rn(w0, r.area);
  l1 = __ddiv_rn(w1, r.area);
  l2 = __ddiv_rn(w2, r.area);
  return true;
}

__device__ __forceinline__ double bary3(double l0, double l1, double l2, double a, double b,
                                        double c) {
  return __dadd_rn(__dadd_rn(__dmul_rn(l0, a), __dmul_rn(l1, b)), __dmul_rn(l2, c));
}

// render_image's buffer set-up (runtime.py:239-241): zbuf = inf, img = background.
__global__ void k_raster_clear(int n_pix, double b0, double b1, double b2, double* __restrict__ zbuf,
                               double* __restrict__ img) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n_pix) return;
  zbuf[p] = __longlong_as_double(0x7ff0000000000000ll);
  img[3 * (int64_t)p] = b0;
  img[3 * (int64_t)p + 1] = b1;
  img[3 * (int64_t)p + 2] = b2;
}

__global__ void k_raster_init(const double* __restrict__ zbuf, int n_pix,
                              unsigned long long* __restrict__ key, unsigned* __restrict__ win) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n_pix) return;
  key[p] = depth_key(zbuf[p]);
  win[p] = 0xffffffffu;
}

// PICK = false: pass 1 (min depth key); PICK = true: pass 2 (min index at the
// min depth). One thread per triangle; the geometry-image mesh's triangles
// cover a few pixels each, and large triangles simply loop longer.
template <bool PICK>
__global__ void __launch_bounds__(256) k_raster_tri(
    const int64_t* __restrict__ tris, int n_tris, const double* __restrict__ sx,
    const double* __restrict__ sy, const double* __restrict__ zn, const double* __restrict__ iw,
    const double* __restrict__ zbuf, int height, int width, unsigned long long* __restrict__ key,
    unsigned* __restrict__ win) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_tris) return;
  RasterTri r;
  if (!raster_setup(tris, t, sx, sy, iw, height, width, r)) return;
  const double z0 = zn[r.i0], z1 = zn[r.i1], z2 = zn[r.i2];
  for (int py = r.ymin; py <= r.ymax; ++py) {
    for (int px = r.xmin; px <= r.xmax; ++px) {
      double l0, l1, l2;
      if (!raster_bary(r, px, py, l0, l1, l2)) continue;
      const double z = bary3(l0, l1, l2, z0, z1, z2);
      const int64_t p = (int64_t)py * width + px;
      if (!(z < zbuf[p])) continue;  // strict test against the initial buffer
      const unsigned long long kz = depth_key(z);
      if (!PICK) {
        if (kz < key[p]) atomicMin(key + p, kz);
      } else if (kz == key[p]) {
        atomicMin(win + p, (unsigned)t);
      }
    }
  }
}

// Per pixel: the winning triangle writes colour and depth (_kernels_nb.py:349-358);
// srgb8 (optional) receives the (linear_to_srgb(img * exposure) * 255 + 0.5)
// u8 pixel of render_image (runtime.py:245) for every pixel, background included.
__global__ void k_raster_resolve(const int64_t* __restrict__ tris, const double* __restrict__ sx,
                                 const double* __restrict__ sy, const double* __restrict__ zn,
                                 const double* __restrict__ iw, const double* __restrict__ colors,
                                 int height, int width, const unsigned* __restrict__ win,
                                 double* __restrict__ zbuf, double* __restrict__ img,
                                 double exposure, uint8_t* __restrict__ srgb8);

__device__ __forceinline__ uint8_t srgb8_of(double v, double exposure) {
  double x = __dmul_rn(v, exposure);
  x = fmin(fmax(x, 0.0), 1.0);  // np.clip (NaN maps to 0 here and in uint8 casts)
  double s = x <= 0.0031308 ? __dmul_rn(x, 12.92)
                            : __dsub_rn(__dmul_rn(1.055, pow(x, 1.0 / 2.4)), 0.055);
  const double q = __dadd_rn(__dmul_rn(s, 255.0), 0.5);
  return (uint8_t)(int)q;
}

__global__ void k_raster_resolve(const int64_t* __restrict__ tris, const double* __restrict__ sx,
                                 const double* __restrict__ sy, const double* __restrict__ zn,
                                 const double* __restrict__ iw, const double* __restrict__ colors,
                                 int height, int width, const unsigned* __restrict__ win,
                                 double* __restrict__ zbuf, double* __restrict__ img,
                                 double exposure, uint8_t* __restrict__ srgb8) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= height * width) return;
  const unsigned t = win[p];
  if (t != 0xffffffffu) {
    RasterTri r;
    raster_setup(tris, (int)t, sx, sy, iw, height, width, r);
    double l0, l1, l2;
    raster_bary(r, p % width, p / width, l0, l1, l2);
    const double q0 = iw[r.i0], q1 = iw[r.i1], q2 = iw[r.i2];
    const double wi = bary3(l0, l1, l2, q0, q1, q2);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double num = bary3(l0, l1, l2, __dmul_rn(colors[3 * r.i0 + c], q0),
                               __dmul_rn(colors[3 * r.i1 + c], q1),
                               __dmul_rn(colors[3 * r.i2 + c], q2));
      img[3 * (int64_t)p + c] = __ddiv_rn(num, wi);
    }
    zbuf[p] = bary3(l0, l1, l2, zn[r.i0], zn[r.i1], zn[r.i2]);
  }
  if (srgb8) {
#pragma unroll
    for (int c = 0; c < 3; ++c) srgb8[3 * (int64_t)p + c] = srgb8_of(img[3 * (int64_t)p + c], exposure);
  }
}

// _project_vertices (runtime.py:247-273) with the camera frame precomputed on
// the host: cam = {position[3], right[3], up[3], fwd[3]}; dot products in the
// order (x r0 + y r1) + z r2. Also scatters the per-sample radiance into the
// per-vertex colour array (render_image, runtime.py:236-237; colors is zeroed
// by the caller).
__global__ void k_raster_project(const double* __restrict__ vertices, int n_vertices,
                                 const double* __restrict__ cam, double f, double aspect,
                                 int width, int height, double* __restrict__ sx,
                                 double* __restrict__ sy, double* __restrict__ zn,
                                 double* __restrict__ iw) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n_vertices) return;
  const double r0 = __dsub_rn(vertices[3 * v], cam[0]);
  const double r1 = __dsub_rn(vertices[3 * v + 1], cam[1]);
  const double r2 = __dsub_rn(vertices[3 * v + 2], cam[2]);
  auto dot = [&](const double* a) {
    return __dadd_rn(__dadd_rn(__dmul_rn(r0, a[0]), __dmul_rn(r1, a[1])), __dmul_rn(r2, a[2]));
  };
  const double x = dot(cam + 3), y = dot(cam + 6), z = dot(cam + 9);
  const double ndc_x = __ddiv_rn(__ddiv_rn(__dmul_rn(x, f), aspect), z);
  const double ndc_y = __ddiv_rn(__dmul_rn(y, f), z);
  sx[v] = __dmul_rn(__dadd_rn(__dmul_rn(ndc_x, 0.5), 0.5), (double)width);
  sy[v] = __dmul_rn(__dsub_rn(0.5, __dmul_rn(ndc_y, 0.5)), (double)height);
  const bool front = z > 1e-3;
  iw[v] = front ? __ddiv_rn(1.0, z) : 0.0;
  zn[v] = front ? z : __longlong_as_double(0x7ff0000000000000ll);
}

__global__ void k_vertex_colors(const float* __restrict__ radiance, const int32_t* __restrict__ src,
                                int n, double* __restrict__ colors) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int v = src ? src[i] : i;
#pragma unroll
  for (int c = 0; c < 3; ++c) colors[3 * (int64_t)v + c] = (double)radiance[3 * (int64_t)i + c];
}

// FrameResult read-back: out[0] = radiance, out[1] = radiance_unclamped as
// float64 (runtime.py:56-62 dtype), so the host receives the final arrays by
// DMA with no host-side conversion.
__global__ void k_widen_frame(const float* __restrict__ rad, const float* __restrict__ radu,
                              int64_t n, double* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    out[i] = (double)rad[i];
    out[n + i] = (double)radu[i];
  }
}

// Per-element sRGB u8 encoding (service.py:181 frame payload).
__global__ void k_encode_srgb8(const double* __restrict__ x, int64_t n, double exposure,
                               uint8_t* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = srgb8_of(x[i], exposure);
}

}  // namespace sss
