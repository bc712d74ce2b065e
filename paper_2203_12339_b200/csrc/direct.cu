// Direct lights with shadow rays: irradiance_direct
// (lighting.py:208-290) with BVH any-hit visibility (lighting.py:101-176,
// _kernels_nb.py:208-298), one thread per surface sample.
//
// Ray / box / triangle tests and the point-light weights use explicit fp64
// round-to-nearest operations (no FMA contraction) in the reference's
// operation order, so visibility bits are those of the reference; the sphere
// light's stratified cone uses cos/sin (libm ulps) and a sequential mean.
// Output: E planar (3, N) doubles (the input of the w0 Haar + top-n path).
#include "sss_common.cuh"

namespace sss {

struct BvhView {
  const double* nmin;   // (M, 3)
  const double* nmax;   // (M, 3)
  const int* left;
  const int* right;
  const int* start;
  const int* count;
  const double* v0;     // (T, 3) leaf order
  const double* e1;
  const double* e2;
};

__device__ __forceinline__ double dsub_(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double ddiv_(double a, double b) { return __ddiv_rn(a, b); }

// _kernels_nb.py:209-232
__device__ __forceinline__ bool tri_hit(const BvhView& B, int t, const double* o, const double* d,
                                        double tmax) {
  const double e1x = B.e1[3 * t], e1y = B.e1[3 * t + 1], e1z = B.e1[3 * t + 2];
  const double e2x = B.e2[3 * t], e2y = B.e2[3 * t + 1], e2z = B.e2[3 * t + 2];
  const double pvx = dsub_(dmul(d[1], e2z), dmul(d[2], e2y));
  const double pvy = dsub_(dmul(d[2], e2x), dmul(d[0], e2z));
  const double pvz = dsub_(dmul(d[0], e2y), dmul(d[1], e2x));
  const double det = dadd(dadd(dmul(e1x, pvx), dmul(e1y, pvy)), dmul(e1z, pvz));
  if (fabs(det) <= 1e-14) return false;
  const double inv = ddiv_(1.0, det);
  const double tvx = dsub_(o[0], B.v0[3 * t]), tvy = dsub_(o[1], B.v0[3 * t + 1]),
               tvz = dsub_(o[2], B.v0[3 * t + 2]);
  const double u = dmul(dadd(dadd(dmul(tvx, pvx), dmul(tvy, pvy)), dmul(tvz, pvz)), inv);
  if (u < 0.0 || u > 1.0) return false;
  const double qvx = dsub_(dmul(tvy, e1z), dmul(tvz, e1y));
  const double qvy = dsub_(dmul(tvz, e1x), dmul(tvx, e1z));
  const double qvz = dsub_(dmul(tvx, e1y), dmul(tvy, e1x));
  const double v = dmul(dadd(dadd(dmul(d[0], qvx), dmul(d[1], qvy)), dmul(d[2], qvz)), inv);
  if (v < 0.0 || dadd(u, v) > 1.0) return false;
  const double tt = dmul(dadd(dadd(dmul(e2x, qvx), dmul(e2y, qvy)), dmul(e2z, qvz)), inv);
  return tt > 1e-9 && tt < tmax;
}

// _kernels_nb.py:236-263
__device__ __forceinline__ bool box_hit(const BvhView& B, int nd, const double* o, const double* d,
                                        double tmax) {
  double tn = 0.0, tf = tmax;
#pragma unroll
  for (int ax = 0; ax < 3; ++ax) {
    const double lo = B.nmin[3 * nd + ax], hi = B.nmax[3 * nd + ax];
    if (d[ax] == 0.0) {
      if (o[ax] < lo || o[ax] > hi) return false;
    } else {
      const double inv = ddiv_(1.0, d[ax]);
      double ta = dmul(dsub_(lo, o[ax]), inv), tb = dmul(dsub_(hi, o[ax]), inv);
      if (ta > tb) { const double s = ta; ta = tb; tb = s; }
      if (ta > tn) tn = ta;
      if (tb < tf) tf = tb;
      if (tn > tf) return false;
    }
  }
  return tn <= tf;
}

// bvh_any_hit for one ray (_kernels_nb.py:267-298)
__device__ bool any_hit(const BvhView& B, const double* o, const double* d, double tmax) {
  int stack[64];
  int top = 1;
  stack[0] = 0;
  while (top > 0) {
    const int nd = stack[--top];
    if (!box_hit(B, nd, o, d, tmax)) continue;
    const int cnt = B.count[nd];
    if (cnt > 0) {
      const int st = B.start[nd];
      for (int t = st; t < st + cnt; ++t)
        if (tri_hit(B, t, o, d, tmax)) return true;
    } else if (top <= 62) {
      stack[top] = B.left[nd];
      stack[top + 1] = B.right[nd];
      top += 2;
    }
  }
  return false;
}

// numpy fresnel_transmittance (dipole.py:135-152) with the same operation order
__device__ __forceinline__ double ft_np(double eta, double ci) {
  ci = fmin(fmax(ci, 0.0), 1.0);
  if (eta == 1.0) return 1.0;
  const double sin2 = ddiv_(dsub_(1.0, dmul(ci, ci)), dmul(eta, eta));
  if (sin2 >= 1.0) return 0.0;
  const double ct = __dsqrt_rn(fmax(dsub_(1.0, sin2), 0.0));
  const double ect = dmul(eta, ct), eci = dmul(eta, ci);
  const double rs = ddiv_(dsub_(ci, ect), dadd(dadd(ci, ect), 1e-300));
  const double rp = ddiv_(dsub_(eci, ct), dadd(dadd(eci, ct), 1e-300));
  const double ft = dsub_(1.0, dmul(0.5, dadd(dmul(rs, rs), dmul(rp, rp))));
  return fmin(fmax(ft, 0.0), 1.0);
}

__device__ __forceinline__ double dot3(const double* a, const double* b) {
  return dadd(dadd(dmul(a[0], b[0]), dmul(a[1], b[1])), dmul(a[2], b[2]));
}

// lights: n x 12 doubles {kind, a[3], b[3], radius, ...}; material[6] = eta
__global__ void __launch_bounds__(128) k_direct_irradiance(
    int N, const float* __restrict__ positions, const float* __restrict__ normals, int n_lights,
    const double* __restrict__ lights, const double* __restrict__ material, double ray_offset,
    double bbox_diag, BvhView B, double* __restrict__ E) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  const double eta = material[6];
  const double p[3] = {(double)positions[3 * i], (double)positions[3 * i + 1],
                       (double)positions[3 * i + 2]};
  const double n[3] = {(double)normals[3 * i], (double)normals[3 * i + 1],
                       (double)normals[3 * i + 2]};
  const double o[3] = {dadd(p[0], dmul(ray_offset, n[0])), dadd(p[1], dmul(ray_offset, n[1])),
                       dadd(p[2], dmul(ray_offset, n[2]))};
  double e0 = 0.0, e1 = 0.0, e2 = 0.0;
  for (int l = 0; l < n_lights; ++l) {
    const double* L = lights + 12 * l;
    const int kind = (int)L[0];
    if (kind == 0) {  // point light
      const double dv[3] = {dsub_(L[1], p[0]), dsub_(L[2], p[1]), dsub_(L[3], p[2])};
      const double dist = __dsqrt_rn(dadd(dadd(dmul(dv[0], dv[0]), dmul(dv[1], dv[1])),
                                          dmul(dv[2], dv[2])));
      const double wi[3] = {ddiv_(dv[0], dist), ddiv_(dv[1], dist), ddiv_(dv[2], dist)};
      const double cs = dot3(n, wi);
      if (cs > 0.0 && !any_hit(B, o, wi, dist)) {
        const double c = fmin(fmax(cs, 0.0), 1.0);
        const double w = ddiv_(dmul(ft_np(eta, c), c), dmul(dist, dist));
        e0 = dadd(e0, dmul(w, L[4]));
        e1 = dadd(e1, dmul(w, L[5]));
        e2 = dadd(e2, dmul(w, L[6]));
      }
    } else if (kind == 1) {  // directional light
      const double wi[3] = {-L[1], -L[2], -L[3]};
      const double cs = dot3(n, wi);
      if (cs > 0.0 && !any_hit(B, o, wi, dadd(dmul(4.0, bbox_diag), 1.0))) {
        const double c = fmin(fmax(cs, 0.0), 1.0);
        const double w = dmul(ft_np(eta, c), c);
        e0 = dadd(e0, dmul(w, L[4]));
        e1 = dadd(e1, dmul(w, L[5]));
        e2 = dadd(e2, dmul(w, L[6]));
      }
    } else {  // sphere light: 8 x 8 midpoint-stratified cone (lighting.py:252-290)
      const double r = L[7];
      double ax[3] = {dsub_(L[1], p[0]), dsub_(L[2], p[1]), dsub_(L[3], p[2])};
      const double dist = __dsqrt_rn(dot3(ax, ax));
      ax[0] = ddiv_(ax[0], dist);
      ax[1] = ddiv_(ax[1], dist);
      ax[2] = ddiv_(ax[2], dist);
      const double sin_max = ddiv_(r, dist);
      const double cos_max = __dsqrt_rn(fmin(fmax(dsub_(1.0, dmul(sin_max, sin_max)), 0.0), 1.0));
      const double omega = dmul(2.0 * 3.141592653589793, dsub_(1.0, cos_max));
      const double hp[3] = {fabs(ax[2]) < 0.9 ? 0.0 : 1.0, 0.0, fabs(ax[2]) < 0.9 ? 1.0 : 0.0};
      double t1[3] = {dsub_(dmul(ax[1], hp[2]), dmul(ax[2], hp[1])),
                      dsub_(dmul(ax[2], hp[0]), dmul(ax[0], hp[2])),
                      dsub_(dmul(ax[0], hp[1]), dmul(ax[1], hp[0]))};
      const double tn = __dsqrt_rn(dot3(t1, t1));
      t1[0] = ddiv_(t1[0], tn);
      t1[1] = ddiv_(t1[1], tn);
      t1[2] = ddiv_(t1[2], tn);
      const double t2[3] = {dsub_(dmul(ax[1], t1[2]), dmul(ax[2], t1[1])),
                            dsub_(dmul(ax[2], t1[0]), dmul(ax[0], t1[2])),
                            dsub_(dmul(ax[0], t1[1]), dmul(ax[1], t1[0]))};
      const double rr = dsub_(dmul(dist, dist), dmul(r, r));
      double acc = 0.0;
      for (int s = 0; s < 64; ++s) {
        const double u1 = ((s >> 3) + 0.5) / 8.0, u2 = ((s & 7) + 0.5) / 8.0;
        const double ct = dsub_(1.0, dmul(u1, dsub_(1.0, cos_max)));
        const double st = __dsqrt_rn(fmin(fmax(dsub_(1.0, dmul(ct, ct)), 0.0), 1.0));
        const double phi = dmul(2.0 * 3.141592653589793, u2);
        double sp, cp;
        sincos(phi, &sp, &cp);
        const double a = dmul(st, cp), bsn = dmul(st, sp);
        const double dir[3] = {dadd(dadd(dmul(ax[0], ct), dmul(t1[0], a)), dmul(t2[0], bsn)),
                               dadd(dadd(dmul(ax[1], ct), dmul(t1[1], a)), dmul(t2[1], bsn)),
                               dadd(dadd(dmul(ax[2], ct), dmul(t1[2], a)), dmul(t2[2], bsn))};
        const double cs = dot3(n, dir);
        if (cs <= 0.0) continue;
        const double proj = dmul(dist, ct);
        const double under = dsub_(dmul(proj, proj), rr);
        const double t_hit = dsub_(proj, __dsqrt_rn(fmax(under, 0.0)));
        if (any_hit(B, o, dir, t_hit)) continue;
        const double c = fmin(fmax(cs, 0.0), 1.0);
        acc = dadd(acc, dmul(ft_np(eta, c), c));
      }
      const double w = dmul(ddiv_(acc, 64.0), omega);
      e0 = dadd(e0, dmul(w, L[4]));
      e1 = dadd(e1, dmul(w, L[5]));
      e2 = dadd(e2, dmul(w, L[6]));
    }
  }
  E[i] = e0;
  E[N + i] = e1;
  E[2 * (size_t)N + i] = e2;
}

}  // namespace sss
