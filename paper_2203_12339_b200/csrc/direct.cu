// Direct lights with shadow rays: irradiance_direct
// (lighting.py:208-290) with BVH any-hit visibility (lighting.py:101-176,
// _kernels_nb.py:208-298). 
//
// Ray / box / triangle tests and the point-light weights use explicit fp64
// round-to-nearest operations (no FMA contraction) in the reference's
// operation order, so visibility bits are those of the reference; the sphere
// light's stratified cone uses cos/sin (libm ulps) and a sequential mean.
// Output: E planar (3, N) doubles (the input of the w0 Haar + top-n path).
#include "sss_common.cuh"

namespace sss {

// Packed BVH: node records of 8 doubles {min[3], max[3], (int left, int
// right), (int start, int count)} (64 B, one L1 line pair), triangle records
// of 10 doubles {v0[3], e1[3], e2[3], pad} in leaf order.
struct BvhView {
  const double2* nodes;  // (M, 4) double2
  const double2* tris;   // (T, 5) double2
};

__device__ __forceinline__ double dsub_(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double ddiv_(double a, double b) { return __ddiv_rn(a, b); }

// a shadow ray: origin, direction and the per-axis 1/d the reference's slab
// test divides by (1.0 / d[ax] is the same value at every node, so it is
// computed once per ray; bitwise unchanged)
struct Ray {
  double o[3], d[3], inv[3];
  double tmax;
};

__device__ __forceinline__ void make_ray(Ray& R, const double* o, const double* d, double tmax) {
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    R.o[a] = o[a];
    R.d[a] = d[a];
    R.inv[a] = d[a] == 0.0 ? 0.0 : ddiv_(1.0, d[a]);
  }
  R.tmax = tmax;
}

// _kernels_nb.py:209-232 (Moller-Trumbore, det <= 1e-14 rejected, t > 1e-9).
// The reference scales each numerator by inv = 1 / det; the division is only
// needed near a decision boundary. A candidate is rejected early, without
// the division, when the numerator's sign or magnitude alone proves the
// reference's test fails (u = du * inv has du's sign times det's, and
// |u| >= |du / det| (1 - 2^-52) > 1 once |du| > |det| (1 + 1e-12)); the
// survivors run the reference's exact sequence, so the answer is unchanged.
__device__ __forceinline__ bool opposite(double num, double det) {
  return fabs(num) > 1e-200 && ((num < 0.0) != (det < 0.0));
}

__device__ __forceinline__ bool tri_hit(const BvhView& B, int t, const Ray& R) {
  const double2* q = B.tris + 5 * (size_t)t;
  const double2 a = __ldg(q), b = __ldg(q + 1), c = __ldg(q + 2), e = __ldg(q + 3),
                f = __ldg(q + 4);
  const double v0x = a.x, v0y = a.y, v0z = b.x, e1x = b.y, e1y = c.x, e1z = c.y;
  const double e2x = e.x, e2y = e.y, e2z = f.x;
  const double* d = R.d;
  const double pvx = dsub_(dmul(d[1], e2z), dmul(d[2], e2y));
  const double pvy = dsub_(dmul(d[2], e2x), dmul(d[0], e2z));
  const double pvz = dsub_(dmul(d[0], e2y), dmul(d[1], e2x));
  const double det = dadd(dadd(dmul(e1x, pvx), dmul(e1y, pvy)), dmul(e1z, pvz));
  if (fabs(det) <= 1e-14) return false;
  const double adet = fabs(det) * (1.0 + 1e-12);
  const double tvx = dsub_(R.o[0], v0x), tvy = dsub_(R.o[1], v0y), tvz = dsub_(R.o[2], v0z);
  const double du = dadd(dadd(dmul(tvx, pvx), dmul(tvy, pvy)), dmul(tvz, pvz));
  if (opposite(du, det) || fabs(du) > adet) return false;
  const double qvx = dsub_(dmul(tvy, e1z), dmul(tvz, e1y));
  const double qvy = dsub_(dmul(tvz, e1x), dmul(tvx, e1z));
  const double qvz = dsub_(dmul(tvx, e1y), dmul(tvy, e1x));
  const double dv = dadd(dadd(dmul(d[0], qvx), dmul(d[1], qvy)), dmul(d[2], qvz));
  if (opposite(dv, det) || fabs(du) + fabs(dv) > fabs(det) * (1.0 + 1e-9)) return false;
  const double dt = dadd(dadd(dmul(e2x, qvx), dmul(e2y, qvy)), dmul(e2z, qvz));
  if (opposite(dt, det)) return false;
  // the reference's exact tests
  const double inv = ddiv_(1.0, det);
  const double u = dmul(du, inv);
  if (u < 0.0 || u > 1.0) return false;
  const double v = dmul(dv, inv);
  if (v < 0.0 || dadd(u, v) > 1.0) return false;
  const double tt = dmul(dt, inv);
  return tt > 1e-9 && tt < R.tmax;
}

// _kernels_nb.py:236-263 (slab test; an axis with d == 0 tests the origin)
__device__ __forceinline__ bool box_hit(const double* lo, const double* hi, const Ray& R) {
  double tn = 0.0, tf = R.tmax;
#pragma unroll
  for (int ax = 0; ax < 3; ++ax) {
    if (R.d[ax] == 0.0) {
      if (R.o[ax] < lo[ax] || R.o[ax] > hi[ax]) return false;
    } else {
      double ta = dmul(dsub_(lo[ax], R.o[ax]), R.inv[ax]);
      double tb = dmul(dsub_(hi[ax], R.o[ax]), R.inv[ax]);
      if (ta > tb) { const double s = ta; ta = tb; tb = s; }
      if (ta > tn) tn = ta;
      if (tb < tf) tf = tb;
      if (tn > tf) return false;
    }
  }
  return tn <= tf;
}

__device__ __forceinline__ bool node_box_hit(const BvhView& B, int nd, const Ray& R) {
  const double2* q = B.nodes + 4 * (size_t)nd;
  const double2 a = __ldg(q), b = __ldg(q + 1), c = __ldg(q + 2);
  const double lo[3] = {a.x, a.y, b.x}, hi[3] = {b.y, c.x, c.y};
  return box_hit(lo, hi, R);
}

// bvh_any_hit for one ray (_kernels_nb.py:267-298), below node `root` (whose
// box is already hit). The answer does not depend on the visiting order or on
// where a box is tested, so both children of an inner node are tested
// together (two independent 64-byte loads in flight) and only the hit ones
// are pushed; the stack holds nodes whose box is hit. `cancel` (shared
// memory, may be null) is polled per pop: another thread of the same ray
// found a hit.
__device__ bool any_hit_from(const BvhView& B, const Ray& R, int root, const volatile int* cancel) {
  int stack[64];
  int top = 1;
  stack[0] = root;
  while (top > 0) {
    if (cancel && *cancel) return false;
    const int nd = stack[--top];
    const double2 e = __ldg(B.nodes + 4 * (size_t)nd + 3);
    const int left = __double2loint(e.x), right = __double2hiint(e.x);
    const int start = __double2loint(e.y), count = __double2hiint(e.y);
    if (count > 0) {
      for (int t = start; t < start + count; ++t)
        if (tri_hit(B, t, R)) return true;
    } else {
      const bool hl = node_box_hit(B, left, R), hr = node_box_hit(B, right, R);
      if (hr && top < 64) stack[top++] = right;
      if (hl && top < 64) stack[top++] = left;
    }
  }
  return false;
}

__device__ __forceinline__ bool any_hit(const BvhView& B, const Ray& R) {
  return node_box_hit(B, 0, R) && any_hit_from(B, R, 0, nullptr);
}

// Part `g` of 2^SPLIT of one ray's any-hit: the subtree reached from the root
// by the SPLIT bits of g (a leaf met on the way belongs to the part whose
// remaining bits are zero). The OR over the parts is the ray's answer.
template <int SPLIT>
__device__ __forceinline__ bool any_hit_part(const BvhView& B, const Ray& R, int g,
                                             const volatile int* cancel) {
  int nd = 0;
#pragma unroll
  for (int lev = 0; lev < SPLIT; ++lev) {
    if (!node_box_hit(B, nd, R)) return false;
    const double2 e = __ldg(B.nodes + 4 * (size_t)nd + 3);
    if (__double2hiint(e.y) > 0) {  // leaf above the split depth
      if (g & ((1 << (SPLIT - lev)) - 1)) return false;
      return any_hit_from(B, R, nd, cancel);
    }
    nd = ((g >> (SPLIT - 1 - lev)) & 1) ? __double2hiint(e.x) : __double2loint(e.x);
  }
  return node_box_hit(B, nd, R) && any_hit_from(B, R, nd, cancel);
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

template <typename PT>
__device__ __forceinline__ void load_point(int i, const PT* __restrict__ positions,
                                           const PT* __restrict__ normals, double ray_offset,
                                           double* p, double* n, double* o) {
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    p[a] = (double)positions[3 * i + a];
    n[a] = (double)normals[3 * i + a];
    o[a] = dadd(p[a], dmul(ray_offset, n[a]));
  }
}

// E[c] += w * L[c] in light order (the reference's per-light accumulation,
// lighting.py:229-290; E starts at exact zeros, so the first light's sum is
// its own product)
__device__ __forceinline__ void add_light(double* E, int N, int i, double w, const double* L) {
  E[i] = dadd(E[i], dmul(w, L[4]));
  E[N + i] = dadd(E[N + i], dmul(w, L[5]));
  E[2 * (size_t)N + i] = dadd(E[2 * (size_t)N + i], dmul(w, L[6]));
}

// point (kind 0) or directional (kind 1) light: one shadow ray per sample
// (lighting.py:229-251); L = 12 doubles {kind, a[3], b[3], radius, ...}.
// 2^SPLIT threads share a ray (any_hit_part): a single light has only one ray
// per sample, so this is where the parallelism comes from.
constexpr int kDirectThreads = 128;

template <int KIND, int SPLIT, typename PT = float>
__global__ void __launch_bounds__(kDirectThreads) k_direct_single(
    int N, const PT* __restrict__ positions, const PT* __restrict__ normals,
    const double* __restrict__ Lp, const double* __restrict__ material, double ray_offset,
    double bbox_diag, BvhView B, double* __restrict__ E) {
  constexpr int P = 1 << SPLIT;
  __shared__ int found[kDirectThreads / P];
  const int r = threadIdx.x >> SPLIT, g = threadIdx.x & (P - 1);
  const int i = blockIdx.x * (kDirectThreads / P) + r;
  if (g == 0) found[r] = 0;
  __syncthreads();
  double L[7];
#pragma unroll
  for (int q = 0; q < 7; ++q) L[q] = Lp[q];
  bool lit = false;
  double w = 0.0;
  if (i < N) {
    const double eta = material[6];
    double p[3], n[3], o[3];
    load_point(i, positions, normals, ray_offset, p, n, o);
    double wi[3], tmax, dist2 = 1.0;
    if (KIND == 0) {
      const double dv[3] = {dsub_(L[1], p[0]), dsub_(L[2], p[1]), dsub_(L[3], p[2])};
      const double dist = __dsqrt_rn(dadd(dadd(dmul(dv[0], dv[0]), dmul(dv[1], dv[1])),
                                          dmul(dv[2], dv[2])));
      wi[0] = ddiv_(dv[0], dist);
      wi[1] = ddiv_(dv[1], dist);
      wi[2] = ddiv_(dv[2], dist);
      tmax = dist;
      dist2 = dmul(dist, dist);
    } else {
      wi[0] = -L[1];
      wi[1] = -L[2];
      wi[2] = -L[3];
      tmax = dadd(dmul(4.0, bbox_diag), 1.0);
    }
    const double cs = dot3(n, wi);
    if (cs > 0.0) {
      Ray R;
      make_ray(R, o, wi, tmax);
      const bool hit = SPLIT == 0 ? any_hit(B, R) : any_hit_part<SPLIT>(B, R, g, &found[r]);
      if (hit) found[r] = 1;
      lit = true;
      const double c = fmin(fmax(cs, 0.0), 1.0);
      w = KIND == 0 ? ddiv_(dmul(ft_np(eta, c), c), dist2) : dmul(ft_np(eta, c), c);
    }
  }
  __syncthreads();
  if (g == 0 && lit && !found[r]) add_light(E, N, i, w, L);
}

// sphere light (kind 2): 8 x 8 midpoint-stratified cone (lighting.py:252-290).
// One thread per (sample, stratum): a CTA holds kSpherePts samples x 64
// strata, the 32 lanes of a warp trace 32 strata of one sample (a narrow,
// coherent cone); per-stratum terms meet in shared memory and one thread sums
// them in stratum order (the reference's sequential mean).
constexpr int kSpherePts = 4;

template <typename PT = float>
__global__ void __launch_bounds__(64 * kSpherePts) k_direct_sphere(
    int N, const PT* __restrict__ positions, const PT* __restrict__ normals,
    const double* __restrict__ Lp, const double* __restrict__ material, double ray_offset,
    BvhView B, double* __restrict__ E) {
  __shared__ double term[kSpherePts][64];
  const int s = threadIdx.x & 63, j = threadIdx.x >> 6;
  const int i = blockIdx.x * kSpherePts + j;
  double L[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) L[q] = Lp[q];
  const double eta = material[6];
  double contrib = 0.0, omega = 0.0;
  if (i < N) {
    double p[3], n[3], o[3];
    load_point(i, positions, normals, ray_offset, p, n, o);
    const double r = L[7];
    double ax[3] = {dsub_(L[1], p[0]), dsub_(L[2], p[1]), dsub_(L[3], p[2])};
    const double dist = __dsqrt_rn(dot3(ax, ax));
    ax[0] = ddiv_(ax[0], dist);
    ax[1] = ddiv_(ax[1], dist);
    ax[2] = ddiv_(ax[2], dist);
    const double sin_max = ddiv_(r, dist);
    const double cos_max = __dsqrt_rn(fmin(fmax(dsub_(1.0, dmul(sin_max, sin_max)), 0.0), 1.0));
    omega = dmul(2.0 * 3.141592653589793, dsub_(1.0, cos_max));
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
    if (cs > 0.0) {
      const double proj = dmul(dist, ct);
      const double under = dsub_(dmul(proj, proj), rr);
      const double t_hit = dsub_(proj, __dsqrt_rn(fmax(under, 0.0)));
      Ray R;
      make_ray(R, o, dir, t_hit);
      if (!any_hit(B, R)) {
        const double c = fmin(fmax(cs, 0.0), 1.0);
        contrib = dmul(ft_np(eta, c), c);
      }
    }
  }
  term[j][s] = contrib;
  __syncthreads();
  if (s == 0 && i < N) {
    double acc = 0.0;
    for (int q = 0; q < 64; ++q) acc = dadd(acc, term[j][q]);  // skipped strata add exact 0
    add_light(E, N, i, dmul(ddiv_(acc, 64.0), omega), L);
  }
}

}  // namespace sss
