// One shadow ray through the packed BVH on the GPU, logging every popped
// node with its box result and every tested triangle: tools only.
#include "../paper_2203_12339_b200/csrc/direct.cu"

namespace {
__global__ void k_probe(sss::BvhView B, const double* ray, int* log, int cap) {
  sss::Ray R;
  sss::make_ray(R, ray, ray + 3, ray[6]);
  int stack[64], top = 1, n = 0;
  stack[0] = 0;
  while (top > 0 && n + 2 < cap) {
    const int nd = stack[--top];
    const double2* q = B.nodes + 4 * (size_t)nd;
    const double2 a = q[0], b = q[1], c = q[2], e = q[3];
    const double lo[3] = {a.x, a.y, b.x}, hi[3] = {b.y, c.x, c.y};
    const bool h = sss::box_hit(lo, hi, R);
    log[n++] = h ? nd : -1 - nd;
    if (!h) continue;
    const int l = __double2loint(e.x), r = __double2hiint(e.x), st = __double2loint(e.y),
              cn = __double2hiint(e.y);
    if (cn > 0) {
      for (int t = st; t < st + cn && n < cap; ++t) log[n++] = sss::tri_hit(B, t, R) ? 1000000 + t : 2000000 + t;
    } else {
      stack[top] = r;
      stack[top + 1] = l;
      top += 2;
    }
  }
  log[n] = -999999999;
}
}  // namespace

extern "C" int direct_probe(const double* nodes, const double* tris, const double* ray, int* log,
                            int cap) {
  const sss::BvhView B{reinterpret_cast<const double2*>(nodes), reinterpret_cast<const double2*>(tris)};
  k_probe<<<1, 1>>>(B, ray, log, cap);
  cudaDeviceSynchronize();
  return (int)cudaGetLastError();
}
