// Layout pass v26 for the flat16 stream: align duplicate columns inside each
// warp iteration so that their x gathers share one L1 wavefront.
//
// A flat16 warp iteration ("window") holds 32 lanes x 16 entries; lane j owns
// 16 entries of one (row, k) segment, in any slot order (the lane's partial
// sum does not depend on it). Consecutive segments of a window are the same
// receiver row's neighbouring terms k, whose column sets overlap (a (row,
// column) pair carries 2.7 of the 8 terms): up to 24 % of a window's kept
// entries repeat a column of another segment (tools/window_dup_stats.py). A
// gather instruction (slot e across the 32 lanes) costs one wavefront per
// distinct x address, so placing the copies of a column in the same slot of
// their segments' lanes shares that wavefront. Greedy per window, one thread:
// walk the window's columns in ascending order (a merge of its segments'
// sorted entry lists); a column present in m >= 2 segments gets the lowest
// slot free in some lane of every one of them; the rest of each segment's
// entries then fill its remaining free slots. Head flags and segment ids do
// not change (lanes keep their segments).
#include "sss_common.cuh"

namespace sss {

__global__ void __launch_bounds__(64) k_flat_align(unsigned n_words, unsigned n_groups,
                                                   const uint32_t* __restrict__ cin,
                                                   const float* __restrict__ vin,
                                                   const uint32_t* __restrict__ heads,
                                                   uint32_t sentinel, uint32_t* __restrict__ cout,
                                                   float* __restrict__ vout) {
  constexpr int E = 16, W = 32 * E;
  const unsigned w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= n_words) return;
  const size_t base = (size_t)w * W;
  const uint32_t h = heads[w];
  // lane ranges of the window's segments (the last window may be partial)
  const int nl = (int)min(32u, n_groups - w * 32u);
  int seg_lo[33], nseg = 0;
  for (int j = 0; j < nl; ++j)
    if (j == 0 || ((h >> j) & 1u)) seg_lo[nseg++] = j;
  seg_lo[nseg] = nl;
  uint16_t freem[32];
  for (int j = 0; j < 32; ++j) freem[j] = 0xffffu;
  uint32_t done[W / 32];
  for (int q = 0; q < W / 32; ++q) done[q] = 0u;
  // merge cursors: the segment's entries in ascending column order are
  // (slot e, lane l0 .. l1-1) for e = 0..15
  int cur[32];
  for (int s = 0; s < nseg; ++s) cur[s] = 0;
  auto entry_of = [&](int s, int r) {  // r-th entry of segment s in sorted order
    const int L = seg_lo[s + 1] - seg_lo[s];
    return (seg_lo[s] + r % L) * E + r / L;  // window-local index lane * 16 + slot
  };
  for (;;) {
    uint32_t cmin = 0xffffffffu;
    for (int s = 0; s < nseg; ++s) {
      const int L = seg_lo[s + 1] - seg_lo[s];
      if (cur[s] < L * E) {
        const uint32_t c = cin[base + entry_of(s, cur[s])];
        if (c < cmin) cmin = c;
      }
    }
    if (cmin >= sentinel) break;  // only padding (or nothing) left
    // segments holding cmin at their cursor
    int mem[32], nm = 0;
    for (int s = 0; s < nseg; ++s) {
      const int L = seg_lo[s + 1] - seg_lo[s];
      if (cur[s] < L * E && cin[base + entry_of(s, cur[s])] == cmin) mem[nm++] = s;
    }
    if (nm >= 2) {
      unsigned common = 0xffffu;
      for (int i = 0; i < nm; ++i) {
        unsigned sf = 0;
        for (int j = seg_lo[mem[i]]; j < seg_lo[mem[i] + 1]; ++j) sf |= freem[j];
        common &= sf;
      }
      if (common) {
        const int e = __ffs(common) - 1;
        for (int i = 0; i < nm; ++i) {
          const int s = mem[i];
          int lane = seg_lo[s];
          while (!((freem[lane] >> e) & 1u)) ++lane;
          freem[lane] &= (uint16_t)~(1u << e);
          const int src = entry_of(s, cur[s]);
          done[src >> 5] |= 1u << (src & 31);
          cout[base + lane * E + e] = cmin;
          vout[base + lane * E + e] = vin[base + src];
        }
      }
    }
    for (int i = 0; i < nm; ++i) ++cur[mem[i]];
  }
  // every other entry (singletons, unplaced duplicates, padding) fills its
  // segment's remaining free slots, both in the original interleaved order
  // (sorted entries, slot-major over the lanes): consecutive sorted columns of
  // a segment stay in one gather instruction, the locality flat16 relies on
  for (int s = 0; s < nseg; ++s) {
    const int l0 = seg_lo[s], L = seg_lo[s + 1] - l0;
    int pos = 0;  // next free position, slot-major: (pos / L, l0 + pos % L)
    for (int r = 0; r < L * E; ++r) {
      const int src = entry_of(s, r);
      if ((done[src >> 5] >> (src & 31)) & 1u) continue;
      int lane = l0 + pos % L, e = pos / L;
      while (!((freem[lane] >> e) & 1u)) { ++pos; lane = l0 + pos % L; e = pos / L; }
      ++pos;
      freem[lane] &= (uint16_t)~(1u << e);
      cout[base + lane * E + e] = cin[base + src];
      vout[base + lane * E + e] = vin[base + src];
    }
  }
}

}  // namespace sss
