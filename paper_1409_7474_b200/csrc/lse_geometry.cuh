// lse_geometry.cuh -- work decomposition of the fused kernels (host + device).
//
// Kept free of CUDA-only constructs so the host driver and a plain C++ unit
// test (tests/test_geometry.py) share the exact code the kernels run.
#pragma once
#ifdef __CUDACC__
#define LSE_HD __host__ __device__ __forceinline__
#else
#define LSE_HD inline
#endif

namespace lse {

// Work geometry of one kernel family (update or partition).
//  interior work: (1) chunks -- word-rows [r_lo, r_hi) x c in [0, nci), chunk c
//  = columns [xoff + 256c, xoff + 256c + 256), one warp each; (2) "B1" lane
//  groups -- the 8-column groups of the right strip [x1, W) of interior rows
//  whose stencil still lies inside the image, packed 32 per warp (each lane
//  its own row); every lane of (1)/(2) runs the interior code.
//  border work: (A) word-rows outside [r_lo, r_hi) -- the blocks [ta, tb) and
//  [ba, bb) -- whole width; (B2) per interior row the left strip [0, xoff)
//  and the right tail beyond the B1 groups.  Border work runs the slower
//  zero-padding code, so its units are short: a border warp unit holds
//  bitems = 32 / bq 8-column lane groups and each group's 32 rows are split
//  over bq lanes of 32 / bq rows (lane = part * bitems + item); bq = 4 by
//  default, 8 or 16 for small images whose border units are the critical
//  path.  A row strip of a
//  multi-GPU run drops the border rows it does not own (its halo rows,
//  recomputed by their owner).
constexpr int kBorderQ = 4;                      // default row parts per border lane group
struct Geo {
  int bq, bitems;    // border row parts per lane group; lane groups (= rows per lane) per unit
  int r_lo, r_hi, nci, xoff, x1;
  int ta, tb, ba, bb;  // part-A word-rows: [ta, tb) above and [ba, bb) below the interior
  int na_row;        // part-A warp units per word-row: ceil(ceil(W / 8) / bitems)
  int nb1_row;       // B1 lane groups per interior row
  int nb2_left;      // B2 left-strip groups per interior row (xoff / 8)
  int nb2_row;       // B2 lane groups per interior row (left + right tail)
  int nA;            // part-A warp units
  int nB1, nB2;      // lane groups
};

// Build the geometry of a kernel whose stencil reaches `top` rows up, `bot`
// rows down and `right` columns right (the left reach must be <= xoff = 8).
LSE_HD long long geo_fdiv(long long a, long long b) { return a >= 0 ? a / b : -((-a + b - 1) / b); }
LSE_HD Geo make_geo(int H, int W, int R, int top, int bot, int right, int bq = kBorderQ) {
  const int HR = (H + 31) / 32;
  Geo g{};
  g.bq = bq;
  g.bitems = 32 / bq;
  g.xoff = 8;
  g.na_row = ((W + 7) / 8 + g.bitems - 1) / g.bitems;
  long long rlo = (top + 31) / 32;
  long long rhi = geo_fdiv(H - 32 - bot, 32) + 1;
  if (rhi > HR) rhi = HR;
  long long nci = geo_fdiv(W - 1 - right - 255 - g.xoff, 256) + 1;
  if (R > 7 || rlo >= rhi || nci <= 0) { rlo = rhi = 0; nci = 0; }
  g.r_lo = (int)rlo;
  g.r_hi = (int)rhi;
  g.nci = (int)nci;
  g.x1 = g.xoff + 256 * g.nci;
  const int ngr = g.nci > 0 ? (W - g.x1 + 7) / 8 : 0;           // right-strip groups
  long long nb1 = g.nci > 0 ? geo_fdiv(W - 8 - right - g.x1, 8) + 1 : 0;
  if (nb1 < 0) nb1 = 0;
  if (nb1 > ngr) nb1 = ngr;
  g.nb1_row = (int)nb1;
  g.nb2_left = g.nci > 0 ? g.xoff / 8 : 0;
  g.nb2_row = g.nb2_left + (ngr - g.nb1_row);
  g.ta = 0;
  g.tb = g.r_lo;
  g.ba = g.r_hi;
  g.bb = HR;
  g.nA = (g.tb - g.ta + g.bb - g.ba) * g.na_row;
  g.nB1 = (g.r_hi - g.r_lo) * g.nb1_row;
  g.nB2 = (g.r_hi - g.r_lo) * g.nb2_row;
  return g;
}

// Row strips: only the word-rows [own_lo, own_hi) are computed.  Returns false
// if an interior row falls outside them (the strip is then unsupported).
LSE_HD bool geo_restrict_rows(Geo& g, int own_lo, int own_hi) {
  if (g.r_lo < g.r_hi && (g.r_lo < own_lo || g.r_hi > own_hi)) return false;
  g.ta = g.ta > own_lo ? g.ta : own_lo;
  g.tb = g.tb < own_hi ? g.tb : own_hi;
  if (g.tb < g.ta) g.tb = g.ta;
  g.ba = g.ba > own_lo ? g.ba : own_lo;
  g.bb = g.bb < own_hi ? g.bb : own_hi;
  if (g.bb < g.ba) g.bb = g.ba;
  g.nA = (g.tb - g.ta + g.bb - g.ba) * g.na_row;
  return true;
}

// the same geometry with no interior (every unit runs the border code)
LSE_HD Geo geo_all_border(const Geo& in, int H) {
  Geo g = in;
  g.r_lo = g.r_hi = 0;
  g.nci = 0;
  g.nb1_row = g.nb2_row = g.nb2_left = 0;
  g.ta = 0;
  g.tb = (H + 31) / 32;
  g.ba = g.bb = g.tb;
  g.nA = ((H + 31) / 32) * g.na_row;
  g.nB1 = g.nB2 = 0;
  return g;
}

// Unit -> lane coordinates.
LSE_HD int chunk_units(const Geo& G) { return (G.r_hi - G.r_lo) * G.nci; }
LSE_HD int interior_units(const Geo& G) {
  return chunk_units(G) + (G.nB1 + 31) / 32;
}
LSE_HD int border_units(const Geo& G) {
  return G.nA + (G.nB2 + G.bitems - 1) / G.bitems;
}
// B1 pack: lane -> (row, x0); false for the unused lanes of the last pack
LSE_HD bool b1_lane(const Geo& G, int pack, int lane, int& r, int& x0) {
  const int g = pack * 32 + lane;
  if (g >= G.nB1) return false;
  r = G.r_lo + g / G.nb1_row;
  x0 = G.x1 + 8 * (g - (r - G.r_lo) * G.nb1_row);
  return true;
}
// Border unit -> the lane group (r, x0) of `lane` (its row part is
// lane / bitems); false for the unused lanes of the last unit.
LSE_HD bool border_lane(const Geo& G, int unit, int lane, int W, int& r,
                                            int& x0) {
  const int item = lane % G.bitems;
  if (unit < G.nA) {
    const int rowidx = unit / G.na_row;
    const int c = unit - rowidx * G.na_row;
    const int ntop = G.tb - G.ta;
    r = rowidx < ntop ? G.ta + rowidx : G.ba + (rowidx - ntop);
    x0 = (c * G.bitems + item) * 8;
    return x0 < W;
  }
  const int g = (unit - G.nA) * G.bitems + item;
  if (g >= G.nB2) return false;
  r = G.r_lo + g / G.nb2_row;
  const int j = g - (r - G.r_lo) * G.nb2_row;
  x0 = j < G.nb2_left ? 8 * j : G.x1 + 8 * (G.nb1_row + j - G.nb2_left);
  return true;
}

}  // namespace lse
