// Host-side check of the fused kernels' work decomposition (lse_geometry.cuh):
// every (word-row, 8-column group) of the image is covered exactly once, and
// every lane given to the interior code has its whole stencil inside the image.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_1409_7474_b200/csrc/lse_geometry.cuh"
using namespace lse;

static int check(int H, int W, int R, int top, int bot, int left, int right, const Geo& G,
                 int own_lo = 0, int own_hi = 1 << 30) {
  const int HR = (H + 31) / 32, NG = (W + 7) / 8;
  std::vector<int> cover((size_t)HR * NG, 0);
  int bad = 0;
  auto interior_ok = [&](int r, int x0) {
    return 32 * r - top >= 0 && 32 * r + 31 + bot <= H - 1 && x0 - left >= 0 &&
           x0 + 7 + right <= W - 1;
  };
  // interior: chunks
  for (int u = 0; u < chunk_units(G); ++u)
    for (int lane = 0; lane < 32; ++lane) {
      const int r = G.r_lo + u / G.nci;
      const int x0 = G.xoff + (u % G.nci) * 256 + 8 * lane;
      if (!interior_ok(r, x0)) { ++bad; }
      if (x0 < W) cover[(size_t)r * NG + x0 / 8]++;
    }
  for (int pk = 0; pk < (G.nB1 + 31) / 32; ++pk)
    for (int lane = 0; lane < 32; ++lane) {
      int r, x0;
      if (!b1_lane(G, pk, lane, r, x0)) continue;
      if (!interior_ok(r, x0)) { ++bad; }
      cover[(size_t)r * NG + x0 / 8]++;
    }
  for (int u = 0; u < border_units(G); ++u)
    for (int lane = 0; lane < G.bitems; ++lane) {   // row part 0 stands for its group
      int r, x0;
      if (!border_lane(G, u, lane, W, r, x0)) continue;
      if (r < 0 || r >= HR || x0 < 0 || x0 >= W || x0 % 8) { ++bad; continue; }
      cover[(size_t)r * NG + x0 / 8]++;
    }
  for (size_t k = 0; k < cover.size(); ++k) {
    const int r = (int)(k / NG);
    if (cover[k] != ((r >= own_lo && r < own_hi) ? 1 : 0)) ++bad;
  }
  if (bad) printf("FAIL H=%d W=%d R=%d reach=(%d,%d,%d,%d): %d problems\n", H, W, R, top, bot,
                  left, right, bad);
  return bad;
}

int main() {
  int fails = 0, cases = 0;
  const int Hs[] = {2, 3, 31, 32, 33, 64, 70, 96, 127, 256, 300, 1024, 4097};
  const int Ws[] = {2, 7, 8, 9, 255, 256, 257, 264, 270, 512, 530, 1024, 1300, 4096, 32768};
  for (int H : Hs)
    for (int W : Ws)
      for (int R = 1; R <= 4; ++R)
      for (int bq = 4; bq <= 16; bq *= 2) {
        fails += check(H, W, R, 1 + R, 1 + R, R + 1, R + 1, make_geo(H, W, R, 1 + R, 1 + R, R + 1, bq)) != 0;
        fails += check(H, W, R, R, R, R, R, make_geo(H, W, R, R, R, R, bq)) != 0;
        Geo a = geo_all_border(make_geo(H, W, R, 1 + R, 1 + R, R + 1, bq), H);
        fails += check(H, W, R, 1 << 20, 1 << 20, 1 << 20, 1 << 20, a) != 0;
        cases += 3;
        // row strips: halo word-rows (first / last) are left to their owners
        const int HR = (H + 31) / 32;
        for (int lo = 0; lo <= 1; ++lo)
          for (int hi = HR - 1; hi <= HR; ++hi) {
            if (hi <= lo) continue;
            Geo s = make_geo(H, W, R, 1 + R, 1 + R, R + 1, bq);
            if (!geo_restrict_rows(s, lo, hi)) continue;
            fails += check(H, W, R, 1 + R, 1 + R, R + 1, R + 1, s, lo, hi) != 0;
            Geo q = make_geo(H, W, R, R, R, R, bq);
            if (!geo_restrict_rows(q, lo, hi)) continue;
            fails += check(H, W, R, R, R, R, R, q, lo, hi) != 0;
            cases += 2;
          }
      }
  printf("%d cases, %d failing\n", cases, fails);
  return fails != 0;
}
