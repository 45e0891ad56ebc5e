/* A plain C caller of the C ABI (include/lse_b200.h): the region evolution of
 * a synthetic two-region image from a square seed, exactly what
 * `lsekit.run(image, SeedSpec(...), default_params(ModelKind.REGION))` does
 * (engine.py:272-277).  Prints "iterations converged mask-hash" so tests can
 * compare it with the Python API.  Build:
 *   gcc -O2 -Iinclude examples/c_abi_region.c -Lpaper_1409_7474_b200/_lib -llse_b200 -lm */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "lse_b200.h"

/* gaussian_kernel(sigma, ts).axis_weights (kernels.py:50-64): exp(-x^2 / 2s^2)
 * over x = k - (ts-1)/2, divided by its sum (numpy's pairwise order for
 * ts <= 15: eight partial sums combined as a tree, then the tail). */
static void gaussian_axis(double sigma, int ts, double* w) {
  const double c = (ts - 1) / 2.0;
  for (int k = 0; k < ts; ++k) {
    const double x = (double)k - c;
    w[k] = exp(-(x * x) / (2.0 * sigma * sigma));
  }
  double s = 0.0;
  if (ts < 8) {
    for (int k = 0; k < ts; ++k) s += w[k];
  } else {
    s = ((w[0] + w[1]) + (w[2] + w[3])) + ((w[4] + w[5]) + (w[6] + w[7]));
    for (int k = 8; k < ts; ++k) s += w[k];
  }
  for (int k = 0; k < ts; ++k) w[k] /= s;
}

int main(void) {
  const int H = 128, W = 128;
  double* img = malloc(sizeof(double) * H * W);
  for (int i = 0; i < H; ++i)
    for (int x = 0; x < W; ++x) img[i * W + x] = (i >= 40 && i < 88 && x >= 40 && x < 88) ? 0.2 : 0.8;
  double wreg[9], wpre[9];
  gaussian_axis(1.0, 9, wreg);
  gaussian_axis(1.0, 9, wpre);
  lse_params p = {0};
  p.model = LSE_MODEL_REGION;
  p.dt = 15.0;
  p.sigma2 = 1.0;
  p.ts_reg = 9;
  p.reinit_period = 1;
  p.reg_period = 1;
  p.max_iters = 300;
  p.conv_check_every = 10;
  p.conv_window = 3;
  p.sigma1 = 1.0;
  p.ts_pre = 9;
  p.edge_gain = 255.0;
  p.reg_weights = wreg;
  p.pre_weights = wpre;
  p.nu = 1.0;
  p.mu = 0.1;
  const double square[8] = {14, 14, 76, 14, 76, 76, 14, 76};
  const long long counts[1] = {4};
  lse_phi0 init = {0};
  init.kind = LSE_PHI0_POLYGONS;
  init.poly_xy = square;
  init.poly_counts = counts;
  init.n_polys = 1;
  init.inside_sign = -1;
  lse_run* run = NULL;
  if (lse_run_create(&run, &p, H, W, img, LSE_IMAGE_F64, &init) != LSE_OK) {
    fprintf(stderr, "create: %s\n", lse_last_error());
    return 1;
  }
  lse_status st;
  if (lse_run_advance(run, p.max_iters, &st) != LSE_OK) {
    fprintf(stderr, "advance: %s\n", lse_last_error());
    return 1;
  }
  unsigned char* mask = malloc(H * W);
  lse_run_read_mask(run, mask, -1, 0);
  uint64_t hsh = 1469598103934665603ull;             /* FNV-1a of the 0/1 mask */
  for (int q = 0; q < H * W; ++q) hsh = (hsh ^ mask[q]) * 1099511628211ull;
  printf("%lld %d %016llx\n", st.iteration, st.converged, (unsigned long long)hsh);
  lse_run_destroy(run);
  free(mask);
  free(img);
  return 0;
}
