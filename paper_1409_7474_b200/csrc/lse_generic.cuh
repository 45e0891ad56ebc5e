// lse_generic.cuh -- exact fp64 field kernels.
//
// These carry a float64 phi field through _advance_once step by step, in
// the reference's operation order, for the iterations the binary-state path
// cannot represent: reinit_period != 1 or reg_period != 1 (engine.py:160-169),
// an injected non-binary state, template sizes outside 3..9, or inputs
// outside the fp32 guard's range (huge dt / intensities).  They also
// implement the stateless public kernels (edge_function, convolve_same,
// gradients, velocities) and the one-time setup passes (seed rasterization,
// image statistics, edge indicator).
#pragma once
#include "lse_device.cuh"
#include "lse_fast.cuh"

namespace lse {

// Separable correlation pass, scipy order (kernels.py:72-76 ->
// scipy NI_Correlate1D symmetric branch), zero padding.
// AXIS 0: along rows (vertical), AXIS 1: along columns (horizontal).
template <int AXIS>
__global__ void k_corr(const double* __restrict__ in, double* __restrict__ out, int H, int W,
                       const double* __restrict__ w, int R) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y;
  if (x >= W) return;
  auto f = [&](int ii, int xx) -> double {
    if (AXIS == 0) return (ii < 0 || ii >= H) ? 0.0 : in[(size_t)ii * W + xx];
    return (xx < 0 || xx >= W) ? 0.0 : in[(size_t)ii * W + xx];
  };
  double acc = dmul(f(i, x), w[0]);
  for (int d = R; d >= 1; --d) {
    double l = AXIS == 0 ? f(i - d, x) : f(i, x - d);
    double r = AXIS == 0 ? f(i + d, x) : f(i, x + d);
    acc = dadd(acc, dmul(dadd(l, r), w[d]));
  }
  out[(size_t)i * W + x] = acc;
}

// full 2-D correlation (ndimage.correlate, mode constant 0): footprint of the
// non-zero weights, row-major order
__global__ void k_corr2d(const double* __restrict__ in, double* __restrict__ out, int H, int W,
                         const double* __restrict__ w2, int ts) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y;
  if (x >= W) return;
  const int R = ts / 2;
  double acc = 0.0;
  bool first = true;
  for (int a = 0; a < ts; ++a)
    for (int b = 0; b < ts; ++b) {
      const double wv = w2[a * ts + b];
      if (wv == 0.0) continue;
      const int ii = i + a - R, xx = x + b - R;
      const double v = (ii < 0 || ii >= H || xx < 0 || xx >= W) ? 0.0 : in[(size_t)ii * W + xx];
      if (first) { acc = dmul(v, wv); first = false; }
      else acc = dadd(acc, dmul(v, wv));
    }
  out[(size_t)i * W + x] = acc;
}

// np.gradient (kernels.py:81-90) of a dense field at (i, x)
__device__ __forceinline__ void np_gradient(const double* f, int H, int W, int i, int x,
                                            double& fx, double& fy) {
  auto v = [&](int ii, int xx) { return f[(size_t)ii * W + xx]; };
  const double c = v(i, x);
  if (x == 0) fx = dsub(v(i, 1), c);
  else if (x == W - 1) fx = dsub(c, v(i, W - 2));
  else fx = dmul(dsub(v(i, x + 1), v(i, x - 1)), 0.5);
  if (i == 0) fy = dsub(v(1, x), c);
  else if (i == H - 1) fy = dsub(c, v(H - 2, x));
  else fy = dmul(dsub(v(i + 1, x), v(i - 1, x)), 0.5);
}

// edge indicator (models.py:78-81) from the smoothed image S
// g32 (the fast path's data plane) is stored pre-multiplied by g32_scale = dt/2.
__global__ void k_edge_g(const double* __restrict__ S, int H, int W, double gain,
                         double* __restrict__ g64, float* __restrict__ g32, long long pitch,
                         double g32_scale) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y;
  if (x >= W) return;
  double fx, fy;
  np_gradient(S, H, W, i, x, fx, fy);
  const double a = dmul(gain, fx), b = dmul(gain, fy);
  const double g = ddiv(1.0, dadd(dadd(1.0, dmul(a, a)), dmul(b, b)));
  if (g64) g64[(size_t)i * pitch + x] = g;
  if (g32) g32[(size_t)i * pitch + x] = (float)(g * g32_scale);
}

__global__ void k_gradient(const double* __restrict__ f, int H, int W, double* fx_out,
                           double* fy_out, double* mag_out) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y;
  if (x >= W) return;
  double fx, fy;
  np_gradient(f, H, W, i, x, fx, fy);
  const size_t o = (size_t)i * W + x;
  if (fx_out) fx_out[o] = fx;
  if (fy_out) fy_out[o] = fy;
  if (mag_out) mag_out[o] = np_hypot(fx, fy);
}

// ----------------------------------------------------- Chan-Vese baseline
// x^1.5 rounded to nearest from a double-double x * sqrt(x): glibc's pow
// (numpy's np.power) is accurate to 0.52 ulp, so this equals it except when
// the exact value lies within ~0.02 ulp of a rounding boundary.
__device__ __forceinline__ double pow_1p5(double x) {
  const double s = __dsqrt_rn(x);
  const double r = __fma_rn(-s, s, x);          // x - s^2 exactly
  const double s_lo = r / (2.0 * s);            // sqrt(x) = s + s_lo + O(ulp^2)
  const double p = __dmul_rn(x, s);
  const double p_lo = __fma_rn(x, s, -p) + x * s_lo;
  return p + p_lo;
}

// Mean curvature (kernels.py:98-115) at (i, x) from the first derivatives px,
// py (np.gradient of phi) with numpy's operation order:
//   num = pxx*py*py - 2*px*py*pxy + pyy*px*px,  den = (px*px + py*py + eps)^1.5
__device__ __forceinline__ double cv_curvature(const double* px, const double* py, int H, int W,
                                               int i, int x, double eps) {
  double pxx, pxy, t, pyy;
  np_gradient(px, H, W, i, x, pxx, pxy);      // d/dx, d/dy of px
  np_gradient(py, H, W, i, x, t, pyy);        // d/dy of py
  const size_t o = (size_t)i * W + x;
  const double ax = px[o], ay = py[o];
  const double num = dadd(dsub(dmul(dmul(pxx, ay), ay), dmul(dmul(dmul(2.0, ax), ay), pxy)),
                          dmul(dmul(pyy, ax), ax));
  const double den = pow_1p5(dadd(dadd(dmul(ax, ax), dmul(ay, ay)), eps));
  return ddiv(num, den);
}

// u = phi + dt * v for the curvature-regularized baseline (models.py:122-141,
// engine.py:155-157): v = [(c+ - c-)(2I - c+ - c-) + mu * kappa] * |grad phi|,
// the data term zero when a side is empty; px/py/mag from k_gradient.
__global__ void k_cv_update(const double* __restrict__ phi, const double* __restrict__ px,
                            const double* __restrict__ py, const double* __restrict__ mag,
                            double* __restrict__ u, int H, int W,
                            const float* __restrict__ data32, const double* __restrict__ data64,
                            long long dpitch, Scalars* sc, double dt, double mu, double eps) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y;
  if (x >= W) return;
  const size_t o = (size_t)i * W + x;
  double data = 0.0;                             // models.py:133-137: zero with an empty side
  if (sc->n_pos != 0 && sc->n_pos != sc->n_total) {
    const size_t od = (size_t)i * dpitch + x;
    const double I = data64 ? data64[od] : (double)data32[od];
    data = dmul(sc->dc, dsub(dsub(dmul(2.0, I), sc->c_pos), sc->c_neg));
  }
  if (mu != 0.0) data = dadd(data, dmul(mu, cv_curvature(px, py, H, W, i, x, eps)));
  const double v = dmul(data, mag[o]);
  if (!phi) {                                    // velocity only (cv_velocity)
    u[o] = v;
    return;
  }
  const double out = dadd(phi[o], dmul(dt, v));
  u[o] = out;
  if (!isfinite(out)) sc->nonfinite = 1;
}

__global__ void k_curvature(const double* __restrict__ px, const double* __restrict__ py, int H,
                            int W, double eps, double* __restrict__ out) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y;
  if (x >= W) return;
  out[(size_t)i * W + x] = cv_curvature(px, py, H, W, i, x, eps);
}

// Exact Euclidean distance transform (scipy.ndimage.distance_transform_edt,
// kernels.py:118-133): squared distances in integers (column pass, then the
// lower envelope of parabolas per row, Felzenszwalb-Huttenlocher, with exact
// fraction comparisons), sqrt correctly rounded.  target(q) = pixel q is a
// "zero" of the transform: the pixels whose distance to the nearest target is
// measured.  Column pass: g = (distance to the nearest target in the column)^2.
constexpr long long kEdtInf = 1LL << 60;
__global__ void k_edt_cols(const double* __restrict__ field, int H, int W, int target_positive,
                           long long* __restrict__ g) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= W) return;
  auto is_target = [&](int i) {
    const bool pos = field[(size_t)i * W + x] > 0.0;
    return target_positive ? pos : !pos;
  };
  long long last = -1;                          // forward: distance to a target above
  for (int i = 0; i < H; ++i) {
    if (is_target(i)) last = i;
    g[(size_t)i * W + x] = last < 0 ? kEdtInf : (long long)(i - last);
  }
  last = -1;
  for (int i = H - 1; i >= 0; --i) {            // backward: below; keep the nearer
    if (is_target(i)) last = i;
    long long d = g[(size_t)i * W + x];
    if (last >= 0 && (long long)(last - i) < d) d = last - i;
    g[(size_t)i * W + x] = d >= kEdtInf ? kEdtInf : d * d;
  }
}

// Row pass: D(i, x) = min_x' g(i, x') + (x - x')^2.  One thread per row; v / zn
// / zd are per-row scratch (W entries each, W + 1 for the breakpoints).
__global__ void k_edt_rows(const long long* __restrict__ g, int H, int W, int* __restrict__ vbuf,
                           long long* __restrict__ znum, long long* __restrict__ zden,
                           double* __restrict__ dist) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= H) return;
  const long long* gr = g + (size_t)i * W;
  int* v = vbuf + (size_t)i * W;
  long long* zn = znum + (size_t)i * (W + 1);
  long long* zd = zden + (size_t)i * (W + 1);
  int k = -1;
  for (int q = 0; q < W; ++q) {
    if (gr[q] >= kEdtInf) continue;
    const long long fq = gr[q] + (long long)q * q;
    while (k >= 0) {
      // intersection with the parabola at v[k]: s = (fq - fv) / (2 (q - v[k]))
      const long long fv = gr[v[k]] + (long long)v[k] * v[k];
      const long long sn = fq - fv, sd = 2LL * (q - v[k]);
      // pop while s <= z[k] (fractions, positive denominators)
      if (k > 0 && sn * zd[k] <= zn[k] * sd) { --k; continue; }
      ++k;
      v[k] = q;
      zn[k] = sn;
      zd[k] = sd;
      break;
    }
    if (k < 0) {
      k = 0;
      v[0] = q;
      zn[0] = -(1LL << 40);                      // -infinity
      zd[0] = 1;
    }
  }
  double* out = dist + (size_t)i * W;
  if (k < 0) {                                   // no target anywhere in reach
    for (int x = 0; x < W; ++x) out[x] = INFINITY;
    return;
  }
  int j = 0;
  for (int x = 0; x < W; ++x) {
    while (j < k && zn[j + 1] <= (long long)x * zd[j + 1]) ++j;   // x >= z[j+1]
    const long long dx = x - v[j];
    out[x] = __dsqrt_rn((double)(gr[v[j]] + dx * dx));
  }
}

// -signed_distance(field > 0) (engine.py:161-165): +distance to the nearest
// non-positive pixel inside, -distance to the nearest positive pixel outside.
__global__ void k_sdf_combine(const double* __restrict__ field, const double* __restrict__ d_to_neg,
                              const double* __restrict__ d_to_pos, double* __restrict__ out,
                              long long n) {
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < n;
       q += (long long)gridDim.x * blockDim.x)
    out[q] = field[q] > 0.0 ? d_to_neg[q] : -d_to_pos[q];
}

// u = phi + dt * v on a dense field (engine.py:155-157) + finiteness flag
// (engine.py:159).  data: I (region) or g (edge), exact values.
template <int MODEL>
__global__ void k_gen_update(const double* __restrict__ phi, double* __restrict__ u, int H, int W,
                             const float* __restrict__ data32, const double* __restrict__ data64,
                             long long dpitch, Scalars* sc, double dt) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y;
  if (MODEL == REGION && x == 0 && i == 0 && sc->zero_vel) sc->degenerate = 1;
  if (x >= W) return;
  double fx, fy;
  np_gradient(phi, H, W, i, x, fx, fy);
  const double h = np_hypot(fx, fy);
  const size_t od = (size_t)i * dpitch + x;
  const double d = data64 ? data64[od] : (double)data32[od];
  const double v = MODEL == REGION ? exact_v_twomean(sc, d, h) : dmul(d, h);
  const double out = dadd(phi[(size_t)i * W + x], dmul(dt, v));
  u[(size_t)i * W + x] = out;
  if (!isfinite(out)) sc->nonfinite = 1;
}

// velocity only (public region_velocity / edge_velocity)
template <int MODEL>
__global__ void k_velocity(const double* __restrict__ phi, double* __restrict__ v_out, int H, int W,
                           const double* __restrict__ data, const Scalars* sc) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y;
  if (x >= W) return;
  double fx, fy;
  np_gradient(phi, H, W, i, x, fx, fy);
  const double h = np_hypot(fx, fy);
  const double d = data[(size_t)i * W + x];
  v_out[(size_t)i * W + x] = MODEL == REGION ? exact_v_twomean(sc, d, h) : dmul(d, h);
}

__global__ void k_binarize(const double* __restrict__ in, double* __restrict__ out, long long n) {
  long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (; k < n; k += (long long)gridDim.x * blockDim.x) out[k] = in[k] > 0.0 ? 1.0 : -1.0;
}

__global__ void k_check_finite(const double* __restrict__ f, long long n, Scalars* sc) {
  long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  bool bad = false;
  for (; k < n; k += (long long)gridDim.x * blockDim.x) bad |= !isfinite(f[k]);
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) sc->nonfinite = 1;
}

// dense field (pitch W) -> vertical-word bits of (f > 0)
__global__ void k_pack_bits(const double* __restrict__ f, uint32_t* __restrict__ bits, RunGeom g) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int r = blockIdx.y;
  if (x >= g.pitch_w) return;
  uint32_t w = 0u;
  if (x < g.W) {
    for (int k = 0; k < 32; ++k) {
      const int i = r * 32 + k;
      if (i >= g.H) break;
      w |= (f[(size_t)i * g.W + x] > 0.0 ? 1u : 0u) << k;
    }
  }
  bits[(size_t)r * g.pitch_w + x] = w;
}

// int8 signs -> bits (b = sign > 0)
__global__ void k_pack_signs(const signed char* __restrict__ s, uint32_t* __restrict__ bits, RunGeom g) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int r = blockIdx.y;
  if (x >= g.pitch_w) return;
  uint32_t w = 0u;
  if (x < g.W) {
    for (int k = 0; k < 32; ++k) {
      const int i = r * 32 + k;
      if (i >= g.H) break;
      w |= (s[(size_t)i * g.W + x] > 0 ? 1u : 0u) << k;
    }
  }
  bits[(size_t)r * g.pitch_w + x] = w;
}

// state -> exact float64 phi (SMOOTH: G*b in scipy order; SCALED: +-s)
__global__ void k_phi_from_bits(const uint32_t* __restrict__ bits, double* __restrict__ out,
                                const ExactCtx* c, int src) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y;
  if (x >= c->W) return;
  double v;
  if (src == SRC_SCALED) v = get_bit(bits, c->pitch_w, i, x) ? c->scale : -c->scale;
  else v = exact_phi_smooth(bits, c->pitch_w, c->H, c->W, c->R, c->w64, i, x);
  out[(size_t)i * c->W + x] = v;
}

// Partition / checkpoint pass over any state representation, ABSOLUTE sums
// (grid.py:112-117 with double-double accumulation) + checkpoint mask
// (engine.py:229) + mismatch count vs the previous checkpoint.
// src: SRC_FIELD (phi dense), SRC_SCALED or SRC_SMOOTH (bits, exact phi).
__global__ void __launch_bounds__(kThreads) k_partition_abs(const double* __restrict__ field,
                                                            const uint32_t* __restrict__ bits,
                                                            const ExactCtx* c, int src,
                                                            uint32_t* pbits, uint32_t* mbits,
                                                            int do_part, int do_ckpt,
                                                            int write_mask_only,
                                                            TilePartial* part, RunGeom g) {
  __shared__ TilePartial s_warp[kThreads / 32];
  const int cbw = kColsPerThread * blockDim.x;
  for (int tile = blockIdx.x; tile < g.ntiles; tile += gridDim.x) {
    const int r = tile / g.ncb;
    const int cx0 = (tile - r * g.ncb) * cbw;
    const int x0 = cx0 + kColsPerThread * threadIdx.x;
    double ah = 0, al = 0, bh = 0, bl = 0;
    long long na = 0, nb = 0;
    unsigned long long mm = 0;
    if (x0 < g.W) {
      for (int cc = 0; cc < 8; ++cc) {
        const int x = x0 + cc;
        uint32_t pw = 0u, mw = 0u;
        if (x < g.W) {
          for (int k = 0; k < 32; ++k) {
            const int i = r * 32 + k;
            if (i >= g.H) break;
            double f;
            if (src == SRC_FIELD) f = field[(size_t)i * g.W + x];
            else if (src == SRC_SCALED) f = get_bit(bits, g.pitch_w, i, x) ? c->scale : -c->scale;
            else f = exact_phi_smooth(bits, g.pitch_w, g.H, g.W, c->R, c->w64, i, x);
            const uint32_t ge = f >= 0.0, gt = f > 0.0;
            pw |= ge << k;
            mw |= gt << k;
            if (do_part) {
              const double I = data_exact(c, i, x);
              if (ge) { dd_add(ah, al, I); ++na; }
              else { dd_add(bh, bl, I); ++nb; }
            }
          }
        }
        const size_t o = (size_t)r * g.pitch_w + x;
        if (do_part) pbits[o] = pw;
        if (write_mask_only) {
          mbits[o] = mw;
        } else if (do_ckpt) {
          mm += __popc(mbits[o] ^ mw);
          mbits[o] = mw;
        }
      }
    }
    // fixed-order CTA reduction (double-double)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int o = 16; o > 0; o >>= 1) {
      double h2 = __shfl_xor_sync(0xffffffffu, ah, o), l2 = __shfl_xor_sync(0xffffffffu, al, o);
      dd_add_dd(ah, al, h2, l2);
      h2 = __shfl_xor_sync(0xffffffffu, bh, o);
      l2 = __shfl_xor_sync(0xffffffffu, bl, o);
      dd_add_dd(bh, bl, h2, l2);
      na += __shfl_xor_sync(0xffffffffu, na, o);
      nb += __shfl_xor_sync(0xffffffffu, nb, o);
      mm += __shfl_xor_sync(0xffffffffu, mm, o);
    }
    __syncthreads();
    if (lane == 0) {
      s_warp[warp].a_hi = ah; s_warp[warp].a_lo = al;
      s_warp[warp].b_hi = bh; s_warp[warp].b_lo = bl;
      s_warp[warp].n_a = na; s_warp[warp].n_b = nb; s_warp[warp].mism = mm;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      TilePartial t{};
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
        dd_add_dd(t.a_hi, t.a_lo, s_warp[w].a_hi, s_warp[w].a_lo);
        dd_add_dd(t.b_hi, t.b_lo, s_warp[w].b_hi, s_warp[w].b_lo);
        t.n_a += s_warp[w].n_a;
        t.n_b += s_warp[w].n_b;
        t.mism += s_warp[w].mism;
      }
      part[tile] = t;
    }
  }
}

__global__ void __launch_bounds__(1024) k_finalize(const TilePartial* part, int n, Scalars* sc,
                                                       int delta, int region, int ckpt,
                                                       long long iter) {
  PartRanges R3{{part, part, part}, {n, 0, 0}};
  finalize_cta(R3, sc, delta != 0, region != 0, ckpt != 0, iter);
}

// stage 1 of the fast path's finalize: CTA b reduces slice b of the partials
constexpr int kFinSlices = 64;
constexpr int kFusedFinSlices = 256;             // the fused pass's (one partial per unit)
__global__ void __launch_bounds__(256) k_finalize_stage1(PartRanges R3, TilePartial* out,
                                                         const Scalars* sc) {
  pdl_wait();
  pdl_launch_dependents();
  if (stop_flag(sc)) return;
  const int n = R3.n[0] + R3.n[1] + R3.n[2];
  const int per = (n + gridDim.x - 1) / gridDim.x;
  const int t0 = min(n, (int)blockIdx.x * per), t1 = min(n, t0 + per);
  reduce_slice(R3, t0, t1, out + blockIdx.x);
}

// row strips: one CTA reduces this rank's slice results to the single partial
// the ranks exchange (fixed order)
__global__ void __launch_bounds__(256) k_reduce_to_one(PartRanges R3, TilePartial* out,
                                                       const Scalars* sc, int check_stop) {
  if (check_stop && stop_flag(sc)) return;
  reduce_slice(R3, 0, R3.n[0] + R3.n[1] + R3.n[2], out);
}

// batched tiles (lse_batch): stage 1 per tile (blockIdx.y = tile) over the
// tile's partials in the single-run order [border units][interior units], so a
// tile's reduction is the one it would get alone
__global__ void __launch_bounds__(256) k_finalize_stage1_tiles(const TilePartial* part,
                                                               TilePartial* out,
                                                               const Scalars* scal, int nb,
                                                               int ni, int T, int ckpt) {
  pdl_wait();
  pdl_launch_dependents();
  const int t = blockIdx.y;
  const Scalars* sc = scal + t;
  if (stop_flag(sc)) return;
  if (sc->model == EDGE && !ckpt) return;
  PartRanges R3{{part + (size_t)t * nb, part + (size_t)T * nb + (size_t)t * ni, part},
                {nb, ni, 0}};
  const int n = nb + ni;
  const int per = (n + gridDim.x - 1) / gridDim.x;
  const int t0 = min(n, (int)blockIdx.x * per), t1 = min(n, t0 + per);
  reduce_slice(R3, t0, t1, out + (size_t)t * gridDim.x + blockIdx.x);
}

// (spec = 1 + fix-list parity after a speculative fused pass: the tile's
// prediction is checked; tile 0's scalars hold the batch's fix-list counters)
__global__ void __launch_bounds__(64) k_finalize_run_tiles(const TilePartial* fin, Scalars* scal,
                                                           int ckpt, long long iter, int spec) {
  pdl_wait();
  pdl_launch_dependents();
  const int t = blockIdx.x;
  Scalars* sc = scal + t;
  if (stop_flag(sc)) return;
  const bool region = sc->model != EDGE;
  if (!region && !ckpt) return;
  const TilePartial* f = fin + (size_t)t * kFinSlices;
  PartRanges R1{{f, f, f}, {kFinSlices, 0, 0}};
  finalize_cta(R1, sc, true, region, ckpt != 0, iter, spec, scal);
}

// batched tiles with few partials per tile: a single-stage finalize per tile
// (blockIdx.x = tile) over the tile's partials in the single-run order
// [border units][interior units] -- what k_finalize_run does for the same
// tile run alone, so the reduction order is the same
__global__ void __launch_bounds__(64) k_finalize_tiles_direct(const TilePartial* part,
                                                              Scalars* scal, int nb, int ni,
                                                              int T, int ckpt, long long iter,
                                                              int spec) {
  pdl_wait();
  pdl_launch_dependents();
  const int t = blockIdx.x;
  Scalars* sc = scal + t;
  if (stop_flag(sc)) return;
  const bool region = sc->model != EDGE;
  if (!region && !ckpt) return;
  PartRanges R3{{part + (size_t)t * nb, part + (size_t)T * nb + (size_t)t * ni, part},
                {nb, ni, 0}};
  finalize_cta(R3, sc, true, region, ckpt != 0, iter, spec, scal);
}

// per-iteration finalize of the fast path (DELTA partials); no-op once stopped
// (spec = 1 + fix-list parity: the partials came from a speculative fused
// pass, whose prediction is checked here -- spec_check)
__global__ void __launch_bounds__(64) k_finalize_run(PartRanges R3, Scalars* sc, int region,
                                                       int ckpt, long long iter, int spec) {
  pdl_wait();
  pdl_launch_dependents();
  if (stop_flag(sc)) return;
  finalize_cta(R3, sc, true, region != 0, ckpt != 0, iter, spec);
}

// image statistics: min, max, max|.| (order-preserving integer atomics)
__device__ __forceinline__ long long dkey(double v) {
  long long b = __double_as_longlong(v);
  return b ^ ((b >> 63) & 0x7fffffffffffffffLL);
}
__device__ __forceinline__ double dkey_inv(long long k) {
  return __longlong_as_double(k ^ ((k >> 63) & 0x7fffffffffffffffLL));
}
__global__ void k_minmax(const float* __restrict__ d32, const double* __restrict__ d64, int H, int W,
                         long long pitch, long long* keys /* [min, max, absmax] */) {
  long long kmin = LLONG_MAX, kmax = LLONG_MIN, kabs = LLONG_MIN;
  for (int i = blockIdx.x; i < H; i += gridDim.x) {
    for (int x = threadIdx.x; x < W; x += blockDim.x) {
      const size_t o = (size_t)i * pitch + x;
      const double v = d64 ? d64[o] : (double)__ldcs(d32 + o);
      const long long k = dkey(v), ka = dkey(fabs(v));
      kmin = k < kmin ? k : kmin;
      kmax = k > kmax ? k : kmax;
      kabs = ka > kabs ? ka : kabs;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    long long a = __shfl_xor_sync(0xffffffffu, kmin, o);
    long long b = __shfl_xor_sync(0xffffffffu, kmax, o);
    long long e = __shfl_xor_sync(0xffffffffu, kabs, o);
    kmin = a < kmin ? a : kmin;
    kmax = b > kmax ? b : kmax;
    kabs = e > kabs ? e : kabs;
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(&keys[0], kmin);
    atomicMax(&keys[1], kmax);
    atomicMax(&keys[2], kabs);
  }
}
__global__ void k_store_minmax(const long long* keys, Scalars* sc) {
  sc->img_min = dkey_inv(keys[0]);
  sc->img_max = dkey_inv(keys[1]);
  sc->img_absmax = dkey_inv(keys[2]);
}

// float64 image -> fp32 plane (+ flag when fp32 is not exact)
__global__ void k_to_f32(const double* __restrict__ in, float* __restrict__ out, int H, int W,
                         long long pitch, int* inexact) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y;
  if (x >= W) return;
  const double v = in[(size_t)i * W + x];
  const float f = (float)v;
  out[(size_t)i * pitch + x] = f;
  if ((double)f != v) *inexact = 1;
}
// float64 dense -> pitched float64
__global__ void k_pitch64(const double* __restrict__ in, double* __restrict__ out, int H, int W,
                          long long pitch) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y;
  if (x >= W) return;
  out[(size_t)i * pitch + x] = in[(size_t)i * W + x];
}
// pitched fp32 plane -> dense float64
__global__ void k_widen(const float* __restrict__ in, double* __restrict__ out, int H, int W,
                        long long pitch) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y;
  if (x >= W) return;
  out[(size_t)i * W + x] = (double)in[(size_t)i * pitch + x];
}

// ---------------------------------------------------- multi-band (VECTOR)
// One iteration's band chain after the fused partition:
//   k_band_sums  per-band sums of the pixels that changed side, one partial per
//                (word-row, 1024-column block); the last CTA to finish folds
//                them (fixed order) into the running sums, the means, the
//                checkpoint bookkeeping (finalize_bands_cta);
//   k_band_peak  D of every pixel exactly (fp64), the fp32 data plane of the
//                fused kernels and max |D| (atomicMax on the ordered bits);
//                the last CTA derives the coefficients of the next update.
// Both "last CTA" hand-offs use a per-run arrival counter (cnt[0], cnt[1]),
// reset by the CTA that consumed it.

// Arrival at the end of a kernel: true in exactly one (the last) CTA, after
// which every other CTA's global writes are visible to it.
__device__ __forceinline__ bool last_cta_arrival(unsigned long long* cnt) {
  __shared__ bool s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned long long total = (unsigned long long)gridDim.x * gridDim.y;
    s_last = atomicAdd(cnt, 1ull) == total - 1;
  }
  __syncthreads();
  if (!s_last) return false;
  __threadfence();
  if (threadIdx.x == 0) *cnt = 0ull;             // ready for the next launch
  return true;
}

// Fixed-order CTA reduction of K band partial arrays at once: the order of
// reduce_slice for every band (each thread a contiguous range, then the xor
// tree, then warps in index order), with the K bands' loads issued together.
__device__ void reduce_bands(const TilePartial* bpart, int nblk, int K, TilePartial* out) {
  __shared__ double g_h[kMaxBands][2][32], g_l[kMaxBands][2][32];
  __shared__ long long g_n[kMaxBands][2][32];
  const int T = blockDim.x, tid = threadIdx.x;
  double ah[kMaxBands], al[kMaxBands], bh[kMaxBands], bl[kMaxBands];
  long long na[kMaxBands], nb[kMaxBands];
#pragma unroll
  for (int k = 0; k < kMaxBands; ++k) { ah[k] = al[k] = bh[k] = bl[k] = 0.0; na[k] = nb[k] = 0; }
  const int per = (nblk + T - 1) / T;
  const int lo = tid * per;
  const int hi = min(lo + per, nblk);
  for (int t = lo; t < hi; ++t) {
#pragma unroll
    for (int k = 0; k < kMaxBands; ++k) {
      if (k >= K) break;
      const TilePartial* p = bpart + (size_t)k * nblk + t;
      const double2 A = __ldcg(reinterpret_cast<const double2*>(&p->a_hi));
      const double2 B = __ldcg(reinterpret_cast<const double2*>(&p->b_hi));
      const longlong2 NN = __ldcg(reinterpret_cast<const longlong2*>(&p->n_a));
      dd_add_dd(ah[k], al[k], A.x, A.y);
      dd_add_dd(bh[k], bl[k], B.x, B.y);
      na[k] += NN.x;
      nb[k] += NN.y;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
    for (int k = 0; k < kMaxBands; ++k) {
      if (k >= K) break;
      dd_shfl_add(ah[k], al[k], o);
      dd_shfl_add(bh[k], bl[k], o);
      na[k] += __shfl_xor_sync(0xffffffffu, na[k], o);
      nb[k] += __shfl_xor_sync(0xffffffffu, nb[k], o);
    }
  }
  const int warp = tid >> 5, lane = tid & 31;
  if (lane == 0)
    for (int k = 0; k < K; ++k) {
      g_h[k][0][warp] = ah[k]; g_l[k][0][warp] = al[k]; g_n[k][0][warp] = na[k];
      g_h[k][1][warp] = bh[k]; g_l[k][1][warp] = bl[k]; g_n[k][1][warp] = nb[k];
    }
  __syncthreads();
  if (tid < K) {
    const int k = tid;
    TilePartial t{};
    for (int w = 0; w < (T + 31) / 32; ++w) {
      dd_add_dd(t.a_hi, t.a_lo, g_h[k][0][w], g_l[k][0][w]);
      dd_add_dd(t.b_hi, t.b_lo, g_h[k][1][w], g_l[k][1][w]);
      t.n_a += g_n[k][0][w];
      t.n_b += g_n[k][1][w];
    }
    out[k] = t;
  }
  __syncthreads();
}

// Reduce the band partials (fixed order) into the running per-band sums and
// means; checkpoint bookkeeping from the fused partition's partials (mism).
// Run by one CTA.  absolute: the partials are full sums (initial state).
__device__ void finalize_bands_cta(const TilePartial* bpart, int nblk, const PartRanges& mism_parts,
                                   Scalars* sc, bool absolute, bool ckpt, long long iter) {
  __shared__ TilePartial s_band[kMaxBands];
  const int K = sc->nbands;
  // no block saw a changed pixel: every partial is zero
  if (absolute || __ldcg(&sc->band_any)) {
    reduce_bands(bpart, nblk, K, s_band);
  } else {
    if (threadIdx.x < K) s_band[threadIdx.x] = TilePartial{};
    __syncthreads();
  }
  unsigned long long mm = 0;
  if (ckpt) {
    __shared__ TilePartial s_m;
    reduce_slice(mism_parts, 0, mism_parts.n[0] + mism_parts.n[1] + mism_parts.n[2], &s_m);
    __syncthreads();
    mm = s_m.mism;
  }
  if (threadIdx.x != 0) return;
  sc->band_any = 0;                                // for the next pass
  // no pixel changed side: the running sums, the means and therefore the
  // data plane, max|D| and the coefficients of the last peak pass stay
  // exactly as they are (grid.py:116-117 over the same partition)
  const bool same = !absolute && sc->band_reuse && sc->band_valid &&
                    s_band[0].n_a == 0 && s_band[0].n_b == 0;
  sc->band_same = same ? 1 : 0;
  if (same) sc->band_reused += 1;
  else sc->band_valid = 0;
  for (int k = 0; k < K && !same; ++k) {
    const TilePartial& t = s_band[k];
    if (absolute) {
      sc->bsp_hi[k] = t.a_hi; sc->bsp_lo[k] = t.a_lo;
      sc->bsn_hi[k] = t.b_hi; sc->bsn_lo[k] = t.b_lo;
    } else {                                       // a: entering P, b: leaving P
      dd_add_dd(sc->bsp_hi[k], sc->bsp_lo[k], t.a_hi, t.a_lo);
      dd_add_dd(sc->bsp_hi[k], sc->bsp_lo[k], -t.b_hi, -t.b_lo);
      dd_add_dd(sc->bsn_hi[k], sc->bsn_lo[k], t.b_hi, t.b_lo);
      dd_add_dd(sc->bsn_hi[k], sc->bsn_lo[k], -t.a_hi, -t.a_lo);
    }
  }
  if (!same) {
    sc->n_pos = absolute ? s_band[0].n_a : sc->n_pos + s_band[0].n_a - s_band[0].n_b;
    const long long np = sc->n_pos, nn = sc->n_total - sc->n_pos;
    sc->zero_vel = (np == 0 || nn == 0) ? 1 : 0;  // grid.py:114-115, models.py:111-113
    if (!sc->zero_vel)
      for (int k = 0; k < K; ++k) {
        sc->bcp[k] = dd_div(sc->bsp_hi[k], sc->bsp_lo[k], (double)np);
        sc->bcm[k] = dd_div(sc->bsn_hi[k], sc->bsn_lo[k], (double)nn);
      }
    sc->peak_bits = 0ull;                          // k_band_peak's atomicMax target
  }
  if (ckpt) {                                      // engine.py:228-236
    sc->n_ckpt += 1;
    if (sc->n_ckpt >= 2) sc->equal_run = (mm == 0) ? sc->equal_run + 1 : 0;
    const long long cw = sc->conv_window;
    if (cw == 1 || (sc->n_ckpt >= cw && sc->equal_run >= cw - 1)) {
      sc->stop = 1;
      sc->converged = 1;
      sc->converged_iter = iter;
    }
  }
}

// Per-band sums of the pixels that changed side (ABS = false: chg bits,
// split by the new partition bit) or of every pixel (ABS = true: split by P),
// one double-double partial per (word-row, 1024-column block) and band, in a
// fixed order (bit order within a word, each thread's four consecutive words
// in column order, the xor tree, warps in index order).  Partial layout:
// part[k * nblk + blk].  The changed bits of a word are taken four at a
// time, so the band loads of four pixels are in flight together; they are
// accumulated in bit order.  A block without changed pixels (the common case
// once the partition settles) writes a zero partial after one 16-byte load
// per thread; a pass without any changed pixel skips the final reduction.
template <bool ABS>
__global__ void __launch_bounds__(256) k_band_sums(const uint32_t* __restrict__ chg,
                                                   const uint32_t* __restrict__ pbits,
                                                   const ExactCtx* c, TilePartial* part,
                                                   RunGeom g, Scalars* sc,
                                                   unsigned long long* cnt, PartRanges mism_parts,
                                                   int ckpt, long long iter) {
  pdl_wait();
  pdl_launch_dependents();
  if (!ABS && stop_flag(sc)) return;
  __shared__ TilePartial s_w[kMaxBands][8];
  const int r = blockIdx.y;
  const int nblk = gridDim.x * gridDim.y, blk = r * gridDim.x + blockIdx.x;
  const int K = c->nbands;
  const int x0 = blockIdx.x * 1024 + threadIdx.x * 4;
  const size_t o0 = (size_t)r * g.pitch_w + x0;
  uint32_t mw[4] = {0u, 0u, 0u, 0u};
  if (x0 < g.W) {                                // pitch_w is a multiple of 8 >= W
    if (ABS) {
      const uint32_t rows = (g.H - r * 32) >= 32 ? 0xffffffffu : ((1u << (g.H - r * 32)) - 1u);
#pragma unroll
      for (int q = 0; q < 4; ++q) mw[q] = x0 + q < g.W ? rows : 0u;
    } else {
      const uint4 v = __ldcg(reinterpret_cast<const uint4*>(chg + o0));
      mw[0] = v.x; mw[1] = v.y; mw[2] = v.z; mw[3] = v.w;
    }
  }
  if (!__syncthreads_or((mw[0] | mw[1] | mw[2] | mw[3]) != 0u)) {
    if (threadIdx.x < K) part[(size_t)threadIdx.x * nblk + blk] = TilePartial{};
  } else {
    if (threadIdx.x == 0) sc->band_any = 1;      // some pixel changed side in this pass
    const float* b32 = c->bands32;
    const double* b64 = c->bands64;
    const size_t bstride = (size_t)c->band_stride, dpitch = (size_t)c->data_pitch;
    double ah[kMaxBands], al[kMaxBands], bh[kMaxBands], bl[kMaxBands];
    long long na = 0, nb = 0;
#pragma unroll
    for (int k = 0; k < kMaxBands; ++k) ah[k] = al[k] = bh[k] = bl[k] = 0.0;
    for (int j = 0; j < 4; ++j) {
      uint32_t m = mw[j];
      if (!m) continue;
      const int x = x0 + j;
      const uint32_t p = pbits[o0 + j];
      while (m) {
        int bs[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          bs[q] = m ? __ffs(m) - 1 : -1;
          m &= m - 1;
        }
        double I[4][kMaxBands];
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int k = 0; k < kMaxBands; ++k) {
            I[q][k] = 0.0;
            if (bs[q] >= 0 && k < K) {
              const size_t e = (size_t)k * bstride + (size_t)(r * 32 + bs[q]) * dpitch + x;
              I[q][k] = b64 ? b64[e] : (double)b32[e];
            }
          }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          if (bs[q] < 0) break;
          const bool in = (p >> bs[q]) & 1u;
#pragma unroll
          for (int k = 0; k < kMaxBands; ++k) {
            if (k >= K) break;
            if (in) dd_add(ah[k], al[k], I[q][k]);
            else dd_add(bh[k], bl[k], I[q][k]);
          }
          if (in) ++na; else ++nb;
        }
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
      for (int k = 0; k < kMaxBands; ++k) {
        if (k >= K) break;
        dd_shfl_add(ah[k], al[k], o);
        dd_shfl_add(bh[k], bl[k], o);
      }
      na += __shfl_xor_sync(0xffffffffu, na, o);
      nb += __shfl_xor_sync(0xffffffffu, nb, o);
    }
    const int warp = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0)
      for (int k = 0; k < K; ++k) {
        s_w[k][warp].a_hi = ah[k]; s_w[k][warp].a_lo = al[k];
        s_w[k][warp].b_hi = bh[k]; s_w[k][warp].b_lo = bl[k];
        s_w[k][warp].n_a = na; s_w[k][warp].n_b = nb;
      }
    __syncthreads();
    if (threadIdx.x < K) {
      const int k = threadIdx.x;
      TilePartial t{};
      for (int w = 0; w < 8; ++w) {
        dd_add_dd(t.a_hi, t.a_lo, s_w[k][w].a_hi, s_w[k][w].a_lo);
        dd_add_dd(t.b_hi, t.b_lo, s_w[k][w].b_hi, s_w[k][w].b_lo);
        t.n_a += s_w[k][w].n_a;
        t.n_b += s_w[k][w].n_b;
      }
      part[(size_t)k * nblk + blk] = t;
    }
  }
  if (!last_cta_arrival(cnt)) return;
  finalize_bands_cta(part, nblk, mism_parts, sc, ABS, ckpt != 0, iter);
}

// The multi-band data term of every pixel for the next update: D exactly in
// fp64 (vector_D's operations; the band constants hoisted), stored rounded to
// fp32 as the fused kernels' data plane, and max |D| (np.abs(data).max()).
// Each CTA takes one 1024-column block of the rows blockIdx.y, +gridDim.y, ..
// (every band load of a row issued before any use), then one atomicMax of
// its maximum on sc->peak_bits (non-negative doubles order like their bits);
// the last CTA turns the peak into the coefficients of the next update.
template <int K>
__global__ void __launch_bounds__(256) k_band_peak(const ExactCtx* __restrict__ c,
                                                   Scalars* __restrict__ sc,
                                                   float* __restrict__ d32,
                                                   unsigned long long* cnt, RunGeom g) {
  pdl_wait();
  pdl_launch_dependents();
  // the means did not move: plane, peak and coefficients are still current
  if (__ldcg(&sc->band_same)) return;
  const float* b32 = c->bands32;
  const double* b64 = c->bands64;
  const long long stride = c->band_stride;
  const int x0 = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
  const bool act = x0 < g.W;
  const bool live = !sc->stop && !sc->zero_vel;
  double cp[K], cm[K], dc[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    cp[k] = sc->bcp[k];
    cm[k] = sc->bcm[k];
    dc[k] = dsub(cp[k], cm[k]);
  }
  unsigned long long m = 0ull;
  if (live && act) {
    for (int i = blockIdx.y; i < g.H; i += gridDim.y) {
      const size_t o = (size_t)i * g.data_pitch + x0;
      double I[K][4];
      if (b64) {
#pragma unroll
        for (int k = 0; k < K; ++k)
#pragma unroll
          for (int q = 0; q < 4; ++q) I[k][q] = b64[k * stride + o + q];
      } else {
        float4 v[K];
#pragma unroll
        for (int k = 0; k < K; ++k) v[k] = __ldcs(reinterpret_cast<const float4*>(b32 + k * stride + o));
#pragma unroll
        for (int k = 0; k < K; ++k) {
          I[k][0] = v[k].x; I[k][1] = v[k].y; I[k][2] = v[k].z; I[k][3] = v[k].w;
        }
      }
      double D[4];
#pragma unroll
      for (int k = 0; k < K; ++k)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const double t = dmul(dc[k], dsub(dsub(dmul(2.0, I[k][q]), cp[k]), cm[k]));
          D[q] = k == 0 ? t : dadd(D[q], t);
        }
      float4 out;
      out.x = (float)D[0]; out.y = (float)D[1]; out.z = (float)D[2]; out.w = (float)D[3];
      reinterpret_cast<float4*>(d32 + o)[0] = out;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (x0 + q >= g.W) break;
        const unsigned long long bb = (unsigned long long)__double_as_longlong(fabs(D[q]));
        m = bb > m ? bb : m;
      }
    }
  }
  for (int o2 = 16; o2 > 0; o2 >>= 1) {
    const unsigned long long v = __shfl_xor_sync(0xffffffffu, m, o2);
    m = v > m ? v : m;
  }
  __shared__ unsigned long long s_m[8];
  if ((threadIdx.x & 31) == 0) s_m[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = s_m[w] > m ? s_m[w] : m;
    if (m) atomicMax(&sc->peak_bits, m);
  }
  if (!last_cta_arrival(cnt)) return;
  if (threadIdx.x != 0 || stop_flag(sc)) return;
  // coefficients of the next update: the fused kernels see the data plane D
  // (fp32) and vf = A * D with A = (dt / 2) / peak
  m = sc->zero_vel ? 0ull : *(volatile unsigned long long*)&sc->peak_bits;
  sc->peak_bits = m;
  const double peak = __longlong_as_double((long long)m);
  sc->peak = peak;
  if (sc->zero_vel || peak == 0.0) {               // models.py:117-118
    sc->zero_vel = 1;
    sc->A = 0.f;
    sc->B = 0.f;
    sc->eps_u = (float)(kGuard * (kErrPhi + 0x1p-22));
    sc->band_valid = 1;
    return;
  }
  const double dt = sc->dt, a = 1.0 / peak;
  sc->A = (float)(0.5 * dt * a);
  sc->B = 0.f;
  // |a| * max|D| = 1; the fp32 plane adds one rounding of D
  const double eps_d = 0x1p-21 * (2.0 + 1.0 + 1.0);
  sc->eps_u = (float)(kGuard * (kErrPhi + dt * (kErrGrad + 1.5 * eps_d + 0x1p-21) +
                                0x1p-22 * (1.0 + 1.5 * dt)));
  sc->band_valid = 1;
}

// 8-bit RGB -> the reference loader's grayscale (fileio.py:28-30, 88): luma
// in float64, ((0.299 R + 0.587 G) + 0.114 B) / 255, no re-quantization.
__global__ void k_luma(const unsigned char* __restrict__ rgb, double* __restrict__ out,
                       long long n) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double R = rgb[3 * i], G = rgb[3 * i + 1], B = rgb[3 * i + 2];
  out[i] = ddiv(dadd(dadd(dmul(0.299, R), dmul(0.587, G)), dmul(0.114, B)), 255.0);
}

// Batched tiles: copy n words (or bytes, via uint32 units) from per-tile
// source pointers into / out of the stacked arrays (blockIdx.y = tile).
__global__ void k_tiles_copy(const uint32_t* const* srcs, uint32_t* const* dsts, long long n) {
  const uint32_t* src = srcs[blockIdx.y];
  uint32_t* dst = dsts[blockIdx.y];
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

// Even-odd seed rasterization at pixel centres (grid.py:58-93), union of
// polygons; emits the state bits of phi0 = where(inside, s, -s) and counts
// the inside pixels (DegenerateSeedError check).
__global__ void k_rasterize(const double* __restrict__ xy, const long long* __restrict__ offs,
                            int n_polys, int inside_sign, uint32_t* bits, signed char* signs,
                            RunGeom g, unsigned long long* n_inside, long long y_off) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int r = blockIdx.y;
  unsigned long long cnt = 0;
  if (x < g.pitch_w) {
    uint32_t w = 0u;
    if (x < g.W) {
      const double cx = dadd((double)x, 0.5);
      for (int k = 0; k < 32; ++k) {
        const int i = r * 32 + k;
        if (i >= g.H) break;
        const double cy = dadd((double)(y_off + i), 0.5);   // global row (row strips)
        bool inside = false;
        for (int p = 0; p < n_polys && !inside; ++p) {
          const long long a = offs[p], e = offs[p + 1];
          const long long nv = e - a;
          bool in_p = false;
          for (long long q = 0; q < nv; ++q) {
            const double x1 = xy[2 * (a + q)], y1 = xy[2 * (a + q) + 1];
            const long long q2 = (q + 1) % nv;
            const double x2 = xy[2 * (a + q2)], y2 = xy[2 * (a + q2) + 1];
            if (y1 == y2) continue;
            const bool crosses = (y1 > cy) != (y2 > cy);
            const double x_hit = dadd(x1, ddiv(dmul(dsub(cy, y1), dsub(x2, x1)), dsub(y2, y1)));
            if (crosses && (cx < x_hit)) in_p = !in_p;
          }
          inside = in_p;
        }
        cnt += inside;
        const bool pos = inside ? (inside_sign > 0) : (inside_sign < 0);
        w |= (pos ? 1u : 0u) << k;
        if (signs) signs[(size_t)i * g.W + x] = pos ? 1 : -1;
      }
    }
    if (bits) bits[(size_t)r * g.pitch_w + x] = w;
  }
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(n_inside, cnt);
}

// Same fill, for polygons with at most kRastEdges edges in total: per block of
// 32 rows the crossing flags and x_hit of every (row, edge) are computed once
// (exactly as grid.py:70-71 evaluates them) and shared by the block's columns.
constexpr int kRastEdges = 64;
__global__ void __launch_bounds__(256) k_rasterize_rows(const double* __restrict__ xy,
                                                        const long long* __restrict__ offs,
                                                        int n_polys, int inside_sign,
                                                        uint32_t* bits, RunGeom g,
                                                        unsigned long long* n_inside,
                                                        long long y_off) {
  __shared__ double s_xhit[32][kRastEdges];
  __shared__ unsigned char s_cross[32][kRastEdges];
  __shared__ short s_poly[kRastEdges];
  const int r = blockIdx.y;
  const int ne = (int)offs[n_polys];
  for (int q = threadIdx.x; q < 32 * ne; q += blockDim.x) {
    const int k = q / ne, e = q - k * ne;
    int p = 0;
    while (offs[p + 1] <= e) ++p;
    const long long a = offs[p], nv = offs[p + 1] - a, qv = e - a;
    const double x1 = xy[2 * e], y1 = xy[2 * e + 1];
    const long long e2 = a + (qv + 1) % nv;
    const double x2 = xy[2 * e2], y2 = xy[2 * e2 + 1];
    const double cy = dadd((double)(y_off + r * 32 + k), 0.5);
    bool crosses = false;
    double xh = 0.0;
    if (y1 != y2) {
      crosses = (y1 > cy) != (y2 > cy);
      xh = dadd(x1, ddiv(dmul(dsub(cy, y1), dsub(x2, x1)), dsub(y2, y1)));
    }
    s_xhit[k][e] = xh;
    s_cross[k][e] = crosses;
    if (k == 0) s_poly[e] = (short)p;
  }
  __syncthreads();
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long cnt = 0;
  if (x < g.pitch_w) {
    uint32_t w = 0u;
    if (x < g.W) {
      const double cx = dadd((double)x, 0.5);
      for (int k = 0; k < 32; ++k) {
        const int i = r * 32 + k;
        if (i >= g.H) break;
        bool inside = false, par = false;
        int cur = 0;
        for (int e = 0; e < ne; ++e) {
          if (s_poly[e] != cur) {          // next polygon: union of even-odd fills
            inside |= par;
            par = false;
            cur = s_poly[e];
          }
          if (s_cross[k][e] && cx < s_xhit[k][e]) par = !par;
        }
        inside |= par;
        cnt += inside;
        const bool pos = inside ? (inside_sign > 0) : (inside_sign < 0);
        w |= (pos ? 1u : 0u) << k;
      }
    }
    bits[(size_t)r * g.pitch_w + x] = w;
  }
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(n_inside, cnt);
}

// Initial partition of a +-s state: P = b, sums of I over b = +1 / b = -1
// (double-double), coalesced (lanes on consecutive columns), one partial per
// CTA (1024 columns x 32 rows) in a fixed order.
__global__ void __launch_bounds__(256) k_partition_init_bits(const uint32_t* __restrict__ bits,
                                                             const ExactCtx* c, uint32_t* pbits,
                                                             TilePartial* part, RunGeom g,
                                                             int own_lo, int own_hi) {
  __shared__ TilePartial s_w[8];
  const int r = blockIdx.y;
  const bool own = r >= own_lo && r < own_hi;   // row strips: halo rows are not counted
  double ah = 0, al = 0, bh = 0, bl = 0;
  long long na = 0, nb = 0;
  for (int j = 0; j < 4; ++j) {
    const int x = blockIdx.x * 1024 + j * 256 + threadIdx.x;
    if (x >= g.pitch_w) continue;
    const uint32_t w = bits[(size_t)r * g.pitch_w + x];
    pbits[(size_t)r * g.pitch_w + x] = w;
    if (x >= g.W || !own) continue;
    for (int k = 0; k < 32; ++k) {
      const int i = r * 32 + k;
      if (i >= g.H) break;
      const double I = data_exact(c, i, x);
      if ((w >> k) & 1u) { dd_add(ah, al, I); ++na; }
      else { dd_add(bh, bl, I); ++nb; }
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    double h2 = __shfl_xor_sync(0xffffffffu, ah, o), l2 = __shfl_xor_sync(0xffffffffu, al, o);
    dd_add_dd(ah, al, h2, l2);
    h2 = __shfl_xor_sync(0xffffffffu, bh, o);
    l2 = __shfl_xor_sync(0xffffffffu, bl, o);
    dd_add_dd(bh, bl, h2, l2);
    na += __shfl_xor_sync(0xffffffffu, na, o);
    nb += __shfl_xor_sync(0xffffffffu, nb, o);
  }
  const int warp = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    s_w[warp].a_hi = ah; s_w[warp].a_lo = al; s_w[warp].b_hi = bh; s_w[warp].b_lo = bl;
    s_w[warp].n_a = na; s_w[warp].n_b = nb;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    TilePartial t{};
    for (int w = 0; w < 8; ++w) {
      dd_add_dd(t.a_hi, t.a_lo, s_w[w].a_hi, s_w[w].a_lo);
      dd_add_dd(t.b_hi, t.b_lo, s_w[w].b_hi, s_w[w].b_lo);
      t.n_a += s_w[w].n_a;
      t.n_b += s_w[w].n_b;
    }
    part[(size_t)r * gridDim.x + blockIdx.x] = t;
  }
}

// checkpoint-style mask bits -> host layout.  mask = (phi > 0) for
// inside_sign > 0, else (phi <= 0) (engine.py:256-259).
__global__ void k_mask_u8(const uint32_t* __restrict__ mbits, RunGeom g, int invert,
                          unsigned char* out) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y;
  if (x >= g.W) return;
  const int b = get_bit(mbits, g.pitch_w, i, x);
  out[(size_t)i * g.W + x] = (unsigned char)(invert ? !b : b);
}
__global__ void k_mask_packed(const uint32_t* __restrict__ mbits, RunGeom g, int invert,
                              unsigned char* out, long long nbytes) {
  const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nbytes) return;
  const long long npx = (long long)g.H * g.W;
  unsigned v = 0;
  for (int k = 0; k < 8; ++k) {
    const long long f = q * 8 + k;
    unsigned bit = 0;
    if (f < npx) {
      const int i = (int)(f / g.W), x = (int)(f - (long long)i * g.W);
      bit = get_bit(mbits, g.pitch_w, i, x);
      if (invert) bit ^= 1u;
    }
    v |= bit << (7 - k);
  }
  out[q] = (unsigned char)v;
}

__global__ void k_bits_differ(const double* a, const double* b, long long n, int* ne) {
  long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  bool d = false;
  for (; k < n; k += (long long)gridDim.x * blockDim.x)
    d |= __double_as_longlong(a[k]) != __double_as_longlong(b[k]);
  if (__any_sync(0xffffffffu, d) && (threadIdx.x & 31) == 0) *ne = 1;
}

// dense region sums over {phi >= 0} / {phi < 0} (grid.py:112-117), per-block
// double-double partials
__global__ void k_region_sums(const double* __restrict__ img, const double* __restrict__ phi,
                              long long n, TilePartial* part) {
  __shared__ TilePartial s_warp[32];
  double ah = 0, al = 0, bh = 0, bl = 0;
  long long na = 0, nb = 0;
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (long long)gridDim.x * blockDim.x) {
    if (phi[k] >= 0.0) { dd_add(ah, al, img[k]); ++na; }
    else { dd_add(bh, bl, img[k]); ++nb; }
  }
  for (int o = 16; o > 0; o >>= 1) {
    double h2 = __shfl_xor_sync(0xffffffffu, ah, o), l2 = __shfl_xor_sync(0xffffffffu, al, o);
    dd_add_dd(ah, al, h2, l2);
    h2 = __shfl_xor_sync(0xffffffffu, bh, o);
    l2 = __shfl_xor_sync(0xffffffffu, bl, o);
    dd_add_dd(bh, bl, h2, l2);
    na += __shfl_xor_sync(0xffffffffu, na, o);
    nb += __shfl_xor_sync(0xffffffffu, nb, o);
  }
  const int warp = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    s_warp[warp].a_hi = ah; s_warp[warp].a_lo = al;
    s_warp[warp].b_hi = bh; s_warp[warp].b_lo = bl;
    s_warp[warp].n_a = na; s_warp[warp].n_b = nb;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    TilePartial t{};
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      dd_add_dd(t.a_hi, t.a_lo, s_warp[w].a_hi, s_warp[w].a_lo);
      dd_add_dd(t.b_hi, t.b_lo, s_warp[w].b_hi, s_warp[w].b_lo);
      t.n_a += s_warp[w].n_a;
      t.n_b += s_warp[w].n_b;
    }
    part[blockIdx.x] = t;
  }
}

}  // namespace lse
