// lse_fast.cuh -- the fused per-iteration kernels of the binary-state path.
//
// One LSE iteration (engine.py:148-174 with reinit_period = reg_period = 1):
//
//   k_update    : b^n (bits) -> phi^n = G*b^n on chip -> |grad phi^n| -> data
//                 term -> u = phi^n + dt v -> b^{n+1} = (u > 0) (bits).
//                 HBM: reads the fp32 data plane (I or g) once, the state bits
//                 (1/8 B/px) and writes 1/8 B/px.
//   k_partition : b^{n+1} -> sign of phi^{n+1} = G*b^{n+1} -> partition bits
//                 {phi >= 0}; incremental c+/c- sums over the pixels that
//                 changed side (sparse exact reads of I); checkpoint mask
//                 {phi > 0} + mismatch count; the last CTA reduces the
//                 fixed-order tile partials and writes the coefficients of
//                 the next update (c+, c-, max|D| closed form, guards) and
//                 the convergence decision (engine.py:228-236).
//
// Arithmetic: phi, |grad phi| and u are evaluated in fp32 with a rigorous
// error bound; any pixel whose decision value lies within that bound of the
// threshold (|u| <= eps_u, |phi| <= eps_phi) is re-evaluated in fp64 with
// the reference's exact operation order (scipy correlate1d order, numpy
// gradient, glibc hypot, no FMA), so every sign decision equals the
// reference's fp64 decision.
#pragma once
#include "lse_device.cuh"

namespace lse {

// Context of the exact (fp64) re-evaluation, resident in device memory.
struct ExactCtx {
  int H, W, R, pitch_w;
  long long data_pitch;
  const float* data32;    // fp32 data plane
  const double* data64;   // exact data (nullptr -> data32 is exact)
  double w64[32];         // w[d] = weight at distance d (R <= 31)
  double dt;
  double scale;           // +-scale state (SRC_SCALED)
  Scalars* scal;
  int model;
};

struct FastParams {
  const uint32_t* bits_in;   // b^n (update) / b^{n+1} (partition)
  uint32_t* bits_out;        // b^{n+1} (update)
  uint32_t* pbits;           // partition bits {phi >= 0}
  uint32_t* mbits;           // checkpoint mask bits {phi > 0}
  const float* data32;
  const float* lut_t;        // fp32 exact vertical-pass value per bit pattern
  const float* lut_s;        // sum of weights of the set bits per pattern
  TilePartial* part;
  Scalars* scal;
  const ExactCtx* ctx;
  RunGeom g;
  float w32[8];
  float dt32;
  float scale32;
  long long iter;            // iteration produced by this launch
};

__device__ __forceinline__ double data_exact(const ExactCtx* c, int i, int x) {
  size_t o = (size_t)i * c->data_pitch + x;
  return c->data64 ? c->data64[o] : (double)c->data32[o];
}

__device__ __noinline__ double exact_phi(const ExactCtx* c, const uint32_t* bits, int src, int i, int x) {
  if (src == SRC_SCALED) return get_bit(bits, c->pitch_w, i, x) ? c->scale : -c->scale;
  return exact_phi_smooth(bits, c->pitch_w, c->H, c->W, c->R, c->w64, i, x);
}

// u = phi + dt * v at (i, x) exactly as _advance_once computes it
// (engine.py:157; models.py:84-90, 101-119; kernels.py:81-95).
__device__ __noinline__ double exact_u(const ExactCtx* c, const uint32_t* bits, int src, int i, int x) {
  const int H = c->H, W = c->W;
  double pc = exact_phi(c, bits, src, i, x);
  double fx, fy;
  if (x == 0) fx = dsub(exact_phi(c, bits, src, i, 1), pc);
  else if (x == W - 1) fx = dsub(pc, exact_phi(c, bits, src, i, W - 2));
  else fx = dmul(dsub(exact_phi(c, bits, src, i, x + 1), exact_phi(c, bits, src, i, x - 1)), 0.5);
  if (i == 0) fy = dsub(exact_phi(c, bits, src, 1, x), pc);
  else if (i == H - 1) fy = dsub(pc, exact_phi(c, bits, src, H - 2, x));
  else fy = dmul(dsub(exact_phi(c, bits, src, i + 1, x), exact_phi(c, bits, src, i - 1, x)), 0.5);
  double h = np_hypot(fx, fy);
  double v;
  const Scalars* sc = c->scal;
  if (c->model == REGION) {
    if (sc->zero_vel) {
      v = 0.0;
    } else {
      double I = data_exact(c, i, x);
      double D = dmul(sc->dc, dsub(dsub(dmul(2.0, I), sc->c_pos), sc->c_neg));
      v = dmul(ddiv(D, sc->peak), h);
    }
  } else {
    v = dmul(data_exact(c, i, x), h);
  }
  atomicAdd(&c->scal->fallbacks, 1ull);
  return dadd(pc, dmul(c->dt, v));
}

// valid-row mask of the window rows i-R .. i+R (bit d <-> row i-R+d)
template <int R>
__device__ __forceinline__ uint32_t row_valid_mask(int i, int H) {
  int lo = R - i;
  lo = lo < 0 ? 0 : lo;
  int hi = H - 1 - i + R;
  hi = hi > 2 * R ? 2 * R : hi;
  if (lo > hi) return 0u;
  return ((2u << hi) - 1u) & ~((1u << lo) - 1u);
}

// One row of phi for NOUT consecutive columns starting at t-index R (the
// t array covers NOUT + 2R columns).  INT: every window row/column lies in
// the image, so the exact-rounded LUT applies; otherwise zero padding
// (b = 0 outside) via the weight-sum LUT: t = 2*S(set & valid) - S(valid).
template <int R, int SRC, bool INT, int NT, int NOUT>
__device__ __forceinline__ void phi_row(const FastParams& P, const uint32_t (&win)[NT],
                                        const uint32_t (&cm)[NT], int m0, int i,
                                        const float* s_lt, const float* s_ls, float (&out)[NOUT]) {
  constexpr uint32_t PM = (1u << (2 * R + 1)) - 1u;
  if (SRC == SRC_SCALED) {
#pragma unroll
    for (int c = 0; c < NOUT; ++c)
      out[c] = ((win[c + R] >> (m0 + R)) & 1u) ? P.scale32 : -P.scale32;
    return;
  }
  uint32_t vr = PM;
  float Lv = 0.f;
  if (!INT) {
    vr = row_valid_mask<R>(i, P.g.H);
    Lv = s_ls[vr];
  }
  float t[NT];
#pragma unroll
  for (int j = 0; j < NT; ++j) {
    uint32_t p = (win[j] >> m0) & PM;
    if (INT) {
      t[j] = s_lt[p];
    } else {
      t[j] = fmaf(2.f, s_ls[p & vr & cm[j]], cm[j] ? -Lv : 0.f);
    }
  }
#pragma unroll
  for (int c = 0; c < NOUT; ++c) {
    float acc = P.w32[0] * t[c + R];
#pragma unroll
    for (int d = 1; d <= R; ++d) acc = fmaf(P.w32[d], t[c + R - d] + t[c + R + d], acc);
    out[c] = acc;
  }
}

template <bool INT>
__device__ __forceinline__ void load_data_row(const FastParams& P, int i, int x0, float (&d)[8]) {
  if (i >= P.g.H) return;
  const float* rowp = P.data32 + (size_t)i * P.g.data_pitch + x0;
  if (INT) {
    float4 a = __ldcs(reinterpret_cast<const float4*>(rowp));
    float4 b = __ldcs(reinterpret_cast<const float4*>(rowp) + 1);
    d[0] = a.x; d[1] = a.y; d[2] = a.z; d[3] = a.w;
    d[4] = b.x; d[5] = b.y; d[6] = b.z; d[7] = b.w;
  } else {
#pragma unroll
    for (int c = 0; c < 8; ++c) d[c] = (x0 + c < P.g.W) ? __ldcs(rowp + c) : 0.f;
  }
}

// ---------------------------------------------------------------- update
template <int R, int MODEL, int SRC, bool INT>
__device__ __forceinline__ void update_tile(const FastParams& P, const uint32_t (*sw)[kSpanMax],
                                            const float* s_lt, const float* s_ls, int r, int x0,
                                            int sbase, float A, float B, float eps_u) {
  constexpr int NT = kColsPerThread + 2 * (R + 1);
  const int H = P.g.H, W = P.g.W;
  const int y0 = r * 32;
  uint32_t cm[NT];
#pragma unroll
  for (int j = 0; j < NT; ++j) {
    int xc = x0 - (R + 1) + j;
    cm[j] = (INT || (xc >= 0 && xc < W)) ? 0xffffffffu : 0u;
  }
  uint32_t win[NT];
  float ra[10], rb[10], rc[10];
  float dcur[8], dnext[8];
  uint32_t ow[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) { ow[c] = 0u; dcur[c] = 0.f; dnext[c] = 0.f; }

  // u on row i from phi rows i-1 (pm), i (p0), i+1 (pp); bit k of the words
  auto u_row = [&](int k, const float (&pm)[10], const float (&p0)[10], const float (&pp)[10],
                   const float (&d)[8]) {
    const int i = y0 + k;
    if (i >= H) return;
    uint32_t fb = 0u;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int x = x0 + c;
      float dx, dy;
      if (INT) {
        dx = p0[c + 2] - p0[c];
        dy = pp[c + 1] - pm[c + 1];
      } else {
        if (x >= W) continue;
        dx = (x == 0) ? 2.f * (p0[c + 2] - p0[c + 1])
                      : (x == W - 1) ? 2.f * (p0[c + 1] - p0[c]) : (p0[c + 2] - p0[c]);
        dy = (i == 0) ? 2.f * (pp[c + 1] - p0[c + 1])
                      : (i == H - 1) ? 2.f * (p0[c + 1] - pm[c + 1]) : (pp[c + 1] - pm[c + 1]);
      }
      float s2 = fmaf(dx, dx, dy * dy);
      float hg = 0.5f * s2 * rsqrtf(fmaxf(s2, 1e-30f));
      float vf = (MODEL == REGION) ? fmaf(A, d[c], B) : d[c];
      float u = fmaf(P.dt32, vf * hg, p0[c + 1]);
      ow[c] |= (u > 0.f ? 1u : 0u) << k;
      if (fabsf(u) <= eps_u) fb |= 1u << c;
    }
    while (fb) {
      const int c = __ffs(fb) - 1;
      fb &= fb - 1;
      double ue = exact_u(P.ctx, P.bits_in, SRC, i, x0 + c);
      ow[c] = (ow[c] & ~(1u << k)) | ((ue > 0.0 ? 1u : 0u) << k);
    }
  };

  // ---- rows -1 .. 15 of phi: window base row y0-1-R
#pragma unroll
  for (int j = 0; j < NT; ++j) win[j] = __funnelshift_r(sw[0][sbase + j], sw[1][sbase + j], 31 - R);
  phi_row<R, SRC, INT, NT, 10>(P, win, cm, 0, y0 - 1, s_lt, s_ls, ra);
  phi_row<R, SRC, INT, NT, 10>(P, win, cm, 1, y0, s_lt, s_ls, rb);
  load_data_row<INT>(P, y0, x0, dcur);
  // three-way register rotation: (ra, rb, rc) = rows (k-1, k, k+1)
  int k = 0;
#pragma unroll 1
  for (; k + 3 <= 15; k += 3) {
    load_data_row<INT>(P, y0 + k + 1, x0, dnext);
    phi_row<R, SRC, INT, NT, 10>(P, win, cm, k + 2, y0 + k + 1, s_lt, s_ls, rc);
    u_row(k, ra, rb, rc, dcur);
    load_data_row<INT>(P, y0 + k + 2, x0, dcur);
    phi_row<R, SRC, INT, NT, 10>(P, win, cm, k + 3, y0 + k + 2, s_lt, s_ls, ra);
    u_row(k + 1, rb, rc, ra, dnext);
    load_data_row<INT>(P, y0 + k + 3, x0, dnext);
    phi_row<R, SRC, INT, NT, 10>(P, win, cm, k + 4, y0 + k + 3, s_lt, s_ls, rb);
    u_row(k + 2, rc, ra, rb, dcur);
#pragma unroll
    for (int c = 0; c < 8; ++c) dcur[c] = dnext[c];
  }
  // k == 15: rows (k-1,k) are in (ra, rb); switch to window base y0+16-R
#pragma unroll
  for (int j = 0; j < NT; ++j) win[j] = __funnelshift_r(sw[1][sbase + j], sw[2][sbase + j], 16 - R);
#pragma unroll 1
  for (; k + 3 <= 30; k += 3) {
    load_data_row<INT>(P, y0 + k + 1, x0, dnext);
    phi_row<R, SRC, INT, NT, 10>(P, win, cm, k + 1 - 16, y0 + k + 1, s_lt, s_ls, rc);
    u_row(k, ra, rb, rc, dcur);
    load_data_row<INT>(P, y0 + k + 2, x0, dcur);
    phi_row<R, SRC, INT, NT, 10>(P, win, cm, k + 2 - 16, y0 + k + 2, s_lt, s_ls, ra);
    u_row(k + 1, rb, rc, ra, dnext);
    load_data_row<INT>(P, y0 + k + 3, x0, dnext);
    phi_row<R, SRC, INT, NT, 10>(P, win, cm, k + 3 - 16, y0 + k + 3, s_lt, s_ls, rb);
    u_row(k + 2, rc, ra, rb, dcur);
#pragma unroll
    for (int c = 0; c < 8; ++c) dcur[c] = dnext[c];
  }
  // k == 30, 31
  load_data_row<INT>(P, y0 + 31, x0, dnext);
  phi_row<R, SRC, INT, NT, 10>(P, win, cm, 31 - 16, y0 + 31, s_lt, s_ls, rc);
  u_row(30, ra, rb, rc, dcur);
  phi_row<R, SRC, INT, NT, 10>(P, win, cm, 32 - 16, y0 + 32, s_lt, s_ls, ra);
  u_row(31, rb, rc, ra, dnext);

  uint32_t* dst = P.bits_out + (size_t)r * P.g.pitch_w + x0;
  if (!INT) {
#pragma unroll
    for (int c = 0; c < 8; ++c) if (x0 + c >= W) ow[c] = 0u;
  }
  reinterpret_cast<uint4*>(dst)[0] = make_uint4(ow[0], ow[1], ow[2], ow[3]);
  reinterpret_cast<uint4*>(dst)[1] = make_uint4(ow[4], ow[5], ow[6], ow[7]);
}

__device__ __forceinline__ void stage_words(const uint32_t* bits, const RunGeom& g, int r, int cx0,
                                            uint32_t (*sw)[kSpanMax]) {
  const int span = kColsPerThread * blockDim.x + 16;
  for (int q = threadIdx.x; q < 3 * span; q += blockDim.x) {
    int rr = q / span;
    int cc = q - rr * span;
    int x = cx0 - 8 + cc;
    int wr = r - 1 + rr;
    uint32_t v = 0u;
    if (x >= 0 && x < g.W && wr >= 0 && wr < g.HR) v = __ldg(&bits[(size_t)wr * g.pitch_w + x]);
    sw[rr][cc] = v;
  }
}

template <int R>
__device__ __forceinline__ void load_luts(const FastParams& P, float* s_lt, float* s_ls) {
  constexpr int NPAT = 1 << (2 * R + 1);
  for (int q = threadIdx.x; q < NPAT; q += blockDim.x) {
    s_lt[q] = __ldg(&P.lut_t[q]);
    s_ls[q] = __ldg(&P.lut_s[q]);
  }
}

template <int R, int MODEL, int SRC>
__global__ void __launch_bounds__(kThreads) k_update(FastParams P) {
  constexpr int NPAT = 1 << (2 * R + 1);
  __shared__ float s_lt[NPAT], s_ls[NPAT];
  __shared__ uint32_t sw[3][kSpanMax];
  const Scalars* sc = P.scal;
  if (*(volatile const int*)&sc->stop) return;
  if (MODEL == REGION && blockIdx.x == 0 && threadIdx.x == 0 && sc->zero_vel) P.scal->degenerate = 1;
  const float A = sc->A, B = sc->B, eps_u = sc->eps_u;
  load_luts<R>(P, s_lt, s_ls);
  const int cbw = kColsPerThread * blockDim.x;
  for (int tile = blockIdx.x; tile < P.g.ntiles; tile += gridDim.x) {
    const int r = tile / P.g.ncb;
    const int cx0 = (tile - r * P.g.ncb) * cbw;
    __syncthreads();
    stage_words(P.bits_in, P.g, r, cx0, sw);
    __syncthreads();
    const int x0 = cx0 + kColsPerThread * threadIdx.x;
    if (x0 >= P.g.W) continue;
    const int y0 = r * 32;
    const int wx0 = cx0 + kColsPerThread * (threadIdx.x & ~31);
    const int wx1 = wx0 + kColsPerThread * 32 - 1;
    const bool interior = SRC == SRC_SMOOTH && y0 - 1 - R >= 0 && y0 + 32 + R <= P.g.H - 1 &&
                          wx0 - (R + 1) >= 0 && wx1 + (R + 1) <= P.g.W - 1;
    const int sbase = x0 - cx0 + 8 - (R + 1);
    if (interior) update_tile<R, MODEL, SRC, true>(P, sw, s_lt, s_ls, r, x0, sbase, A, B, eps_u);
    else update_tile<R, MODEL, SRC, false>(P, sw, s_lt, s_ls, r, x0, sbase, A, B, eps_u);
  }
}

// ------------------------------------------------------------- finalize
// Region coefficients of the next update from the running sums.
__device__ inline void region_coeffs(Scalars* sc) {
  const long long np = sc->n_pos, nn = sc->n_total - sc->n_pos;
  const double dt = sc->dt;
  sc->zero_vel = 0;
  if (np == 0 || nn == 0) {                       // grid.py:114-115, models.py:111-113
    sc->zero_vel = 1;
  } else {
    double cp = dd_div(sc->sp_hi, sc->sp_lo, (double)np);
    double cm = dd_div(sc->sn_hi, sc->sn_lo, (double)nn);
    double dc = dsub(cp, cm);
    // max |D| over the image (models.py:116) is attained at the extreme
    // intensities: D(I) is monotone in I under round-to-nearest.
    double dmax = fabs(dmul(dc, dsub(dsub(dmul(2.0, sc->img_max), cp), cm)));
    double dmin = fabs(dmul(dc, dsub(dsub(dmul(2.0, sc->img_min), cp), cm)));
    double peak = dmax > dmin ? dmax : dmin;
    sc->c_pos = cp;
    sc->c_neg = cm;
    sc->dc = dc;
    sc->peak = peak;
    if (peak == 0.0) {                             // models.py:117-118
      sc->zero_vel = 1;
    } else {
      double a = 2.0 * dc / peak;
      double b = -dc * (cp + cm) / peak;
      sc->A = (float)a;
      sc->B = (float)b;
      double eps_d = 0x1p-21 * (fabs(a) * sc->img_absmax + fabs(b) + 1.0);
      sc->eps_u = (float)(4.0 * (0x1p-18 + dt * (0x1p-16 + 1.5 * eps_d + 0x1p-21) +
                                 0x1p-22 * (1.0 + 1.5 * dt)));
    }
  }
  if (sc->zero_vel) {
    sc->A = 0.f;
    sc->B = 0.f;
    sc->eps_u = (float)(4.0 * (0x1p-18 + 0x1p-22));
  }
}

// Whole-CTA reduction of the tile partials in a fixed order, then the
// scalar bookkeeping (single thread).
__device__ void finalize_cta(const TilePartial* part, int n, Scalars* sc, bool delta, bool region,
                             bool ckpt, long long iter) {
  __shared__ double f_ah[kThreads], f_al[kThreads], f_bh[kThreads], f_bl[kThreads];
  __shared__ long long f_na[kThreads], f_nb[kThreads];
  __shared__ unsigned long long f_mm[kThreads];
  const int T = blockDim.x, tid = threadIdx.x;
  double ah = 0, al = 0, bh = 0, bl = 0;
  long long na = 0, nb = 0;
  unsigned long long mm = 0;
  const int per = (n + T - 1) / T;
  const int lo = tid * per;
  const int hi = lo + per < n ? lo + per : n;
  for (int t = lo; t < hi; ++t) {
    const TilePartial* q = part + t;
    dd_add_dd(ah, al, __ldcg(&q->a_hi), __ldcg(&q->a_lo));
    dd_add_dd(bh, bl, __ldcg(&q->b_hi), __ldcg(&q->b_lo));
    na += __ldcg(&q->n_a);
    nb += __ldcg(&q->n_b);
    mm += __ldcg(&q->mism);
  }
  f_ah[tid] = ah; f_al[tid] = al; f_bh[tid] = bh; f_bl[tid] = bl;
  f_na[tid] = na; f_nb[tid] = nb; f_mm[tid] = mm;
  __syncthreads();
  for (int s = T / 2; s > 0; s >>= 1) {
    if (tid < s) {
      double h1 = f_ah[tid], l1 = f_al[tid];
      dd_add_dd(h1, l1, f_ah[tid + s], f_al[tid + s]);
      f_ah[tid] = h1; f_al[tid] = l1;
      double h2 = f_bh[tid], l2 = f_bl[tid];
      dd_add_dd(h2, l2, f_bh[tid + s], f_bl[tid + s]);
      f_bh[tid] = h2; f_bl[tid] = l2;
      f_na[tid] += f_na[tid + s];
      f_nb[tid] += f_nb[tid + s];
      f_mm[tid] += f_mm[tid + s];
    }
    __syncthreads();
  }
  if (tid == 0) {
    if (region) {
      if (delta) {
        dd_add_dd(sc->sp_hi, sc->sp_lo, f_ah[0], f_al[0]);
        dd_add_dd(sc->sp_hi, sc->sp_lo, -f_bh[0], -f_bl[0]);
        dd_add_dd(sc->sn_hi, sc->sn_lo, f_bh[0], f_bl[0]);
        dd_add_dd(sc->sn_hi, sc->sn_lo, -f_ah[0], -f_al[0]);
        sc->n_pos += f_na[0] - f_nb[0];
      } else {
        sc->sp_hi = f_ah[0]; sc->sp_lo = f_al[0];
        sc->sn_hi = f_bh[0]; sc->sn_lo = f_bl[0];
        sc->n_pos = f_na[0];
      }
      region_coeffs(sc);
    }
    if (ckpt) {                                    // engine.py:228-236
      sc->n_ckpt += 1;
      if (sc->n_ckpt >= 2) sc->equal_run = (f_mm[0] == 0) ? sc->equal_run + 1 : 0;
      const long long cw = sc->conv_window;
      if (cw == 1 || (sc->n_ckpt >= cw && sc->equal_run >= cw - 1)) {
        sc->stop = 1;
        sc->converged = 1;
        sc->converged_iter = iter;
      }
    }
    sc->ticket = 0u;
    __threadfence();
  }
}

// ------------------------------------------------------------- partition
template <int R, bool INT, bool PART, bool CKPT, bool MASKONLY>
__device__ __forceinline__ void partition_tile(const FastParams& P, const uint32_t (*sw)[kSpanMax],
                                               const float* s_lt, const float* s_ls, int r, int x0,
                                               int sbase, float eps_phi, double& acc_in,
                                               double& acc_out, long long& n_in, long long& n_out,
                                               unsigned long long& mism) {
  constexpr int NT = kColsPerThread + 2 * R;
  const int H = P.g.H, W = P.g.W;
  const int y0 = r * 32;
  uint32_t cm[NT];
#pragma unroll
  for (int j = 0; j < NT; ++j) {
    int xc = x0 - R + j;
    cm[j] = (INT || (xc >= 0 && xc < W)) ? 0xffffffffu : 0u;
  }
  uint32_t win[NT];
  uint32_t pw[8], mw[8];
  float ph[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) { pw[c] = 0u; mw[c] = 0u; }
  auto do_row = [&](int k, int m0) {
    const int i = y0 + k;
    if (i >= H) return;
    phi_row<R, SRC_SMOOTH, INT, NT, 8>(P, win, cm, m0, i, s_lt, s_ls, ph);
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      if (!INT && x0 + c >= W) continue;
      const float f = ph[c];
      uint32_t ge, gt;
      if (fabsf(f) <= eps_phi) {
        double e = exact_phi(P.ctx, P.bits_in, SRC_SMOOTH, i, x0 + c);
        ge = e >= 0.0;
        gt = e > 0.0;
        atomicAdd(&P.scal->fallbacks, 1ull);
      } else {
        ge = gt = f > 0.f;
      }
      pw[c] |= ge << k;
      mw[c] |= gt << k;
    }
  };
#pragma unroll
  for (int j = 0; j < NT; ++j) win[j] = __funnelshift_r(sw[0][sbase + j], sw[1][sbase + j], 32 - R);
#pragma unroll 1
  for (int k = 0; k < 16; ++k) do_row(k, k);
#pragma unroll
  for (int j = 0; j < NT; ++j) win[j] = __funnelshift_r(sw[1][sbase + j], sw[2][sbase + j], 16 - R);
#pragma unroll 1
  for (int k = 16; k < 32; ++k) do_row(k, k - 16);

  const size_t base = (size_t)r * P.g.pitch_w + x0;
  if (PART) {
    uint4 o0 = reinterpret_cast<const uint4*>(P.pbits + base)[0];
    uint4 o1 = reinterpret_cast<const uint4*>(P.pbits + base)[1];
    uint32_t old[8] = {o0.x, o0.y, o0.z, o0.w, o1.x, o1.y, o1.z, o1.w};
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      if (!INT && x0 + c >= W) { pw[c] = 0u; continue; }
      uint32_t ch = old[c] ^ pw[c];
      while (ch) {
        const int b = __ffs(ch) - 1;
        ch &= ch - 1;
        const double I = data_exact(P.ctx, y0 + b, x0 + c);
        if ((pw[c] >> b) & 1u) { acc_in += I; ++n_in; }
        else { acc_out += I; ++n_out; }
      }
    }
    reinterpret_cast<uint4*>(P.pbits + base)[0] = make_uint4(pw[0], pw[1], pw[2], pw[3]);
    reinterpret_cast<uint4*>(P.pbits + base)[1] = make_uint4(pw[4], pw[5], pw[6], pw[7]);
  }
  if (MASKONLY) {
#pragma unroll
    for (int c = 0; c < 8; ++c)
      if (!INT && x0 + c >= W) mw[c] = 0u;
    reinterpret_cast<uint4*>(P.mbits + base)[0] = make_uint4(mw[0], mw[1], mw[2], mw[3]);
    reinterpret_cast<uint4*>(P.mbits + base)[1] = make_uint4(mw[4], mw[5], mw[6], mw[7]);
  } else if (CKPT) {
    uint4 o0 = reinterpret_cast<const uint4*>(P.mbits + base)[0];
    uint4 o1 = reinterpret_cast<const uint4*>(P.mbits + base)[1];
    uint32_t old[8] = {o0.x, o0.y, o0.z, o0.w, o1.x, o1.y, o1.z, o1.w};
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      if (!INT && x0 + c >= W) mw[c] = 0u;
      mism += __popc(old[c] ^ mw[c]);
    }
    reinterpret_cast<uint4*>(P.mbits + base)[0] = make_uint4(mw[0], mw[1], mw[2], mw[3]);
    reinterpret_cast<uint4*>(P.mbits + base)[1] = make_uint4(mw[4], mw[5], mw[6], mw[7]);
  }
}

// Deterministic CTA reduction of the per-thread partials into one tile
// partial (fixed shuffle pattern, warps combined in index order).
__device__ __forceinline__ void cta_tile_partial(TilePartial* dst, double a, double b, long long na,
                                                 long long nb, unsigned long long mm,
                                                 TilePartial* s_w) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
    na += __shfl_xor_sync(0xffffffffu, na, o);
    nb += __shfl_xor_sync(0xffffffffu, nb, o);
    mm += __shfl_xor_sync(0xffffffffu, mm, o);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    s_w[warp].a_hi = a; s_w[warp].b_hi = b;
    s_w[warp].n_a = na; s_w[warp].n_b = nb; s_w[warp].mism = mm;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    TilePartial t{};
    double ah = 0, al = 0, bh = 0, bl = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      dd_add(ah, al, s_w[w].a_hi);
      dd_add(bh, bl, s_w[w].b_hi);
      t.n_a += s_w[w].n_a;
      t.n_b += s_w[w].n_b;
      t.mism += s_w[w].mism;
    }
    t.a_hi = ah; t.a_lo = al; t.b_hi = bh; t.b_lo = bl;
    *dst = t;
  }
}

template <int R, bool PART, bool CKPT, bool MASKONLY>
__global__ void __launch_bounds__(kThreads) k_partition(FastParams P) {
  constexpr int NPAT = 1 << (2 * R + 1);
  __shared__ float s_lt[NPAT], s_ls[NPAT];
  __shared__ uint32_t sw[3][kSpanMax];
  __shared__ TilePartial s_warp[kThreads / 32];
  __shared__ unsigned int s_ticket;
  Scalars* sc = P.scal;
  if (!MASKONLY && *(volatile const int*)&sc->stop) return;
  const float eps_phi = sc->eps_phi;
  load_luts<R>(P, s_lt, s_ls);
  const int cbw = kColsPerThread * blockDim.x;
  for (int tile = blockIdx.x; tile < P.g.ntiles; tile += gridDim.x) {
    const int r = tile / P.g.ncb;
    const int cx0 = (tile - r * P.g.ncb) * cbw;
    __syncthreads();
    stage_words(P.bits_in, P.g, r, cx0, sw);
    __syncthreads();
    const int x0 = cx0 + kColsPerThread * threadIdx.x;
    double a = 0.0, b = 0.0;
    long long na = 0, nb = 0;
    unsigned long long mm = 0;
    if (x0 < P.g.W) {
      const int y0 = r * 32;
      const int wx0 = cx0 + kColsPerThread * (threadIdx.x & ~31);
      const int wx1 = wx0 + kColsPerThread * 32 - 1;
      const bool interior = y0 - R >= 0 && y0 + 31 + R <= P.g.H - 1 && wx0 - R >= 0 &&
                            wx1 + R <= P.g.W - 1;
      const int sbase = x0 - cx0 + 8 - R;
      if (interior)
        partition_tile<R, true, PART, CKPT, MASKONLY>(P, sw, s_lt, s_ls, r, x0, sbase, eps_phi, a, b, na, nb, mm);
      else
        partition_tile<R, false, PART, CKPT, MASKONLY>(P, sw, s_lt, s_ls, r, x0, sbase, eps_phi, a, b, na, nb, mm);
    }
    if (!MASKONLY) cta_tile_partial(P.part + tile, a, b, na, nb, mm, s_warp);
  }
  if (MASKONLY) return;
  // last CTA to finish reduces every tile partial (threadFenceReduction idiom)
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_ticket = atomicAdd(&sc->ticket, 1u);
  }
  __syncthreads();
  if (s_ticket == gridDim.x - 1) {
    __threadfence();
    finalize_cta(P.part, P.g.ntiles, sc, /*delta=*/true, PART, CKPT, P.iter);
  }
}

}  // namespace lse
