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
  int skip_uniform;          // skip warp blocks whose whole stencil window is uniform
  int nchunk;                // 256-column chunks per word-row
  int nseg;                  // partition segments (kSegChunks chunks) per word-row
};

constexpr int kChunk = 256;      // columns per warp chunk (32 lanes x 8 columns)
constexpr int kSegChunks = 16;   // chunks per partition segment (partial granularity)

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

// One row of phi for NOUT consecutive columns; the t array covers NOUT + 2R
// columns and phi column c is centred on t index c + R.  INT: all window rows
// and columns lie in the image, so the exact-rounded LUT applies; otherwise
// zero padding (b = 0 outside) via the weight-sum LUT:
// t = 2*S(set & valid) - S(valid).
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
    const uint32_t p = (win[j] >> m0) & PM;
    if (INT) t[j] = s_lt[p];
    else t[j] = fmaf(2.f, s_ls[p & vr & cm[j]], cm[j] ? -Lv : 0.f);
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
    const float4 a = __ldcs(reinterpret_cast<const float4*>(rowp));
    const float4 b = __ldcs(reinterpret_cast<const float4*>(rowp) + 1);
    d[0] = a.x; d[1] = a.y; d[2] = a.z; d[3] = a.w;
    d[4] = b.x; d[5] = b.y; d[6] = b.z; d[7] = b.w;
  } else {
#pragma unroll
    for (int c = 0; c < 8; ++c) d[c] = (x0 + c < P.g.W) ? __ldcs(rowp + c) : 0.f;
  }
}

__device__ __forceinline__ float sqrt_approx(float x) {
  float y;
  asm("sqrt.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// state words of column xc in word-row wr (0 outside the image)
template <bool INT>
__device__ __forceinline__ uint32_t word_at(const FastParams& P, int wr, int xc) {
  if (!INT && (wr < 0 || wr >= P.g.HR || xc < 0 || xc >= P.g.W)) return 0u;
  return __ldg(&P.bits_in[(size_t)wr * P.g.pitch_w + xc]);
}

// ---------------------------------------------------------------- update
// One lane: columns x0..x0+7 of word-row r (32 rows).  phi rows -1..32 are
// rebuilt from the bit state (t columns x0-R-1 .. x0+8+R); three phi rows
// are kept in registers while walking down the rows.
template <int R, int MODEL, int SRC, bool INT>
__device__ __forceinline__ void update_block(const FastParams& P, const float* s_lt,
                                             const float* s_ls, int r, int x0, float A, float B,
                                             float eps_u, const uint32_t (&prev)[8 + 2 * (R + 1)],
                                             const uint32_t (&cur)[8 + 2 * (R + 1)]) {
  constexpr int NT = kColsPerThread + 2 * (R + 1);
  const int H = P.g.H, W = P.g.W;
  const int y0 = r * 32;
  const float hdt = 0.5f * P.dt32;        // h below is 2|grad phi|
  uint32_t cm[NT], win[NT];
#pragma unroll
  for (int j = 0; j < NT; ++j) {
    const int xc = x0 - (R + 1) + j;
    cm[j] = (INT || (xc >= 0 && xc < W)) ? 0xffffffffu : 0u;
    win[j] = __funnelshift_r(prev[j], cur[j], 31 - R);   // base row y0-1-R
  }
  float pm[10], p0[10], pn[10], dcur[8], dnext[8];
  uint32_t ow[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) { ow[c] = 0u; dcur[c] = 0.f; dnext[c] = 0.f; }
  phi_row<R, SRC, INT, NT, 10>(P, win, cm, 0, y0 - 1, s_lt, s_ls, pm);
  phi_row<R, SRC, INT, NT, 10>(P, win, cm, 1, y0, s_lt, s_ls, p0);
  load_data_row<INT>(P, y0, x0, dcur);
#pragma unroll 1
  for (int k = 0; k < 32; ++k) {
    const int kk = k + 1;                  // phi row produced in this step
    if (kk == 16) {                        // switch to window base y0+16-R
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        const int xc = x0 - (R + 1) + j;
        win[j] = __funnelshift_r(word_at<INT>(P, r, xc), word_at<INT>(P, r + 1, xc), 16 - R);
      }
    }
    const int m0 = kk < 16 ? kk + 1 : kk - 16;
    if (kk < 32) load_data_row<INT>(P, y0 + kk, x0, dnext);
    phi_row<R, SRC, INT, NT, 10>(P, win, cm, m0, y0 + kk, s_lt, s_ls, pn);
    const int i = y0 + k;
    if (i < H) {
      const uint32_t bitk = 1u << k;
      uint32_t fb = 0u;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const int x = x0 + c;
        float dx, dy;
        if (INT) {
          dx = p0[c + 2] - p0[c];
          dy = pn[c + 1] - pm[c + 1];
        } else {
          if (x >= W) continue;
          dx = (x == 0) ? 2.f * (p0[c + 2] - p0[c + 1])
                        : (x == W - 1) ? 2.f * (p0[c + 1] - p0[c]) : (p0[c + 2] - p0[c]);
          dy = (i == 0) ? 2.f * (pn[c + 1] - p0[c + 1])
                        : (i == H - 1) ? 2.f * (p0[c + 1] - pm[c + 1]) : (pn[c + 1] - pm[c + 1]);
        }
        const float h = sqrt_approx(fmaf(dx, dx, dy * dy));
        const float vf = (MODEL == REGION) ? fmaf(A, dcur[c], B) : dcur[c];
        const float u = fmaf(hdt, vf * h, p0[c + 1]);
        if (u > 0.f) ow[c] |= bitk;
        if (fabsf(u) <= eps_u) fb |= 1u << c;
      }
      while (fb) {                          // near-tie: exact fp64 decision
        const int c = __ffs(fb) - 1;
        fb &= fb - 1;
        const double ue = exact_u(P.ctx, P.bits_in, SRC, i, x0 + c);
        ow[c] = ue > 0.0 ? (ow[c] | bitk) : (ow[c] & ~bitk);
      }
    }
#pragma unroll
    for (int c = 0; c < 10; ++c) { pm[c] = p0[c]; p0[c] = pn[c]; }
#pragma unroll
    for (int c = 0; c < 8; ++c) dcur[c] = dnext[c];
  }
  if (!INT) {
#pragma unroll
    for (int c = 0; c < 8; ++c) if (x0 + c >= W) ow[c] = 0u;
  }
  uint32_t* dst = P.bits_out + (size_t)r * P.g.pitch_w + x0;
  reinterpret_cast<uint4*>(dst)[0] = make_uint4(ow[0], ow[1], ow[2], ow[3]);
  reinterpret_cast<uint4*>(dst)[1] = make_uint4(ow[4], ow[5], ow[6], ow[7]);
}

template <int R>
__device__ __forceinline__ void load_luts(const FastParams& P, float* s_lt, float* s_ls) {
  constexpr int NPAT = 1 << (2 * R + 1);
  for (int q = threadIdx.x; q < NPAT; q += blockDim.x) {
    s_lt[q] = __ldg(&P.lut_t[q]);
    s_ls[q] = __ldg(&P.lut_s[q]);
  }
}

// Work unit = (word-row, 256-column chunk), one warp each, grid-strided.  A
// chunk whose every lane sees a uniform stencil window (all bits of rows
// y0-32 .. y0+63 equal over its t columns, away from the image border) has
// phi constant there, hence |grad phi| == 0, v == 0 and u == phi exactly, so
// b^{n+1} == b^n: the chunk is copied without touching the data plane.
template <int R, int MODEL, int SRC>
__global__ void __launch_bounds__(kThreads, 4) k_update(FastParams P) {
  constexpr int NPAT = 1 << (2 * R + 1);
  constexpr int NT = kColsPerThread + 2 * (R + 1);
  __shared__ float s_lt[NPAT], s_ls[NPAT];
  const Scalars* sc = P.scal;
  if (*(volatile const int*)&sc->stop) return;
  if (MODEL == REGION && blockIdx.x == 0 && threadIdx.x == 0 && sc->zero_vel) P.scal->degenerate = 1;
  const float A = sc->A, B = sc->B, eps_u = sc->eps_u;
  load_luts<R>(P, s_lt, s_ls);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int nwarp = gridDim.x * (blockDim.x >> 5);
  const int nunits = P.g.HR * P.nchunk;
  for (int unit = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); unit < nunits;
       unit += nwarp) {
    const int r = unit / P.nchunk;
    const int cx = (unit - r * P.nchunk) * kChunk;
    const int x0 = cx + kColsPerThread * lane;
    const int y0 = r * 32;
    const bool interior = SRC == SRC_SMOOTH && y0 - 1 - R >= 0 && y0 + 32 + R <= P.g.H - 1 &&
                          cx - (R + 1) >= 0 && cx + kChunk - 1 + (R + 1) <= P.g.W - 1;
    uint32_t prev[NT], cur[NT];
    if (interior) {
      uint32_t a = ~0u, o = 0u;
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        const int xc = x0 - (R + 1) + j;
        prev[j] = word_at<true>(P, r - 1, xc);
        cur[j] = word_at<true>(P, r, xc);
        const uint32_t nx = word_at<true>(P, r + 1, xc);
        a &= prev[j] & cur[j] & nx;
        o |= prev[j] | cur[j] | nx;
      }
      if (P.skip_uniform && __all_sync(0xffffffffu, a == ~0u || o == 0u)) {
        uint32_t* dst = P.bits_out + (size_t)r * P.g.pitch_w + x0;
        reinterpret_cast<uint4*>(dst)[0] = make_uint4(cur[R + 1], cur[R + 2], cur[R + 3], cur[R + 4]);
        reinterpret_cast<uint4*>(dst)[1] = make_uint4(cur[R + 5], cur[R + 6], cur[R + 7], cur[R + 8]);
        continue;
      }
      update_block<R, MODEL, SRC, true>(P, s_lt, s_ls, r, x0, A, B, eps_u, prev, cur);
    } else {
      if (x0 >= P.g.W) continue;
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        const int xc = x0 - (R + 1) + j;
        prev[j] = word_at<false>(P, r - 1, xc);
        cur[j] = word_at<false>(P, r, xc);
      }
      update_block<R, MODEL, SRC, false>(P, s_lt, s_ls, r, x0, A, B, eps_u, prev, cur);
    }
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
// One lane: columns x0..x0+7 of word-row r.  Signs of phi^{n+1} = G*b^{n+1}
// (t columns x0-R .. x0+7+R, no row halo), partition bits {phi >= 0} with the
// incremental c+/c- sums, checkpoint mask {phi > 0} with the mismatch count.
template <int R, bool INT>
__device__ __forceinline__ void partition_block(const FastParams& P, const float* s_lt,
                                                const float* s_ls, int r, int x0, float eps_phi,
                                                const uint32_t (&prev)[8 + 2 * R],
                                                const uint32_t (&cur)[8 + 2 * R],
                                                uint32_t (&pw)[8], uint32_t (&mw)[8]) {
  constexpr int NT = kColsPerThread + 2 * R;
  const int H = P.g.H, W = P.g.W;
  const int y0 = r * 32;
  uint32_t cm[NT], win[NT];
#pragma unroll
  for (int j = 0; j < NT; ++j) {
    const int xc = x0 - R + j;
    cm[j] = (INT || (xc >= 0 && xc < W)) ? 0xffffffffu : 0u;
    win[j] = __funnelshift_r(prev[j], cur[j], 32 - R);     // base row y0-R
  }
  float ph[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) { pw[c] = 0u; mw[c] = 0u; }
#pragma unroll 1
  for (int k = 0; k < 32; ++k) {
    if (k == 16) {                                          // base row y0+16-R
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        const int xc = x0 - R + j;
        win[j] = __funnelshift_r(word_at<INT>(P, r, xc), word_at<INT>(P, r + 1, xc), 16 - R);
      }
    }
    const int i = y0 + k;
    if (i >= H) break;
    phi_row<R, SRC_SMOOTH, INT, NT, 8>(P, win, cm, k < 16 ? k : k - 16, i, s_lt, s_ls, ph);
    const uint32_t bitk = 1u << k;
    uint32_t fb = 0u;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      if (!INT && x0 + c >= W) continue;
      if (ph[c] > 0.f) { pw[c] |= bitk; mw[c] |= bitk; }
      if (fabsf(ph[c]) <= eps_phi) fb |= 1u << c;
    }
    while (fb) {
      const int c = __ffs(fb) - 1;
      fb &= fb - 1;
      const double e = exact_phi(P.ctx, P.bits_in, SRC_SMOOTH, i, x0 + c);
      atomicAdd(&P.scal->fallbacks, 1ull);
      pw[c] = e >= 0.0 ? (pw[c] | bitk) : (pw[c] & ~bitk);
      mw[c] = e > 0.0 ? (mw[c] | bitk) : (mw[c] & ~bitk);
    }
  }
}

// Work unit = (word-row, segment of kSegChunks chunks), one warp each; the
// warp's deltas over the segment form one partial (fixed geometry =>
// deterministic and independent of how the rows are split across GPUs).
template <int R, bool PART, bool CKPT, bool MASKONLY>
__global__ void __launch_bounds__(kThreads, 4) k_partition(FastParams P) {
  constexpr int NPAT = 1 << (2 * R + 1);
  constexpr int NT = kColsPerThread + 2 * R;
  __shared__ float s_lt[NPAT], s_ls[NPAT];
  __shared__ unsigned int s_ticket;
  Scalars* sc = P.scal;
  if (!MASKONLY && *(volatile const int*)&sc->stop) return;
  const float eps_phi = sc->eps_phi;
  load_luts<R>(P, s_lt, s_ls);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int nwarp = gridDim.x * (blockDim.x >> 5);
  const int nunits = P.g.HR * P.nseg;
  for (int unit = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); unit < nunits;
       unit += nwarp) {
    const int r = unit / P.nseg;
    const int seg = unit - r * P.nseg;
    double a_in = 0.0, a_out = 0.0;
    long long n_in = 0, n_out = 0;
    unsigned long long mism = 0;
    for (int ch = seg * kSegChunks; ch < (seg + 1) * kSegChunks && ch < P.nchunk; ++ch) {
      const int cx = ch * kChunk;
      const int x0 = cx + kColsPerThread * lane;
      const int y0 = r * 32;
      const bool interior = y0 - R >= 0 && y0 + 31 + R <= P.g.H - 1 && cx - R >= 0 &&
                            cx + kChunk - 1 + R <= P.g.W - 1;
      uint32_t pw[8], mw[8], prev[NT], cur[NT];
      if (interior) {
        uint32_t a = ~0u, o = 0u;
#pragma unroll
        for (int j = 0; j < NT; ++j) {
          const int xc = x0 - R + j;
          prev[j] = word_at<true>(P, r - 1, xc);
          cur[j] = word_at<true>(P, r, xc);
          const uint32_t nx = word_at<true>(P, r + 1, xc);
          a &= prev[j] & cur[j] & nx;
          o |= prev[j] | cur[j] | nx;
        }
        if (P.skip_uniform && __all_sync(0xffffffffu, a == ~0u || o == 0u)) {
          // phi = +-c everywhere in the block: sign(phi) = b
#pragma unroll
          for (int c = 0; c < 8; ++c) pw[c] = mw[c] = cur[R + c];
        } else {
          partition_block<R, true>(P, s_lt, s_ls, r, x0, eps_phi, prev, cur, pw, mw);
        }
      } else {
        if (x0 >= P.g.W) continue;
#pragma unroll
        for (int j = 0; j < NT; ++j) {
          const int xc = x0 - R + j;
          prev[j] = word_at<false>(P, r - 1, xc);
          cur[j] = word_at<false>(P, r, xc);
        }
        partition_block<R, false>(P, s_lt, s_ls, r, x0, eps_phi, prev, cur, pw, mw);
        if (x0 + 8 > P.g.W) {
#pragma unroll
          for (int c = 0; c < 8; ++c) if (x0 + c >= P.g.W) { pw[c] = 0u; mw[c] = 0u; }
        }
      }
      const size_t base = (size_t)r * P.g.pitch_w + x0;
      if (MASKONLY) {
        reinterpret_cast<uint4*>(P.mbits + base)[0] = make_uint4(mw[0], mw[1], mw[2], mw[3]);
        reinterpret_cast<uint4*>(P.mbits + base)[1] = make_uint4(mw[4], mw[5], mw[6], mw[7]);
        continue;
      }
      if (PART) {
        const uint4 o0 = reinterpret_cast<const uint4*>(P.pbits + base)[0];
        const uint4 o1 = reinterpret_cast<const uint4*>(P.pbits + base)[1];
        const uint32_t old[8] = {o0.x, o0.y, o0.z, o0.w, o1.x, o1.y, o1.z, o1.w};
        uint32_t any = 0u;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          uint32_t ch2 = old[c] ^ pw[c];
          any |= ch2;
          while (ch2) {
            const int b = __ffs(ch2) - 1;
            ch2 &= ch2 - 1;
            const double I = data_exact(P.ctx, y0 + b, x0 + c);
            if ((pw[c] >> b) & 1u) { a_in += I; ++n_in; }
            else { a_out += I; ++n_out; }
          }
        }
        if (any) {
          reinterpret_cast<uint4*>(P.pbits + base)[0] = make_uint4(pw[0], pw[1], pw[2], pw[3]);
          reinterpret_cast<uint4*>(P.pbits + base)[1] = make_uint4(pw[4], pw[5], pw[6], pw[7]);
        }
      }
      if (CKPT) {
        const uint4 o0 = reinterpret_cast<const uint4*>(P.mbits + base)[0];
        const uint4 o1 = reinterpret_cast<const uint4*>(P.mbits + base)[1];
        const uint32_t old[8] = {o0.x, o0.y, o0.z, o0.w, o1.x, o1.y, o1.z, o1.w};
#pragma unroll
        for (int c = 0; c < 8; ++c) mism += __popc(old[c] ^ mw[c]);
        reinterpret_cast<uint4*>(P.mbits + base)[0] = make_uint4(mw[0], mw[1], mw[2], mw[3]);
        reinterpret_cast<uint4*>(P.mbits + base)[1] = make_uint4(mw[4], mw[5], mw[6], mw[7]);
      }
    }
    if (MASKONLY) continue;
    // warp partial for this unit (fixed xor-shuffle order)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a_in += __shfl_xor_sync(0xffffffffu, a_in, o);
      a_out += __shfl_xor_sync(0xffffffffu, a_out, o);
      n_in += __shfl_xor_sync(0xffffffffu, n_in, o);
      n_out += __shfl_xor_sync(0xffffffffu, n_out, o);
      mism += __shfl_xor_sync(0xffffffffu, mism, o);
    }
    if (lane == 0) {
      TilePartial t{};
      t.a_hi = a_in;
      t.b_hi = a_out;
      t.n_a = n_in;
      t.n_b = n_out;
      t.mism = mism;
      P.part[unit] = t;
    }
  }
  if (MASKONLY) return;
  // last CTA to finish reduces every unit partial (threadFenceReduction idiom)
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_ticket = atomicAdd(&sc->ticket, 1u);
  }
  __syncthreads();
  if (s_ticket == gridDim.x - 1) {
    __threadfence();
    finalize_cta(P.part, nunits, sc, /*delta=*/true, PART, CKPT, P.iter);
  }
}

}  // namespace lse
