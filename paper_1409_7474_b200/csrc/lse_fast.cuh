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
#include "lse_geometry.cuh"

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
  int nbands;             // VECTOR: bands of the image (band-major planes)
  const float* bands32;   // VECTOR: fp32 band planes (data_pitch rows)
  const double* bands64;  // VECTOR: exact band planes (nullptr -> bands32 exact)
  long long band_stride;  // elements per band plane
  const double* lut64;    // R <= 4: wt() of every all-valid 2R+1-row pattern (host_t64)
};

// Guard certification (validation builds, -DLSE_CHECK_BOUND): every fp32
// decision value of the fused kernels is compared with the reference's fp64
// value; each thread accumulates into its own slot (no contention).
struct CheckSlot {
  float ru, rp;              // max |u32 - u64| / eps_u, max |phi32 - phi64| / eps_phi
  float umin, pmin;          // min |u64|, min |phi64| (the closest decision to a tie)
  unsigned bad_u, bad_p;     // fp32 decisions outside the guard band that differ from fp64
  unsigned long long n;      // decision values checked
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
  float2 w2[8];              // (w, w) pairs: uniform operands of the packed FFMA2 pass
  float dt32;
  float scale32;
  long long iter;            // iteration produced by this launch
  int skip_uniform;          // skip warp blocks whose whole stencil window is uniform
  int nchunk;                // partition chunks (kChunk columns) per word-row
  int nchunk_u;              // update chunks (kUpdChunk columns) per word-row
  int nseg;                  // partition segments per interior word-row
  int seg_chunks;            // chunks per partition segment (partial granularity)
  Geo gu, gp;                // work geometry: update / partition
  unsigned long long* work;  // dynamic work counter (monotonic across launches)
  unsigned long long work_base;  // value of *work when this launch started
  int own_lo, own_hi;        // word-rows whose pixels count in the partials (row strips)
  unsigned long long* trace; // LSE_UNIT_TRACE builds: (start, end) ns of every unit
  uint32_t* chg;             // multi-band runs: changed-partition bits of this pass
  // batched tiles (lse_batch): ntiles equal tiles stacked in the arrays above,
  // tile t at word-row t * tile_hr; scal / ctx are per-tile arrays and gu / gp
  // the geometry of one tile (single runs: ntiles = 1, tile 0 is the image)
  int ntiles, tile_hr, tile_h;
  long long tile_words, tile_data;
  CheckSlot* chk;            // validation builds: per-thread certification slots (or null)
  long long chk_cap;
  // speculative fused iteration: pixels whose decision waits for the true
  // coefficients, (x, row) pairs; entries counted in scal->fix_n[fix_par]
  int2* fix;
  unsigned int fix_cap;
  int fix_par;
  unsigned int* fix_cnt;     // the fix-list counters (by parity): scal->fix_n of the run / tile 0
  int fix_row0;              // row offset of this view in the list's frame (batched tile views)
  int redo_only;             // batched redo pass: only the tiles whose scal->redo is set
};

// exact-path frame of tile t (its context, state and first image row)
__device__ __forceinline__ const ExactCtx* tile_ctx(const FastParams& P, int t) {
  return P.ctx + t;
}
__device__ __forceinline__ const uint32_t* tile_bits(const FastParams& P, int t) {
  return P.bits_in + (size_t)t * P.tile_words;
}
__device__ __forceinline__ int tile_y0(const FastParams& P, int t) { return t * P.tile_hr * 32; }

// Unit tracing (profiling builds only, -DLSE_UNIT_TRACE): each warp stamps the
// global timer when it grabs a unit; the interval up to its next grab is the
// unit's service time.
#ifdef LSE_UNIT_TRACE
__device__ __forceinline__ unsigned long long lse_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define LSE_TRACE_ENTRY const unsigned long long tr_entry = lse_now();
#define LSE_TRACE_DECL unsigned long long tr_t0 = 0; int tr_prev = -1; bool tr_first = true;
#define LSE_TRACE_MARK(unit)                                                        \
  do {                                                                              \
    const unsigned long long tr_now = lse_now();                                    \
    if (P.trace && lane == 0 && tr_prev >= 0) {                                     \
      P.trace[2 * tr_prev] = tr_t0;                                                 \
      P.trace[2 * tr_prev + 1] = tr_now;                                            \
    }                                                                               \
    if (P.trace && tr_first && threadIdx.x == 0) {                                  \
      P.trace[2 * nunits + 2 * blockIdx.x] = tr_entry;                              \
      P.trace[2 * nunits + 2 * blockIdx.x + 1] = tr_now;                            \
    }                                                                               \
    if (P.trace && lane == 0 && (unit) < 0)                                         \
      P.trace[2 * nunits + 2 * 4096 + blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32] = tr_now; \
    tr_first = false;                                                               \
    tr_t0 = tr_now;                                                                 \
    tr_prev = (unit);                                                               \
  } while (0)
#else
#define LSE_TRACE_ENTRY
#define LSE_TRACE_DECL
#define LSE_TRACE_MARK(unit) do { } while (0)
#endif

constexpr int kChunk = 256;      // partition: columns per warp chunk (32 lanes x 8 columns)
constexpr int kPartitionCtasPerSm = 4;   // partition occupancy (launch bound and grid)
#ifndef LSE_UPDATE_CTAS
#define LSE_UPDATE_CTAS 4
#endif
constexpr int kUpdateCtasPerSm = LSE_UPDATE_CTAS;   // update occupancy (launch bound and grid)
#ifndef LSE_FUSED_CTAS
#define LSE_FUSED_CTAS 3
#endif
// fused pass: 3 CTAs (12 warps) per SM at 168 registers measured faster than
// 4 at 128 (C5 766 -> 775 Gpix-it/s: the spills of the tighter budget cost
// more than the extra warps hide)
constexpr int kFusedCtasPerSm = LSE_FUSED_CTAS;
constexpr int kUpdCols = 8;      // update: columns per lane
constexpr int kUpdChunk = 32 * kUpdCols;   // update: columns per warp chunk


__device__ __forceinline__ double data_exact(const ExactCtx* c, int i, int x) {
  size_t o = (size_t)i * c->data_pitch + x;
  return c->data64 ? c->data64[o] : (double)c->data32[o];
}

// Exact velocity of the two-mean models at intensity I and |grad phi| = h:
// region (models.py:109-119) or mean separation (models.py:152-162).
__device__ __forceinline__ double exact_v_twomean(const Scalars* sc, double I, double h) {
  if (sc->zero_vel) return 0.0;
  if (sc->model == ZHANG) return dmul(dmul(sc->nu, ddiv(dsub(I, sc->mid), sc->peak)), h);
  const double D = dmul(sc->dc, dsub(dsub(dmul(2.0, I), sc->c_pos), sc->c_neg));
  return dmul(ddiv(D, sc->peak), h);
}

// Band value k at (i, x) exactly.
__device__ __forceinline__ double band_exact(const ExactCtx* c, int k, int i, int x) {
  const size_t o = (size_t)k * c->band_stride + (size_t)i * c->data_pitch + x;
  return c->bands64 ? c->bands64[o] : (double)c->bands32[o];
}

// Multi-band data term D = sum_k (c+_k - c-_k)(2 I_k - c+_k - c-_k), bands
// accumulated left to right (oracle/lse_oracle.py region_velocity_bands; K = 1
// is region_velocity's D exactly).
__device__ __forceinline__ double vector_D(const ExactCtx* c, const Scalars* sc, int i, int x) {
  double D = 0.0;
  for (int k = 0; k < c->nbands; ++k) {
    const double I = band_exact(c, k, i, x);
    const double cp = sc->bcp[k], cm = sc->bcm[k];
    const double t = dmul(dsub(cp, cm), dsub(dsub(dmul(2.0, I), cp), cm));
    D = k == 0 ? t : dadd(D, t);
  }
  return D;
}

// exact velocity factor of any two-mean model at (i, x), h = |grad phi|
__device__ __forceinline__ double exact_v_at(const ExactCtx* c, int i, int x, double h) {
  const Scalars* sc = c->scal;
  if (sc->zero_vel) return 0.0;
  if (c->model == VECTOR) return dmul(ddiv(vector_D(c, sc, i, x), sc->peak), h);
  return exact_v_twomean(sc, data_exact(c, i, x), h);
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
  if (c->model != EDGE) {
    v = exact_v_at(c, i, x, h);
  } else {
    v = dmul(data_exact(c, i, x), h);
  }
  atomicAdd(&c->scal->fallbacks, 1ull);
  return dadd(pc, dmul(c->dt, v));
}

// ------------------------------------------------ fast exact evaluators
// Same arithmetic as exact_u / exact_phi, but the bit window around the
// pixel is gathered up front (two independent word loads per column), so a
// near-tie costs one round of L2 latency instead of hundreds of dependent
// loads.  val/valid hold, per window column, the signs and the in-image mask
// of window rows r0 .. r0+NR-1.
// (CG: the state is rewritten inside the running kernel -- the resident
// kernels of lse_resident.cuh -- so its words are read at L2, never through
// the non-coherent path)
template <bool CG>
__device__ __forceinline__ uint32_t state_word(const uint32_t* p) {
  return CG ? __ldcg(p) : __ldg(p);
}
template <int NR, int NC, bool CG = false>
__device__ __forceinline__ void gather_window(const ExactCtx* c, const uint32_t* bits, int r0,
                                              int xc0, uint32_t (&val)[NC], uint32_t (&valid)[NC]) {
  const int H = c->H, W = c->W, HR = (H + 31) >> 5;
  const int wr = r0 >> 5;                      // arithmetic shift: r0 may be negative
  const int sh = r0 & 31;
  uint32_t rows_ok = 0u;
#pragma unroll
  for (int k = 0; k < NR; ++k) rows_ok |= (r0 + k >= 0 && r0 + k < H) ? (1u << k) : 0u;
#pragma unroll
  for (int cc = 0; cc < NC; ++cc) {
    const int xc = xc0 + cc;
    uint32_t lo = 0u, hi = 0u;
    if (xc >= 0 && xc < W) {
      if (wr >= 0 && wr < HR) lo = state_word<CG>(&bits[(size_t)wr * c->pitch_w + xc]);
      if (wr + 1 >= 0 && wr + 1 < HR) hi = state_word<CG>(&bits[(size_t)(wr + 1) * c->pitch_w + xc]);
      valid[cc] = rows_ok;
    } else {
      valid[cc] = 0u;
    }
    val[cc] = __funnelshift_r(lo, hi, sh);
  }
}

// exact vertical scipy pass at window row rr (centre), column cc
template <int R, int NC>
__device__ __forceinline__ double wt(const ExactCtx* c, const uint32_t (&val)[NC],
                                     const uint32_t (&valid)[NC], int rr, int cc) {
  // (interior pixels take the branch-free table path of exact_u_fast /
  // exact_phi_fast; here each table lookup sits behind a data-dependent
  // branch.  Always computing the explicit sum instead measured far worse:
  // the unrolled sums' registers spill the fused kernel's hot loop.)
  constexpr uint32_t PM = (1u << (2 * R + 1)) - 1u;
  if (R <= 4 && c->lut64 && ((valid[cc] >> (rr - R)) & PM) == PM)
    return __ldg(&c->lut64[(val[cc] >> (rr - R)) & PM]);   // the same value, tabulated
  auto b = [&](int k) -> double {
    if (!((valid[cc] >> k) & 1u)) return 0.0;
    return ((val[cc] >> k) & 1u) ? 1.0 : -1.0;
  };
  double acc = dmul(b(rr), c->w64[0]);
#pragma unroll
  for (int d = R; d >= 1; --d) acc = dadd(acc, dmul(dadd(b(rr - d), b(rr + d)), c->w64[d]));
  return acc;
}

// exact horizontal pass at window row rr, window column cc (t zero outside)
template <int R, int NC>
__device__ __forceinline__ double wphi(const ExactCtx* c, const uint32_t (&val)[NC],
                                       const uint32_t (&valid)[NC], int rr, int cc) {
  double acc = dmul(wt<R, NC>(c, val, valid, rr, cc), c->w64[0]);
#pragma unroll
  for (int d = R; d >= 1; --d)
    acc = dadd(acc, dmul(dadd(wt<R, NC>(c, val, valid, rr, cc - d),
                              wt<R, NC>(c, val, valid, rr, cc + d)), c->w64[d]));
  return acc;
}

#ifndef LSE_EXACT_INTERIOR
#define LSE_EXACT_INTERIOR 1
#endif
// Interior pixels (the whole window inside the image, R <= 4): every vertical
// value is a table entry, so all of them are loaded at once -- no per-value
// branch to serialise the loads (the general path above takes ~45 dependent
// L2 round trips, ~10 us per evaluation) -- then combined in scipy's order.
template <int R, int NC, bool CG = false>
__device__ __forceinline__ void interior_window(const ExactCtx* c, const uint32_t* bits, int r0,
                                                int xc0, uint32_t (&val)[NC]) {
  const int HR = (c->H + 31) >> 5;
  const int wr = r0 >> 5, sh = r0 & 31;
  const uint32_t* p = bits + (size_t)wr * c->pitch_w + xc0;
  const bool two = wr + 1 < HR;
#pragma unroll
  for (int cc = 0; cc < NC; ++cc) {
    const uint32_t lo = state_word<CG>(p + cc);
    const uint32_t hi = two ? state_word<CG>(p + c->pitch_w + cc) : 0u;
    val[cc] = __funnelshift_r(lo, hi, sh);
  }
}
template <int R, int NC>
__device__ __forceinline__ void lut_row(const double* lut, const uint32_t (&val)[NC], int rr,
                                        double (&t)[NC]) {
  constexpr uint32_t PM = (1u << (2 * R + 1)) - 1u;
#pragma unroll
  for (int cc = 0; cc < NC; ++cc) t[cc] = __ldg(&lut[(val[cc] >> (rr - R)) & PM]);
}
// wphi's sum over one row of vertical values (same order)
template <int R, int NC>
__device__ __forceinline__ double wphi_row(const double (&t)[NC], int cc, const double (&w)[R + 1]) {
  double acc = dmul(t[cc], w[0]);
#pragma unroll
  for (int d = R; d >= 1; --d) acc = dadd(acc, dmul(dadd(t[cc - d], t[cc + d]), w[d]));
  return acc;
}

// phi^{n+1} at (i, x) exactly (partition near-ties)
template <int R, bool CG = false>
__device__ __noinline__ double exact_phi_fast(const ExactCtx* c, const uint32_t* bits, int i, int x,
                                              bool count = true) {
  constexpr int NR = 2 * R + 1, NC = 2 * R + 1;
  if (LSE_EXACT_INTERIOR && R <= 4 && c->lut64 && i >= R && i <= c->H - 1 - R && x >= R &&
      x <= c->W - 1 - R) {
    double w[R + 1];
#pragma unroll
    for (int d = 0; d <= R; ++d) w[d] = c->w64[d];
    uint32_t v[NC];
    interior_window<R, NC, CG>(c, bits, i - R, x - R, v);
    double t[NC];
    lut_row<R, NC>(c->lut64, v, R, t);
    if (count) atomicAdd(&c->scal->fallbacks, 1ull);
    return wphi_row<R, NC>(t, R, w);
  }
  uint32_t val[NC], valid[NC];
  gather_window<NR, NC, CG>(c, bits, i - R, x - R, val, valid);
  if (count) atomicAdd(&c->scal->fallbacks, 1ull);
  return wphi<R, NC>(c, val, valid, R, R);
}

// u at (i, x) exactly (update near-ties): phi at the pixel and its four
// neighbours (np.gradient one-sided at the image border), glibc hypot,
// the model's velocity, u = phi + dt * v.
template <int R, int SRC, bool CG = false>
__device__ __noinline__ double exact_u_fast(const ExactCtx* c, const uint32_t* bits, int i, int x,
                                            bool count = true) {
  constexpr int NR = 2 * R + 3, NC = 2 * R + 3;
  const int H = c->H, W = c->W;
  // the pixel's data value is loaded with the window (one round of latency
  // for both; the multi-band term reads its bands later)
  const double Iv = c->model != VECTOR ? data_exact(c, i, x) : 0.0;
  if (LSE_EXACT_INTERIOR && SRC != SRC_SCALED && R <= 4 && c->lut64 && i >= R + 1 &&
      i <= H - 2 - R && x >= R + 1 && x <= W - 2 - R) {
    // interior: rows i-1, i, i+1 of the window (rr = R .. R+2), central differences
    double w[R + 1];
#pragma unroll
    for (int d = 0; d <= R; ++d) w[d] = c->w64[d];
    uint32_t v[NC];
    interior_window<R, NC, CG>(c, bits, i - 1 - R, x - 1 - R, v);
    double tu[NC], tc[NC], td[NC];
    lut_row<R, NC>(c->lut64, v, R, tu);
    lut_row<R, NC>(c->lut64, v, R + 1, tc);
    lut_row<R, NC>(c->lut64, v, R + 2, td);
    const double pc = wphi_row<R, NC>(tc, R + 1, w);
    const double fx = dmul(dsub(wphi_row<R, NC>(tc, R + 2, w), wphi_row<R, NC>(tc, R, w)), 0.5);
    const double fy = dmul(dsub(wphi_row<R, NC>(td, R + 1, w), wphi_row<R, NC>(tu, R + 1, w)), 0.5);
    const double h = np_hypot(fx, fy);
    double v2;
    if (c->model == EDGE) v2 = dmul(Iv, h);
    else if (c->model == VECTOR) v2 = exact_v_at(c, i, x, h);
    else v2 = exact_v_twomean(c->scal, Iv, h);
    if (count) atomicAdd(&c->scal->fallbacks, 1ull);
    return dadd(pc, dmul(c->dt, v2));
  }
  uint32_t val[NC], valid[NC];
  gather_window<NR, NC, CG>(c, bits, i - 1 - R, x - 1 - R, val, valid);
  auto ph = [&](int di, int dx) -> double {      // phi at (i + di, x + dx)
    if (SRC == SRC_SCALED) {
      const int cc = R + 1 + dx, rr = R + 1 + di;
      return ((val[cc] >> rr) & 1u) ? c->scale : -c->scale;
    }
    return wphi<R, NC>(c, val, valid, R + 1 + di, R + 1 + dx);
  };
  const double pc = ph(0, 0);
  double fx, fy;
  if (x == 0) fx = dsub(ph(0, 1), pc);
  else if (x == W - 1) fx = dsub(pc, ph(0, -1));
  else fx = dmul(dsub(ph(0, 1), ph(0, -1)), 0.5);
  if (i == 0) fy = dsub(ph(1, 0), pc);
  else if (i == H - 1) fy = dsub(pc, ph(-1, 0));
  else fy = dmul(dsub(ph(1, 0), ph(-1, 0)), 0.5);
  const double h = np_hypot(fx, fy);
  double v;
  const Scalars* sc = c->scal;
  if (c->model == EDGE) v = dmul(Iv, h);
  else if (c->model == VECTOR) v = exact_v_at(c, i, x, h);
  else v = exact_v_twomean(sc, Iv, h);           // exact_v_at's two-mean branch
  if (count) atomicAdd(&c->scal->fallbacks, 1ull);
  return dadd(pc, dmul(c->dt, v));
}

#ifdef LSE_CHECK_BOUND
__device__ __forceinline__ CheckSlot* check_slot(const FastParams& P) {
  if (!P.chk) return nullptr;
  const long long s =
      ((long long)blockIdx.y * gridDim.x + blockIdx.x) * blockDim.x + threadIdx.x;
  return s < P.chk_cap ? P.chk + s : nullptr;
}
// u32: the fused kernel's fp32 u at (i, x) (frame of ctx / bits); the kernel's
// decision off the guard band is u32 > 0
template <int R, int SRC>
__device__ __noinline__ void check_u(const FastParams& P, const ExactCtx* c, const uint32_t* bits,
                                     int i, int x, float u32, float eps) {
  CheckSlot* k = check_slot(P);
  if (!k) return;
  const double u64 = exact_u_fast<R, SRC>(c, bits, i, x, false);
  k->ru = fmaxf(k->ru, (float)(fabs((double)u32 - u64) / (double)eps));
  k->umin = fminf(k->umin, (float)fabs(u64));
  if (fabsf(u32) > eps && ((u32 > 0.f) != (u64 > 0.0))) k->bad_u += 1u;
  k->n += 1ull;
}
// phi32: the partition's fp32 phi^{n+1}; decisions phi >= 0 and phi > 0
template <int R>
__device__ __noinline__ void check_phi(const FastParams& P, const ExactCtx* c, const uint32_t* bits,
                                       int i, int x, float p32, float eps) {
  CheckSlot* k = check_slot(P);
  if (!k) return;
  const double p64 = exact_phi_fast<R>(c, bits, i, x, false);
  k->rp = fmaxf(k->rp, (float)(fabs((double)p32 - p64) / (double)eps));
  k->pmin = fminf(k->pmin, (float)fabs(p64));
  if (fabsf(p32) > eps && ((p32 > 0.f) != (p64 > 0.0))) k->bad_p += 1u;
  k->n += 1ull;
}
#define LSE_CHECK_U(R_, SRC_, P_, C_, B_, I_, X_, U_, E_) check_u<R_, SRC_>(P_, C_, B_, I_, X_, U_, E_)
#define LSE_CHECK_PHI(R_, P_, C_, B_, I_, X_, V_, E_) check_phi<R_>(P_, C_, B_, I_, X_, V_, E_)
#else
#define LSE_CHECK_U(...) do { } while (0)
#define LSE_CHECK_PHI(...) do { } while (0)
#endif

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
  // each t (vertical pass of one column) is folded into the <= 2R+1 outputs
  // it touches as soon as it is looked up: no t[] array stays live
#pragma unroll
  for (int j = 0; j < NT; ++j) {
    const uint32_t p = (win[j] >> m0) & PM;
    float t;
    if (INT) t = s_lt[p];
    else t = fmaf(2.f, s_ls[p & vr & cm[j]], cm[j] ? -Lv : 0.f);
#pragma unroll
    for (int c = 0; c < NOUT; ++c) {
      const int d = j - c - R;                     // t column offset from output c
      if (d < -R || d > R) continue;
      const float wd = P.w32[d < 0 ? -d : d];
      if (d == -R) out[c] = wd * t;                // first contribution to out[c]
      else out[c] = fmaf(wd, t, out[c]);
    }
  }
}

template <bool INT, int CPL>
__device__ __forceinline__ void load_data_row(const FastParams& P, int i, int x0, float (&d)[CPL]) {
  if (i >= P.g.H) return;
  const float* rowp = P.data32 + (size_t)i * P.g.data_pitch + x0;
  if (INT) {
#pragma unroll
    for (int q = 0; q < CPL / 4; ++q) {
      const float4 a = __ldcs(reinterpret_cast<const float4*>(rowp) + q);
      d[4 * q + 0] = a.x; d[4 * q + 1] = a.y; d[4 * q + 2] = a.z; d[4 * q + 3] = a.w;
    }
  } else {
#pragma unroll
    for (int c = 0; c < CPL; ++c) d[c] = (x0 + c < P.g.W) ? __ldcs(rowp + c) : 0.f;
  }
}

// fused pass: decide the guard band of the coefficients used exactly in the
// pass (so an iteration whose coefficients did not move needs no fix list)
#ifndef LSE_SPEC_INLINE
#define LSE_SPEC_INLINE 1
#endif
// codegen knobs of the fused loop (A/B builds)
#ifndef LSE_LUT_EXPLICIT
#define LSE_LUT_EXPLICIT 0
#endif
#ifndef LSE_TIE_PARAM
#define LSE_TIE_PARAM 1
#endif
#if LSE_TIE_PARAM
#define LSE_TIE_P P
#else
#define LSE_TIE_P Pn
#endif
#ifndef LSE_PAIR_MIN
#define LSE_PAIR_MIN 1
#endif
#ifndef LSE_STEP_UNROLL
#define LSE_STEP_UNROLL 2
#endif
constexpr int kStepUnroll = LSE_STEP_UNROLL;

// three-input minimum (FMNMX3, sm_100+)
__device__ __forceinline__ float fmin3(float a, float b, float c) {
  float r;
  asm("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

__device__ __forceinline__ float sqrt_approx(float x) {
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// state words of column xc in word-row wr (0 outside the image)
template <bool INT>
__device__ __forceinline__ uint32_t word_at(const FastParams& P, int wr, int xc) {
  if (!INT && (wr < 0 || wr >= P.g.HR || xc < 0 || xc >= P.g.W)) return 0u;
  return __ldg(&P.bits_in[(size_t)wr * P.g.pitch_w + xc]);
}

// ---------------------------------------------------------------- update
// ------------------------------------------------- interior update block
// Specialised copy of update_block for interior units (the >98% case):
//  * LUT addressing is one SHF + one LOP3 per t: the windows are kept
//    pre-shifted by 2 (byte offsets) and the 2 KB LUT is 2 KB-aligned in
//    shared memory, so ((win >> m0) & mask) | base is the LDS address;
//  * the data plane (I or g) streams through a 4-row cp.async ring in shared
//    memory, issued 3 rows ahead, so no register copies wait on HBM.
constexpr int kRing = 4;                        // rows in flight per warp (power of 2)

__device__ __forceinline__ float lds_f32(uint32_t addr) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ float2 lds_f32x2(uint32_t addr) {
  float2 v;
  asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(addr));
  return v;
}
__device__ __forceinline__ void cp_async16(uint32_t saddr, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(saddr), "l"(g));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N)); }

// ---- TMA (bulk async copy + mbarrier) variant of the data ring, A/B builds
// only (-DLSE_TMA_RING=1, `make tma`): one elected lane copies a whole 1 KB
// row of a chunk unit per instruction and the warp waits on an mbarrier,
// instead of two 16-byte cp.async per lane and row.  Measured slower (C5 673
// vs 772 Gpix-it/s, same box: a convergence point, the elected-lane branch
// and an mbarrier wait per 2-row step cost more than the 4 LDGSTS they
// replace in this issue-bound loop), so the default build keeps the per-lane
// ring, which also serves the lane-scattered B1 units.
#ifndef LSE_TMA_RING
#define LSE_TMA_RING 0
#endif
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile("{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
               "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
               "@!p bra WAIT_%=;\n\t}" ::"r"(bar), "r"(parity) : "memory");
}

template <int R, int NT, int NOUT, int SRC = SRC_SMOOTH>
__device__ __forceinline__ void phi_row_int(const FastParams& P, const uint32_t (&win4)[NT],
                                            int m0, uint32_t lut_base, float (&out)[NOUT]) {
  constexpr uint32_t PM4 = ((1u << (2 * R + 1)) - 1u) << 2;
  if (SRC == SRC_SCALED) {                       // phi = +-s (binary initial state)
#pragma unroll
    for (int c = 0; c < NOUT; ++c)
      out[c] = ((win4[c + R] >> (m0 + R + 2)) & 1u) ? P.scale32 : -P.scale32;
    return;
  }
#pragma unroll
  for (int j = 0; j < NT; ++j) {
    const float t = lds_f32(((win4[j] >> m0) & PM4) | lut_base);
#pragma unroll
    for (int c = 0; c < NOUT; ++c) {
      const int d = j - c - R;
      if (d < -R || d > R) continue;
      const float wd = P.w32[d < 0 ? -d : d];
      if (d == -R) out[c] = wd * t;
      else out[c] = fmaf(wd, t, out[c]);
    }
  }
}

// ---- packed fp32x2 arithmetic (FFMA2 / FMUL2 / FADD2 on sm_100a)
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{.reg .b64 ra, rb, rc, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
      "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) {
  float2 d;
  asm("{.reg .b64 ra, rb, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "mul.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;}"
      : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
__device__ __forceinline__ float2 fsub2(float2 a, float2 b) {
  float2 d;
  asm("{.reg .b64 ra, rb, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "sub.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;}"
      : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}

// Two phi rows at once (window offsets m0 and m0+1) as (row, row+1) pairs, so
// the horizontal pass runs on the packed FFMA2 pipe: out[c] = sum_d w_d t(c+d).
// The vertical values of both rows come from one lookup in the pair table:
// entry i of the 2R+2-bit window is (t(i & low 2R+1 bits), t(i >> 1)) -- the
// same fp32 values as two t-LUT lookups.  win8 holds the window words
// pre-shifted by 3 (byte offsets of 8-byte entries).  The table is a
// file-scope __shared__ array: the partition addresses it as [offset + UR]
// (no add); in the update ptxas keeps the base in a per-thread register and
// spends one IADD per lookup.  (An OR-with-aligned-base variant removed that
// add but measured no faster, and static __shared__ alignment is relative to
// the user window, so it was dropped.)
__shared__ __align__(16) float2 g_pair_lut[1 << (2 * 4 + 2)];      // R <= 4

template <int R, int NT, int NOUT, int SRC = SRC_SMOOTH>
__device__ __forceinline__ void phi_rows2_int(const FastParams& P, const uint32_t (&win8)[NT],
                                              int m0, uint32_t lut2_base, float2 (&out)[NOUT]) {
  constexpr uint32_t PM8 = ((1u << (2 * R + 2)) - 1u) << 3;
  if (SRC == SRC_SCALED) {
#pragma unroll
    for (int c = 0; c < NOUT; ++c) {
      const uint32_t w = win8[c + R] >> (m0 + R + 3);
      out[c] = make_float2((w & 1u) ? P.scale32 : -P.scale32,
                           (w & 2u) ? P.scale32 : -P.scale32);
    }
    return;
  }
#pragma unroll
  for (int j = 0; j < NT; ++j) {
#if LSE_LUT_EXPLICIT
    uint32_t tb;
    asm("mov.u32 %0, _ZN3lse10g_pair_lutE;" : "=r"(tb));   // the table's shared address
    const float2 t = lds_f32x2(tb + ((win8[j] >> m0) & PM8));
#else
    const float2 t = *reinterpret_cast<const float2*>(
        reinterpret_cast<const char*>(g_pair_lut) + ((win8[j] >> m0) & PM8));
#endif
#pragma unroll
    for (int c = 0; c < NOUT; ++c) {
      const int d = j - c - R;
      if (d < -R || d > R) continue;
      const float2 wd = P.w2[d < 0 ? -d : d];
      if (d == -R) out[c] = fmul2(wd, t);
      else out[c] = ffma2(wd, t, out[c]);
    }
  }
}

// Near-tie columns of one interior row.  The fused loops flag whole rows
// (one running min per row keeps the loop short); these recompute the row's
// fp32 values with exactly the loop's operations -- phi_rows2_int's packed
// lanes are independent FMAs, so a row's values do not depend on which row
// it was paired with -- and return the columns that need the fp64 decision.
template <int R, int MODEL, int CPL, int SRC, bool SPEC = false>
__device__ __noinline__ uint32_t update_tie_cols(const FastParams& P, uint32_t lut_base, int r,
                                                 int x0, int k, float A, float B, float eps_u,
                                                 float delta = 0.f, float eps_t = 0.f) {
  constexpr int NT = CPL + 2 * (R + 1);
  constexpr int NP = CPL + 2;
  const int y0 = r * 32;
  const int base = y0 + k - 1 - R;               // phi rows k-1 .. k+2 at m0 = 0 .. 3
  const uint32_t* wp = P.bits_in + (size_t)(base >> 5) * P.g.pitch_w + (x0 - (R + 1));
  uint32_t win4[NT];
#pragma unroll
  for (int j = 0; j < NT; ++j)
    win4[j] = __funnelshift_r(__ldg(wp + j), __ldg(wp + P.g.pitch_w + j), base & 31) << 3;
  float2 pa[NP], pb[NP];
  phi_rows2_int<R, NT, NP, SRC>(P, win4, 0, lut_base, pa);     // rows k-1, k
  phi_rows2_int<R, NT, NP, SRC>(P, win4, 2, lut_base, pb);     // rows k+1, k+2
  const float* drow = P.data32 + (size_t)(y0 + k) * P.g.data_pitch + x0;
  uint32_t cols = 0u;
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    const float dy = __fsub_rn(pb[c + 1].x, pa[c + 1].x);
    const float dx = __fsub_rn(pa[c + 2].y, pa[c].y);
    const float h = sqrt_approx(__fmaf_rn(dx, dx, __fmul_rn(dy, dy)));
    const float d = __ldg(drow + c);
    const float vf = (MODEL == REGION) ? __fmaf_rn(A, d, B) : d;
    const float u = __fmaf_rn(vf, h, pa[c + 1].y);
    // SPEC: the speculative band |u| - delta h <= e0 (eps_u holds e0), the
    // fused loop's test on the same values; bits 16.. mark the band's columns
    // within the guard eps_t of the coefficients used (decided exactly there)
    if ((SPEC ? __fmaf_rn(-delta, h, fabsf(u)) : fabsf(u)) <= eps_u) cols |= 1u << c;
    if (SPEC && fabsf(u) <= eps_t) cols |= 1u << (16 + c);
  }
  // (all columns if nothing matched; SPEC callers flag row pairs, so a row
  // may legitimately have no match there)
  return (cols || SPEC) ? cols : (1u << CPL) - 1u;
}

// a pixel whose speculative decision waits for the true coefficients
// (rows in the list's frame: the stacked rows of a batch)
__device__ __forceinline__ void spec_append(const FastParams& P, int i, int x) {
  const unsigned q = atomicAdd(&P.fix_cnt[P.fix_par], 1u);
  if (q < P.fix_cap) P.fix[q] = make_int2(x, i + P.fix_row0);
}

template <int R, bool EXACT = false>
__device__ __noinline__ uint32_t partition_tie_cols(const FastParams& P, uint32_t lut_base, int r,
                                                    int x0, int k, float eps_phi) {
  constexpr int NT = kColsPerThread + 2 * R;
  const int base = r * 32 + k - R;               // phi row k at m0 = 0
  const uint32_t* wp = P.bits_in + (size_t)(base >> 5) * P.g.pitch_w + (x0 - R);
  uint32_t win4[NT];
#pragma unroll
  for (int j = 0; j < NT; ++j)
    win4[j] = __funnelshift_r(__ldg(wp + j), __ldg(wp + P.g.pitch_w + j), base & 31) << 3;
  float2 ph[8];
  phi_rows2_int<R, NT, 8>(P, win4, 0, lut_base, ph);
  uint32_t cols = 0u;
#pragma unroll
  for (int c = 0; c < 8; ++c)
    if (fabsf(ph[c].x) <= eps_phi) cols |= 1u << c;
  return (cols || EXACT) ? cols : 0xffu;        // EXACT: row pairs flagged (fused pass)
}

constexpr int kRing2 = 8;                       // data rows buffered per warp (2-row steps)

// Interior update block, two rows per step (see update_block_int for the
// design); phi rows are kept as (row, row+1) pairs.
//
// FUSED (the speculative fused iteration, single runs): the same pass also
// yields the partition of its input state -- the centre values pp.y / pn.x
// are phi^n itself -- as pw (phi >= 0) / mw (phi > 0) words, near ties
// resolved exactly; the update's coefficients are a prediction, so instead of
// the eps_u guard every pixel with |u| - delta h <= eps_u (eps_u then holds
// the band's e0) goes to the fix list (spec_append), decided by k_spec_fix.
template <int R, int MODEL, int CPL, int SRC, bool FUSED = false>
__device__ __forceinline__ void update_block_int2(const FastParams& P, uint32_t lut_base,
                                                  float* ring, int r, int x0, float A, float B,
                                                  float eps_u,
                                                  const uint32_t (&prev)[CPL + 2 * (R + 1)],
                                                  const uint32_t (&cur)[CPL + 2 * (R + 1)],
                                                  int tile, float delta, uint32_t (&pw)[CPL],
                                                  uint32_t (&mw)[CPL], const FastParams& Pn,
                                                  const uint32_t* wslot = nullptr,
                                                  float eps_t = 0.f, uint32_t tma_bars = 0u) {
  // Pn: the launch parameters as seen by the noinline tie helpers (the CTA's
  // shared copy: passing the kernel parameter block by reference to a noinline
  // function makes every thread copy it to local memory first)
  constexpr int NT = CPL + 2 * (R + 1);
  constexpr int NP = CPL + 2;
  constexpr uint32_t kSlot = 32 * CPL * 4;
  const int y0 = r * 32;
  const int lane = threadIdx.x & 31;
  uint32_t win4[NT];
#pragma unroll
  for (int j = 0; j < NT; ++j) win4[j] = __funnelshift_r(prev[j], cur[j], 31 - R) << 3;
  const uint32_t ring_s = (uint32_t)__cvta_generic_to_shared(ring) + lane * CPL * 4;
  const size_t dpitch = P.g.data_pitch;
  const float* gsrc = P.data32 + (size_t)y0 * dpitch + x0;
  // (A/B builds) chunk units: whole rows by bulk copies of one lane, signalled
  // on the warp's four mbarriers (one per slot pair; 16 steps = 4 phases each,
  // so every unit starts at parity 0)
  const bool tma = LSE_TMA_RING && FUSED && tma_bars != 0u;
  const uint32_t ring_w = ring_s - lane * CPL * 4;             // the warp's ring, lane 0's view
  const float* grow = gsrc - lane * CPL;                        // the chunk's first column
  if (tma) {
    if (lane == 0) {
#pragma unroll
      for (int q = 0; q < kRing2 - 2; q += 2) {
        const uint32_t bar = tma_bars + 8 * (q >> 1);
        mbar_expect_tx(bar, 2 * kSlot);
        bulk_g2s(ring_w + q * kSlot, grow + (size_t)q * dpitch, kSlot, bar);
        bulk_g2s(ring_w + (q + 1) * kSlot, grow + (size_t)(q + 1) * dpitch, kSlot, bar);
      }
    }
    gsrc += (kRing2 - 2) * dpitch;
  } else {
#pragma unroll
  for (int q = 0; q < kRing2 - 2; q += 2) {    // rows 0 .. 5 in flight, 2 per group
#pragma unroll
    for (int v = 0; v < CPL / 4; ++v) {
      cp_async16(ring_s + q * kSlot + v * 16, gsrc + 4 * v);
      cp_async16(ring_s + (q + 1) * kSlot + v * 16, gsrc + dpitch + 4 * v);
    }
    cp_async_commit();
    gsrc += 2 * dpitch;
  }
  }
  float2 pp[NP], pn[NP];
  uint32_t ow[CPL];
  uint32_t fbrows = 0u, pfrows = 0u;
#pragma unroll
  for (int c = 0; c < CPL; ++c) ow[c] = 0u;
  if (FUSED) {
#pragma unroll
    for (int c = 0; c < CPL; ++c) pw[c] = 0u;
  }
  phi_rows2_int<R, NT, NP, SRC>(P, win4, 0, lut_base, pp);     // rows -1, 0
  const uint32_t* wrow = P.bits_in + (size_t)r * P.g.pitch_w + (x0 - (R + 1));
#pragma unroll kStepUnroll
  for (int s = 0; s < 16; ++s) {
    if (tma) {
      if (2 * s + kRing2 - 2 < 32) {
        __syncwarp();                             // every lane has read the slots being refilled
        if (lane == 0) {
          const int q = (2 * s + kRing2 - 2) & (kRing2 - 1);
          const uint32_t bar = tma_bars + 8 * (q >> 1);
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          mbar_expect_tx(bar, 2 * kSlot);
          bulk_g2s(ring_w + q * kSlot, grow + (size_t)(2 * s + kRing2 - 2) * dpitch, kSlot, bar);
          bulk_g2s(ring_w + (q + 1) * kSlot, grow + (size_t)(2 * s + kRing2 - 1) * dpitch, kSlot, bar);
        }
      }
    } else {
      if (2 * s + kRing2 - 2 < 32) {
        const uint32_t d0 = ring_s + ((2 * s + kRing2 - 2) & (kRing2 - 1)) * kSlot;
#pragma unroll
        for (int v = 0; v < CPL / 4; ++v) {
          cp_async16(d0 + v * 16, gsrc + 4 * v);
          cp_async16(d0 + kSlot + v * 16, gsrc + dpitch + 4 * v);
        }
        gsrc += 2 * dpitch;
      }
      cp_async_commit();
    }
    if (s == 8) {                               // window base y0+16-R for rows >= 17
      if (FUSED) {                              // staged in shared memory at the unit start
        // (an asm load: a plain one lets the compiler re-derive the value from
        // the global words it was built from -- the loads this avoids)
        const uint32_t ws = (uint32_t)__cvta_generic_to_shared(wslot) + 4 * lane;
#pragma unroll
        for (int j = 0; j < NT; ++j) asm volatile("ld.shared.u32 %0, [%1];" : "=r"(win4[j]) : "r"(ws + 128 * j));
      } else {
#pragma unroll
        for (int j = 0; j < NT; ++j)
          win4[j] = __funnelshift_r(__ldg(wrow + j), __ldg(wrow + P.g.pitch_w + j), 16 - R) << 3;
      }
    }
    const int kn = 2 * s + 1;                   // first phi row of this step's pair
    phi_rows2_int<R, NT, NP, SRC>(P, win4, s < 8 ? kn + 1 : kn - 16, lut_base, pn);
    if (tma) mbar_wait(tma_bars + 8 * (s & 3), (s >> 2) & 1);
    else cp_async_wait<kRing2 / 2 - 1>();        // rows 2s, 2s+1 have landed
    float d0[CPL], d1[CPL];
    {
      const uint32_t src0 = ring_s + ((2 * s) & (kRing2 - 1)) * kSlot;
#pragma unroll
      for (int v = 0; v < CPL / 4; ++v) {
        float4 q0, q1;
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(q0.x), "=f"(q0.y), "=f"(q0.z), "=f"(q0.w) : "r"(src0 + v * 16));
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(q1.x), "=f"(q1.y), "=f"(q1.z), "=f"(q1.w) : "r"(src0 + kSlot + v * 16));
        d0[4 * v] = q0.x; d0[4 * v + 1] = q0.y; d0[4 * v + 2] = q0.z; d0[4 * v + 3] = q0.w;
        d1[4 * v] = q1.x; d1[4 * v + 1] = q1.y; d1[4 * v + 2] = q1.z; d1[4 * v + 3] = q1.w;
      }
    }
    float umin0 = 3.0e38f, umin1 = 3.0e38f, pmin0 = 3.0e38f;
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      // rows 2s (centre pp.y) and 2s+1 (centre pn.x); dy = phi(k+1) - phi(k-1)
      const float2 dy = fsub2(pn[c + 1], pp[c + 1]);
      const float2 dx = make_float2(pp[c + 2].y - pp[c].y, pn[c + 2].x - pn[c].x);
      const float2 s2 = ffma2(dx, dx, fmul2(dy, dy));
      const float h0 = sqrt_approx(s2.x), h1 = sqrt_approx(s2.y);      // 2|grad phi|
      const float vf0 = (MODEL == REGION) ? fmaf(A, d0[c], B) : d0[c];
      const float vf1 = (MODEL == REGION) ? fmaf(A, d1[c], B) : d1[c];
      const float u0 = fmaf(vf0, h0, pp[c + 1].y);
      const float u1 = fmaf(vf1, h1, pn[c + 1].x);
      ow[c] = __funnelshift_l(__float_as_uint(u0), ow[c], 1);
      ow[c] = __funnelshift_l(__float_as_uint(u1), ow[c], 1);
      if (FUSED) {
        pw[c] = __funnelshift_l(__float_as_uint(pp[c + 1].y), pw[c], 1);
        pw[c] = __funnelshift_l(__float_as_uint(pn[c + 1].x), pw[c], 1);
#if LSE_PAIR_MIN
        // one minimum per row pair (three-input FMNMX): the pair's rows are
        // then searched column by column (exact matches only)
        umin0 = fmin3(umin0, fmaf(-delta, h0, fabsf(u0)), fmaf(-delta, h1, fabsf(u1)));
        pmin0 = fmin3(pmin0, fabsf(pp[c + 1].y), fabsf(pn[c + 1].x));
#else
        umin0 = fminf(umin0, fmaf(-delta, h0, fabsf(u0)));
        umin1 = fminf(umin1, fmaf(-delta, h1, fabsf(u1)));
        pmin0 = fminf(pmin0, fminf(fabsf(pp[c + 1].y), fabsf(pn[c + 1].x)));
#endif
      } else {
        umin0 = fminf(umin0, fabsf(u0));
        umin1 = fminf(umin1, fabsf(u1));
        LSE_CHECK_U(R, SRC, P, tile_ctx(P, tile), tile_bits(P, tile),
                    y0 - tile_y0(P, tile) + 2 * s, x0 + c, u0, eps_u);
        LSE_CHECK_U(R, SRC, P, tile_ctx(P, tile), tile_bits(P, tile),
                    y0 - tile_y0(P, tile) + 2 * s + 1, x0 + c, u1, eps_u);
      }
    }
    if (FUSED) {
#if LSE_PAIR_MIN
      if (umin0 <= eps_u) fbrows |= 3u << (2 * s);
#else
      if (umin0 <= eps_u) fbrows |= 1u << (2 * s);
      if (umin1 <= eps_u) fbrows |= 2u << (2 * s);
#endif
      if (pmin0 <= P.scal->eps_phi) pfrows |= 3u << (2 * s);
    } else {
      if (umin0 <= eps_u) fbrows |= 1u << (2 * s);
      if (umin1 <= eps_u) fbrows |= 2u << (2 * s);
    }
#pragma unroll
    for (int c = 0; c < NP; ++c) pp[c] = pn[c];
  }
  cp_async_wait<0>();
#pragma unroll
  for (int c = 0; c < CPL; ++c) ow[c] = ~__brev(ow[c]);   // bit k = (u_k > 0) off ties
  while (fbrows) {
    const int k = __ffs(fbrows) - 1;
    fbrows &= fbrows - 1;
    const uint32_t bitk = 1u << k;
    uint32_t cols = update_tie_cols<R, MODEL, CPL, SRC, FUSED>(LSE_TIE_P, lut_base, r, x0, k, A,
                                                               B, eps_u, delta, eps_t);
    uint32_t exact_cols = cols >> 16;
    cols &= 0xffffu;
    while (cols) {
      const int c = __ffs(cols) - 1;
      cols &= cols - 1;
      if (FUSED) {
        // decided by k_spec_fix unless the coefficients turn out unchanged;
        // the guard band of the ones used is decided exactly now (final if
        // they are unchanged, as they are once the partition settles)
        // (batched edge tiles run with their exact coefficients: nothing to fix)
        if (tile_ctx(P, tile)->model != EDGE) spec_append(P, y0 + k, x0 + c);
        if (!LSE_SPEC_INLINE || !((exact_cols >> c) & 1u)) continue;
      }
      const bool pos = exact_u_fast<R, SRC>(tile_ctx(P, tile), tile_bits(P, tile),
                                            y0 - tile_y0(P, tile) + k, x0 + c) > 0.0;
#pragma unroll
      for (int q = 0; q < CPL; ++q)
        if (q == c) ow[q] = pos ? (ow[q] | bitk) : (ow[q] & ~bitk);
    }
  }
  if (FUSED) {
    // partition of the input state: bit k = phi_k >= +0 off ties, then the
    // exact signs of the tie columns (as partition_block)
#pragma unroll
    for (int c = 0; c < CPL; ++c) mw[c] = pw[c] = ~__brev(pw[c]);
    const float eps_phi = P.scal->eps_phi;
    while (pfrows) {
      const int k = __ffs(pfrows) - 1;
      pfrows &= pfrows - 1;
      const uint32_t bitk = 1u << k;
      uint32_t cols = partition_tie_cols<R, true>(LSE_TIE_P, lut_base, r, x0, k, eps_phi);
      while (cols) {
        const int c = __ffs(cols) - 1;
        cols &= cols - 1;
        const double e = exact_phi_fast<R>(tile_ctx(P, tile), tile_bits(P, tile),
                                           y0 - tile_y0(P, tile) + k, x0 + c);
#pragma unroll
        for (int q = 0; q < CPL; ++q) {
          if (q == c) {
            pw[q] = e >= 0.0 ? (pw[q] | bitk) : (pw[q] & ~bitk);
            mw[q] = e > 0.0 ? (mw[q] | bitk) : (mw[q] & ~bitk);
          }
        }
      }
    }
  }
  uint32_t* dst = P.bits_out + (size_t)r * P.g.pitch_w + x0;
#pragma unroll
  for (int q = 0; q < CPL / 4; ++q)
    reinterpret_cast<uint4*>(dst)[q] = make_uint4(ow[4 * q], ow[4 * q + 1], ow[4 * q + 2], ow[4 * q + 3]);
}

// Split-warp interior block for small images: the warp's lanes form NS row
// parts of 32/NS lanes; part p takes rows p*RP .. p*RP+RP-1 (RP = 32/NS) of
// the same 8-column groups (a warp unit covers 256/NS columns), so a unit is
// RP/2 row pairs long instead of 16.  Each part keeps its own window with base
// row h0 - 1 - R, so the window offsets -- and the whole instruction stream --
// are the same in every part; the RP-bit pieces of each state word are merged
// by log2(NS) shuffles.  Every lane of the warp calls it (act = false: no work,
// still shuffles).  wlo/whi: word-rows r-1, r (part 0) or r, r+1 (parts >= 1).
template <int R, int MODEL, int CPL, int SRC, int NS>
__device__ __forceinline__ void update_block_split(const FastParams& P, uint32_t lut_base,
                                                  float* ring, int r, int x0, float A, float B,
                                                  float eps_u,
                                                  const uint32_t (&wlo)[CPL + 2 * (R + 1)],
                                                  const uint32_t (&whi)[CPL + 2 * (R + 1)],
                                                  int tile, bool act) {
  constexpr int NT = CPL + 2 * (R + 1);
  constexpr int NP = CPL + 2;
  constexpr uint32_t kSlot = 32 * CPL * 4;
  constexpr int RP = 32 / NS;                   // rows per part
  static_assert(NS == 2 || NS == 4, "row parts");
  static_assert(RP >= R + 1, "part window must fit in two words");
  const int lane = threadIdx.x & 31;
  const int h0 = (lane / (32 / NS)) * RP;       // first row of this lane's part
  const int y0 = r * 32;
  uint32_t ow[CPL];
#pragma unroll
  for (int c = 0; c < CPL; ++c) ow[c] = 0u;
  if (act) {
    uint32_t win4[NT];
    const int sh = h0 ? h0 - 1 - R : 31 - R;    // window base row y0 + h0 - 1 - R
#pragma unroll
    for (int j = 0; j < NT; ++j) win4[j] = __funnelshift_r(wlo[j], whi[j], sh) << 3;
    const uint32_t ring_s = (uint32_t)__cvta_generic_to_shared(ring) + lane * CPL * 4;
    const size_t dpitch = P.g.data_pitch;
    const float* gsrc = P.data32 + (size_t)(y0 + h0) * dpitch + x0;
#pragma unroll
    for (int q = 0; q < kRing2 - 2; q += 2) {  // rows 0 .. 5 of the part in flight
#pragma unroll
      for (int v = 0; v < CPL / 4; ++v) {
        cp_async16(ring_s + q * kSlot + v * 16, gsrc + 4 * v);
        cp_async16(ring_s + (q + 1) * kSlot + v * 16, gsrc + dpitch + 4 * v);
      }
      cp_async_commit();
      gsrc += 2 * dpitch;
    }
    float2 pp[NP], pn[NP];
    uint32_t fbrows = 0u;
    phi_rows2_int<R, NT, NP, SRC>(P, win4, 0, lut_base, pp);   // rows h0-1, h0
#pragma unroll 2
    for (int s = 0; s < RP / 2; ++s) {
      if (2 * s + kRing2 - 2 < RP) {
        const uint32_t d0 = ring_s + ((2 * s + kRing2 - 2) & (kRing2 - 1)) * kSlot;
#pragma unroll
        for (int v = 0; v < CPL / 4; ++v) {
          cp_async16(d0 + v * 16, gsrc + 4 * v);
          cp_async16(d0 + kSlot + v * 16, gsrc + dpitch + 4 * v);
        }
        gsrc += 2 * dpitch;
      }
      cp_async_commit();
      phi_rows2_int<R, NT, NP, SRC>(P, win4, 2 * s + 2, lut_base, pn);
      cp_async_wait<kRing2 / 2 - 1>();
      float d0[CPL], d1[CPL];
      {
        const uint32_t src0 = ring_s + ((2 * s) & (kRing2 - 1)) * kSlot;
#pragma unroll
        for (int v = 0; v < CPL / 4; ++v) {
          float4 q0, q1;
          asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                       : "=f"(q0.x), "=f"(q0.y), "=f"(q0.z), "=f"(q0.w) : "r"(src0 + v * 16));
          asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                       : "=f"(q1.x), "=f"(q1.y), "=f"(q1.z), "=f"(q1.w) : "r"(src0 + kSlot + v * 16));
          d0[4 * v] = q0.x; d0[4 * v + 1] = q0.y; d0[4 * v + 2] = q0.z; d0[4 * v + 3] = q0.w;
          d1[4 * v] = q1.x; d1[4 * v + 1] = q1.y; d1[4 * v + 2] = q1.z; d1[4 * v + 3] = q1.w;
        }
      }
      float umin0 = 3.0e38f, umin1 = 3.0e38f;
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        const float2 dy = fsub2(pn[c + 1], pp[c + 1]);
        const float2 dx = make_float2(pp[c + 2].y - pp[c].y, pn[c + 2].x - pn[c].x);
        const float2 s2 = ffma2(dx, dx, fmul2(dy, dy));
        const float h0v = sqrt_approx(s2.x), h1v = sqrt_approx(s2.y);   // 2|grad phi|
        const float vf0 = (MODEL == REGION) ? fmaf(A, d0[c], B) : d0[c];
        const float vf1 = (MODEL == REGION) ? fmaf(A, d1[c], B) : d1[c];
        const float u0 = fmaf(vf0, h0v, pp[c + 1].y);
        const float u1 = fmaf(vf1, h1v, pn[c + 1].x);
        ow[c] = __funnelshift_l(__float_as_uint(u0), ow[c], 1);
        ow[c] = __funnelshift_l(__float_as_uint(u1), ow[c], 1);
        umin0 = fminf(umin0, fabsf(u0));
        umin1 = fminf(umin1, fabsf(u1));
        LSE_CHECK_U(R, SRC, P, tile_ctx(P, tile), tile_bits(P, tile),
                    y0 - tile_y0(P, tile) + h0 + 2 * s, x0 + c, u0, eps_u);
        LSE_CHECK_U(R, SRC, P, tile_ctx(P, tile), tile_bits(P, tile),
                    y0 - tile_y0(P, tile) + h0 + 2 * s + 1, x0 + c, u1, eps_u);
      }
      if (umin0 <= eps_u) fbrows |= 1u << (h0 + 2 * s);
      if (umin1 <= eps_u) fbrows |= 2u << (h0 + 2 * s);
#pragma unroll
      for (int c = 0; c < NP; ++c) pp[c] = pn[c];
    }
    cp_async_wait<0>();
    // RP appended sign bits: after the reversal rows h0 .. h0+RP-1 sit in the
    // top RP bits
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      const uint32_t v = ~__brev(ow[c]) & (0xffffffffu << (32 - RP));
      ow[c] = v >> (32 - RP - h0);
    }
    while (fbrows) {
      const int k = __ffs(fbrows) - 1;
      fbrows &= fbrows - 1;
      const uint32_t bitk = 1u << k;
      uint32_t cols = update_tie_cols<R, MODEL, CPL, SRC>(P, lut_base, r, x0, k, A, B, eps_u);
      while (cols) {
        const int c = __ffs(cols) - 1;
        cols &= cols - 1;
        const bool pos = exact_u_fast<R, SRC>(tile_ctx(P, tile), tile_bits(P, tile),
                                              y0 - tile_y0(P, tile) + k, x0 + c) > 0.0;
#pragma unroll
        for (int q = 0; q < CPL; ++q)
          if (q == c) ow[q] = pos ? (ow[q] | bitk) : (ow[q] & ~bitk);
      }
    }
  }
#pragma unroll
  for (int m = 32 / NS; m < 32; m <<= 1)
#pragma unroll
    for (int c = 0; c < CPL; ++c) ow[c] |= __shfl_xor_sync(0xffffffffu, ow[c], m);
  if (!act || h0) return;
  uint32_t* dst = P.bits_out + (size_t)r * P.g.pitch_w + x0;
#pragma unroll
  for (int q = 0; q < CPL / 4; ++q)
    reinterpret_cast<uint4*>(dst)[q] = make_uint4(ow[4 * q], ow[4 * q + 1], ow[4 * q + 2], ow[4 * q + 3]);
}

// Shared lookup tables: the t-LUT and s-LUT (2^(2R+1) floats each) and the
// pair table (2^(2R+2) float2).  phi_rows2_int adds the pair table's shared
// address to the byte offset; with the table a static __shared__ array that
// address is a link-time constant the compiler folds into the LDS immediate.
struct SharedLuts {
  float* lt;
  float* ls;
  uint32_t lt2;                                  // pair table (shared address, g_pair_lut)
};

template <int R>
__device__ __forceinline__ void load_luts(const FastParams& P, const SharedLuts& L) {
  constexpr int NPAT = 1 << (2 * R + 1);
  for (int q = threadIdx.x; q < NPAT; q += blockDim.x) {
    L.lt[q] = __ldg(&P.lut_t[q]);
    L.ls[q] = __ldg(&P.lut_s[q]);
  }
  float2* lt2 = g_pair_lut;                     // 2 NPAT entries
  for (int q = threadIdx.x; q < 2 * NPAT; q += blockDim.x)
    lt2[q] = make_float2(__ldg(&P.lut_t[q & (NPAT - 1)]), __ldg(&P.lut_t[q >> 1]));
}

__device__ __forceinline__ int grab_unit(const FastParams& P, int lane) {
  // dynamic unit scheduling: grabs are counted from this launch's base, so the
  // counter never needs a reset (each warp makes exactly one failing grab)
  unsigned long long g = 0;
  if (lane == 0) g = atomicAdd(P.work, 1ull) - P.work_base;
  g = (unsigned long long)__shfl_sync(0xffffffffu, (long long)g, 0);
  return g > 0x7fffffffull ? 0x7fffffff : (int)g;     // out of window: treated as "no work" 
}

// INT = true : interior units (exact-rounded LUT, central differences, and
// the uniform-window skip: a chunk whose every lane sees all-equal bits over
// rows y0-32 .. y0+63 of its t columns has phi constant there, hence
// |grad phi| == 0, v == 0 and u == phi exactly, so b^{n+1} == b^n and the
// chunk is copied without reading the data plane).
// INT = false: border units (zero padding, one-sided gradients).
// Border rows k0 .. k0 + nrows - 1 of the lane block (r, x0): zero
// padding / one-sided gradients (update_block's arithmetic on a row range).
// ow[c] gets bit k for the rows of the range only.
// FUSED: eps_u holds the speculative band's e0; flagged pixels go to the fix
// list instead of the exact path (see update_block_int2).
template <int R, int MODEL, int SRC, int CPL, bool FUSED = false>
__device__ __forceinline__ void update_rows_border(const FastParams& P, const float* s_lt,
                                                   const float* s_ls, int r, int x0, int k0,
                                                   int nrows, float A, float B, float eps_u,
                                                   uint32_t (&ow)[CPL], float delta = 0.f) {
  constexpr int NT = CPL + 2 * (R + 1);
  constexpr int NP = CPL + 2;
  const int H = P.g.H, W = P.g.W;
  const int y0 = r * 32;
  const int base = y0 + k0 - 1 - R;              // window row 0 (phi row y0+k0-1 at m0 = 0)
  const int wr = base >> 5, sh = base & 31;
  uint32_t cm[NT], win[NT];
#pragma unroll
  for (int j = 0; j < NT; ++j) {
    const int xc = x0 - (R + 1) + j;
    cm[j] = (xc >= 0 && xc < W) ? 0xffffffffu : 0u;
    win[j] = __funnelshift_r(word_at<false>(P, wr, xc), word_at<false>(P, wr + 1, xc), sh);
  }
  float pm[NP], p0[NP], pn[NP], dcur[CPL], dnext[CPL];
  uint32_t fbrows = 0u;
  // flagged pixels of the first 8 rows of the range (bit 8 (k - k0) + c): border
  // ranges are at most 8 rows, so only those pixels take the fp64 evaluation
  // (a whole flagged row cost 8 general-path evaluations of ~10 us each and
  // made single border units the critical path of mid-size images)
  static_assert(CPL <= 8, "column mask");
  unsigned long long fbm = 0ull;
#pragma unroll
  for (int c = 0; c < CPL; ++c) { ow[c] = 0u; dcur[c] = 0.f; dnext[c] = 0.f; }
  phi_row<R, SRC, false, NT, NP>(P, win, cm, 0, y0 + k0 - 1, s_lt, s_ls, pm);
  phi_row<R, SRC, false, NT, NP>(P, win, cm, 1, y0 + k0, s_lt, s_ls, p0);
  load_data_row<false, CPL>(P, y0 + k0, x0, dcur);
#pragma unroll 1
  for (int k = k0; k < k0 + nrows; ++k) {
    const int kk = k + 1;                        // phi row produced in this step
    if (kk < k0 + nrows) load_data_row<false, CPL>(P, y0 + kk, x0, dnext);
    phi_row<R, SRC, false, NT, NP>(P, win, cm, kk - k0 + 1, y0 + kk, s_lt, s_ls, pn);
    const int i = y0 + k;
    if (i < H) {
      const uint32_t bitk = 1u << k;
      uint32_t fb = 0u;
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        const int x = x0 + c;
        if (x >= W) continue;
        const float dx = (x == 0) ? 2.f * (p0[c + 2] - p0[c + 1])
                         : (x == W - 1) ? 2.f * (p0[c + 1] - p0[c]) : (p0[c + 2] - p0[c]);
        const float dy = (i == 0) ? 2.f * (pn[c + 1] - p0[c + 1])
                         : (i == H - 1) ? 2.f * (p0[c + 1] - pm[c + 1]) : (pn[c + 1] - pm[c + 1]);
        const float h = sqrt_approx(fmaf(dx, dx, dy * dy));
        // h = 2|grad phi|; A, B (region) and the g plane (edge) carry dt/2
        const float vf = (MODEL == REGION) ? fmaf(A, dcur[c], B) : dcur[c];
        const float u = fmaf(vf, h, p0[c + 1]);
        if (u > 0.f) ow[c] |= bitk;
        if ((FUSED ? fmaf(-delta, h, fabsf(u)) : fabsf(u)) <= eps_u) fb |= 1u << c;
        if (!FUSED) LSE_CHECK_U(R, SRC, P, P.ctx, P.bits_in, y0 + k, x, u, eps_u);
      }
      if (fb) {
        fbrows |= bitk;
        if (k - k0 < 8) fbm |= (unsigned long long)fb << (8 * (k - k0));
      }
    }
#pragma unroll
    for (int c = 0; c < NP; ++c) { pm[c] = p0[c]; p0[c] = pn[c]; }
#pragma unroll
    for (int c = 0; c < CPL; ++c) dcur[c] = dnext[c];
  }
  while (fbrows) {                               // near ties: exact fp64 decisions
    const int k = __ffs(fbrows) - 1;
    fbrows &= fbrows - 1;
    const uint32_t bitk = 1u << k;
    const uint32_t cols = (k - k0 < 8) ? (uint32_t)(fbm >> (8 * (k - k0))) & 0xffu : 0xffu;
#pragma unroll 1
    for (int c = 0; c < CPL; ++c) {
      if (x0 + c >= W) break;
      if (!((cols >> c) & 1u)) continue;
      // fused pass: a flagged pixel goes to the fix list and is also decided
      // exactly with the coefficients used (final if they turn out unchanged)
      if (FUSED) {
        if (P.ctx->model != EDGE) spec_append(P, y0 + k, x0 + c);
        if (!LSE_SPEC_INLINE) continue;
      }
      const bool pos = exact_u_fast<R, SRC>(P.ctx, P.bits_in, y0 + k, x0 + c) > 0.0;
#pragma unroll
      for (int q = 0; q < CPL; ++q)
        if (q == c) ow[q] = pos ? (ow[q] | bitk) : (ow[q] & ~bitk);
    }
  }
}

// Border unit: bitems lane groups x bq row parts.  Called by every lane of
// the warp (the parts are merged with shuffles); not
// inlined, so its register needs do not constrain the interior loop.
template <int R, int MODEL, int SRC>
__device__ __forceinline__ void border_update_body(const FastParams& P, const float* s_lt,
                                                   const float* s_ls, int unit, float A, float B,
                                                   float eps_u, bool stopped) {
  constexpr int CPL = kUpdCols;
  const int lane = threadIdx.x & 31;
  int r = 0, x0 = 0;
  const bool act = border_lane(P.gu, unit, lane, P.g.W, r, x0);
  const int items = P.gu.bitems;                 // lane groups per unit = rows per lane
  if (stopped) {                                 // converged tile: keep its state
    if (!act || lane >= items) return;
    const uint32_t* src = P.bits_in + (size_t)r * P.g.pitch_w + x0;
    uint32_t* dst = P.bits_out + (size_t)r * P.g.pitch_w + x0;
#pragma unroll
    for (int q = 0; q < CPL / 4; ++q)
      reinterpret_cast<uint4*>(dst)[q] = reinterpret_cast<const uint4*>(src)[q];
    return;
  }
  uint32_t ow[CPL];
#pragma unroll
  for (int c = 0; c < CPL; ++c) ow[c] = 0u;
  if (act)
    update_rows_border<R, MODEL, SRC, CPL>(P, s_lt, s_ls, r, x0, (lane / items) * items, items,
                                           A, B, eps_u, ow);
  for (int o = items; o < 32; o <<= 1) {
#pragma unroll
    for (int c = 0; c < CPL; ++c) ow[c] |= __shfl_xor_sync(0xffffffffu, ow[c], o);
  }
  if (!act || lane >= items) return;
  uint32_t* dst = P.bits_out + (size_t)r * P.g.pitch_w + x0;
#pragma unroll
  for (int q = 0; q < CPL / 4; ++q)
    reinterpret_cast<uint4*>(dst)[q] = make_uint4(ow[4 * q], ow[4 * q + 1], ow[4 * q + 2], ow[4 * q + 3]);
}

// the tile-local view of a batched launch: every pointer at the tile's first
// row, the tile's scalars / context, the tile's height
__device__ __forceinline__ void tile_view(FastParams& Q, int tile) {
  Q.bits_in += (size_t)tile * Q.tile_words;
  Q.bits_out += (size_t)tile * Q.tile_words;
  Q.pbits += (size_t)tile * Q.tile_words;
  Q.mbits += (size_t)tile * Q.tile_words;
  Q.data32 += (size_t)tile * Q.tile_data;
  Q.scal += tile;
  Q.ctx += tile;
  Q.g.H = Q.tile_h;
  Q.g.HR = Q.tile_hr;
  Q.fix_row0 += tile * Q.tile_hr * 32;
}

template <int R, int MODEL, int SRC, bool BATCH>
__device__ __noinline__ void border_update_unit(const FastParams& P, const float* s_lt,
                                                const float* s_ls, int unit, int tile, float A,
                                                float B, float eps_u, bool stopped) {
  if (!BATCH) {
    border_update_body<R, MODEL, SRC>(P, s_lt, s_ls, unit, A, B, eps_u, false);
    return;
  }
  FastParams Q = P;
  tile_view(Q, tile);
  border_update_body<R, MODEL, SRC>(Q, s_lt, s_ls, unit, A, B, eps_u, stopped);
}

// One launch covers every unit: [border units][interior units] (border first,
// so their longer latency overlaps the interior work of the other warps).
// BATCH: every unit of every tile, [all border units][all interior units];
// the tile's scalars (stop, A, B, guards) are read per unit.
// NS > 1: split-warp units of 256/NS columns (update_block_split) for small
// images.
// The unit loop of k_update (also the redo pass of k_spec_fix): the launch's
// units are grabbed from P.work until exhausted.
template <int R, int MODEL, int SRC, bool BATCH, int NS>
__device__ __forceinline__ void update_units(const FastParams& P, const FastParams& s_P,
                                             const SharedLuts& luts, const float* s_lt,
                                             const float* s_ls, float* s_ring) {
  constexpr int CPL = kUpdCols;
  constexpr int NT = CPL + 2 * (R + 1);
  LSE_TRACE_ENTRY
  const Scalars* sc = P.scal;
  float A = sc->A, B = sc->B, eps_u = sc->eps_u;
  const int lane = threadIdx.x & 31;
  const int nb = border_units(P.gu);
  constexpr int LPP = 32 / NS;                   // lanes per row part
  const int ni = NS > 1 ? NS * chunk_units(P.gu) + (P.gu.nB1 + LPP - 1) / LPP
                        : interior_units(P.gu);
  const int T = BATCH ? P.ntiles : 1;
  const int nunits = T * (nb + ni);
  LSE_TRACE_DECL
  for (;;) {
    const int unit = grab_unit(P, lane);
    LSE_TRACE_MARK(unit < nunits ? unit : -1);
    if (unit >= nunits) break;
    int tile = 0, lu = unit;
    bool stopped = false;
    if (BATCH) {
      if (unit < T * nb) {
        tile = unit / nb;
        lu = unit - tile * nb;
      } else {
        const int iu = unit - T * nb;
        tile = iu / ni;
        lu = nb + (iu - tile * ni);
      }
      const Scalars* st = P.scal + tile;
      if (P.redo_only && !__ldcg(&st->redo)) continue;   // (its speculative update stands)
      stopped = stop_flag(st) != 0;
      A = st->A;
      B = st->B;
      eps_u = st->eps_u;
    }
    int r = 0, x0 = 0;
    if (lu < nb) {
      border_update_unit<R, MODEL, SRC, BATCH>(s_P, s_lt, s_ls, lu, tile, A, B, eps_u, stopped);
      continue;
    }
    const int iu = lu - nb;
    bool act = true;
    const int nch = chunk_units(P.gu);
    if (NS > 1) {                                 // sub-chunks; lanes L, L+LPP, .. share columns
      if (iu < NS * nch) {
        const int ch = iu / NS;
        r = P.gu.r_lo + ch / P.gu.nci;
        x0 = P.gu.xoff + (ch % P.gu.nci) * kUpdChunk + (iu % NS) * (kUpdChunk / NS) +
             CPL * (lane % LPP);
      } else {
        act = b1_lane(P.gu, 0, (iu - NS * nch) * LPP + (lane % LPP), r, x0);
      }
    } else if (iu < nch) {
      r = P.gu.r_lo + iu / P.gu.nci;
      x0 = P.gu.xoff + (iu % P.gu.nci) * kUpdChunk + CPL * lane;
    } else {
      act = b1_lane(P.gu, iu - nch, lane, r, x0);
    }
    if (BATCH) r += tile * P.tile_hr;             // row of the tile in the stacked arrays
    if constexpr (NS > 1) {
      // window words of this lane's part: rows r-1, r (part 0) or r, r+1
      uint32_t wlo[NT], whi[NT];
      uint32_t a = ~0u, o = 0u;
      if (act) {
        const uint32_t* wp =
            P.bits_in + (size_t)(r - 1 + (lane >= LPP)) * P.g.pitch_w + (x0 - (R + 1));
#pragma unroll
        for (int j = 0; j < NT; ++j) {
          wlo[j] = __ldg(wp + j);
          whi[j] = __ldg(wp + P.g.pitch_w + j);
          a &= wlo[j] & whi[j];
          o |= wlo[j] | whi[j];
        }
      }
      if (stopped || (P.skip_uniform && __all_sync(0xffffffffu, !act || a == ~0u || o == 0u))) {
        if (!act || lane >= LPP) continue;
        uint32_t* dst = P.bits_out + (size_t)r * P.g.pitch_w + x0;
#pragma unroll
        for (int q = 0; q < CPL / 4; ++q)
          reinterpret_cast<uint4*>(dst)[q] = make_uint4(whi[R + 1 + 4 * q], whi[R + 2 + 4 * q],
                                                        whi[R + 3 + 4 * q], whi[R + 4 + 4 * q]);
        continue;
      }
      update_block_split<R, MODEL, CPL, SRC, NS>(P, luts.lt2,
                                            s_ring + (threadIdx.x >> 5) * kRing2 * 32 * CPL, r,
                                            x0, A, B, eps_u, wlo, whi, tile, act);
      continue;
    }
    uint32_t prev[NT], cur[NT];
    uint32_t a = ~0u, o = 0u;
    if (act) {
      const uint32_t* wp = P.bits_in + (size_t)(r - 1) * P.g.pitch_w + (x0 - (R + 1));
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        prev[j] = __ldg(wp + j);
        cur[j] = __ldg(wp + P.g.pitch_w + j);
        if (P.skip_uniform) {
          const uint32_t nx = __ldg(wp + 2 * (size_t)P.g.pitch_w + j);
          a &= prev[j] & cur[j] & nx;
          o |= prev[j] | cur[j] | nx;
        }
      }
    }
    // uniform-window skip: phi constant over the block's stencil => b unchanged
    // (a converged tile of a batch keeps its state the same way)
    if (stopped || (P.skip_uniform && __all_sync(0xffffffffu, !act || a == ~0u || o == 0u))) {
      if (!act) continue;
      uint32_t* dst = P.bits_out + (size_t)r * P.g.pitch_w + x0;
#pragma unroll
      for (int q = 0; q < CPL / 4; ++q)
        reinterpret_cast<uint4*>(dst)[q] = make_uint4(cur[R + 1 + 4 * q], cur[R + 2 + 4 * q],
                                                      cur[R + 3 + 4 * q], cur[R + 4 + 4 * q]);
      continue;
    }
    if (!act) continue;
    uint32_t npw[CPL], nmw[CPL];                  // (partition words: fused pass only)
    update_block_int2<R, MODEL, CPL, SRC>(P, luts.lt2,
                                          s_ring + (threadIdx.x >> 5) * kRing2 * 32 * CPL, r, x0,
                                          A, B, eps_u, prev, cur, tile, 0.f, npw, nmw, s_P);
  }
}

template <int R, int MODEL, int SRC, bool BATCH, int NS>
__global__ void __launch_bounds__(kThreads, kUpdateCtasPerSm) k_update(FastParams P) {
  constexpr int CPL = kUpdCols;
  constexpr int NPAT = 1 << (2 * R + 1);
  __shared__ float s_lt[NPAT];
  __shared__ float s_ls[NPAT];
  __shared__ __align__(16) float s_ring[(kThreads / 32) * kRing2 * 32 * CPL];
  // the noinline border path reads the launch parameters from this shared
  // copy: handing it the kernel parameter block itself would force a
  // per-thread local-memory copy of the block (taking its address)
  __shared__ FastParams s_P;
  const SharedLuts luts{s_lt, s_ls, (uint32_t)__cvta_generic_to_shared(g_pair_lut)};
  load_luts<R>(P, luts);                         // static data: before the dependency wait
  if (threadIdx.x == 0) s_P = P;
  __syncthreads();
  pdl_wait();
  pdl_launch_dependents();
  if (!BATCH && stop_flag(P.scal)) return;
  if (MODEL == REGION && blockIdx.x == 0) {      // sticky degenerate (engine.py:239-240)
    for (int t = threadIdx.x; t < (BATCH ? P.ntiles : 1); t += blockDim.x)
      if (P.scal[t].zero_vel && !P.scal[t].stop && P.scal[t].model != EDGE)
        P.scal[t].degenerate = 1;
  }
  update_units<R, MODEL, SRC, BATCH, NS>(P, s_P, luts, s_lt, s_ls, s_ring);
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
    double a, b;
    if (sc->model == ZHANG) {                      // models.py:152-155
      const double m = dmul(0.5, dadd(cp, cm));
      const double pmax = fabs(dsub(sc->img_max, m)), pmin = fabs(dsub(sc->img_min, m));
      peak = pmax > pmin ? pmax : pmin;
      sc->mid = m;
      a = sc->nu / peak;
      b = -sc->nu * m / peak;
    } else {
      a = 2.0 * dc / peak;
      b = -dc * (cp + cm) / peak;
    }
    sc->c_pos = cp;
    sc->c_neg = cm;
    sc->dc = dc;
    sc->peak = peak;
    if (peak == 0.0) {                             // models.py:117-118, 156-157
      sc->zero_vel = 1;
    } else {
      sc->A = (float)(0.5 * dt * a);    // kernels evaluate u = phi + (A I + B) * 2|grad phi|
      sc->B = (float)(0.5 * dt * b);
      double eps_d = 0x1p-21 * (fabs(a) * sc->img_absmax + fabs(b) + 1.0);
      // |v / |grad phi|| <= 1 for the region model, <= |nu| for zhang
      const double vs = sc->model == ZHANG ? fmax(1.0, fabs(sc->nu)) : 1.0;
      sc->eps_u = (float)(kGuard * (kErrPhi + dt * vs * (kErrGrad + 1.5 * eps_d + 0x1p-21) +
                                    0x1p-22 * (1.0 + 1.5 * dt * vs)));
    }
  }
  if (sc->zero_vel) {
    sc->A = 0.f;
    sc->B = 0.f;
    sc->eps_u = (float)(kGuard * (kErrPhi + 0x1p-22));
  }
}

// Whole-CTA reduction of the unit partials in a fixed order (each thread a
// contiguous range, then a fixed xor-shuffle tree, then warps in index order;
// deterministic for a given n and blockDim), followed by the scalar
// bookkeeping on one thread.  Launched as its own 1-CTA x 1024-thread kernel.
__device__ __forceinline__ void dd_shfl_add(double& hi, double& lo, int o) {
  const double h2 = __shfl_xor_sync(0xffffffffu, hi, o);
  const double l2 = __shfl_xor_sync(0xffffffffu, lo, o);
  dd_add_dd(hi, lo, h2, l2);
}

// The partials form one virtual array: part0[0..n0) ++ part1[0..n1) ++ part2[0..n2).
struct PartRanges {
  const TilePartial* p[3];
  int n[3];
};

__device__ __forceinline__ const TilePartial* part_at(const PartRanges& R3, int t) {
  if (t < R3.n[0]) return R3.p[0] + t;
  t -= R3.n[0];
  if (t < R3.n[1]) return R3.p[1] + t;
  return R3.p[2] + (t - R3.n[1]);
}

// Fixed-order CTA reduction of the virtual partial array slice [t0, t1) into
// one double-double partial (written by thread 0 to *out) -- stage 1 of the
// finalize, run by many CTAs.
__device__ void reduce_slice(const PartRanges& R3, int t0, int t1, TilePartial* out) {
  __shared__ double g_ah[32], g_al[32], g_bh[32], g_bl[32];
  __shared__ long long g_na[32], g_nb[32];
  __shared__ unsigned long long g_mm[32];
  const int T = blockDim.x, tid = threadIdx.x;
  double ah = 0, al = 0, bh = 0, bl = 0;
  long long na = 0, nb = 0;
  unsigned long long mm = 0;
  const int n = t1 - t0;
  const int per = (n + T - 1) / T;
  const int lo = t0 + tid * per;
  const int hi = min(lo + per, t1);
  for (int t = lo; t < hi; ++t) {
    const TilePartial* p = part_at(R3, t);
    const double2 A = __ldcg(reinterpret_cast<const double2*>(&p->a_hi));
    const double2 B = __ldcg(reinterpret_cast<const double2*>(&p->b_hi));
    const longlong2 NN = __ldcg(reinterpret_cast<const longlong2*>(&p->n_a));
    dd_add_dd(ah, al, A.x, A.y);
    dd_add_dd(bh, bl, B.x, B.y);
    na += NN.x;
    nb += NN.y;
    mm += __ldcg(&p->mism);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    dd_shfl_add(ah, al, o);
    dd_shfl_add(bh, bl, o);
    na += __shfl_xor_sync(0xffffffffu, na, o);
    nb += __shfl_xor_sync(0xffffffffu, nb, o);
    mm += __shfl_xor_sync(0xffffffffu, mm, o);
  }
  const int warp = tid >> 5, lane = tid & 31;
  if (lane == 0) {
    g_ah[warp] = ah; g_al[warp] = al; g_bh[warp] = bh; g_bl[warp] = bl;
    g_na[warp] = na; g_nb[warp] = nb; g_mm[warp] = mm;
  }
  __syncthreads();
  if (tid == 0) {
    TilePartial t{};
    for (int w = 0; w < (T + 31) / 32; ++w) {
      dd_add_dd(t.a_hi, t.a_lo, g_ah[w], g_al[w]);
      dd_add_dd(t.b_hi, t.b_lo, g_bh[w], g_bl[w]);
      t.n_a += g_na[w];
      t.n_b += g_nb[w];
      t.mism += g_mm[w];
    }
    *out = t;
  }
}

// Check of a speculative update (spec = 1 + parity of its fix list) against
// the coefficients just computed, and the flag band of the next one.
// Not flagged means |u_g| - delta*h > e0 (the kernels' fp32 test is exact
// enough: fl(|u| - delta h) > e0 implies |u| - delta h > e0).  With vf_g =
// A' I + B' the kernel's, vf_t = A I + B the true coefficient of I, and
// |vf_g - vf_t| <= |A - A'| max|I| + |B - B'| + 2^-23 max|vf| (two FMA
// roundings), |u_g - u_t| <= |vf_g - vf_t| h + 2^-23 |u_g| (1 + tiny): so
// delta (1 - 2^-20) >= (that bound) (1 + 2^-20) and e0 (1 - 2^-20) >= eps_u of
// the true coefficients give |u_t| > eps_u with sign(u_t) = sign(u_g), i.e.
// the unflagged decisions are the ones the non-speculative update makes.
// exact coefficients of an update (what the exact evaluators read)
struct ExactCoefs {
  double cp, cm, dc, peak, mid;
  int zero;
};
__device__ __forceinline__ ExactCoefs exact_coefs(const Scalars* sc) {
  return ExactCoefs{sc->c_pos, sc->c_neg, sc->dc, sc->peak, sc->mid, sc->zero_vel};
}

// base: the scalars holding the fix-list counters and the redo work counter
// (the run's own; tile 0's for every tile of a batch)
__device__ __forceinline__ void spec_check(Scalars* sc, float A0, float B0, float delta0, float e00,
                                           int spec, const ExactCoefs& k0, Scalars* base) {
  const double am = sc->img_absmax * (1.0 + 0x1p-20);
  const double A = sc->A, B = sc->B, a0 = A0, b0 = B0;
  const double D = (fabs(A - a0) * am + fabs(B - b0)) * (1.0 + 0x1p-40);
  const double vfm = fmax(fabs(A) * am + fabs(B), fabs(a0) * am + fabs(b0));
  if (spec) {
    const unsigned nfix = base->fix_n[spec - 1];
    const bool ok = nfix <= base->fix_cap &&
                    (double)delta0 * (1.0 - 0x1p-20) >= (D + 0x1p-22 * vfm) * (1.0 + 0x1p-20) &&
                    (double)e00 * (1.0 - 0x1p-20) >= (double)sc->eps_u;
    sc->redo = ok ? 0 : 1;
    // coefficients bit-identical to the ones the pass used (the partition did
    // not move): its decisions -- the guard band decided exactly in the pass
    // -- are final and the fix list is not needed
    const ExactCoefs k1 = exact_coefs(sc);
    const bool same = LSE_SPEC_INLINE && (float)A == A0 && (float)B == B0 && k1.zero == k0.zero &&
                      k1.cp == k0.cp && k1.cm == k0.cm && k1.dc == k0.dc && k1.peak == k0.peak &&
                      k1.mid == k0.mid;
    sc->fix_needed = same ? 0 : 1;
    if (ok) {
      if (!same) sc->spec_fixes += nfix;
    } else {
      sc->spec_redos += 1;
      base->work2 = 0;
      if (base != sc) atomicOr(&base->redo_any, 1);
    }
  }
  // next band: 4x the last move of the coefficients plus a floor; none when
  // they still move by more than 1/8 of the velocity scale (early iterations)
  const double nd = 4.0 * D + 0x1p-14 * vfm;
  sc->spec_delta = nd <= vfm * 0x1p-3 ? (float)(nd * (1.0 + 0x1p-20)) : -1.0f;
  sc->spec_e0 = (float)((double)sc->eps_u * 1.25);
}

__device__ void finalize_cta(const PartRanges& R3, Scalars* sc, bool delta, bool region,
                             bool ckpt, long long iter, int spec = 0, Scalars* base = nullptr) {
  const int n = R3.n[0] + R3.n[1] + R3.n[2];
  __shared__ double f_ah[32], f_al[32], f_bh[32], f_bl[32];
  __shared__ long long f_na[32], f_nb[32];
  __shared__ unsigned long long f_mm[32];
  const int T = blockDim.x, tid = threadIdx.x;
  double ah = 0, al = 0, bh = 0, bl = 0;
  long long na = 0, nb = 0;
  unsigned long long mm = 0;
  const int per = (n + T - 1) / T;
  const int lo = tid * per;
  const int hi = lo + per < n ? lo + per : n;
  int t = lo;
  for (; t + 4 <= hi; t += 4) {          // 4 partials in flight per thread
    double2 A[4], B[4];
    longlong2 NN[4];
    unsigned long long M[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const TilePartial* p = part_at(R3, t + q);
      A[q] = __ldcg(reinterpret_cast<const double2*>(&p->a_hi));
      B[q] = __ldcg(reinterpret_cast<const double2*>(&p->b_hi));
      NN[q] = __ldcg(reinterpret_cast<const longlong2*>(&p->n_a));
      M[q] = __ldcg(&p->mism);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      dd_add_dd(ah, al, A[q].x, A[q].y);
      dd_add_dd(bh, bl, B[q].x, B[q].y);
      na += NN[q].x;
      nb += NN[q].y;
      mm += M[q];
    }
  }
  for (; t < hi; ++t) {
    const TilePartial* p = part_at(R3, t);
    const double2 A = __ldcg(reinterpret_cast<const double2*>(&p->a_hi));
    const double2 B = __ldcg(reinterpret_cast<const double2*>(&p->b_hi));
    const longlong2 NN = __ldcg(reinterpret_cast<const longlong2*>(&p->n_a));
    dd_add_dd(ah, al, A.x, A.y);
    dd_add_dd(bh, bl, B.x, B.y);
    na += NN.x;
    nb += NN.y;
    mm += __ldcg(&p->mism);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    dd_shfl_add(ah, al, o);
    dd_shfl_add(bh, bl, o);
    na += __shfl_xor_sync(0xffffffffu, na, o);
    nb += __shfl_xor_sync(0xffffffffu, nb, o);
    mm += __shfl_xor_sync(0xffffffffu, mm, o);
  }
  const int warp = tid >> 5, lane = tid & 31;
  if (lane == 0) {
    f_ah[warp] = ah; f_al[warp] = al; f_bh[warp] = bh; f_bl[warp] = bl;
    f_na[warp] = na; f_nb[warp] = nb; f_mm[warp] = mm;
  }
  __syncthreads();
  if (tid == 0) {
    double sah = 0, sal = 0, sbh = 0, sbl = 0;
    long long sna = 0, snb = 0;
    unsigned long long smm = 0;
    for (int w = 0; w < (T + 31) / 32; ++w) {
      dd_add_dd(sah, sal, f_ah[w], f_al[w]);
      dd_add_dd(sbh, sbl, f_bh[w], f_bl[w]);
      sna += f_na[w];
      snb += f_nb[w];
      smm += f_mm[w];
    }
    if (region) {
      const float A0 = sc->A, B0 = sc->B, delta0 = sc->spec_delta, e00 = sc->spec_e0;
      const ExactCoefs k0 = exact_coefs(sc);
      if (delta) {
        dd_add_dd(sc->sp_hi, sc->sp_lo, sah, sal);
        dd_add_dd(sc->sp_hi, sc->sp_lo, -sbh, -sbl);
        dd_add_dd(sc->sn_hi, sc->sn_lo, sbh, sbl);
        dd_add_dd(sc->sn_hi, sc->sn_lo, -sah, -sal);
        sc->n_pos += sna - snb;
      } else {
        sc->sp_hi = sah; sc->sp_lo = sal;
        sc->sn_hi = sbh; sc->sn_lo = sbl;
        sc->n_pos = sna;
      }
      region_coeffs(sc);
      spec_check(sc, A0, B0, delta0, e00, spec, k0, base ? base : sc);
    }
    if (ckpt) {                                    // engine.py:228-236
      sc->n_ckpt += 1;
      if (sc->n_ckpt >= 2) sc->equal_run = (smm == 0) ? sc->equal_run + 1 : 0;
      const long long cw = sc->conv_window;
      if (cw == 1 || (sc->n_ckpt >= cw && sc->equal_run >= cw - 1)) {
        sc->stop = 1;
        sc->converged = 1;
        sc->converged_iter = iter;
        // a batched tile converging after a speculative pass: the pass has
        // written b^{iter+1}; the redo pass puts b^{iter} back (a stopped
        // tile's units copy their state)
        if (spec && base && base != sc) {
          sc->redo = 1;
          base->work2 = 0;
          atomicOr(&base->redo_any, 1);
        }
      }
    }
  }
}

// ------------------------------------------------------------- partition
// One lane: columns x0..x0+7 of word-row r.  Signs of phi^{n+1} = G*b^{n+1}
// (t columns x0-R .. x0+7+R, no row halo), partition bits {phi >= 0} with the
// incremental c+/c- sums, checkpoint mask {phi > 0} with the mismatch count.
template <int R, bool INT>
__device__ __forceinline__ void partition_block(const FastParams& P, const float* s_lt,
                                                const float* s_ls, uint32_t lut_base, int r,
                                                int x0, float eps_phi,
                                                const uint32_t (&prev)[8 + 2 * R],
                                                const uint32_t (&cur)[8 + 2 * R],
                                                uint32_t (&pw)[8], uint32_t (&mw)[8], int tile) {
  constexpr int NT = kColsPerThread + 2 * R;
  const int H = P.g.H, W = P.g.W;
  const int y0 = r * 32;
  uint32_t cm[NT], win[NT];
#pragma unroll
  for (int j = 0; j < NT; ++j) {
    const int xc = x0 - R + j;
    cm[j] = (INT || (xc >= 0 && xc < W)) ? 0xffffffffu : 0u;
    win[j] = __funnelshift_r(prev[j], cur[j], 32 - R);     // base row y0-R
    if (INT) win[j] <<= 3;                                  // byte offsets for phi_rows2_int
  }
  float ph[8];
  uint32_t fbrows = 0u;
#pragma unroll
  for (int c = 0; c < 8; ++c) { pw[c] = 0u; mw[c] = 0u; }
  if (INT) {
    // row pairs (k, k+1), k = 2 kk
#pragma unroll 1
    for (int kk = 0; kk < 16; ++kk) {
      const int k = 2 * kk;
      if (kk == 8) {                                        // base row y0+16-R
#pragma unroll
        for (int j = 0; j < NT; ++j) {
          const int xc = x0 - R + j;
          win[j] = __funnelshift_r(word_at<INT>(P, r, xc), word_at<INT>(P, r + 1, xc), 16 - R)
                   << 3;
        }
      }
      float2 ph2[8];
      phi_rows2_int<R, NT, 8>(P, win, k < 16 ? k : k - 16, lut_base, ph2);
      float pmin0 = 3.0e38f, pmin1 = 3.0e38f;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        pw[c] = __funnelshift_l(__float_as_uint(ph2[c].x), pw[c], 1);   // sign bits, reversed
        pw[c] = __funnelshift_l(__float_as_uint(ph2[c].y), pw[c], 1);
        pmin0 = fminf(pmin0, fabsf(ph2[c].x));
        pmin1 = fminf(pmin1, fabsf(ph2[c].y));
        LSE_CHECK_PHI(R, P, tile_ctx(P, tile), tile_bits(P, tile), y0 - tile_y0(P, tile) + k,
                      x0 + c, ph2[c].x, eps_phi);
        LSE_CHECK_PHI(R, P, tile_ctx(P, tile), tile_bits(P, tile), y0 - tile_y0(P, tile) + k + 1,
                      x0 + c, ph2[c].y, eps_phi);
      }
      if (pmin0 <= eps_phi) fbrows |= 1u << k;
      if (pmin1 <= eps_phi) fbrows |= 2u << k;
    }
  } else {
#pragma unroll 1
    for (int k = 0; k < 32; ++k) {
      if (k == 16) {                                        // base row y0+16-R
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
      bool tie = false;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        if (x0 + c >= W) continue;
        if (ph[c] > 0.f) pw[c] |= bitk;
        tie |= fabsf(ph[c]) <= eps_phi;
      }
      if (tie) fbrows |= bitk;
    }
  }
  if (INT) {
#pragma unroll
    for (int c = 0; c < 8; ++c) pw[c] = ~__brev(pw[c]);    // bit k = phi_k >= +0 off ties
  }
#pragma unroll
  for (int c = 0; c < 8; ++c) mw[c] = pw[c];               // phi > 0 unless phi == 0 (tie path)
  // near ties: exact fp64 sign for the tie columns of the flagged rows
  while (fbrows) {
    const int k = __ffs(fbrows) - 1;
    fbrows &= fbrows - 1;
    const uint32_t bitk = 1u << k;
    uint32_t cols = INT ? partition_tie_cols<R>(P, lut_base, r, x0, k, eps_phi) : 0xffu;
    while (cols) {
      const int c = __ffs(cols) - 1;
      cols &= cols - 1;
      if (!INT && x0 + c >= W) break;
      const double e = exact_phi_fast<R>(tile_ctx(P, tile), tile_bits(P, tile),
                                         y0 - tile_y0(P, tile) + k, x0 + c);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        if (q == c) {
          pw[q] = e >= 0.0 ? (pw[q] | bitk) : (pw[q] & ~bitk);
          mw[q] = e > 0.0 ? (mw[q] | bitk) : (mw[q] & ~bitk);
        }
      }
    }
  }
}

struct LaneDelta {
  double a_in, a_out;
  long long n_in, n_out;
  unsigned long long mism;
};

// P / M bit bookkeeping of one lane block (8 words) + the partition deltas.
__device__ __forceinline__ uint4 lds_u4(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}

// sold: shared address of this lane's old P words (and, +1024, old M words)
// staged by cp.async at the unit start (fused pass), 0: read global memory
template <bool PART, bool CKPT, bool MASKONLY>
__device__ __forceinline__ void partition_commit(const FastParams& P, int r, int x0,
                                                 const uint32_t (&pw)[8], const uint32_t (&mw)[8],
                                                 LaneDelta& d, int tile = 0, uint32_t sold = 0u) {
  const int y0 = r * 32;
  const size_t base = (size_t)r * P.g.pitch_w + x0;
  // a row strip's halo word-rows are owned (and counted) by the neighbour
  const bool own = r >= P.own_lo && r < P.own_hi;
  if (MASKONLY) {
    reinterpret_cast<uint4*>(P.mbits + base)[0] = make_uint4(mw[0], mw[1], mw[2], mw[3]);
    reinterpret_cast<uint4*>(P.mbits + base)[1] = make_uint4(mw[4], mw[5], mw[6], mw[7]);
    return;
  }
  if (PART) {
    const uint4 o0 = sold ? lds_u4(sold) : reinterpret_cast<const uint4*>(P.pbits + base)[0];
    const uint4 o1 = sold ? lds_u4(sold + 16) : reinterpret_cast<const uint4*>(P.pbits + base)[1];
    const uint32_t old[8] = {o0.x, o0.y, o0.z, o0.w, o1.x, o1.y, o1.z, o1.w};
    uint32_t any = 0u;
    if (P.chg) {
      // multi-band runs: record the changed pixels; k_band_sums folds every
      // band's sums over them (the fused kernel keeps one band's registers)
      uint32_t cw[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        cw[c] = own ? old[c] ^ pw[c] : 0u;
        any |= cw[c];
      }
      reinterpret_cast<uint4*>(P.chg + base)[0] = make_uint4(cw[0], cw[1], cw[2], cw[3]);
      reinterpret_cast<uint4*>(P.chg + base)[1] = make_uint4(cw[4], cw[5], cw[6], cw[7]);
    } else {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      uint32_t chg = old[c] ^ pw[c];
      any |= chg;
      if (!own) chg = 0u;
      while (chg) {
        const int b = __ffs(chg) - 1;
        chg &= chg - 1;
        const double I = data_exact(tile_ctx(P, tile), y0 - tile_y0(P, tile) + b, x0 + c);
        if ((pw[c] >> b) & 1u) { d.a_in += I; ++d.n_in; }
        else { d.a_out += I; ++d.n_out; }
      }
    }
    }
    if (any) {
      reinterpret_cast<uint4*>(P.pbits + base)[0] = make_uint4(pw[0], pw[1], pw[2], pw[3]);
      reinterpret_cast<uint4*>(P.pbits + base)[1] = make_uint4(pw[4], pw[5], pw[6], pw[7]);
    }
  }
  if (CKPT) {
    const uint4 o0 = sold ? lds_u4(sold + 1024) : reinterpret_cast<const uint4*>(P.mbits + base)[0];
    const uint4 o1 = sold ? lds_u4(sold + 1040) : reinterpret_cast<const uint4*>(P.mbits + base)[1];
    const uint32_t old[8] = {o0.x, o0.y, o0.z, o0.w, o1.x, o1.y, o1.z, o1.w};
#pragma unroll
    for (int c = 0; c < 8; ++c) d.mism += own ? __popc(old[c] ^ mw[c]) : 0;
    reinterpret_cast<uint4*>(P.mbits + base)[0] = make_uint4(mw[0], mw[1], mw[2], mw[3]);
    reinterpret_cast<uint4*>(P.mbits + base)[1] = make_uint4(mw[4], mw[5], mw[6], mw[7]);
  }
}

// Border rows k0 .. k0 + nrows - 1 of the partition lane block (r, x0):
// signs of phi^{n+1} with zero padding (partition_block's arithmetic on a row
// range); pw / mw get bit k for the rows of the range only.
template <int R>
__device__ __forceinline__ void partition_rows_border(const FastParams& P, const float* s_lt,
                                                      const float* s_ls, int r, int x0, int k0,
                                                      int nrows, float eps_phi, uint32_t (&pw)[8],
                                                      uint32_t (&mw)[8]) {
  constexpr int NT = kColsPerThread + 2 * R;
  const int H = P.g.H, W = P.g.W;
  const int y0 = r * 32;
  const int base = y0 + k0 - R;                  // window row 0 (phi row y0+k0 at m0 = 0)
  const int wr = base >> 5, sh = base & 31;
  uint32_t cm[NT], win[NT];
#pragma unroll
  for (int j = 0; j < NT; ++j) {
    const int xc = x0 - R + j;
    cm[j] = (xc >= 0 && xc < W) ? 0xffffffffu : 0u;
    win[j] = __funnelshift_r(word_at<false>(P, wr, xc), word_at<false>(P, wr + 1, xc), sh);
  }
  float ph[8];
  uint32_t fbrows = 0u;
  unsigned long long fbm = 0ull;                 // near-tie pixels (see update_rows_border)
#pragma unroll
  for (int c = 0; c < 8; ++c) { pw[c] = 0u; mw[c] = 0u; }
#pragma unroll 1
  for (int k = k0; k < k0 + nrows; ++k) {
    const int i = y0 + k;
    if (i >= H) break;
    phi_row<R, SRC_SMOOTH, false, NT, 8>(P, win, cm, k - k0, i, s_lt, s_ls, ph);
    const uint32_t bitk = 1u << k;
    uint32_t tie = 0u;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      if (x0 + c >= W) continue;
      if (ph[c] > 0.f) pw[c] |= bitk;
      if (fabsf(ph[c]) <= eps_phi) tie |= 1u << c;
      LSE_CHECK_PHI(R, P, P.ctx, P.bits_in, i, x0 + c, ph[c], eps_phi);
    }
    if (tie) {
      fbrows |= bitk;
      if (k - k0 < 8) fbm |= (unsigned long long)tie << (8 * (k - k0));
    }
  }
#pragma unroll
  for (int c = 0; c < 8; ++c) mw[c] = pw[c];     // phi > 0 unless phi == 0 (tie path)
  while (fbrows) {                               // near ties: exact fp64 signs
    const int k = __ffs(fbrows) - 1;
    fbrows &= fbrows - 1;
    const uint32_t bitk = 1u << k;
    const uint32_t cols = (k - k0 < 8) ? (uint32_t)(fbm >> (8 * (k - k0))) & 0xffu : 0xffu;
#pragma unroll 1
    for (int c = 0; c < 8; ++c) {
      if (x0 + c >= W) break;
      if (!((cols >> c) & 1u)) continue;
      const double e = exact_phi_fast<R>(P.ctx, P.bits_in, y0 + k, x0 + c);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        if (q == c) {
          pw[q] = e >= 0.0 ? (pw[q] | bitk) : (pw[q] & ~bitk);
          mw[q] = e > 0.0 ? (mw[q] | bitk) : (mw[q] & ~bitk);
        }
      }
    }
  }
}

// Border partition unit (all lanes call it): the row quarters of each lane
// group are merged, then the group's first lane commits the whole word.
template <int R, bool PART, bool CKPT, bool MASKONLY>
__device__ __forceinline__ void border_partition_body(const FastParams& P, const float* s_lt,
                                                      const float* s_ls, int unit, float eps_phi,
                                                      LaneDelta& d) {
  const int lane = threadIdx.x & 31;
  int r = 0, x0 = 0;
  const bool act = border_lane(P.gp, unit, lane, P.g.W, r, x0);
  const int items = P.gp.bitems;                 // lane groups per unit = rows per lane
  uint32_t pw[8], mw[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) { pw[c] = 0u; mw[c] = 0u; }
  if (act)
    partition_rows_border<R>(P, s_lt, s_ls, r, x0, (lane / items) * items, items, eps_phi, pw,
                             mw);
  for (int o = items; o < 32; o <<= 1) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      pw[c] |= __shfl_xor_sync(0xffffffffu, pw[c], o);
      mw[c] |= __shfl_xor_sync(0xffffffffu, mw[c], o);
    }
  }
  if (!act || lane >= items) return;
  partition_commit<PART, CKPT, MASKONLY>(P, r, x0, pw, mw, d);
}

template <int R, bool PART, bool CKPT, bool MASKONLY, bool BATCH>
__device__ __noinline__ void border_partition_unit(const FastParams& P, const float* s_lt,
                                                   const float* s_ls, int unit, int tile,
                                                   bool part_t, float eps_phi, LaneDelta& d) {
  if (!BATCH) {
    border_partition_body<R, PART, CKPT, MASKONLY>(P, s_lt, s_ls, unit, eps_phi, d);
    return;
  }
  FastParams Q = P;
  tile_view(Q, tile);
  if (part_t) border_partition_body<R, true, CKPT, false>(Q, s_lt, s_ls, unit, eps_phi, d);
  else border_partition_body<R, false, CKPT, false>(Q, s_lt, s_ls, unit, eps_phi, d);
}

// Units: [border units][interior (word-row, segment of seg_chunks chunks)]
// [interior B1 packs]; each unit's deltas form one partial at part[unit]
// (fixed geometry => deterministic).  A separate finalize then reduces all
// partials in a fixed order.  BATCH: [all tiles' border units][all tiles'
// interior units]; a tile's partials are reduced by its own finalize CTA.
template <int R, bool PART, bool CKPT, bool MASKONLY, bool BATCH>
__global__ void __launch_bounds__(kThreads, kPartitionCtasPerSm) k_partition(FastParams P) {
  constexpr int NT = kColsPerThread + 2 * R;
  constexpr int NPAT = 1 << (2 * R + 1);
  __shared__ float s_lt[NPAT];
  __shared__ float s_ls[NPAT];
  LSE_TRACE_ENTRY
  __shared__ FastParams s_P;                     // see k_update
  const SharedLuts luts{s_lt, s_ls, (uint32_t)__cvta_generic_to_shared(g_pair_lut)};
  load_luts<R>(P, luts);                         // static data: before the dependency wait
  if (threadIdx.x == 0) s_P = P;
  __syncthreads();
  pdl_wait();
  pdl_launch_dependents();
  Scalars* sc = P.scal;
  if (!BATCH && !MASKONLY && stop_flag(sc)) return;
  const float eps_phi = sc->eps_phi;
  const int lane = threadIdx.x & 31;
  const int nseg = P.nseg;
  const int nb = border_units(P.gp);
  const int nsu = (P.gp.r_hi - P.gp.r_lo) * nseg;
  const int ni = nsu + (P.gp.nB1 + 31) / 32;
  const int T = BATCH ? P.ntiles : 1;
  const int nunits = T * (nb + ni);
  LSE_TRACE_DECL
  for (;;) {
    const int unit = grab_unit(P, lane);
    LSE_TRACE_MARK(unit < nunits ? unit : -1);
    if (unit >= nunits) break;
    int tile = 0, lu = unit;
    bool part_t = PART;
    if (BATCH) {
      if (unit < T * nb) {
        tile = unit / nb;
        lu = unit - tile * nb;
      } else {
        const int iu = unit - T * nb;
        tile = iu / ni;
        lu = nb + (iu - tile * ni);
      }
      const Scalars* st = P.scal + tile;
      part_t = PART && st->model != EDGE;
      // converged tiles, and edge tiles off the checkpoints, have nothing to do
      if (stop_flag(st) || (!part_t && !CKPT)) continue;
    }
    LaneDelta d{0.0, 0.0, 0, 0, 0ull};
    if (lu < nb) {
      border_partition_unit<R, PART, CKPT, MASKONLY, BATCH>(s_P, s_lt, s_ls, lu, tile, part_t,
                                                           eps_phi, d);
    } else {
      const int iu = lu - nb;
      int r = 0, c0 = 0, c1 = 1, xb = 0;
      bool active = true, chunked = false;
      if (iu < nsu) {
        chunked = true;
        r = P.gp.r_lo + iu / nseg;
        c0 = (iu % nseg) * P.seg_chunks;
        c1 = min(c0 + P.seg_chunks, P.gp.nci);
        xb = P.gp.xoff + kColsPerThread * lane;
      } else {
        active = b1_lane(P.gp, iu - nsu, lane, r, xb);
      }
      if (BATCH) r += tile * P.tile_hr;
      for (int ch = c0; ch < c1; ++ch) {
        const int x0 = chunked ? xb + ch * kChunk : xb;
        uint32_t pw[8], mw[8], prev[NT], cur[NT];
        uint32_t a = ~0u, o = 0u;
        if (active) {
#pragma unroll
          for (int j = 0; j < NT; ++j) {
            const int xc = x0 - R + j;
            prev[j] = word_at<true>(P, r - 1, xc);
            cur[j] = word_at<true>(P, r, xc);
            if (P.skip_uniform) {
              const uint32_t nx = word_at<true>(P, r + 1, xc);
              a &= prev[j] & cur[j] & nx;
              o |= prev[j] | cur[j] | nx;
            }
          }
        }
        if (P.skip_uniform && __all_sync(0xffffffffu, !active || a == ~0u || o == 0u)) {
          if (!active) continue;
#pragma unroll
          for (int c = 0; c < 8; ++c) pw[c] = mw[c] = cur[R + c];   // sign(phi) = b
        } else if (!active) {
          continue;
        } else {
          partition_block<R, true>(P, s_lt, s_ls, luts.lt2, r,
                                   x0, eps_phi, prev, cur, pw, mw, tile);
        }
        if (!BATCH || part_t == PART) partition_commit<PART, CKPT, MASKONLY>(P, r, x0, pw, mw, d, tile);
        else partition_commit<false, CKPT, false>(P, r, x0, pw, mw, d, tile);
      }
    }
    if (MASKONLY) continue;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      d.a_in += __shfl_xor_sync(0xffffffffu, d.a_in, o);
      d.a_out += __shfl_xor_sync(0xffffffffu, d.a_out, o);
      d.n_in += __shfl_xor_sync(0xffffffffu, d.n_in, o);
      d.n_out += __shfl_xor_sync(0xffffffffu, d.n_out, o);
      d.mism += __shfl_xor_sync(0xffffffffu, d.mism, o);
    }
    if (lane == 0) {
      TilePartial t{};
      t.a_hi = d.a_in;
      t.b_hi = d.a_out;
      t.n_a = d.n_in;
      t.n_b = d.n_out;
      t.mism = d.mism;
      P.part[unit] = t;
    }
  }
}


// ------------------------------------------- speculative fused iteration
// One pass per iteration instead of update + partition: k_update_fused reads
// b^n, rebuilds phi^n once and from it derives both
//   * the partition of iteration n (P bits, the c+/c- deltas, the checkpoint
//     mask) -- exactly what k_partition computes from the same b^n, and
//   * b^{n+1} with the coefficients of iteration n-1 as the prediction of
//     iteration n's (the partition that defines them is being computed in
//     the same pass).
// The finalize then derives the true coefficients and checks the prediction
// (spec_check): if it held, only the pixels in the flag band were undecided
// and k_spec_fix decides them exactly; otherwise k_spec_fix redoes the whole
// update with the true coefficients.  Either way b^{n+1} is the state the
// two-pass iteration produces, bit for bit.

template <int R, bool CKPT>
__device__ __noinline__ void border_fused_unit(const FastParams& P, const float* s_lt,
                                               const float* s_ls, int unit, float A, float B,
                                               float e0, float delta, LaneDelta& d) {
  constexpr int CPL = kUpdCols;
  const int lane = threadIdx.x & 31;
  int r = 0, x0 = 0;
  const bool act = border_lane(P.gu, unit, lane, P.g.W, r, x0);
  const int items = P.gu.bitems;
  uint32_t ow[CPL], pw[CPL], mw[CPL];
#pragma unroll
  for (int c = 0; c < CPL; ++c) { ow[c] = 0u; pw[c] = 0u; mw[c] = 0u; }
  if (act) {
    const int k0 = (lane / items) * items;
    update_rows_border<R, REGION, SRC_SMOOTH, CPL, true>(P, s_lt, s_ls, r, x0, k0, items, A, B,
                                                         e0, ow, delta);
    partition_rows_border<R>(P, s_lt, s_ls, r, x0, k0, items, P.scal->eps_phi, pw, mw);
  }
  for (int o = items; o < 32; o <<= 1) {
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      ow[c] |= __shfl_xor_sync(0xffffffffu, ow[c], o);
      pw[c] |= __shfl_xor_sync(0xffffffffu, pw[c], o);
      mw[c] |= __shfl_xor_sync(0xffffffffu, mw[c], o);
    }
  }
  if (!act || lane >= items) return;
  uint32_t* dst = P.bits_out + (size_t)r * P.g.pitch_w + x0;
#pragma unroll
  for (int q = 0; q < CPL / 4; ++q)
    reinterpret_cast<uint4*>(dst)[q] = make_uint4(ow[4 * q], ow[4 * q + 1], ow[4 * q + 2], ow[4 * q + 3]);
  partition_commit<true, CKPT, false>(P, r, x0, pw, mw, d);
}

// Single runs, region / zhang, smoothed state, unsplit units: the update's
// work geometry (gu) for both halves, one partial per unit (part[unit]).
template <int R>
constexpr int fused_smem_bytes() {
  // per warp: data ring, window of rows 16..31, old P and M words (2 x 1 KB)
  return (kThreads / 32) * ((kRing2 * 32 * kUpdCols + (kUpdCols + 2 * (R + 1)) * 32) * 4 + 2048) +
         (LSE_TMA_RING ? (kThreads / 32) * 32 : 0);             // (A/B builds: 4 mbarriers per warp)
}

// BATCH: every unit of every tile ([all tiles' border][all tiles' interior],
// the batched update's order), each with its tile's coefficients and band;
// converged tiles keep their state; edge tiles run with their exact
// coefficients (A = 1, B = 0, delta = 0: nothing to predict) and produce
// partition words only for the checkpoint masks.
template <int R, bool CKPT, bool BATCH>
__global__ void __launch_bounds__(kThreads, kFusedCtasPerSm) k_update_fused(FastParams P) {
  constexpr int CPL = kUpdCols;
  constexpr int NT = CPL + 2 * (R + 1);
  constexpr int NPAT = 1 << (2 * R + 1);
  // (the border code's zero-padded rows read only the weight-sum table)
  __shared__ float s_ls[NPAT];
  // dynamic shared memory (fused_smem_bytes): the data rings, then per warp
  // the window of rows 16..31 of its unit, built at the unit start (word j of
  // lane l at [j][l]) so the mid-unit switch reads shared memory
  extern __shared__ __align__(16) float s_dyn[];
  LSE_TRACE_ENTRY
  float* s_ring = s_dyn;
  auto s_win = reinterpret_cast<uint32_t (*)[NT][32]>(s_dyn + (kThreads / 32) * kRing2 * 32 * CPL);
  // per warp: the old P / M words of the unit's block, staged at the unit start
  const uint32_t s_old = (uint32_t)__cvta_generic_to_shared(s_dyn) +
                         (kThreads / 32) * (kRing2 * 32 * CPL + NT * 32) * 4 +
                         (threadIdx.x >> 5) * 2048 + (threadIdx.x & 31) * 32;
  __shared__ FastParams s_P;                     // see k_update
  const SharedLuts luts{nullptr, s_ls, (uint32_t)__cvta_generic_to_shared(g_pair_lut)};
  // (A/B builds) the warp's mbarriers, after everything else in dynamic shared memory
  const uint32_t s_bars = LSE_TMA_RING
      ? (uint32_t)__cvta_generic_to_shared(s_dyn) +
            (kThreads / 32) * ((kRing2 * 32 * CPL + NT * 32) * 4 + 2048) + (threadIdx.x >> 5) * 32
      : 0u;
  if (LSE_TMA_RING && (threadIdx.x & 31) == 0) {
#pragma unroll
    for (int q = 0; q < 4; ++q) mbar_init(s_bars + 8 * q, 1u);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  {
    for (int q = threadIdx.x; q < NPAT; q += blockDim.x) s_ls[q] = __ldg(&P.lut_s[q]);
    for (int q = threadIdx.x; q < 2 * NPAT; q += blockDim.x)
      g_pair_lut[q] = make_float2(__ldg(&P.lut_t[q & (NPAT - 1)]), __ldg(&P.lut_t[q >> 1]));
  }
  const float* s_lt = nullptr;
  if (threadIdx.x == 0) s_P = P;
  __syncthreads();
  pdl_wait();
  pdl_launch_dependents();
  const Scalars* sc = P.scal;
  if (!BATCH && stop_flag(sc)) return;
  if (BATCH && blockIdx.x == 0 && threadIdx.x == 0) P.scal->redo_any = 0;   // (this iteration's)
  float A = sc->A, B = sc->B, e0 = sc->spec_e0, delta = sc->spec_delta;
  float eps_t = sc->eps_u;
  const int lane = threadIdx.x & 31;
  const int nb = border_units(P.gu);
  const int nch = chunk_units(P.gu);
  const int ni = interior_units(P.gu);
  const int T = BATCH ? P.ntiles : 1;
  const int nunits = T * (nb + ni);
  float* ring = s_ring + (threadIdx.x >> 5) * kRing2 * 32 * CPL;
  uint32_t (&win_b)[NT][32] = s_win[threadIdx.x >> 5];
  // (Also loading the next unit's window before this one's commit measured
  // slower: 775 -> 764 Gpix-it/s on C5, the live window words cost more than
  // the latency they hid.)
  // The next unit is grabbed when this one starts and read at its end (the
  // atomic's round trip overlaps the unit; same grab count: one failing grab
  // per warp).
  int unit = grab_unit(P, lane);
  LSE_TRACE_DECL
  for (;;) {
    LSE_TRACE_MARK(unit < nunits ? unit : -1);
    if (unit >= nunits) break;
    unsigned long long g_next = 0;
    if (lane == 0) g_next = atomicAdd(P.work, 1ull) - P.work_base;
    LaneDelta d{0.0, 0.0, 0, 0, 0ull};
    int tile = 0, lu = unit;
    bool stopped = false, part_t = true;
    if (BATCH) {
      if (unit < T * nb) {
        tile = unit / nb;
        lu = unit - tile * nb;
      } else {
        const int iu = unit - T * nb;
        tile = iu / ni;
        lu = nb + (iu - tile * ni);
      }
      const Scalars* st = P.scal + tile;
      stopped = stop_flag(st) != 0;
      A = st->A;
      B = st->B;
      e0 = st->spec_e0;
      delta = st->spec_delta;
      eps_t = st->eps_u;
      part_t = st->model != EDGE || CKPT;        // edge tiles: checkpoint masks only
    }
    if (lu < nb) {
      if (!BATCH) {
        border_fused_unit<R, CKPT>(s_P, s_lt, s_ls, lu, A, B, e0, delta, d);
      } else {
        FastParams Q = s_P;
        tile_view(Q, tile);
        if (stopped) border_update_body<R, REGION, SRC_SMOOTH>(Q, s_lt, s_ls, lu, A, B, e0, true);
        else border_fused_unit<R, CKPT>(Q, s_lt, s_ls, lu, A, B, e0, delta, d);
      }
    } else {
      const int iu = lu - nb;
      int r = 0, x0 = 0;
      bool act = true;
      if (iu < nch) {
        r = P.gu.r_lo + iu / P.gu.nci;
        x0 = P.gu.xoff + (iu % P.gu.nci) * kUpdChunk + CPL * lane;
      } else {
        act = b1_lane(P.gu, iu - nch, lane, r, x0);
      }
      if (BATCH) r += tile * P.tile_hr;           // row of the tile in the stacked arrays
      uint32_t prev[NT], cur[NT];
      uint32_t a = ~0u, o = 0u;
      if (act) {
        // old P (and M) words of the block: in flight until the commit
        const size_t wb = (size_t)r * P.g.pitch_w + x0;
        cp_async16(s_old, P.pbits + wb);
        cp_async16(s_old + 16, P.pbits + wb + 4);
        if (CKPT) {
          cp_async16(s_old + 1024, P.mbits + wb);
          cp_async16(s_old + 1040, P.mbits + wb + 4);
        }
      }
      cp_async_commit();
      if (act) {
        const uint32_t* wp = P.bits_in + (size_t)(r - 1) * P.g.pitch_w + (x0 - (R + 1));
#pragma unroll
        for (int j = 0; j < NT; ++j) {
          prev[j] = __ldg(wp + j);
          cur[j] = __ldg(wp + P.g.pitch_w + j);
          const uint32_t nx = __ldg(wp + 2 * (size_t)P.g.pitch_w + j);
          if (P.skip_uniform) {
            a &= prev[j] & cur[j] & nx;
            o |= prev[j] | cur[j] | nx;
          }
          win_b[j][lane] = __funnelshift_r(cur[j], nx, 16 - R) << 3;
        }
      }
      uint32_t pw[CPL], mw[CPL];
      if (stopped || (P.skip_uniform && __all_sync(0xffffffffu, !act || a == ~0u || o == 0u))) {
        // uniform window: phi has the sign of b everywhere, b^{n+1} = b^n
        // (a converged tile of a batch keeps its state the same way)
        if (act) {
          uint32_t* dst = P.bits_out + (size_t)r * P.g.pitch_w + x0;
#pragma unroll
          for (int q = 0; q < CPL / 4; ++q)
            reinterpret_cast<uint4*>(dst)[q] = make_uint4(cur[R + 1 + 4 * q], cur[R + 2 + 4 * q],
                                                          cur[R + 3 + 4 * q], cur[R + 4 + 4 * q]);
#pragma unroll
          for (int c = 0; c < CPL; ++c) pw[c] = mw[c] = cur[R + 1 + c];
          cp_async_wait<0>();
          if (!stopped) {
            if (part_t) partition_commit<true, CKPT, false>(P, r, x0, pw, mw, d, tile, s_old);
            else partition_commit<false, CKPT, false>(P, r, x0, pw, mw, d, tile, s_old);
          }
        }
      } else if (act) {
        // (its final cp.async wait covers the old words too)
        update_block_int2<R, REGION, CPL, SRC_SMOOTH, true>(P, luts.lt2, ring, r, x0, A, B, e0,
                                                            prev, cur, tile, delta, pw, mw, s_P,
                                                            &win_b[0][0], eps_t,
                                                            iu < nch ? s_bars : 0u);
        if (!BATCH || part_t) partition_commit<true, CKPT, false>(P, r, x0, pw, mw, d, tile, s_old);
        else partition_commit<false, CKPT, false>(P, r, x0, pw, mw, d, tile, s_old);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      d.a_in += __shfl_xor_sync(0xffffffffu, d.a_in, o);
      d.a_out += __shfl_xor_sync(0xffffffffu, d.a_out, o);
      d.n_in += __shfl_xor_sync(0xffffffffu, d.n_in, o);
      d.n_out += __shfl_xor_sync(0xffffffffu, d.n_out, o);
      d.mism += __shfl_xor_sync(0xffffffffu, d.mism, o);
    }
    if (lane == 0) {
      TilePartial t{};
      t.a_hi = d.a_in;
      t.b_hi = d.a_out;
      t.n_a = d.n_in;
      t.n_b = d.n_out;
      t.mism = d.mism;
      P.part[unit] = t;
    }
    g_next = (unsigned long long)__shfl_sync(0xffffffffu, (long long)g_next, 0);
    unit = g_next > 0x7fffffffull ? 0x7fffffff : (int)g_next;
  }
}

// After the finalize of a speculative update, two launches (both no-ops once
// the run has stopped):
//   k_spec_fix  -- small grid: the sticky degenerate flag, the next update's
//                  fix-list counter, and -- unless the update is to be redone
//                  -- the fix list's pixels decided exactly (u in fp64 in the
//                  reference's operation order, exact_u_fast) and patched;
//   k_spec_redo -- the update grid: returns at once unless scal->redo, else
//                  redoes the whole update with the true coefficients (its own
//                  work counter scal->work2, reset by the finalize).
template <int R, bool BATCH>
__global__ void __launch_bounds__(256) k_spec_fix(const FastParams P) {
  pdl_wait();
  pdl_launch_dependents();
  Scalars* sc = P.scal;                          // (tile 0 of a batch: the list's counters)
  if (!BATCH && stop_flag(sc)) return;
  const bool skip = !BATCH && (__ldcg(&sc->redo) != 0 || __ldcg(&sc->fix_needed) == 0);
  const unsigned n = min(__ldcg(&P.fix_cnt[P.fix_par]), P.fix_cap);
  if (blockIdx.x == 0) {
    for (int t = threadIdx.x; t < (BATCH ? P.ntiles : 1); t += blockDim.x) {
      Scalars* st = sc + t;                      // sticky degenerate (engine.py:239-240)
      if (st->zero_vel && st->model != EDGE && !st->stop) st->degenerate = 1;
    }
    if (threadIdx.x == 0) {
      P.fix_cnt[P.fix_par ^ 1] = 0u;             // the next speculative update's list
      if (!BATCH && !skip) sc->fallbacks += n;   // (counted once: no contended atomics)
    }
  }
  if (skip) return;
  const int tile_rows = P.tile_hr * 32;
  const unsigned stride = gridDim.x * blockDim.x;
  for (unsigned q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += stride) {
    const int2 e = __ldcg(&P.fix[q]);
    int t = 0, i = e.y;
    if (BATCH) {
      t = e.y / tile_rows;
      i = e.y - t * tile_rows;
      const Scalars* st = sc + t;
      if (__ldcg(&st->stop) || __ldcg(&st->redo) || !__ldcg(&st->fix_needed)) continue;
    }
    const bool pos = exact_u_fast<R, SRC_SMOOTH>(P.ctx + t, P.bits_in + (size_t)t * P.tile_words, i,
                                                 e.x, false) > 0.0;
    uint32_t* w = P.bits_out + (size_t)(e.y >> 5) * P.g.pitch_w + e.x;
    const uint32_t bit = 1u << (e.y & 31);
    if (pos) atomicOr(w, bit);
    else atomicAnd(w, ~bit);
  }
}

// the redo pass proper: a noinline body over the CTA's shared copy of the
// parameters, so the (almost always) early-returning kernel never copies its
// parameter block to local memory
template <int R, bool BATCH>
__device__ __noinline__ void spec_redo_body(const FastParams& P, float* s_lt, float* s_ls,
                                            float* s_ring) {
  const SharedLuts luts{s_lt, s_ls, (uint32_t)__cvta_generic_to_shared(g_pair_lut)};
  load_luts<R>(P, luts);
  __syncthreads();
  update_units<R, REGION, SRC_SMOOTH, BATCH, 1>(P, P, luts, s_lt, s_ls, s_ring);
}

// BATCH: the tiles whose scal->redo is set (a failed prediction, or a tile
// that converged in this iteration: its state goes back to b^{iter})
template <int R, bool BATCH>
__global__ void __launch_bounds__(kThreads, kUpdateCtasPerSm) k_spec_redo(const FastParams P) {
  constexpr int CPL = kUpdCols;
  constexpr int NPAT = 1 << (2 * R + 1);
  __shared__ float s_lt[NPAT];
  __shared__ float s_ls[NPAT];
  __shared__ __align__(16) float s_ring[(kThreads / 32) * kRing2 * 32 * CPL];
  __shared__ FastParams s_P;
  pdl_wait();
  pdl_launch_dependents();
  if (BATCH ? !__ldcg(&P.scal->redo_any) : (stop_flag(P.scal) || !__ldcg(&P.scal->redo))) return;
  if (threadIdx.x == 0) {
    s_P = P;
    s_P.redo_only = BATCH ? 1 : 0;
  }
  __syncthreads();
  spec_redo_body<R, BATCH>(s_P, s_lt, s_ls, s_ring);
}

}  // namespace lse
