// lse_device.cuh -- device-side data layout and exact-arithmetic helpers.
//
// HBM layout (one run):
//   * state b^n : bit-packed "vertical words": word (r, x) holds the signs of
//     rows 32r..32r+31 of column x (bit k <-> row 32r+k, 1 <-> phi > 0).
//     With reinit_period = reg_period = 1 the carried field is exactly
//     phi^n = G_sigma2 * b^n (engine.py:160-169), so 1 bit/pixel is the whole
//     state and phi is re-derived on chip each iteration.
//   * P : partition bits {phi >= 0} (grid.py:112), M : last checkpoint mask
//     {phi > 0} (engine.py:229), same layout.
//   * data : fp32 copy of the image (region) or edge indicator g (edge),
//     row pitch a multiple of 8 floats, plus exact fp64 values when fp32 is
//     not exact (read only by the rare exact re-evaluations).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace lse {

constexpr int kThreads = 128;            // threads per CTA of the tiled kernels
constexpr int kColsPerThread = 8;        // columns per thread (one 32-row word each)
constexpr int kSpanMax = kColsPerThread * kThreads + 16;

// ZHANG and VECTOR run the REGION kernels (their data term is an affine image
// of one fp32 data plane); VECTOR = region data term summed over K bands
enum Model : int { EDGE = 0, REGION = 1, ZHANG = 2, VECTOR = 3, CHAN_VESE = 4 };
constexpr int kMaxBands = 4;
enum Src : int { SRC_SMOOTH = 0, SRC_SCALED = 1, SRC_FIELD = 2 };

// A-priori error bounds of the fp32 evaluation.  phi32 is a
// (2R+1 <= 9)-term FMA chain over table values: table rounding <= 2^-23 (the
// zero-padded form 2 S - L; 2^-25 for the exact-rounded interior values),
// weight rounding <= 2^-24, nine FMA roundings <= 2^-25 each (|partial sums|
// <= 1): |phi32 - phi| <= 5.1e-7 < 0.54 * 2^-20.  h = 2|grad phi| from four such
// values (one-sided differences double them): <= 5.66 * 5.1e-7 + roundings
// (differences, squares, sqrt.approx at 2^-23 relative) < 2^-18 + 2^-21.  The
// guards are kGuard times these bounds.
constexpr double kErrPhi = 0x1p-20;
constexpr double kErrGrad = 0x1p-18;
constexpr double kGuard = 4.0;

// Per-run scalars shared by the kernels of one run (device resident).
struct __align__(16) Scalars {
  double sp_hi, sp_lo, sn_hi, sn_lo;  // running sums of I over {phi>=0} / {phi<0} (double-double)
  long long n_pos, n_total;
  double c_pos, c_neg, dc, peak;      // region coefficients of the next update (models.py:109-118)
  double mid, nu;                     // zhang: m = (c+ + c-)/2, speed constant (models.py:152-162)
  // vector (multi-band) region model: per-band running sums and means
  double bsp_hi[kMaxBands], bsp_lo[kMaxBands], bsn_hi[kMaxBands], bsn_lo[kMaxBands];
  double bcp[kMaxBands], bcm[kMaxBands];
  unsigned long long peak_bits;       // max |D| of the current pass (ordered double bits)
  int nbands, pad2_;
  double img_min, img_max, img_absmax;
  float A, B, eps_u, eps_phi;         // fp32 fast path: D/peak ~= A*I + B ; near-tie guards
  int zero_vel;                       // next update has v == 0 (degenerate, models.py:111-118)
  int degenerate;                     // sticky (engine.py:239-240)
  int stop;                           // set at convergence: later launches are no-ops
  int converged;
  long long converged_iter;
  long long n_ckpt, equal_run;        // checkpoint history (engine.py:228-236)
  unsigned int ticket;                // last-CTA-done counter
  int nonfinite;                      // generic path finiteness flag (engine.py:159, 172)
  unsigned long long fallbacks;       // fp64 near-tie re-evaluations
  long long conv_window;
  double dt;
  int model;
  // speculative fused iteration (k_update<..., FUSED>): the update of
  // iteration n runs with the coefficients of iteration n-1 while the same
  // pass computes the partition that defines iteration n's own; every pixel
  // with |u| - spec_delta * h <= spec_e0 goes to the fix list and is decided
  // exactly once the true coefficients are known (k_spec_fix), or the whole
  // update is redone when the coefficients moved more than spec_delta
  int redo;                           // the last speculative update must be redone
  int fix_needed;                     // its coefficients moved: the fix list decides the band
  int redo_any;                       // batches (tile 0's copy): some tile's update is redone
  float spec_delta, spec_e0;          // flag band of the next speculative update (delta < 0: none)
  unsigned int fix_n[2];              // fix-list entries of the speculative update (by parity)
  unsigned int fix_cap;               // fix-list capacity
  unsigned long long work2;           // work counter of the redo pass
  unsigned long long spec_redos, spec_fixes;   // statistics
  // multi-band runs: the data plane, peak and coefficients of the last peak
  // pass are a function of the band means alone; when a partition changed
  // no pixel the means are bit-identical and the peak pass is not repeated
  int band_valid;                     // the last peak pass completed (plane + coefficients)
  int band_same;                      // this pass: the means did not move (peak pass skipped)
  int band_reuse;                     // reuse enabled (LSE_BAND_REUSE, default 1)
  int band_any;                       // k_band_sums: some block of this pass saw a changed pixel
  unsigned long long band_reused;     // statistics: peak passes skipped
};

// Per-tile partial (fixed tile geometry => deterministic, GPU-count independent
// reduction order).  DELTA mode: a = I entering P, b = I leaving P.
// ABSOLUTE mode: a = sum over P, b = sum over not-P.
struct __align__(16) TilePartial {
  double a_hi, a_lo, b_hi, b_lo;
  long long n_a, n_b;
  unsigned long long mism;
  long long pad_;
};

struct RunGeom {
  int H, W, HR, pitch_w;    // image rows/cols, word rows, words per word-row
  long long data_pitch;     // floats/doubles per image row in data buffers
  int ncb, ntiles;          // column blocks (of 8*kThreads columns), tiles
};

// ------------------------------------------------- programmatic dependent launch
// The per-iteration kernels are launched with programmatic stream
// serialization: a kernel may start (its static prologue: LUT loads) while its
// predecessor drains, and waits here before touching the predecessor's
// results.  Without the launch attribute both are no-ops.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// A run's stop flag.  It is only written by earlier kernels of the stream
// (finalize passes), which are complete and visible once pdl_wait() returns,
// so an L2 (.cg) load suffices -- a volatile access compiles to a
// system-scope strong load on the critical path of every short kernel.
template <typename S>
__device__ __forceinline__ int stop_flag(const S* sc) { return __ldcg(&sc->stop); }
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// ---------------------------------------------------------------- exact ops
// numpy / scipy evaluate every float64 operation separately with round-to-
// nearest (no FMA on x86-64 baseline builds); these wrappers stop nvcc from
// contracting them so the device reproduces the reference bit-for-bit.
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }

// glibc >= 2.35 hypot, non-FMA branch (Borges, "An improved algorithm for
// hypot(a,b)") -- the libm routine np.hypot calls on x86-64 (kernels.py:95).
__device__ __forceinline__ double hypot_kernel(double ax, double ay) {
  double h = __dsqrt_rn(dadd(dmul(ax, ax), dmul(ay, ay)));
  double t1, t2;
  if (h <= dmul(2.0, ay)) {
    double delta = dsub(h, ay);
    t1 = dmul(ax, dsub(dmul(2.0, delta), ax));
    t2 = dmul(dsub(delta, dmul(2.0, dsub(ax, ay))), delta);
  } else {
    double delta = dsub(h, ax);
    t1 = dmul(dmul(2.0, delta), dsub(ax, dmul(2.0, ay)));
    t2 = dadd(dmul(dsub(dmul(4.0, delta), ay), ay), dmul(delta, delta));
  }
  return dsub(h, ddiv(dadd(t1, t2), dmul(2.0, h)));
}

__device__ inline double np_hypot(double x, double y) {
  if (!isfinite(x) || !isfinite(y)) {
    if (isinf(x) || isinf(y)) return __longlong_as_double(0x7ff0000000000000LL);
    return x + y;
  }
  x = fabs(x);
  y = fabs(y);
  double ax = x < y ? y : x, ay = x < y ? x : y;
  const double SCALE = 0x1p-600, LARGE = 0x1p+511, TINY = 0x1p-511, EPS = 0x1p-54;
  if (ax > LARGE) {
    if (ay <= dmul(ax, EPS)) return dadd(ax, ay);
    return ddiv(hypot_kernel(dmul(ax, SCALE), dmul(ay, SCALE)), SCALE);
  }
  if (ay < TINY) {
    if (ax >= ddiv(ay, EPS)) return dadd(ax, ay);
    return dmul(hypot_kernel(ddiv(ax, SCALE), ddiv(ay, SCALE)), SCALE);
  }
  if (ay <= dmul(ax, EPS)) return dadd(ax, ay);
  return hypot_kernel(ax, ay);
}

// ------------------------------------------------------- double-double sums
__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e) {
  s = dadd(a, b);
  double bb = dsub(s, a);
  e = dadd(dsub(a, dsub(s, bb)), dsub(b, bb));
}
__device__ __forceinline__ void dd_add(double& hi, double& lo, double x) {
  double s, e;
  two_sum(hi, x, s, e);
  e = dadd(e, lo);
  hi = dadd(s, e);
  lo = dsub(e, dsub(hi, s));
}
__device__ __forceinline__ void dd_add_dd(double& hi, double& lo, double xh, double xl) {
  double s, e;
  two_sum(hi, xh, s, e);
  e = dadd(e, dadd(lo, xl));
  hi = dadd(s, e);
  lo = dsub(e, dsub(hi, s));
}
// (hi + lo) / n, nearly correctly rounded
__device__ __forceinline__ double dd_div(double hi, double lo, double n) {
  double q = ddiv(hi, n);
  double r = dadd(__fma_rn(-q, n, hi), lo);
  return dadd(q, ddiv(r, n));
}

// ------------------------------------------------------------- bit access
__device__ __forceinline__ int get_bit(const uint32_t* bits, int pitch_w, int i, int x) {
  return (int)((__ldg(&bits[(size_t)(i >> 5) * pitch_w + x]) >> (i & 31)) & 1u);
}

// Exact vertical scipy pass (kernels.py:73-74) over the binary field b
// (b = +1/-1 inside, 0 outside the image) at (i, x): out = b0*w0, then for
// d = R..1: out += (b[i-d] + b[i+d]) * w[d].
__device__ inline double exact_t(const uint32_t* bits, int pitch_w, int H, int R,
                                 const double* w64, int i, int x) {
  auto b = [&](int ii) -> double {
    if (ii < 0 || ii >= H) return 0.0;
    return get_bit(bits, pitch_w, ii, x) ? 1.0 : -1.0;
  };
  double acc = dmul(b(i), w64[0]);
  for (int d = R; d >= 1; --d) acc = dadd(acc, dmul(dadd(b(i - d), b(i + d)), w64[d]));
  return acc;
}

// Exact phi = G * b at (i, x): horizontal scipy pass (kernels.py:75-76) over
// the exact vertical pass; zero padding outside the columns.
__device__ inline double exact_phi_smooth(const uint32_t* bits, int pitch_w, int H, int W, int R,
                                          const double* w64, int i, int x) {
  auto tv = [&](int xc) -> double {
    if (xc < 0 || xc >= W) return 0.0;
    return exact_t(bits, pitch_w, H, R, w64, i, xc);
  };
  double acc = dmul(tv(x), w64[0]);
  for (int d = R; d >= 1; --d) acc = dadd(acc, dmul(dadd(tv(x - d), tv(x + d)), w64[d]));
  return acc;
}

}  // namespace lse
