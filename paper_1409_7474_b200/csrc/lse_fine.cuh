// lse_fine.cuh -- per-pixel update / partition kernels for small images.
//
// The tiled kernels (lse_fast.cuh) give each lane a block of 8 columns x
// 32 (or 32/NS) rows; on a small image there are only a few such blocks per
// SM, so an iteration costs the serial latency of one block rather than its
// throughput.  Here every thread owns one pixel: a warp is one state word
// (lane k = row 32r + k of column x), a CTA eight adjacent columns of one
// word-row.  The state word of the next iteration is one __ballot_sync.
//
// The arithmetic is the tiled kernels' arithmetic pixel by pixel: the same
// vertical LUT values (exact-rounded t where a pixel's window lies inside the
// image, the zero-padding weight-sum form otherwise -- chosen per pixel here,
// per lane block there), the same left-to-right horizontal FMA order, the
// same gradient / velocity / u expressions and the same near-tie guards.
// Every decision therefore equals the reference's fp64 decision, as on the
// tiled path: outside the guard band the fp32 sign is provably right, inside
// it the fp64 restatement decides.  The partition partials are one per CTA
// of kFineCols state words (CTAP: images of at most kFineCtaParts CTAs, the
// words' sums added in plain fp64 in column order) or one per state word
// (larger images), so only the grouping of the c+/c- sums differs from the
// tiled path.
#pragma once

namespace lse {

constexpr int kFineCols = 8;                     // columns (warps) per CTA

// The CTA's state words: word-rows r-1, r, r+1 (r = blockIdx.y) of columns
// xb .. xb+SW-1, 0 outside the image; the LUT stores made before are published
// by the same barrier.
template <int SW>
__device__ __forceinline__ void fine_stage_words(const FastParams& P, int xb, uint32_t (&s_w)[3][SW]) {
  const int r = blockIdx.y;
  for (int q = threadIdx.x; q < 3 * SW; q += blockDim.x) {
    const int row = q / SW, col = q - row * SW;
    s_w[row][col] = word_at<false>(P, r - 1 + row, xb + col);
  }
  __syncthreads();
}

template <int R>
__device__ __forceinline__ void fine_load_luts(const FastParams& P, float* s_lt, float* s_ls) {
  constexpr int NPAT = 1 << (2 * R + 1);
  for (int q = threadIdx.x; q < NPAT; q += blockDim.x) {
    s_lt[q] = __ldg(&P.lut_t[q]);
    s_ls[q] = __ldg(&P.lut_s[q]);
  }
}

// t values (vertical pass) of window row offset m for window columns j,
// exact-rounded LUT inside the image, zero padding via the weight-sum form
template <int R, int NC>
__device__ __forceinline__ void fine_trow(const uint32_t (&win)[NC], const uint32_t (&cm)[NC],
                                          int m, bool in, uint32_t vr, float Lv,
                                          const float* s_lt, const float* s_ls, float (&t)[NC]) {
  constexpr uint32_t PM = (1u << (2 * R + 1)) - 1u;
  if (in) {                                      // one branch per row, not per column
#pragma unroll
    for (int j = 0; j < NC; ++j) t[j] = s_lt[(win[j] >> m) & PM];
  } else {
#pragma unroll
    for (int j = 0; j < NC; ++j)
      t[j] = fmaf(2.f, s_ls[(win[j] >> m) & PM & vr & cm[j]], cm[j] ? -Lv : 0.f);
  }
}
// horizontal pass centred on window column j0 + R, left to right
template <int R, int NC>
__device__ __forceinline__ float fine_hsum(const FastParams& P, const float (&t)[NC], int j0) {
  float out = 0.f;
#pragma unroll
  for (int d = -R; d <= R; ++d) {
    const float wd = P.w32[d < 0 ? -d : d];
    out = (d == -R) ? wd * t[j0 + R + d] : fmaf(wd, t[j0 + R + d], out);
  }
  return out;
}

// b^n -> b^{n+1} (engine.py:155-169 for one pixel per thread).  Grid:
// (ceil(W / kFineCols), HR), block kFineCols warps.  Each lane computes phi
// of its own row at columns x-1, x, x+1; phi at rows i-1 / i+1 comes from the
// neighbouring lanes (lanes 0 and 31 compute their outside neighbour).
template <int R, int MODEL, int SRC>
__global__ void __launch_bounds__(32 * kFineCols, 4) k_update_fine(FastParams P) {
  constexpr int NPAT = 1 << (2 * R + 1);
  constexpr int NC = 2 * R + 3;                  // window columns x-R-1 .. x+R+1
  constexpr int SW = kFineCols + 2 * (R + 1);   // state words staged per word-row
  __shared__ float s_lt[NPAT];
  __shared__ float s_ls[NPAT];
  __shared__ uint32_t s_w[3][SW];                // word-rows r-1, r, r+1; 0 outside
  fine_load_luts<R>(P, s_lt, s_ls);
  pdl_wait();
  pdl_launch_dependents();
  Scalars* sc = P.scal;
  if (stop_flag(sc)) return;
  const int lane = threadIdx.x & 31;
  const int x = blockIdx.x * kFineCols + (threadIdx.x >> 5);
  const int r = blockIdx.y;
  const int H = P.g.H, W = P.g.W;
  const int i = r * 32 + lane;
  // this pixel's data value, in flight while the words are staged
  const float d = (x < W && i < H) ? __ldg(P.data32 + (size_t)i * P.g.data_pitch + x) : 0.f;
  fine_stage_words<SW>(P, blockIdx.x * kFineCols - (R + 1), s_w);
  if (MODEL == REGION && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0 &&
      sc->zero_vel && sc->model != EDGE)
    sc->degenerate = 1;                          // sticky degenerate (engine.py:239-240)
  const float A = sc->A, B = sc->B, eps_u = sc->eps_u;
  if (x >= W) return;                            // whole warps
  // window of each column: 32 rows from i-R-1, from word-rows (r-1, r) for
  // the first R+1 lanes and (r, r+1) for the others
  const int up = lane > R ? 1 : 0;
  const int sh = up ? lane - R - 1 : lane + 31 - R;
  const uint32_t* wlo = &s_w[up][threadIdx.x >> 5];   // this column's first staged words
  const uint32_t* whi = wlo + SW;
  uint32_t win[NC], cm[NC];
#pragma unroll
  for (int j = 0; j < NC; ++j) {
    const int xc = x - (R + 1) + j;
    cm[j] = (xc >= 0 && xc < W) ? 0xffffffffu : 0u;
    win[j] = __funnelshift_r(wlo[j], whi[j], sh);
  }
  const bool cols_in = x - R - 1 >= 0 && x + R + 1 <= W - 1;
  auto row_in = [&](int row) { return cols_in && row - R >= 0 && row + R <= H - 1; };
  float pm, p0, pn, pl, pr;                      // phi at (i-1,x) (i,x) (i+1,x) (i,x-1) (i,x+1)
  if (SRC == SRC_SCALED) {                       // phi = +-s (binary initial state)
    auto ps = [&](int j, int m) { return ((win[j] >> (m + R)) & 1u) ? P.scale32 : -P.scale32; };
    pm = ps(R + 1, 0);
    p0 = ps(R + 1, 1);
    pn = ps(R + 1, 2);
    pl = ps(R, 1);
    pr = ps(R + 2, 1);
  } else {
    float t[NC];
    {
      const bool in = row_in(i);
      const uint32_t v0 = in ? 0u : row_valid_mask<R>(i, H);
      fine_trow<R, NC>(win, cm, 1, in, v0, in ? 0.f : s_ls[v0], s_lt, s_ls, t);
      pl = fine_hsum<R, NC>(P, t, 0);
      p0 = fine_hsum<R, NC>(P, t, 1);
      pr = fine_hsum<R, NC>(P, t, 2);
    }
    pm = __shfl_up_sync(0xffffffffu, p0, 1);
    pn = __shfl_down_sync(0xffffffffu, p0, 1);
    if (lane == 0 || lane == 31) {               // the row outside this warp
      const int m = lane == 0 ? 0 : 2, row = i - 1 + m;
      const bool in = row_in(row);
      const uint32_t v = in ? 0u : row_valid_mask<R>(row, H);
      fine_trow<R, NC>(win, cm, m, in, v, in ? 0.f : s_ls[v], s_lt, s_ls, t);
      const float pe = fine_hsum<R, NC>(P, t, 1);
      if (lane == 0) pm = pe;
      else pn = pe;
    }
  }
  bool bit = false;
  if (i < H) {
    // np.gradient: central differences, one-sided at the image border
    const float dx = (x == 0) ? 2.f * (pr - p0) : (x == W - 1) ? 2.f * (p0 - pl) : (pr - pl);
    const float dy = (i == 0) ? 2.f * (pn - p0) : (i == H - 1) ? 2.f * (p0 - pm) : (pn - pm);
    const float h = sqrt_approx(fmaf(dx, dx, dy * dy));     // 2 |grad phi|
    const float vf = (MODEL == REGION) ? fmaf(A, d, B) : d; // A, B / the g plane carry dt/2
    const float u = fmaf(vf, h, p0);
    bit = u > 0.f;
    LSE_CHECK_U(R, SRC, P, P.ctx, P.bits_in, i, x, u, eps_u);
    if (fabsf(u) <= eps_u)                       // near tie: the reference's fp64 decision
      bit = exact_u_fast<R, SRC>(P.ctx, P.bits_in, i, x) > 0.0;
  }
  const uint32_t word = __ballot_sync(0xffffffffu, bit);
  if (lane == 0) P.bits_out[(size_t)r * P.g.pitch_w + x] = word;
}

// Partition / checkpoint pass over b^{n+1} (engine.py:168-169, grid.py:102-118,
// engine.py:228-236): P = {phi >= 0} and M = {phi > 0} words, the sums over
// the pixels that changed side (CTAP: one partial per CTA, its words' plain
// fp64 sums added in column order; else one per state word, index r * W + x),
// multi-band runs record the changed bits instead.
// (The two-stage finalize of the tiled path follows; folding it into the
// last CTA of this kernel measured slower: one CTA then reduces every word's
// partial.)
// CTAP: one partial per CTA (small images: the finalize is then a single
// stage); else one per state word (the layout the two-stage finalize prefers).
template <int R, bool PART, bool CKPT, bool CTAP>
__global__ void __launch_bounds__(32 * kFineCols) k_partition_fine(FastParams P) {
  constexpr int NPAT = 1 << (2 * R + 1);
  constexpr int NC = 2 * R + 1;                  // window columns x-R .. x+R
  constexpr int SW = kFineCols + 2 * R;
  __shared__ float s_lt[NPAT];
  __shared__ float s_ls[NPAT];
  __shared__ uint32_t s_w[3][SW];
  fine_load_luts<R>(P, s_lt, s_ls);
  pdl_wait();
  pdl_launch_dependents();
  Scalars* sc = P.scal;
  if (stop_flag(sc)) return;
  fine_stage_words<SW>(P, blockIdx.x * kFineCols - R, s_w);
  const float eps_phi = sc->eps_phi;
  const int lane = threadIdx.x & 31;
  const int x = blockIdx.x * kFineCols + (threadIdx.x >> 5);
  const int r = blockIdx.y;
  const int H = P.g.H, W = P.g.W;
  if (!CTAP && x >= W) return;                   // whole warps (no CTA barrier below)
  const int i = r * 32 + lane;
  double a_in = 0.0, a_out = 0.0;
  long long n_in = 0, n_out = 0;
  unsigned long long mism = 0ull;
  if (CTAP ? x < W : true) {                     // (whole warps)
  // window of each column: 32 rows from i-R (word-rows (r-1, r) for the
  // first R lanes, (r, r+1) for the others)
  const int up = lane >= R ? 1 : 0;
  const int sh = up ? lane - R : lane + 32 - R;
  const uint32_t* wlo = &s_w[up][threadIdx.x >> 5];
  const uint32_t* whi = wlo + SW;
  uint32_t win[NC], cm[NC];
#pragma unroll
  for (int j = 0; j < NC; ++j) {
    const int xc = x - R + j;
    cm[j] = (xc >= 0 && xc < W) ? 0xffffffffu : 0u;
    win[j] = __funnelshift_r(wlo[j], whi[j], sh);
  }
  const bool act = i < H;
  const bool in = i - R >= 0 && i + R <= H - 1 && x - R >= 0 && x + R <= W - 1;
  float t[NC];
  const uint32_t v0 = in ? 0u : row_valid_mask<R>(i, H);
  fine_trow<R, NC>(win, cm, 0, in, v0, in ? 0.f : s_ls[v0], s_lt, s_ls, t);
  const float ph = fine_hsum<R, NC>(P, t, 0);
  bool pb = act && ph > 0.f, mb = pb;
  if (act) LSE_CHECK_PHI(R, P, P.ctx, P.bits_in, i, x, ph, eps_phi);
  if (act && fabsf(ph) <= eps_phi) {             // near tie: exact fp64 sign
    const double e = exact_phi_fast<R>(P.ctx, P.bits_in, i, x);
    pb = e >= 0.0;
    mb = e > 0.0;
  }
  const uint32_t pw = __ballot_sync(0xffffffffu, pb);
  const uint32_t mw = __ballot_sync(0xffffffffu, mb);
  const size_t o = (size_t)r * P.g.pitch_w + x;
  if (PART) {
    const uint32_t chg = P.pbits[o] ^ pw;
    if (P.chg) {
      if (lane == 0) P.chg[o] = chg;
    } else if ((chg >> lane) & 1u) {
      const double I = data_exact(P.ctx, i, x);
      if (pb) { a_in = I; n_in = 1; }
      else { a_out = I; n_out = 1; }
    }
    if (chg && lane == 0) P.pbits[o] = pw;
  }
  if (CKPT) {
    if (lane == 0) {
      mism = __popc(P.mbits[o] ^ mw);
      P.mbits[o] = mw;
    }
  }
  }
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) {
    a_in += __shfl_xor_sync(0xffffffffu, a_in, s);
    a_out += __shfl_xor_sync(0xffffffffu, a_out, s);
    n_in += __shfl_xor_sync(0xffffffffu, n_in, s);
    n_out += __shfl_xor_sync(0xffffffffu, n_out, s);
  }
  if (!CTAP) {
    if (lane == 0) {
      TilePartial t{};
      t.a_hi = a_in;
      t.b_hi = a_out;
      t.n_a = n_in;
      t.n_b = n_out;
      t.mism = mism;
      P.part[(size_t)r * W + x] = t;
    }
    return;
  }
  // one partial per CTA (its words in column order)
  __shared__ double s_a[kFineCols], s_b[kFineCols];
  __shared__ long long s_na[kFineCols], s_nb[kFineCols];
  __shared__ unsigned long long s_m[kFineCols];
  const int wq = threadIdx.x >> 5;
  if (lane == 0) {
    s_a[wq] = a_in; s_b[wq] = a_out; s_na[wq] = n_in; s_nb[wq] = n_out; s_m[wq] = mism;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    TilePartial t{};
    for (int w = 0; w < kFineCols; ++w) {
      t.a_hi += s_a[w];
      t.b_hi += s_b[w];
      t.n_a += s_na[w];
      t.n_b += s_nb[w];
      t.mism += s_m[w];
    }
    P.part[(size_t)blockIdx.y * gridDim.x + blockIdx.x] = t;
  }
}

}  // namespace lse
