// lse_resident.cuh -- a whole advance() call as ONE resident kernel (small images).
//
// On a small image an iteration of the per-pixel kernels (lse_fine.cuh) is a
// chain of three launches -- update, partition, finalize -- each a few
// microseconds of launch + drain latency around well under a microsecond of
// work (C1, 256^2: ~11 us per iteration).  Here the whole image is resident
// on chip for the call: every warp owns one task (the 32 rows of a word-row x
// kResCols adjacent columns, lane = row), keeps its pixels' data values in
// registers for all iterations, and the iterations are separated by barriers
// instead of kernel boundaries:
//
//   per iteration n (state b^n in global memory, read at L2):
//     phi^n = G * b^n at the task's pixels and one column either side
//       (zero padding / one-sided gradient at the image border exactly as
//        k_update_fine), |grad phi^n|;
//     [region / zhang, n > first]  P^n = {phi^n >= 0}, sums of I over the
//       pixels that changed side, checkpoint mask + mismatches -> one partial
//       per CTA -> barrier -> every CTA reduces all partials in the same fixed
//       order (double-double) and derives the coefficients (region_coeffs) and
//       the convergence state redundantly -- no broadcast step;
//     u = phi + (A I + B) 2|grad phi| -> b^{n+1} (near ties in fp64, the
//       reference's operation order) -> global -> barrier.
//
//   * phi is rebuilt once per iteration (the two-pass path rebuilds it in the
//     update and again in the partition);
//   * the barrier is a cluster barrier when the tasks fit one cluster of <= 16
//     CTAs (hardware barrier, ~0.3 us; the CTAs' partials go straight into
//     every CTA's shared memory), else a grid barrier of a cooperative launch
//     (one CTA per SM, up to three tasks per warp: images up to ~1.8 Mpx);
//   * edge runs need one barrier per iteration (two on checkpoints).
//
// The arithmetic of every decision is the per-pixel kernels' (same LUT values,
// FMA order, gradient, guards, exact evaluators), so the decisions are the
// reference's; only the grouping of the c+/c- sums differs (per lane over its
// columns, lanes and warps by xor trees, CTAs by a double-double tree).
// engine.py:148-174 (one iteration), :222-240 (checkpoints), grid.py:102-118.
#pragma once

namespace lse {

constexpr int kResWarps = 16;                   // warps per CTA (128 registers per thread)
constexpr int kResThreads = 32 * kResWarps;
constexpr int kResCols = 8;                     // columns per warp task
constexpr int kResClusterMax = 16;              // CTAs of the one-cluster mode

struct ResidentArgs {
  uint32_t* bits[2];       // state ping-pong (b^n in bits[cur])
  int cur0;                // buffer holding the state at iteration it0
  int scaled;              // that state is the +-scale initial field (SRC_SCALED)
  long long it0, steps;    // iterations it0+1 .. it0+steps
  long long cce;           // conv_check_every
  int ntasks, ncb;         // warp tasks = HR * ncb, ncb = ceil(W / kResCols)
  TilePartial* parts;      // one partial per CTA
  unsigned int* sync;      // grid barrier arrival counter (zero at launch; GRID only)
};

// All CTAs of the launch: memory written before is visible (at L2) after.
// (Grid barrier: every CTA polls the arrival counter itself.  Publishing the
// epoch on a second line for the others to poll measured slower -- the
// release costs the last arriver two more L2 round trips: C2 107 -> 98
// Gpix-it/s.)
template <bool GRID>
__device__ __forceinline__ void res_sync(unsigned int* ctr, unsigned int& epoch) {
  if (GRID) {
    __syncthreads();
    if (threadIdx.x == 0) {
      epoch += gridDim.x;
      __threadfence();
      atomicAdd(ctr, 1u);
      unsigned int v;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
      } while (v < epoch);
    }
    __syncthreads();
  } else {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\t"
                 "barrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
}

// one-cluster mode: a CTA's partial goes straight into every CTA's shared memory
struct __align__(16) ResPart {
  double a, b;
  long long na, nb;
  unsigned long long mm;
  long long pad_;
};
__device__ __forceinline__ uint32_t res_smem(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint32_t res_mapa(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void res_st_cluster(uint32_t addr, long long v) {
  asm volatile("st.shared::cluster.b64 [%0], %1;" ::"r"(addr), "l"(v) : "memory");
}

// vertical-pass values of window row offset m for every window column
// (fine_trow with the column mask derived from the column index)
template <int R, int NC>
__device__ __forceinline__ void res_trow(const uint32_t (&win)[NC], int xw0, int W, int m, bool in,
                                         uint32_t vr, float Lv, const float* s_lt,
                                         const float* s_ls, float (&t)[NC]) {
  constexpr uint32_t PM = (1u << (2 * R + 1)) - 1u;
  if (in) {
#pragma unroll
    for (int j = 0; j < NC; ++j) t[j] = s_lt[(win[j] >> m) & PM];
  } else {
#pragma unroll
    for (int j = 0; j < NC; ++j) {
      const bool cin = (unsigned)(xw0 + j) < (unsigned)W;
      t[j] = fmaf(2.f, s_ls[cin ? ((win[j] >> m) & PM & vr) : 0u], cin ? -Lv : 0.f);
    }
  }
}

// checkpoint bookkeeping of finalize_cta (engine.py:228-236)
__device__ __forceinline__ void res_checkpoint(Scalars* sc, unsigned long long mism, long long iter) {
  sc->n_ckpt += 1;
  if (sc->n_ckpt >= 2) sc->equal_run = (mism == 0) ? sc->equal_run + 1 : 0;
  const long long cw = sc->conv_window;
  if (cw == 1 || (sc->n_ckpt >= cw && sc->equal_run >= cw - 1)) {
    sc->stop = 1;
    sc->converged = 1;
    sc->converged_iter = iter;
  }
}

// phase timing (profiling builds, -DLSE_RES_TRACE): CTA 0 / thread 0 accumulates
// the SM clock per phase and prints the totals when the call ends
#ifdef LSE_RES_TRACE
#define RES_T(k) do { if (tid == 0 && blockIdx.x == 0) { const long long c_ = clock64(); tr[k] += c_ - tr_last; tr_last = c_; } } while (0)
#else
#define RES_T(k) do { } while (0)
#endif

// NT: tasks per warp (larger images on a full cooperative grid).  Edge runs
// have constant coefficients: a warp finishes one task (phi -> checkpoint
// words -> update) before the next.  Region / zhang runs need the coefficients
// between the partition and the update of an iteration, so a warp keeps phi
// and |grad phi| of all its tasks across the barrier (NT > 1: some of them in
// local memory -- one store and one load per pixel and iteration, far cheaper
// than rebuilding phi).
template <int R, int MODEL, bool GRID, int NT>
__global__ void __launch_bounds__(kResThreads, 1) k_resident(FastParams P, ResidentArgs A) {
  constexpr int CW = kResCols;
  constexpr int NPAT = 1 << (2 * R + 1);
  constexpr int NC = CW + 2 * R + 2;             // window columns x0-R-1 .. x0+CW+R
  constexpr int NSW = sizeof(Scalars) / 4, NCW = sizeof(ExactCtx) / 4;
  static_assert(sizeof(Scalars) % 4 == 0 && sizeof(ExactCtx) % 4 == 0, "word copies");
  __shared__ float s_lt[NPAT];
  __shared__ float s_ls[NPAT];
  __shared__ uint32_t s_w[kResWarps][3][NC];     // word-rows r-1, r, r+1 of the window columns
  __shared__ Scalars s_sc;                       // this CTA's copy (every CTA derives the same)
  __shared__ ExactCtx s_ctx;                     // exact-evaluator context over s_sc
  __shared__ double s_pa[kResWarps], s_pb[kResWarps];
  __shared__ int s_na[kResWarps], s_nb[kResWarps], s_mm[kResWarps];
  __shared__ ResPart s_parts[kResClusterMax];    // one-cluster mode: every CTA's partial
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  fine_load_luts<R>(P, s_lt, s_ls);
  {
    const uint32_t* gs = reinterpret_cast<const uint32_t*>(P.scal);
    uint32_t* ss = reinterpret_cast<uint32_t*>(&s_sc);
    for (int q = tid; q < NSW; q += kResThreads) ss[q] = __ldcg(gs + q);
    const uint32_t* gc = reinterpret_cast<const uint32_t*>(P.ctx);
    uint32_t* cs = reinterpret_cast<uint32_t*>(&s_ctx);
    for (int q = tid; q < NCW; q += kResThreads) cs[q] = __ldcg(gc + q);
  }
  __syncthreads();
  if (tid == 0) s_ctx.scal = &s_sc;
  __syncthreads();
  if (s_sc.stop) return;                         // (every CTA alike)
  const unsigned long long fallbacks0 = s_sc.fallbacks;
  unsigned int epoch = 0u;
  if (!GRID) res_sync<GRID>(A.sync, epoch);      // every CTA of the cluster is running (DSMEM)

  const int H = P.g.H, W = P.g.W, HR = P.g.HR, pitch_w = P.g.pitch_w;
  // task t of this warp: consecutive warps of the launch take adjacent tasks
  int tk_r[NT], tk_x0[NT];
  bool tk_on[NT];
  float d[NT][CW];                               // this lane's data values, all iterations
  uint32_t pold[NT], mold[NT];                   // lane c: partition / checkpoint word of column x0+c
#pragma unroll
  for (int t = 0; t < NT; ++t) {
    const int task = (t * (int)gridDim.x + (int)blockIdx.x) * kResWarps + warp;
    tk_on[t] = task < A.ntasks;
    tk_r[t] = tk_on[t] ? task / A.ncb : 0;
    tk_x0[t] = tk_on[t] ? (task - tk_r[t] * A.ncb) * CW : 0;
    const int i = tk_r[t] * 32 + lane;
#pragma unroll
    for (int c = 0; c < CW; ++c)
      d[t][c] = (tk_on[t] && i < H && tk_x0[t] + c < W)
                    ? __ldg(P.data32 + (size_t)i * P.g.data_pitch + tk_x0[t] + c) : 0.f;
    pold[t] = mold[t] = 0u;
    if (tk_on[t] && lane < CW && tk_x0[t] + lane < W) {
      const size_t wofs = (size_t)tk_r[t] * pitch_w + tk_x0[t] + lane;
      pold[t] = __ldcg(P.pbits + wofs);
      mold[t] = __ldcg(P.mbits + wofs);
    }
  }
  const float eps_phi = s_sc.eps_phi;
  const int up = lane > R ? 1 : 0;
  const int sh = up ? lane - R - 1 : lane + 31 - R;

  int cur = A.cur0;
  long long to_ckpt = (A.cce - (A.it0 + 1) % A.cce) % A.cce;   // iterations from it0+1 to the next checkpoint
  const long long it_end = A.it0 + A.steps;
#ifdef LSE_RES_TRACE
  long long tr[24] = {0}, tr_last = clock64();
#endif
  for (long long n = A.it0;; ++n) {
    RES_T(7);
    const uint32_t* bits = A.bits[cur];
    uint32_t* bits_next = A.bits[cur ^ 1];
    const bool first = n == A.it0;
    const bool scaled = first && A.scaled;
    const bool more = n != it_end;               // an update n -> n+1 follows
    // partition / checkpoint of b^n (owed by update n; not on entry)
    const bool do_part = !first && MODEL == REGION;
    const bool do_ckpt = !first && to_ckpt == 0;
    if (!first) to_ckpt = to_ckpt == 0 ? A.cce - 1 : to_ckpt - 1;
    double a_in = 0.0, a_out = 0.0;
    int n_in = 0, n_out = 0, mism = 0;           // (a warp's pixels: 32-bit counts)
    float p0a[NT][CW], hha[NT][CW];              // phi^n and 2 |grad phi^n| at the lane's pixels

    // b^{n+1} of task (r, x0) from p0 / hh and the coefficients; near ties in fp64
    auto update_task = [&](int t, int r, int x0, float Av, float Bv, float eps_u) {
      const int i = r * 32 + lane;
      const float (&p0)[CW] = p0a[t];
      const float (&hh)[CW] = hha[t];
      float u[CW];
#pragma unroll
      for (int c = 0; c < CW; ++c) {
        const float vf = (MODEL == REGION) ? fmaf(Av, d[t][c], Bv) : d[t][c];   // carry dt/2
        u[c] = fmaf(vf, hh[c], p0[c]);
      }
      float umin = fabsf(u[0]);
#pragma unroll
      for (int c = 1; c < CW; ++c) umin = fminf(umin, fabsf(u[c]));
      uint32_t wnew = 0u;
      if (!__any_sync(0xffffffffu, umin <= eps_u)) {
#pragma unroll
        for (int c = 0; c < CW; ++c) {
          const uint32_t w = __ballot_sync(0xffffffffu, u[c] > 0.f);
          if (lane == c) wnew = w;
        }
      } else {                                   // near ties: the reference's fp64 decision
        uint32_t b8 = 0u, tie8 = 0u;             // bit c: column x0 + c
#pragma unroll
        for (int c = 0; c < CW; ++c) {
          b8 |= (u[c] > 0.f) ? (1u << c) : 0u;
          tie8 |= (fabsf(u[c]) <= eps_u) ? (1u << c) : 0u;
        }
#pragma unroll 1
        for (int c = 0; c < CW; ++c)
          if ((tie8 >> c) & 1u) {
            const double e = scaled ? exact_u_fast<R, SRC_SCALED, true>(&s_ctx, bits, i, x0 + c)
                                    : exact_u_fast<R, SRC_SMOOTH, true>(&s_ctx, bits, i, x0 + c);
            b8 = (b8 & ~(1u << c)) | (e > 0.0 ? (1u << c) : 0u);
          }
#pragma unroll
        for (int c = 0; c < CW; ++c) {
          const uint32_t w = __ballot_sync(0xffffffffu, (b8 >> c) & 1u);
          if (lane == c) wnew = w;
        }
      }
      if (lane < CW && x0 + lane < W) bits_next[(size_t)r * pitch_w + x0 + lane] = wnew;
    };

#pragma unroll
    for (int t = 0; t < NT; ++t) {
      const int r = tk_r[t], x0 = tk_x0[t];
      const int i = r * 32 + lane;
      const bool rowok = tk_on[t] && i < H;
      float (&p0)[CW] = p0a[t];
      float (&hh)[CW] = hha[t];
      if (tk_on[t]) {
        for (int q = lane; q < 3 * NC; q += 32) {
          const int row = q / NC, col = q - row * NC;
          const int wr = r - 1 + row, xc = x0 - R - 1 + col;
          s_w[warp][row][col] = (wr >= 0 && wr < HR && xc >= 0 && xc < W)
                                    ? __ldcg(bits + (size_t)wr * pitch_w + xc) : 0u;
        }
        __syncwarp();
        RES_T(8);
        // window of each column: 32 rows from i-R-1 (k_update_fine's frame)
        uint32_t win[NC];
#pragma unroll
        for (int j = 0; j < NC; ++j) win[j] = __funnelshift_r(s_w[warp][up][j], s_w[warp][up + 1][j], sh);
        __syncwarp();
        RES_T(9);
        float pm[CW], pn[CW];
        float pc[CW + 2];                        // phi of row i at columns x0-1 .. x0+CW
        if (scaled) {                            // phi = +-s (binary initial state)
          auto ps = [&](int j, int m) { return ((win[j] >> (m + R)) & 1u) ? P.scale32 : -P.scale32; };
#pragma unroll
          for (int j0 = 0; j0 < CW + 2; ++j0) pc[j0] = ps(j0 + R, 1);
#pragma unroll
          for (int c = 0; c < CW; ++c) {
            pm[c] = ps(c + R + 1, 0);
            pn[c] = ps(c + R + 1, 2);
          }
        } else {
          float tv[NC];
          const bool cols_in = x0 - R - 1 >= 0 && x0 + CW + R <= W - 1;
          auto row_in = [&](int row) { return cols_in && row - R >= 0 && row + R <= H - 1; };
          {
            const bool in = row_in(i);
            const uint32_t v0 = in ? 0u : row_valid_mask<R>(i, H);
            res_trow<R, NC>(win, x0 - R - 1, W, 1, in, v0, in ? 0.f : s_ls[v0], s_lt, s_ls, tv);
#pragma unroll
            for (int j0 = 0; j0 < CW + 2; ++j0) pc[j0] = fine_hsum<R, NC>(P, tv, j0);
          }
          RES_T(10);
#pragma unroll
          for (int c = 0; c < CW; ++c) {
            pm[c] = __shfl_up_sync(0xffffffffu, pc[c + 1], 1);
            pn[c] = __shfl_down_sync(0xffffffffu, pc[c + 1], 1);
          }
          RES_T(11);
          // the row outside this warp, on its two edge lanes (spreading it over
          // 2 CW lanes -- one horizontal sum each from the staged words, then
          // shuffles back -- measured slower: C1 9.85 -> 9.5 Gpix-it/s)
          if (lane == 0 || lane == 31) {
            const int m = lane == 0 ? 0 : 2, row = i - 1 + m;
            const bool in = row_in(row);
            const uint32_t v = in ? 0u : row_valid_mask<R>(row, H);
            res_trow<R, NC>(win, x0 - R - 1, W, m, in, v, in ? 0.f : s_ls[v], s_lt, s_ls, tv);
#pragma unroll
            for (int c = 0; c < CW; ++c) {
              const float pe = fine_hsum<R, NC>(P, tv, c + 1);
              if (lane == 0) pm[c] = pe;
              else pn[c] = pe;
            }
          }
          RES_T(12);
        }
        // np.gradient: central differences, one-sided at the image border --
        // branch-free: the missing neighbour is replaced by the centre and the
        // difference doubled (2 (b - a) and (b - a) 1 are exact scalings)
        const bool yt = i == 0, yb = i == H - 1 && !yt;
        const float sy = (yt || yb) ? 2.f : 1.f;
#pragma unroll
        for (int c = 0; c < CW; ++c) {
          const int x = x0 + c;
          p0[c] = pc[c + 1];
          const bool xl = x == 0, xr = x == W - 1 && !xl;
          const float xa = xl ? p0[c] : pc[c], xb = xr ? p0[c] : pc[c + 2];
          const float ya = yt ? p0[c] : pm[c], yb2 = yb ? p0[c] : pn[c];
          const float dx = (xb - xa) * ((xl || xr) ? 2.f : 1.f);
          const float dy = (yb2 - ya) * sy;
          hh[c] = sqrt_approx(fmaf(dx, dx, dy * dy));
          // pixels outside the image: phi = -1, |grad| = 0 (never positive,
          // never a near tie), so the loops below need no validity tests
          if (!(rowok && x < W)) {
            p0[c] = -1.f;
            hh[c] = 0.f;
          }
        }
      } else {
#pragma unroll
        for (int c = 0; c < CW; ++c) {
          p0[c] = -1.f;
          hh[c] = 0.f;
        }
      }
      RES_T(0);

      if ((do_part || do_ckpt) && tk_on[t]) {
        // signs of phi^n; near ties (rare: one warp-wide test on the smallest
        // |phi| of the lane) take the exact fp64 sign
        const bool wlane = lane < CW && x0 + lane < W;
        const size_t wofs = (size_t)r * pitch_w + x0 + lane;
        float amin = fabsf(p0[0]);
#pragma unroll
        for (int c = 1; c < CW; ++c) amin = fminf(amin, fabsf(p0[c]));
        uint32_t pnew = pold[t], mnew = mold[t];
        uint32_t pb8 = 0u;                       // bit c: this lane's pixel of column c is in P
        if (!__any_sync(0xffffffffu, amin <= eps_phi)) {
#pragma unroll
          for (int c = 0; c < CW; ++c) {
            const bool pb = p0[c] > 0.f;
            const uint32_t pw = __ballot_sync(0xffffffffu, pb);
            pb8 |= pb ? (1u << c) : 0u;
            if (lane == c) {
              if (do_part) pnew = pw;
              if (do_ckpt) mnew = pw;            // {phi > 0} = {phi >= 0} without ties
            }
          }
        } else {
          uint32_t tie8 = 0u;
#pragma unroll
          for (int c = 0; c < CW; ++c) {
            pb8 |= (p0[c] > 0.f) ? (1u << c) : 0u;
            tie8 |= (fabsf(p0[c]) <= eps_phi) ? (1u << c) : 0u;
          }
          uint32_t mb8 = pb8;
#pragma unroll 1
          for (int c = 0; c < CW; ++c)
            if ((tie8 >> c) & 1u) {
              const double e = exact_phi_fast<R, true>(&s_ctx, bits, i, x0 + c);
              pb8 = (pb8 & ~(1u << c)) | (e >= 0.0 ? (1u << c) : 0u);
              mb8 = (mb8 & ~(1u << c)) | (e > 0.0 ? (1u << c) : 0u);
            }
#pragma unroll
          for (int c = 0; c < CW; ++c) {
            const uint32_t pw = __ballot_sync(0xffffffffu, (pb8 >> c) & 1u);
            const uint32_t mw = __ballot_sync(0xffffffffu, (mb8 >> c) & 1u);
            if (lane == c) {
              if (do_part) pnew = pw;
              if (do_ckpt) mnew = mw;
            }
          }
        }
        // sums of I over the pixels that changed side (few columns change)
        if (do_part && __any_sync(0xffffffffu, wlane && pnew != pold[t])) {
#pragma unroll
          for (int c = 0; c < CW; ++c) {
            const uint32_t chg = __shfl_sync(0xffffffffu, pnew ^ pold[t], c);
            if ((chg >> lane) & 1u) {
              const double I = s_ctx.data64 ? data_exact(&s_ctx, i, x0 + c) : (double)d[t][c];
              if ((pb8 >> c) & 1u) { a_in += I; n_in += 1; }
              else { a_out += I; n_out += 1; }
            }
          }
        }
        if (wlane) {
          if (do_part && pnew != pold[t]) P.pbits[wofs] = pnew;
          if (do_ckpt) {
            mism += __popc(mold[t] ^ mnew);
            P.mbits[wofs] = mnew;
            mold[t] = mnew;
          }
          pold[t] = pnew;
        }
      }
      RES_T(13);
      // edge runs: constant coefficients, the update follows at once (on a
      // checkpoint that turns out converged, b^{n+1} lands in the buffer that
      // is then not adopted)
      if (MODEL == EDGE && more && tk_on[t]) update_task(t, r, x0, 0.f, 0.f, s_sc.eps_u);
    }

    if (do_part || do_ckpt) {
      // warp totals (few pixels change side: most warps have none to add)
      if (__any_sync(0xffffffffu, n_in + n_out != 0)) {
#pragma unroll
        for (int s = 16; s > 0; s >>= 1) {
          a_in += __shfl_xor_sync(0xffffffffu, a_in, s);
          a_out += __shfl_xor_sync(0xffffffffu, a_out, s);
          n_in += __shfl_xor_sync(0xffffffffu, n_in, s);
          n_out += __shfl_xor_sync(0xffffffffu, n_out, s);
        }
      }
      if (do_ckpt) {                             // (lanes 0 .. CW-1 hold the mismatches)
#pragma unroll
        for (int s = CW / 2; s > 0; s >>= 1) mism += __shfl_xor_sync(0xffffffffu, mism, s);
      }
      if (lane == 0) {
        s_pa[warp] = a_in; s_pb[warp] = a_out; s_na[warp] = n_in; s_nb[warp] = n_out;
        s_mm[warp] = mism;
      }
      RES_T(14);
      __syncthreads();
      RES_T(15);
      if (warp == 0) {                           // this CTA's partial: its warps by xor tree
        const bool lw = lane < kResWarps;
        double ca = lw ? s_pa[lane] : 0.0, cb = lw ? s_pb[lane] : 0.0;
        int cna = lw ? s_na[lane] : 0, cnb = lw ? s_nb[lane] : 0, cmm = lw ? s_mm[lane] : 0;
#pragma unroll
        for (int s = kResWarps / 2; s > 0; s >>= 1) {
          ca += __shfl_xor_sync(0xffffffffu, ca, s);
          cb += __shfl_xor_sync(0xffffffffu, cb, s);
          cna += __shfl_xor_sync(0xffffffffu, cna, s);
          cnb += __shfl_xor_sync(0xffffffffu, cnb, s);
          cmm += __shfl_xor_sync(0xffffffffu, cmm, s);
        }
        if (GRID) {
          if (lane == 0) {
            TilePartial tp{};
            tp.a_hi = ca; tp.b_hi = cb; tp.n_a = cna; tp.n_b = cnb; tp.mism = (unsigned long long)cmm;
            A.parts[blockIdx.x] = tp;
          }
        } else if (lane < (int)gridDim.x) {
          // one cluster: straight into slot [this CTA] of CTA `lane`'s shared memory
          const uint32_t ra = res_mapa(res_smem(&s_parts[blockIdx.x]), (uint32_t)lane);
          res_st_cluster(ra, __double_as_longlong(ca));
          res_st_cluster(ra + 8, __double_as_longlong(cb));
          res_st_cluster(ra + 16, (long long)cna);
          res_st_cluster(ra + 24, (long long)cnb);
          res_st_cluster(ra + 32, (long long)cmm);
        }
      }
      RES_T(1);
      res_sync<GRID>(A.sync, epoch);
      RES_T(2);
      if (warp == 0) {                           // every CTA: all partials, fixed order
        double ah = 0, al = 0, bh = 0, bl = 0;
        long long na = 0, nb = 0;
        unsigned long long mm = 0;
        if (GRID) {
          for (int q = lane; q < (int)gridDim.x; q += 32) {
            const TilePartial* pp = A.parts + q;
            const double2 SA = __ldcg(reinterpret_cast<const double2*>(&pp->a_hi));
            const double2 SB = __ldcg(reinterpret_cast<const double2*>(&pp->b_hi));
            const longlong2 NN = __ldcg(reinterpret_cast<const longlong2*>(&pp->n_a));
            dd_add_dd(ah, al, SA.x, SA.y);
            dd_add_dd(bh, bl, SB.x, SB.y);
            na += NN.x;
            nb += NN.y;
            mm += __ldcg(&pp->mism);
          }
        } else if (lane < (int)gridDim.x) {
          const volatile ResPart* pp = &s_parts[lane];
          ah = pp->a; bh = pp->b; na = pp->na; nb = pp->nb; mm = pp->mm;
        }
        RES_T(16);
        int np2 = 1;
        while (np2 < (int)gridDim.x && np2 < 32) np2 <<= 1;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          if (o < np2) {                         // (lanes beyond the CTA count hold zeros)
            if (MODEL == REGION) {
              dd_shfl_add(ah, al, o);
              dd_shfl_add(bh, bl, o);
              na += __shfl_xor_sync(0xffffffffu, na, o);
              nb += __shfl_xor_sync(0xffffffffu, nb, o);
            }
            mm += __shfl_xor_sync(0xffffffffu, mm, o);
          }
        }
        RES_T(17);
        if (lane == 0) {
          Scalars* sc = &s_sc;
          if (do_part) {                         // finalize_cta, delta mode
            dd_add_dd(sc->sp_hi, sc->sp_lo, ah, al);
            dd_add_dd(sc->sp_hi, sc->sp_lo, -bh, -bl);
            dd_add_dd(sc->sn_hi, sc->sn_lo, bh, bl);
            dd_add_dd(sc->sn_hi, sc->sn_lo, -ah, -al);
            sc->n_pos += na - nb;
            region_coeffs(sc);
          }
          if (do_ckpt) res_checkpoint(sc, mm, n);
        }
        RES_T(18);
      }
      __syncthreads();
      RES_T(3);
      if (s_sc.stop) break;                      // converged at n: b^n stays the state
    }
    if (!more) break;

    // ---- update n -> n+1 (region / zhang: with the coefficients just derived)
    if (MODEL == REGION) {
      const float Av = s_sc.A, Bv = s_sc.B, eps_u = s_sc.eps_u;
      if (tid == 0 && s_sc.zero_vel && s_sc.model != EDGE)
        s_sc.degenerate = 1;                     // sticky degenerate (engine.py:239-240)
#pragma unroll
      for (int t = 0; t < NT; ++t)
        if (tk_on[t]) update_task(t, tk_r[t], tk_x0[t], Av, Bv, eps_u);
    }
    RES_T(4);
    res_sync<GRID>(A.sync, epoch);
    RES_T(5);
    cur ^= 1;
  }
#ifdef LSE_RES_TRACE
  if (tid == 0 && blockIdx.x == 0)
    printf("res trace (cycles, %lld its): phi+grad %lld cta %lld sync1 %lld finalize %lld update %lld "
           "sync2 %lld loop %lld fallbacks %llu\n", A.steps, tr[0], tr[1], tr[2], tr[3], tr[4], tr[5],
           tr[7], s_sc.fallbacks - fallbacks0);
  if (tid == 0 && blockIdx.x == 0)
    printf("  phi: stage %lld win %lld hsum %lld shfl %lld outer %lld grad %lld | part: cols(+edge update) %lld tree %lld "
           "bar %lld cta %lld | fin: load %lld tree %lld coef %lld bar %lld\n", tr[8], tr[9], tr[10],
           tr[11], tr[12], tr[0], tr[13], tr[14], tr[15], tr[1], tr[16], tr[17], tr[18], tr[3]);
#endif

  // ---- write the scalars back (CTA 0's copy; every CTA adds its own near-tie count)
  __syncthreads();
  const unsigned long long mine = s_sc.fallbacks - fallbacks0;
  __syncthreads();
  if (blockIdx.x == 0) {
    if (tid == 0) s_sc.fallbacks = fallbacks0;
    __syncthreads();
    uint32_t* gs = reinterpret_cast<uint32_t*>(P.scal);
    const uint32_t* ss = reinterpret_cast<const uint32_t*>(&s_sc);
    for (int q = tid; q < NSW; q += kResThreads) gs[q] = ss[q];
  }
  res_sync<GRID>(A.sync, epoch);
  if (tid == 0 && mine) atomicAdd(&P.scal->fallbacks, mine);
}

}  // namespace lse
