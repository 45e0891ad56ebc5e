// lse_api.cu -- C ABI (include/lse_b200.h): the run handle and its driver.
//
// The driver mirrors EvolutionRun (engine.py:193-269).  Per iteration it
// picks one of two device paths:
//   * fast  : binary state (reinit_period = reg_period = 1, 3 <= ts_reg <= 9)
//             -> k_update + k_partition (two launches, no host sync; a
//             device stop flag turns later launches into no-ops after
//             convergence);
//   * generic: exact fp64 field kernels (any other cadence, injected
//             non-binary states, out-of-range inputs), host-synchronised so
//             NumericalInstabilityError can name the iteration.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <climits>
#include <cmath>
#include <cstddef>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "lse_b200.h"
#include "lse_device.cuh"
#include "lse_fast.cuh"
#include "lse_generic.cuh"
#include "lse_fine.cuh"
#include "lse_resident.cuh"
#include "lse_contours.cuh"

using namespace lse;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CK(x)                                                                            \
  do {                                                                                   \
    cudaError_t e_ = (x);                                                                \
    if (e_ != cudaSuccess)                                                               \
      return fail(LSE_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_));        \
  } while (0)

std::atomic<long long> g_launches{0};

#define CKL()                                                                            \
  do {                                                                                   \
    g_launches.fetch_add(1, std::memory_order_relaxed);                                  \
    cudaError_t e_ = cudaGetLastError();                                                 \
    if (e_ != cudaSuccess)                                                               \
      return fail(LSE_ERR_CUDA, std::string("launch: ") + cudaGetErrorString(e_));       \
  } while (0)

#define TRY(x)                 \
  do {                         \
    int rc_ = (x);             \
    if (rc_ != LSE_OK) return rc_; \
  } while (0)

inline long long round_up(long long a, long long b) { return (a + b - 1) / b * b; }

// Per-iteration kernels are launched with programmatic stream serialization
// (each waits in pdl_wait before reading its predecessor's results), so a
// kernel's launch and static prologue overlap the previous kernel's tail.
// LSE_NO_PDL=1 launches them plainly (A/B measurements).
bool pdl_enabled() {
  static const bool on = std::getenv("LSE_NO_PDL") == nullptr;
  return on;
}

template <typename... KArgs, typename... Args>
int launch_pdl_smem(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                    Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, args...);
  if (e != cudaSuccess) return fail(LSE_ERR_CUDA, std::string("launch: ") + cudaGetErrorString(e));
  return LSE_OK;
}

template <typename... KArgs, typename... Args>
int launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, cudaStream_t st, Args... args) {
  return launch_pdl_smem(kern, grid, block, 0, st, args...);
}

// a kernel with dynamic shared memory: opt in to the size and to the carveout
// that keeps kUpdateCtasPerSm CTAs resident (once per kernel)
template <typename... KArgs>
int prepare_smem(void (*kern)(KArgs...), size_t smem) {
  static std::vector<const void*> done;
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  const void* key = reinterpret_cast<const void*>(kern);
  if (std::find(done.begin(), done.end(), key) != done.end()) return LSE_OK;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                          cudaSharedmemCarveoutMaxShared));
  done.push_back(key);
  return LSE_OK;
}

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

template <typename T>
int dalloc(T** p, size_t n) {
  *p = nullptr;
  if (n == 0) n = 1;
  CK(cudaMalloc((void**)p, n * sizeof(T)));
  return LSE_OK;
}

int check_device() {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0)
    return fail(LSE_ERR_NODEVICE, std::string("no CUDA device: ") + cudaGetErrorString(e));
  return LSE_OK;
}

// exact vertical-pass value of a full-window bit pattern (host, same order as
// the device and scipy; built with -ffp-contract=off)
double host_t64(unsigned p, int R, const double* w) {
  auto b = [&](int k) { return ((p >> k) & 1u) ? 1.0 : -1.0; };
  volatile double acc = b(R) * w[0];
  for (int d = R; d >= 1; --d) {
    volatile double s = b(R - d) + b(R + d);
    volatile double m = s * w[d];
    acc = acc + m;
  }
  return acc;
}

// near-tie guards (lse_device.cuh: kGuard x the a-priori fp32 error bounds)
const double kEpsPhi = kGuard * kErrPhi;

double edge_eps_u(double dt) {
  return kGuard * (kErrPhi + dt * (kErrGrad + 1.5 * 0x1p-22 + 0x1p-21) + 0x1p-22 * (1.0 + 1.5 * dt));
}

}  // namespace

// Guard certification (validation builds, -DLSE_CHECK_BOUND): process-wide
// per-thread slots every checked launch accumulates into (lse_check_stats).
namespace {
#ifdef LSE_CHECK_BOUND
constexpr long long kCheckSlots = 1LL << 21;
CheckSlot* g_chk = nullptr;
long long g_check_every = 1;
__global__ void k_check_reset(CheckSlot* s, long long n) {
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n;
       q += (long long)gridDim.x * blockDim.x)
    s[q] = CheckSlot{0.f, 0.f, 3.0e38f, 3.0e38f, 0u, 0u, 0ull};
}
CheckSlot* check_slots() {
  if (!g_chk) {
    if (cudaMalloc(&g_chk, kCheckSlots * sizeof(CheckSlot)) != cudaSuccess) return nullptr;
    k_check_reset<<<512, 256>>>(g_chk, kCheckSlots);
    cudaDeviceSynchronize();
    if (const char* e = std::getenv("LSE_CHECK_EVERY")) g_check_every = std::max(1LL, std::atoll(e));
  }
  return g_chk;
}
#endif
// the certification slots of the launches of iteration `it` (null: unchecked)
void set_check(FastParams& P, long long it) {
#ifdef LSE_CHECK_BOUND
  CheckSlot* s = check_slots();
  const bool on = s && it % g_check_every == 0;
  P.chk = on ? s : nullptr;
  P.chk_cap = on ? kCheckSlots : 0;
#else
  (void)it;
  P.chk = nullptr;
  P.chk_cap = 0;
#endif
}
}  // namespace

// one-stage finalize cutoff of the tiled kernels (lone runs and every tile of
// a batch: both sites read the run's copy, so a batched tile and the same
// tile alone reduce alike); LSE_ONESTAGE_MAX_PARTS overrides it at creation
constexpr long long kOneStageMaxParts = 768;

struct lse_run {
  lse_params p{};
  std::vector<double> wreg, wpre;
  int H = 0, W = 0, R = 0;
  RunGeom g{};
  long long npx = 0;
  int nthr = kThreads;
  cudaStream_t st = nullptr;
  // data plane
  float* d_data32 = nullptr;
  double* d_data64 = nullptr;
  bool fp32_exact = true;
  // multi-band runs (LSE_MODEL_BANDS): band planes; d_data32 then holds the
  // per-pass data term D written by k_band_peak
  int nbands = 1;
  float* d_bands32 = nullptr;
  double* d_bands64 = nullptr;
  uint32_t* d_chg = nullptr;
  TilePartial* d_bpart = nullptr;
  unsigned long long* d_pmax = nullptr;   // band chain arrival counters (2, zeroed)
  // reusable device scratch for per-call buffers (mask read-back, injected
  // signs, seed polygons, flags): no cudaMalloc / cudaFree -- each of which
  // can stall the device -- on the per-job paths
  unsigned char* d_scratch = nullptr;
  size_t scratch_cap = 0;
  double* d_poly = nullptr;
  long long* d_offs = nullptr;
  size_t poly_cap = 0, offs_cap = 0;
  int* d_flag = nullptr;
  // Chan-Vese baseline: derivative planes and distance-transform scratch
  double* d_px = nullptr;
  double* d_py = nullptr;
  double* d_mag = nullptr;
  long long* d_edt_g = nullptr;
  int* d_edt_v = nullptr;
  long long* d_edt_zn = nullptr;
  long long* d_edt_zd = nullptr;
  double* d_dist[2] = {nullptr, nullptr};
  double img_absmax = 0.0;
  // state
  uint32_t* d_bits[2] = {nullptr, nullptr};
  uint32_t* d_P = nullptr;
  uint32_t* d_M = nullptr;
  uint32_t* d_mask = nullptr;
  TilePartial* d_part = nullptr;
  Scalars* d_scal = nullptr;
  Scalars* h_scal = nullptr;
  float* d_lut_t = nullptr;
  float* d_lut_s = nullptr;
  ExactCtx* d_ctx = nullptr;
  ExactCtx h_ctx{};
  double* d_w64 = nullptr;
  double* d_lut64 = nullptr;   // exact vertical-pass values of the interior patterns
  long long* d_keys = nullptr;
  unsigned long long* d_count = nullptr;
  double* d_F[2] = {nullptr, nullptr};
  double* d_U = nullptr;
  double* d_T = nullptr;
  // host mirror of the state
  int mode = SRC_SCALED;
  int cur = 0, curF = 0;
  double scale = 1.0;
  bool field_valid = false;
  long long iteration = 0;
  bool converged = false;
  bool degenerate = false;
  bool prepared = false;
  long long fast_iters = 0, generic_iters = 0;
  // fast-path batch bookkeeping: output buffer of each launched iteration
  std::vector<std::pair<long long, int>> launched;
  // profiling
  bool prof = false;
  std::vector<cudaEvent_t> evpool;
  size_t evused = 0;
  // e0..e1 an update (upd), e1..e2 a partition + finalize (part); a fused
  // iteration records its pass as the update and finalize + fix as the rest
  struct EvRec { cudaEvent_t e0, e1, e2; bool upd, part; };
  std::vector<EvRec> evrec;
  double t_update = 0, t_part = 0;
  long long n_update = 0, n_part = 0;
  int grid_update = 0, grid_part = 0;
  int skip_uniform = 1;
  int nchunk = 1, nchunk_u = 1, nseg = 1, seg_chunks = 1;
  Geo gu{}, gu_all{}, gp{};   // work geometry: update, update with no interior, partition
  long long ni_upd = 0, nb_upd[2] = {0, 0}, ni_part = 0, nb_part = 0;
  long long ni_upd_split = 0;  // interior update units in split-warp mode
  int split_parts = 1;         // small images: 256/split_parts-column split-warp update units
  unsigned long long* d_work = nullptr;
  TilePartial* d_part_fin = nullptr;
  TilePartial* d_part_init = nullptr;
  unsigned long long work_next = 0;   // host mirror of the monotonic work counter
  cudaEvent_t t_begin = nullptr, t_end = nullptr;
  // row strips (multi-GPU): word-rows [own_lo, own_hi) are this rank's, the
  // others are halo copies of the neighbours' rows; the partition phase
  // reduces to one partial at strip_out and the ranks finalize together
  bool strip = false;
  bool fine = false;           // small image: per-pixel kernels (lse_fine.cuh)
  long long onestage_max = kOneStageMaxParts;   // tiled partition: one-stage finalize cutoff
  int own_lo = 0, own_hi = 0;
  TilePartial* strip_out = nullptr;
  bool strip_part = false, strip_ckpt = false;   // phases owed by the last update
  cudaEvent_t pev[2] = {nullptr, nullptr};       // profiling events of the pending update
  // speculative fused iteration (k_update_fused): eligible runs, fix list
  bool fused = false;
  bool strip_fused = false;      // the partials owed to lse_strip_finalize came from a fused pass
  FastParams strip_fp{};         // ... whose fix / redo launches follow that finalize
  int2* d_fix = nullptr;
  unsigned int fix_cap = 0;
  long long fused_iters = 0;
  // resident kernel (lse_resident.cuh): whole advance() calls of small images
  // in one launch -- one cluster (res_grid false) or a cooperative grid
  bool resident = false, res_grid = false;
  int res_ctas = 0, res_tasks = 0, res_nt = 1;
  TilePartial* d_res_parts = nullptr;
  unsigned int* d_sync = nullptr;
  long long resident_calls = 0;
  long long res_base_it = -1;    // first iteration base / buffer of the resident launches since collect
  int res_base_cur = 0;
};

namespace {

// models whose velocity uses the two region means (partition sums each pass)
bool two_mean(int model) {
  return model == LSE_MODEL_REGION || model == LSE_MODEL_ZHANG || model == LSE_MODEL_BANDS ||
         model == LSE_MODEL_CV;
}
bool is_bands(const lse_run* r) { return r->p.model == LSE_MODEL_BANDS; }
bool is_cv(const lse_run* r) { return r->p.model == LSE_MODEL_CV; }

// grow-only per-run scratch (its contents do not survive the call)
template <typename T>
int scratch(lse_run* r, size_t n, T** out) {
  const size_t bytes = std::max<size_t>(n * sizeof(T), 256);
  if (bytes > r->scratch_cap) {
    if (r->d_scratch) {
      cudaStreamSynchronize(r->st);
      cudaFree(r->d_scratch);
      r->d_scratch = nullptr;
      r->scratch_cap = 0;
    }
    TRY(dalloc(&r->d_scratch, bytes));
    r->scratch_cap = bytes;
  }
  *out = reinterpret_cast<T*>(r->d_scratch);
  return LSE_OK;
}

template <typename T>
int grow(lse_run* r, T** buf, size_t* cap, size_t n) {
  if (n <= *cap) return LSE_OK;
  if (*buf) {
    cudaStreamSynchronize(r->st);
    cudaFree(*buf);
    *buf = nullptr;
  }
  TRY(dalloc(buf, n));
  *cap = n;
  return LSE_OK;
}

int run_flag(lse_run* r, int** out) {
  if (!r->d_flag) TRY(dalloc(&r->d_flag, 4));
  *out = r->d_flag;
  return LSE_OK;
}

// LSE_BORDER_Q: row parts per border lane group (a power of two, 1 .. 16)
int parse_border_q(const char* v) {
  const int q = std::atoi(v);
  return q >= 16 ? 16 : q >= 8 ? 8 : q >= 4 ? 4 : q >= 2 ? 2 : 1;
}

// partials of the per-pixel partition: one per CTA of kFineCols columns up to
// kFineCtaParts CTAs, else one per state word
constexpr long long kFineCtaParts = 768;
bool fine_cta_parts(const lse_run* r) {
  return (long long)r->g.HR * ((r->W + kFineCols - 1) / kFineCols) <= kFineCtaParts;
}
long long fine_parts(const lse_run* r) {
  return fine_cta_parts(r) ? (long long)r->g.HR * ((r->W + kFineCols - 1) / kFineCols)
                           : (long long)r->g.HR * r->W;
}

FastParams fast_params(lse_run* r) {
  FastParams P{};
  P.pbits = r->d_P;
  P.mbits = r->d_M;
  P.data32 = r->d_data32;
  P.lut_t = r->d_lut_t;
  P.lut_s = r->d_lut_s;
  P.part = r->d_part;
  P.scal = r->d_scal;
  P.ctx = r->d_ctx;
  P.g = r->g;
  for (int d = 0; d < 8; ++d) {
    P.w32[d] = d <= r->R ? (float)r->h_ctx.w64[d] : 0.f;
    P.w2[d] = make_float2(P.w32[d], P.w32[d]);
  }
  P.dt32 = (float)r->p.dt;
  P.scale32 = (float)r->scale;
  P.skip_uniform = r->skip_uniform;
  P.nchunk = r->nchunk;
  P.nchunk_u = r->nchunk_u;
  P.nseg = r->nseg;
  P.seg_chunks = r->seg_chunks;
  P.work = r->d_work;
  P.gu = r->gu;
  P.gp = r->gp;
  P.own_lo = r->own_lo;
  P.own_hi = r->own_hi;
  P.chg = is_bands(r) ? r->d_chg : nullptr;
  P.ntiles = 1;
  P.fix_cnt = r->d_scal->fix_n;                  // (device address: no dereference)
  P.tile_hr = r->g.HR;
  P.tile_h = r->H;
  P.tile_words = (long long)r->g.HR * r->g.pitch_w;
  P.tile_data = (long long)r->H * r->g.data_pitch;
  return P;
}

// one wave of CTAs (ctas_per_sm resident per SM, the kernels' launch bound)
int fast_grid(long long warp_units, int ctas_per_sm = 4) {
  const long long ctas = (warp_units + 3) / 4;
  return (int)std::max<long long>(1, std::min<long long>(ctas, (long long)num_sms() * ctas_per_sm));
}

dim3 grid2(int W, int H, int bx = 128) { return dim3((W + bx - 1) / bx, H); }

int upload_ctx(lse_run* r) {
  r->h_ctx.scale = r->scale;
  CK(cudaMemcpyAsync(r->d_ctx, &r->h_ctx, sizeof(ExactCtx), cudaMemcpyHostToDevice, r->st));
  return LSE_OK;
}

int ensure_generic(lse_run* r) {
  if (r->d_F[0]) return LSE_OK;
  TRY(dalloc(&r->d_F[0], r->npx));
  TRY(dalloc(&r->d_F[1], r->npx));
  TRY(dalloc(&r->d_U, r->npx));
  TRY(dalloc(&r->d_T, r->npx));
  return LSE_OK;
}

// current state -> dense exact field in F[curF]
int materialize(lse_run* r) {
  if (r->field_valid) return LSE_OK;
  TRY(ensure_generic(r));
  TRY(upload_ctx(r));
  k_phi_from_bits<<<grid2(r->W, r->H), 128, 0, r->st>>>(r->d_bits[r->cur], r->d_F[r->curF],
                                                         r->d_ctx, r->mode);
  CKL();
  r->field_valid = true;
  return LSE_OK;
}

int launch_partition_abs(lse_run* r, int src, bool part, bool ckpt, bool mask_only,
                         uint32_t* mbits) {
  const double* field = src == SRC_FIELD ? r->d_F[r->curF] : nullptr;
  int grid = std::min(r->g.ntiles, num_sms() * 8);
  k_partition_abs<<<grid, r->nthr, 0, r->st>>>(field, r->d_bits[r->cur], r->d_ctx, src, r->d_P,
                                               mbits, part, ckpt, mask_only, r->d_part, r->g);
  CKL();
  return LSE_OK;
}


// partition sums / coefficients for the current state (region / zhang models)
int band_chain(lse_run* r, bool absolute, bool ckpt, long long it);

int prepare(lse_run* r) {
  if (r->prepared) return LSE_OK;
  TRY(upload_ctx(r));
  if (is_bands(r)) {
    if (r->mode != SRC_SCALED || r->field_valid)
      return fail(LSE_ERR_UNSUPPORTED, "multi-band runs start from seeds or signs");
    const dim3 gr((r->g.pitch_w + 1023) / 1024, r->g.HR);
    k_partition_init_bits<<<gr, 256, 0, r->st>>>(r->d_bits[r->cur], r->d_ctx, r->d_P,
                                                 r->d_part_init, r->g, r->own_lo, r->own_hi);
    CKL();
    TRY(band_chain(r, true, false, r->iteration));
  } else if (two_mean(r->p.model)) {
    if (r->mode == SRC_SCALED && !r->field_valid) {
      // +-s state: P = b; coalesced double-double sums, one partial per CTA
      const dim3 gr((r->g.pitch_w + 1023) / 1024, r->g.HR);
      k_partition_init_bits<<<gr, 256, 0, r->st>>>(r->d_bits[r->cur], r->d_ctx, r->d_P,
                                                   r->d_part_init, r->g, r->own_lo, r->own_hi);
      CKL();
      k_finalize<<<1, 1024, 0, r->st>>>(r->d_part_init, (int)(gr.x * gr.y), r->d_scal, 0, 1, 0,
                                        r->iteration);
      CKL();
    } else {
      TRY(launch_partition_abs(r, r->mode == SRC_FIELD ? SRC_FIELD : r->mode, true, false, false,
                               r->d_M));
      k_finalize<<<1, 1024, 0, r->st>>>(r->d_part, r->g.ntiles, r->d_scal, 0, 1, 0,
                                        r->iteration);
      CKL();
    }
  }
  r->prepared = true;
  return LSE_OK;
}

cudaEvent_t next_event(lse_run* r) {
  if (r->evused == r->evpool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    r->evpool.push_back(e);
  }
  return r->evpool[r->evused++];
}

// reserve the work-counter window of one dynamically scheduled launch
unsigned long long take_work(lse_run* r, long long units, int grid) {
  const unsigned long long base = r->work_next;
  r->work_next += (unsigned long long)units + (unsigned long long)grid * 4;
  return base;
}

#ifdef LSE_UNIT_TRACE
// Profiling builds: LSE_UNIT_TRACE_FILE=path appends, for launches
// [LSE_UNIT_TRACE_SKIP, +LSE_UNIT_TRACE_COUNT) of the fused kernels, one
// line per launch: "<kernel> <units> <nb> <grid> s0 e0 ... | exit a b
// stamps p q" (ns, relative to the launch's first CTA entry; p / q are
// global-timer stamps taken by 1-thread kernels just before and after).
// Nothing synchronizes between launches: the buffers are read back when the
// run next waits for the device (collect), so the pipeline is undisturbed.
__global__ void k_stamp(unsigned long long* slot) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  *slot = t;
}
struct TraceRec {
  unsigned long long* d;
  long long n, nb, cap;
  int grid;
  const char* name;
};
std::vector<TraceRec> g_traces;
long long g_trace_launch = 0;
constexpr long long kTrCta = 2 * 4096, kTrWarp = 4 * 4096;
unsigned long long* trace_begin_st(cudaStream_t st, long long n, int grid, const char* name,
                                   long long nb) {
  const char* f = std::getenv("LSE_UNIT_TRACE_FILE");
  if (!f) return nullptr;
  const long long skip = std::getenv("LSE_UNIT_TRACE_SKIP") ? std::atoll(std::getenv("LSE_UNIT_TRACE_SKIP")) : 0;
  const long long cnt = std::getenv("LSE_UNIT_TRACE_COUNT") ? std::atoll(std::getenv("LSE_UNIT_TRACE_COUNT")) : 4;
  const long long k = g_trace_launch++;
  if (k < skip || k >= skip + cnt) return nullptr;
  TraceRec t{nullptr, n, nb, 2 * n + kTrCta + kTrWarp + 2, grid, name};
  cudaMalloc(&t.d, t.cap * sizeof(unsigned long long));
  cudaMemsetAsync(t.d, 0, t.cap * sizeof(unsigned long long), st);
  k_stamp<<<1, 1, 0, st>>>(t.d + t.cap - 2);
  g_traces.push_back(t);
  return t.d;
}
void trace_after_st(cudaStream_t st, unsigned long long* d) {
  if (d) k_stamp<<<1, 1, 0, st>>>(d + g_traces.back().cap - 1);
}
unsigned long long* trace_begin(lse_run* r, long long n, int grid, const char* name, long long nb) {
  return trace_begin_st(r->st, n, grid, name, nb);
}
void trace_after(lse_run* r, unsigned long long* d) { trace_after_st(r->st, d); }
void trace_flush() {
  if (g_traces.empty()) return;
  FILE* fp = std::fopen(std::getenv("LSE_UNIT_TRACE_FILE"), "a");
  for (auto& t : g_traces) {
    std::vector<unsigned long long> h(t.cap);
    cudaMemcpy(h.data(), t.d, t.cap * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    cudaFree(t.d);
    if (!fp) continue;
    const long long m = t.n + t.grid;
    unsigned long long t0 = ~0ull;
    for (long long u = 0; u < m; ++u) if (h[2 * u] && h[2 * u] < t0) t0 = h[2 * u];
    std::fprintf(fp, "%s %lld %lld %d", t.name, t.n, t.nb, t.grid);
    for (long long u = 0; u < m; ++u)
      std::fprintf(fp, " %lld %lld", h[2 * u] ? (long long)(h[2 * u] - t0) : -1,
                   h[2 * u + 1] ? (long long)(h[2 * u + 1] - t0) : -1);
    unsigned long long emax = 0, emin = ~0ull;
    for (long long w = 0; w < 4 * t.grid; ++w) {
      const unsigned long long e = h[2 * t.n + kTrCta + w];
      if (e) { emax = e > emax ? e : emax; emin = e < emin ? e : emin; }
    }
    std::fprintf(fp, " | exit %lld %lld stamps %lld %lld\n", (long long)(emin - t0),
                 (long long)(emax - t0), (long long)h[t.cap - 2] - (long long)t0,
                 (long long)h[t.cap - 1] - (long long)t0);
  }
  if (fp) std::fclose(fp);
  g_traces.clear();
}
#endif

template <int R, int MODEL, int SRC>
int launch_update(lse_run* r, FastParams P) {
  if (r->fine) {
    const dim3 g((r->W + kFineCols - 1) / kFineCols, r->g.HR);
    TRY(launch_pdl(k_update_fine<R, MODEL, SRC>, g, 32 * kFineCols, r->st, P));
    return LSE_OK;
  }
  const int ns = r->split_parts;
  const long long n = r->nb_upd[0] + (ns > 1 ? r->ni_upd_split : r->ni_upd);
  const int g = fast_grid(n, kUpdateCtasPerSm);
  P.work_base = take_work(r, n, g);
#ifdef LSE_UNIT_TRACE
  P.trace = trace_begin(r, n, g, "update", r->nb_upd[0]);
#endif
  if (ns == 4) TRY(launch_pdl(k_update<R, MODEL, SRC, false, 4>, g, kThreads, r->st, P));
  else if (ns == 2) TRY(launch_pdl(k_update<R, MODEL, SRC, false, 2>, g, kThreads, r->st, P));
  else TRY(launch_pdl(k_update<R, MODEL, SRC, false, 1>, g, kThreads, r->st, P));
#ifdef LSE_UNIT_TRACE
  trace_after(r, P.trace);
#endif
  return LSE_OK;
}

template <int R, bool PART, bool CKPT, bool MASKONLY>
int launch_partition(lse_run* r, FastParams P) {
  const bool fine = r->fine && !MASKONLY;
  const long long n = fine ? fine_parts(r) : r->nb_part + r->ni_part;
  if (fine) {
    const dim3 gf((r->W + kFineCols - 1) / kFineCols, r->g.HR);
    // one partial per CTA and a single-stage finalize on small images
    // (256^2: 13.2 -> 11.5 us per iteration); per-word partials and the
    // two stages below beyond kFineCtaParts CTAs (512^2: 27.7 vs 29.0 us)
    if (fine_cta_parts(r)) {
      TRY(launch_pdl(k_partition_fine<R, PART, CKPT, true>, gf, 32 * kFineCols, r->st, P));
    } else {
      TRY(launch_pdl(k_partition_fine<R, PART, CKPT, false>, gf, 32 * kFineCols, r->st, P));
    }
    if (fine_cta_parts(r) && !is_bands(r)) {
      PartRanges RF{{r->d_part, r->d_part, r->d_part}, {(int)n, 0, 0}};
      TRY(launch_pdl(k_finalize_run, 1, 64, r->st, RF, r->d_scal, PART ? 1 : 0, CKPT ? 1 : 0,
                     (long long)P.iter, 0));
      return LSE_OK;
    }
  } else {
  const int g = fast_grid(n, kPartitionCtasPerSm);
  P.work_base = take_work(r, n, g);
#ifdef LSE_UNIT_TRACE
  P.trace = MASKONLY ? nullptr : trace_begin(r, n, g, "partition", r->nb_part);
#endif
  TRY(launch_pdl(k_partition<R, PART, CKPT, MASKONLY, false>, g, kThreads, r->st, P));
#ifdef LSE_UNIT_TRACE
  trace_after(r, P.trace);
#endif
  }
  if (!MASKONLY) {
    // two-stage fixed-order reduction of all unit partials -> the next
    // update's coefficients (64 CTAs reduce contiguous slices, 1 CTA the rest)
    PartRanges R3{{r->d_part, r->d_part, r->d_part}, {(int)n, 0, 0}};
    if (!is_bands(r) && !r->strip && n <= r->onestage_max) {
      // few partials (small images): a single-stage finalize, one launch less
      TRY(launch_pdl(k_finalize_run, 1, 64, r->st, R3, r->d_scal, PART ? 1 : 0, CKPT ? 1 : 0,
                     (long long)P.iter, 0));
      return LSE_OK;
    }
    if (!is_bands(r)) {
      TRY(launch_pdl(k_finalize_stage1, kFinSlices, 256, r->st, R3, r->d_part_fin,
                     (const Scalars*)r->d_scal));
    }
    PartRanges R1{{r->d_part_fin, r->d_part_fin, r->d_part_fin}, {kFinSlices, 0, 0}};
    if (is_bands(r)) {
      TRY(band_chain(r, false, CKPT, P.iter));
      return LSE_OK;
    }
    if (r->strip) {
      // row strips: this rank's contribution; the ranks exchange it and
      // finalize together (lse_strip_finalize)
      k_reduce_to_one<<<1, 256, 0, r->st>>>(R1, r->strip_out, r->d_scal, 1);
    } else {
      TRY(launch_pdl(k_finalize_run, 1, 64, r->st, R1, r->d_scal, PART ? 1 : 0, CKPT ? 1 : 0,
                     (long long)P.iter, 0));
    }
    CKL();
  }
  return LSE_OK;
}

// One fast iteration in two phases: PH_UPDATE launches the update of
// iteration `it` (b^n -> b^{n+1}) and makes b^{n+1} the current state;
// PH_PARTITION launches the partition / checkpoint pass over it.  A single-GPU
// run does both back to back; a row strip exchanges its halo rows in between.
enum Phase : int { PH_BOTH = 0, PH_UPDATE = 1, PH_PARTITION = 2 };

template <int R, int MODEL>
int launch_fast_R(lse_run* r, long long it, bool ckpt, int phase) {
  FastParams P = fast_params(r);
  P.iter = it;
  set_check(P, it);
  if (phase != PH_PARTITION) {
    P.bits_in = r->d_bits[r->cur];
    P.bits_out = r->d_bits[r->cur ^ 1];
    if (r->prof) {
      r->pev[0] = next_event(r);
      r->pev[1] = next_event(r);
      cudaEventRecord(r->pev[0], r->st);
    }
    if (r->mode == SRC_SCALED) TRY((launch_update<R, MODEL, SRC_SCALED>(r, P)));
    else TRY((launch_update<R, MODEL, SRC_SMOOTH>(r, P)));
    if (r->prof) cudaEventRecord(r->pev[1], r->st);
    r->cur ^= 1;
    r->mode = SRC_SMOOTH;
    r->field_valid = false;
    r->launched.emplace_back(it, r->cur);
    r->strip_part = MODEL == REGION || ckpt;
    r->strip_ckpt = ckpt;
    if (phase == PH_UPDATE) {
      if (r->prof) r->evrec.push_back({r->pev[0], r->pev[1], r->pev[1], true, false});
      return LSE_OK;
    }
  } else if (r->prof) {
    r->pev[0] = r->pev[1] = next_event(r);       // partition phase alone
    cudaEventRecord(r->pev[1], r->st);
  }
  P.bits_in = r->d_bits[r->cur];
  bool launched_part = false;
  if (MODEL == REGION) {
    if (ckpt) TRY((launch_partition<R, true, true, false>(r, P)));
    else TRY((launch_partition<R, true, false, false>(r, P)));
    launched_part = true;
  } else if (ckpt) {
    TRY((launch_partition<R, false, true, false>(r, P)));
    launched_part = true;
  }
  if (r->prof) {
    cudaEvent_t e2 = next_event(r);
    cudaEventRecord(e2, r->st);
    r->evrec.push_back({r->pev[0], r->pev[1], e2, phase != PH_PARTITION, launched_part});
  }
  return LSE_OK;
}

template <int MODEL>
int launch_fast_model(lse_run* r, long long it, bool ckpt, int phase) {
  switch (r->R) {
    case 1: return launch_fast_R<1, MODEL>(r, it, ckpt, phase);
    case 2: return launch_fast_R<2, MODEL>(r, it, ckpt, phase);
    case 3: return launch_fast_R<3, MODEL>(r, it, ckpt, phase);
    case 4: return launch_fast_R<4, MODEL>(r, it, ckpt, phase);
  }
  return fail(LSE_ERR_ARG, "unsupported template radius");
}

int launch_fast(lse_run* r, long long it, bool ckpt, int phase = PH_BOTH) {
  // the mean-separation model differs only in its finalize coefficients
  if (two_mean(r->p.model)) return launch_fast_model<REGION>(r, it, ckpt, phase);
  return launch_fast_model<EDGE>(r, it, ckpt, phase);
}

// One speculative fused iteration (lse_fast.cuh, k_update_fused): the
// partition of the current state b^{it-1} (its checkpoint when ckpt_prev)
// and the update it-1 -> it in one pass, then the finalize of iteration it-1
// (true coefficients of update it, prediction check) and k_spec_fix (fix list
// or full redo).  Only after an update whose partition is still owed.
// the fix-list decision and the redo pass after a fused pass's finalize
template <int R>
int launch_spec_tail(lse_run* r, const FastParams& P) {
  TRY(launch_pdl(k_spec_fix<R, false>, num_sms(), 256, r->st, P));
  FastParams Q = P;                              // the redo pass has its own work counter
  Q.work = &r->d_scal->work2;
  Q.work_base = 0;
  const long long n = r->nb_upd[0] + r->ni_upd;
  TRY(launch_pdl(k_spec_redo<R, false>, fast_grid(n, kUpdateCtasPerSm), kThreads, r->st, Q));
  return LSE_OK;
}

template <int R>
int launch_fused_R(lse_run* r, long long it, bool ckpt_prev, TilePartial* strip_out = nullptr) {
  FastParams P = fast_params(r);
  P.iter = it - 1;
  set_check(P, it);
  P.bits_in = r->d_bits[r->cur];
  P.bits_out = r->d_bits[r->cur ^ 1];
  P.fix = r->d_fix;
  P.fix_cap = r->fix_cap;
  P.fix_par = (int)(it & 1);
  const long long n = r->nb_upd[0] + r->ni_upd;
  const int g = fast_grid(n, kFusedCtasPerSm);
  P.work_base = take_work(r, n, g);
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (r->prof) {
    e0 = next_event(r);
    e1 = next_event(r);
    cudaEventRecord(e0, r->st);
  }
  constexpr size_t smem = fused_smem_bytes<R>();
#ifdef LSE_UNIT_TRACE
  P.trace = trace_begin(r, n, g, "fused", r->nb_upd[0]);
#endif
  if (ckpt_prev) {
    TRY(prepare_smem(k_update_fused<R, true, false>, smem));
    TRY(launch_pdl_smem(k_update_fused<R, true, false>, g, kThreads, smem, r->st, P));
  } else {
    TRY(prepare_smem(k_update_fused<R, false, false>, smem));
    TRY(launch_pdl_smem(k_update_fused<R, false, false>, g, kThreads, smem, r->st, P));
  }
#ifdef LSE_UNIT_TRACE
  trace_after(r, P.trace);
#endif
  if (r->prof) cudaEventRecord(e1, r->st);
  PartRanges R3{{r->d_part, r->d_part, r->d_part}, {(int)n, 0, 0}};
  const int spec = 1 + P.fix_par;
  if (strip_out) {
    // row strips: this rank's partial of the partition of b^{it-1}; the ranks
    // exchange them, then lse_strip_finalize checks the prediction and
    // launches the fix / redo pass (launch_spec_tail)
    TRY(launch_pdl(k_finalize_stage1, kFusedFinSlices, 256, r->st, R3, r->d_part_fin,
                   (const Scalars*)r->d_scal));
    PartRanges R1{{r->d_part_fin, r->d_part_fin, r->d_part_fin}, {kFusedFinSlices, 0, 0}};
    k_reduce_to_one<<<1, 256, 0, r->st>>>(R1, strip_out, r->d_scal, 1);
    CKL();
    r->strip_fused = true;
    r->strip_fp = P;
  } else if (n <= r->onestage_max) {
    TRY(launch_pdl(k_finalize_run, 1, 64, r->st, R3, r->d_scal, 1, ckpt_prev ? 1 : 0, it - 1,
                   spec));
  } else {
    // (one partial per unit, ~131 k on C5: a wider first stage)
    TRY(launch_pdl(k_finalize_stage1, kFusedFinSlices, 256, r->st, R3, r->d_part_fin,
                   (const Scalars*)r->d_scal));
    PartRanges R1{{r->d_part_fin, r->d_part_fin, r->d_part_fin}, {kFusedFinSlices, 0, 0}};
    TRY(launch_pdl(k_finalize_run, 1, 64, r->st, R1, r->d_scal, 1, ckpt_prev ? 1 : 0, it - 1,
                   spec));
  }
  if (!strip_out) TRY(launch_spec_tail<R>(r, P));
  if (r->prof) {
    cudaEvent_t e2 = next_event(r);
    cudaEventRecord(e2, r->st);
    r->evrec.push_back({e0, e1, e2, true, true});
  }
  r->cur ^= 1;
  r->mode = SRC_SMOOTH;
  r->field_valid = false;
  r->launched.emplace_back(it, r->cur);
  r->fused_iters++;
  return LSE_OK;
}

int launch_fused(lse_run* r, long long it, bool ckpt_prev, TilePartial* strip_out = nullptr) {
  switch (r->R) {
    case 1: return launch_fused_R<1>(r, it, ckpt_prev, strip_out);
    case 2: return launch_fused_R<2>(r, it, ckpt_prev, strip_out);
    case 3: return launch_fused_R<3>(r, it, ckpt_prev, strip_out);
    case 4: return launch_fused_R<4>(r, it, ckpt_prev, strip_out);
  }
  return fail(LSE_ERR_ARG, "unsupported template radius");
}

int launch_spec_tail_any(lse_run* r, const FastParams& P) {
  switch (r->R) {
    case 1: return launch_spec_tail<1>(r, P);
    case 2: return launch_spec_tail<2>(r, P);
    case 3: return launch_spec_tail<3>(r, P);
    case 4: return launch_spec_tail<4>(r, P);
  }
  return fail(LSE_ERR_ARG, "unsupported template radius");
}

// wait for the device, fold profiling events, detect convergence
int collect(lse_run* r) {
  unsigned long long work = 0;
  CK(cudaMemcpyAsync(r->h_scal, r->d_scal, sizeof(Scalars), cudaMemcpyDeviceToHost, r->st));
  CK(cudaMemcpyAsync(&work, r->d_work, sizeof(work), cudaMemcpyDeviceToHost, r->st));
  CK(cudaStreamSynchronize(r->st));
#ifdef LSE_UNIT_TRACE
  trace_flush();
#endif
  // every dynamically scheduled launch must have made exactly its reserved
  // number of grabs (units + one failing grab per warp) unless it was stopped
  if (!r->h_scal->stop && work != r->work_next) {
    char msg[128];
    std::snprintf(msg, sizeof(msg), "work-counter mismatch: device %llu, expected %llu", work,
                  r->work_next);
    return fail(LSE_ERR_CUDA, msg);
  }
  if (r->prof) {
    for (auto& e : r->evrec) {
      float ms = 0.f;
      if (e.upd) {
        cudaEventElapsedTime(&ms, e.e0, e.e1);
        r->t_update += ms;
        r->n_update++;
      }
      if (e.part) {
        cudaEventElapsedTime(&ms, e.e1, e.e2);
        r->t_part += ms;
        r->n_part++;
      }
    }
  }
  r->evrec.clear();
  r->evused = 0;
  const Scalars& s = *r->h_scal;
  r->degenerate = s.degenerate != 0;
  if (s.converged && !r->converged) {
    r->converged = true;
    r->iteration = s.converged_iter;
    for (auto& pr : r->launched)
      if (pr.first == s.converged_iter) r->cur = pr.second;
    // resident launches alternate the two state buffers from their base
    if (r->res_base_it >= 0)
      r->cur = r->res_base_cur ^ (int)((s.converged_iter - r->res_base_it) & 1);
  }
  r->res_base_it = -1;
  r->launched.clear();
  return LSE_OK;
}

bool fp32_ok(lse_run* r) {
  if (is_cv(r)) return false;                    // continuous field: the fp64 path
  if (r->R < 1 || r->R > 4) return false;
  if (!(r->p.dt <= 1e6)) return false;
  if (two_mean(r->p.model) && !(r->img_absmax <= 1e6)) return false;
  if (r->p.model == LSE_MODEL_ZHANG && !(std::fabs(r->p.nu) <= 1e6)) return false;
  if (r->mode == SRC_SCALED && !(r->scale >= 1e-3 && r->scale <= 1e6)) return false;
  // +-s in fp32: exact, or its rounding (s 2^-24) far inside the phi bound
  if (r->mode == SRC_SCALED && (double)(float)r->scale != r->scale && !(r->scale <= 4.0)) return false;
  return true;
}

// ------------------------------------------------------- resident kernel
// (lse_resident.cuh) whole advance() calls of small single images in one
// launch.  LSE_RESIDENT=0 keeps the per-iteration launches, 2 forces the
// cooperative-grid barrier where one cluster would do (tests / A-B).
template <int R, int MODEL, bool GRID, int NT>
int resident_launch_k(lse_run* r, const FastParams& P, const ResidentArgs& A) {
  auto kern = k_resident<R, MODEL, GRID, NT>;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)r->res_ctas);
  cfg.blockDim = dim3(kResThreads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = r->st;
  cudaLaunchAttribute at[1];
  if (GRID) {
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
  } else {
    if (r->res_ctas > 8)
      CK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)r->res_ctas;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
  }
  cfg.attrs = at;
  cfg.numAttrs = 1;
  CK(cudaLaunchKernelEx(&cfg, kern, P, A));
  CKL();
  return LSE_OK;
}

template <int R, int MODEL>
int resident_launch_rm(lse_run* r, const FastParams& P, const ResidentArgs& A) {
  if (r->res_nt > 1) {                           // (several tasks per warp: grid launches only)
    if (r->res_nt == 2) return resident_launch_k<R, MODEL, true, 2>(r, P, A);
    return resident_launch_k<R, MODEL, true, 3>(r, P, A);
  }
  if (r->res_grid) return resident_launch_k<R, MODEL, true, 1>(r, P, A);
  return resident_launch_k<R, MODEL, false, 1>(r, P, A);
}

template <int MODEL>
int resident_launch_m(lse_run* r, const FastParams& P, const ResidentArgs& A) {
  switch (r->R) {
    case 1: return resident_launch_rm<1, MODEL>(r, P, A);
    case 2: return resident_launch_rm<2, MODEL>(r, P, A);
    case 3: return resident_launch_rm<3, MODEL>(r, P, A);
    case 4: return resident_launch_rm<4, MODEL>(r, P, A);
  }
  return fail(LSE_ERR_ARG, "unsupported template radius");
}

// can this run's launch shape be resident on the device?  (decided once)
template <bool GRID>
int resident_capacity(int ctas) {
  // occupancy of the widest instantiation stands for all (same launch bounds)
  auto kern = k_resident<4, REGION, GRID, 1>;
  if (GRID) {
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kResThreads, 0) != cudaSuccess)
      return 0;
    return per_sm * num_sms();
  }
  if (ctas > 8 &&
      cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)ctas);
  cfg.blockDim = dim3(kResThreads);
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)ctas;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int nclusters = 0;
  if (cudaOccupancyMaxActiveClusters(&nclusters, kern, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return nclusters > 0 ? ctas : 0;
}

constexpr int kResMaxTasksPerWarp = 3;           // k_resident NT

void resident_setup(lse_run* r) {
  r->resident = false;
  int mode = 1;
  if (const char* v = std::getenv("LSE_RESIDENT")) {
    mode = std::atoi(v);
  } else {
    // a knob that selects a variant of the per-iteration kernels (tests, A/B)
    // asks for those kernels
    for (const char* k : {"LSE_FINE_MAX_PX", "LSE_SPLIT_PARTS", "LSE_BORDER_Q", "LSE_FUSED",
                          "LSE_FIX_CAP", "LSE_ONESTAGE_MAX_PARTS"})
      if (std::getenv(k)) mode = 0;
  }
#ifdef LSE_CHECK_BOUND
  mode = 0;                                      // validation builds certify the per-iteration kernels
#endif
  if (mode == 0 || is_bands(r) || is_cv(r) || r->strip || r->R < 1 || r->R > 4) return;
  // up to kResMaxTasksPerWarp tasks per warp of a full cooperative grid
  // (~1.8 Mpx); larger images run the tiled kernels.  LSE_RESIDENT_MAX_PX
  // lowers the limit (A/B against the tiled / per-pixel kernels).
  if (const char* v = std::getenv("LSE_RESIDENT_MAX_PX"))
    if (r->npx > std::atoll(v)) return;
  const int ncb = (r->W + kResCols - 1) / kResCols;
  const long long tasks = (long long)r->g.HR * ncb;
  long long ctas = (tasks + kResWarps - 1) / kResWarps;
  int nt = 1;
  bool grid = mode == 2 || ctas > kResClusterMax;
  if (!grid && resident_capacity<false>((int)ctas) < ctas) grid = true;
  if (grid) {
    const int cap = resident_capacity<true>((int)ctas);
    if (cap <= 0) return;
    if (ctas > cap) {
      nt = (int)((ctas + cap - 1) / cap);
      if (nt > kResMaxTasksPerWarp) return;
      ctas = (ctas + nt - 1) / nt;               // balanced: every warp has nt or nt-1 tasks
    }
  }
  r->resident = true;
  r->res_grid = grid;
  r->res_ctas = (int)ctas;
  r->res_tasks = (int)tasks;
  r->res_nt = nt;
}

// is the whole call [it0+1, it0+steps] on the fast binary-state path?
bool fp32_ok(lse_run* r);
bool resident_now(lse_run* r) {
  return r->resident && r->p.reinit_period == 1 && r->p.reg_period == 1 &&
         r->mode != SRC_FIELD && fp32_ok(r);
}

int launch_resident(lse_run* r, long long steps) {
  if (!r->d_res_parts) {
    TRY(dalloc(&r->d_res_parts, (size_t)r->res_ctas));
    TRY(dalloc(&r->d_sync, 64));
  }
  FastParams P = fast_params(r);
  ResidentArgs A{};
  A.bits[0] = r->d_bits[0];
  A.bits[1] = r->d_bits[1];
  A.cur0 = r->cur;
  A.scaled = r->mode == SRC_SCALED ? 1 : 0;
  A.it0 = r->iteration;
  A.steps = steps;
  A.cce = r->p.conv_check_every;
  A.ncb = (r->W + kResCols - 1) / kResCols;
  A.ntasks = r->res_tasks;
  A.parts = r->d_res_parts;
  A.sync = r->d_sync;
  if (r->res_grid) CK(cudaMemsetAsync(r->d_sync, 0, 64 * sizeof(unsigned int), r->st));
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (r->prof) {
    e0 = next_event(r);
    e1 = next_event(r);
    cudaEventRecord(e0, r->st);
  }
  if (two_mean(r->p.model)) TRY(resident_launch_m<REGION>(r, P, A));
  else TRY(resident_launch_m<EDGE>(r, P, A));
  if (r->prof) {
    cudaEventRecord(e1, r->st);
    r->evrec.push_back({e0, e1, e1, true, false});
  }
  if (r->res_base_it < 0) {                      // (collect: the buffer of a converged iteration)
    r->res_base_it = A.it0;
    r->res_base_cur = A.cur0;
  }
  r->cur = A.cur0 ^ (int)(steps & 1);
  r->mode = SRC_SMOOTH;
  r->field_valid = false;
  r->iteration = A.it0 + steps;
  r->fast_iters += steps;
  r->resident_calls++;
  return LSE_OK;
}

// -signed_distance(f > 0) of a dense field (engine.py:161-165) into out (may
// alias f): two exact distance transforms (kernels.py:118-133).
int edt_buffers(lse_run* r) {
  if (r->d_edt_g) return LSE_OK;
  TRY(dalloc(&r->d_edt_g, r->npx));
  TRY(dalloc(&r->d_edt_v, r->npx));
  TRY(dalloc(&r->d_edt_zn, (size_t)r->H * (r->W + 1)));
  TRY(dalloc(&r->d_edt_zd, (size_t)r->H * (r->W + 1)));
  TRY(dalloc(&r->d_dist[0], r->npx));
  TRY(dalloc(&r->d_dist[1], r->npx));
  return LSE_OK;
}

int neg_signed_distance(cudaStream_t st, const double* f, double* out, int H, int W,
                        long long* g, int* v, long long* zn, long long* zd, double* d0,
                        double* d1) {
  for (int pos = 0; pos < 2; ++pos) {
    k_edt_cols<<<(W + 127) / 128, 128, 0, st>>>(f, H, W, pos, g);
    CKL();
    k_edt_rows<<<(H + 127) / 128, 128, 0, st>>>(g, H, W, v, zn, zd, pos ? d1 : d0);
    CKL();
  }
  k_sdf_combine<<<num_sms() * 8, 256, 0, st>>>(f, d0, d1, out, (long long)H * W);
  CKL();
  return LSE_OK;
}

int run_neg_sdf(lse_run* r, const double* f, double* out) {
  TRY(edt_buffers(r));
  return neg_signed_distance(r->st, f, out, r->H, r->W, r->d_edt_g, r->d_edt_v, r->d_edt_zn,
                             r->d_edt_zd, r->d_dist[0], r->d_dist[1]);
}

double key_to_double(long long q) {
  const long long b = q ^ ((q >> 63) & 0x7fffffffffffffffLL);
  double d;
  std::memcpy(&d, &b, 8);
  return d;
}

// min / max of a dense field (re-init guard: both signs present?)
int field_minmax(lse_run* r, const double* f, double* mn, double* mx) {
  long long init[3] = {LLONG_MAX, LLONG_MIN, LLONG_MIN};
  CK(cudaMemcpyAsync(r->d_keys, init, sizeof(init), cudaMemcpyHostToDevice, r->st));
  k_minmax<<<std::min(r->H, num_sms() * 8), 256, 0, r->st>>>(nullptr, f, r->H, r->W, r->W,
                                                            r->d_keys);
  CKL();
  long long k[3];
  CK(cudaMemcpyAsync(k, r->d_keys, sizeof(k), cudaMemcpyDeviceToHost, r->st));
  CK(cudaStreamSynchronize(r->st));
  *mn = key_to_double(k[0]);
  *mx = key_to_double(k[1]);
  return LSE_OK;
}

int generic_iteration(lse_run* r, long long it, bool reinit_now, bool reg_now, bool ckpt) {
  if (is_bands(r))
    return fail(LSE_ERR_UNSUPPORTED, "multi-band runs need the binary-state fast path "
                                     "(reinit_period = reg_period = 1, 3 <= ts_reg <= 9)");
  TRY(ensure_generic(r));
  TRY(materialize(r));
  CK(cudaMemsetAsync(&r->d_scal->nonfinite, 0, sizeof(int), r->st));
  const double* phi = r->d_F[r->curF];
  const bool cv = is_cv(r);
  if (cv) {
    // models.py:122-141 on the fp64 field
    if (!r->d_px) {
      TRY(dalloc(&r->d_px, r->npx));
      TRY(dalloc(&r->d_py, r->npx));
      TRY(dalloc(&r->d_mag, r->npx));
    }
    k_gradient<<<grid2(r->W, r->H), 128, 0, r->st>>>(phi, r->H, r->W, r->d_px, r->d_py, r->d_mag);
    CKL();
    k_cv_update<<<grid2(r->W, r->H), 128, 0, r->st>>>(
        phi, r->d_px, r->d_py, r->d_mag, r->d_U, r->H, r->W, r->d_data32, r->d_data64,
        r->g.data_pitch, r->d_scal, r->p.dt, r->p.mu, 1e-10);
  } else if (two_mean(r->p.model))
    k_gen_update<REGION><<<grid2(r->W, r->H), 128, 0, r->st>>>(
        phi, r->d_U, r->H, r->W, r->d_data32, r->d_data64, r->g.data_pitch, r->d_scal, r->p.dt);
  else
    k_gen_update<EDGE><<<grid2(r->W, r->H), 128, 0, r->st>>>(
        phi, r->d_U, r->H, r->W, r->d_data32, r->d_data64, r->g.data_pitch, r->d_scal, r->p.dt);
  CKL();
  // the reference skips reinit/smoothing when u is not finite and raises
  // either way; computing them regardless is harmless (phi is not committed)
  if (reinit_now && cv) {
    // rebuild the distance field around the zero set when both classes exist
    // (engine.py:161-165); otherwise u is kept as it is
    double mn, mx;
    TRY(field_minmax(r, r->d_U, &mn, &mx));
    if (mx > 0.0 && mn <= 0.0) TRY(run_neg_sdf(r, r->d_U, r->d_U));
  } else if (reinit_now) {
    k_binarize<<<num_sms() * 8, 256, 0, r->st>>>(r->d_U, r->d_U, r->npx);
    CKL();
  }
  double* out = r->d_F[r->curF ^ 1];
  if (reg_now) {
    k_corr<0><<<grid2(r->W, r->H), 128, 0, r->st>>>(r->d_U, r->d_T, r->H, r->W, r->d_w64, r->R);
    CKL();
    k_corr<1><<<grid2(r->W, r->H), 128, 0, r->st>>>(r->d_T, out, r->H, r->W, r->d_w64, r->R);
    CKL();
  } else {
    CK(cudaMemcpyAsync(out, r->d_U, r->npx * sizeof(double), cudaMemcpyDeviceToDevice, r->st));
  }
  k_check_finite<<<num_sms() * 8, 256, 0, r->st>>>(out, r->npx, r->d_scal);
  CKL();
  int nonfinite = 0;
  CK(cudaMemcpyAsync(&r->h_scal->nonfinite, &r->d_scal->nonfinite, sizeof(int),
                     cudaMemcpyDeviceToHost, r->st));
  CK(cudaStreamSynchronize(r->st));
  nonfinite = r->h_scal->nonfinite;
  if (nonfinite) return LSE_ERR_INSTABILITY;   // engine.py:172-173; phi untouched
  // commit
  r->curF ^= 1;
  r->mode = SRC_FIELD;
  r->field_valid = true;
  if (!cv && reinit_now && reg_now && r->R >= 1 && r->R <= 4) {
    // phi = G * b exactly: carry the state as bits from here on
    k_pack_bits<<<dim3((r->g.pitch_w + 127) / 128, r->g.HR), 128, 0, r->st>>>(r->d_U,
                                                                              r->d_bits[r->cur],
                                                                              r->g);
    CKL();
    r->mode = SRC_SMOOTH;
  }
  const bool region = two_mean(r->p.model);
  if (region || ckpt) {
    // partition from the exact field (field_valid => F[curF] is phi^{n+1})
    const double* field = r->d_F[r->curF];
    int grid = std::min(r->g.ntiles, num_sms() * 8);
    k_partition_abs<<<grid, r->nthr, 0, r->st>>>(field, r->d_bits[r->cur], r->d_ctx, SRC_FIELD,
                                                 r->d_P, r->d_M, region, ckpt, 0, r->d_part, r->g);
    CKL();
    k_finalize<<<1, 1024, 0, r->st>>>(r->d_part, r->g.ntiles, r->d_scal, 0, region, ckpt, it);
    CKL();
  }
  r->iteration = it;
  r->generic_iters++;
  TRY(collect(r));
  return LSE_OK;
}

// multi-band runs: the pass after each partition -- band sums over the
// changed pixels (or all pixels), per-band means, the data term D of every
// pixel (fp32 plane for the fused kernels) and its peak, the coefficients
int band_chain(lse_run* r, bool absolute, bool ckpt, long long it) {
  const dim3 gr((r->g.pitch_w + 1023) / 1024, r->g.HR);
  const int n = (int)(r->fine ? fine_parts(r) : r->nb_part + r->ni_part);
  PartRanges M{{r->d_part, r->d_part, r->d_part}, {ckpt ? n : 0, 0, 0}};
  unsigned long long* cnt = r->d_pmax;          // [0]: band sums, [1]: band peak arrivals
  if (absolute)
    TRY(launch_pdl(k_band_sums<true>, gr, 256, r->st, (const uint32_t*)nullptr,
                   (const uint32_t*)r->d_P, (const ExactCtx*)r->d_ctx, r->d_bpart, r->g,
                   r->d_scal, cnt, M, ckpt ? 1 : 0, it));
  else
    TRY(launch_pdl(k_band_sums<false>, gr, 256, r->st, (const uint32_t*)r->d_chg,
                   (const uint32_t*)r->d_P, (const ExactCtx*)r->d_ctx, r->d_bpart, r->g,
                   r->d_scal, cnt, M, ckpt ? 1 : 0, it));
  // peak pass: one wave -- as many CTAs as fit on the SMs at once (a partial
  // second wave measured ~2 % slower per iteration on C3), each a 1024-column
  // block of every gy-th row
  const int gx = (r->W + 1023) / 1024;
  int peak_cps = 0;
  switch (r->nbands) {
    case 1: cudaOccupancyMaxActiveBlocksPerMultiprocessor(&peak_cps, k_band_peak<1>, 256, 0); break;
    case 2: cudaOccupancyMaxActiveBlocksPerMultiprocessor(&peak_cps, k_band_peak<2>, 256, 0); break;
    case 3: cudaOccupancyMaxActiveBlocksPerMultiprocessor(&peak_cps, k_band_peak<3>, 256, 0); break;
    default: cudaOccupancyMaxActiveBlocksPerMultiprocessor(&peak_cps, k_band_peak<4>, 256, 0); break;
  }
  if (const char* v = std::getenv("LSE_PEAK_CPS")) peak_cps = std::atoi(v);
  peak_cps = std::max(1, peak_cps);
  const int gy = std::max(1, std::min(r->H, num_sms() * peak_cps / gx));
  const dim3 gp(gx, gy);
  const ExactCtx* cctx = r->d_ctx;
  switch (r->nbands) {
    case 1: TRY(launch_pdl(k_band_peak<1>, gp, 256, r->st, cctx, r->d_scal, r->d_data32, cnt + 1, r->g)); break;
    case 2: TRY(launch_pdl(k_band_peak<2>, gp, 256, r->st, cctx, r->d_scal, r->d_data32, cnt + 1, r->g)); break;
    case 3: TRY(launch_pdl(k_band_peak<3>, gp, 256, r->st, cctx, r->d_scal, r->d_data32, cnt + 1, r->g)); break;
    default: TRY(launch_pdl(k_band_peak<4>, gp, 256, r->st, cctx, r->d_scal, r->d_data32, cnt + 1, r->g)); break;
  }
  return LSE_OK;
}

// multi-band image: n_bands planes (band-major, each H x W), float32 or float64
int upload_bands(lse_run* r, const void* image, int fmt) {
  if (fmt != LSE_IMAGE_F32 && fmt != LSE_IMAGE_F64)
    return fail(LSE_ERR_ARG, "multi-band images are float32 or float64 planes");
  const int H = r->H, W = r->W, K = r->nbands;
  const long long pitch = r->g.data_pitch, stride = pitch * H;
  int* d_flag = nullptr;
  double* tmp64 = nullptr;
  TRY(run_flag(r, &d_flag));
  CK(cudaMemsetAsync(d_flag, 0, sizeof(int), r->st));
  if (fmt == LSE_IMAGE_F32) {
    for (int k = 0; k < K; ++k)
      CK(cudaMemcpy2DAsync(r->d_bands32 + k * stride, pitch * sizeof(float),
                           (const float*)image + (size_t)k * H * W, W * sizeof(float),
                           W * sizeof(float), H, cudaMemcpyHostToDevice, r->st));
  } else {
    TRY(dalloc(&tmp64, (size_t)K * H * W));
    CK(cudaMemcpyAsync(tmp64, image, (size_t)K * H * W * sizeof(double), cudaMemcpyHostToDevice,
                       r->st));
    for (int k = 0; k < K; ++k) {
      k_to_f32<<<grid2(W, H), 128, 0, r->st>>>(tmp64 + (size_t)k * H * W,
                                               r->d_bands32 + k * stride, H, W, pitch, d_flag);
      CKL();
    }
  }
  int inexact = 0;
  CK(cudaMemcpyAsync(&inexact, d_flag, sizeof(int), cudaMemcpyDeviceToHost, r->st));
  CK(cudaStreamSynchronize(r->st));
  if (inexact) {
    if (!r->d_bands64) TRY(dalloc(&r->d_bands64, (size_t)K * stride));
    for (int k = 0; k < K; ++k) {
      k_pitch64<<<grid2(W, H), 128, 0, r->st>>>(tmp64 + (size_t)k * H * W,
                                                r->d_bands64 + k * stride, H, W, pitch);
      CKL();
    }
  } else if (r->d_bands64) {
    cudaFree(r->d_bands64);
    r->d_bands64 = nullptr;
  }
  // max |I| over the bands (fp32 guard preconditions)
  double absmax = 0.0;
  for (int k = 0; k < K; ++k) {
    long long init[3] = {LLONG_MAX, LLONG_MIN, LLONG_MIN};
    CK(cudaMemcpyAsync(r->d_keys, init, sizeof(init), cudaMemcpyHostToDevice, r->st));
    k_minmax<<<std::min(H, num_sms() * 8), 256, 0, r->st>>>(
        r->d_bands32 + k * stride, r->d_bands64 ? r->d_bands64 + k * stride : nullptr, H, W,
        pitch, r->d_keys);
    CKL();
    k_store_minmax<<<1, 1, 0, r->st>>>(r->d_keys, r->d_scal);
    CKL();
    CK(cudaMemcpyAsync(r->h_scal, r->d_scal, sizeof(Scalars), cudaMemcpyDeviceToHost, r->st));
    CK(cudaStreamSynchronize(r->st));
    absmax = std::max(absmax, r->h_scal->img_absmax);
  }
  r->img_absmax = absmax;
  if (tmp64) cudaFree(tmp64);
  r->fp32_exact = !inexact;
  r->h_ctx.data32 = r->d_data32;
  r->h_ctx.data64 = nullptr;
  r->h_ctx.bands32 = r->d_bands32;
  r->h_ctx.bands64 = r->d_bands64;
  return upload_ctx(r);
}

void fill_status(lse_run* r, lse_status* s, long long instab) {
  if (!s) return;
  s->iteration = r->iteration;
  s->converged = r->converged;
  s->degenerate = r->degenerate;
  s->instability_iteration = instab;
  s->exact_fallbacks = r->h_scal ? (long long)r->h_scal->fallbacks : 0;
  s->fast_iterations = r->fast_iters;
  s->generic_iterations = r->generic_iters;
}

// Large pageable float32 images: staged through two cached pinned buffers, the
// host-side copies spread over a few threads (a plain cudaMemcpy from pageable
// memory is staged by the driver on one thread at ~10 GB/s: 0.36 s for a
// 32768^2 image; this path reaches the PCIe rate).  Pinned sources and small
// images take the direct copy.
constexpr size_t kStageBytes = 64u << 20;
constexpr int kStageThreads = 6;
struct StageBufs {
  void* buf[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
  std::mutex mu;
};
StageBufs g_stage;

int h2d_rows(lse_run* r, void* dst, size_t dpitch_b, const void* src, int H, size_t row_b) {
  cudaPointerAttributes at{};
  const bool pageable = cudaPointerGetAttributes(&at, src) != cudaSuccess ||
                        at.type == cudaMemoryTypeUnregistered;
  cudaGetLastError();
  if (!pageable || row_b * H < 4 * kStageBytes || row_b > kStageBytes) {
    CK(cudaMemcpy2DAsync(dst, dpitch_b, src, row_b, row_b, H, cudaMemcpyHostToDevice, r->st));
    return LSE_OK;
  }
  std::lock_guard<std::mutex> lock(g_stage.mu);
  for (int k = 0; k < 2; ++k)
    if (!g_stage.buf[k]) {
      CK(cudaHostAlloc(&g_stage.buf[k], kStageBytes, cudaHostAllocDefault));
      CK(cudaEventCreateWithFlags(&g_stage.ev[k], cudaEventDisableTiming));
    }
  const int rows_per = (int)(kStageBytes / row_b);
  int k = 0;
  for (int y = 0; y < H; y += rows_per, k ^= 1) {
    const int n = std::min(rows_per, H - y);
    CK(cudaEventSynchronize(g_stage.ev[k]));       // the copy that last used this buffer is done
    char* b = static_cast<char*>(g_stage.buf[k]);
    const char* s0 = reinterpret_cast<const char*>(src) + (size_t)y * row_b;
    const size_t bytes = (size_t)n * row_b, per = (bytes / kStageThreads + 4095) & ~(size_t)4095;
    std::thread th[kStageThreads];
    int nt = 0;
    for (size_t o = 0; o < bytes; o += per)
      th[nt++] = std::thread([=] { std::memcpy(b + o, s0 + o, std::min(per, bytes - o)); });
    for (int t = 0; t < nt; ++t) th[t].join();
    CK(cudaMemcpy2DAsync(reinterpret_cast<char*>(dst) + (size_t)y * dpitch_b, dpitch_b, b, row_b,
                         row_b, n, cudaMemcpyHostToDevice, r->st));
    CK(cudaEventRecord(g_stage.ev[k], r->st));
  }
  return LSE_OK;
}

// Large results into pageable host memory (the 1 byte/pixel mask of a big
// scene): the same two pinned buffers, the DMA of one chunk overlapping the
// threaded host copy of the previous one.
int d2h_bytes(lse_run* r, unsigned char* out, const unsigned char* d_src, size_t nbytes) {
  cudaPointerAttributes at{};
  const bool pageable = cudaPointerGetAttributes(&at, out) != cudaSuccess ||
                        at.type == cudaMemoryTypeUnregistered;
  cudaGetLastError();
  if (!pageable || nbytes < 4 * kStageBytes) {
    CK(cudaMemcpyAsync(out, d_src, nbytes, cudaMemcpyDeviceToHost, r->st));
    return LSE_OK;
  }
  std::lock_guard<std::mutex> lock(g_stage.mu);
  for (int k = 0; k < 2; ++k)
    if (!g_stage.buf[k]) {
      CK(cudaHostAlloc(&g_stage.buf[k], kStageBytes, cudaHostAllocDefault));
      CK(cudaEventCreateWithFlags(&g_stage.ev[k], cudaEventDisableTiming));
    }
  auto drain = [&](int k, size_t o, size_t n) -> int {
    CK(cudaEventSynchronize(g_stage.ev[k]));
    const char* b = static_cast<const char*>(g_stage.buf[k]);
    unsigned char* d0 = out + o;
    const size_t per = (n / kStageThreads + 4095) & ~(size_t)4095;
    std::thread th[kStageThreads];
    int nt = 0;
    for (size_t q = 0; q < n; q += per)
      th[nt++] = std::thread([=] { std::memcpy(d0 + q, b + q, std::min(per, n - q)); });
    for (int t = 0; t < nt; ++t) th[t].join();
    return LSE_OK;
  };
  size_t prev_o = 0, prev_n = 0;
  int k = 0;
  for (size_t o = 0; o < nbytes; o += kStageBytes, k ^= 1) {
    const size_t n = std::min(kStageBytes, nbytes - o);
    CK(cudaMemcpyAsync(g_stage.buf[k], d_src + o, n, cudaMemcpyDeviceToHost, r->st));
    CK(cudaEventRecord(g_stage.ev[k], r->st));
    if (prev_n) TRY(drain(k ^ 1, prev_o, prev_n));
    prev_o = o;
    prev_n = n;
  }
  if (prev_n) TRY(drain(k ^ 1, prev_o, prev_n));
  return LSE_OK;
}

int upload_image(lse_run* r, const void* image, int is_f32) {
  const int H = r->H, W = r->W;
  const long long pitch = r->g.data_pitch;
  double* tmp64 = nullptr;
  int* d_flag = nullptr;
  TRY(run_flag(r, &d_flag));
  CK(cudaMemsetAsync(d_flag, 0, sizeof(int), r->st));
  if (is_f32 == LSE_IMAGE_F32) {
    TRY(h2d_rows(r, r->d_data32, pitch * sizeof(float), image, H, (size_t)W * sizeof(float)));
    r->fp32_exact = true;
  } else {
    TRY(dalloc(&tmp64, r->npx));
    if (is_f32 == LSE_IMAGE_RGB8) {
      // 8-bit RGB, decoded to the loader's float64 luma on the device
      unsigned char* d8 = nullptr;
      TRY(dalloc(&d8, 3 * r->npx));
      TRY(h2d_rows(r, d8, 3 * (size_t)W, image, H, 3 * (size_t)W));
      k_luma<<<(unsigned)((r->npx + 255) / 256), 256, 0, r->st>>>(d8, tmp64, r->npx);
      CKL();
      CK(cudaStreamSynchronize(r->st));
      cudaFree(d8);
    } else {
      TRY(h2d_rows(r, tmp64, (size_t)W * sizeof(double), image, H, (size_t)W * sizeof(double)));
    }
    k_to_f32<<<grid2(W, H), 128, 0, r->st>>>(tmp64, r->d_data32, H, W, pitch, d_flag);
    CKL();
    int inexact = 0;
    CK(cudaMemcpyAsync(&inexact, d_flag, sizeof(int), cudaMemcpyDeviceToHost, r->st));
    CK(cudaStreamSynchronize(r->st));
    r->fp32_exact = !inexact;
  }
  if (two_mean(r->p.model)) {
    if (!r->fp32_exact) {
      if (!r->d_data64) TRY(dalloc(&r->d_data64, (size_t)pitch * H));
      k_pitch64<<<grid2(W, H), 128, 0, r->st>>>(tmp64, r->d_data64, H, W, pitch);
      CKL();
    } else if (r->d_data64) {
      cudaFree(r->d_data64);
      r->d_data64 = nullptr;
    }
  } else {
    // edge model: g = edge_function(I) on the device (engine.py:210-211)
    double* I64 = tmp64;
    if (!I64) {
      TRY(dalloc(&I64, r->npx));
      k_widen<<<grid2(W, H), 128, 0, r->st>>>(r->d_data32, I64, H, W, pitch);
      CKL();
      tmp64 = I64;
    }
    double *T = nullptr, *S = nullptr, *wpre = nullptr;
    TRY(dalloc(&T, r->npx));
    TRY(dalloc(&S, r->npx));
    const int Rp = (int)r->wpre.size() / 2;
    std::vector<double> wp(Rp + 1);
    for (int d = 0; d <= Rp; ++d) wp[d] = r->wpre[Rp - d];
    TRY(dalloc(&wpre, wp.size()));
    CK(cudaMemcpyAsync(wpre, wp.data(), wp.size() * sizeof(double), cudaMemcpyHostToDevice, r->st));
    k_corr<0><<<grid2(W, H), 128, 0, r->st>>>(I64, T, H, W, wpre, Rp);
    CKL();
    k_corr<1><<<grid2(W, H), 128, 0, r->st>>>(T, S, H, W, wpre, Rp);
    CKL();
    if (!r->d_data64) TRY(dalloc(&r->d_data64, (size_t)pitch * H));
    k_edge_g<<<grid2(W, H), 128, 0, r->st>>>(S, H, W, r->p.edge_gain, r->d_data64, r->d_data32,
                                              pitch, 0.5 * r->p.dt);
    CKL();
    CK(cudaStreamSynchronize(r->st));
    cudaFree(T);
    cudaFree(S);
    cudaFree(wpre);
    r->fp32_exact = false;
  }
  // image statistics for the closed-form normalizer / guards
  long long init[3] = {LLONG_MAX, LLONG_MIN, LLONG_MIN};
  CK(cudaMemcpyAsync(r->d_keys, init, sizeof(init), cudaMemcpyHostToDevice, r->st));
  k_minmax<<<std::min(H, num_sms() * 8), 256, 0, r->st>>>(r->d_data32, r->d_data64, H, W, pitch,
                                                          r->d_keys);
  CKL();
  k_store_minmax<<<1, 1, 0, r->st>>>(r->d_keys, r->d_scal);
  CKL();
  CK(cudaMemcpyAsync(r->h_scal, r->d_scal, sizeof(Scalars), cudaMemcpyDeviceToHost, r->st));
  CK(cudaStreamSynchronize(r->st));
  r->img_absmax = r->h_scal->img_absmax;
  if (tmp64) cudaFree(tmp64);
  // (two-mean models: the statistics above are the image's; NaN / inf order
  // above every finite key, so one of them makes max |I| non-finite)
  if (two_mean(r->p.model) && !std::isfinite(r->img_absmax))
    return fail(LSE_ERR_ARG, "grid contains non-finite values");
  r->h_ctx.data32 = r->d_data32;
  r->h_ctx.data64 = r->d_data64;
  r->prepared = false;
  return LSE_OK;
}

int set_state(lse_run* r, const lse_phi0* s) {
  if (!s) return fail(LSE_ERR_ARG, "null state");
  const int H = r->H, W = r->W;
  dim3 gw((r->g.pitch_w + 127) / 128, r->g.HR);
  r->launched.clear();
  if (s->kind == LSE_PHI0_POLYGONS) {
    if (s->n_polys < 1) return fail(LSE_ERR_ARG, "at least one seed polygon is required");
    std::vector<long long> offs(s->n_polys + 1, 0);
    for (long long k = 0; k < s->n_polys; ++k) offs[k + 1] = offs[k] + s->poly_counts[k];
    TRY(grow(r, &r->d_poly, &r->poly_cap, 2 * offs.back()));
    TRY(grow(r, &r->d_offs, &r->offs_cap, offs.size()));
    double* dxy = r->d_poly;
    long long* doffs = r->d_offs;
    CK(cudaMemcpyAsync(dxy, s->poly_xy, 2 * offs.back() * sizeof(double), cudaMemcpyHostToDevice,
                       r->st));
    CK(cudaMemcpyAsync(doffs, offs.data(), offs.size() * sizeof(long long), cudaMemcpyHostToDevice,
                       r->st));
    CK(cudaMemsetAsync(r->d_count, 0, sizeof(unsigned long long), r->st));
    if (offs.back() <= kRastEdges)
      k_rasterize_rows<<<dim3((r->g.pitch_w + 255) / 256, r->g.HR), 256, 0, r->st>>>(
          dxy, doffs, (int)s->n_polys, s->inside_sign, r->d_bits[r->cur], r->g, r->d_count, s->row_offset);
    else
      k_rasterize<<<gw, 128, 0, r->st>>>(dxy, doffs, (int)s->n_polys, s->inside_sign,
                                         r->d_bits[r->cur], nullptr, r->g, r->d_count,
                                         s->row_offset);
    CKL();
    unsigned long long cnt = 0;
    CK(cudaMemcpyAsync(&cnt, r->d_count, sizeof(cnt), cudaMemcpyDeviceToHost, r->st));
    CK(cudaStreamSynchronize(r->st));
    // (a row strip's seed count is global: the coordinator checks it)
    if (cnt == 0 && !r->strip)
      return fail(LSE_ERR_DEGENERATE_SEED, "seed polygons cover no pixel centers");
    if ((long long)cnt == r->npx && !r->strip)
      return fail(LSE_ERR_DEGENERATE_SEED, "seed polygons cover the entire grid");
    r->mode = SRC_SCALED;
    r->scale = 1.0;
    r->field_valid = false;
  } else if (s->kind == LSE_PHI0_SIGNS) {
    if (!(s->scale > 0.0) || !std::isfinite(s->scale)) return fail(LSE_ERR_ARG, "bad sign scale");
    signed char* d = nullptr;
    TRY(scratch(r, r->npx, &d));
    CK(cudaMemcpyAsync(d, s->signs, r->npx, cudaMemcpyHostToDevice, r->st));
    k_pack_signs<<<gw, 128, 0, r->st>>>(d, r->d_bits[r->cur], r->g);
    CKL();
    CK(cudaStreamSynchronize(r->st));
    r->mode = SRC_SCALED;
    r->scale = s->scale;
    r->field_valid = false;
  } else if (s->kind == LSE_PHI0_FIELD) {
    TRY(ensure_generic(r));
    r->curF = 0;
    CK(cudaMemcpyAsync(r->d_F[0], s->field, r->npx * sizeof(double), cudaMemcpyHostToDevice,
                       r->st));
    r->mode = SRC_FIELD;
    r->field_valid = true;
    // recognise fields the bit state represents exactly: +-s, or G * b
    if (r->R >= 1 && r->R <= 4) {
      k_pack_bits<<<gw, 128, 0, r->st>>>(r->d_F[0], r->d_bits[r->cur], r->g);
      CKL();
      double first = 0.0;
      CK(cudaMemcpyAsync(&first, r->d_F[0], sizeof(double), cudaMemcpyDeviceToHost, r->st));
      CK(cudaStreamSynchronize(r->st));
      const double sc = std::fabs(first);
      int cand[2] = {SRC_SCALED, SRC_SMOOTH};
      for (int src : cand) {
        if (src == SRC_SCALED && !(sc > 0.0 && std::isfinite(sc))) continue;
        r->scale = sc;
        TRY(upload_ctx(r));
        k_phi_from_bits<<<grid2(W, H), 128, 0, r->st>>>(r->d_bits[r->cur], r->d_F[1], r->d_ctx,
                                                         src);
        CKL();
        // compare bitwise
        int* d_ne = nullptr;
        TRY(run_flag(r, &d_ne));
        CK(cudaMemsetAsync(d_ne, 0, sizeof(int), r->st));
        const long long n = r->npx;
        const double* a = r->d_F[0];
        const double* b = r->d_F[1];
        k_bits_differ<<<num_sms() * 8, 256, 0, r->st>>>(a, b, n, d_ne);
        CKL();
        int ne = 1;
        CK(cudaMemcpyAsync(&ne, d_ne, sizeof(int), cudaMemcpyDeviceToHost, r->st));
        CK(cudaStreamSynchronize(r->st));
        if (!ne) {
          r->mode = src;
          break;
        }
      }
      if (r->mode != SRC_SCALED) r->scale = 1.0;
    }
  } else {
    return fail(LSE_ERR_ARG, "unknown state kind");
  }
  if (is_cv(r) && s->kind == LSE_PHI0_POLYGONS) {
    // init_state (engine.py:128-132): the distance field of the seed mask,
    // -signed_distance(phi0 > 0) for either inside sign
    TRY(ensure_generic(r));
    r->curF = 0;
    TRY(upload_ctx(r));
    k_phi_from_bits<<<grid2(W, H), 128, 0, r->st>>>(r->d_bits[r->cur], r->d_F[0], r->d_ctx,
                                                     SRC_SCALED);
    CKL();
    TRY(run_neg_sdf(r, r->d_F[0], r->d_F[0]));
    r->mode = SRC_FIELD;
    r->field_valid = true;
  }
  r->iteration = s->iteration;
  r->converged = s->converged != 0;
  r->degenerate = s->degenerate != 0;
  // device bookkeeping: sticky degenerate from the state, no stop; the
  // checkpoint history (n_ckpt, equal_run, M) is kept as in the reference
  CK(cudaMemcpyAsync(r->h_scal, r->d_scal, sizeof(Scalars), cudaMemcpyDeviceToHost, r->st));
  CK(cudaStreamSynchronize(r->st));
  r->h_scal->degenerate = r->degenerate;
  r->h_scal->stop = 0;
  r->h_scal->converged = 0;
  r->h_scal->ticket = 0;
  CK(cudaMemcpyAsync(r->d_scal, r->h_scal, sizeof(Scalars), cudaMemcpyHostToDevice, r->st));
  TRY(upload_ctx(r));
  CK(cudaStreamSynchronize(r->st));
  r->prepared = false;
  return LSE_OK;
}

}  // namespace

// ======================================================================= C ABI
extern "C" {

int lse_abi_version(void) { return LSE_ABI_VERSION; }
const char* lse_last_error(void) { return g_err.c_str(); }
int lse_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

namespace {
struct StripInfo {
  int own_lo, own_hi;
  long long n_total;
};

int create_impl(lse_run** out, const lse_params* p, long long height, long long width,
                const void* image, int image_is_f32, const lse_phi0* init, const StripInfo* si) {
  if (!out || !p || !image || !init) return fail(LSE_ERR_ARG, "null argument");
  *out = nullptr;
  if (height < 2 || width < 2) return fail(LSE_ERR_ARG, "gradient needs at least a 2x2 field");
  if (height > (1LL << 30) || width > (1LL << 30)) return fail(LSE_ERR_ARG, "grid too large");
  if (!two_mean(p->model) && p->model != LSE_MODEL_EDGE)
    return fail(LSE_ERR_UNSUPPORTED, "unknown model");
  if (p->model == LSE_MODEL_CV && (height < 3 || width < 3))
    return fail(LSE_ERR_ARG, "curvature needs at least a 3x3 field");
  if (p->ts_reg < 1 || p->ts_reg % 2 == 0 || !p->reg_weights)
    return fail(LSE_ERR_ARG, "ts_reg must be an odd number >= 1");
  if (p->ts_reg > 63) return fail(LSE_ERR_ARG, "ts_reg > 63 is not supported");
  if (p->model == LSE_MODEL_BANDS) {
    if (p->n_bands < 1 || p->n_bands > kMaxBands)
      return fail(LSE_ERR_ARG, "n_bands must be 1..4");
    if (p->reinit_period != 1 || p->reg_period != 1 || p->ts_reg < 3 || p->ts_reg > 9)
      return fail(LSE_ERR_UNSUPPORTED, "multi-band runs need the binary-state fast path "
                                       "(reinit_period = reg_period = 1, 3 <= ts_reg <= 9)");
    if (init->kind == LSE_PHI0_FIELD)
      return fail(LSE_ERR_UNSUPPORTED, "multi-band runs start from seeds or signs");
  }
  if (p->model == LSE_MODEL_EDGE && (p->ts_pre < 1 || p->ts_pre % 2 == 0 || !p->pre_weights))
    return fail(LSE_ERR_ARG, "ts_pre must be an odd number >= 1");
  TRY(check_device());
  lse_run* r = new lse_run();
  r->p = *p;
  r->wreg.assign(p->reg_weights, p->reg_weights + p->ts_reg);
  if (p->model == LSE_MODEL_EDGE) r->wpre.assign(p->pre_weights, p->pre_weights + p->ts_pre);
  r->p.reg_weights = nullptr;
  r->p.pre_weights = nullptr;
  r->H = (int)height;
  r->W = (int)width;
  r->R = p->ts_reg / 2;
  r->npx = height * width;
  r->g.H = r->H;
  r->g.W = r->W;
  r->g.HR = (r->H + 31) / 32;
  r->g.pitch_w = (int)round_up(r->W, 8);
  r->g.data_pitch = round_up(r->W, 8);
  long long need_thr = round_up((r->W + kColsPerThread - 1) / kColsPerThread, 32);
  r->nthr = (int)std::min<long long>(kThreads, need_thr);
  r->g.ncb = (r->W + kColsPerThread * r->nthr - 1) / (kColsPerThread * r->nthr);
  r->g.ntiles = r->g.HR * r->g.ncb;
  r->own_lo = 0;
  r->own_hi = r->g.HR;
  if (si) {
    r->strip = true;
    r->own_lo = si->own_lo;
    r->own_hi = si->own_hi;
  }
  r->nchunk = (r->W + kChunk - 1) / kChunk;
  r->nchunk_u = (r->W + kUpdChunk - 1) / kUpdChunk;
  {
    const int R = r->R, H = r->H, W = r->W;
    // border row parts (lse_geometry.cuh): border units are the critical path
    // of small images -- 2-row border lanes when there is no interior at all,
    // 4-row lanes when the interior units are split (see below), else 8
    const long long warps_u = (long long)num_sms() * kUpdateCtasPerSm * (kThreads / 32);
    int bq = kBorderQ;
    {
      const Geo g0 = make_geo(H, W, R, 1 + R, 1 + R, R + 1);
      const long long ni0 = (long long)(g0.r_hi - g0.r_lo) * g0.nci + (g0.nB1 + 31) / 32;
      bq = ni0 == 0 ? 16 : ni0 < 2 * warps_u ? 8 : kBorderQ;
    }
    // the partition keeps the default border lanes (its units carry the
    // partials, so a batched tile and the same tile alone group them alike)
    int bqp = kBorderQ;
    if (const char* bv = std::getenv("LSE_BORDER_Q"))
      bq = bqp = parse_border_q(bv);
    r->gu = make_geo(H, W, R, 1 + R, 1 + R, R + 1, bq);   // update reaches R+1 rows/columns
    r->gp = make_geo(H, W, R, R, R, R, bqp);              // partition reaches R
    if (si && (!geo_restrict_rows(r->gu, si->own_lo, si->own_hi) ||
               !geo_restrict_rows(r->gp, si->own_lo, si->own_hi))) {
      delete r;
      return fail(LSE_ERR_UNSUPPORTED, "strip too thin for its stencil");
    }
    r->gu_all = geo_all_border(r->gu, H);
    r->ni_upd = (long long)(r->gu.r_hi - r->gu.r_lo) * r->gu.nci + (r->gu.nB1 + 31) / 32;
    // too few full units to keep every warp busy for several rounds: split
    // them into 2 or 4 row parts (shorter units, more of them)
    {
      int ns = 1;
      while (ns < 4 && (long long)ns * r->ni_upd < 2 * warps_u) ns *= 2;
      const char* hv = std::getenv("LSE_SPLIT_PARTS");
      if (hv) ns = std::atoi(hv) >= 4 ? 4 : std::atoi(hv) >= 2 ? 2 : 1;
      r->split_parts = ns;
      r->ni_upd_split = (long long)ns * (r->gu.r_hi - r->gu.r_lo) * r->gu.nci +
                        (r->gu.nB1 + 32 / ns - 1) / (32 / ns);
    }
    r->nb_upd[0] = border_units(r->gu);
    r->nb_upd[1] = r->gu_all.nA;
    // partition segments: >= ~8 interior units per resident warp, <= 16 chunks
    // (fixed by the image geometry only)
    const long long warps = (long long)num_sms() * 16;
    const long long wi = r->gp.nci, hi_rows = r->gp.r_hi - r->gp.r_lo;
    long long sc = wi > 0 ? (hi_rows * wi) / (8 * warps) : 1;
    sc = std::max<long long>(1, std::min<long long>(16, sc));
    r->seg_chunks = (int)sc;
    r->nseg = wi > 0 ? (int)((wi + sc - 1) / sc) : 0;
    r->ni_part = hi_rows * r->nseg + (r->gp.nB1 + 31) / 32;
    r->nb_part = border_units(r->gp);
  }
  // small single images run the per-pixel kernels: an iteration is then
  // bound by one pixel's latency instead of one lane block's
  {
    long long fine_max = 450000;                  // ~670^2: measured crossover
    if (const char* fv = std::getenv("LSE_FINE_MAX_PX")) fine_max = std::atoll(fv);
    r->fine = !r->strip && r->R >= 1 && r->R <= 4 && r->npx <= fine_max;
    if (const char* ov = std::getenv("LSE_ONESTAGE_MAX_PARTS")) r->onestage_max = std::atoll(ov);
    // product default of the exact uniform-window skip (lse_run_set_option
    // changes it per run); LSE_SKIP_UNIFORM=0 makes every new run dense
    if (const char* sv = std::getenv("LSE_SKIP_UNIFORM")) r->skip_uniform = std::atoi(sv) != 0;
  }
  // speculative fused iterations (one pass per iteration): single tiled runs
  // of the region / zhang models with unsplit update units; LSE_FUSED=0 keeps
  // the two-pass iteration (A/B); validation builds check the two-pass path
  {
    bool fz = !r->fine && r->split_parts == 1 && r->R >= 1 && r->R <= 4 &&
              (p->model == LSE_MODEL_REGION || p->model == LSE_MODEL_ZHANG);
#ifdef LSE_CHECK_BOUND
    fz = false;
#endif
    if (const char* fv = std::getenv("LSE_FUSED")) fz = fz && std::atoi(fv) != 0;
    r->fused = fz;
    // fix list: pixels in the speculative band (a tiny fraction near the
    // fronts); more than this and the iteration is redone instead
    r->fix_cap = fz ? (unsigned)std::min<long long>(std::max<long long>(r->npx / 256, 4096),
                                                    1LL << 22)
                    : 0u;
    if (const char* cv = std::getenv("LSE_FIX_CAP"))   // (tests: force the redo pass)
      if (fz) r->fix_cap = (unsigned)std::max(0LL, std::atoll(cv));
  }
  resident_setup(r);
  const long long nparts = std::max<long long>(
      std::max<long long>(std::max<long long>(r->g.ntiles, r->ni_part + r->nb_part),
                          r->fused ? r->nb_upd[0] + r->ni_upd : 0LL),
      r->fine ? fine_parts(r) : 0LL);
  auto cleanup = [&](int rc) {
    lse_run_destroy(r);
    return rc;
  };
  if (cudaStreamCreateWithFlags(&r->st, cudaStreamNonBlocking) != cudaSuccess)
    return cleanup(fail(LSE_ERR_CUDA, "stream creation failed"));
  const size_t nbits = (size_t)r->g.HR * r->g.pitch_w;
  int rc = LSE_OK;
  if ((rc = dalloc(&r->d_data32, (size_t)r->g.data_pitch * r->H)) ||
      (rc = dalloc(&r->d_bits[0], nbits)) || (rc = dalloc(&r->d_bits[1], nbits)) ||
      (rc = dalloc(&r->d_P, nbits)) || (rc = dalloc(&r->d_M, nbits)) ||
      (rc = dalloc(&r->d_mask, nbits)) || (rc = dalloc(&r->d_part, nparts)) ||
      (rc = dalloc(&r->d_scal, 1)) || (rc = dalloc(&r->d_lut_t, 512)) ||
      (rc = dalloc(&r->d_lut_s, 512)) || (rc = dalloc(&r->d_ctx, 1)) ||
      (rc = dalloc(&r->d_w64, 32)) || (rc = dalloc(&r->d_keys, 3)) ||
      (rc = dalloc(&r->d_count, 1)) || (rc = dalloc(&r->d_work, 1)) ||
      (rc = dalloc(&r->d_part_fin, std::max(kFinSlices, kFusedFinSlices))) ||
      (rc = dalloc(&r->d_part_init, (size_t)r->g.HR * ((r->g.pitch_w + 1023) / 1024))))
    return cleanup(rc);
  if (r->fused && (rc = dalloc(&r->d_fix, r->fix_cap))) return cleanup(rc);
  if (p->model == LSE_MODEL_BANDS &&
      ((rc = dalloc(&r->d_bands32, (size_t)p->n_bands * r->g.data_pitch * r->H)) ||
       (rc = dalloc(&r->d_chg, nbits)) ||
       (rc = dalloc(&r->d_pmax, 2)) ||
       (rc = dalloc(&r->d_bpart, (size_t)p->n_bands * r->g.HR * ((r->g.pitch_w + 1023) / 1024)))))
    return cleanup(rc);
  if (r->d_pmax && cudaMemset(r->d_pmax, 0, 2 * sizeof(unsigned long long)) != cudaSuccess)
    return cleanup(fail(LSE_ERR_CUDA, "cudaMemset"));
  if (cudaMallocHost((void**)&r->h_scal, sizeof(Scalars)) != cudaSuccess)
    return cleanup(fail(LSE_ERR_CUDA, "pinned alloc failed"));
  cudaMemsetAsync(r->d_work, 0, sizeof(unsigned long long), r->st);
  cudaMemsetAsync(r->d_bits[0], 0, nbits * 4, r->st);
  cudaMemsetAsync(r->d_bits[1], 0, nbits * 4, r->st);
  cudaMemsetAsync(r->d_P, 0, nbits * 4, r->st);
  cudaMemsetAsync(r->d_M, 0, nbits * 4, r->st);
  // weights: w64[d] = weight at distance d (axis_weights[R - d])
  std::memset(&r->h_ctx, 0, sizeof(ExactCtx));
  for (int d = 0; d <= r->R; ++d) r->h_ctx.w64[d] = r->wreg[r->R - d];
  r->h_ctx.H = r->H;
  r->h_ctx.W = r->W;
  r->h_ctx.R = r->R;
  r->h_ctx.pitch_w = r->g.pitch_w;
  r->h_ctx.data_pitch = r->g.data_pitch;
  r->h_ctx.dt = p->dt;
  r->h_ctx.scale = 1.0;
  r->h_ctx.scal = r->d_scal;
  r->h_ctx.model = p->model == LSE_MODEL_REGION  ? REGION
                   : p->model == LSE_MODEL_ZHANG ? ZHANG
                   : p->model == LSE_MODEL_BANDS ? VECTOR
                   : p->model == LSE_MODEL_CV    ? CHAN_VESE
                                                 : EDGE;
  cudaMemcpyAsync(r->d_w64, r->h_ctx.w64, 32 * sizeof(double), cudaMemcpyHostToDevice, r->st);
  // LUTs for the fast path (R <= 4)
  if (r->R >= 1 && r->R <= 4) {
    const int np = 1 << (2 * r->R + 1);
    std::vector<float> lt(512, 0.f), ls(512, 0.f);
    for (int q = 0; q < np; ++q) {
      lt[q] = (float)host_t64((unsigned)q, r->R, r->h_ctx.w64);
      double s = 0.0;
      for (int k = 0; k <= 2 * r->R; ++k)
        if ((q >> k) & 1) s += r->h_ctx.w64[std::abs(k - r->R)];
      ls[q] = (float)s;
    }
    std::vector<double> lt64(512, 0.0);
    for (int q = 0; q < np; ++q) lt64[q] = host_t64((unsigned)q, r->R, r->h_ctx.w64);
    if (!r->d_lut64 && dalloc(&r->d_lut64, 512) != LSE_OK) return cleanup(LSE_ERR_CUDA);
    cudaMemcpyAsync(r->d_lut64, lt64.data(), 512 * sizeof(double), cudaMemcpyHostToDevice, r->st);
    r->h_ctx.lut64 = r->d_lut64;
    cudaMemcpyAsync(r->d_lut_t, lt.data(), 512 * sizeof(float), cudaMemcpyHostToDevice, r->st);
    cudaMemcpyAsync(r->d_lut_s, ls.data(), 512 * sizeof(float), cudaMemcpyHostToDevice, r->st);
    cudaStreamSynchronize(r->st);
  }
  // scalars
  Scalars s0;
  std::memset(&s0, 0, sizeof(s0));
  s0.n_total = si ? si->n_total : r->npx;
  s0.dt = p->dt;
  s0.model = r->h_ctx.model;
  s0.nu = p->nu;
  s0.nbands = p->model == LSE_MODEL_BANDS ? p->n_bands : 1;
  s0.conv_window = p->conv_window;
  s0.eps_phi = (float)kEpsPhi;
  s0.eps_u = (float)edge_eps_u(p->dt);
  s0.spec_delta = -1.0f;
  s0.fix_cap = r->fix_cap;
  s0.band_reuse = 1;
  if (const char* v = std::getenv("LSE_BAND_REUSE")) s0.band_reuse = std::atoi(v) != 0;
  if (p->model == LSE_MODEL_EDGE) {
    // a batched edge tile runs the fused pass with its exact coefficients:
    // band = the guard band, decided exactly in the pass, no fix list
    s0.spec_delta = 0.0f;
    s0.spec_e0 = (float)(edge_eps_u(p->dt) * 1.25);
  }
  if (p->model == LSE_MODEL_EDGE) s0.A = 1.0f;   // vf = 1 * g + 0 in a batched launch
  if (cudaMemcpyAsync(r->d_scal, &s0, sizeof(s0), cudaMemcpyHostToDevice, r->st) != cudaSuccess)
    return cleanup(fail(LSE_ERR_CUDA, "scalar upload failed"));
  if (p->model == LSE_MODEL_BANDS) {
    r->nbands = p->n_bands;
    r->h_ctx.nbands = p->n_bands;
    r->h_ctx.band_stride = (long long)r->g.data_pitch * r->H;
    if ((rc = upload_bands(r, image, image_is_f32))) return cleanup(rc);
  } else if ((rc = upload_image(r, image, image_is_f32))) {
    return cleanup(rc);
  }
  if ((rc = set_state(r, init))) return cleanup(rc);
  *out = r;
  return LSE_OK;
}
}  // namespace

int lse_run_create(lse_run** out, const lse_params* p, long long height, long long width,
                   const void* image, int image_is_f32, const lse_phi0* init) {
  return create_impl(out, p, height, width, image, image_is_f32, init, nullptr);
}

// ------------------------------------------------------------- row strips
int lse_strip_create(lse_run** out, const lse_params* p, long long height, long long width,
                     const void* image, int image_is_f32, const lse_phi0* init, int own_lo,
                     int own_hi, long long n_total) {
  if (!out || !p || !init) return fail(LSE_ERR_ARG, "null argument");
  if (p->reinit_period != 1 || p->reg_period != 1 || p->ts_reg < 3 || p->ts_reg > 9)
    return fail(LSE_ERR_UNSUPPORTED,
                "row strips run the binary-state fast path (reinit_period = reg_period = 1, "
                "3 <= ts_reg <= 9)");
  if (init->kind == LSE_PHI0_FIELD)
    return fail(LSE_ERR_UNSUPPORTED, "row strips start from seeds or signs");
  if (p->model == LSE_MODEL_BANDS)
    return fail(LSE_ERR_UNSUPPORTED, "multi-band runs are single-GPU");
  const long long HR = (height + 31) / 32;
  if (own_lo < 0 || own_lo > 1 || own_hi <= own_lo || own_hi > HR || own_hi < HR - 1)
    return fail(LSE_ERR_ARG, "a strip owns all its word-rows but at most one halo row per side");
  if (n_total < height * width) return fail(LSE_ERR_ARG, "n_total smaller than the strip");
  StripInfo si{own_lo, own_hi, n_total};
  return create_impl(out, p, height, width, image, image_is_f32, init, &si);
}

int lse_strip_image_range(lse_run* r, double* out3) {
  if (!r || !out3 || !r->strip) return fail(LSE_ERR_ARG, "not a row strip");
  CK(cudaMemcpyAsync(r->h_scal, r->d_scal, sizeof(Scalars), cudaMemcpyDeviceToHost, r->st));
  CK(cudaStreamSynchronize(r->st));
  out3[0] = r->h_scal->img_min;
  out3[1] = r->h_scal->img_max;
  out3[2] = r->h_scal->img_absmax;
  return LSE_OK;
}

int lse_strip_set_image_range(lse_run* r, const double* in3) {
  if (!r || !in3 || !r->strip) return fail(LSE_ERR_ARG, "not a row strip");
  CK(cudaStreamSynchronize(r->st));
  CK(cudaMemcpy(&r->d_scal->img_min, in3, 3 * sizeof(double), cudaMemcpyHostToDevice));
  r->img_absmax = in3[2];
  return LSE_OK;
}

int lse_strip_prepare(lse_run* r, void* part_out) {
  if (!r || !part_out || !r->strip) return fail(LSE_ERR_ARG, "not a row strip");
  if (r->mode != SRC_SCALED || r->field_valid || !fp32_ok(r))
    return fail(LSE_ERR_UNSUPPORTED, "row strips need a binary state on the fast path");
  TRY(upload_ctx(r));
  CK(cudaMemsetAsync(r->d_work, 0, sizeof(unsigned long long), r->st));
  r->work_next = 0;
  r->strip_fused = false;
  if (r->fused)
    CK(cudaMemsetAsync(reinterpret_cast<char*>(r->d_scal) + offsetof(Scalars, fix_n), 0,
                       sizeof(unsigned int) * 2, r->st));
  const dim3 gr((r->g.pitch_w + 1023) / 1024, r->g.HR);
  k_partition_init_bits<<<gr, 256, 0, r->st>>>(r->d_bits[r->cur], r->d_ctx, r->d_P,
                                               r->d_part_init, r->g, r->own_lo, r->own_hi);
  CKL();
  PartRanges R1{{r->d_part_init, r->d_part_init, r->d_part_init}, {(int)(gr.x * gr.y), 0, 0}};
  k_reduce_to_one<<<1, 256, 0, r->st>>>(R1, (TilePartial*)part_out, r->d_scal, 0);
  CKL();
  return LSE_OK;
}

int lse_strip_update(lse_run* r, int* partition_next) {
  if (!r || !r->strip) return fail(LSE_ERR_ARG, "not a row strip");
  if (!r->prepared) return fail(LSE_ERR_ARG, "lse_strip_prepare / lse_strip_finalize first");
  if (r->mode == SRC_FIELD || !fp32_ok(r))
    return fail(LSE_ERR_UNSUPPORTED, "row strips need a binary state on the fast path");
  const long long it = r->iteration + 1;
  TRY(launch_fast(r, it, it % r->p.conv_check_every == 0, PH_UPDATE));
  r->iteration = it;
  r->fast_iters++;
  if (partition_next) *partition_next = r->strip_part ? 1 : 0;
  return LSE_OK;
}

int lse_strip_partition(lse_run* r, void* part_out) {
  if (!r || !r->strip) return fail(LSE_ERR_ARG, "not a row strip");
  if (!r->strip_part) return LSE_OK;
  if (!part_out) return fail(LSE_ERR_ARG, "null partial");
  r->strip_out = (TilePartial*)part_out;
  TRY(launch_fast(r, r->iteration, r->strip_ckpt, PH_PARTITION));
  return LSE_OK;
}

int lse_strip_fused(lse_run* r, void* part_out) {
  if (!r || !r->strip || !part_out) return fail(LSE_ERR_ARG, "bad arguments");
  if (!r->fused)
    return fail(LSE_ERR_UNSUPPORTED, "this strip runs the two-pass iteration (lse_strip_update)");
  if (!r->prepared || !r->strip_part || r->strip_fused)
    return fail(LSE_ERR_ARG, "lse_strip_fused follows an update whose partition is owed");
  if (r->mode == SRC_FIELD || !fp32_ok(r))
    return fail(LSE_ERR_UNSUPPORTED, "row strips need a binary state on the fast path");
  const long long it = r->iteration + 1;
  TRY(launch_fused(r, it, r->strip_ckpt, (TilePartial*)part_out));
  r->iteration = it;
  r->fast_iters++;
  r->strip_part = true;                          // b^{it}'s partition is owed now
  r->strip_ckpt = it % r->p.conv_check_every == 0;
  return LSE_OK;
}

int lse_strip_finalize(lse_run* r, const void* parts, int nparts, int absolute) {
  if (!r || !r->strip || !parts || nparts < 1) return fail(LSE_ERR_ARG, "bad arguments");
  const TilePartial* tp = (const TilePartial*)parts;
  if (absolute) {
    if (two_mean(r->p.model)) {
      k_finalize<<<1, 1024, 0, r->st>>>(tp, nparts, r->d_scal, 0, 1, 0, r->iteration);
      CKL();
    }
    r->prepared = true;
    return LSE_OK;
  }
  PartRanges R{{tp, tp, tp}, {nparts, 0, 0}};
  if (r->strip_fused) {
    // the partition of iteration it-1 (fused pass): its coefficients check
    // the speculative update it, then the fix list or the redo
    const FastParams& P = r->strip_fp;
    k_finalize_run<<<1, 64, 0, r->st>>>(R, r->d_scal, 1, (P.iter % r->p.conv_check_every) == 0,
                                          P.iter, 1 + P.fix_par);
    CKL();
    TRY(launch_spec_tail_any(r, P));
    r->strip_fused = false;
    return LSE_OK;
  }
  if (!r->strip_part) return LSE_OK;
  k_finalize_run<<<1, 64, 0, r->st>>>(R, r->d_scal, two_mean(r->p.model) ? 1 : 0,
                                        r->strip_ckpt ? 1 : 0, r->iteration, 0);
  CKL();
  r->strip_part = false;
  return LSE_OK;
}

int lse_strip_sync(lse_run* r, lse_status* st) {
  if (!r || !r->strip) return fail(LSE_ERR_ARG, "not a row strip");
  TRY(collect(r));
  fill_status(r, st, -1);
  return LSE_OK;
}

void* lse_run_stream(lse_run* r) { return r ? (void*)r->st : nullptr; }

void* lse_run_bits_row(lse_run* r, int word_row) {
  if (!r || word_row < 0 || word_row >= r->g.HR) return nullptr;
  return r->d_bits[r->cur] + (size_t)word_row * r->g.pitch_w;
}

int lse_run_geometry(lse_run* r, int* word_rows, int* pitch_words) {
  if (!r) return fail(LSE_ERR_ARG, "null run");
  if (word_rows) *word_rows = r->g.HR;
  if (pitch_words) *pitch_words = r->g.pitch_w;
  return LSE_OK;
}

int lse_run_load_image(lse_run* r, const void* image, int image_is_f32) {
  if (!r || !image) return fail(LSE_ERR_ARG, "null argument");
  if (is_bands(r)) {
    TRY(upload_bands(r, image, image_is_f32));
    r->prepared = false;                         // the data term depends on the bands
    return LSE_OK;
  }
  return upload_image(r, image, image_is_f32);
}

int lse_run_set_state(lse_run* r, const lse_phi0* st) {
  if (!r) return fail(LSE_ERR_ARG, "null run");
  return set_state(r, st);
}

int lse_run_advance(lse_run* r, long long n_steps, lse_status* st) {
  if (!r) return fail(LSE_ERR_ARG, "null run");
  if (r->strip) return fail(LSE_ERR_ARG, "row strips advance through the lse_strip_* phases");
  if (n_steps < 0) return fail(LSE_ERR_ARG, "n_steps must be >= 0");
  if (r->converged || r->iteration >= r->p.max_iters || n_steps == 0) {
    fill_status(r, st, -1);
    return LSE_OK;
  }
  const long long steps = std::min(n_steps, r->p.max_iters - r->iteration);
  TRY(prepare(r));
  // re-base the dynamic work counter (a stopped launch makes no grabs)
  CK(cudaMemsetAsync(r->d_work, 0, sizeof(unsigned long long), r->st));
  r->work_next = 0;
  const long long it0 = r->iteration;
  const long long cce = r->p.conv_check_every;
  bool pending = false;
  // fused runs: the partition of the last update's output is owed to the next
  // pass (a fused iteration) or to the trailing partition phase
  bool owe = false;
  long long owe_it = 0;
  if (r->fused)
    CK(cudaMemsetAsync(reinterpret_cast<char*>(r->d_scal) + offsetof(Scalars, fix_n), 0,
                       sizeof(unsigned int) * 2, r->st));
  if (resident_now(r)) {
    // small image: the whole call is one resident kernel (lse_resident.cuh);
    // very long calls in launches of 2^20 iterations (the grid barrier counts
    // arrivals in 32 bits; a launch after convergence returns at once)
    for (long long done = 0; done < steps;) {
      const long long n = std::min<long long>(steps - done, 1LL << 20);
      TRY(launch_resident(r, n));
      done += n;
    }
    TRY(collect(r));
    fill_status(r, st, -1);
    return LSE_OK;
  }
  for (long long it = it0 + 1; it <= it0 + steps; ++it) {
    const bool reinit_now = r->p.reinit_period > 0 && it % r->p.reinit_period == 0;
    const bool reg_now = it % r->p.reg_period == 0;
    const bool ckpt = it % r->p.conv_check_every == 0;
    if (reinit_now && reg_now && r->mode != SRC_FIELD && fp32_ok(r)) {
      if (r->fused) {
        if (owe) TRY(launch_fused(r, it, owe_it % cce == 0));
        else TRY(launch_fast(r, it, ckpt, PH_UPDATE));
        owe = true;
        owe_it = it;
      } else {
        TRY(launch_fast(r, it, ckpt));
      }
      r->iteration = it;
      r->fast_iters++;
      pending = true;
    } else {
      if (owe) {
        TRY(launch_fast(r, owe_it, owe_it % cce == 0, PH_PARTITION));
        owe = false;
      }
      if (pending) {
        TRY(collect(r));
        pending = false;
        if (r->converged) break;
      }
      int rc = generic_iteration(r, it, reinit_now, reg_now, ckpt);
      if (rc == LSE_ERR_INSTABILITY) {
        fill_status(r, st, it);
        char msg[160];
        std::snprintf(msg, sizeof(msg), "numerical instability: non-finite level-set values at "
                                        "iteration %lld", it);
        return fail(LSE_ERR_INSTABILITY, msg);
      }
      TRY(rc);
      if (r->converged) break;
    }
  }
  if (owe) TRY(launch_fast(r, owe_it, owe_it % cce == 0, PH_PARTITION));
  if (pending) TRY(collect(r));
  fill_status(r, st, -1);
  return LSE_OK;
}

int lse_run_status(lse_run* r, lse_status* st) {
  if (!r || !st) return fail(LSE_ERR_ARG, "null argument");
  fill_status(r, st, -1);
  return LSE_OK;
}

int lse_run_read_phi(lse_run* r, double* out) {
  if (!r || !out) return fail(LSE_ERR_ARG, "null argument");
  TRY(ensure_generic(r));
  const double* src;
  if (r->field_valid) {
    src = r->d_F[r->curF];
  } else {
    TRY(upload_ctx(r));
    k_phi_from_bits<<<grid2(r->W, r->H), 128, 0, r->st>>>(r->d_bits[r->cur], r->d_U, r->d_ctx,
                                                           r->mode);
    CKL();
    src = r->d_U;
  }
  TRY(d2h_bytes(r, reinterpret_cast<unsigned char*>(out), reinterpret_cast<const unsigned char*>(src),
                (size_t)r->npx * sizeof(double)));
  CK(cudaStreamSynchronize(r->st));
  return LSE_OK;
}

int lse_run_read_mask(lse_run* r, unsigned char* out, int inside_sign, int packed) {
  if (!r || !out) return fail(LSE_ERR_ARG, "null argument");
  TRY(upload_ctx(r));
  if (r->mode == SRC_SMOOTH && !r->field_valid && r->R >= 1 && r->R <= 4) {
    FastParams P = fast_params(r);
    P.bits_in = r->d_bits[r->cur];
    P.mbits = r->d_mask;
    CK(cudaMemsetAsync(r->d_work, 0, sizeof(unsigned long long), r->st));
    r->work_next = 0;
    switch (r->R) {
      case 1: TRY((launch_partition<1, false, false, true>(r, P))); break;
      case 2: TRY((launch_partition<2, false, false, true>(r, P))); break;
      case 3: TRY((launch_partition<3, false, false, true>(r, P))); break;
      case 4: TRY((launch_partition<4, false, false, true>(r, P))); break;
    }
    CKL();
  } else {
    const int src = r->field_valid ? SRC_FIELD : r->mode;
    if (src == SRC_SMOOTH) TRY(materialize(r));
    TRY(launch_partition_abs(r, r->field_valid ? SRC_FIELD : src, false, false, true, r->d_mask));
  }
  const int invert = inside_sign > 0 ? 0 : 1;
  unsigned char* d_out = nullptr;
  if (packed) {
    const long long nbytes = (r->npx + 7) / 8;
    TRY(scratch(r, nbytes, &d_out));
    k_mask_packed<<<(unsigned)((nbytes + 255) / 256), 256, 0, r->st>>>(r->d_mask, r->g, invert,
                                                                      d_out, nbytes);
    CKL();
    CK(cudaMemcpyAsync(out, d_out, nbytes, cudaMemcpyDeviceToHost, r->st));
  } else {
    TRY(scratch(r, r->npx, &d_out));
    k_mask_u8<<<grid2(r->W, r->H), 128, 0, r->st>>>(r->d_mask, r->g, invert, d_out);
    CKL();
    TRY(d2h_bytes(r, out, d_out, (size_t)r->npx));
  }
  CK(cudaStreamSynchronize(r->st));
  return LSE_OK;
}

long long lse_launch_count(void) { return g_launches.load(); }

int lse_check_enabled(void) {
#ifdef LSE_CHECK_BOUND
  return 1;
#else
  return 0;
#endif
}

int lse_check_stats(double* out, int reset) {
  if (!out) return fail(LSE_ERR_ARG, "null argument");
#ifdef LSE_CHECK_BOUND
  CheckSlot* d = check_slots();
  if (!d) return fail(LSE_ERR_CUDA, "no certification slots");
  CK(cudaDeviceSynchronize());
  std::vector<CheckSlot> h(kCheckSlots);
  CK(cudaMemcpy(h.data(), d, kCheckSlots * sizeof(CheckSlot), cudaMemcpyDeviceToHost));
  double ru = 0, rp = 0, umin = 3.0e38, pmin = 3.0e38, bu = 0, bp = 0, n = 0, used = 0;
  for (const CheckSlot& k : h) {
    if (!k.n) continue;
    ru = std::max(ru, (double)k.ru);
    rp = std::max(rp, (double)k.rp);
    umin = std::min(umin, (double)k.umin);
    pmin = std::min(pmin, (double)k.pmin);
    bu += k.bad_u;
    bp += k.bad_p;
    n += (double)k.n;
    used += 1;
  }
  const double v[8] = {ru, rp, umin, pmin, bu, bp, n, used};
  std::memcpy(out, v, sizeof(v));
  if (reset) {
    k_check_reset<<<512, 256>>>(d, kCheckSlots);
    CK(cudaDeviceSynchronize());
  }
  return LSE_OK;
#else
  (void)reset;
  return fail(LSE_ERR_UNSUPPORTED, "not a certification build (make check)");
#endif
}

int lse_run_set_option(lse_run* r, const char* name, long long value) {
  if (!r || !name) return fail(LSE_ERR_ARG, "null argument");
  if (!std::strcmp(name, "skip_uniform")) {
    r->skip_uniform = value != 0;
    return LSE_OK;
  }
  return fail(LSE_ERR_ARG, std::string("unknown option ") + name);
}

int lse_run_begin_timing(lse_run* r) {
  if (!r) return fail(LSE_ERR_ARG, "null run");
  if (!r->t_begin) CK(cudaEventCreate(&r->t_begin));
  if (!r->t_end) CK(cudaEventCreate(&r->t_end));
  CK(cudaEventRecord(r->t_begin, r->st));
  return LSE_OK;
}

int lse_run_end_timing(lse_run* r, double* ms) {
  if (!r || !ms) return fail(LSE_ERR_ARG, "null argument");
  if (!r->t_begin || !r->t_end) return fail(LSE_ERR_ARG, "timing not started");
  CK(cudaEventRecord(r->t_end, r->st));
  CK(cudaEventSynchronize(r->t_end));
  float f = 0.f;
  CK(cudaEventElapsedTime(&f, r->t_begin, r->t_end));
  *ms = f;
  return LSE_OK;
}

int lse_run_spec_stats(lse_run* r, long long* out4) {
  if (!r || !out4) return fail(LSE_ERR_ARG, "null argument");
  CK(cudaMemcpyAsync(r->h_scal, r->d_scal, sizeof(Scalars), cudaMemcpyDeviceToHost, r->st));
  CK(cudaStreamSynchronize(r->st));
  out4[0] = r->fused_iters;
  out4[1] = (long long)r->h_scal->spec_redos;
  out4[2] = (long long)r->h_scal->spec_fixes;
  out4[3] = r->fused ? 1 : 0;
  return LSE_OK;
}

int lse_run_resident_stats(lse_run* r, long long* out5) {
  if (!r || !out5) return fail(LSE_ERR_ARG, "null argument");
  out5[0] = r->resident ? 1 : 0;
  out5[1] = r->res_grid ? 1 : 0;
  out5[2] = r->res_ctas;
  out5[3] = r->resident_calls;
  out5[4] = r->res_nt;
  return LSE_OK;
}

int lse_run_band_stats(lse_run* r, long long* out2) {
  if (!r || !out2) return fail(LSE_ERR_ARG, "null argument");
  CK(cudaMemcpyAsync(r->h_scal, r->d_scal, sizeof(Scalars), cudaMemcpyDeviceToHost, r->st));
  CK(cudaStreamSynchronize(r->st));
  out2[0] = (long long)r->h_scal->band_reused;
  out2[1] = r->h_scal->band_reuse;
  return LSE_OK;
}

int lse_run_set_profiling(lse_run* r, int enabled) {
  if (!r) return fail(LSE_ERR_ARG, "null run");
  r->prof = enabled != 0;
  r->t_update = r->t_part = 0;
  r->n_update = r->n_part = 0;
  return LSE_OK;
}

int lse_run_kernel_times(lse_run* r, double* update_ms, long long* update_launches,
                         double* partition_ms, long long* partition_launches) {
  if (!r) return fail(LSE_ERR_ARG, "null run");
  if (update_ms) *update_ms = r->t_update;
  if (update_launches) *update_launches = r->n_update;
  if (partition_ms) *partition_ms = r->t_part;
  if (partition_launches) *partition_launches = r->n_part;
  return LSE_OK;
}

// ------------------------------------------------------------ batched tiles
// lse_batch: many equal-size runs advanced together, one launch per kernel
// per iteration for all of them (512 tiles of 1024^2 are each
// far too small to fill a B200).  The tiles' state is stacked in shared
// arrays while the batch advances and written back to the runs afterwards,
// so every run stays usable on its own (status, read_phi, read_mask).
}  // extern "C"

struct lse_batch {
  std::vector<lse_run*> runs;
  int T = 0;
  // update geometry of one tile: the batch has work for every warp, so its
  // border units keep the default 8-row lanes whatever a lone tile would
  // use (the update has no partials, so this changes no reduction order; the
  // partition uses the single run's geometry and partial grouping)
  Geo gu{};
  cudaStream_t st = nullptr;
  uint32_t* bits[2] = {nullptr, nullptr};
  uint32_t* P = nullptr;
  uint32_t* M = nullptr;
  float* data32 = nullptr;
  double* data64 = nullptr;
  Scalars* scal = nullptr;
  Scalars* h_scal = nullptr;
  ExactCtx* ctx = nullptr;
  TilePartial* part = nullptr;
  TilePartial* part_fin = nullptr;
  unsigned long long* work = nullptr;
  unsigned long long work_next = 0;
  const uint32_t** d_src = nullptr;          // per-tile pointer tables for k_tiles_copy
  uint32_t** d_dst = nullptr;
  long long tile_words = 0, tile_data = 0, nb_upd = 0, ni_upd = 0, nb_part = 0, ni_part = 0;
  int tile_hr = 0;
  int cur = 0;
  // speculative fused iterations (batches with region / zhang tiles)
  bool fused = false;
  int2* fix = nullptr;
  unsigned int fix_cap = 0;
  // device-event timing of whole lse_batch_advance calls (bench support)
  bool timing = false;
  cudaEvent_t ev[2] = {nullptr, nullptr};
  double t_ms = 0.0;
  long long t_calls = 0;
};

namespace {

// copy n uint32 words per tile: src[t] -> dst[t] (device pointer tables)
int tiles_copy(lse_batch* b, const std::vector<const void*>& src, const std::vector<void*>& dst,
               long long n_words) {
  CK(cudaMemcpyAsync(b->d_src, src.data(), b->T * sizeof(void*), cudaMemcpyHostToDevice, b->st));
  CK(cudaMemcpyAsync(b->d_dst, dst.data(), b->T * sizeof(void*), cudaMemcpyHostToDevice, b->st));
  const int gx = (int)std::min<long long>(64, (n_words + 255) / 256);
  k_tiles_copy<<<dim3(gx, b->T), 256, 0, b->st>>>(b->d_src, b->d_dst, n_words);
  CKL();
  CK(cudaStreamSynchronize(b->st));             // the host tables are reused at once
  return LSE_OK;
}

FastParams batch_params(lse_batch* b, int sel) {
  lse_run* r0 = b->runs[0];
  FastParams P = fast_params(r0);
  P.pbits = b->P;
  P.mbits = b->M;
  P.data32 = b->data32;
  P.part = b->part;
  P.scal = b->scal;
  P.ctx = b->ctx;
  P.work = b->work;
  P.bits_in = b->bits[sel];
  P.bits_out = b->bits[sel ^ 1];
  P.ntiles = b->T;
  P.tile_hr = b->tile_hr;
  P.tile_h = r0->H;
  P.tile_words = b->tile_words;
  P.tile_data = b->tile_data;
  P.gu = b->gu;
  P.g.H = b->T * b->tile_hr * 32;             // the stacked arrays
  P.g.HR = b->T * b->tile_hr;
  P.own_lo = 0;
  P.own_hi = P.g.HR;
  P.fix = b->fix;
  P.fix_cap = b->fix_cap;
  P.fix_cnt = b->scal->fix_n;                 // the batch's counters: tile 0's scalars
  return P;
}

unsigned long long batch_take_work(lse_batch* b, long long units, int grid) {
  const unsigned long long base = b->work_next;
  b->work_next += (unsigned long long)units + (unsigned long long)grid * 4;
  return base;
}

// phase: the batched plain update of iteration it (b^{it-1} -> b^{it})
template <int R>
int batch_update(lse_batch* b, long long it, int src) {
  FastParams P = batch_params(b, b->cur);
  P.iter = it;
  set_check(P, it);
  {
    const long long n = (long long)b->T * (b->nb_upd + b->ni_upd);
    const int g = fast_grid(n, kUpdateCtasPerSm);
    P.work_base = batch_take_work(b, n, g);
#ifdef LSE_UNIT_TRACE
    P.trace = trace_begin_st(b->st, n, g, "batch-update", (long long)b->T * b->nb_upd);
#endif
    if (src == SRC_SCALED)
      TRY(launch_pdl(k_update<R, REGION, SRC_SCALED, true, 1>, g, kThreads, b->st, P));
    else
      TRY(launch_pdl(k_update<R, REGION, SRC_SMOOTH, true, 1>, g, kThreads, b->st, P));
#ifdef LSE_UNIT_TRACE
    trace_after_st(b->st, P.trace);
    P.trace = nullptr;
#endif
  }
  b->cur ^= 1;
  return LSE_OK;
}

// phase: the batched partition / checkpoint pass over the current state
// (iteration it) and the per-tile finalize
template <int R>
int batch_partition(lse_batch* b, long long it, bool ckpt, bool any_region) {
  if (!any_region && !ckpt) return LSE_OK;
  FastParams P = batch_params(b, b->cur);
  P.iter = it;
  set_check(P, it);
  P.bits_in = b->bits[b->cur];
  const long long n = (long long)b->T * (b->nb_part + b->ni_part);
  const int g = fast_grid(n, kPartitionCtasPerSm);
  P.work_base = batch_take_work(b, n, g);
#ifdef LSE_UNIT_TRACE
  P.trace = trace_begin_st(b->st, n, g, "batch-partition", (long long)b->T * b->nb_part);
#endif
  if (ckpt) TRY(launch_pdl(k_partition<R, true, true, false, true>, g, kThreads, b->st, P));
  else TRY(launch_pdl(k_partition<R, true, false, false, true>, g, kThreads, b->st, P));
#ifdef LSE_UNIT_TRACE
  trace_after_st(b->st, P.trace);
#endif
  if (b->nb_part + b->ni_part <= b->runs[0]->onestage_max) {   // as a lone tile: one stage
    TRY(launch_pdl(k_finalize_tiles_direct, b->T, 64, b->st, (const TilePartial*)b->part, b->scal,
                   (int)b->nb_part, (int)b->ni_part, b->T, ckpt ? 1 : 0, it, 0));
    return LSE_OK;
  }
  TRY(launch_pdl(k_finalize_stage1_tiles, dim3(kFinSlices, b->T), 256, b->st,
                 (const TilePartial*)b->part, b->part_fin, (const Scalars*)b->scal,
                 (int)b->nb_part, (int)b->ni_part, b->T, ckpt ? 1 : 0));
  TRY(launch_pdl(k_finalize_run_tiles, b->T, 64, b->st, (const TilePartial*)b->part_fin,
                 b->scal, ckpt ? 1 : 0, it, 0));
  return LSE_OK;
}

template <int R>
int batch_iteration(lse_batch* b, long long it, bool ckpt, int src, bool any_region) {
  TRY(batch_update<R>(b, it, src));
  return batch_partition<R>(b, it, ckpt, any_region);
}

// One speculative fused iteration of every tile (batched): the
// partition of b^{it-1} (its checkpoint when ckpt_prev) and the update it-1 ->
// it in one pass, the per-tile finalize with each region tile's prediction
// check, the fix list, the redo of the tiles that need it.
template <int R>
int batch_fused(lse_batch* b, long long it, bool ckpt_prev) {
  FastParams P = batch_params(b, b->cur);
  P.iter = it - 1;
  set_check(P, it);
  P.fix_par = (int)(it & 1);
  const long long nu = b->nb_upd + b->ni_upd;
  const long long n = (long long)b->T * nu;
  const int g = fast_grid(n, kFusedCtasPerSm);
  P.work_base = batch_take_work(b, n, g);
  constexpr size_t smem = fused_smem_bytes<R>();
  if (ckpt_prev) {
    TRY(prepare_smem(k_update_fused<R, true, true>, smem));
    TRY(launch_pdl_smem(k_update_fused<R, true, true>, g, kThreads, smem, b->st, P));
  } else {
    TRY(prepare_smem(k_update_fused<R, false, true>, smem));
    TRY(launch_pdl_smem(k_update_fused<R, false, true>, g, kThreads, smem, b->st, P));
  }
  const int spec = 1 + P.fix_par;
  if (nu <= b->runs[0]->onestage_max) {
    TRY(launch_pdl(k_finalize_tiles_direct, b->T, 64, b->st, (const TilePartial*)b->part, b->scal,
                   (int)b->nb_upd, (int)b->ni_upd, b->T, ckpt_prev ? 1 : 0, it - 1, spec));
  } else {
    TRY(launch_pdl(k_finalize_stage1_tiles, dim3(kFinSlices, b->T), 256, b->st,
                   (const TilePartial*)b->part, b->part_fin, (const Scalars*)b->scal,
                   (int)b->nb_upd, (int)b->ni_upd, b->T, ckpt_prev ? 1 : 0));
    TRY(launch_pdl(k_finalize_run_tiles, b->T, 64, b->st, (const TilePartial*)b->part_fin,
                   b->scal, ckpt_prev ? 1 : 0, it - 1, spec));
  }
  TRY(launch_pdl(k_spec_fix<R, true>, num_sms(), 256, b->st, P));
  FastParams Q = P;                              // the redo pass has its own work counter
  Q.work = &b->scal->work2;
  Q.work_base = 0;
  TRY(launch_pdl(k_spec_redo<R, true>, fast_grid(n, kUpdateCtasPerSm), kThreads, b->st, Q));
  b->cur ^= 1;
  return LSE_OK;
}

}  // namespace

extern "C" {

int lse_batch_create(lse_batch** out, lse_run* const* runs, int n) {
  if (!out || !runs || n < 1) return fail(LSE_ERR_ARG, "bad arguments");
  *out = nullptr;
  lse_run* r0 = runs[0];
  for (int t = 0; t < n; ++t) {
    lse_run* r = runs[t];
    if (!r || r->strip) return fail(LSE_ERR_ARG, "batch tiles must be plain runs");
    if (r->H != r0->H || r->W != r0->W || r->R != r0->R || r->p.dt != r0->p.dt ||
        r->p.ts_reg != r0->p.ts_reg || r->wreg != r0->wreg ||
        r->p.conv_check_every != r0->p.conv_check_every ||
        r->p.conv_window != r0->p.conv_window || r->p.max_iters != r0->p.max_iters ||
        r->skip_uniform != r0->skip_uniform)
      return fail(LSE_ERR_ARG, "batch tiles must share size and evolution parameters");
    if (r->p.reinit_period != 1 || r->p.reg_period != 1 || r->R < 1 || r->R > 4)
      return fail(LSE_ERR_UNSUPPORTED, "batches run the binary-state fast path only");
    if (is_bands(r)) return fail(LSE_ERR_UNSUPPORTED, "multi-band runs are not batched");
  }
  lse_batch* b = new lse_batch();
  b->runs.assign(runs, runs + n);
  b->T = n;
  b->tile_hr = r0->g.HR;
  b->tile_words = (long long)r0->g.HR * r0->g.pitch_w;
  b->tile_data = (long long)r0->g.HR * 32 * r0->g.data_pitch;
  b->gu = make_geo(r0->H, r0->W, r0->R, 1 + r0->R, 1 + r0->R, r0->R + 1, kBorderQ);
  if (const char* bv = std::getenv("LSE_BORDER_Q"))
    b->gu = make_geo(r0->H, r0->W, r0->R, 1 + r0->R, 1 + r0->R, r0->R + 1, parse_border_q(bv));
  b->nb_upd = border_units(b->gu);
  b->ni_upd = r0->ni_upd;
  b->nb_part = r0->nb_part;
  b->ni_part = r0->ni_part;
  auto cleanup = [&](int rc) {
    lse_batch_destroy(b);
    return rc;
  };
  if (cudaStreamCreateWithFlags(&b->st, cudaStreamNonBlocking) != cudaSuccess)
    return cleanup(fail(LSE_ERR_CUDA, "stream creation failed"));
  bool any64 = false;
  for (auto* r : b->runs) any64 |= r->d_data64 != nullptr;
  const size_t nw = (size_t)n * b->tile_words, nd = (size_t)n * b->tile_data;
  int rc;
  if ((rc = dalloc(&b->bits[0], nw)) || (rc = dalloc(&b->bits[1], nw)) ||
      (rc = dalloc(&b->P, nw)) || (rc = dalloc(&b->M, nw)) || (rc = dalloc(&b->data32, nd)) ||
      (any64 && (rc = dalloc(&b->data64, nd))) || (rc = dalloc(&b->scal, n)) ||
      (rc = dalloc(&b->ctx, n)) ||
      (rc = dalloc(&b->part, (size_t)n * (b->nb_upd + b->ni_upd + b->nb_part + b->ni_part))) ||
      (rc = dalloc(&b->part_fin, (size_t)n * kFinSlices)) || (rc = dalloc(&b->work, 1)) ||
      (rc = dalloc(&b->d_src, n)) || (rc = dalloc(&b->d_dst, n)))
    return cleanup(rc);
  if (cudaMallocHost((void**)&b->h_scal, n * sizeof(Scalars)) != cudaSuccess)
    return cleanup(fail(LSE_ERR_CUDA, "pinned alloc failed"));
  {
    // batched fused iterations are opt-in (LSE_FUSED_BATCH=1): on C4's
    // 1024^2 tiles the border units -- ~30 % of the update's work -- pay the
    // partition's zero-padded recomputation on top of the update's, and the
    // fused pass measured 306 us vs 126 + 65 us for update + partition (64
    // tiles); the next step is deriving the border partition from the
    // update's own phi rows, as the interior units do
    bool fz = true;
#ifdef LSE_CHECK_BOUND
    fz = false;
#endif
    const char* bv = std::getenv("LSE_FUSED_BATCH");
    fz = fz && bv && std::atoi(bv) != 0;
    if (const char* fv = std::getenv("LSE_FUSED")) fz = fz && std::atoi(fv) != 0;
    b->fused = fz;
    if (fz) {
      const long long px = (long long)n * r0->H * r0->W;
      b->fix_cap = (unsigned)std::min<long long>(std::max<long long>(px / 256, 4096), 1LL << 22);
      if (const char* cv = std::getenv("LSE_FIX_CAP"))
        b->fix_cap = (unsigned)std::max(0LL, std::atoll(cv));
      if ((rc = dalloc(&b->fix, std::max<unsigned>(1u, b->fix_cap)))) return cleanup(rc);
    }
  }
  // static data planes and per-tile contexts (tile t at word-row t * tile_hr)
  std::vector<ExactCtx> ctx(n);
  for (int t = 0; t < n; ++t) {
    lse_run* r = b->runs[t];
    CK(cudaStreamSynchronize(r->st));
    CK(cudaMemcpyAsync(b->data32 + t * b->tile_data, r->d_data32,
                       (size_t)r->H * r->g.data_pitch * sizeof(float), cudaMemcpyDeviceToDevice,
                       b->st));
    if (r->d_data64)
      CK(cudaMemcpyAsync(b->data64 + t * b->tile_data, r->d_data64,
                         (size_t)r->H * r->g.data_pitch * sizeof(double),
                         cudaMemcpyDeviceToDevice, b->st));
    ctx[t] = r->h_ctx;
    ctx[t].data32 = b->data32 + t * b->tile_data;
    ctx[t].data64 = r->d_data64 ? b->data64 + t * b->tile_data : nullptr;
    ctx[t].scal = b->scal + t;
  }
  CK(cudaMemcpyAsync(b->ctx, ctx.data(), n * sizeof(ExactCtx), cudaMemcpyHostToDevice, b->st));
  CK(cudaStreamSynchronize(b->st));
  *out = b;
  return LSE_OK;
}

int lse_batch_advance(lse_batch* b, long long n_steps, lse_status* statuses) {
  if (!b) return fail(LSE_ERR_ARG, "null batch");
  if (n_steps < 0) return fail(LSE_ERR_ARG, "n_steps must be >= 0");
  const int T = b->T;
  lse_run* r0 = b->runs[0];
  const long long it0 = r0->iteration;
  bool all_done = true;
  for (auto* r : b->runs) {
    if (r->iteration != it0 && !r->converged)
      return fail(LSE_ERR_ARG, "batch tiles must be at the same iteration");
    if (r->mode == SRC_FIELD || !fp32_ok(r) || r->mode != r0->mode || r->scale != r0->scale)
      return fail(LSE_ERR_UNSUPPORTED, "batch tiles need binary states on the fast path");
    all_done &= r->converged;
  }
  const long long steps = std::min(n_steps, r0->p.max_iters - it0);
  if (steps > 0 && !all_done) {
    for (auto* r : b->runs) {
      TRY(upload_ctx(r));
      TRY(prepare(r));
    }
    for (auto* r : b->runs) CK(cudaStreamSynchronize(r->st));
    if (b->timing) CK(cudaEventRecord(b->ev[0], b->st));
    // gather: state, partition and checkpoint bits, scalars
    std::vector<const void*> src(T);
    std::vector<void*> dst(T);
    b->cur = 0;
    auto gather = [&](auto srcf, uint32_t* base, long long words) -> int {
      for (int t = 0; t < T; ++t) {
        src[t] = srcf(b->runs[t]);
        dst[t] = base + t * b->tile_words;
      }
      return tiles_copy(b, src, dst, words);
    };
    TRY(gather([](lse_run* r) { return (const void*)r->d_bits[r->cur]; }, b->bits[0], b->tile_words));
    TRY(gather([](lse_run* r) { return (const void*)r->d_P; }, b->P, b->tile_words));
    TRY(gather([](lse_run* r) { return (const void*)r->d_M; }, b->M, b->tile_words));
    for (int t = 0; t < T; ++t) {
      src[t] = b->runs[t]->d_scal;
      dst[t] = b->scal + t;
    }
    TRY(tiles_copy(b, src, dst, sizeof(Scalars) / 4));
    CK(cudaMemsetAsync(b->work, 0, sizeof(unsigned long long), b->st));
    b->work_next = 0;
    bool any_region = false;
    for (auto* r : b->runs) any_region |= two_mean(r->p.model);
    // speculative fused iterations when some tile has a partition to compute
    // every iteration (edge-only batches keep the update-only iterations)
    const bool fz = b->fused && any_region;
    if (fz) {
      // fresh fix-list counters, its capacity and the batch redo flag (tile
      // 0's scalars hold the batch's list state)
      CK(cudaMemsetAsync(reinterpret_cast<char*>(b->scal) + offsetof(Scalars, fix_n), 0,
                         sizeof(unsigned int) * 2, b->st));
      CK(cudaMemsetAsync(reinterpret_cast<char*>(b->scal) + offsetof(Scalars, redo_any), 0,
                         sizeof(int), b->st));
      CK(cudaMemcpyAsync(reinterpret_cast<char*>(b->scal) + offsetof(Scalars, fix_cap),
                         &b->fix_cap, sizeof(unsigned int), cudaMemcpyHostToDevice, b->st));
    }
    const long long cce = r0->p.conv_check_every;
    bool owe = false;                            // the partition of owe_it is owed (fused)
    long long owe_it = 0;
    int src_mode = r0->mode;
    for (long long it = it0 + 1; it <= it0 + steps; ++it) {
      const bool ckpt = it % cce == 0;
      int rc = LSE_ERR_ARG;
      switch (r0->R) {
        case 1: rc = fz && owe ? batch_fused<1>(b, it, owe_it % cce == 0)
                 : fz ? batch_update<1>(b, it, src_mode)
                      : batch_iteration<1>(b, it, ckpt, src_mode, any_region); break;
        case 2: rc = fz && owe ? batch_fused<2>(b, it, owe_it % cce == 0)
                 : fz ? batch_update<2>(b, it, src_mode)
                      : batch_iteration<2>(b, it, ckpt, src_mode, any_region); break;
        case 3: rc = fz && owe ? batch_fused<3>(b, it, owe_it % cce == 0)
                 : fz ? batch_update<3>(b, it, src_mode)
                      : batch_iteration<3>(b, it, ckpt, src_mode, any_region); break;
        case 4: rc = fz && owe ? batch_fused<4>(b, it, owe_it % cce == 0)
                 : fz ? batch_update<4>(b, it, src_mode)
                      : batch_iteration<4>(b, it, ckpt, src_mode, any_region); break;
      }
      TRY(rc);
      owe = fz;
      owe_it = it;
      src_mode = SRC_SMOOTH;
    }
    if (owe) {                                   // the partition of the last iteration
      int rc = LSE_ERR_ARG;
      const bool ck = owe_it % cce == 0;
      switch (r0->R) {
        case 1: rc = batch_partition<1>(b, owe_it, ck, any_region); break;
        case 2: rc = batch_partition<2>(b, owe_it, ck, any_region); break;
        case 3: rc = batch_partition<3>(b, owe_it, ck, any_region); break;
        case 4: rc = batch_partition<4>(b, owe_it, ck, any_region); break;
      }
      TRY(rc);
    }
    // collect + scatter back into the runs
    unsigned long long work = 0;
    CK(cudaMemcpyAsync(b->h_scal, b->scal, T * sizeof(Scalars), cudaMemcpyDeviceToHost, b->st));
    CK(cudaMemcpyAsync(&work, b->work, sizeof(work), cudaMemcpyDeviceToHost, b->st));
    CK(cudaStreamSynchronize(b->st));
#ifdef LSE_UNIT_TRACE
    trace_flush();
#endif
    if (work != b->work_next) {
      char msg[128];
      std::snprintf(msg, sizeof(msg), "batch work-counter mismatch: device %llu, expected %llu",
                    work, b->work_next);
      return fail(LSE_ERR_CUDA, msg);
    }
    auto scatter = [&](auto dstf, const uint32_t* base, long long words) -> int {
      for (int t = 0; t < T; ++t) {
        src[t] = base + t * b->tile_words;
        dst[t] = dstf(b->runs[t]);
      }
      return tiles_copy(b, src, dst, words);
    };
    TRY(scatter([](lse_run* r) { return (void*)r->d_bits[r->cur]; }, b->bits[b->cur], b->tile_words));
    TRY(scatter([](lse_run* r) { return (void*)r->d_P; }, b->P, b->tile_words));
    TRY(scatter([](lse_run* r) { return (void*)r->d_M; }, b->M, b->tile_words));
    for (int t = 0; t < T; ++t) {
      src[t] = b->scal + t;
      dst[t] = b->runs[t]->d_scal;
    }
    TRY(tiles_copy(b, src, dst, sizeof(Scalars) / 4));
    if (b->timing) {
      CK(cudaEventRecord(b->ev[1], b->st));
      CK(cudaEventSynchronize(b->ev[1]));
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, b->ev[0], b->ev[1]));
      b->t_ms += ms;
      b->t_calls += 1;
    }
    for (int t = 0; t < T; ++t) {
      lse_run* r = b->runs[t];
      const Scalars& s = b->h_scal[t];
      *r->h_scal = s;
      if (!r->converged) {
        r->iteration = s.converged ? s.converged_iter : it0 + steps;
        r->converged = s.converged != 0;
        r->fast_iters += steps;
      }
      r->degenerate = s.degenerate != 0;
      r->mode = SRC_SMOOTH;
      r->field_valid = false;
      r->prepared = true;
      r->launched.clear();
    }
  }
  if (statuses)
    for (int t = 0; t < T; ++t) fill_status(b->runs[t], statuses + t, -1);
  return LSE_OK;
}

int lse_batch_set_timing(lse_batch* b, int enabled) {
  if (!b) return fail(LSE_ERR_ARG, "null batch");
  if (enabled && !b->ev[0]) {
    CK(cudaEventCreate(&b->ev[0]));
    CK(cudaEventCreate(&b->ev[1]));
  }
  b->timing = enabled != 0;
  b->t_ms = 0.0;
  b->t_calls = 0;
  return LSE_OK;
}

int lse_batch_elapsed(lse_batch* b, double* ms, long long* calls) {
  if (!b || !ms) return fail(LSE_ERR_ARG, "null argument");
  *ms = b->t_ms;
  if (calls) *calls = b->t_calls;
  return LSE_OK;
}

void lse_batch_destroy(lse_batch* b) {
  if (!b) return;
  if (b->st) cudaStreamSynchronize(b->st);
  for (cudaEvent_t e : b->ev)
    if (e) cudaEventDestroy(e);
  void* ptrs[] = {b->bits[0], b->bits[1], b->P, b->M, b->data32, b->data64, b->scal,
                  b->ctx, b->part, b->part_fin, b->work, (void*)b->d_src, (void*)b->d_dst,
                  (void*)b->fix};
  for (void* q : ptrs)
    if (q) cudaFree(q);
  if (b->h_scal) cudaFreeHost(b->h_scal);
  if (b->st) cudaStreamDestroy(b->st);
  delete b;
}

void lse_run_destroy(lse_run* r) {
  if (!r) return;
  if (r->st) cudaStreamSynchronize(r->st);
  void* ptrs[] = {r->d_px, r->d_py, r->d_mag, r->d_edt_g, r->d_edt_v, r->d_edt_zn,
                  r->d_edt_zd, r->d_dist[0], r->d_dist[1],
                  r->d_scratch, r->d_poly, r->d_offs, r->d_flag,
                  r->d_bands32, r->d_bands64, r->d_chg, r->d_bpart, r->d_pmax, r->d_lut64,
                  r->d_work, r->d_part_fin, r->d_part_init, r->d_data32, r->d_data64, r->d_bits[0], r->d_bits[1], r->d_P, r->d_M,
                  r->d_mask, r->d_part, r->d_scal, r->d_lut_t, r->d_lut_s, r->d_ctx,
                  r->d_w64, r->d_keys, r->d_count, r->d_F[0], r->d_F[1], r->d_U, r->d_T,
                  r->d_fix, r->d_res_parts, r->d_sync};
  for (void* q : ptrs)
    if (q) cudaFree(q);
  if (r->h_scal) cudaFreeHost(r->h_scal);
  for (auto e : r->evpool) cudaEventDestroy(e);
  if (r->t_begin) cudaEventDestroy(r->t_begin);
  if (r->t_end) cudaEventDestroy(r->t_end);
  if (r->st) cudaStreamDestroy(r->st);
  delete r;
}


}  // extern "C"

// ------------------------------------------------------- stateless kernels
namespace {

struct DevBuf {
  void* p = nullptr;
  ~DevBuf() { if (p) cudaFree(p); }
};

template <typename T>
int dbuf(DevBuf& b, size_t n) {
  T* q = nullptr;
  TRY(dalloc(&q, n));
  b.p = q;
  return LSE_OK;
}

std::vector<double> taps_from_axis(const double* w, int ts) {
  const int R = ts / 2;
  std::vector<double> out(R + 1);
  for (int d = 0; d <= R; ++d) out[d] = w[R - d];
  return out;
}

int conv_device(const double* d_in, double* d_tmp, double* d_out, int H, int W, const double* w,
                int ts) {
  auto taps = taps_from_axis(w, ts);
  DevBuf dw;
  TRY(dbuf<double>(dw, taps.size()));
  CK(cudaMemcpy(dw.p, taps.data(), taps.size() * sizeof(double), cudaMemcpyHostToDevice));
  k_corr<0><<<grid2(W, H), 128>>>(d_in, d_tmp, H, W, (double*)dw.p, ts / 2);
  CKL();
  k_corr<1><<<grid2(W, H), 128>>>(d_tmp, d_out, H, W, (double*)dw.p, ts / 2);
  CKL();
  CK(cudaDeviceSynchronize());
  return LSE_OK;
}

// region coefficients (c+, c-, peak) of (image, phi) into a device Scalars
int region_scalars(const double* d_img, const double* d_phi, int H, int W, Scalars* d_sc,
                   Scalars* h_sc, int model = REGION, double nu = 0.0) {
  const long long n = (long long)H * W;
  const int blocks = std::min<long long>((n + 255) / 256, num_sms() * 4);
  DevBuf part, keys;
  TRY(dbuf<TilePartial>(part, blocks));
  TRY(dbuf<long long>(keys, 3));
  Scalars s0;
  std::memset(&s0, 0, sizeof(s0));
  s0.n_total = n;
  s0.model = model;
  s0.nu = nu;
  CK(cudaMemcpy(d_sc, &s0, sizeof(s0), cudaMemcpyHostToDevice));
  long long init[3] = {LLONG_MAX, LLONG_MIN, LLONG_MIN};
  CK(cudaMemcpy(keys.p, init, sizeof(init), cudaMemcpyHostToDevice));
  k_minmax<<<std::min(H, num_sms() * 8), 256>>>(nullptr, d_img, H, W, W, (long long*)keys.p);
  CKL();
  k_store_minmax<<<1, 1>>>((long long*)keys.p, d_sc);
  CKL();
  k_region_sums<<<blocks, 256>>>(d_img, d_phi, n, (TilePartial*)part.p);
  CKL();
  k_finalize<<<1, 1024>>>((TilePartial*)part.p, blocks, d_sc, 0, 1, 0, 0);
  CKL();
  CK(cudaMemcpy(h_sc, d_sc, sizeof(Scalars), cudaMemcpyDeviceToHost));
  return LSE_OK;
}

}  // namespace

extern "C" {

int lse_edge_function(const double* image, long long h, long long w, const double* weights,
                      int ts, double gain, double* g_out) {
  if (!image || !weights || !g_out || ts < 1 || ts % 2 == 0) return fail(LSE_ERR_ARG, "bad arguments");
  if (h < 2 || w < 2) return fail(LSE_ERR_ARG, "gradient needs at least a 2x2 field");
  TRY(check_device());
  const long long n = h * w;
  DevBuf a, b, c;
  TRY(dbuf<double>(a, n));
  TRY(dbuf<double>(b, n));
  TRY(dbuf<double>(c, n));
  CK(cudaMemcpy(a.p, image, n * sizeof(double), cudaMemcpyHostToDevice));
  TRY(conv_device((double*)a.p, (double*)b.p, (double*)c.p, (int)h, (int)w, weights, ts));
  k_edge_g<<<grid2((int)w, (int)h), 128>>>((double*)c.p, (int)h, (int)w, gain, (double*)a.p,
                                           nullptr, w, 1.0);
  CKL();
  CK(cudaMemcpy(g_out, a.p, n * sizeof(double), cudaMemcpyDeviceToHost));
  return LSE_OK;
}

int lse_convolve_same(const double* f, long long h, long long w, const double* weights, int ts,
                      double* out) {
  if (!f || !weights || !out || ts < 1 || ts % 2 == 0 || h < 1 || w < 1)
    return fail(LSE_ERR_ARG, "bad arguments");
  TRY(check_device());
  const long long n = h * w;
  DevBuf a, b, c;
  TRY(dbuf<double>(a, n));
  TRY(dbuf<double>(b, n));
  TRY(dbuf<double>(c, n));
  CK(cudaMemcpy(a.p, f, n * sizeof(double), cudaMemcpyHostToDevice));
  TRY(conv_device((double*)a.p, (double*)b.p, (double*)c.p, (int)h, (int)w, weights, ts));
  CK(cudaMemcpy(out, c.p, n * sizeof(double), cudaMemcpyDeviceToHost));
  return LSE_OK;
}

int lse_correlate2d(const double* f, long long h, long long w, const double* weights, int ts,
                    double* out) {
  if (!f || !weights || !out || ts < 1 || ts % 2 == 0 || h < 1 || w < 1)
    return fail(LSE_ERR_ARG, "bad arguments");
  TRY(check_device());
  const long long n = h * w;
  DevBuf a, b, dw;
  TRY(dbuf<double>(a, n));
  TRY(dbuf<double>(b, n));
  TRY(dbuf<double>(dw, (size_t)ts * ts));
  CK(cudaMemcpy(a.p, f, n * sizeof(double), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dw.p, weights, (size_t)ts * ts * sizeof(double), cudaMemcpyHostToDevice));
  k_corr2d<<<grid2((int)w, (int)h), 128>>>((double*)a.p, (double*)b.p, (int)h, (int)w,
                                           (double*)dw.p, ts);
  CKL();
  CK(cudaMemcpy(out, b.p, n * sizeof(double), cudaMemcpyDeviceToHost));
  return LSE_OK;
}

int lse_gradient(const double* f, long long h, long long w, double* fx, double* fy,
                 double* magnitude) {
  if (!f) return fail(LSE_ERR_ARG, "bad arguments");
  if (h < 2 || w < 2) return fail(LSE_ERR_ARG, "gradient needs at least a 2x2 field");
  TRY(check_device());
  const long long n = h * w;
  DevBuf a, bx, by, bm;
  TRY(dbuf<double>(a, n));
  TRY(dbuf<double>(bx, n));
  TRY(dbuf<double>(by, n));
  TRY(dbuf<double>(bm, n));
  CK(cudaMemcpy(a.p, f, n * sizeof(double), cudaMemcpyHostToDevice));
  k_gradient<<<grid2((int)w, (int)h), 128>>>((double*)a.p, (int)h, (int)w, (double*)bx.p,
                                             (double*)by.p, (double*)bm.p);
  CKL();
  if (fx) CK(cudaMemcpy(fx, bx.p, n * sizeof(double), cudaMemcpyDeviceToHost));
  if (fy) CK(cudaMemcpy(fy, by.p, n * sizeof(double), cudaMemcpyDeviceToHost));
  if (magnitude) CK(cudaMemcpy(magnitude, bm.p, n * sizeof(double), cudaMemcpyDeviceToHost));
  return LSE_OK;
}

int lse_binarize(const double* phi, long long n, double* out) {
  if (!phi || !out || n < 0) return fail(LSE_ERR_ARG, "bad arguments");
  if (n == 0) return LSE_OK;
  TRY(check_device());
  DevBuf a;
  TRY(dbuf<double>(a, n));
  CK(cudaMemcpy(a.p, phi, n * sizeof(double), cudaMemcpyHostToDevice));
  k_binarize<<<num_sms() * 8, 256>>>((double*)a.p, (double*)a.p, n);
  CKL();
  CK(cudaMemcpy(out, a.p, n * sizeof(double), cudaMemcpyDeviceToHost));
  return LSE_OK;
}

int lse_region_means(const double* image, const double* phi, long long h, long long w,
                     double* c_plus, double* c_minus) {
  if (!image || !phi || h < 1 || w < 1) return fail(LSE_ERR_ARG, "bad arguments");
  TRY(check_device());
  const long long n = h * w;
  DevBuf a, b, sc;
  TRY(dbuf<double>(a, n));
  TRY(dbuf<double>(b, n));
  TRY(dbuf<Scalars>(sc, 1));
  CK(cudaMemcpy(a.p, image, n * sizeof(double), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(b.p, phi, n * sizeof(double), cudaMemcpyHostToDevice));
  Scalars hs;
  TRY(region_scalars((double*)a.p, (double*)b.p, (int)h, (int)w, (Scalars*)sc.p, &hs));
  if (hs.n_pos == 0 || hs.n_pos == n)
    return fail(LSE_ERR_DEGENERATE, "one side of the partition is empty");
  if (c_plus) *c_plus = hs.c_pos;
  if (c_minus) *c_minus = hs.c_neg;
  return LSE_OK;
}

namespace {
// region_velocity (models.py:101-119) / zhang_velocity (models.py:144-162)
int two_mean_velocity(const double* image, const double* phi, long long h, long long w,
                      int model, double nu, double* v_out, int* degenerate) {
  if (!image || !phi || !v_out || h < 1 || w < 1) return fail(LSE_ERR_ARG, "bad arguments");
  TRY(check_device());
  const long long n = h * w;
  DevBuf a, b, v, sc;
  TRY(dbuf<double>(a, n));
  TRY(dbuf<double>(b, n));
  TRY(dbuf<double>(v, n));
  TRY(dbuf<Scalars>(sc, 1));
  CK(cudaMemcpy(a.p, image, n * sizeof(double), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(b.p, phi, n * sizeof(double), cudaMemcpyHostToDevice));
  Scalars hs;
  TRY(region_scalars((double*)a.p, (double*)b.p, (int)h, (int)w, (Scalars*)sc.p, &hs, model, nu));
  if (degenerate) *degenerate = hs.zero_vel;
  if (hs.zero_vel) {
    // models.py:111-118, 156-157: zero field, degenerate = True, gradient not evaluated
    std::memset(v_out, 0, n * sizeof(double));
    return LSE_OK;
  }
  if (h < 2 || w < 2) return fail(LSE_ERR_ARG, "gradient needs at least a 2x2 field");
  k_velocity<REGION><<<grid2((int)w, (int)h), 128>>>((double*)b.p, (double*)v.p, (int)h, (int)w,
                                                     (double*)a.p, (Scalars*)sc.p);
  CKL();
  CK(cudaMemcpy(v_out, v.p, n * sizeof(double), cudaMemcpyDeviceToHost));
  return LSE_OK;
}
}  // namespace

int lse_region_velocity(const double* image, const double* phi, long long h, long long w,
                        double* v_out, int* degenerate) {
  return two_mean_velocity(image, phi, h, w, REGION, 0.0, v_out, degenerate);
}

int lse_curvature(const double* phi, long long h, long long w, double eps_guard, double* out) {
  if (!phi || !out) return fail(LSE_ERR_ARG, "bad arguments");
  if (!(eps_guard > 0.0)) return fail(LSE_ERR_ARG, "eps_guard must be positive");
  if (h < 3 || w < 3) return fail(LSE_ERR_ARG, "curvature needs at least a 3x3 field");
  TRY(check_device());
  const long long n = h * w;
  DevBuf a, px, py, k;
  TRY(dbuf<double>(a, n));
  TRY(dbuf<double>(px, n));
  TRY(dbuf<double>(py, n));
  TRY(dbuf<double>(k, n));
  CK(cudaMemcpy(a.p, phi, n * sizeof(double), cudaMemcpyHostToDevice));
  k_gradient<<<grid2((int)w, (int)h), 128>>>((double*)a.p, (int)h, (int)w, (double*)px.p,
                                             (double*)py.p, nullptr);
  CKL();
  k_curvature<<<grid2((int)w, (int)h), 128>>>((double*)px.p, (double*)py.p, (int)h, (int)w,
                                              eps_guard, (double*)k.p);
  CKL();
  CK(cudaMemcpy(out, k.p, n * sizeof(double), cudaMemcpyDeviceToHost));
  return LSE_OK;
}

int lse_signed_distance(const unsigned char* mask, long long h, long long w, double* out) {
  if (!mask || !out || h < 1 || w < 1) return fail(LSE_ERR_ARG, "bad arguments");
  TRY(check_device());
  const long long n = h * w;
  long long objs = 0;
  for (long long q = 0; q < n; ++q) objs += mask[q] != 0;
  if (objs == 0) return fail(LSE_ERR_ARG, "mask has no object pixels");
  if (objs == n) return fail(LSE_ERR_ARG, "mask has no background pixels");
  std::vector<double> f(n);
  for (long long q = 0; q < n; ++q) f[q] = mask[q] ? 1.0 : -1.0;
  DevBuf a, g, v, zn, zd, d0, d1, o;
  TRY(dbuf<double>(a, n));
  TRY(dbuf<long long>(g, n));
  TRY(dbuf<int>(v, n));
  TRY(dbuf<long long>(zn, h * (w + 1)));
  TRY(dbuf<long long>(zd, h * (w + 1)));
  TRY(dbuf<double>(d0, n));
  TRY(dbuf<double>(d1, n));
  TRY(dbuf<double>(o, n));
  CK(cudaMemcpy(a.p, f.data(), n * sizeof(double), cudaMemcpyHostToDevice));
  TRY(neg_signed_distance(0, (double*)a.p, (double*)o.p, (int)h, (int)w, (long long*)g.p,
                          (int*)v.p, (long long*)zn.p, (long long*)zd.p, (double*)d0.p,
                          (double*)d1.p));
  CK(cudaMemcpy(out, o.p, n * sizeof(double), cudaMemcpyDeviceToHost));
  for (long long q = 0; q < n; ++q) out[q] = -out[q];   // positive outside (kernels.py:131-133)
  return LSE_OK;
}

int lse_cv_velocity(const double* image, const double* phi, long long h, long long w, double mu,
                    double* v_out) {
  if (!image || !phi || !v_out) return fail(LSE_ERR_ARG, "bad arguments");
  if (h < 3 || w < 3) return fail(LSE_ERR_ARG, "curvature needs at least a 3x3 field");
  TRY(check_device());
  const long long n = h * w;
  DevBuf a, b, px, py, mag, v, sc;
  TRY(dbuf<double>(a, n));
  TRY(dbuf<double>(b, n));
  TRY(dbuf<double>(px, n));
  TRY(dbuf<double>(py, n));
  TRY(dbuf<double>(mag, n));
  TRY(dbuf<double>(v, n));
  TRY(dbuf<Scalars>(sc, 1));
  CK(cudaMemcpy(a.p, image, n * sizeof(double), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(b.p, phi, n * sizeof(double), cudaMemcpyHostToDevice));
  Scalars hs;
  TRY(region_scalars((double*)a.p, (double*)b.p, (int)h, (int)w, (Scalars*)sc.p, &hs));
  k_gradient<<<grid2((int)w, (int)h), 128>>>((double*)b.p, (int)h, (int)w, (double*)px.p,
                                             (double*)py.p, (double*)mag.p);
  CKL();
  k_cv_update<<<grid2((int)w, (int)h), 128>>>(nullptr, (double*)px.p, (double*)py.p,
                                              (double*)mag.p, (double*)v.p, (int)h, (int)w,
                                              nullptr, (double*)a.p, w, (Scalars*)sc.p, 0.0, mu,
                                              1e-10);
  CKL();
  CK(cudaMemcpy(v_out, v.p, n * sizeof(double), cudaMemcpyDeviceToHost));
  return LSE_OK;
}

int lse_zhang_velocity(const double* image, const double* phi, long long h, long long w, double nu,
                       double* v_out, int* degenerate) {
  return two_mean_velocity(image, phi, h, w, ZHANG, nu, v_out, degenerate);
}

int lse_edge_velocity(const double* g, const double* phi, long long h, long long w, double* v_out) {
  if (!g || !phi || !v_out) return fail(LSE_ERR_ARG, "bad arguments");
  if (h < 2 || w < 2) return fail(LSE_ERR_ARG, "gradient needs at least a 2x2 field");
  TRY(check_device());
  const long long n = h * w;
  DevBuf a, b, v;
  TRY(dbuf<double>(a, n));
  TRY(dbuf<double>(b, n));
  TRY(dbuf<double>(v, n));
  CK(cudaMemcpy(a.p, g, n * sizeof(double), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(b.p, phi, n * sizeof(double), cudaMemcpyHostToDevice));
  k_velocity<EDGE><<<grid2((int)w, (int)h), 128>>>((double*)b.p, (double*)v.p, (int)h, (int)w,
                                                   (double*)a.p, nullptr);
  CKL();
  CK(cudaMemcpy(v_out, v.p, n * sizeof(double), cudaMemcpyDeviceToHost));
  return LSE_OK;
}

int lse_rasterize_seeds(const double* poly_xy, const long long* poly_counts, long long n_polys,
                        int inside_sign, long long h, long long w, signed char* out) {
  if (!poly_xy || !poly_counts || !out || n_polys < 1 || h < 1 || w < 1)
    return fail(LSE_ERR_ARG, "bad arguments");
  TRY(check_device());
  std::vector<long long> offs(n_polys + 1, 0);
  for (long long k = 0; k < n_polys; ++k) offs[k + 1] = offs[k] + poly_counts[k];
  RunGeom g{};
  g.H = (int)h;
  g.W = (int)w;
  g.HR = (int)((h + 31) / 32);
  g.pitch_w = (int)w;
  DevBuf dxy, doffs, dsig, dcnt;
  TRY(dbuf<double>(dxy, 2 * offs.back()));
  TRY(dbuf<long long>(doffs, offs.size()));
  TRY(dbuf<signed char>(dsig, h * w));
  TRY(dbuf<unsigned long long>(dcnt, 1));
  CK(cudaMemcpy(dxy.p, poly_xy, 2 * offs.back() * sizeof(double), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(doffs.p, offs.data(), offs.size() * sizeof(long long), cudaMemcpyHostToDevice));
  CK(cudaMemset(dcnt.p, 0, sizeof(unsigned long long)));
  k_rasterize<<<dim3((unsigned)((w + 127) / 128), g.HR), 128>>>(
      (double*)dxy.p, (long long*)doffs.p, (int)n_polys, inside_sign, nullptr,
      (signed char*)dsig.p, g, (unsigned long long*)dcnt.p, 0);
  CKL();
  unsigned long long cnt = 0;
  CK(cudaMemcpy(&cnt, dcnt.p, sizeof(cnt), cudaMemcpyDeviceToHost));
  if (cnt == 0) return fail(LSE_ERR_DEGENERATE_SEED, "seed polygons cover no pixel centers");
  if ((long long)cnt == h * w) return fail(LSE_ERR_DEGENERATE_SEED, "seed polygons cover the entire grid");
  CK(cudaMemcpy(out, dsig.p, h * w, cudaMemcpyDeviceToHost));
  return LSE_OK;
}

}  // extern "C"

// ------------------------------------------------------------------ contours
struct lse_contours {
  std::vector<long long> offsets{0};   // point offsets, n_contours + 1
  std::vector<double> xy;              // (x, y) = (col + 0.5, row + 0.5) per point
};

namespace {

// extract_contours (engine.py:280-294) of a dense device field on stream st.
int contours_device(const double* d_phi, long long H, long long W, cudaStream_t st,
                    lse_contours* out) {
  const long long rows = std::max(H - 1, 1LL);
  DevBuf cnt, off, fl, sg;
  TRY(dbuf<long long>(cnt, rows));
  TRY(dbuf<long long>(off, rows + 1));
  TRY(dbuf<unsigned>(fl, 1));
  CK(cudaMemsetAsync(fl.p, 0, sizeof(unsigned), st));
  k_contour_rows<false><<<(unsigned)rows, kContourThreads, 0, st>>>(
      d_phi, H, W, (long long*)cnt.p, nullptr, nullptr, (unsigned*)fl.p);
  CKL();
  k_contour_scan<<<1, 1024, 0, st>>>((const long long*)cnt.p, rows, (long long*)off.p);
  CKL();
  long long total = 0;
  unsigned signs = 0;
  CK(cudaMemcpyAsync(&total, (long long*)off.p + rows, sizeof(long long), cudaMemcpyDeviceToHost,
                     st));
  CK(cudaMemcpyAsync(&signs, fl.p, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (signs != 3u || total == 0) return LSE_OK;      // single-signed: no zero crossing
  TRY(dbuf<Seg>(sg, total));
  k_contour_rows<true><<<(unsigned)rows, kContourThreads, 0, st>>>(
      d_phi, H, W, nullptr, (const long long*)off.p, (Seg*)sg.p, nullptr);
  CKL();
  std::vector<Seg> segs(total);
  CK(cudaMemcpyAsync(segs.data(), sg.p, total * sizeof(Seg), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  const auto lines = ms_assemble(segs);
  long long npts = 0;
  for (const auto& l : lines) npts += (long long)l.size();
  out->offsets.reserve(lines.size() + 1);
  out->xy.reserve(2 * npts);
  for (const auto& l : lines) {
    for (const MsPoint& q : l) {
      out->xy.push_back(q.c + 0.5);
      out->xy.push_back(q.r + 0.5);
    }
    out->offsets.push_back((long long)out->xy.size() / 2);
  }
  return LSE_OK;
}

}  // namespace

extern "C" {

int lse_contours_from_field(const double* phi, int phi_on_device, long long h, long long w,
                            lse_contours** out) {
  if (!phi || !out || h < 1 || w < 1) return fail(LSE_ERR_ARG, "bad arguments");
  *out = nullptr;
  TRY(check_device());
  DevBuf a;
  const double* d = phi;
  if (!phi_on_device) {
    TRY(dbuf<double>(a, h * w));
    CK(cudaMemcpy(a.p, phi, h * w * sizeof(double), cudaMemcpyHostToDevice));
    d = (const double*)a.p;
  }
  auto* c = new lse_contours();
  const int rc = contours_device(d, h, w, 0, c);
  if (rc != LSE_OK) {
    delete c;
    return rc;
  }
  *out = c;
  return LSE_OK;
}

int lse_run_contours(lse_run* r, lse_contours** out) {
  if (!r || !out) return fail(LSE_ERR_ARG, "null argument");
  if (r->strip) return fail(LSE_ERR_ARG, "contours of a row strip: gather the strips' phi");
  *out = nullptr;
  TRY(ensure_generic(r));
  const double* src;
  if (r->field_valid) {
    src = r->d_F[r->curF];
  } else {
    TRY(upload_ctx(r));
    k_phi_from_bits<<<grid2(r->W, r->H), 128, 0, r->st>>>(r->d_bits[r->cur], r->d_U, r->d_ctx,
                                                           r->mode);
    CKL();
    src = r->d_U;
  }
  auto* c = new lse_contours();
  const int rc = contours_device(src, r->H, r->W, r->st, c);
  if (rc != LSE_OK) {
    delete c;
    return rc;
  }
  *out = c;
  return LSE_OK;
}

int lse_contours_size(const lse_contours* c, long long* n_contours, long long* n_points) {
  if (!c || !n_contours || !n_points) return fail(LSE_ERR_ARG, "null argument");
  *n_contours = (long long)c->offsets.size() - 1;
  *n_points = c->offsets.back();
  return LSE_OK;
}

int lse_contours_read(const lse_contours* c, long long* offsets, double* xy) {
  if (!c || !offsets || (!xy && c->offsets.back() > 0)) return fail(LSE_ERR_ARG, "null argument");
  memcpy(offsets, c->offsets.data(), c->offsets.size() * sizeof(long long));
  if (!c->xy.empty()) memcpy(xy, c->xy.data(), c->xy.size() * sizeof(double));
  return LSE_OK;
}

void lse_contours_destroy(lse_contours* c) { delete c; }

}  // extern "C"
