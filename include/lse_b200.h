/*
 * lse_b200.h -- C ABI of the B200-native fast level-set-evolution (LSE) path.
 *
 * The reference (`lsekit` 0.1.0, pure Python) has no FFI: its drop-in
 * boundary is the Python module API (lsekit/__init__.py:3-32).  The entry
 * points below are the seams a maintainer would bind from that API; each
 * names the reference function it replaces.  Plain pointers and sizes only:
 * images/fields are row-major (H, W) host arrays unless stated otherwise.
 * All calls are synchronous with respect to the caller (they return after
 * the device work finished) and thread-safe per handle.
 *
 * Errors: every int-returning call returns LSE_OK (0) or an LSE_ERR_* code;
 * lse_last_error() gives the message of the calling thread's last failure.
 */
#ifndef LSE_B200_H
#define LSE_B200_H

#ifdef __cplusplus
extern "C" {
#endif

#define LSE_ABI_VERSION 6

#define LSE_OK 0
#define LSE_ERR_ARG 1            /* ValueError in the reference               */
#define LSE_ERR_CUDA 2           /* device/runtime failure                    */
#define LSE_ERR_INSTABILITY 3    /* NumericalInstabilityError (engine.py:29)  */
#define LSE_ERR_DEGENERATE 4     /* DegeneratePartitionError (grid.py:20)     */
#define LSE_ERR_NODEVICE 5       /* no CUDA device visible                    */
#define LSE_ERR_DEGENERATE_SEED 6 /* DegenerateSeedError (grid.py:16)         */
#define LSE_ERR_UNSUPPORTED 7    /* configuration outside the device paths    */

#define LSE_MODEL_EDGE 0         /* ModelKind.EDGE   (models.py:30)  E_Td, Eq. 14 */
#define LSE_MODEL_REGION 1       /* ModelKind.REGION (models.py:31)  R_Td, Eq. 17 */
#define LSE_MODEL_ZHANG 2        /* ModelKind.ZHANG  (models.py:33)  mean separation (models.py:144-162) */
#define LSE_MODEL_CV 4           /* ModelKind.CHAN_VESE (models.py:32): curvature-regularized
                                    baseline (models.py:122-141), distance re-init (generic path) */
#define LSE_MODEL_BANDS 3        /* region data term summed over n_bands bands (
                                    a restatement -- the reference is single-band) */

/* EvolutionParams + ModelParams (engine.py:40-81, models.py:44-68).  The
 * Gaussian 1-D weights are passed in exactly as
 * gaussian_kernel(sigma, ts).axis_weights (kernels.py:50-64) computes them,
 * so host and oracle share one weight vector bit-for-bit. */
typedef struct lse_params {
  int model;
  double dt;
  double sigma2;
  int ts_reg;
  int reinit_period;
  int reg_period;
  long long max_iters;
  long long conv_check_every;
  long long conv_window;
  double sigma1;
  int ts_pre;
  double edge_gain;
  const double* reg_weights; /* ts_reg values */
  const double* pre_weights; /* ts_pre values (edge model) */
  double nu;                 /* ModelParams.nu (zhang model speed constant) */
  int n_bands;               /* LSE_MODEL_BANDS: bands of the image (1..4), band-major */
  double mu;                 /* ModelParams.mu (LSE_MODEL_CV curvature weight) */
} lse_params;

#define LSE_PHI0_FIELD 0     /* float64 (H, W) level-set field                 */
#define LSE_PHI0_SIGNS 1     /* int8 (H, W) in {-1, +1}; phi = sign * scale     */
#define LSE_PHI0_POLYGONS 2  /* seed polygons, rasterized on the device         */

/* Initial / injected state: EvolutionState (engine.py:98-103) or a SeedSpec
 * (grid.py:34-55) rasterized by rasterize_seeds (grid.py:76-93). */
typedef struct lse_phi0 {
  int kind;
  const double* field;            /* LSE_PHI0_FIELD                          */
  const signed char* signs;       /* LSE_PHI0_SIGNS                          */
  double scale;                   /* LSE_PHI0_SIGNS magnitude (> 0)          */
  const double* poly_xy;          /* LSE_PHI0_POLYGONS: concatenated (x, y)  */
  const long long* poly_counts;   /* vertices per polygon                    */
  long long n_polys;
  int inside_sign;                /* +1 / -1                                 */
  long long iteration;            /* EvolutionState.iteration                */
  int converged;                  /* EvolutionState.converged                */
  int degenerate;                 /* EvolutionState.degenerate               */
  long long row_offset;           /* LSE_PHI0_POLYGONS: global row of local row 0
                                     (row strips; 0 otherwise)               */
} lse_phi0;

typedef struct lse_status {
  long long iteration;             /* EvolutionState.iteration                */
  int converged;                   /* EvolutionState.converged                */
  int degenerate;                  /* EvolutionState.degenerate (sticky)      */
  long long instability_iteration; /* NumericalInstabilityError.iteration / -1 */
  long long exact_fallbacks;       /* fp64 re-evaluations of near-tie pixels  */
  long long fast_iterations;       /* iterations run by the fused bit-state path */
  long long generic_iterations;    /* iterations run by the fp64 field path   */
} lse_status;

typedef struct lse_run lse_run;

/* ---- library ----------------------------------------------------------- */
int lse_abi_version(void);
const char* lse_last_error(void);
int lse_device_count(void);

/* Image formats of lse_run_create / lse_run_load_image (image_is_f32). */
#define LSE_IMAGE_F64 0     /* float64 (H, W)                                     */
#define LSE_IMAGE_F32 1     /* float32 (H, W)                                     */
#define LSE_IMAGE_RGB8 2    /* uint8 (H, W, 3): decoded to the loader's luma
                               ((0.299 R + 0.587 G) + 0.114 B) / 255 in float64
                               (fileio.py:28-30, 88) on the device            */

/* ---- the resumable driver: EvolutionRun (engine.py:193-269) -------------- */

/* EvolutionRun.__init__ (engine.py:202-216): uploads the image, builds the
 * edge indicator on the device for the edge model (engine.py:210-211), and
 * sets the initial state (init_state, engine.py:123-133).  image is float64
 * (image_is_f32 = 0) or float32 (image_is_f32 = 1). */
int lse_run_create(lse_run** out, const lse_params* p, long long height, long long width,
                   const void* image, int image_is_f32, const lse_phi0* init);

/* Replace the image of an existing run (same shape), keeping its buffers. */
int lse_run_load_image(lse_run* run, const void* image, int image_is_f32);

/* EvolutionRun.state = ... (engine.py:207, 239): inject a state; the
 * checkpoint history is kept, as in the reference. */
int lse_run_set_state(lse_run* run, const lse_phi0* st);

/* EvolutionRun.advance(n_steps) (engine.py:242-254), i.e. up to n_steps
 * calls of _advance_once (engine.py:148-174) + convergence bookkeeping
 * (engine.py:222-240).  Returns LSE_ERR_INSTABILITY with
 * st->instability_iteration set when the update produced NaN/Inf; the state
 * then stays at the last good iteration (engine.py:150-153). */
int lse_run_advance(lse_run* run, long long n_steps, lse_status* st);

int lse_run_status(lse_run* run, lse_status* st);

/* EvolutionRun.state.phi: float64 (H, W), bit-identical to the reference's
 * G * b when the state is binary-regularized. */
int lse_run_read_phi(lse_run* run, double* out);

/* EvolutionRun.mask() (engine.py:256-259): (phi > 0) if inside_sign > 0
 * else (phi <= 0).  packed = 0 -> uint8 (H, W) of 0/1; packed = 1 -> row-major
 * bits, numpy.packbits(mask, axis=None) order (ceil(H*W/8) bytes). */
int lse_run_read_mask(lse_run* run, unsigned char* out, int inside_sign, int packed);

/* Device-event timing on the run's stream: everything the run enqueues
 * between begin and end (bench support). */
int lse_run_begin_timing(lse_run* run);
int lse_run_end_timing(lse_run* run, double* ms);

/* Run options.  "skip_uniform" (default 1, or the environment's
 * LSE_SKIP_UNIFORM at creation): let the fused kernels copy warp blocks
 * whose whole stencil window is uniform (exactly unchanged by the update)
 * instead of recomputing them; 0 forces the dense pass. */
int lse_run_set_option(lse_run* run, const char* name, long long value);

/* Number of kernel launches this library has issued (process-wide). */
long long lse_launch_count(void);

/* Guard certification (the validation build liblse_b200_check.so, `make
 * check`): every fp32 decision value of the fused kernels -- u of the update,
 * phi of the partition -- is also evaluated in the reference's fp64 order
 * (every LSE_CHECK_EVERY-th iteration, default 1).  lse_check_stats fills
 * out[8] = {max |u32-u64|/eps_u, max |phi32-phi64|/eps_phi, min |u64|,
 * min |phi64|, fp32 decisions outside the guard band that differ from fp64
 * (u, phi), values checked, thread slots used}; reset != 0 clears them.
 * lse_check_enabled() is 1 in that build only. */
int lse_check_enabled(void);
int lse_check_stats(double* out, int reset);

/* Device-event timing of the fused kernels (bench/roofline support). */
int lse_run_set_profiling(lse_run* run, int enabled);
int lse_run_kernel_times(lse_run* run, double* update_ms, long long* update_launches,
                         double* partition_ms, long long* partition_launches);

/* Speculative fused iterations (single tiled region / zhang runs; the
 * library's own execution strategy, invisible in the results): out[4] =
 * {fused iterations launched, of which redone whole, pixels decided from the
 * fix list, fused path enabled (0/1)}.  LSE_FUSED=0 at creation disables it. */
int lse_run_spec_stats(lse_run* run, long long* out4);

/* Multi-band runs: out[2] = {peak passes reused (a partition that moved no
 * pixel leaves the band means, the data term D, max|D| and the coefficients
 * bit-identical, so the pass over every pixel is not repeated), reuse
 * enabled (0/1)}.  LSE_BAND_REUSE=0 at creation disables the reuse. */
int lse_run_band_stats(lse_run* run, long long* out2);

/* Small single images (lse_resident.cuh): a whole lse_run_advance call runs as
 * one resident kernel -- iterations separated by cluster / grid barriers
 * instead of kernel launches (replaces the launch chain of engine.py:242-254's
 * loop; same results).  out[5] = {resident path enabled (0/1), barrier kind
 * (0 one thread-block cluster, 1 cooperative grid), CTAs of the launch,
 * advance calls served, tasks (32 rows x 8 columns) per warp}.
 * LSE_RESIDENT=0 at creation disables it, 2 forces the grid barrier. */
int lse_run_resident_stats(lse_run* run, long long* out5);

void lse_run_destroy(lse_run* run);

/* ---- batched tiles -----------------------------------------
 * Many equal-size runs advanced together with one launch per kernel per
 * iteration for all of them.  Tiles share size and evolution parameters and
 * may differ in model (region / zhang / edge), image and seeds; each must be on
 * the binary-state fast path (reinit_period = reg_period = 1) at the same
 * iteration.  Each tile evolves exactly as it would alone: the per-tile
 * reductions keep the single-run order.  After lse_batch_advance the run
 * handles hold the new states (status, read_phi, read_mask work per tile);
 * statuses (n entries, optional) receive their lse_status.  The batch
 * borrows the runs: destroy it before them. */
typedef struct lse_batch lse_batch;
int lse_batch_create(lse_batch** out, lse_run* const* runs, int n_runs);
int lse_batch_advance(lse_batch* batch, long long n_steps, lse_status* statuses);
/* Device-event timing of whole lse_batch_advance calls (gather, iterations,
 * scatter on the batch's stream): set_timing(1) clears and starts it,
 * elapsed returns the summed milliseconds and the number of timed calls. */
int lse_batch_set_timing(lse_batch* batch, int enabled);
int lse_batch_elapsed(lse_batch* batch, double* ms, long long* calls);
void lse_batch_destroy(lse_batch* batch);

/* ---- row strips: one rank's share of a multi-GPU run --------
 * A rank owns whole word-rows (32 image rows) of the global grid and holds
 * one halo word-row of each neighbour.  Per iteration of _advance_once
 * (engine.py:148-174), with the exchanges between the phases done by the
 * caller's communicator on lse_run_stream(run):
 *   lse_strip_update      update of iteration n+1 (b^n -> b^{n+1})
 *   <halo exchange>       own first/last word-row -> neighbours' halo rows
 *                         (lse_run_bits_row pointers, pitch_words uint32 each)
 *   lse_strip_partition   partition / checkpoint pass -> one partial
 *                         (LSE_PARTIAL_BYTES) per rank, if *partition_next
 *   <allgather>           the ranks' partials, in rank order
 *   lse_strip_finalize    c+/c-, coefficients, convergence -- identical on
 *                         every rank (same partials, same fixed order)
 * Setup: lse_strip_create (local rows incl. halos, seeds in local
 * coordinates, n_total = global pixel count), lse_strip_image_range ->
 * allreduce min/max/max|.| -> lse_strip_set_image_range, lse_strip_prepare
 * -> allgather -> lse_strip_finalize(absolute = 1).  Row strips run the
 * binary-state fast path only (reinit_period = reg_period = 1). */
#define LSE_PARTIAL_BYTES 64
int lse_strip_create(lse_run** out, const lse_params* p, long long height, long long width,
                     const void* image, int image_is_f32, const lse_phi0* init, int own_lo,
                     int own_hi, long long n_total);
int lse_strip_image_range(lse_run* run, double* min_max_absmax);
int lse_strip_set_image_range(lse_run* run, const double* min_max_absmax);
int lse_strip_prepare(lse_run* run, void* partial_out);
int lse_strip_update(lse_run* run, int* partition_next);
int lse_strip_partition(lse_run* run, void* partial_out);
int lse_strip_finalize(lse_run* run, const void* partials, int n_partials, int absolute);
/* One-pass iteration of a strip (the speculative fused pass):
 * the partition of the current state -- owed by the last lse_strip_update or
 * lse_strip_fused -- and the update of the next iteration in one launch
 * sequence; partial_out receives this rank's partition partial.  The ranks
 * exchange them, lse_strip_finalize(absolute = 0) checks the prediction and
 * decides the undecided pixels (or redoes the update); only then exchange the
 * halo rows.  LSE_ERR_UNSUPPORTED when the strip runs the two-pass iteration
 * (lse_run_spec_stats out[3] == 0). */
int lse_strip_fused(lse_run* run, void* partial_out);
int lse_strip_sync(lse_run* run, lse_status* st);
void* lse_run_stream(lse_run* run);
void* lse_run_bits_row(lse_run* run, int word_row);
int lse_run_geometry(lse_run* run, int* word_rows, int* pitch_words);

/* ---- stateless kernels of the public API --------------------------------- */

/* edge_function (models.py:71-81): g = 1/(1 + (gain fx)^2 + (gain fy)^2). */
int lse_edge_function(const double* image, long long h, long long w,
                      const double* weights, int ts, double gain, double* g_out);

/* convolve_same (kernels.py:67-78), separable, zero padding. */
int lse_convolve_same(const double* f, long long h, long long w,
                      const double* weights, int ts, double* out);

/* convolve_same with a non-separable Kernel2D (kernels.py:77-78,
 * ndimage.correlate, zero padding); weights is ts x ts row-major. */
int lse_correlate2d(const double* f, long long h, long long w,
                    const double* weights, int ts, double* out);

/* gradient_central / gradient_magnitude (kernels.py:81-95). */
int lse_gradient(const double* f, long long h, long long w,
                 double* fx, double* fy, double* magnitude);

/* binarize (grid.py:96-99). */
int lse_binarize(const double* phi, long long n, double* out);

/* region_means (grid.py:102-118); LSE_ERR_DEGENERATE on an empty side. */
int lse_region_means(const double* image, const double* phi, long long h, long long w,
                     double* c_plus, double* c_minus);

/* region_velocity (models.py:101-119) and edge_velocity (models.py:84-90). */
int lse_region_velocity(const double* image, const double* phi, long long h, long long w,
                        double* v_out, int* degenerate);
int lse_edge_velocity(const double* g, const double* phi, long long h, long long w,
                      double* v_out);

/* curvature (kernels.py:98-115), signed_distance (kernels.py:118-133; mask
 * uint8 0/1, exact Euclidean, positive outside), cv_velocity (models.py:
 * 122-141, eps_guard 1e-10 as the reference calls it). */
int lse_curvature(const double* phi, long long h, long long w, double eps_guard, double* out);
int lse_signed_distance(const unsigned char* mask, long long h, long long w, double* out);
int lse_cv_velocity(const double* image, const double* phi, long long h, long long w, double mu,
                    double* v_out);

/* zhang_velocity (models.py:144-162); *degenerate as region_velocity. */
int lse_zhang_velocity(const double* image, const double* phi, long long h, long long w, double nu,
                       double* v_out, int* degenerate);

/* rasterize_seeds (grid.py:76-93): +-1 as int8; LSE_ERR_DEGENERATE_SEED when
 * the union covers no pixel centre or every pixel centre. */
int lse_rasterize_seeds(const double* poly_xy, const long long* poly_counts, long long n_polys,
                        int inside_sign, long long h, long long w, signed char* out);

/* ---- zero-level contours (extract_contours, engine.py:280-294) ---------- */

/* Marching squares at level 0 (scikit-image find_contours, fully_connected
 * 'low', positive_orientation 'low'): polylines of (x, y) = (col + 0.5,
 * row + 0.5) points, in the published assembly's order; none when phi is
 * single-signed.  The result is host memory owned by the handle. */
typedef struct lse_contours lse_contours;
int lse_contours_from_field(const double* phi, int phi_on_device, long long h, long long w,
                            lse_contours** out);
/* contours of a run's current phi, computed on the device without a phi
 * download (EvolutionRun.contours, engine.py:260-261; the trace, 214-238) */
int lse_run_contours(lse_run* run, lse_contours** out);
int lse_contours_size(const lse_contours* c, long long* n_contours, long long* n_points);
/* offsets: n_contours + 1 point offsets; xy: 2 * n_points doubles */
int lse_contours_read(const lse_contours* c, long long* offsets, double* xy);
void lse_contours_destroy(lse_contours* c);

#ifdef __cplusplus
}
#endif
#endif /* LSE_B200_H */
