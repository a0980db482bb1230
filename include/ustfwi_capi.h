/*
 * ustfwi_capi.h — C ABI of the B200-native TD-FWI gradient engine (libustfwi_b200.so).
 *
 * This is the drop-in boundary for the hot path of arXiv 2102.00755 as implemented by
 * the reference C++ library (/root/reference/proj/include/ustfwi). Every entry point
 * names the reference interface it replaces (file:line, paths relative to
 * proj/include/ustfwi/). Plain pointers and sizes only: no torch, no C++ types.
 * The C++ drop-in headers (include/ustfwi/*.hpp) wrap these calls back into the
 * reference's value types and exceptions; INTEGRATION.md shows the bindings.
 *
 * Conventions
 *   - Every function returns a status: USTFWI_OK (0) or one of USTFWI_ERR_*.
 *     USTFWI_ERR_INVALID   <-> std::invalid_argument   (grid.hpp:35-51, medium.hpp:41-57)
 *     USTFWI_ERR_NUMERICAL <-> ustfwi::NumericalError  (core/errors.hpp:10-12)
 *     The message of the last failure is returned by ustfwi_last_error() (per thread).
 *   - Host buffers are owned by the caller. The API is fp64 at the boundary
 *     (field.hpp:38,89); device arithmetic is fp32 (loss and adjoint-source scan fp64).
 *   - Fields are row-major with the last axis fastest (field.hpp:14-17). 1-D and 2-D
 *     grids are accepted and run as 3-D grids with leading singleton axes.
 *   - A context is the device analogue of one SpectralEngine + its WaveSteppers
 *     (engine.hpp:14-16, "one engine per worker"): not thread-safe, one CUDA stream.
 *   - There is NO CPU fallback: without a usable sm_100 device, ustfwi_gpu_create fails
 *     with USTFWI_ERR_CUDA.
 */
#ifndef USTFWI_CAPI_H
#define USTFWI_CAPI_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define USTFWI_API __attribute__((visibility("default")))
#else
#define USTFWI_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define USTFWI_OK 0
#define USTFWI_ERR_INVALID 1
#define USTFWI_ERR_NUMERICAL 2
#define USTFWI_ERR_CUDA 3
#define USTFWI_ERR_OOM 4
#define USTFWI_ERR_NCCL 5

#define USTFWI_STAGGER_NONE 0  /* Stagger::none  (spectral.hpp:15) */
#define USTFWI_STAGGER_PLUS 1  /* Stagger::plus  */
#define USTFWI_STAGGER_MINUS 2 /* Stagger::minus */

/* Field-for-field image of ustfwi::Grid (grid/grid.hpp:14-20); unused axes are 0. */
typedef struct ustfwi_grid {
    int ndim;
    int dims[3];
    double dx[3];
    double dt;
    int nt;
    int pml_size[3];
    double c_ref;
} ustfwi_grid;

USTFWI_API const char* ustfwi_last_error(void);
USTFWI_API const char* ustfwi_version(void);

/* ------------------------------------------------------------------------------------
 * Host-side setup (C++ in the library; no device needed)
 * ------------------------------------------------------------------------------------ */

/* Grid::validate (grid.hpp:35-51). */
USTFWI_API int ustfwi_grid_validate(const ustfwi_grid* grid);
/* choose_pml_size (grid.hpp:70-86). */
USTFWI_API int ustfwi_choose_pml_size(int ndim, const int* interior, int* pml_out);
/* make_grid (grid.hpp:91-103). */
USTFWI_API int ustfwi_make_grid(int ndim, const int* interior, double dx, double c_max, double duration,
                     double cfl, ustfwi_grid* out);
/* make_pml (grid.hpp:153-178): regular/staggered are concatenated per axis (sum of dims). */
USTFWI_API int ustfwi_make_pml(const ustfwi_grid* grid, double alpha, double* regular, double* staggered);
/* shell_indices (solver/medium.hpp:168-178) with erode (:137-165). Two-call protocol:
 * out == NULL queries *count; otherwise writes min(*count, n) indices, sets *count = n. */
USTFWI_API int ustfwi_shell_indices(int ndim, const int* dims, const uint8_t* mask, int thickness,
                         size_t* out, size_t* count);
/* ball_mask (solver/medium.hpp:181-198). */
USTFWI_API int ustfwi_ball_mask(int ndim, const int* dims, const double* center, double radius_points,
                     uint8_t* out);
/* synth_source_pulse (solver/simulate.hpp:124-148); same two-call protocol via *len. */
USTFWI_API int ustfwi_synth_source_pulse(const ustfwi_grid* grid, double center_freq_fraction, double c0_min,
                              double* out, int* len);
/* design_kaiser_lowpass (grid/filter.hpp:38-66): odd-length Kaiser FIR taps with unit DC gain;
 * two-call protocol via *len (out == NULL queries the length). */
USTFWI_API int ustfwi_design_kaiser_lowpass(double dt, double cutoff_hz, double transition, double atten_db,
                                            double* out, int* len);
/* Encoding realization (SPEC.md stochastic_estimators, EncodingRealization :277-280, RNG
 * contract :331-334): Rademacher weights w_i in {-1,+1} and delays d_i ~ U[0,1] quantized to
 * delay_steps_i = round(d_i * tau / dt), from a counter-based stream keyed by
 * (master_seed, iteration, index). Bit-identical for identical keys. */
USTFWI_API int ustfwi_draw_realization(size_t n_src, double tau, double dt, uint64_t master_seed,
                            uint64_t iteration, uint64_t index, int8_t* weights,
                            int32_t* delay_steps, double* delays_unit);

/* fp64 host FFT over interleaved complex data [dims] (row-major): the reference's
 * ComplexFft (core/fft.hpp:75-118; FFTW conventions: forward e^{-i}, unnormalised; inverse
 * e^{+i}, scaled by 1/N when normalize != 0). Serves the fp64 setup utilities of the drop-in
 * headers (spectral_derivative, fourier_shift, RealFft); never the device hot path. */
USTFWI_API int ustfwi_host_fft(int ndim, const int* dims, double* data, int inverse, int normalize);

/* ------------------------------------------------------------------------------------
 * Device engine
 * ------------------------------------------------------------------------------------ */
typedef struct ustfwi_gpu_ctx ustfwi_gpu_ctx;

/* SpectralEngine(grid) (engine.hpp:19-79): validates the grid, builds the per-axis FFT
 * plans / wavenumber and stagger tables on `device`, allocates state for two steppers. */
USTFWI_API int ustfwi_gpu_create(int device, const ustfwi_grid* grid, ustfwi_gpu_ctx** out);
USTFWI_API void ustfwi_gpu_destroy(ustfwi_gpu_ctx* ctx);

/* Medium (solver/medium.hpp:26-58) + the per-medium part of the WaveStepper constructor
 * (engine.hpp:184-259): CFL guard (NumericalError), c0^2, dt*rho0, dt/rho0 staggered via
 * fourier_shift. alpha0 may be NULL (lossless); gamma may be NULL. alpha0 != 0 enables the
 * power-law absorption of update_pressure (engine.hpp:233-246,327-343; dispersion term
 * unless y == 2) and the absorption terms of the c0 gradient (gradient.hpp:63-74,183-203). */
USTFWI_API int ustfwi_gpu_set_medium(ustfwi_gpu_ctx* ctx, const double* c0, const double* rho0,
                          const double* alpha0, double y, const uint8_t* gamma, double c0_min,
                          double c0_max);

/* GradientOptions::dispersion_enabled (adjoint/gradient.hpp:22-32): the dispersion term of the
 * adjoint and time-reversal steppers and of the gradient's absorption terms (gradient.hpp:56,
 * 381-384, 424-426); the forward simulation keeps it (default StepperOptions). Default 1. */
USTFWI_API int ustfwi_gpu_set_gradient_options(ustfwi_gpu_ctx* ctx, int dispersion_enabled);

/* GradientParam of the next gradient (adjoint/gradient.hpp:9, GradientAccumulator :50-142):
 * USTFWI_PARAM_C0 (default), USTFWI_PARAM_ALPHA0, USTFWI_PARAM_Y. USTFWI_PARAM_RHO0 is
 * rejected with USTFWI_ERR_INVALID (the reference branch is defective). */
#define USTFWI_PARAM_C0 0
#define USTFWI_PARAM_RHO0 1
#define USTFWI_PARAM_ALPHA0 2
#define USTFWI_PARAM_Y 3
USTFWI_API int ustfwi_gpu_set_gradient_param(ustfwi_gpu_ctx* ctx, int param);

/* SourceSet (solver/medium.hpp:74-85), generalised to encoded super-sources: source i fires
 * at flat index pos[i] with sample(i, n) = w_i * sig[sig_off[i] + n - delay_i] when
 * 0 <= n - delay_i < sig_off[i+1] - sig_off[i], else 0. weights / delay_steps may be NULL
 * (w = 1, delay = 0): the plain reference SourceSet. */
USTFWI_API int ustfwi_gpu_set_sources(ustfwi_gpu_ctx* ctx, size_t n_src, const size_t* pos,
                           const size_t* sig_off, const double* sig, const double* weights,
                           const int32_t* delay_steps);
/* SensorArray (solver/medium.hpp:88-91). */
USTFWI_API int ustfwi_gpu_set_sensors(ustfwi_gpu_ctx* ctx, size_t n_sensors, const size_t* pos);
/* Simulation length of the following forward / gradient calls (Grid::nt, grid.hpp:18):
 * delayed source encoding runs over the extended duration T + tau, nt_ext = nt +
 * ceil(tau/dt). Observed data must be re-uploaded afterwards. */
USTFWI_API int ustfwi_gpu_set_nt(ustfwi_gpu_ctx* ctx, int nt);

/* simulate_forward (solver/simulate.hpp:30-105). data_out: [n_sensors * nt] sensor-major
 * (SensorData, medium.hpp:94-114). If boundary_thickness > 0 the shell trace
 * (BoundaryTrace, medium.hpp:118-133) is recorded; trace_out (nullable) receives
 * [nt * n_shell] step-major and *n_shell_out the shell size. */
USTFWI_API int ustfwi_gpu_forward(ustfwi_gpu_ctx* ctx, int boundary_thickness, double* data_out,
                       double* trace_out, size_t* n_shell_out);

/* gradient_time_reversal / compute_gradient TR branch (adjoint/gradient.hpp:333-464,478-488)
 * for GradientParam::c0: forward with shell record, adjoint source (reverse, Kahan loss,
 * cumsum; :264-289), interleaved adjoint + time-reversal replay with in-kernel c0
 * correlation, gradient zeroed outside gamma. observed: [n_sensors * nt] sensor-major. */
USTFWI_API int ustfwi_gpu_gradient_tr(ustfwi_gpu_ctx* ctx, const double* observed, int boundary_thickness,
                           double* grad_out, double* loss_out);

/* evaluate_loss (adjoint/gradient.hpp:491-505). */
USTFWI_API int ustfwi_gpu_evaluate_loss(ustfwi_gpu_ctx* ctx, const double* observed, double* loss_out);

/* SpectralEngine::derivative (engine.hpp:118-121): out = d/dx_axis f on the grid staggered
 * by stagger (USTFWI_STAGGER_*). Test/diagnostic entry of the K1 passes. */
USTFWI_API int ustfwi_gpu_derivative(ustfwi_gpu_ctx* ctx, const double* f, int axis, int stagger,
                          double* out);

/* SpectralEngine::half_shift (engine.hpp:131-137): band-limited shift by direction * dx/2
 * along axis (the Nyquist bin keeps its real part). */
USTFWI_API int ustfwi_gpu_half_shift(ustfwi_gpu_ctx* ctx, const double* f, int axis, int direction, double* out);

/* ---- WaveStepper, step by step (solver/engine.hpp:170-386) ----
 * A context hosts two steppers (which = 0, 1) on its bound medium. init = the constructor with
 * StepperOptions {pml_enabled, absorption_sign, dispersion_enabled} (:170-177,184-259) and a
 * zero state; update_velocity_density (:270-292); inject = inject_mass_source for n positions
 * applied in order (:296-300); enforce = enforce_shell with density values (:304-307);
 * refresh_pressure = refresh_pressure_from_density (:311-316); update_pressure (:318-347; a
 * NumericalError every 64th step when p[0] is not finite); read = pressure() / velocity()[a] /
 * the split densities as fp64 (field 0 p, 1..ndim v_a, 4..3+ndim rho_a); gather = p at n
 * positions. The hot path (forward / gradient) never goes through these calls. */
USTFWI_API int ustfwi_gpu_stepper_init(ustfwi_gpu_ctx* ctx, int which, int pml_enabled, double absorption_sign,
                                       int dispersion_enabled);
USTFWI_API int ustfwi_gpu_stepper_reset(ustfwi_gpu_ctx* ctx, int which);
USTFWI_API int ustfwi_gpu_stepper_update_velocity_density(ustfwi_gpu_ctx* ctx, int which);
USTFWI_API int ustfwi_gpu_stepper_inject(ustfwi_gpu_ctx* ctx, int which, size_t n, const size_t* idx,
                                         const double* amplitude);
USTFWI_API int ustfwi_gpu_stepper_enforce(ustfwi_gpu_ctx* ctx, int which, size_t n, const size_t* idx,
                                          const double* values);
USTFWI_API int ustfwi_gpu_stepper_refresh_pressure(ustfwi_gpu_ctx* ctx, int which);
USTFWI_API int ustfwi_gpu_stepper_update_pressure(ustfwi_gpu_ctx* ctx, int which);
USTFWI_API int ustfwi_gpu_stepper_read(ustfwi_gpu_ctx* ctx, int which, int field, double* out);
USTFWI_API int ustfwi_gpu_stepper_gather(ustfwi_gpu_ctx* ctx, int which, size_t n, const size_t* idx, double* out);
USTFWI_API int ustfwi_gpu_stepper_step_index(ustfwi_gpu_ctx* ctx, int which, int* out);

/* ---- device-resident variants (inputs already in HBM; used by the benchmark and by the
 *      multi-GPU mini-batch driver) ---- */
USTFWI_API int ustfwi_gpu_upload_observed(ustfwi_gpu_ctx* ctx, const double* observed);
/* One TR gradient from the uploaded observed data; the result stays on the device and is
 * ADDED to the context's mini-batch accumulator when accumulate != 0 (else replaces it). */
USTFWI_API int ustfwi_gpu_run_gradient(ustfwi_gpu_ctx* ctx, int boundary_thickness, int accumulate);
/* Copy the accumulator (gradient and loss, divided by `scale_div` >= 1) to the host. */
USTFWI_API int ustfwi_gpu_download_gradient(ustfwi_gpu_ctx* ctx, double scale_div, double* grad_out,
                                 double* loss_out);
/* Device pointer of the fp32 gradient accumulator (N floats) and its loss (1 double). */
USTFWI_API int ustfwi_gpu_accumulator(ustfwi_gpu_ctx* ctx, float** grad_dev, double** loss_dev);
USTFWI_API int ustfwi_gpu_synchronize(ustfwi_gpu_ctx* ctx);
/* Stream the engine launches on (cudaStream_t as void*). */
USTFWI_API void* ustfwi_gpu_stream(ustfwi_gpu_ctx* ctx);
/* Number of kernel launches issued by this context since creation. */
USTFWI_API uint64_t ustfwi_gpu_launch_count(const ustfwi_gpu_ctx* ctx);
/* Shell size of the last forward with boundary recording. */
USTFWI_API size_t ustfwi_gpu_shell_size(const ustfwi_gpu_ctx* ctx);

/* ---- per-launch-class device timing (CUDA events on the engine stream) ---- */
#define USTFWI_KERNEL_Y 0    /* y-pencil FFT passes */
#define USTFWI_KERNEL_X 1    /* x-pencil FFT * kappa * D_x * IFFT passes */
#define USTFWI_KERNEL_ZVEL 2 /* fused z c2r + velocity update + r2c */
#define USTFWI_KERNEL_ZRHO 3 /* fused z c2r + density/pressure/sparse/correlation + r2c */
#define USTFWI_KERNEL_AUX 4
#define USTFWI_KERNEL_CHAIN 5 /* fused y-x-y chain (y forward, x * kappa * D_x * inverse, y inverse) */
#define USTFWI_KERNEL_KINDS 6
/* Fused y-x-y chain kernel wait statistics (only with USTFWI_CHAIN_STATS=1; diagnostics):
 * out[0] CTAs, out[1] units, out[2] deferred tile loads, out[3] dependency-wait cycles,
 * out[4] tile-wait cycles, summed over CTAs since the previous call. */
USTFWI_API int ustfwi_gpu_chain_stats(uint64_t* out5);
/* SM partition of the TR gradient's adjoint / replay pair loop (green contexts; no reference
 * counterpart, the reference runs both steppers on the host thread in turn, gradient.hpp:443-461):
 * SMs of the adjoint and of the replay stream, 0 / 0 when both share the device. */
USTFWI_API int ustfwi_gpu_partition(ustfwi_gpu_ctx* ctx, int* adjoint_sms, int* replay_sms);
/* Enable/disable event timing of every launch and reset the counters. */
USTFWI_API int ustfwi_gpu_set_profiling(ustfwi_gpu_ctx* ctx, int enable);
/* Accumulated device time, launch count and algorithmic bytes (minimum HBM traffic of the
 * launches: half-spectrum and field reads + writes) of one launch class. */
USTFWI_API int ustfwi_gpu_kernel_stats(ustfwi_gpu_ctx* ctx, int kind, double* total_ms,
                                       uint64_t* launches, double* bytes);

/* ---- mini-batch mean over GPUs (SPEC.md average_estimates :314-322, worker-count
 *      independence :328,337; PAPER §4.5) ---- */
/* ncclGetUniqueId into 128 bytes. */
USTFWI_API int ustfwi_nccl_unique_id(char id_out[128]);
/* Bind an NCCL communicator (one rank per GPU) to the context. */
USTFWI_API int ustfwi_gpu_comm_init(ustfwi_gpu_ctx* ctx, const char id[128], int nranks, int rank);
/* Reserve `slots` per-realization gradient slots on this rank (cleared to zero). A mini-batch
 * of B realizations over W ranks uses slots = ceil(B / W); realization r runs on rank r mod W
 * in slot r / W (an idle rank keeps empty slots and still joins the mean). */
USTFWI_API int ustfwi_gpu_batch_reserve(ustfwi_gpu_ctx* ctx, int slots);
/* One TR gradient from the uploaded observed data into `slot` (masked gradient + loss). */
USTFWI_API int ustfwi_gpu_run_gradient_slot(ustfwi_gpu_ctx* ctx, int boundary_thickness, int slot);
/* Deterministic mean: all-gather every rank's slots (NCCL, when a communicator is bound), sum
 * the B realizations in realization order in fp64 and scale by 1/B into the accumulator (read
 * with ustfwi_gpu_download_gradient(ctx, 1, ...)); the loss likewise. The result is
 * bit-identical for every world size. */
USTFWI_API int ustfwi_gpu_batch_mean(ustfwi_gpu_ctx* ctx, int batch);

/* ---- SLBFGS curvature history on the device (Algorithm 2 / Appendix D; SPEC.md
 * optimizer: two_loop_recursion, LbfgsState with m_h = 64). fp64 vectors of length n; S, Y
 * rings, rho_i and H0 = gamma I (gamma = <s,y>/<y,y> of the newest pair) stay in HBM. ---- */
typedef struct ustfwi_lbfgs ustfwi_lbfgs;
USTFWI_API int ustfwi_lbfgs_create(int device, size_t n, int history, ustfwi_lbfgs** out);
USTFWI_API int ustfwi_lbfgs_destroy(ustfwi_lbfgs* h);
/* Forget all pairs (H0 = I). */
USTFWI_API int ustfwi_lbfgs_reset(ustfwi_lbfgs* h);
/* updateBuffer(s, S), updateBuffer(y, Y) (Algorithm 2); the pair is rejected (*accepted = 0)
 * unless <s,y> > reject_tol * |s| |y| (SPEC design decision, default 1e-10). Host or device
 * vectors (unified addressing; device vectors stay in HBM). */
USTFWI_API int ustfwi_lbfgs_push(ustfwi_lbfgs* h, const double* s, const double* y, double reject_tol, int* accepted);
/* out = H_k g by the two-loop recursion (empty history: g). Host or device vectors. */
USTFWI_API int ustfwi_lbfgs_apply(ustfwi_lbfgs* h, const double* g, double* out);
/* Number of stored pairs and the current H0 scaling. */
USTFWI_API int ustfwi_lbfgs_pairs(const ustfwi_lbfgs* h, int* count, double* gamma);

/* ---- multigrid transfer on the device (§3.3, Appendix C) ----
 * fourier_interpolate (grid/spectral.hpp:166-212): field [dims] -> out [new_dims], every
 * target dim even and >= 4, every source dim even; blackman != 0 applies the separable
 * Blackman taper (prolong_model). Host fp64 buffers. */
USTFWI_API int ustfwi_fourier_interpolate(int device, int ndim, const int* dims, const double* field,
                                          const int* new_dims, int blackman, double* out);
/* lowpass_filter_timeseries (grid/filter.hpp:88-101) of n_series rows of len samples. */
USTFWI_API int ustfwi_lowpass_timeseries(int device, size_t n_series, size_t len, const double* sig, double dt,
                                         double cutoff_hz, double transition, double atten_db, double* out);
/* restrict_data: [n_series][nt] -> [n_series][ceil(nt/eta)], Fourier
 * resampling, Kaiser low-pass (transition 0.1, 60 dB) at cutoff_hz, scale eta^(ndim-1).
 * out == NULL: only *nt_out is set. */
USTFWI_API int ustfwi_restrict_traces(int device, size_t n_series, size_t nt, const double* data, int eta, int ndim,
                                      double dt_fine, double cutoff_hz, double* out, size_t* nt_out);

#ifdef __cplusplus
}
#endif

#endif /* USTFWI_CAPI_H */
