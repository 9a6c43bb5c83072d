/*
 * ptycho_b200.h -- C ABI of the B200 rPIE hot path (libptycho_b200.so).
 *
 * Plain pointers and sizes only; no torch types.  Every device pointer is a
 * raw CUDA device address borrowed for the duration of the call; `stream` is a
 * cudaStream_t passed as void*.  All calls are stream-ordered and return a
 * host status (PTY_OK or PTY_ERR_*); data-dependent failures detected on the
 * device (bounds, degenerate probe/object, negative intensity) are OR-ed into
 * a device int32 status word that the caller reads after synchronising.
 *
 * Reference interfaces replaced (paths relative to /root/reference/pkg/src/ptychokit):
 *   pty_sweep            engine.py:173-243  sweep()  (inner loop engine.py:191-233)
 *                          + fields.py:87-107 crop / paste_add_inplace
 *                          + engine.py:104-150 magnitude_correct / update_object / update_probe
 *   pty_sweep_subpixel   (extension) simulate.py:157-166 extract_view applied to the sweep's crops
 *   pty_fft2             fields.py:71-84 propagate()  (centered=1), and the
 *                          uncentered np.fft.fft2/ifft2 of registration.py:47,71
 *   pty_register_batch   registration.py:43-128 cross_power_spectrum / coarse_shift /
 *                          refine_shift / register  (+ posref.py:57-84 sensors)
 *   pty_adam_apply       posref.py:87-113 adam_step + apply_correction
 *   pty_init_probes      engine.py:83-95 (mode-1 back-propagation, mode Gram-Schmidt)
 *   pty_orthogonalize    engine.py:153-164 _orthogonalize_modes
 *   pty_check_patterns   engine.py:111-112 (DataError on I < 0), checked once at upload
 *   pty_magnitude_correct / pty_update_object / pty_update_probe
 *                        engine.py:104-150 (the per-visit functions, one call each)
 *   pty_cross_power_spectrum / pty_coarse_argmax / pty_upsampled_idft / pty_argmax_abs
 *                        registration.py:43-120 (the per-pair pipeline, step by step)
 *   pty_adam_step / pty_apply_correction
 *                        posref.py:87-113 (one position)
 *   pty_batch_contrib / pty_batch_apply / pty_batch_finalize
 *                        batched (semi-parallel) extension -- no reference
 *                        counterpart; CPU statement oracle/batched.py
 */
#ifndef PTYCHO_B200_H
#define PTYCHO_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PTY_ABI_VERSION 1

#if defined(__GNUC__)
#define PTY_API __attribute__((visibility("default")))
#else
#define PTY_API
#endif

/* host status and device status bits (paper_2205_04295_b200/errors.py) */
#define PTY_OK              0
#define PTY_ERR_BOUNDS      (1 << 0)  /* crop box outside the canvas        -> BoundsError */
#define PTY_ERR_PROBE_ZERO  (1 << 1)  /* max sum_m |P_m|^2 == 0              -> DegenerateInputError */
#define PTY_ERR_OBJECT_ZERO (1 << 2)  /* max |o_j|^2 == 0 with probe update  -> DegenerateInputError */
#define PTY_ERR_NEGATIVE_I  (1 << 3)  /* measured intensity < 0              -> DataError */
#define PTY_ERR_ARGUMENT    (1 << 8)  /* bad argument                        -> ParameterError */
#define PTY_ERR_CUDA        (1 << 9)  /* CUDA runtime error                  -> NativeError */

#define PTY_DTYPE_C64  0   /* complex64  (float2 interleaved), real = float32 */
#define PTY_DTYPE_C128 1   /* complex128 (double2 interleaved), real = float64 */

#define PTY_SENSE_NONE    0
#define PTY_SENSE_XCORR_A 1   /* posref.py:66-76 register(o_j, o'_j, "raw") */
#define PTY_SENSE_XCORR_B 2   /* posref.py:79-84 register(total, I_j, "raw") */

/*
 * One reconstruction (a "slot") swept by pty_sweep.  Several slots in one call
 * are independent reconstructions advanced in lock step (replica mode); one
 * slot is the reference's sequential sweep.
 */
typedef struct PtySlot {
    void*          obj;          /* [H][Wc] complex, row-major, updated in place   */
    int32_t        H, Wc;        /* canvas shape                                    */
    int32_t        r0, c0;       /* canvas origin (engine.py:77-81)                 */
    void*          probes;       /* [M][W][W] complex, updated in place             */
    const void*    patterns;     /* [N][W][W] real (measured intensity I)           */
    const void*    patterns_t;   /* [N][W][W] real, each pattern transposed         */
    const double*  positions;    /* [N][2] (x, y) float64                           */
    const int32_t* order;        /* [N] visit order of this sweep (engine.py:177-181) */
    void*          stage;        /* posref staging [N][2][W][W] complex or NULL     */
    double*        err_out;      /* [3]: err_num, err_den, modulus_worst (written)  */
    int32_t*       status;       /* device status word of this slot (OR-ed)         */
} PtySlot;

typedef struct PtySweepArgs {
    int32_t dtype;               /* PTY_DTYPE_*                                    */
    int32_t window;              /* W: power of two, 16..512                        */
    int32_t modes;               /* M: 1..8                                         */
    int32_t n_positions;         /* N (same for every slot)                          */
    int32_t n_slots;
    const PtySlot* slots;        /* HOST array of n_slots descriptors               */
    double  alpha_obj, alpha_probe, beta, gamma, epsilon_rel;
    int32_t update_probe;        /* update_probe_modes && alpha_probe > 0           */
    int32_t track_modulus;       /* track_modulus_error                             */
    int32_t sense;               /* PTY_SENSE_*: what pty_sweep stages for posref   */
    void*   workspace;           /* device scratch, >= pty_sweep_workspace_bytes()  */
    int64_t workspace_bytes;
} PtySweepArgs;

PTY_API int pty_abi_version(void);

/* Number of kernels this library has launched in the process (all devices). */
PTY_API int64_t pty_launch_count(void);

/* Microbenchmark of the sweep kernel's software grid barrier: `ctas` CTAs of
 * 512 threads (0 = one per SM) cross `iters` barriers; synchronous. */
PTY_API int pty_barrier_bench(int32_t iters, int32_t ctas, double* ns_per_barrier);

/* Debug: globaltimer stamps [steps][5][grid] of the last pty_sweep run with
 * PTY_TIMELINE=<steps> in the environment (k=0 step start, k=1..4 end of
 * P1..P4 per CTA).  Returns the number of stamps, copies min(n, cap). */
PTY_API int64_t pty_timeline(uint64_t* out, int64_t cap, int32_t* grid);

/* SM count, max cooperative CTAs for the sweep kernel, compute capability. */
PTY_API int pty_device_info(int32_t* sm_count, int32_t* coop_ctas, int32_t* cc_major, int32_t* cc_minor);

/* bytes of device workspace pty_sweep needs for these sizes */
PTY_API int64_t pty_sweep_workspace_bytes(int32_t dtype, int32_t window, int32_t modes,
                                  int32_t n_positions, int32_t n_slots);

/* One full sweep (every position of every slot) as one cooperative kernel. */
PTY_API int pty_sweep(const PtySweepArgs* args, void* stream);

/* Opt-in subpixel reconstruction gather (extension, no reference counterpart;
 * SolverConfig.subpixel_gather): the sweep of pty_sweep with every crop shifted
 * by its position's residual (simulate.py:157-166 applied to reconstruction)
 * and the object update shifted back before the paste.  Same arguments as
 * pty_sweep (workspace unused); track_modulus must be 0. */
PTY_API int pty_sweep_subpixel(const PtySweepArgs* args, void* stream);

/* In-place batched 2D FFT of `batch` W x W complex fields.
 * centered=1: fields.py propagate (fftshift . fft2 . ifftshift, norm="ortho");
 * centered=0: np.fft.fft2 (inverse=0, unnormalised) / np.fft.ifft2 (inverse=1, 1/W^2). */
PTY_API int pty_fft2(void* data, int32_t dtype, int32_t window, int32_t batch, int32_t inverse,
             int32_t centered, void* stream);

/*
 * Batched registration (registration.py:123-128) of n pairs.
 * work: [n][2][W][W] complex; plane 0 = reference, plane 1 = moving on entry
 *       (overwritten).  real_inputs = 1: ref_real/mov_real ([n][W][W] real)
 *       are loaded instead and `work` is only scratch; real_inputs = 2 (dtype
 *       C128 only): ref_real points at complex64 pairs [n][2][W][W] that are
 *       widened to float64 while loading (fp32 states registered in float64).
 * weighting: 0 = "phase", 1 = "raw".  kappa in {1} U [2, 1000].
 * Outputs (device): dy, dx, peak [n] float64; ok [n] int32 (0 = degenerate spectrum).
 */
PTY_API int pty_register_batch(void* work, const void* ref_real, const void* mov_real,
                       int32_t real_inputs, int32_t dtype, int32_t window, int32_t n,
                       int32_t weighting, int32_t kappa,
                       double* dy, double* dx, double* peak, int32_t* ok,
                       void* scratch, int64_t scratch_bytes, void* stream);
PTY_API int64_t pty_register_scratch_bytes(int32_t window, int32_t n, int32_t kappa);

/* Adam + clamp for n sensed positions (posref.py:87-113), float64.
 * index[k] (or k when index == NULL) is the position id of sensed entry k. */
PTY_API int pty_adam_apply(double* positions, double* m, double* v, int64_t* t,
                   const double* gx, const double* gy, const int32_t* ok,
                   const int32_t* index, int32_t n,
                   double step_size, double beta1, double beta2, double eps_adam,
                   double max_correction, double xmin, double ymin, double xmax, double ymax,
                   void* stream);

/* engine.py:83-95: probes[0] = propagate(sqrt(max(mean_j I_j, 0)), backward) and
 * probes[p] = GS(probes[0] * noise[p-1]) scaled to 1% of mode-1 power.
 * noise: [M-1][W][W] complex128 from default_rng([init_seed, p]) (host numpy). */
PTY_API int pty_init_probes(void* probes, int32_t dtype, const void* patterns, int32_t n_patterns,
                    const double* noise, int32_t window, int32_t modes,
                    void* scratch, int64_t scratch_bytes, void* stream);

/* engine.py:153-164 power-preserving Gram-Schmidt over M modes, in place. */
PTY_API int pty_orthogonalize(void* probes, int32_t dtype, int32_t window, int32_t modes, void* stream);

/* OR PTY_ERR_NEGATIVE_I into *status if any of count intensities is < 0. */
PTY_API int pty_check_patterns(const void* patterns, int32_t dtype, int64_t count, int32_t* status,
                       void* stream);

/*
 * Batched (semi-parallel) rPIE, one batch of positions of ONE reconstruction.
 * pty_batch_contrib computes every position of `batch` against the batch-start
 * state and leaves the summed update terms in the caller-owned accumulators:
 *   obj_acc   [H][3][Wc]  real: object numerator (re, im), denominator, the three
 *                         planes interleaved per canvas row (a row band is contiguous)
 *   probe_acc [2M+1][W][W] real: probe numerator (re, im) per mode, denominator
 * (real = float for PTY_DTYPE_C64, double for C128).  Ranks that split a batch
 * all-reduce (sum) both accumulators, then every rank calls pty_batch_apply.
 * patterns_t is the diffraction stack transposed per pattern (I^T[j][kc][u]),
 * the layout the column passes stream.
 * err_part [n_positions][W][3] is indexed by visit rank (visit0 + k) and
 * reduced once per sweep by pty_batch_finalize (deterministic order).
 */
typedef struct PtyBatchArgs {
    int32_t dtype, window, modes, n_positions;
    void*   obj;
    int32_t H, Wc, r0, c0;
    void*   probes;
    const void*    patterns;     /* [N][W][W] real                              */
    const void*    patterns_t;   /* [N][W][W] real, each pattern transposed     */
    const double*  positions;    /* [N][2] (x, y) float64                       */
    const int32_t* batch;        /* [n_batch] position ids (this rank's slice)  */
    int32_t n_batch, visit0;
    double  alpha_obj, alpha_probe, beta, gamma, epsilon_rel;
    int32_t update_probe, track_modulus, sense;
    void*   stage;               /* [N][2][W][W] complex posref staging or NULL */
    void*   obj_acc;
    void*   probe_acc;
    double* err_part;
    int32_t* status;
    void*   workspace;
    int64_t workspace_bytes;
} PtyBatchArgs;

PTY_API int64_t pty_batch_workspace_bytes(int32_t dtype, int32_t window, int32_t modes,
                                          int32_t n_batch, int32_t H, int32_t Wc);
PTY_API int pty_batch_contrib(const PtyBatchArgs* args, void* stream);
PTY_API int pty_batch_apply(const PtyBatchArgs* args, void* stream);
/* dst[i] += src[i] for n real values of the dtype's real type (an owner rank
 * adding the halo rows of another rank's object accumulator). */
PTY_API int pty_accumulate(void* dst, const void* src, int64_t n, int32_t dtype, void* stream);
PTY_API int pty_batch_finalize(const double* err_part, int32_t n_visits, int32_t window,
                               double* err_out, void* stream);

/*
 * Per-visit / per-pair public functions of the reference, one call each
 * (pty_visit.cu).  All fields are W x W complex (real where noted) device
 * arrays of the given dtype; `scratch` is device scratch of at least the
 * *_scratch_bytes() size.  Data-dependent failures are OR-ed into *status.
 */
PTY_API int64_t pty_visit_scratch_bytes(int32_t dtype, int32_t window, int32_t modes);

/* engine.py:104-120 magnitude_correct: psi_det[m] = propagate(P_m * o_j),
 * corrected[m] = propagate(sqrt(I) / sqrt(total + eps) * psi_det[m], backward);
 * I (real) < 0 anywhere -> PTY_ERR_NEGATIVE_I.  probes/corrected/psi_det: [M][W][W]. */
PTY_API int pty_magnitude_correct(int32_t dtype, int32_t window, int32_t modes, const void* probes,
                                  const void* o_j, const void* intensity, double epsilon_rel,
                                  void* corrected, void* psi_det, int32_t* status,
                                  void* scratch, int64_t scratch_bytes, void* stream);

/* engine.py:123-137 update_object: out = o_j + alpha numer / denom (zero probe -> PTY_ERR_PROBE_ZERO). */
PTY_API int pty_update_object(int32_t dtype, int32_t window, int32_t modes, const void* o_j,
                              const void* probes, const void* corrected, double alpha_obj, double gamma,
                              double epsilon_rel, void* out, int32_t* status,
                              void* scratch, int64_t scratch_bytes, void* stream);

/* engine.py:140-150 update_probe (one mode; zero crop -> PTY_ERR_OBJECT_ZERO). */
PTY_API int pty_update_probe(int32_t dtype, int32_t window, const void* probe, const void* o_j,
                             const void* corrected, double alpha_probe, double beta, double epsilon_rel,
                             void* out, int32_t* status, void* scratch, int64_t scratch_bytes, void* stream);

/* registration.py:43-56 cross_power_spectrum of n pairs (work as pty_register_batch):
 * xps [n][W][W] = F(ref) conj(F(mov)) (uncentered), whitened when weighting = 0
 * ("phase"); ok[k] = 0 when the spectrum is identically zero. */
PTY_API int pty_cross_power_spectrum(void* work, const void* ref_real, const void* mov_real,
                                     int32_t real_inputs, int32_t dtype, int32_t window, int32_t n,
                                     int32_t weighting, void* xps, int32_t* ok,
                                     void* scratch, int64_t scratch_bytes, void* stream);

/* registration.py:67-81 coarse_shift, given corr = ifft2(xps) [n][W][W]:
 * argmax of |corr| over signed lags, ties -> (|dy|+|dx|, dy, dx) smallest. */
PTY_API int pty_coarse_argmax(const void* corr, int32_t dtype, int32_t window, int32_t n,
                              double* dy, double* dx, double* peak, void* stream);

/* registration.py:84-96 upsampled_idft: out[n_rows][n_cols] = er @ xps @ ec / W^2 at
 * fractional lags rows[], cols[] (device float64 arrays). */
PTY_API int64_t pty_upsampled_idft_scratch_bytes(int32_t dtype, int32_t window, int32_t n_rows);
PTY_API int pty_upsampled_idft(const void* xps, int32_t dtype, int32_t window, const double* rows,
                               int32_t n_rows, const double* cols, int32_t n_cols, void* out,
                               void* scratch, int64_t scratch_bytes, void* stream);

/* np.argmax(np.abs(x)) over n complex values (first maximum) -> *idx, *val. */
PTY_API int pty_argmax_abs(const void* x, int32_t dtype, int64_t n, int64_t* idx, double* val, void* stream);

/* posref.py:87-99 adam_step for position j; delta[2] = clipped (dx, dy). */
PTY_API int pty_adam_step(double* m, double* v, int64_t* t, int32_t j, double gx, double gy,
                          double step_size, double beta1, double beta2, double eps_adam,
                          double max_correction, double* delta, void* stream);

/* posref.py:102-113 apply_correction for position j; *inside = 1 when no clamping. */
PTY_API int pty_apply_correction(double* positions, int32_t j, double dx, double dy, double xmin,
                                 double ymin, double xmax, double ymax, int32_t* inside, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* PTYCHO_B200_H */
