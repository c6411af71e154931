/*
 * mdcuda.h -- C ABI of the B200 (sm_100a) Wiener + RRRL deconvolution library.
 *
 * Drop-in boundary for the hot path of the reference package `motiondeblur`
 * (arXiv:1212.2245). The reference has no FFI: its boundary is the Python API
 * (`motiondeblur/__init__.py:7-62`) plus the duck-typed convolver protocol
 * `blur / adjoint / adjoint_pair` (`deconv.py:295-376`). Every entry point below replaces
 * one of those calls; the Python mirror in `paper_1212_2245_b200/` binds them with ctypes
 * (see INTEGRATION.md). Signatures carry plain pointers, sizes and scalars only.
 *
 * Conventions
 *   - Images are batches of frames, `[batch, height, width]`, row-major, contiguous,
 *     in the plan's dtype (MD_F64: double, MD_F32: float), resident in DEVICE memory
 *     unless the function name ends in `_host`.
 *   - `stream` is a `cudaStream_t` passed as `void*` (NULL = legacy default stream).
 *   - Every function returns MD_OK (0) or a negative MD_E* status; `md_last_error()`
 *     returns a thread-local message for the last failure. MD_EINVAL maps to Python
 *     ValueError, MD_ECONTRACT to ContractError (core.py:39-40), MD_ECUDA to RuntimeError.
 */
#ifndef MDCUDA_H
#define MDCUDA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MDCUDA_ABI_VERSION 1

/* status codes */
#define MD_OK 0
#define MD_EINVAL (-1)     /* bad parameter / shape / unsupported size   -> ValueError    */
#define MD_ECONTRACT (-2)  /* non-positive data where positivity required -> ContractError */
#define MD_ECUDA (-3)      /* CUDA runtime failure                          -> RuntimeError  */
#define MD_ENOMEM (-4)     /* device allocation failed                      -> MemoryError   */

/* arithmetic type */
#define MD_F64 0
#define MD_F32 1

/* PSF kinds (core.py:83-86) */
#define MD_PSF_GENERAL_2D 0
#define MD_PSF_GENERAL_1D 1
#define MD_PSF_BOX_1D 2

/* blur axis of 1D kinds (core.py:89-93) */
#define MD_AXIS_NONE (-1)
#define MD_AXIS_VERTICAL 0
#define MD_AXIS_HORIZONTAL 1

/* convolver realisation used inside the iterations (deconv.py:295-403, 566-579) */
#define MD_CONV_BOX 0        /* clamped sliding-window box   (_BoxConvolver, Scenario.BOX_1D)   */
#define MD_CONV_SPATIAL 1    /* clamped direct summation     (_SpatialConvolver)                */
#define MD_CONV_FOURIER 2    /* periodic along the blur axis (_FourierConvolver1D, FOURIER_1D)  */
#define MD_CONV_FOURIER2D 3  /* periodic 2D                  (_FourierConvolver2D, FOURIER_2D)  */

/* how the iterate is initialised */
#define MD_INIT_WIENER 0     /* DeblurPipeline.run_timed: u0 = max(Wiener(f), floor) (deconv.py:653-672) */
#define MD_INIT_CLAMPED 1    /* rrrl_deblur / rl_deblur:  u0 = max(f, floor)         (deconv.py:524-559) */

/* flags */
#define MD_FLAG_RL 1u            /* identity penaliser and alpha = 0: plain RL (rl_deblur)        */
#define MD_FLAG_NO_FUSED 2u      /* force the multi-kernel path even where a fused kernel applies */
#define MD_FLAG_FORCE_FFT2D 4u   /* 2D periodic convolver through 2D FFTs, not direct taps        */
#define MD_FLAG_GENERIC_LINES 8u /* 1D blur: generic per-iteration line kernel, not the fast one  */
#define MD_FLAG_BIG_FFT 16u      /* 2D Wiener through the two-level FFT passes at any size        */

typedef struct md_plan md_plan; /* opaque */

/* Problem description -- mirrors DeblurPipeline(shape, psf, params, scenario)
 * (deconv.py:611-643) and make_convolver(psf, shape, mode) (deconv.py:379-403). */
typedef struct md_plan_desc {
    int32_t height, width;        /* frame shape (rows, cols)                                     */
    int32_t dtype;                /* MD_F64 | MD_F32                                               */
    int32_t psf_kind;             /* MD_PSF_*                                                      */
    int32_t psf_axis;             /* MD_AXIS_* (1D kinds)                                          */
    int32_t psf_rows, psf_cols;   /* weight array shape; 1D kinds: rows = taps, cols = 1           */
    int32_t center_row, center_col; /* 2D: (cy, cx); 1D kinds: center_row = centre index          */
    double box_length;            /* MD_PSF_BOX_1D only (Psf.length)                               */
    const double *psf_weights;    /* HOST pointer, psf_rows*psf_cols normalised weights            */
    int32_t conv;                 /* MD_CONV_*                                                     */
    int32_t init;                 /* MD_INIT_*                                                     */
    int32_t iterations;           /* DeconvParams.iterations                                       */
    uint32_t flags;               /* MD_FLAG_*                                                     */
    double wiener_k, alpha, eps_data, eps_reg, floor; /* DeconvParams (core.py:242-247)            */
} md_plan_desc;

/* library */
int32_t md_abi_version(void);
const char *md_last_error(void);
int32_t md_device_sm_count(void);

/* plans (DeblurPipeline.__init__, deconv.py:611-643; make_convolver, deconv.py:379-403) */
/* A 1D PSF whose blur axis exceeds the on-chip line kernels (Wiener: 8192 float / 4096 double
   samples; iterations: 4096 float / 2048 double) is planned as a plane with a one-row (one-column)
   PSF and the same boundary; that route needs power-of-two sides, else MD_EINVAL.           */
int32_t md_plan_create(const md_plan_desc *desc, md_plan **out);
int32_t md_plan_destroy(md_plan *plan);
/* scratch bytes a run over `batch` frames needs (allocated lazily, owned by the plan) */
int64_t md_plan_scratch_bytes(const md_plan *plan, int64_t batch);
/* human-readable description of the kernels the plan launches (for logs / DESIGN.md) */
const char *md_plan_describe(const md_plan *plan);
/* frames per internal chunk (0 = automatic, bounded by ~1 GiB of scratch) */
int32_t md_plan_set_chunk(md_plan *plan, int64_t frames);
/* enable / disable the fused persistent kernel where the plan supports it */
int32_t md_plan_set_fused(md_plan *plan, int32_t on);
int32_t md_plan_is_fused(const md_plan *plan);
/* the 1D cluster kernel's launch geometry: CTAs per cluster, co-resident clusters, CTAs per SM
 * (all 0 when the plan does not use it); SMs busy = clusters x CTAs / CTAs per SM */
int32_t md_plan_fused_geometry(const md_plan *plan, int32_t *cluster_ctas, int32_t *resident_clusters,
                               int32_t *ctas_per_sm);

/* the pipeline: Wiener (or clamp) init + iterations (DeblurPipeline.run, deconv.py:653-693;
 * rrrl_deblur deconv.py:537-559; rl_deblur deconv.py:524-534). f and u are device arrays.
 * Capturable: between cudaStreamBeginCapture/EndCapture on `stream` it records its launches
 * into the caller's CUDA graph (call it once uncaptured first with the same batch, so the
 * plan's scratch is already sized; replays are ordered only by the stream they run on). */
int32_t md_run(md_plan *plan, const void *f, void *u, int64_t batch, void *stream);
/* same, but f/u are HOST float64 arrays; H2D, dtype conversion, run, D2H all inside.
 * Copies are chunked through the plan's pinned staging buffers. */
int32_t md_run_host(md_plan *plan, const double *f, double *u, int64_t batch, void *stream);
/* md_run with CUDA events between launch groups on `stream`; synchronises. ms_out[4]:
 * [0] init (Wiener or clamp) ms, [1] RRRL iteration kernels ms, [2] layout transposes ms,
 * [3] number of launch groups timed. */
int32_t md_run_profile(md_plan *plan, const void *f, void *u, int64_t batch, void *stream,
                       double *ms_out);
/* host frame types for md_run_host_ex */
#define MD_IO_F64 0
#define MD_IO_F32 1
#define MD_IO_U8 2    /* 8-bit grey frames (camera / PGM capture); as an OUTPUT type of
                         md_run_host_ex: the reference's write_pgm quantisation
                         clip(floor(u + 0.5), 0, 255) (pgm.py:56-58) */
/* md_run from HOST frames of type in_type to HOST results of type out_type. Chunks are
 * pipelined over internal streams (H2D of chunk c+1 overlaps compute of chunk c and D2H of
 * chunk c-1); pinned host buffers make the copies asynchronous. Synchronises `stream`. */
int32_t md_run_host_ex(md_plan *plan, const void *f, int32_t in_type, void *u, int32_t out_type,
                       int64_t batch, void *stream);
/* element type conversion of n DEVICE values on `stream` (no sync): any MD_IO_* to float32 /
 * float64, or float32 / float64 to MD_IO_U8 (write_pgm quantisation) -- the device half of the
 * host entries, exported for callers that stage their own copies (e.g. a PSF bank pipelining
 * several plans) */
int32_t md_convert(const void *in, int32_t in_type, void *out, int32_t out_type, int64_t n, void *stream);
/* md_run with one CUDA event per launch group: group_ms[i] / group_kind[i] (0 init, 1 iteration
 * kernel(s), 2 layout) for i < *n_groups; the fused kernel is one group for all iterations */
int32_t md_run_profile_groups(md_plan *plan, const void *f, void *u, int64_t batch, void *stream,
                              double *group_ms, int32_t *group_kind, int32_t max_groups,
                              int32_t *n_groups);
/* number of kernel launches md_run issues for one call (for the bench's gpu_launches) */
int32_t md_run_launch_count(const md_plan *plan, int64_t batch);

/* Wiener filter only, unclamped (wiener_1d deconv.py:275-288 / wiener_2d deconv.py:257-272) */
int32_t md_wiener(md_plan *plan, const void *f, void *out, int64_t batch, void *stream);

/* convolver protocol (deconv.py:295-376): which = 0 blur, 1 adjoint */
int32_t md_convolve(md_plan *plan, const void *in, void *out, int64_t batch, int32_t which,
                    void *stream);
int32_t md_adjoint_pair(md_plan *plan, const void *p, const void *q, void *out_p, void *out_q,
                        int64_t batch, void *stream);

/* step-level operations (deconv.py:142-229, 415-446). n = element count / frame shape. */
int32_t md_robust_weight(int32_t dtype, const void *f, const void *b, void *out, int64_t n,
                         double eps_data, double floor, int32_t assume_floored, void *stream);
int32_t md_diffusion(int32_t dtype, const void *u, void *out, int64_t batch, int32_t height,
                     int32_t width, double eps_reg, void *stream);
/* u' = u*num/den assembled from blurred b, optional weight w and diffusion d (_combine) */
int32_t md_rrrl_step(md_plan *plan, const void *u, const void *f, const void *b, const void *w,
                     const void *d, void *out, int64_t batch, double alpha, void *stream);
/* r1(x) = x - 1 - ln x through the device divergence table (DivergenceLut.r1, deconv.py:114-134) */
int32_t md_lut_r1(int32_t dtype, const void *x, void *out, int64_t n, void *stream);
/* copy the 133,057-entry float64 table to the host (DivergenceLut.table, deconv.py:101-112) */
int32_t md_lut_table(double *host_out, int64_t count);
/* x = max(x, 1e-12) in place (_blur_guarded, deconv.py:415-418) */
int32_t md_guard(int32_t dtype, void *x, int64_t n, void *stream);
/* natural-order complex FFT of `lines` contiguous lines of length n (power of two <= 2^20), in
 * place; dtype MD_F64 = complex128 (interleaved double pairs), MD_F32 = complex64; forward
 * unnormalised, inverse scaled by 1/n (FourierPlan.forward / inverse, fft.py:52-117) */
int32_t md_fft(int32_t dtype, void *z, int32_t n, int64_t lines, int32_t inverse, void *stream);
/* min over n elements, written to *out_host (positivity contracts, deconv.py:410-412) */
int32_t md_min(int32_t dtype, const void *x, int64_t n, double *out_host, void *stream);

/* ---- DivergenceLut with non-default parameters (DivergenceLut.build, deconv.py:95-112): the
 * caller owns a device table of `count` doubles; slope / intercept as the reference derives
 * them (deconv.py:108-111). Evaluation follows the reference's rounding order. */
/* table[i] = (delta + step i) - 1 - ln(delta + step i) */
int32_t md_lut_build(double *table, int64_t count, double delta, double step, void *stream);
/* DivergenceLut.r1 (deconv.py:114-134) with that table, float64 */
int32_t md_lut_r1_custom(const double *table, int64_t count, double delta, double step, double upper,
                         double direct_below, double slope, double intercept, const double *x,
                         double *out, int64_t n, void *stream);
/* _weight_arrays / robust_weight (deconv.py:142-180) with that table */
int32_t md_robust_weight_custom(int32_t dtype, const double *table, int64_t count, double delta,
                                double step, double upper, double direct_below, double slope,
                                double intercept, const void *f, const void *b, void *out, int64_t n,
                                double eps_data, double floor, int32_t assume_floored, void *stream);

/* ---- plan-free pointwise steps for a caller-supplied convolver object (the reference's
 * duck-typed protocol, deconv.py:456-457, 549-550): the caller's blur / adjoint_pair run
 * wherever they run, these two run here */
/* out = max(in, floor)  (np.maximum(f, floor): rl_deblur / rrrl_deblur, deconv.py:529, 554) */
int32_t md_clamp(int32_t dtype, const void *in, void *out, int64_t n, double floor, void *stream);
/* out = (w ?) f / b  (_combine's ratio, deconv.py:425-430) */
int32_t md_ratio(int32_t dtype, const void *f, const void *b, const void *w, void *out, int64_t n,
                 void *stream);
/* out = u * (num + a D+) / max(den - a D-, 1e-12); den NULL = RL form, d NULL = no TV
 * (_combine, deconv.py:421-446) */
int32_t md_combine(int32_t dtype, const void *u, const void *num, const void *den, const void *d,
                   void *out, int64_t n, double alpha, void *stream);

/* ---- one image split into row slabs over ranks (c5; driver: paper_1212_2245_b200/slab.py).
 * Plans must be 2D direct-tap plans created with MD_FLAG_BIG_FFT. Slab buffers hold the
 * rank's rows plus `top`/`bottom` halo rows; pointers passed to md_slab_iterate point at the
 * first OWN row (halo rows live before / after it). */
/* halo depth in rows needed above / below a slab for one iteration */
int32_t md_slab_halo(const md_plan *plan, int32_t *top, int32_t *bottom);
/* device copy of the Wiener multiplier's storage columns [col0, col0+cols) (plan-owned) */
int32_t md_slab_prepare(md_plan *plan, int32_t col0, int32_t cols, void **mult_block);
/* two-level FFT along the rows of a [rows][W] complex slab (forward: optional real input) */
int32_t md_slab_rows_fft(md_plan *plan, void *z, const void *real_in, int32_t rows, int32_t inv,
                         double scale, void *stream);
/* forward column transform, x multiplier block, inverse, on a [H][cols] complex block */
int32_t md_slab_cols_filter(md_plan *plan, void *zc, int32_t cols, const void *mult_block,
                            void *stream);
/* u0 = max(Re z / (H W), floor), fpos = max(f, floor) for `rows` rows */
int32_t md_slab_wiener_epilogue(md_plan *plan, const void *z, const void *f, void *u0,
                                void *fpos, int32_t rows, void *stream);
/* one RRRL iteration of a slab whose first own row is global row `row0` */
int32_t md_slab_iterate(md_plan *plan, const void *u, const void *fpos, void *p, void *w,
                        void *u_out, int32_t rows, int32_t row0, void *stream);
/* the same iteration in pieces, so the halo exchange can overlap the rows that do not need it:
 * stage A (blur -> p, W) over rows [a_begin, a_end) of [-adj.ht, rows + adj.hb), stage B
 * (adjoint pair + TV + update) over own rows [b_begin, b_end); empty ranges are skipped */
int32_t md_slab_stage(md_plan *plan, const void *u, const void *fpos, void *p, void *w,
                      void *u_out, int32_t rows, int32_t row0, int32_t a_begin, int32_t a_end,
                      int32_t b_begin, int32_t b_end, void *stream);
/* margins of the halo-free bands: stage A rows [a_in, S - a_in) read no halo u, stage B rows
 * [b_in, S - b_in) need only those p / W rows (slab.py: interior first, boundary after the
 * exchange); adj_top / adj_bottom: the full stage A range is [-adj_top, S + adj_bottom) */
int32_t md_slab_bands(const md_plan *plan, int32_t *a_in, int32_t *b_in, int32_t *adj_top,
                      int32_t *adj_bottom);

#ifdef __cplusplus
}
#endif
#endif /* MDCUDA_H */
