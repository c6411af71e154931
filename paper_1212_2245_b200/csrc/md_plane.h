// md_plane.h -- argument blocks for the 2D kernels (direct taps and 2D FFT).
#pragma once

#include "md_internal.h"

namespace md {

// out[y, x] += w * in[y + dy, x + dx]
struct PlaneTap {
    int dy, dx;
    double w;
};

// a tap list plus the halo it needs around an output tile
struct PlaneHalo {
    int nt;
    int ht, hb, hl, hr;   // rows above / below, cols left / right
};

struct StagePlaneArgs {
    const void *u;        // current iterate
    const void *f;        // observation (floored unless floor_f)
    void *p, *w;          // stage A outputs (w unused for RL)
    void *u_out;          // stage B output
    int H, W, periodic;
    PlaneHalo blur, adj;
    const PlaneTap *blur_taps, *adj_taps;   // device
    double alpha, eps_d2, eps_r2, floor;
    int has_d, floor_f, general_weight;
    LutView lut;
};

struct ConvPlaneArgs {
    const void *in;
    void *out;
    int H, W, periodic;
    PlaneHalo h;
    const PlaneTap *taps;
};

template <typename T> cudaError_t launch_stage_plane(const StagePlaneArgs &, bool robust, int64_t, cudaStream_t);
template <typename T> cudaError_t launch_conv_plane(const ConvPlaneArgs &, int64_t, cudaStream_t);
template <typename T> cudaError_t launch_diffusion(const void *u, void *out, int64_t batch, int H, int W,
                                                   double eps_r2, cudaStream_t);
template <typename T> cudaError_t launch_robust_weight(const void *f, const void *b, void *out, int64_t n,
                                                       double eps2, double floor, int floored,
                                                       const LutView &lut, cudaStream_t);
template <typename T> cudaError_t launch_ratio(const void *f, const void *b, const void *w, void *out, int64_t n,
                                               cudaStream_t);
template <typename T> cudaError_t launch_combine(const void *u, const void *num, const void *den, const void *d,
                                                 void *out, int64_t n, double alpha, cudaStream_t);
template <typename T> cudaError_t launch_guard(void *x, int64_t n, cudaStream_t);
template <typename T> cudaError_t launch_lut_r1(const void *x, void *out, int64_t n, const LutView &lut, cudaStream_t);
template <typename T> cudaError_t launch_min(const void *x, int64_t n, double *partial, int nblocks, cudaStream_t);
template <typename T> cudaError_t launch_convert(const void *in, void *out, int64_t n, int to_double, cudaStream_t);
// host-frame type conversion: in_type / out_type are MD_IO_F64 (0), MD_IO_F32 (1), MD_IO_U8 (2)
template <typename T> cudaError_t launch_convert_in(const void *in, int in_type, void *out, int64_t n, cudaStream_t);
template <typename T> cudaError_t launch_convert_out(const void *in, void *out, int out_type, int64_t n, cudaStream_t);

// ---- 2D FFT (md_fft2d.cu) ----
// row-pass epilogues
enum { R_LOAD_REAL = 0, R_LOAD_PAIR = 1, R_LOAD_COMPLEX = 2 };
enum { R_EPI_NONE = 0, R_EPI_STORE_PAIR = 1, R_EPI_WIENER = 2, R_EPI_STAGE_A = 3, R_EPI_STAGE_B = 4 };

struct Fft2Args {
    int H, W, log2H, log2W;
    const void *twH, *twW;      // cx_t<T> twiddles for the column / row lengths
    // row pass
    int load;                   // R_LOAD_*
    const void *ra, *rb;        // real inputs (rb may be null -> zero imaginary part)
    void *z;                    // complex work field [batch][H][W] (bit-reversed along x after fwd)
    int inv;                    // 1: inverse DIT first (input z is a spectrum)
    int epi;                    // R_EPI_*
    int fwd_after;              // 1: forward DIF of the epilogue's packed output, stored to z
    void *oa, *ob;              // epilogue real outputs
    const void *f;              // observation (stage A: floored; Wiener: raw -> writes fpos to ob)
    const void *u;              // current iterate (stage B)
    const void *dpre;           // stage B: the TV divergence precomputed per pixel (k_diffusion), or null
    double floor, alpha, eps_d2, eps_r2, scale;
    int has_d, robust;
    LutView lut;
    // frame pairing (Wiener init): real frames 2z and 2z+1 ride in the real / imaginary part of
    // complex field z (h is real, so the filter maps each part to itself); nreal = real frames
    int pairs;
    int64_t nreal;
    // column pass
    const void *filt;           // cx_t<T>[H][W] in storage (bit-reversed) coordinates, or null
    int conj_filt, col_inv;     // multiply by conj(filt); run the inverse DIT after the multiply
};

template <typename T> cudaError_t launch_fft2_rows(const Fft2Args &, int64_t batch, cudaStream_t);
template <typename T> cudaError_t launch_fft2_cols(const Fft2Args &, int64_t batch, cudaStream_t);

}  // namespace md
