// md_fft_big.h -- interface of the two-level FFT passes (md_fft_big.cu).
#pragma once

#include <algorithm>

#include "md_internal.h"

namespace md {

// TW_FILT_INV: forward sub-DFT, x filter, inverse sub-DFT, then the TW_INV twiddle -- the
// middle of a filtered axis (F2, filter, I2) in one pass
enum { TW_NONE = 0, TW_FWD = 1, TW_INV = 2, TW_FILT_INV = 3 };

struct SubFftArgs {
    void *z;                     // complex field, [batch] frames of `frame` elements
    const void *ra, *rb;         // optional real inputs (first forward pass)
    int64_t frame, rframe;
    int A, B, G, log2L, log2Lother, N;
    int64_t sa, sb, es;          // line (a, b) base = a*sa + b*sb, element stride es
    const void *twL;             // W_L^k, k < L/2 (sub-transform)
    const void *twN;             // W_N^k, k < N/2 (inter-pass twiddles)
    int inv, tw_mode, tw_digit_is_a;
    const void *filt;            // multiply by filt[address] after the pass (last forward pass)
    int conj_filt;
    double scale;
    // optional Wiener epilogue instead of storing z (last inverse pass): u = max(Re z * scale,
    // floor) (or unclamped), fpos = max(f, floor), real fields indexed like z
    void *wu, *wfpos;
    const void *wf;
    double floor;
    int clamp;
};

// one axis of a two-level transform: N = N1 * N2, twiddle tables in the plan dtype
struct BigAxis {
    int N, N1, N2, l1, l2;
    const void *twN, *twN1, *twN2;
};

void split_axis(int N, int *N1, int *N2);
template <typename T> cudaError_t launch_subfft(const SubFftArgs &, int64_t batch, cudaStream_t);
// the pass kernel specialised for a compile-time sub-transform length 2^6 .. 2^10 (float64;
// md_fft_big_ct.cu), or nullptr (then the generic kernel runs)
template <typename T> void (*subfft_ct_kernel(int log2L, bool line_fast, int tw_mode))(SubFftArgs);
template <typename T>
cudaError_t big_axis(const BigAxis &ax, void *z, int H, int W, int axis, int inv, const void *ra, const void *rb,
                     const void *filt, int conj_filt, double scale_last, int64_t batch, cudaStream_t st);
// filtered transform along one axis: forward (F1, then F2 + filter + I2 fused), inverse I1;
// with wu set, the last pass writes the Wiener result instead of z (see SubFftArgs)
template <typename T>
cudaError_t big_axis_filter(const BigAxis &ax, void *z, int H, int W, int axis, const void *filt, int conj_filt,
                            int64_t batch, cudaStream_t st);
// inverse transform along one axis whose last pass writes u / fpos (Wiener epilogue)
template <typename T>
cudaError_t big_axis_inv_wiener(const BigAxis &ax, void *z, int H, int W, int axis, double scale, const void *f,
                                void *u, void *fpos, double floor, int clamp, int64_t batch, cudaStream_t st);
// natural-order transforms of contiguous lines (md_fft_api.cu)
template <typename T> int fft_lines_max_single();
template <typename T>
cudaError_t launch_fft_lines_nat(void *z, int n, int64_t lines, const void *tw, int inverse, cudaStream_t st);
template <typename T>
cudaError_t launch_fft_perm(const void *in, void *out, const BigAxis &ax, int64_t lines, int to_natural,
                            cudaStream_t st);
template <typename T>
cudaError_t launch_big_wiener_epilogue(const void *z, const void *f, void *u, void *fpos, int64_t n, double scale,
                                       double floor, int clamp, cudaStream_t st);

}  // namespace md
