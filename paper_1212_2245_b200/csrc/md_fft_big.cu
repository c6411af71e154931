// md_fft_big.cu -- two-level ("four-step") FFT passes for transform lengths beyond one
// block's shared memory (the 16384^2 single-image config), and for the
// column transforms of a row slab's all-to-all-transposed block.
//
// A length-N transform along an axis, N = N1 * N2 with j = j1 + N1 j2, runs as two passes,
// each a batch of short sub-transforms staged through shared memory:
//   F1: for each j1, DIF over j2 (stride N1)   -> position j1 + N1 p holds k2 = rev(p);
//       multiply by W_N^{j1 rev(p)}
//   F2: for each p,  DIF over j1 (stride 1)    -> position q + N1 p holds k = rev(p) + N2 rev(q)
// and the inverse undoes them in reverse order (DIT, conjugate twiddles). The spectrum is
// held in this "storage order"; filters computed by the same passes line up with it, so no
// permutation is ever executed (fft.py:87-117 convention: unnormalised forward, 1/N inverse).
//
// Generic line geometry: line (a, b) starts at a*sa + b*sb and has L elements at stride es;
// a block transforms G lines with consecutive b.
#include "md_fft_big_kernel.cuh"

namespace md {

// u0 = max(Re z * scale, floor) (or unclamped), fpos = max(f, floor)
template <typename T>
__global__ void k_big_wiener_epilogue(const void *z_, const T *__restrict__ f, T *__restrict__ u, T *__restrict__ fpos,
                                      int64_t n, T scale, T floor, int clamp) {
    const cx_t<T> *z = static_cast<const cx_t<T> *>(z_);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        T v = z[i].x * scale;
        if (clamp) v = v > floor ? v : floor;
        u[i] = v;
        if (fpos) {
            const T fv = f[i];
            fpos[i] = fv > floor ? fv : floor;
        }
    }
}

template <typename T>
cudaError_t launch_subfft(const SubFftArgs &a0, int64_t batch, cudaStream_t st) {
    if (a0.frame >= (1ll << 31)) return cudaErrorNotSupported;     // 32-bit in-frame offsets
    SubFftArgs a = a0;
    const int L = 1 << a.log2L;
    a.G = std::max(1, std::min(16, 2048 / L));   // power of two (L is)
    const size_t smem = ((size_t)a.G * fline_stride<sizeof(cx_t<T>)>(L) + L + 1) * sizeof(cx_t<T>);
    auto pick = [&](auto lf) {
        constexpr bool LF = decltype(lf)::value;
        return a.tw_mode == TW_FWD ? k_subfft<T, LF, TW_FWD, 0>
               : (a.tw_mode == TW_INV ? k_subfft<T, LF, TW_INV, 0>
                                      : (a.tw_mode == TW_FILT_INV ? k_subfft<T, LF, TW_FILT_INV, 0> : k_subfft<T, LF, TW_NONE, 0>));
    };
    using KernT = void (*)(SubFftArgs);
    KernT kern = subfft_ct_kernel<T>(a.log2L, a.es == 1, a.tw_mode);      // compile-time length, if any
    if (!kern) kern = a.es == 1 ? pick(std::true_type{}) : pick(std::false_type{});
    cudaError_t e = func_smem_attr((const void *)kern, smem);
    if (e != cudaSuccess) return e;
    const int blocks_b = (a.B + a.G - 1) / a.G;
    for (int64_t b0 = 0; b0 < batch; b0 += 65535) {
        const int nb = (int)((batch - b0) < 65535 ? (batch - b0) : 65535);
        SubFftArgs ab = a;
        ab.z = static_cast<char *>(a.z) + b0 * a.frame * (int64_t)sizeof(cx_t<T>);
        if (a.ra) ab.ra = static_cast<const char *>(a.ra) + b0 * a.rframe * (int64_t)sizeof(T);
        if (a.rb) ab.rb = static_cast<const char *>(a.rb) + b0 * a.rframe * (int64_t)sizeof(T);
        if (a.wu) ab.wu = static_cast<char *>(a.wu) + b0 * a.rframe * (int64_t)sizeof(T);
        if (a.wfpos) ab.wfpos = static_cast<char *>(a.wfpos) + b0 * a.rframe * (int64_t)sizeof(T);
        if (a.wf) ab.wf = static_cast<const char *>(a.wf) + b0 * a.rframe * (int64_t)sizeof(T);
        kern<<<dim3((unsigned)(a.A * blocks_b), nb), 256, smem, st>>>(ab);
    }
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_big_wiener_epilogue(const void *z, const void *f, void *u, void *fpos, int64_t n, double scale,
                                       double floor, int clamp, cudaStream_t st) {
    int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 32);
    k_big_wiener_epilogue<T><<<blocks, 256, 0, st>>>(z, static_cast<const T *>(f), static_cast<T *>(u),
                                                     static_cast<T *>(fpos), n, T(scale), T(floor), clamp);
    return cudaGetLastError();
}

// ---- axis plans -------------------------------------------------------------------------

// split N = N1 * N2, N1 >= N2, both factors <= 1024 (N <= 2^20, the reference's limit, fft.py:45)
void split_axis(int N, int *N1, int *N2) {
    int l = 0;
    while ((1 << l) < N) ++l;
    const int l2 = l / 2, l1 = l - l2;
    *N1 = 1 << l1;
    *N2 = 1 << l2;
}

// Forward (inv = 0) or inverse (inv = 1) two-pass transform along the rows (axis = 1,
// length W) or columns (axis = 0, length H) of a [batch][H][W] complex field.
// the two passes of one axis: "1" = sub-DFT over j2 (length N2, stride N1), lines j1;
// "2" = sub-DFT over j1 (length N1, stride 1), lines p
static void axis_passes(const BigAxis &ax, void *z, int H, int W, int axis, SubFftArgs &p1, SubFftArgs &p2) {
    const int N = axis == 1 ? W : H;
    const int N1 = ax.N1, N2 = ax.N2;
    p1 = SubFftArgs{};
    p2 = SubFftArgs{};
    for (SubFftArgs *p : {&p1, &p2}) {
        p->z = z; p->frame = (int64_t)H * W; p->rframe = (int64_t)H * W;
        p->N = N; p->twN = ax.twN; p->scale = 1.0;
    }
    if (axis == 1) {
        p1.A = H; p1.sa = W; p1.B = N1; p1.sb = 1; p1.es = N1;
        p2.A = H; p2.sa = W; p2.B = N2; p2.sb = N1; p2.es = 1;
    } else {
        p1.A = N1; p1.sa = W; p1.B = W; p1.sb = 1; p1.es = (int64_t)N1 * W;
        p2.A = N2; p2.sa = (int64_t)N1 * W; p2.B = W; p2.sb = 1; p2.es = W;
    }
    p1.log2L = ax.l2; p1.twL = ax.twN2; p1.log2Lother = ax.l1;
    p2.log2L = ax.l1; p2.twL = ax.twN1; p2.log2Lother = ax.l2;
    p1.tw_digit_is_a = axis == 0;
    p2.tw_digit_is_a = axis == 0;
}

template <typename T>
cudaError_t big_axis_filter(const BigAxis &ax, void *z, int H, int W, int axis, const void *filt, int conj_filt,
                            int64_t batch, cudaStream_t st) {
    SubFftArgs p1, p2;
    axis_passes(ax, z, H, W, axis, p1, p2);
    cudaError_t e;
    p1.tw_mode = TW_FWD;
    if ((e = launch_subfft<T>(p1, batch, st)) != cudaSuccess) return e;
    p2.tw_mode = TW_FILT_INV; p2.filt = filt; p2.conj_filt = conj_filt;
    if ((e = launch_subfft<T>(p2, batch, st)) != cudaSuccess) return e;
    p1.tw_mode = TW_NONE; p1.inv = 1;
    return launch_subfft<T>(p1, batch, st);
}

template <typename T>
cudaError_t big_axis_inv_wiener(const BigAxis &ax, void *z, int H, int W, int axis, double scale, const void *f,
                                void *u, void *fpos, double floor, int clamp, int64_t batch, cudaStream_t st) {
    SubFftArgs p1, p2;
    axis_passes(ax, z, H, W, axis, p1, p2);
    cudaError_t e;
    p2.tw_mode = TW_INV; p2.inv = 1;
    if ((e = launch_subfft<T>(p2, batch, st)) != cudaSuccess) return e;
    p1.tw_mode = TW_NONE; p1.inv = 1; p1.scale = scale;
    p1.wu = u; p1.wfpos = fpos; p1.wf = f; p1.floor = floor; p1.clamp = clamp;
    return launch_subfft<T>(p1, batch, st);
}

template <typename T>
cudaError_t big_axis(const BigAxis &ax, void *z, int H, int W, int axis, int inv, const void *ra, const void *rb,
                     const void *filt, int conj_filt, double scale_last, int64_t batch, cudaStream_t st) {
    const int N = axis == 1 ? W : H;
    const int N1 = ax.N1, N2 = ax.N2;
    SubFftArgs p1{}, p2{};
    for (SubFftArgs *p : {&p1, &p2}) {
        p->z = z; p->frame = (int64_t)H * W; p->rframe = (int64_t)H * W;
        p->N = N; p->twN = ax.twN; p->inv = inv; p->scale = 1.0;
    }
    // pass "1" : sub-DFT over j2 (length N2, stride N1), lines j1 = 0..N1-1
    // pass "2" : sub-DFT over j1 (length N1, stride 1),  lines p  = 0..N2-1
    if (axis == 1) {
        p1.A = H; p1.sa = W; p1.B = N1; p1.sb = 1; p1.es = N1;
        p2.A = H; p2.sa = W; p2.B = N2; p2.sb = N1; p2.es = 1;
    } else {
        p1.A = N1; p1.sa = W; p1.B = W; p1.sb = 1; p1.es = (int64_t)N1 * W;
        p2.A = N2; p2.sa = (int64_t)N1 * W; p2.B = W; p2.sb = 1; p2.es = W;
    }
    p1.log2L = ax.l2; p1.twL = ax.twN2; p1.log2Lother = ax.l1;
    p2.log2L = ax.l1; p2.twL = ax.twN1; p2.log2Lother = ax.l2;
    p1.tw_digit_is_a = axis == 0;          // the j1 digit: line index b (rows) or a (columns)
    p2.tw_digit_is_a = axis == 0;          // the p digit likewise
    cudaError_t e;
    if (!inv) {
        p1.tw_mode = TW_FWD; p1.ra = ra; p1.rb = rb;
        p2.tw_mode = TW_NONE; p2.filt = filt; p2.conj_filt = conj_filt; p2.scale = scale_last;
        if ((e = launch_subfft<T>(p1, batch, st)) != cudaSuccess) return e;
        return launch_subfft<T>(p2, batch, st);
    }
    p2.tw_mode = TW_INV;                   // conj W_N^{j1 rev(p)} after the sub-IDFT over j1
    p1.tw_mode = TW_NONE; p1.scale = scale_last;
    if ((e = launch_subfft<T>(p2, batch, st)) != cudaSuccess) return e;
    return launch_subfft<T>(p1, batch, st);
}

template cudaError_t launch_big_wiener_epilogue<double>(const void *, const void *, void *, void *, int64_t, double,
                                                        double, int, cudaStream_t);
template cudaError_t launch_big_wiener_epilogue<float>(const void *, const void *, void *, void *, int64_t, double,
                                                       double, int, cudaStream_t);
template cudaError_t big_axis_filter<double>(const BigAxis &, void *, int, int, int, const void *, int, int64_t,
                                             cudaStream_t);
template cudaError_t big_axis_filter<float>(const BigAxis &, void *, int, int, int, const void *, int, int64_t,
                                            cudaStream_t);
template cudaError_t big_axis_inv_wiener<double>(const BigAxis &, void *, int, int, int, double, const void *, void *,
                                                 void *, double, int, int64_t, cudaStream_t);
template cudaError_t big_axis_inv_wiener<float>(const BigAxis &, void *, int, int, int, double, const void *, void *,
                                                void *, double, int, int64_t, cudaStream_t);
template cudaError_t big_axis<double>(const BigAxis &, void *, int, int, int, int, const void *, const void *,
                                      const void *, int, double, int64_t, cudaStream_t);
template cudaError_t big_axis<float>(const BigAxis &, void *, int, int, int, int, const void *, const void *,
                                     const void *, int, double, int64_t, cudaStream_t);

}  // namespace md
