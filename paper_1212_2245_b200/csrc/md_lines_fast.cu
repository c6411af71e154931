// md_lines_fast.cu -- the fast RRRL iteration kernel for 1D blur (lines), one launch per
// iteration, warp-per-line with register windows (see md_linefast.cuh).
//
// Replaces _iterate_rrrl with a box / 1D convolver (deconv.py:512-521) and its callees:
// _blur_guarded (415-418), _weight_arrays (142-162), _diffusion_arrays (187-213) and
// _combine (421-446); a general 1D kernel is applied as a dense tap vector over a
// compile-time window [-R, R] (conv.py:141-173 / deconv.py:329-356 semantics: clamped or
// periodic continuation via the smem halo), a box as an O(1) sliding sum (md_lines_box_*.cu).
//
// Block = 8 warps = 8 lines of one frame (+2 halo lines each side for the TV stencil).
//   load u (12 lines), fpos (8 lines) -> fill halos
//   phase 1: diffusivity g on 10 lines; blur -> b -> W, p on own line (warp-local)
//   barrier
//   phase 2: adjoint pair (num, den) + TV divergence + update -> global
#include "md_lines_fast_kernel.cuh"

namespace md {

int line_radius(const LineConv &c) {
    int lo, hi;
    if (c.kind == LINE_BOX) {
        lo = c.ends ? c.elo : c.lo;
        hi = c.ends ? c.ehi : c.hi;
    } else {
        lo = c.center - c.ntaps + 1;
        hi = c.center;
    }
    return std::max(-lo, hi);
}

bool iter_fast_supported(int dtype, int n, const LineConv &blur, const LineConv &adj) {
    const int r = std::max(line_radius(blur), line_radius(adj));
    if (r > 16 || n % SEG != 0 || n < SEG) return false;
    const int hw = r <= 8 ? 8 : 16;
    if (hw > n) return false;   // halo wider than the line: keep the generic kernel
    const size_t es = dtype == 0 ? 8 : 4;
    return (size_t)(5 * FTL + 6) * xline_len(n, hw) * es <= 200 * 1024;
}

template <typename T>
cudaError_t launch_iter_fast(const IterFastDesc &d, bool robust, int64_t batch, cudaStream_t st) {
    const int r = std::max(line_radius(d.blur), line_radius(d.adj));
    // boxes (odd, even, fractional length): O(1) sliding sums + end corrections
    if (d.blur.kind == LINE_BOX && d.adj.kind == LINE_BOX && r >= 1 && r <= 15 && robust) {
        const cudaError_t e = r <= 8 ? launch_iter_fast_box_a<T>(d, r, batch, st) : launch_iter_fast_box_b<T>(d, r, batch, st);
        if (e != cudaErrorNotSupported) return e;
    }
    auto go = [&](auto rtag) -> cudaError_t {
        constexpr int RR = decltype(rtag)::value;
        IterFastArgs<T, RR> a{};
        a.u_in = static_cast<const T *>(d.u_in);
        a.fpos = static_cast<const T *>(d.fpos);
        a.u_out = static_cast<T *>(d.u_out);
        a.n = d.n; a.m = d.m; a.periodic = d.blur.periodic;
        fill_dense<T, RR>(a.wb, d.blur, d.taps_blur_host);
        fill_dense<T, RR>(a.wa, d.adj, d.taps_adj_host);
        a.alpha = T(d.alpha); a.eps_d2 = T(d.eps_d2); a.eps_r2 = T(d.eps_r2); a.has_d = d.has_d;
        a.lut = d.lut;
        return launch_iter_fast_k<T, RR>(robust ? k_iter_lines_fast<T, RR, true, 0, false>
                                                : k_iter_lines_fast<T, RR, false, 0, false>,
                                         a, batch, st);
    };
    if (r <= 4) return go(std::integral_constant<int, 4>{});
    if (r <= 8) return go(std::integral_constant<int, 8>{});
    return go(std::integral_constant<int, 16>{});
}

template cudaError_t launch_iter_fast<double>(const IterFastDesc &, bool, int64_t, cudaStream_t);
template cudaError_t launch_iter_fast<float>(const IterFastDesc &, bool, int64_t, cudaStream_t);

}  // namespace md
