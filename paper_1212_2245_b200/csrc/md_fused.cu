// md_fused.cu -- host dispatch of the cluster-resident iteration kernel
// (md_fused_kernel.cuh): dense-tap instantiations here, symmetric-box ones in md_fused_box*.cu.
#include <cstdlib>

#include "md_fused_kernel.cuh"

namespace md {

// ---------------------------------------------------------------------------------- host

// lines per warp: float64 uses 2 (16-line CTAs); float uses 4 unless MD_FUSED_LPW=2 (tuning knob)
int fused_lpw(int dtype) {
    if (dtype == 0) return 2;
    static int v = [] {
        const char *e = getenv("MD_FUSED_LPW");
        return (e && atoi(e) == 2) ? 2 : 4;
    }();
    return v;
}

bool fused_lines_supported(int dtype, int n, int m, unsigned flags) {
    if (flags & 2u) return false;                  // MD_FLAG_NO_FUSED
    if (n % SEG != 0 || n / SEG > 32 || n < 64) return false;
    const int rl = FU_WARPS * fused_lpw(dtype);
    if (m % rl != 0) return false;
    const int cl = m / rl;
    return cl >= 2 && cl <= 16;
}

template <typename T>
cudaError_t launch_fused_lines(const FusedLinesArgs &d, int64_t batch, cudaStream_t st) {
    const int r = std::max(line_radius(d.blur), line_radius(d.adj));
    const int lpw = fused_lpw(sizeof(T) == 8 ? 0 : 1);
    // symmetric integer box (odd length, default centre): O(1) sliding-sum specialisation
    if (d.blur.kind == LINE_BOX && !d.blur.ends && d.blur.lo == -d.blur.hi && d.adj.lo == -d.adj.hi &&
        d.blur.hi == d.adj.hi && d.blur.hi >= 1 && d.blur.hi <= 15 && d.robust)
        return launch_fused_box<T>(d, d.blur.hi, batch, st);
    auto go = [&](auto rtag, auto ltag) -> cudaError_t {
        constexpr int RR = decltype(rtag)::value;
        constexpr int LP = decltype(ltag)::value;
        FusedKArgs<T, RR> a{};
        a.u0 = static_cast<const T *>(d.u_in);
        a.fpos = static_cast<const T *>(d.fpos);
        a.out = static_cast<T *>(d.u_out);
        a.n = d.n; a.m = d.m; a.iterations = d.iterations; a.out_vert = d.out_vert;
        a.periodic = d.blur.periodic;
        a.cl = d.m / (FU_WARPS * LP);
        fill_dense<T, RR>(a.wb, d.blur, d.taps_blur_host);
        fill_dense<T, RR>(a.wa, d.adj, d.taps_adj_host);
        a.alpha = T(d.alpha); a.eps_d2 = T(d.eps_d2); a.eps_r2 = T(d.eps_r2); a.has_d = d.has_d;
        a.lut = d.lut;
        return launch_fused_t<T, RR, LP, 0>(a, d.robust != 0, batch, st);
    };
    using I2 = std::integral_constant<int, 2>;
    using I4 = std::integral_constant<int, 4>;
    if (lpw == 2 || sizeof(T) == 8) {
        if (r <= 4) return go(std::integral_constant<int, 4>{}, I2{});
        if (r <= 8) return go(std::integral_constant<int, 8>{}, I2{});
        return go(std::integral_constant<int, 16>{}, I2{});
    }
    if (r <= 4) return go(std::integral_constant<int, 4>{}, I4{});
    if (r <= 8) return go(std::integral_constant<int, 8>{}, I4{});
    return go(std::integral_constant<int, 16>{}, I4{});
}

template cudaError_t launch_fused_lines<double>(const FusedLinesArgs &, int64_t, cudaStream_t);
template cudaError_t launch_fused_lines<float>(const FusedLinesArgs &, int64_t, cudaStream_t);

}  // namespace md
