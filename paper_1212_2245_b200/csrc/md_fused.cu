// md_fused.cu -- host dispatch of the cluster-resident iteration kernel
// (md_fused_kernel.cuh): dense-tap instantiations here, box ones in md_fused_box*.cu.

#include "md_fused_kernel.cuh"

namespace md {

// ---------------------------------------------------------------------------------- host

// lines per warp (fused_lp in md_fused_kernel.cuh): float64 2; float 4, or 2 for radii above 8
int fused_lpw(int dtype, int radius) { return dtype == 0 ? 2 : (radius > 8 ? 2 : 4); }

bool fused_lines_supported(int dtype, int n, int m, unsigned flags, int radius) {
    if (flags & 2u) return false;                  // MD_FLAG_NO_FUSED
    if (n % SEG != 0 || n / SEG > 32 || n < 64) return false;
    // float64, radius <= 16: any line count the cluster can hold (2..16 CTAs of 4..rows lines)
    if (dtype == 0 && radius <= 16) return m >= 8 && (m + 15) / 16 <= fused64_rows();
    const int rl = FU_WARPS * fused_lpw(dtype, radius);
    if (m % rl != 0) return false;
    const int cl = m / rl;
    return cl >= 2 && cl <= 16;
}

template <typename T>
cudaError_t launch_fused_lines(const FusedLinesArgs &d, int64_t batch, cudaStream_t st) {
    const int r = std::max(line_radius(d.blur), line_radius(d.adj));
    if (sizeof(T) == 8 && r <= 16) return launch_fused64(d, batch, st);
    if (d.floor_f) return cudaErrorNotSupported;          // the raw-observation mode is float64-kernel only
    // boxes (odd, even, fractional length): O(1) sliding sum + end corrections
    if (d.blur.kind == LINE_BOX && d.adj.kind == LINE_BOX && r >= 1 && r <= 15 && d.robust) {
        const cudaError_t e = launch_fused_box<T>(d, r, batch, st);
        if (e != cudaErrorNotSupported) return e;
    }
    auto go = [&](auto rtag) -> cudaError_t {
        constexpr int RR = decltype(rtag)::value;
        constexpr int LP = fused_lp<T, RR>();
        FusedKArgs<T, RR> a{};
        a.u0 = static_cast<const T *>(d.u_in);
        a.fpos = static_cast<const T *>(d.fpos);
        a.out = static_cast<T *>(d.u_out);
        a.query = d.query;
        a.n = d.n; a.m = d.m; a.iterations = d.iterations; a.out_vert = d.out_vert;
        a.periodic = d.blur.periodic;
        a.cl = d.m / (FU_WARPS * LP);
        fill_dense<T, RR>(a.wb, d.blur, d.taps_blur_host);
        fill_dense<T, RR>(a.wa, d.adj, d.taps_adj_host);
        a.alpha = T(d.alpha); a.eps_d2 = T(d.eps_d2); a.eps_r2 = T(d.eps_r2); a.has_d = d.has_d;
        a.lut = d.lut;
        return launch_fused_t<T, RR, LP>(d.robust ? k_fused_lines<T, RR, LP, true, 0, false>
                                                  : k_fused_lines<T, RR, LP, false, 0, false>,
                                         a, batch, st, d.query_geom);
    };
    if (r <= 4) return go(std::integral_constant<int, 4>{});
    if (r <= 8) return go(std::integral_constant<int, 8>{});
    return go(std::integral_constant<int, 16>{});
}

template cudaError_t launch_fused_lines<double>(const FusedLinesArgs &, int64_t, cudaStream_t);
template cudaError_t launch_fused_lines<float>(const FusedLinesArgs &, int64_t, cudaStream_t);

}  // namespace md
