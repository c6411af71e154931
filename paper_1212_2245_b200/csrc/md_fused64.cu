// md_fused64.cu -- host dispatch of the float64 cluster-resident iteration kernel
// (md_fused64_kernel.cuh): box radii 1..16 (sliding sums; 9..16 in md_fused64_b.cu) and dense
// line taps up to radius 16.

#include "md_fused64_kernel.cuh"

namespace md {

int fused64_rows() { return F64_NW * F64_LPW; }

cudaError_t launch_fused64_box_hi(const FusedLinesArgs &d, int radius, int64_t batch, cudaStream_t st);

cudaError_t launch_fused64(const FusedLinesArgs &d, int64_t batch, cudaStream_t st) {
    const int r = std::max(line_radius(d.blur), line_radius(d.adj));
    if (r > 16 || (!d.lut.p64 && !d.query)) return cudaErrorNotSupported;   // plan-time queries run before the table exists
    if (d.blur.kind == LINE_BOX && d.adj.kind == LINE_BOX && r >= 1 && d.robust) {
        cudaError_t e = cudaErrorNotSupported;
        switch (r) {
            case 1: e = launch_fused64_box_r<1>(d, batch, st); break;
            case 2: e = launch_fused64_box_r<2>(d, batch, st); break;
            case 3: e = launch_fused64_box_r<3>(d, batch, st); break;
            case 4: e = launch_fused64_box_r<4>(d, batch, st); break;
            case 5: e = launch_fused64_box_r<5>(d, batch, st); break;
            case 6: e = launch_fused64_box_r<6>(d, batch, st); break;
            case 7: e = launch_fused64_box_r<7>(d, batch, st); break;
            case 8: e = launch_fused64_box_r<8>(d, batch, st); break;
            default: e = launch_fused64_box_hi(d, r, batch, st); break;
        }
        if (e != cudaErrorNotSupported) return e;
    }
    auto go = [&](auto rtag) -> cudaError_t {
        constexpr int RR = decltype(rtag)::value;
        FusedKArgs<double, RR> a{};
        a.u0 = static_cast<const double *>(d.u_in);
        a.fpos = static_cast<const double *>(d.fpos);
        a.out = static_cast<double *>(d.u_out);
        a.query = d.query;
        a.n = d.n; a.m = d.m; a.iterations = d.iterations; a.out_vert = d.out_vert;
        a.periodic = d.blur.periodic;
        a.cl = 0;
        fill_dense<double, RR>(a.wb, d.blur, d.taps_blur_host);
        fill_dense<double, RR>(a.wa, d.adj, d.taps_adj_host);
        a.alpha = d.alpha; a.eps_d2 = d.eps_d2; a.eps_r2 = d.eps_r2; a.has_d = d.has_d;
        a.lut = d.lut;
        a.floor = d.floor; a.floor_f = d.floor_f;
        return launch_fused64_t<RR, F64_NW, F64_LPW>(d.robust ? k_fused_lines64<RR, F64_NW, F64_LPW, true, 0, false>
                                                              : k_fused_lines64<RR, F64_NW, F64_LPW, false, 0, false>,
                                                     a, d.lut.p64, batch, st, d.query_geom);
    };
    if (r <= 4) return go(std::integral_constant<int, 4>{});
    if (r <= 8) return go(std::integral_constant<int, 8>{});
    // radius 9-12 (e.g. a 17-tap kernel centred off the middle): 25 dense taps instead of 33
    if (r <= 12) return go(std::integral_constant<int, 12>{});
    return go(std::integral_constant<int, 16>{});
}

}  // namespace md
