// md_fused_box_a -- symmetric-box specialisations of the fused kernel, radius 1..8.
#include "md_fused_kernel.cuh"

namespace md {

template <typename T, int RR, int LP>
static cudaError_t go_lp(const FusedLinesArgs &d, int64_t batch, cudaStream_t st) {
    FusedKArgs<T, RR> a{};
    a.u0 = static_cast<const T *>(d.u_in);
    a.fpos = static_cast<const T *>(d.fpos);
    a.out = static_cast<T *>(d.u_out);
    a.n = d.n; a.m = d.m; a.iterations = d.iterations; a.out_vert = d.out_vert;
    a.periodic = d.blur.periodic;
    a.cl = d.m / (8 * LP);
    a.alpha = T(d.alpha); a.eps_d2 = T(d.eps_d2); a.eps_r2 = T(d.eps_r2); a.has_d = d.has_d;
    a.lut = d.lut;
    a.box_wi = T(d.blur.wi);
    return launch_fused_t<T, RR, LP, RR>(a, true, batch, st);
}

template <typename T>
cudaError_t launch_fused_box_parta(const FusedLinesArgs &d, int radius, int64_t batch, cudaStream_t st) {
    const int lpw = fused_lpw(sizeof(T) == 8 ? 0 : 1);
    auto go = [&](auto rtag) -> cudaError_t {
        constexpr int RR = decltype(rtag)::value;
        if constexpr (sizeof(T) == 8) {
            return go_lp<T, RR, 2>(d, batch, st);
        } else {
            return lpw == 2 ? go_lp<T, RR, 2>(d, batch, st) : go_lp<T, RR, 4>(d, batch, st);
        }
    };
    switch (radius) {
        case 1: return go(std::integral_constant<int, 1>{});
        case 2: return go(std::integral_constant<int, 2>{});
        case 3: return go(std::integral_constant<int, 3>{});
        case 4: return go(std::integral_constant<int, 4>{});
        case 5: return go(std::integral_constant<int, 5>{});
        case 6: return go(std::integral_constant<int, 6>{});
        case 7: return go(std::integral_constant<int, 7>{});
        case 8: return go(std::integral_constant<int, 8>{});
        default: return cudaErrorInvalidValue;
    }
}

template cudaError_t launch_fused_box_parta<double>(const FusedLinesArgs &, int, int64_t, cudaStream_t);
template cudaError_t launch_fused_box_parta<float>(const FusedLinesArgs &, int, int64_t, cudaStream_t);

}  // namespace md
