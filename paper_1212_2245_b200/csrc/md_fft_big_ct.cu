// md_fft_big_ct.cu -- two-level FFT pass kernels with the sub-transform length fixed at compile
// time (2^6 .. 2^10: every split of the 2^12 .. 2^20-point axes the large-image Wiener, the
// slab column passes and the transform API use), float64. See k_subfft (md_fft_big_kernel.cuh).
#include "md_fft_big_kernel.cuh"

namespace md {

namespace {
template <int LOG2L, bool LF>
void (*pick_tw(int tw_mode))(SubFftArgs) {
    switch (tw_mode) {
        case TW_FWD: return k_subfft<double, LF, TW_FWD, LOG2L>;
        case TW_INV: return k_subfft<double, LF, TW_INV, LOG2L>;
        case TW_FILT_INV: return k_subfft<double, LF, TW_FILT_INV, LOG2L>;
        default: return k_subfft<double, LF, TW_NONE, LOG2L>;
    }
}
template <int LOG2L>
void (*pick_lf(bool line_fast, int tw_mode))(SubFftArgs) {
    return line_fast ? pick_tw<LOG2L, true>(tw_mode) : pick_tw<LOG2L, false>(tw_mode);
}
}  // namespace

template <>
void (*subfft_ct_kernel<double>(int log2L, bool line_fast, int tw_mode))(SubFftArgs) {
    switch (log2L) {
        case 6: return pick_lf<6>(line_fast, tw_mode);
        case 7: return pick_lf<7>(line_fast, tw_mode);
        case 8: return pick_lf<8>(line_fast, tw_mode);
        case 9: return pick_lf<9>(line_fast, tw_mode);
        case 10: return pick_lf<10>(line_fast, tw_mode);
        default: return nullptr;
    }
}

template <>
void (*subfft_ct_kernel<float>(int, bool, int))(SubFftArgs) {
    return nullptr;
}

}  // namespace md
