// md_fft_big_kernel.cuh -- the two-level FFT pass kernel (k_subfft), shared by md_fft_big.cu
// (host side, generic-length instantiations) and md_fft_big_ct.cu (compile-time lengths).
#pragma once
#include "md_fft.cuh"
#include "md_fft_big.h"

namespace md {

// LINE_FAST: contiguous lines (es == 1); TW: the inter-pass twiddle mode (TW_NONE / FWD / INV),
// compile-time so that each pass carries only its own epilogue
// LOG2L > 0: the sub-transform length is a compile-time constant (the c5 / large-image lengths
// 2^6 .. 2^10, md_fft_big_ct.cu) -- with it the line count per block, the padded stride and the
// 256-thread loops are constants, so the stage loops unroll and their shift / mask / address
// arithmetic folds (the generic kernel spent ~100 of its ~180 instructions per element on it);
// LOG2L = 0: any length, from the arguments
constexpr int subfft_lines(int log2l) { return (2048 >> log2l) < 1 ? 1 : ((2048 >> log2l) > 16 ? 16 : (2048 >> log2l)); }

// measurement option (off): register stage groups of MD_SUBFFT_GROUPS stages in the
// constant-length kernels (md_fft.cuh); 3 with MD_SUBFFT_MINB=4 (<= 64 registers) was the
// fastest variant -- c5 Wiener 17.6 -> 15.8 ms -- but it is not bit-compatible with the
// parity fixtures. With the option off the kernel is unchanged.
#ifndef MD_SUBFFT_GROUPS
#define MD_SUBFFT_GROUPS 0
#endif
#if MD_SUBFFT_GROUPS
#ifndef MD_SUBFFT_MINB
#define MD_SUBFFT_MINB 4
#endif
#define MD_SUBFFT_DIF(...) do { if constexpr (LOG2L > 0) fft_dif_lines_ct<LOG2L, subfft_lines(LOG2L), BD, MD_SUBFFT_GROUPS>(s, ls, twL); else fft_dif_lines<true, BD>(s, log2L, G, ls, twL); } while (0)
#define MD_SUBFFT_DIT(...) do { if constexpr (LOG2L > 0) fft_dit_inv_lines_ct<LOG2L, subfft_lines(LOG2L), BD, MD_SUBFFT_GROUPS>(s, ls, twL); else fft_dit_inv_lines<true, BD>(s, log2L, G, ls, twL); } while (0)
#define MD_SUBFFT_BOUNDS __launch_bounds__(256, LOG2L > 0 ? MD_SUBFFT_MINB : 1)
#else
#define MD_SUBFFT_DIF(...) fft_dif_lines<true, BD>(s, log2L, G, ls, twL)
#define MD_SUBFFT_DIT(...) fft_dit_inv_lines<true, BD>(s, log2L, G, ls, twL)
#define MD_SUBFFT_BOUNDS __launch_bounds__(256)
#endif
template <typename T, bool LINE_FAST, int TW, int LOG2L>
__global__ void MD_SUBFFT_BOUNDS
k_subfft(SubFftArgs a) {
    using C = cx_t<T>;
    constexpr int BD = 256;                    // launch_subfft always uses 256 threads
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C *s = reinterpret_cast<C *>(smem_raw);
    const int log2L = LOG2L ? LOG2L : a.log2L;
    const int L = 1 << log2L, G = LOG2L ? subfft_lines(LOG2L) : a.G;
    const int ls = fline_stride<sizeof(C)>(L);   // padded line stride (md_fft.cuh)
    const int blocks_b = (a.B + G - 1) / G;
    const int ai = blockIdx.x / blocks_b, b0 = (blockIdx.x - ai * blocks_b) * G;
    const int64_t fr = blockIdx.y;
    C *z = static_cast<C *>(a.z) + fr * a.frame;
    const T *ra = a.ra ? static_cast<const T *>(a.ra) + fr * a.rframe : nullptr;
    const T *rb = a.rb ? static_cast<const T *>(a.rb) + fr * a.rframe : nullptr;
    // offsets within a frame fit 32 bits (launch_subfft checks frame < 2^31): cheaper address math
    const int sb = (int)a.sb, es = (int)a.es;
    const int base = ai * (int)a.sa + b0 * sb;
    constexpr bool line_fast = LINE_FAST;      // contiguous lines: iterate along the line
#ifndef MD_SUBFFT_U
#define MD_SUBFFT_U 4
#endif
    constexpr int U = MD_SUBFFT_U;             // global loads in flight per thread
    const int n = G * L, bd = BD;
    const int lg = 31 - __clz(G);              // G is a power of two
    auto coords = [&](int idx, int &g, int &e) {
        if (line_fast) { g = idx >> log2L; e = idx & (L - 1); }
        else { e = idx >> lg; g = idx & (G - 1); }
    };
#ifndef MD_SUBFFT_CP_ASYNC
#define MD_SUBFFT_CP_ASYNC 1
#endif
    if (MD_SUBFFT_CP_ASYNC) {
        // cp.async (global -> shared, no register round trip, every element of the block in
        // flight at once): one 16-byte copy per complex element, two 8-byte (4-byte) copies for a
        // real pair; lines past the batch and a missing second field zero-filled
        for (int idx = threadIdx.x; idx < n; idx += bd) {
            int g, e;
            coords(idx, g, e);
            const bool ok = b0 + g < a.B;
            const int o = ok ? base + g * sb + e * es : 0;
            C *d = &s[g * ls + fpad<sizeof(C)>(e)];
            const uint32_t da = (uint32_t)__cvta_generic_to_shared(d);
            if (ra) {
                constexpr int ES = (int)sizeof(T);
                const uint32_t db = da + ES;
                const T *pa = ra + o, *pb = rb ? rb + o : ra;
                const int na = ok ? ES : 0, nb2 = ok && rb ? ES : 0;
                if (ES == 8) {
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(da), "l"(pa), "r"(na) : "memory");
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(db), "l"(pb), "r"(nb2) : "memory");
                } else {
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(da), "l"(pa), "r"(na) : "memory");
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(db), "l"(pb), "r"(nb2) : "memory");
                }
            } else {
                const C *pz = z + o;
                if (sizeof(C) == 16)
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(da), "l"(pz), "r"(ok ? 16 : 0) : "memory");
                else
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(da), "l"(pz), "r"(ok ? 8 : 0) : "memory");
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    } else {
    for (int i0 = threadIdx.x; i0 < n; i0 += U * bd) {
        C v[U];
#pragma unroll
        for (int k = 0; k < U; ++k) {
            const int idx = i0 + k * bd;
            int g, e;
            coords(idx, g, e);
            v[k] = mkc<T>(T(0), T(0));
            if (idx < n && b0 + g < a.B) {
                const int o = base + g * sb + e * es;
                if (ra) v[k] = mkc<T>(ra[o], rb ? rb[o] : T(0));
                else v[k] = z[o];
            }
        }
#pragma unroll
        for (int k = 0; k < U; ++k) {
            const int idx = i0 + k * bd;
            if (idx >= n) break;
            int g, e;
            coords(idx, g, e);
            s[g * ls + fpad<sizeof(C)>(e)] = v[k];
        }
    }
    }
    C *twL = s + G * ls;                       // sub-transform twiddles staged in shared memory
    stage_twiddles<BD>(twL, static_cast<const C *>(a.twL), log2L);   // stage-major (md_fft.cuh)
    if (MD_SUBFFT_CP_ASYNC) asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    const C *filt = static_cast<const C *>(a.filt);
    if (TW == TW_FILT_INV) {
        MD_SUBFFT_DIF();
        for (int idx = threadIdx.x; idx < n; idx += bd) {
            int g, e;
            coords(idx, g, e);
            if (b0 + g >= a.B) continue;
            const C fl = filt[base + g * sb + e * es];
            C &v = s[g * ls + fpad<sizeof(C)>(e)];
            v = a.conj_filt ? cmulc(v, fl) : cmul(v, fl);
        }
        __syncthreads();
        MD_SUBFFT_DIT();
    } else if (a.inv) {
        MD_SUBFFT_DIT();
    } else {
        MD_SUBFFT_DIF();
    }
    // inter-pass twiddle W_N^{+-(digit * rev(pos))}, digit = line (FWD) or element (INV) index
    const C *twN = static_cast<const C *>(a.twN);
    const int N = a.N;
    const T scale = T(a.scale);
    constexpr bool FILT_EPI = TW != TW_FILT_INV;        // the fused mode filtered in shared memory
    constexpr int TWM = TW == TW_FILT_INV ? TW_INV : TW;
    T *wu = static_cast<T *>(a.wu), *wfp = static_cast<T *>(a.wfpos);
    const T *wf = static_cast<const T *>(a.wf);
    const T wfloor = T(a.floor);
    for (int i0 = threadIdx.x; i0 < n; i0 += U * bd) {
        // table and filter operands first: loads after the z stores below would wait on them
        C tw[U], fl[U];
#pragma unroll
        for (int k = 0; k < U; ++k) {
            const int idx = i0 + k * bd;
            int g, e;
            coords(idx, g, e);
            tw[k] = fl[k] = mkc<T>(T(1), T(0));
            if (idx >= n || b0 + g >= a.B) continue;
            if (TWM != TW_NONE) {
                const int lb = a.tw_digit_is_a ? ai : b0 + g;                 // line digit
                const int re = (int)(__brev((unsigned)e) >> (32 - log2L));     // rev(pos) in the line
                const int rl = (int)(__brev((unsigned)lb) >> (32 - a.log2Lother));
                // FWD (after F1): W_N^{line * rev(e)};  INV (after I2): conj W_N^{e * rev(line)}
                const int kk = TWM == TW_FWD ? (int)(((int64_t)lb * re) & (N - 1)) : (int)(((int64_t)e * rl) & (N - 1));
                const C w = twN[kk & (N / 2 - 1)];
                tw[k] = kk < N / 2 ? w : mkc<T>(-w.x, -w.y);
            }
            if (FILT_EPI && filt) fl[k] = filt[base + g * sb + e * es];
        }
#pragma unroll
        for (int k = 0; k < U; ++k) {
            const int idx = i0 + k * bd;
            int g, e;
            coords(idx, g, e);
            if (idx >= n || b0 + g >= a.B) continue;
            C v = s[g * ls + fpad<sizeof(C)>(e)];
            if (TWM != TW_NONE) v = TWM == TW_FWD ? cmul(v, tw[k]) : cmulc(v, tw[k]);
            if (FILT_EPI && filt) v = a.conj_filt ? cmulc(v, fl[k]) : cmul(v, fl[k]);
            if (scale != T(1)) v = cscale(v, scale);
            const int o = base + g * sb + e * es;
            if (TW == TW_NONE && wu) {
                // Wiener epilogue (deconv.py:666-672): real part, clamp, floored observation
                const T x = v.x;
                wu[fr * a.rframe + o] = a.clamp ? (x > wfloor ? x : wfloor) : x;
                if (wfp) {
                    const T fv = wf[fr * a.rframe + o];
                    wfp[fr * a.rframe + o] = fv > wfloor ? fv : wfloor;
                }
            } else {
                z[o] = v;
            }
        }
    }
}

}  // namespace md
