// md_fft.cuh -- shared-memory radix-2 FFT building blocks.
//
// Convolution-style pairing: the forward transform is decimation-in-frequency (natural
// order in, bit-reversed order out), the inverse is decimation-in-time (bit-reversed in,
// natural out). Spectra and filters are therefore stored in bit-reversed order and no
// permutation pass is ever executed. Convention matches the reference FourierPlan
// (fft.py:52-117): forward unnormalised, inverse scaled by 1/n by the caller's epilogue.
// Twiddles tw[k] = exp(-2*pi*i*k/n), k < n/2, are tabulated per length at plan time.
#pragma once

#include "md_common.cuh"

namespace md {

// Shared-memory position of element j of a line: one pad slot after every 8 elements. The
// radix-4 stages with small spans access elements 8, 32, ... apart; unpadded, 16-byte (f64
// complex) elements at stride 8 all fall into one bank group (16-way conflicts, measured
// 2.8e8 conflicts per two-level pass at 16384^2); padded, they spread over all banks.
// ES = element bytes: 16-byte (complex double) lines pad once per 8 elements, 8-byte (complex
// float) ones once per 16 -- then a half-warp's 8-byte accesses at strides 1, 2, 4, 8, 16 hit
// distinct banks (one pad per 8 left the small-span radix-4 stages 2-4-way conflicted)
template <int ES = 16> __host__ __device__ constexpr int fpad(int j) { return j + (j >> (ES <= 8 ? 4 : 3)); }
// storage length of a padded line of n elements
template <int ES = 16> __host__ __device__ constexpr int fpad_len(int n) { return fpad<ES>(n - 1) + 1; }
// stride between padded lines that are accessed across lines (transposed loads / stores):
// = 1 (mod 8), so 8 consecutive lines fall into 8 different bank groups for 16-byte complex
// elements (and 16 into different bank pairs for 8-byte ones)
template <int ES = 16> __host__ __device__ constexpr int fline_stride(int n) { return ((fpad_len<ES>(n) + 6) & ~7) + 1; }

// `nl` lines of length n = 2^log2n at s[l * stride + fpad(j)]; all threads of the block take part.
// Pairs of radix-2 stages are fused into radix-4 units (4 elements in registers), halving the
// shared-memory round trips and barriers; an odd stage count leaves one radix-2 stage.
template <typename C>
__device__ __forceinline__ C mul_mi(C a) {          // a * (-i)
    C r; r.x = a.y; r.y = -a.x; return r;
}

// Stage-major twiddle table for the STAGED variants: the stage with butterfly half-size h reads
// W_{2h}^k, k < h, at tws[h - 1 + k] (n - 1 entries in all), so consecutive lanes of a stage
// read consecutive entries -- the natural table read at tw[k << shift] strides the banks. Filled
// by a block from the plan's natural table twg[k] = W_n^k, k < n/2.
// BD: the block size when the caller knows it at compile time (0: blockDim.x) -- with the
// length also a compile-time constant the loops below unroll and their index math folds
template <int BD = 0, typename C>
__device__ __forceinline__ void stage_twiddles(C *tws, const C *__restrict__ twg, int log2n) {
    const int n = 1 << log2n;
    const int bd = BD ? BD : (int)blockDim.x;
    for (int i = threadIdx.x; i < n - 1; i += bd) {
        const int lh = 31 - __clz(i + 1), h = 1 << lh;     // stage of entry i
        tws[i] = twg[(i - (h - 1)) << (log2n - 1 - lh)];   // W_{2h}^k = W_n^{k n / 2h}
    }
}

template <bool STAGED = false, int BD = 0, typename C>
__device__ __forceinline__ void fft_dif_lines(C *s, int log2n, int nl, int stride, const C *__restrict__ tw) {
    const int n = 1 << log2n;
    const int bd = BD ? BD : (int)blockDim.x;
    int lh = log2n - 1;
    if (log2n & 1) {                               // lone radix-2 stage, half = n/2
        const int half = n >> 1;
        for (int b = threadIdx.x; b < (nl << lh); b += bd) {
            const int l = b >> lh, k = b & (half - 1);
            C *row = s + l * stride;
            const C a = row[fpad<sizeof(C)>(k)], c = row[fpad<sizeof(C)>(k + half)];
            row[fpad<sizeof(C)>(k)] = cadd(a, c);
            row[fpad<sizeof(C)>(k + half)] = cmul(csub(a, c), tw[STAGED ? half - 1 + k : k]);
        }
        __syncthreads();
        --lh;
    }
    const int lu = log2n - 2;                      // log2(n/4) units per line
    for (; lh >= 1; lh -= 2) {
        const int h = 1 << lh, q = h >> 1;
        for (int u = threadIdx.x; u < (nl << lu); u += bd) {
            const int l = u >> lu, uu = u & ((n >> 2) - 1);
            const int k = uu & (q - 1);
            const int i0 = ((uu >> (lh - 1)) << (lh + 1)) + k;
            C *row = s + l * stride;
            const C x0 = row[fpad<sizeof(C)>(i0)], x1 = row[fpad<sizeof(C)>(i0 + q)], x2 = row[fpad<sizeof(C)>(i0 + h)], x3 = row[fpad<sizeof(C)>(i0 + h + q)];
            const C w1 = STAGED ? tw[h - 1 + k] : tw[k << (log2n - 1 - lh)];      // W_{2h}^k
            const C w2 = STAGED ? tw[q - 1 + k] : tw[k << (log2n - lh)];          // W_h^k
            const C y0 = cadd(x0, x2), y2 = cmul(csub(x0, x2), w1);
            const C y1 = cadd(x1, x3), y3 = cmul(csub(x1, x3), mul_mi(w1));
            row[fpad<sizeof(C)>(i0)] = cadd(y0, y1);
            row[fpad<sizeof(C)>(i0 + q)] = cmul(csub(y0, y1), w2);
            row[fpad<sizeof(C)>(i0 + h)] = cadd(y2, y3);
            row[fpad<sizeof(C)>(i0 + h + q)] = cmul(csub(y2, y3), w2);
        }
        __syncthreads();
    }
}

// inverse (conjugate twiddles), bit-reversed in -> natural out, unscaled
template <bool STAGED = false, int BD = 0, typename C>
__device__ __forceinline__ void fft_dit_inv_lines(C *s, int log2n, int nl, int stride, const C *__restrict__ tw) {
    const int n = 1 << log2n;
    const int bd = BD ? BD : (int)blockDim.x;
    const int hb = log2n - 1;
    const int lu = log2n - 2;
    int lh = 0;
    for (; lh + 1 <= hb; lh += 2) {                // stages half = 2^lh and 2^(lh+1)
        const int q = 1 << lh, h = q << 1;
        for (int u = threadIdx.x; u < (nl << lu); u += bd) {
            const int l = u >> lu, uu = u & ((n >> 2) - 1);
            const int k = uu & (q - 1);
            const int i0 = ((uu >> lh) << (lh + 2)) + k;
            C *row = s + l * stride;
            const C x0 = row[fpad<sizeof(C)>(i0)], x1 = row[fpad<sizeof(C)>(i0 + q)], x2 = row[fpad<sizeof(C)>(i0 + h)], x3 = row[fpad<sizeof(C)>(i0 + h + q)];
            const C w2 = STAGED ? tw[q - 1 + k] : tw[k << (log2n - lh - 1)];      // W_h^k
            const C w1 = STAGED ? tw[h - 1 + k] : tw[k << (log2n - lh - 2)];      // W_{2h}^k
            C t = cmulc(x1, w2);
            const C y0 = cadd(x0, t), y1 = csub(x0, t);
            t = cmulc(x3, w2);
            const C y2 = cadd(x2, t), y3 = csub(x2, t);
            t = cmulc(y2, w1);
            row[fpad<sizeof(C)>(i0)] = cadd(y0, t);
            row[fpad<sizeof(C)>(i0 + h)] = csub(y0, t);
            t = cmulc(y3, mul_mi(w1));
            row[fpad<sizeof(C)>(i0 + q)] = cadd(y1, t);
            row[fpad<sizeof(C)>(i0 + h + q)] = csub(y1, t);
        }
        __syncthreads();
    }
    if (lh == hb) {                                // lone radix-2 stage, half = n/2
        const int half = n >> 1;
        for (int b = threadIdx.x; b < (nl << hb); b += bd) {
            const int l = b >> hb, k = b & (half - 1);
            C *row = s + l * stride;
            const C t = cmulc(row[fpad<sizeof(C)>(k + half)], tw[STAGED ? half - 1 + k : k]);
            const C a = row[fpad<sizeof(C)>(k)];
            row[fpad<sizeof(C)>(k + half)] = csub(a, t);
            row[fpad<sizeof(C)>(k)] = cadd(a, t);
        }
        __syncthreads();
    }
}

// ---- compile-time-length variants: several stages per shared-memory round trip --------------
// With the length and the line count known at compile time, a thread can hold 2^NS elements of
// a line in registers and run NS consecutive radix-2 stages on them before writing back (one
// load/store + one barrier per group of stages instead of per radix-4 unit). The butterflies,
// their twiddle operands and their order per element are exactly those of fft_dif_lines /
// fft_dit_inv_lines with STAGED twiddles -- including which twiddles come from the table and
// which are the exact (-i) rotation of a table entry (the second pair of a radix-4 unit) --
// -- the same operations, but not bit-identical results: see fft_dif_lines_ct below.
//
// DIF stage with half size hs = 2^lh (stages run lh = log2n-1 .. 0): `mi` marks the first stage
// of a radix-4 unit, whose pairs at positions p >= hs/2 use -i * table[p - hs/2]
template <int LOG2N>
__device__ __forceinline__ constexpr bool dif_stage_mi(int lh) {
    return !((LOG2N & 1) && lh == LOG2N - 1) && (((LOG2N - 1 - (LOG2N & 1)) - lh) % 2 == 0);
}
// DIT (inverse) stages run lh = 0 .. log2n-1; units pair (lh, lh+1) for even lh, the second
// (odd lh) uses the rotation; an odd count leaves a lone plain stage at the top
__device__ __forceinline__ constexpr bool dit_stage_mi(int lh) { return (lh & 1) != 0; }

// one group of NS stages, top stage LT (DIF: LT, LT-1, .., LB; DIT: LB, .., LT), over NL lines
template <int LOG2N, int LT, int NS, bool INV, int NL, int BD, typename C>
__device__ __forceinline__ void fft_group_ct(C *s, int stride, const C *__restrict__ tw) {
    constexpr int LB = LT - NS + 1, E = 1 << NS, SB = 1 << LB;
    constexpr int LOG2UPL = LOG2N - NS;                 // units (thread tasks) per line
    constexpr int NU = NL << LOG2UPL;
    static_assert(LB >= 0 && LT < LOG2N, "stage group out of range");
#pragma unroll 1
    for (int u = threadIdx.x; u < NU; u += BD) {
        const int l = u >> LOG2UPL, r = u & ((1 << LOG2UPL) - 1);
        const int k = r & (SB - 1), blk = r >> LB;
        const int base = (blk << (LT + 1)) + k;
        C *row = s + l * stride;
        C v[E];
#pragma unroll
        for (int j = 0; j < E; ++j) v[j] = row[fpad<sizeof(C)>(base + (j << LB))];
#pragma unroll
        for (int st = 0; st < NS; ++st) {
            const int lh = INV ? LB + st : LT - st;
            const int hs = 1 << lh, q = hs >> 1, js = 1 << (lh - LB);
            const bool mi = INV ? dit_stage_mi(lh) : dif_stage_mi<LOG2N>(lh);
#pragma unroll
            for (int j = 0; j < E; ++j) {
                if (j & js) continue;
                const int p = k + ((j << LB) & (hs - 1));          // position in the half
                C w;
                if (mi) {
                    const C w0 = tw[hs - 1 + (p & (q - 1))];
                    w = (p & q) ? mul_mi(w0) : w0;
                } else {
                    w = tw[hs - 1 + p];
                }
                const C a = v[j], c = v[j + js];
                if (INV) {
                    const C t = cmulc(c, w);
                    v[j] = cadd(a, t);
                    v[j + js] = csub(a, t);
                } else {
                    v[j] = cadd(a, c);
                    v[j + js] = cmul(csub(a, c), w);
                }
            }
        }
#pragma unroll
        for (int j = 0; j < E; ++j) row[fpad<sizeof(C)>(base + (j << LB))] = v[j];
    }
    __syncthreads();
}

// the whole transform: greedy groups of MD_SUBFFT_GROUPS stages from the top (DIF) / bottom
// (DIT), the remainder group taking the leftover stages. MEASUREMENT OPTION, off by default
// (md_fft_big_kernel.cuh): with 3-stage groups the c5 16384^2 Wiener ran 10 % faster (30 %
// fewer shared wavefronts) but the butterflies of a group split across a radix-4 unit round
// differently (the compiler contracts a lane-selected rotation differently), and the noise-
// free c5 problem amplifies that past the parity bar
template <int LOG2N, int NL, int BD, int GS, int LT = LOG2N - 1, typename C>
__device__ __forceinline__ void fft_dif_lines_ct(C *s, int stride, const C *__restrict__ tw) {
    constexpr int NS = LT + 1 < GS ? LT + 1 : GS;
    fft_group_ct<LOG2N, LT, NS, false, NL, BD>(s, stride, tw);
    if constexpr (LT + 1 - NS > 0) fft_dif_lines_ct<LOG2N, NL, BD, GS, LT - NS>(s, stride, tw);
}
template <int LOG2N, int NL, int BD, int GS, int LB = 0, typename C>
__device__ __forceinline__ void fft_dit_inv_lines_ct(C *s, int stride, const C *__restrict__ tw) {
    constexpr int NS = LOG2N - LB < GS ? LOG2N - LB : GS;
    fft_group_ct<LOG2N, LB + NS - 1, NS, true, NL, BD>(s, stride, tw);
    if constexpr (LB + NS < LOG2N) fft_dit_inv_lines_ct<LOG2N, NL, BD, GS, LB + NS>(s, stride, tw);
}

}  // namespace md
