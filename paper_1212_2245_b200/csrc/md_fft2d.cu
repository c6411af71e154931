// md_fft2d.cu -- 2D FFT passes for the FOURIER_2D scenario with dense kernels (the
// _FourierConvolver2D / wiener_2d path, deconv.py:257-272, 359-376, 660-664; fft.py:165-170,
// 274-280) and for PSF spectra.
//
// A 2D transform is a row pass (length W, contiguous) and a column pass (length H). The
// forward direction is DIF, so a spectrum is held in "storage coordinates" -- bit-reversed
// along both axes -- and filters are computed in the same coordinates; inverse passes are
// DIT and return natural order. Pointwise RRRL work is fused into the row passes:
//   row pass  : [load] -> [inverse DIT] -> epilogue -> [forward DIF of the packed result]
//   col pass  : DIF -> x filter (or conj) -> DIT        (or DIF only, for spectra)
// With this fusion one FOURIER_2D iteration is 4 launches:
//   rows(inv, stage A: b -> W, p; pack p + iW; fwd) -> cols(x conj h) ->
//   rows(inv, stage B: adjoint pair + TV + update; pack u'; fwd) -> cols(x h)
#include "md_fft.cuh"
#include <cstdlib>
#include "md_plane.h"

namespace md {

// TV divergence at (y, x) straight from global memory (the row pass owns one row only)
template <typename T>
__device__ T tv_div_global(const T *__restrict__ u, int H, int W, int y, int x, T eps_r2) {
    auto at = [&](int yy, int xx) { return __ldg(u + (int64_t)yy * W + xx); };
    auto gfun = [&](int yy, int xx) {
        const T c = at(yy, xx);
        T q = T(0);
        if (xx + 1 < W) { const T d = at(yy, xx + 1) - c; q += d * d; }
        if (xx > 0) { const T d = c - at(yy, xx - 1); q += d * d; }
        if (yy + 1 < H) { const T d = at(yy + 1, xx) - c; q += d * d; }
        if (yy > 0) { const T d = c - at(yy - 1, xx); q += d * d; }
        return T(0.5) / sqrt(T(0.5) * q + eps_r2);
    };
    const T u0 = at(y, x), gc = gfun(y, x);
    T d = T(0);
    if (x + 1 < W) d += (gc + gfun(y, x + 1)) * (at(y, x + 1) - u0);
    if (x > 0) d -= (gfun(y, x - 1) + gc) * (u0 - at(y, x - 1));
    if (y + 1 < H) d += (gc + gfun(y + 1, x)) * (at(y + 1, x) - u0);
    if (y > 0) d -= (gfun(y - 1, x) + gc) * (u0 - at(y - 1, x));
    return d;
}

template <typename T>
__global__ void __launch_bounds__(256)
k_fft2_rows(Fft2Args a, int rb, int staged) {
    // `rb` consecutive rows per block (all threads busy in every FFT stage)
    using C = cx_t<T>;
    constexpr int U = 4;                              // global loads in flight per thread
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C *s = reinterpret_cast<C *>(smem_raw);
    const int H = a.H, W = a.W, lw = a.log2W;
    const int y0 = blockIdx.x * rb;
    const int64_t fsz = (int64_t)H * W;
    const int64_t fr = blockIdx.y;
    const int64_t base = fr * fsz + (int64_t)y0 * W;      // rb rows are contiguous
    // real frames: with pairing, frames 2 fr (real part) and 2 fr + 1 (imaginary part)
    const int64_t fa = a.pairs ? 2 * fr : fr;
    const bool has_b = a.pairs && fa + 1 < a.nreal;
    const int64_t rbase_a = fa * fsz + (int64_t)y0 * W, rbase_b = rbase_a + fsz;
    const int ne = rb * W;
    const int bd = blockDim.x;
    C *z = static_cast<C *>(a.z);
    const int LS = fpad_len<sizeof(C)>(W);                       // padded row stride (md_fft.cuh)
    auto sp = [&](int i) { return (i >> lw) * LS + fpad<sizeof(C)>(i & (W - 1)); };
    // twiddles staged in shared memory behind the rows: the butterflies read them every stage
    C *tw = s + rb * LS;
    {
        const C *twg = static_cast<const C *>(a.twW);
        if (staged) stage_twiddles(tw, twg, lw);      // stage-major: conflict-free per-stage reads
        else for (int k = threadIdx.x; k < (W >> 1); k += blockDim.x) tw[k] = twg[k];
    }

    if (a.load == R_LOAD_COMPLEX) {
        for (int i0 = threadIdx.x; i0 < ne; i0 += U * bd) {
            C v[U];
#pragma unroll
            for (int k = 0; k < U; ++k) if (i0 + k * bd < ne) v[k] = z[base + i0 + k * bd];
#pragma unroll
            for (int k = 0; k < U; ++k) if (i0 + k * bd < ne) s[sp(i0 + k * bd)] = v[k];
        }
    } else {
        const T *ra = static_cast<const T *>(a.ra);
        // R_LOAD_PAIR: second real field at rb (same frame); pairing: the next frame of ra
        const T *rbp = a.pairs ? (has_b ? ra + rbase_b : nullptr)
                               : (a.rb ? static_cast<const T *>(a.rb) + rbase_a : nullptr);
        for (int i0 = threadIdx.x; i0 < ne; i0 += U * bd) {
            T xa[U], xb[U];
#pragma unroll
            for (int k = 0; k < U; ++k) {
                const int i = i0 + k * bd;
                xa[k] = i < ne ? ra[rbase_a + i] : T(0);
                xb[k] = (i < ne && rbp) ? rbp[i] : T(0);
            }
#pragma unroll
            for (int k = 0; k < U; ++k) if (i0 + k * bd < ne) s[sp(i0 + k * bd)] = mkc<T>(xa[k], xb[k]);
        }
    }
    __syncthreads();
    if (a.inv && lw > 0) {
        if (staged) fft_dit_inv_lines<true>(s, lw, rb, LS, tw);
        else fft_dit_inv_lines<false>(s, lw, rb, LS, tw);
    }

    const T scale = T(a.scale), floor = T(a.floor);
    const T eps_d2 = T(a.eps_d2), eps_r2 = T(a.eps_r2), alpha = T(a.alpha);   // converted once
    if (a.epi != R_EPI_NONE) {
        for (int i0 = threadIdx.x; i0 < ne; i0 += U * bd) {
            // global operands of U elements first: the stores below could alias them, so a
            // load issued after a store would wait for it
            T g0[U], g1[U];
#pragma unroll
            for (int k = 0; k < U; ++k) {
                const int i = i0 + k * bd;
                g0[k] = g1[k] = T(0);
                if (i >= ne) continue;
                if (a.epi == R_EPI_WIENER && a.ob) {
                    g0[k] = static_cast<const T *>(a.f)[rbase_a + i];
                    if (has_b) g1[k] = static_cast<const T *>(a.f)[rbase_b + i];
                } else if (a.epi == R_EPI_STAGE_A) {
                    g0[k] = static_cast<const T *>(a.f)[base + i];
                } else if (a.epi == R_EPI_STAGE_B) {
                    g0[k] = static_cast<const T *>(a.u)[base + i];
                    if (a.dpre) g1[k] = static_cast<const T *>(a.dpre)[base + i];
                }
            }
#pragma unroll
            for (int k = 0; k < U; ++k) {
                const int i = i0 + k * bd;
                if (i >= ne) continue;
                const C v = s[sp(i)];
                const int64_t o = base + i;
                C packed = mkc<T>(T(0), T(0));
                if (a.epi == R_EPI_STORE_PAIR) {
                    static_cast<T *>(a.oa)[o] = v.x * scale;
                    if (a.ob) static_cast<T *>(a.ob)[o] = v.y * scale;
                } else if (a.epi == R_EPI_WIENER) {
                    T w = v.x * scale, w1 = v.y * scale;
                    if (floor > T(0)) {                  // u0 = max(Wiener, floor)
                        w = w > floor ? w : floor;
                        w1 = w1 > floor ? w1 : floor;
                    }
                    static_cast<T *>(a.oa)[rbase_a + i] = w;
                    if (has_b) static_cast<T *>(a.oa)[rbase_b + i] = w1;
                    if (a.ob) {
                        static_cast<T *>(a.ob)[rbase_a + i] = g0[k] > floor ? g0[k] : floor;
                        if (has_b) static_cast<T *>(a.ob)[rbase_b + i] = g1[k] > floor ? g1[k] : floor;
                    }
                    packed = mkc<T>(w, T(0));
                } else if (a.epi == R_EPI_STAGE_A) {
                    T b = v.x * scale;
                    b = b > T(kGuard) ? b : T(kGuard);
                    const T fp = g0[k];
                    const T ratio = fp / b;
                    if (a.robust) {
                        const T wv = robust_weight_floored<T>(a.lut, fp, b, eps_d2);
                        packed = mkc<T>(wv * ratio, wv);
                    } else {
                        packed = mkc<T>(ratio, T(0));
                    }
                } else {  // R_EPI_STAGE_B
                    const T *u = static_cast<const T *>(a.u) + fr * fsz;
                    const int y = y0 + (i >> lw), x = i & (W - 1);
                    const T uv = g0[k];
                    // the divergence from one pass over the frame (k_diffusion: each diffusivity
                    // once, not five times per pixel) or evaluated here from global memory
                    const T d = !a.has_d ? T(0) : (a.dpre ? g1[k] : tv_div_global<T>(u, H, W, y, x, eps_r2));
                    const T un = a.robust ? combine_px<T, true>(uv, v.x * scale, v.y * scale, d, alpha, a.has_d != 0)
                                          : combine_px<T, false>(uv, v.x * scale, T(0), d, alpha, a.has_d != 0);
                    static_cast<T *>(a.oa)[o] = un;
                    packed = mkc<T>(un, T(0));
                }
                s[sp(i)] = packed;
            }
        }
        __syncthreads();
    }
    if (a.fwd_after) {
        if (lw > 0) {
            if (staged) fft_dif_lines<true>(s, lw, rb, LS, tw);
            else fft_dif_lines<false>(s, lw, rb, LS, tw);
        }
        for (int i = threadIdx.x; i < ne; i += blockDim.x) z[base + i] = s[sp(i)];
    } else if (a.epi == R_EPI_NONE) {
        for (int i = threadIdx.x; i < ne; i += blockDim.x) z[base + i] = s[sp(i)];
    }
}

template <typename T>
__global__ void __launch_bounds__(256)
k_fft2_cols(Fft2Args a, int lcw) {
    using C = cx_t<T>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C *s = reinterpret_cast<C *>(smem_raw);
    const int H = a.H, W = a.W, cs = fline_stride<sizeof(C)>(H);      // padded column stride (md_fft.cuh)
    const int cw = 1 << lcw;                                // a power of two: shifts, no division
    const int x0 = blockIdx.x * cw;
    const int64_t base = blockIdx.y * (int64_t)H * W;
    C *z = static_cast<C *>(a.z);
    C *tw = s + cw * cs;                              // staged twiddles (see k_fft2_rows)
    {
        const C *twg = static_cast<const C *>(a.twH);
        stage_twiddles(tw, twg, a.log2H);
    }
    // element idx -> (row y, column c), columns fastest: a warp reads whole row segments of the
    // block's columns (coalesced), and the padded column stride (= 1 mod 8) keeps the shared
    // stores conflict-free. U loads in flight per thread (a load after a shared store could not
    // be hoisted above it: z may alias as far as the compiler knows)
    constexpr int U = 4;
    const int n = cw * H, bd = blockDim.x;
#ifndef MD_FFT2_COLS_CP_ASYNC
#define MD_FFT2_COLS_CP_ASYNC 1
#endif
#if MD_FFT2_COLS_CP_ASYNC
    // cp.async (global -> shared, no register round trip): the whole block of columns in flight at
    // once, columns past the frame zero-filled
    for (int idx = threadIdx.x; idx < n; idx += bd) {
        const int y = idx >> lcw, c = idx & (cw - 1);
        const bool ok = x0 + c < W;
        const C *src = ok ? z + base + (int64_t)y * W + x0 + c : z;
        const uint32_t d = (uint32_t)__cvta_generic_to_shared(&s[c * cs + fpad<sizeof(C)>(y)]);
        if (sizeof(C) == 16)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(ok ? 16 : 0) : "memory");
        else
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(src), "r"(ok ? 8 : 0) : "memory");
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
#else
    for (int i0 = threadIdx.x; i0 < n; i0 += U * bd) {
        C v[U];
#pragma unroll
        for (int k = 0; k < U; ++k) {
            const int idx = i0 + k * bd;
            const int y = idx >> lcw, c = idx & (cw - 1);
            v[k] = (idx < n && x0 + c < W) ? z[base + (int64_t)y * W + x0 + c] : mkc<T>(T(0), T(0));
        }
#pragma unroll
        for (int k = 0; k < U; ++k) {
            const int idx = i0 + k * bd;
            if (idx >= n) break;
            const int y = idx >> lcw, c = idx & (cw - 1);
            s[c * cs + fpad<sizeof(C)>(y)] = v[k];
        }
    }
#endif
    __syncthreads();
    if (a.log2H > 0) fft_dif_lines<true>(s, a.log2H, cw, cs, tw);
    if (a.filt) {
        // the same row-segment order for the (natural-layout) multiplier: coalesced reads (a
        // column-major walk read one 16-byte element per 4 KB row)
        const C *filt = static_cast<const C *>(a.filt);
        for (int i0 = threadIdx.x; i0 < n; i0 += U * bd) {
            C f[U];
#pragma unroll
            for (int k = 0; k < U; ++k) {
                const int idx = i0 + k * bd;
                const int y = idx >> lcw, c = idx & (cw - 1);
                f[k] = (idx < n && x0 + c < W) ? __ldg(filt + (int64_t)y * W + x0 + c) : mkc<T>(T(0), T(0));
            }
#pragma unroll
            for (int k = 0; k < U; ++k) {
                const int idx = i0 + k * bd;
                const int y = idx >> lcw, c = idx & (cw - 1);
                if (idx >= n || x0 + c >= W) continue;
                C &e = s[c * cs + fpad<sizeof(C)>(y)];
                e = a.conj_filt ? cmulc(e, f[k]) : cmul(e, f[k]);
            }
        }
        __syncthreads();
    }
    if (a.col_inv && a.log2H > 0) fft_dit_inv_lines<true>(s, a.log2H, cw, cs, tw);
    for (int idx = threadIdx.x; idx < cw * H; idx += blockDim.x) {
        const int y = idx >> lcw, c = idx & (cw - 1);
        if (x0 + c < W) z[base + (int64_t)y * W + x0 + c] = s[c * cs + fpad<sizeof(C)>(y)];
    }
}

template <typename T>
cudaError_t launch_fft2_rows(const Fft2Args &a, int64_t batch, cudaStream_t st) {
    int rb = 2048 / a.W;                      // ~2048 elements per block
    rb = rb < 1 ? 1 : (rb > a.H ? a.H : rb);
    // stage-major twiddles (W - 1 entries) unless they would not fit (the plan-time float64
    // spectrum of an 8192-sample line): then the natural table (W / 2)
    size_t smem = ((size_t)rb * fpad_len<sizeof(cx_t<T>)>(a.W) + a.W + 1) * sizeof(cx_t<T>);
    int staged = 1;
    if (smem > 227 * 1024) {
        smem = ((size_t)rb * fpad_len<sizeof(cx_t<T>)>(a.W) + a.W / 2 + 1) * sizeof(cx_t<T>);
        staged = 0;
    }
    cudaError_t e = func_smem_attr((const void *)k_fft2_rows<T>, smem);
    if (e != cudaSuccess) return e;
    // `batch` counts complex fields; with pairing the real pointers advance two frames per field
    const int64_t fr = (int64_t)a.H * a.W;
    const int64_t rstep = a.pairs ? 2 : 1;
    for (int64_t b0 = 0; b0 < batch; b0 += 65535) {
        const int nb = (int)((batch - b0) < 65535 ? (batch - b0) : 65535);
        Fft2Args ab = a;
        auto sh = [&](const void *p, size_t es, int64_t step) -> const void * {
            return p ? static_cast<const char *>(p) + step * b0 * fr * es : nullptr;
        };
        ab.ra = sh(a.ra, sizeof(T), rstep);
        ab.rb = sh(a.rb, sizeof(T), rstep);
        ab.z = const_cast<void *>(sh(a.z, sizeof(cx_t<T>), 1));
        ab.oa = const_cast<void *>(sh(a.oa, sizeof(T), rstep));
        ab.ob = const_cast<void *>(sh(a.ob, sizeof(T), rstep));
        ab.f = sh(a.f, sizeof(T), rstep);
        ab.u = sh(a.u, sizeof(T), 1);
        ab.nreal = a.nreal - rstep * b0;
        k_fft2_rows<T><<<dim3(a.H / rb, nb), 256, smem, st>>>(ab, rb, staged);
    }
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_fft2_cols(const Fft2Args &a, int64_t batch, cudaStream_t st) {
    // columns per block: up to one 128-byte line per row (8 float64 / 16 float32 complex
    // columns) -- 16 float64 columns (78 KB of shared memory, 2 blocks/SM) ran the 256^2
    // Wiener column pass 20 % slower than 8 (39 KB); 4 was slower again
    constexpr int kColW = 128 / (int)sizeof(cx_t<T>);
    // 1024-high columns: 2 per block (32 KB, 4 blocks/SM) measured 1.8 % faster on the c3 iterations
    // than 4 (64 KB); 8 and 1 slower (MD_FFT2_COLW, scripts/c3_hash_probe.py)
    int cw = a.H >= 1024 ? 2048 / a.H : 4096 / a.H;
    cw = cw > kColW ? kColW : (cw < 1 ? 1 : cw);          // a power of two (H is)
    static const int cw_env = [] { const char *v = std::getenv("MD_FFT2_COLW"); return v ? std::atoi(v) : 0; }();
    if (cw_env > 0) cw = cw_env;                          // measurement knob (a power of two)
    int lcw = 0;
    while ((1 << lcw) < cw) ++lcw;
    const size_t smem = ((size_t)cw * fline_stride<sizeof(cx_t<T>)>(a.H) + a.H + 1) * sizeof(cx_t<T>);
    cudaError_t e = func_smem_attr((const void *)k_fft2_cols<T>, smem);
    if (e != cudaSuccess) return e;
    const int64_t fr = (int64_t)a.H * a.W;
    for (int64_t b0 = 0; b0 < batch; b0 += 65535) {
        const int nb = (int)((batch - b0) < 65535 ? (batch - b0) : 65535);
        Fft2Args ab = a;
        ab.z = static_cast<char *>(a.z) + b0 * fr * sizeof(cx_t<T>);
        k_fft2_cols<T><<<dim3((a.W + cw - 1) / cw, nb), 256, smem, st>>>(ab, lcw);
    }
    return cudaGetLastError();
}

template cudaError_t launch_fft2_rows<double>(const Fft2Args &, int64_t, cudaStream_t);
template cudaError_t launch_fft2_rows<float>(const Fft2Args &, int64_t, cudaStream_t);
template cudaError_t launch_fft2_cols<double>(const Fft2Args &, int64_t, cudaStream_t);
template cudaError_t launch_fft2_cols<float>(const Fft2Args &, int64_t, cudaStream_t);

}  // namespace md
