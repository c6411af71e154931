// md_capi.cu -- the C ABI (include/mdcuda.h): plans, constant tables and kernel dispatch.
//
// A plan is the B200 counterpart of DeblurPipeline.__init__ (deconv.py:611-643) and
// make_convolver (deconv.py:379-403): it validates the problem, picks the kernel path,
// uploads the PSF taps, builds the twiddle tables, the divergence table (deconv.py:101-112)
// and the Wiener multiplier conj(h)/(|h|^2+K) (deconv.py:253-254) ON THE DEVICE, and owns
// the scratch fields. md_run is DeblurPipeline.run (deconv.py:653-693) for a batch.
//
// Kernel paths
//   LINES        1D PSFs (box or general, any convolver mode): k_wiener_lines + one
//                k_iter_lines launch per iteration (md_lines.cu).
//   PLANE_DIRECT 2D PSFs with a modest tap count: 2D-FFT Wiener + two direct-tap stage
//                kernels per iteration (md_plane.cu), periodic or clamped.
//   PLANE_FFT    2D PSFs with many taps: 2D-FFT Wiener + 4 fused FFT passes per iteration
//                (md_fft2d.cu).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>
#include <string>
#include <vector>

#include "../../include/mdcuda.h"
#include "md_fused.h"
#include "md_fused_plane.h"
#include "md_lines_fast.h"
#include "md_plane_fast.h"
#include "md_fft_big.h"
#include "md_plane.h"

using namespace md;

namespace {

// internal plan flag (not in mdcuda.h): a 1D PSF handed over from the line route as a plane
constexpr uint32_t kFlagLinePlane = 1u << 16;

thread_local std::string g_err;

int fail(int code, const std::string &msg) {
    g_err = msg;
    return code;
}

#define CU(expr)                                                                                   \
    do {                                                                                           \
        cudaError_t _e = (expr);                                                                   \
        if (_e != cudaSuccess) return fail(MD_ECUDA, std::string(#expr ": ") + cudaGetErrorString(_e)); \
    } while (0)

bool is_pow2(int n) { return n >= 1 && (n & (n - 1)) == 0; }

// a non-sticky error left by a call whose failure was handled (e.g. a kernel variant whose
// shared-memory attribute is refused, then another path taken) must not be reported by the
// next entry point's launch check
inline void clear_stale_error() { (void)cudaGetLastError(); }
int ilog2(int n) { int l = 0; while ((1 << l) < n) ++l; return l; }

enum Path { PATH_LINES = 0, PATH_PLANE_DIRECT = 1, PATH_PLANE_FFT = 2 };

// optional per-launch-group CUDA events (md_run_profile): kind 0 = init (Wiener / clamp),
// 1 = RRRL iterations, 2 = layout (transposes)
enum { PK_INIT = 0, PK_ITER = 1, PK_LAYOUT = 2, PK_KINDS = 3 };
struct Prof {
    std::vector<cudaEvent_t> ev;     // persistent per-thread pool (created once, reused)
    std::vector<int> kind;
    int n = 0;
    bool active = false;
    cudaEvent_t get(int i) {
        while ((int)ev.size() <= i) {
            cudaEvent_t e;
            cudaEventCreate(&e);
            ev.push_back(e);
            kind.push_back(0);
        }
        return ev[i];
    }
};
thread_local Prof g_prof_pool;
thread_local Prof *g_prof = nullptr;
inline void prof_mark(cudaStream_t st, int kind) {
    if (!g_prof) return;
    cudaEventRecord(g_prof->get(g_prof->n + 1), st);
    g_prof->kind[g_prof->n + 1] = kind;
    ++g_prof->n;
}

// ---------------------------------------------------------------- plan-time kernels
__global__ void k_build_lut(double *t64, float *t32, float2 *p32, double2 *p64) {
    auto val = [](int i) {
        const double x = kLutDelta + (1.0 / kLutInvStep) * (double)i;   // deconv.py:106-108
        return x - 1.0 - log(x);
    };
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < kLutCount; i += gridDim.x * blockDim.x) {
        const double v = val(i);
        t64[i] = v;
        t32[i] = (float)v;
        if (i + 1 < kLutCount) {
            const double step = val(i + 1) - v;      // the reference's T[i+1] - T[i] (deconv.py:131-133)
            p32[i] = make_float2((float)v, (float)step);
            p64[i] = make_double2(v, step);
        }
    }
}

__global__ void k_build_twiddles(double2 *t64, float2 *t32, int n) {
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n / 2; k += gridDim.x * blockDim.x) {
        double s, c;
        sincospi(-2.0 * (double)k / (double)n, &s, &c);
        t64[k] = make_double2(c, s);
        t32[k] = make_float2((float)c, (float)s);
    }
}

// mult = conj(h) / (|h|^2 + K) (or h itself when K < 0), converted to the plan dtype
__global__ void k_make_filter(const double2 *h, int64_t count, double K, double2 *o64, float2 *o32) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
        const double2 v = h[i];
        double2 r;
        if (K >= 0.0) {
            const double den = v.x * v.x + v.y * v.y + K;
            r = make_double2(v.x / den, -v.y / den);
        } else {
            r = v;
        }
        if (o64) o64[i] = r;
        if (o32) o32[i] = make_float2((float)r.x, (float)r.y);
    }
}

// dst[k] = src[bitrev(k)] for complex elements of `es` bytes (bit-reversed -> natural order)
__global__ void k_unbitrev(const unsigned char *src, unsigned char *dst, int n, int log2n, int es) {
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        const int r = (int)(__brev((unsigned)k) >> (32 - log2n));
        for (int b = 0; b < es; ++b) dst[(size_t)k * es + b] = src[(size_t)r * es + b];
    }
}

// scatter a direct-tap list into a zeroed H x W grid, centre at (0, 0), wrapped (fft.py:204-221)
// m[H][W] = m1[x] (axis 1) or m1[y] (axis 0): a 1D multiplier over a plane, byte-generic
__global__ void k_replicate_filter(const unsigned char *m1, unsigned char *m, int H, int W, int axis, int es) {
    const int64_t n = (int64_t)H * W;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = axis == 1 ? i % W : i / W;
        for (int b = 0; b < es; ++b) m[i * es + b] = m1[k * es + b];
    }
}

__global__ void k_embed_taps(double *z, int H, int W, const PlaneTap *taps, int nt) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nt; t += gridDim.x * blockDim.x) {
        const int y = ((-taps[t].dy) % H + H) % H, x = ((-taps[t].dx) % W + W) % W;
        z[(size_t)y * W + x] = taps[t].w;
    }
}

// set while this thread enqueues into a stream under capture: buffers cannot be reallocated
// then (an earlier graph may still reference the old one)
thread_local bool tl_capturing = false;

// Plan scratch. Once a CUDA graph has captured a run that uses the buffer, the graph holds its
// address: a later (uncaptured) run that needs more scratch gets a new buffer, and the old one is
// retired -- kept alive until the plan is destroyed -- so every captured graph stays valid.
struct DevBuf {
    void *p = nullptr;
    size_t bytes = 0;
    bool captured = false;               // some graph recorded launches that use `p`
    std::vector<void *> retired;
    void release() {
        if (p) cudaFree(p);
        for (void *q : retired) cudaFree(q);
        retired.clear();
        p = nullptr;
        bytes = 0;
        captured = false;
    }
    int ensure(size_t b) {
        if (tl_capturing) captured = true;
        if (b <= bytes) return MD_OK;
        if (tl_capturing) return fail(MD_EINVAL, "plan scratch must be sized by an uncaptured run before stream capture");
        if (captured) {
            retired.push_back(p);        // still referenced by a graph: keep it
            p = nullptr;
            bytes = 0;
            captured = false;
        } else if (p) {
            cudaFree(p);
            p = nullptr;
            bytes = 0;
        }
        if (cudaMalloc(&p, b) != cudaSuccess) { cudaGetLastError(); return fail(MD_ENOMEM, "device allocation failed"); }
        bytes = b;
        return MD_OK;
    }
};

}  // namespace

struct md_plan {
    md_plan_desc d{};
    std::vector<double> w, wrev;
    int es = 8;                 // element size
    int path = PATH_LINES;
    bool robust = true, has_d = true;
    // lines
    int vert = 0, n = 0, m = 0, log2n = -1;
    LineConv lblur{}, ladj{};
    double *d_taps_blur = nullptr, *d_taps_adj = nullptr;
    // plane
    PlaneHalo hblur{}, hadj{};
    PlaneTap *d_ptaps_blur = nullptr, *d_ptaps_adj = nullptr;
    std::vector<PlaneTap> htaps_blur, htaps_adj;
    bool fast_plane = false;    // register-blocked direct-tap stage kernels apply
    bool big = false;           // two-level FFT passes for the 2D Wiener step (large images)
    int line_axis = -1;         // a 1D PSF routed as a plane: its blur axis (1 rows, 0 columns) --
                                // the Wiener step is then 1D along that axis (wiener_1d semantics)
    BigAxis bigH{}, bigW{};
    std::vector<void *> owned;  // extra device tables
    int periodic = 0;
    // FFT tables (dtype copies; fp64 masters are temporaries)
    void *d_tw_n = nullptr, *d_tw_H = nullptr, *d_tw_W = nullptr;
    void *d_mult = nullptr;     // Wiener multiplier (lines: [n]; plane: [H][W] storage coords)
    void *d_mult_nat = nullptr; // lines: the same multiplier in natural frequency order
    bool wiener_reg = false;    // register four-step FFT kernel for the line Wiener step
    void *d_hspec = nullptr;    // PSF spectrum (PLANE_FFT iterations)
    // LUT
    double *d_lut64 = nullptr;
    float *d_lut32 = nullptr;
    float2 *d_lutp32 = nullptr;
    double2 *d_lutp64 = nullptr;
    LutView lut{};
    // scratch / staging
    DevBuf scratch, stage, partial;
    void *h_pin = nullptr;
    size_t h_pin_bytes = 0;
    int64_t chunk = 0;          // frames per internal chunk (0 = auto)
    cudaStream_t hstream[3] = {nullptr, nullptr, nullptr};
    cudaEvent_t ev_start = nullptr, ev_done[3] = {nullptr, nullptr, nullptr};
    int ensure_host_streams() {
        if (hstream[0]) return MD_OK;
        for (int s = 0; s < 3; ++s) {
            if (cudaStreamCreateWithFlags(&hstream[s], cudaStreamNonBlocking) != cudaSuccess ||
                cudaEventCreateWithFlags(&ev_done[s], cudaEventDisableTiming) != cudaSuccess)
                return fail(MD_ECUDA, "stream creation failed");
        }
        if (cudaEventCreateWithFlags(&ev_start, cudaEventDisableTiming) != cudaSuccess)
            return fail(MD_ECUDA, "event creation failed");
        return MD_OK;
    }
    int fused_clusters = 0;     // resident clusters of the fused-lines kernel (0 = unknown)
    int fused_geom[2] = {0, 0}; // its cluster size (CTAs) and CTAs per SM
    // concurrent use: host-side enqueue under a per-plan lock; a call on another stream than the
    // previous one waits (device side) for it, since both would use the plan's scratch
    std::recursive_mutex mu;
    int use_depth = 0;
    cudaEvent_t use_done = nullptr;
    cudaStream_t use_stream = nullptr;
    bool use_any = false;
    bool fused = false;         // whole-iteration-loop fused kernel applies
    bool fused_plane = false;   // cluster-resident 2D iteration loop (md_fused_plane.cu)
    bool fast_lines = false;    // register-window iteration kernel applies
    std::string describe;

    int64_t frame_elems() const { return (int64_t)d.height * d.width; }
    ~md_plan() {
        for (void *p : {(void *)d_taps_blur, (void *)d_taps_adj, (void *)d_ptaps_blur, (void *)d_ptaps_adj, d_tw_n,
                        d_tw_H, d_tw_W, d_mult, d_mult_nat, d_hspec, (void *)d_lut64, (void *)d_lut32,
                        (void *)d_lutp32, (void *)d_lutp64})
            if (p) cudaFree(p);
        for (void *p : owned) cudaFree(p);
        scratch.release();
        stage.release();
        partial.release();
        if (h_pin) cudaFreeHost(h_pin);
        for (int s = 0; s < 3; ++s) {
            if (hstream[s]) cudaStreamDestroy(hstream[s]);
            if (ev_done[s]) cudaEventDestroy(ev_done[s]);
        }
        if (ev_start) cudaEventDestroy(ev_start);
        if (use_done) cudaEventDestroy(use_done);
    }
};

namespace {

// divergence table (deconv.py:101-112, 137-139): values in both precisions plus (value, step)
// pairs for the float kernels' single-load interpolation
int build_lut(md_plan *P) {
    CU(cudaMalloc(&P->d_lut64, kLutCount * sizeof(double)));
    CU(cudaMalloc(&P->d_lut32, kLutCount * sizeof(float)));
    CU(cudaMalloc(&P->d_lutp32, (kLutCount - 1) * sizeof(float2)));
    CU(cudaMalloc(&P->d_lutp64, (kLutCount - 1) * sizeof(double2)));
    k_build_lut<<<(kLutCount + 255) / 256, 256>>>(P->d_lut64, P->d_lut32, P->d_lutp32, P->d_lutp64);
    CU(cudaGetLastError());
    CU(cudaDeviceSynchronize());
    P->lut.t64 = P->d_lut64;
    P->lut.t32 = P->d_lut32;
    P->lut.p32 = P->d_lutp32;
    P->lut.p64 = P->d_lutp64;
    return MD_OK;
}

template <typename X>
int upload(X **dst, const X *src, size_t count) {
    CU(cudaMalloc(dst, std::max<size_t>(count, 1) * sizeof(X)));
    if (count) CU(cudaMemcpy(*dst, src, count * sizeof(X), cudaMemcpyHostToDevice));
    return MD_OK;
}

int build_twiddles(int n, int dtype, void **out) {
    if (n < 2) { CU(cudaMalloc(out, 16)); return MD_OK; }
    double2 *t64 = nullptr;
    float2 *t32 = nullptr;
    CU(cudaMalloc(&t64, (n / 2) * sizeof(double2)));
    CU(cudaMalloc(&t32, (n / 2) * sizeof(float2)));
    k_build_twiddles<<<(n / 2 + 255) / 256, 256>>>(t64, t32, n);
    CU(cudaGetLastError());
    CU(cudaDeviceSynchronize());
    if (dtype == MD_F64) { cudaFree(t32); *out = t64; }
    else { cudaFree(t64); *out = t32; }
    return MD_OK;
}

int build_big_axis(int N, int dtype, BigAxis *ax, std::vector<void *> &owned) {
    ax->N = N;
    split_axis(N, &ax->N1, &ax->N2);
    ax->l1 = ilog2(ax->N1);
    ax->l2 = ilog2(ax->N2);
    void *a = nullptr, *b = nullptr, *c = nullptr;
    int rc = build_twiddles(N, dtype, &a);
    if (!rc) rc = build_twiddles(ax->N1, dtype, &b);
    if (!rc) rc = build_twiddles(ax->N2, dtype, &c);
    if (rc) return rc;
    owned.push_back(a); owned.push_back(b); owned.push_back(c);
    ax->twN = a; ax->twN1 = b; ax->twN2 = c;
    return MD_OK;
}

// spectrum of a real H x W array (natural layout) in storage coordinates, fp64;
// for H == 1 this is one row transform (1D spectra)
int spectrum_f64(const std::vector<double> &emb, int H, int W, double2 **out) {
    void *twH = nullptr, *twW = nullptr;
    int rc = build_twiddles(W, MD_F64, &twW);
    if (rc) return rc;
    rc = build_twiddles(H, MD_F64, &twH);
    if (rc) return rc;
    double *d_emb = nullptr;
    rc = upload(&d_emb, emb.data(), emb.size());
    if (rc) return rc;
    double2 *z = nullptr;
    CU(cudaMalloc(&z, (size_t)H * W * sizeof(double2)));
    Fft2Args a{};
    a.H = H; a.W = W; a.log2H = ilog2(H); a.log2W = ilog2(W);
    a.twH = twH; a.twW = twW;
    a.load = R_LOAD_REAL; a.ra = d_emb; a.z = z; a.epi = R_EPI_NONE; a.fwd_after = 1;
    CU(launch_fft2_rows<double>(a, 1, 0));
    if (H > 1) {
        a.filt = nullptr; a.col_inv = 0;
        CU(launch_fft2_cols<double>(a, 1, 0));
    }
    CU(cudaDeviceSynchronize());
    cudaFree(d_emb); cudaFree(twH); cudaFree(twW);
    *out = z;
    return MD_OK;
}

int make_filter(const double2 *h64, int64_t count, double K, int dtype, void **out) {
    void *o = nullptr;
    CU(cudaMalloc(&o, count * (dtype == MD_F64 ? sizeof(double2) : sizeof(float2))));
    k_make_filter<<<(int)std::min<int64_t>((count + 255) / 256, 4096), 256>>>(
        h64, count, K, dtype == MD_F64 ? (double2 *)o : nullptr, dtype == MD_F32 ? (float2 *)o : nullptr);
    CU(cudaGetLastError());
    CU(cudaDeviceSynchronize());
    *out = o;
    return MD_OK;
}

// PSF taps for the direct 2D path: blur reads u[y + cy - jy, x + cx - jx]; the adjoint
// (reflected kernel, core.py:204-220) reads u[y - cy + jy, x - cx + jx].
void plane_taps(const md_plan &P, bool adjoint, std::vector<PlaneTap> &taps, PlaneHalo &h) {
    const int sy = P.d.psf_rows, sx = P.d.psf_cols, cy = P.d.center_row, cx = P.d.center_col;
    taps.clear();
    int dymin = 0, dymax = 0, dxmin = 0, dxmax = 0;
    for (int i = 0; i < sy; ++i) {
        const int jy = adjoint ? sy - 1 - i : i;
        for (int jx0 = 0; jx0 < sx; ++jx0) {
            const int jx = adjoint ? sx - 1 - jx0 : jx0;
            const double w = P.w[(size_t)jy * sx + jx];
            if (w == 0.0) continue;
            PlaneTap t;
            t.dy = adjoint ? jy - cy : cy - jy;
            t.dx = adjoint ? jx - cx : cx - jx;
            t.w = w;
            taps.push_back(t);
            dymin = std::min(dymin, t.dy); dymax = std::max(dymax, t.dy);
            dxmin = std::min(dxmin, t.dx); dxmax = std::max(dxmax, t.dx);
        }
    }
    h.nt = (int)taps.size();
    h.ht = -dymin; h.hb = dymax; h.hl = -dxmin; h.hr = dxmax;
}

// 1D convolution descriptor for one direction (conv.py:141-173, deconv.py:310-326)
LineConv line_conv(const md_plan &P, bool adjoint, bool box, int periodic) {
    LineConv c{};
    const int T = P.d.psf_rows;
    const int center = adjoint ? T - 1 - P.d.center_row : P.d.center_row;
    c.periodic = periodic;
    c.ntaps = T;
    c.center = center;
    if (box) {
        const double L = P.d.box_length;
        const int whole = (int)std::floor(L);
        const bool frac = L != (double)whole;
        c.kind = LINE_BOX;
        c.wi = 1.0 / (frac ? L : (double)whole);
        // the 1/L factor: integer L multiplies by (1.0 / whole), fractional by (1.0 / length)
        if (frac) {
            c.lo = center - T + 2; c.hi = center - 1;
            c.ends = 1; c.elo = center - T + 1; c.ehi = center;
            c.we = (L - whole) / (2.0 * L);
        } else {
            c.lo = center - T + 1; c.hi = center;
        }
        c.ntaps = 0;   // no tap table needed
    } else {
        c.kind = LINE_TAPS;
    }
    return c;
}

int validate(const md_plan_desc *d) {
    if (d->height < 1 || d->width < 1) return fail(MD_EINVAL, "image must be a non-empty 2D grid");
    if (d->dtype != MD_F64 && d->dtype != MD_F32) return fail(MD_EINVAL, "dtype must be MD_F64 or MD_F32");
    if (d->psf_kind < 0 || d->psf_kind > 2) return fail(MD_EINVAL, "unknown PSF kind");
    if (d->psf_rows < 1 || d->psf_cols < 1 || !d->psf_weights) return fail(MD_EINVAL, "PSF weights missing");
    if (d->psf_kind != MD_PSF_GENERAL_2D && d->psf_cols != 1) return fail(MD_EINVAL, "1D PSF weights must be a vector");
    if (d->psf_kind != MD_PSF_GENERAL_2D && d->psf_axis != MD_AXIS_VERTICAL && d->psf_axis != MD_AXIS_HORIZONTAL)
        return fail(MD_EINVAL, "1D PSF kinds need a blur axis");
    if (!(d->wiener_k > 0.0)) return fail(MD_EINVAL, "wiener_k must be positive");
    if (d->alpha < 0.0) return fail(MD_EINVAL, "alpha must be non-negative");
    if (d->iterations < 0) return fail(MD_EINVAL, "iterations must be a non-negative integer");
    if (d->flags & MD_FLAG_RL) {
        // rl_deblur (deconv.py:524-534) clamps with any floor and has no robust / TV terms
        if (!std::isfinite(d->floor)) return fail(MD_EINVAL, "floor must be finite");
    } else if (!(d->eps_data > 0.0 && d->eps_reg > 0.0 && d->floor > 0.0)) {
        return fail(MD_EINVAL, "eps_data, eps_reg and floor must be positive");
    }
    if (d->conv < MD_CONV_BOX || d->conv > MD_CONV_FOURIER2D) return fail(MD_EINVAL, "unknown convolver mode");
    return MD_OK;
}

template <typename T> int lines_fused_clusters(md_plan &P);

}  // namespace

// RAII guard of an entry point that uses a plan's scratch (see md_plan::mu)
class PlanUse {
  public:
    PlanUse(md_plan *P, cudaStream_t st) : P_(P), st_(st), lk_(P->mu) {
        outer_ = P_->use_depth++ == 0;
        // under stream capture (the caller builds a CUDA graph) the launches are recorded, not
        // run: no cross-stream event edges -- replays are ordered by the stream they replay on
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        if (outer_) {
            if (cudaStreamIsCapturing(st_, &cs) != cudaSuccess) cudaGetLastError();
            else if (cs != cudaStreamCaptureStatusNone) outer_ = false, captured_ = tl_capturing = true;
        }
        if (outer_ && P_->use_any && P_->use_stream != st_) cudaStreamWaitEvent(st_, P_->use_done, 0);
    }
    ~PlanUse() {
        if (outer_) {
            if (P_->use_done || cudaEventCreateWithFlags(&P_->use_done, cudaEventDisableTiming) == cudaSuccess) {
                cudaEventRecord(P_->use_done, st_);
                P_->use_stream = st_;
                P_->use_any = true;
            }
        }
        if (captured_) tl_capturing = false;
        --P_->use_depth;
    }
    PlanUse(const PlanUse &) = delete;
    PlanUse &operator=(const PlanUse &) = delete;

  private:
    md_plan *P_;
    cudaStream_t st_;
    std::unique_lock<std::recursive_mutex> lk_;
    bool outer_ = false, captured_ = false;
};

// ======================================================================== C ABI
// error reporting for the C-ABI entries defined in other translation units (md_custom_lut.cu)
namespace md {
int set_error(int code, const char *msg) { return fail(code, msg); }
}  // namespace md

extern "C" {

int32_t md_abi_version(void) { return MDCUDA_ABI_VERSION; }
const char *md_last_error(void) { return g_err.c_str(); }

int32_t md_device_sm_count(void) {
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms;
}

int32_t md_plan_create(const md_plan_desc *desc, md_plan **out) {
    if (!desc || !out) return fail(MD_EINVAL, "null argument");
    *out = nullptr;
    int rc = validate(desc);
    if (rc) return rc;
    clear_stale_error();
    md_plan *P = new md_plan();
    P->d = *desc;
    P->w.assign(desc->psf_weights, desc->psf_weights + (size_t)desc->psf_rows * desc->psf_cols);
    P->d.psf_weights = nullptr;
    P->es = desc->dtype == MD_F64 ? 8 : 4;
    P->robust = !(desc->flags & MD_FLAG_RL);
    P->has_d = !(desc->flags & MD_FLAG_RL) && desc->alpha > 0.0;
    const int H = desc->height, W = desc->width;
    const bool wiener = desc->init == MD_INIT_WIENER;
    auto bail = [&](int code) { delete P; return code; };
    char buf[512];

    if (desc->psf_kind != MD_PSF_GENERAL_2D) {
        // ---------------------------------------------------------------- LINES
        P->path = PATH_LINES;
        P->vert = desc->psf_axis == MD_AXIS_VERTICAL;
        P->n = P->vert ? H : W;
        P->m = P->vert ? W : H;
        const int T = desc->psf_rows;
        if (T > P->n) return bail(fail(MD_EINVAL, "PSF support exceeds the image dimensions"));
        const bool isbox = desc->psf_kind == MD_PSF_BOX_1D;
        if (desc->conv == MD_CONV_BOX && !isbox) return bail(fail(MD_EINVAL, "box convolver requires a uniform-box PSF"));
        const int periodic = (desc->conv == MD_CONV_FOURIER || desc->conv == MD_CONV_FOURIER2D) ? 1 : 0;
        if (periodic) {
            const bool ok = desc->conv == MD_CONV_FOURIER ? is_pow2(P->n) : (is_pow2(H) && is_pow2(W));
            if (!ok) return bail(fail(MD_EINVAL, "transform length must be a power of two"));
        }
        if (wiener && !is_pow2(P->n)) return bail(fail(MD_EINVAL, "the blur axis must have power-of-two extent"));
        const bool use_box = isbox;   // box taps realised as a sliding window in every mode
        P->lblur = line_conv(*P, false, use_box, periodic);
        P->ladj = line_conv(*P, true, use_box, periodic);
        P->wrev.assign(P->w.rbegin(), P->w.rend());
        if (!use_box) {
            if ((rc = upload(&P->d_taps_blur, P->w.data(), P->w.size()))) return bail(rc);
            if ((rc = upload(&P->d_taps_adj, P->wrev.data(), P->wrev.size()))) return bail(rc);
        }
        P->fast_lines = !(desc->flags & MD_FLAG_GENERIC_LINES) &&
                        iter_fast_supported(desc->dtype, P->n, P->lblur, P->ladj);
        const size_t lim = desc->dtype == MD_F64 ? 4096 : 8192;
        const char *beyond = nullptr;
        if (wiener && (size_t)P->n > lim) beyond = "blur-axis length above the on-chip FFT limit";
        else if (desc->iterations > 0 && !P->fast_lines && !iter_lines_fits(desc->dtype, P->n, 2 * T))
            beyond = "blur-axis length above the on-chip line-iteration limit";
        else if (!conv_lines_fits(desc->dtype, P->n, 2 * T))
            beyond = "blur-axis length above the on-chip line-convolution limit";
        if (beyond) {
            // lines longer than one CTA holds: the same problem as a plane with a one-row (one-
            // column) PSF -- two-level FFT Wiener (its spectrum is constant across the lines) and
            // direct-tap iterations with the same boundary (box and spatial: edge-replicated;
            // Fourier 1D: periodic along the blur axis). Needs power-of-two sides for the Wiener.
            delete P;
            md_plan_desc d2 = *desc;
            d2.psf_kind = MD_PSF_GENERAL_2D;
            d2.psf_axis = MD_AXIS_NONE;
            const bool vert = desc->psf_axis == MD_AXIS_VERTICAL;
            d2.psf_rows = vert ? T : 1;
            d2.psf_cols = vert ? 1 : T;
            d2.center_row = vert ? desc->center_row : 0;
            d2.center_col = vert ? 0 : desc->center_row;
            d2.box_length = 0.0;
            d2.conv = desc->conv == MD_CONV_FOURIER ? MD_CONV_FOURIER2D
                                                    : (desc->conv == MD_CONV_BOX ? MD_CONV_SPATIAL : desc->conv);
            d2.flags &= ~MD_FLAG_FORCE_FFT2D;
            d2.flags |= kFlagLinePlane;
            if (md_plan_create(&d2, out) != MD_OK) return fail(MD_EINVAL, beyond);
            (*out)->describe = std::string("1D PSF beyond the on-chip line limits as a plane; ") + (*out)->describe;
            return MD_OK;
        }
        if (is_pow2(P->n)) P->log2n = ilog2(P->n);
        if (is_pow2(P->n) && (size_t)P->n <= lim) {      // line FFT tables (Wiener step)
            if ((rc = build_twiddles(P->n, desc->dtype, &P->d_tw_n))) return bail(rc);
            std::vector<double> emb(P->n, 0.0);       // fft.py:192-201
            for (int j = 0; j < T; ++j) emb[((j - desc->center_row) % P->n + P->n) % P->n] = P->w[j];
            double2 *h64 = nullptr;
            if ((rc = spectrum_f64(emb, 1, P->n, &h64))) return bail(rc);
            rc = make_filter(h64, P->n, desc->wiener_k, desc->dtype, &P->d_mult);
            cudaFree(h64);
            if (rc) return bail(rc);
            const int ces = desc->dtype == MD_F64 ? 16 : 8;
            CU(cudaMalloc(&P->d_mult_nat, (size_t)P->n * ces));
            if (P->n > 1) {
                k_unbitrev<<<(P->n + 255) / 256, 256>>>((const unsigned char *)P->d_mult, (unsigned char *)P->d_mult_nat,
                                                        P->n, P->log2n, ces);
            } else {
                CU(cudaMemcpy(P->d_mult_nat, P->d_mult, ces, cudaMemcpyDeviceToDevice));
            }
            CU(cudaGetLastError());
            CU(cudaDeviceSynchronize());
            P->wiener_reg = !(desc->flags & MD_FLAG_GENERIC_LINES) && wiener_reg_supported(desc->dtype, P->n);
        }
        // default: the cluster kernel -- float, and float64 for line radii <= 16 (the
        // shuffle-window / st.async-halo kernel, md_fused64_kernel.cuh); wider float64 kernels
        // keep the per-iteration kernel, opt-in via md_plan_set_fused
        const int lrad = std::max(line_radius(P->lblur), line_radius(P->ladj));
        P->fused = (desc->dtype == MD_F32 || lrad <= 16) && P->fast_lines &&
                   fused_lines_supported(desc->dtype, P->n, P->m, desc->flags, lrad);
        if (P->fused)
            P->fused_clusters = desc->dtype == MD_F32 ? lines_fused_clusters<float>(*P) : lines_fused_clusters<double>(*P);
        snprintf(buf, sizeof buf, "lines: n=%d m=%d %s %s %s, %s", P->n, P->m, P->vert ? "vertical" : "horizontal",
                 use_box ? "box" : "taps", periodic ? "periodic" : "clamped",
                 P->fused ? "fused cluster iteration kernel"
                          : (P->fast_lines ? "k_wiener_lines + k_iter_lines_fast per iteration"
                                           : "k_wiener_lines + k_iter_lines per iteration"));
    } else {
        // ---------------------------------------------------------------- PLANE
        if (desc->psf_rows > H || desc->psf_cols > W) return bail(fail(MD_EINVAL, "PSF support exceeds the image dimensions"));
        if (desc->conv == MD_CONV_BOX) return bail(fail(MD_EINVAL, "box convolver requires a uniform-box PSF"));
        if (!(desc->center_row >= 0 && desc->center_row < desc->psf_rows && desc->center_col >= 0 &&
              desc->center_col < desc->psf_cols))
            return bail(fail(MD_EINVAL, "PSF center must lie inside the support"));
        P->periodic = desc->conv != MD_CONV_SPATIAL;
        // a 1D PSF past the line kernels' limits (kFlagLinePlane): only its blur axis is
        // transformed (wiener_1d, deconv.py:275-288; fft.py:63-66 constrains that axis alone)
        if ((desc->flags & kFlagLinePlane) && (desc->psf_rows == 1) != (desc->psf_cols == 1))
            P->line_axis = desc->psf_rows == 1 ? 1 : 0;
        const bool pow2 = P->line_axis >= 0 ? is_pow2(P->line_axis == 1 ? W : H) : (is_pow2(H) && is_pow2(W));
        if ((P->periodic || wiener) && !pow2)
            return bail(fail(MD_EINVAL, P->line_axis >= 0 ? "the blur axis must have power-of-two extent"
                                                          : "2D Fourier convolution needs power-of-two dimensions"));
        std::vector<PlaneTap> tb, ta;
        plane_taps(*P, false, tb, P->hblur);
        plane_taps(*P, true, ta, P->hadj);
        const int maxh = std::max(std::max(P->hadj.ht, P->hadj.hb), std::max(P->hadj.hl, P->hadj.hr));
        const bool direct_ok = maxh <= 40;
        const int lim = desc->dtype == MD_F64 ? 4096 : 8192;
        P->big = pow2 && (P->line_axis >= 0 || std::max(H, W) > lim || (desc->flags & MD_FLAG_BIG_FFT)) &&
                 (P->periodic || wiener);
        bool use_fft = P->periodic && ((desc->flags & MD_FLAG_FORCE_FFT2D) || P->hblur.nt > 96 || !direct_ok);
        if (!P->periodic && !direct_ok) return bail(fail(MD_EINVAL, "PSF too large for the direct clamped path"));
        if (P->big && use_fft) {
            if (!direct_ok || P->hblur.nt > kPlaneMaxTaps)
                return bail(fail(MD_EINVAL, "image side above the on-chip 2D FFT limit for a dense PSF"));
            use_fft = false;    // large images iterate with direct taps; only the Wiener step needs FFTs
        }
        if (P->line_axis >= 0 ? (std::max(H, W) > (1 << 20) || (int64_t)H * W >= (1ll << 31))
                              : std::max(H, W) > 65536)
            return bail(fail(MD_EINVAL, "transform length above the two-level FFT limit"));
        P->path = use_fft ? PATH_PLANE_FFT : PATH_PLANE_DIRECT;
        if ((rc = upload(&P->d_ptaps_blur, tb.data(), tb.size()))) return bail(rc);
        if ((rc = upload(&P->d_ptaps_adj, ta.data(), ta.size()))) return bail(rc);
        P->htaps_blur = tb;
        P->htaps_adj = ta;
        P->fast_plane = !(desc->flags & MD_FLAG_GENERIC_LINES) && plane_fast_supported(P->hblur, P->hadj, tb, ta, desc->dtype);
        if (pow2 && P->big && P->line_axis >= 0) {
            // the 1D spectrum along the blur axis in the two-level storage order, its Wiener
            // multiplier replicated over the other axis (so the passes' filter index is the
            // frame address, as for 2D)
            const int ax = P->line_axis, N = ax == 1 ? W : H;
            BigAxis n64{};
            std::vector<void *> tmp;
            if ((rc = build_big_axis(N, MD_F64, &n64, tmp)) ||
                (rc = build_big_axis(N, desc->dtype, ax == 1 ? &P->bigW : &P->bigH, P->owned)))
                return bail(rc);
            double *emb = nullptr;
            double2 *h64 = nullptr;
            CU(cudaMalloc(&emb, (size_t)N * sizeof(double)));
            CU(cudaMalloc(&h64, (size_t)N * sizeof(double2)));
            CU(cudaMemset(emb, 0, (size_t)N * sizeof(double)));
            k_embed_taps<<<(tb.size() + 255) / 256, 256>>>(emb, ax == 1 ? 1 : N, ax == 1 ? N : 1, P->d_ptaps_blur,
                                                         (int)tb.size());
            CU(cudaGetLastError());
            CU(big_axis<double>(n64, h64, ax == 1 ? 1 : N, ax == 1 ? N : 1, ax, 0, emb, nullptr, nullptr, 0, 1.0, 1, 0));
            CU(cudaDeviceSynchronize());
            cudaFree(emb);
            for (void *p : tmp) cudaFree(p);
            void *m1 = nullptr;
            rc = make_filter(h64, N, desc->wiener_k, desc->dtype, &m1);
            cudaFree(h64);
            if (rc) return bail(rc);
            const int ces = desc->dtype == MD_F64 ? 16 : 8;
            CU(cudaMalloc(&P->d_mult, (size_t)H * W * ces));
            k_replicate_filter<<<1024, 256>>>((const unsigned char *)m1, (unsigned char *)P->d_mult, H, W, ax, ces);
            CU(cudaGetLastError());
            CU(cudaDeviceSynchronize());
            cudaFree(m1);
        } else if (pow2 && P->big) {
            BigAxis h64{}, w64{};
            std::vector<void *> tmp;
            if ((rc = build_big_axis(H, MD_F64, &h64, tmp)) || (rc = build_big_axis(W, MD_F64, &w64, tmp)) ||
                (rc = build_big_axis(H, desc->dtype, &P->bigH, P->owned)) ||
                (rc = build_big_axis(W, desc->dtype, &P->bigW, P->owned)))
                return bail(rc);
            double *emb = nullptr;
            double2 *h64s = nullptr;
            CU(cudaMalloc(&emb, (size_t)H * W * sizeof(double)));
            CU(cudaMalloc(&h64s, (size_t)H * W * sizeof(double2)));
            CU(cudaMemset(emb, 0, (size_t)H * W * sizeof(double)));
            k_embed_taps<<<(tb.size() + 255) / 256, 256>>>(emb, H, W, P->d_ptaps_blur, (int)tb.size());
            CU(cudaGetLastError());
            CU(big_axis<double>(w64, h64s, H, W, 1, 0, emb, nullptr, nullptr, 0, 1.0, 1, 0));
            CU(big_axis<double>(h64, h64s, H, W, 0, 0, nullptr, nullptr, nullptr, 0, 1.0, 1, 0));
            CU(cudaDeviceSynchronize());
            cudaFree(emb);
            for (void *p : tmp) cudaFree(p);
            rc = make_filter(h64s, (int64_t)H * W, desc->wiener_k, desc->dtype, &P->d_mult);
            cudaFree(h64s);
            if (rc) return bail(rc);
        } else if (pow2 && (P->periodic || wiener)) {
            if ((rc = build_twiddles(H, desc->dtype, &P->d_tw_H))) return bail(rc);
            if ((rc = build_twiddles(W, desc->dtype, &P->d_tw_W))) return bail(rc);
            std::vector<double> emb((size_t)H * W, 0.0);       // fft.py:204-221
            for (int jy = 0; jy < desc->psf_rows; ++jy)
                for (int jx = 0; jx < desc->psf_cols; ++jx) {
                    const int y = ((jy - desc->center_row) % H + H) % H;
                    const int x = ((jx - desc->center_col) % W + W) % W;
                    emb[(size_t)y * W + x] = P->w[(size_t)jy * desc->psf_cols + jx];
                }
            double2 *h64 = nullptr;
            if ((rc = spectrum_f64(emb, H, W, &h64))) return bail(rc);
            rc = make_filter(h64, (int64_t)H * W, desc->wiener_k, desc->dtype, &P->d_mult);
            if (!rc && use_fft) rc = make_filter(h64, (int64_t)H * W, -1.0, desc->dtype, &P->d_hspec);
            cudaFree(h64);
            if (rc) return bail(rc);
        }
        // float: small frames run the whole iteration loop on one cluster (measured faster)
        P->fused_plane = desc->dtype == MD_F32 && P->path == PATH_PLANE_DIRECT && !P->big && P->fast_plane &&
                         !(desc->flags & MD_FLAG_NO_FUSED) &&
                         fused_plane_supported(H, W, P->hblur, P->hadj, tb, ta, desc->dtype);
        snprintf(buf, sizeof buf, "plane: %dx%d %s, %d taps (halo %d/%d/%d/%d), %s", H, W,
                 P->periodic ? "periodic" : "clamped", P->hblur.nt, P->hblur.ht, P->hblur.hb, P->hblur.hl,
                 P->hblur.hr, use_fft ? "2D FFT convolver (4 launches/iteration)"
                                      : (P->big ? "two-level FFT Wiener, direct taps (2 launches/iteration)"
                                                : (P->fused_plane ? "direct taps, fused cluster iteration kernel"
                                                                  : "direct taps (2 launches/iteration)")));
    }
    P->describe = buf;
    // divergence table (deconv.py:101-112, 137-139)
    if ((rc = build_lut(P))) return bail(rc);
    *out = P;
    return MD_OK;
}

int32_t md_plan_destroy(md_plan *plan) {
    delete plan;
    return MD_OK;
}

const char *md_plan_describe(const md_plan *plan) { return plan ? plan->describe.c_str() : ""; }

}  // extern "C"

// ======================================================================== execution
namespace {

// scratch fields per frame (in elements of the plan dtype)
constexpr int64_t kChunkScratch = 4ll << 30;

// per-plan scratch bound: 4 GiB, or a sixteenth of the device memory on smaller GPUs (plans are
// cached by the Python layer, several may hold scratch at once)
int64_t chunk_scratch_cap() {
    static int64_t cap = [] {
        size_t fr = 0, total = 0;
        if (cudaMemGetInfo(&fr, &total) != cudaSuccess) { cudaGetLastError(); return kChunkScratch; }
        return std::max<int64_t>(256ll << 20, std::min<int64_t>(kChunkScratch, (int64_t)(total / 16)));
    }();
    return cap;
}

bool lines_pipelined(const md_plan &P) {
    return P.path == PATH_LINES && P.fused && P.wiener_reg && P.d.init == MD_INIT_WIENER && P.d.iterations > 0;
}

int scratch_fields(const md_plan &P) {
    switch (P.path) {
        case PATH_LINES: return lines_pipelined(P) ? 4 : 3;   // (fpos, A) x 2 sets | fpos, A, B
        case PATH_PLANE_DIRECT: return 5;   // fpos, A, B, p, W
        default: return 5;                  // fpos, A, B, z (complex = 2)
    }
}

int64_t auto_chunk(const md_plan &P, int64_t batch) {
    if (P.chunk > 0) return std::min(P.chunk, batch);
    // keep one chunk's scratch within chunk_scratch_cap(): large chunks, because every launch ends on a
    // partial wave of clusters (measured: 4096 c1 frames as one chunk 8.21 ms, as four pipelined
    // chunks 8.30 ms)
    const int64_t per = (int64_t)scratch_fields(P) * P.frame_elems() * P.es;
    int64_t c = std::max<int64_t>(1, chunk_scratch_cap() / std::max<int64_t>(per, 1));
    if (lines_pipelined(P) && P.fused_clusters > 0 && batch > c) {
        // whole rounds of the resident clusters per chunk, the rounds spread evenly over the
        // chunks: no chunk ends on a nearly empty round
        const int64_t R = P.fused_clusters;
        const int64_t rounds = (batch + R - 1) / R, chunks = (batch + c - 1) / c;
        c = std::max<int64_t>(R, (rounds + chunks - 1) / chunks * R);
    }
    return std::min(c, batch);
}

template <typename T>
FusedLinesArgs fused_args(md_plan &P, const void *A, const void *FP, void *u, bool raw_f = false) {
    FusedLinesArgs fa{};
    fa.u_in = A; fa.fpos = FP; fa.u_out = u; fa.n = P.n; fa.m = P.m; fa.iterations = P.d.iterations;
    fa.floor_f = raw_f ? 1 : 0; fa.floor = P.d.floor;
    fa.out_vert = P.vert; fa.blur = P.lblur; fa.adj = P.ladj;
    fa.taps_blur_host = P.w.data(); fa.taps_adj_host = P.wrev.data();
    fa.alpha = P.d.alpha; fa.eps_d2 = P.d.eps_data * P.d.eps_data; fa.eps_r2 = P.d.eps_reg * P.d.eps_reg;
    fa.has_d = P.has_d; fa.robust = P.robust; fa.lut = P.lut;
    return fa;
}

// 2D-FFT convolver iterations: the TV divergence from k_diffusion (MD_FFT2_DPRE=0: evaluated in
// the update pass, five diffusivities per pixel -- for A/B runs)
inline bool fft2_dpre() {
    static const bool on = [] { const char *v = std::getenv("MD_FFT2_DPRE"); return !v || std::atoi(v) != 0; }();
    return on;
}

// float64 cluster kernel on horizontal lines: it floors the raw observation itself (the input is
// already line-major), so the Wiener step writes no fpos field -- one field pass fewer per frame
// (MD_F64_RAW_F=0: the fpos field as before, for A/B runs)
template <typename T>
bool lines_raw_f(const md_plan &P) {
    static const bool on = [] { const char *v = std::getenv("MD_F64_RAW_F"); return !v || std::atoi(v) != 0; }();
    return on && sizeof(T) == 8 && !P.vert && P.d.init == MD_INIT_WIENER &&
           std::max(line_radius(P.lblur), line_radius(P.ladj)) <= 16;
}

// the whole RRRL loop of nb frames: one launch of the cluster kernel
template <typename T>
int lines_fused_launch(md_plan &P, const void *A, const void *FP, void *u, int64_t nb, cudaStream_t st,
                       bool raw_f = false) {
    FusedLinesArgs fa = fused_args<T>(P, A, FP, u, raw_f);
    CU(launch_fused_lines<T>(fa, nb, st));
    return MD_OK;
}

// resident cluster count of the plan's fused kernel (0 when it cannot be determined)
template <typename T>
int lines_fused_clusters(md_plan &P) {
    int n = 0;
    FusedLinesArgs fa = fused_args<T>(P, nullptr, nullptr, nullptr);
    fa.query = &n;
    fa.query_geom = P.fused_geom;
    return launch_fused_lines<T>(fa, 1, nullptr) == cudaSuccess ? n : 0;
}

// Wiener step of nb frames along lines (clamped), result `out` (line-major unless out_vert),
// optionally fpos = max(f, floor) line-major
template <typename T>
int lines_wiener(md_plan &P, const void *f, void *out, int out_vert, void *fpos, int64_t nb, cudaStream_t st,
                 bool pdl = false) {
    WienerLinesArgs a{};
    a.pdl = pdl ? 1 : 0;
    a.in = f; a.n = P.n; a.log2n = P.log2n; a.m = P.m; a.in_vert = P.vert;
    a.mult = P.d_mult; a.tw = P.d_tw_n; a.floor = P.d.floor; a.clamp = 1;
    a.out = out; a.out_vert = out_vert; a.fpos = fpos;
    if (P.wiener_reg) {
        a.mult = P.d_mult_nat;
        CU(launch_wiener_reg<T>(a, nb, st));
    } else {
        CU(launch_wiener_lines<T>(a, nb, st));
    }
    return MD_OK;
}

// chunks of the fused-lines path, pipelined on one stream: the Wiener step of chunk c+1 is a
// programmatic dependent launch of chunk c's cluster iteration kernel, so it starts once that
// grid's last wave is resident and runs on the SMs the wave leaves free; its last block waits for
// the iteration kernel, so the next iteration kernel (a plain launch) starts after both. Scratch
// holds two (fpos, u0) sets.
template <typename T>
int run_lines_pipelined(md_plan &P, const void *f, void *u, int64_t batch, cudaStream_t st) {
    const int64_t chunk = auto_chunk(P, batch);
    const int64_t fe = P.frame_elems(), fb = fe * (int64_t)sizeof(T) * chunk;
    int rc = P.scratch.ensure((size_t)4 * fb);
    if (rc) return rc;
    char *scr = (char *)P.scratch.p;
    void *FP[2] = {scr, scr + 2 * fb}, *A[2] = {scr + fb, scr + 3 * fb};
    auto fin = [&](int64_t c) { return static_cast<const char *>(f) + c * chunk * fe * (int64_t)sizeof(T); };
    auto uout = [&](int64_t c) { return static_cast<char *>(u) + c * chunk * fe * (int64_t)sizeof(T); };
    const int64_t C = (batch + chunk - 1) / chunk;
    auto nbof = [&](int64_t c) { return std::min(chunk, batch - c * chunk); };
    const bool raw = lines_raw_f<T>(P);
    rc = lines_wiener<T>(P, fin(0), A[0], 0, raw ? nullptr : FP[0], nbof(0), st, false);
    if (rc) return rc;
    prof_mark(st, PK_INIT);
    for (int64_t c = 0; c < C; ++c) {
        const int s = (int)(c & 1);
        rc = lines_fused_launch<T>(P, A[s], raw ? fin(c) : FP[s], uout(c), nbof(c), st, raw);
        if (rc) return rc;
        if (c + 1 < C) {
            rc = lines_wiener<T>(P, fin(c + 1), A[s ^ 1], 0, raw ? nullptr : FP[s ^ 1], nbof(c + 1), st, true);
            if (rc) return rc;
        }
    }
    prof_mark(st, PK_ITER);     // one mark: events between the launches would serialise them
    return MD_OK;
}

template <typename T>
int run_lines(md_plan &P, const void *f, void *u, int64_t nb, char *scr, cudaStream_t st) {
    const int64_t fb = P.frame_elems() * (int64_t)sizeof(T) * nb;
    void *FP = scr, *A = scr + fb, *B = scr + 2 * fb;
    const int K = P.d.iterations;
    const bool wiener = P.d.init == MD_INIT_WIENER;
    const bool raw = P.fused && lines_raw_f<T>(P);
    if (wiener) {
        const int rc = K == 0 ? lines_wiener<T>(P, f, u, P.vert, nullptr, nb, st)
                              : lines_wiener<T>(P, f, A, 0, raw ? nullptr : FP, nb, st);
        if (rc) return rc;
        prof_mark(st, PK_INIT);
        if (K == 0) return MD_OK;
    } else {
        if (K == 0) { CU(launch_clamp2<T>(f, u, nullptr, P.frame_elems() * nb, P.d.floor, st)); return MD_OK; }
        if (P.vert) {
            // native [n rows][m cols] -> line-major [m][n]
            CU(launch_transpose<T>(f, A, FP, P.n, P.m, P.d.floor, 1, nb, st));
        } else {
            CU(launch_clamp2<T>(f, A, FP, P.frame_elems() * nb, P.d.floor, st));
        }
        prof_mark(st, PK_INIT);
    }
    if (P.fused) {
        const int rc = lines_fused_launch<T>(P, A, raw ? f : FP, u, nb, st, raw);
        if (rc) return rc;
        prof_mark(st, PK_ITER);
        return MD_OK;
    }
    if (P.fast_lines) {
        IterFastDesc fd{};
        fd.fpos = FP; fd.n = P.n; fd.m = P.m; fd.blur = P.lblur; fd.adj = P.ladj;
        fd.taps_blur_host = P.w.data(); fd.taps_adj_host = P.wrev.data();
        fd.alpha = P.d.alpha; fd.eps_d2 = P.d.eps_data * P.d.eps_data; fd.eps_r2 = P.d.eps_reg * P.d.eps_reg;
        fd.has_d = P.has_d; fd.lut = P.lut;
        void *cur = A;
        for (int k = 0; k < K; ++k) {
            const bool last = k == K - 1;
            void *dst = (last && !P.vert) ? u : (cur == A ? B : A);
            fd.u_in = cur; fd.u_out = dst;
            CU(launch_iter_fast<T>(fd, P.robust, nb, st));
            prof_mark(st, PK_ITER);
            cur = dst;
        }
        if (P.vert) {
            CU(launch_transpose<T>(cur, u, nullptr, P.m, P.n, 0.0, 0, nb, st));
            prof_mark(st, PK_LAYOUT);
        }
        return MD_OK;
    }
    IterLinesArgs it{};
    it.n = P.n; it.m = P.m; it.blur = P.lblur; it.adj = P.ladj;
    it.taps_blur = P.d_taps_blur; it.taps_adj = P.d_taps_adj;
    it.alpha = P.d.alpha; it.eps_d2 = P.d.eps_data * P.d.eps_data; it.eps_r2 = P.d.eps_reg * P.d.eps_reg;
    it.has_d = P.has_d; it.lut = P.lut; it.fpos = FP;
    void *cur = A;
    for (int k = 0; k < K; ++k) {
        const bool last = k == K - 1;
        void *dst = (last && !P.vert) ? u : (cur == A ? B : A);
        it.u_in = cur; it.u_out = dst;
        CU(launch_iter_lines<T>(it, P.robust, nb, st));
        prof_mark(st, PK_ITER);
        cur = dst;
    }
    if (P.vert) {
        CU(launch_transpose<T>(cur, u, nullptr, P.m, P.n, 0.0, 0, nb, st));
        prof_mark(st, PK_LAYOUT);
    }
    return MD_OK;
}

template <typename T>
Fft2Args fft2_base(const md_plan &P) {
    Fft2Args a{};
    a.H = P.d.height; a.W = P.d.width; a.log2H = ilog2(a.H); a.log2W = ilog2(a.W);
    a.twH = P.d_tw_H; a.twW = P.d_tw_W;
    a.lut = P.lut;
    a.eps_d2 = P.d.eps_data * P.d.eps_data; a.eps_r2 = P.d.eps_reg * P.d.eps_reg;
    a.alpha = P.d.alpha; a.has_d = P.has_d; a.robust = P.robust;
    a.scale = 1.0 / ((double)a.H * (double)a.W);
    return a;
}

// Wiener 2D: rows fwd -> cols (x M, inv) -> rows inv + epilogue; optionally leaves the
// row-transformed clamped result in z for the first FFT-path iteration
template <typename T>
int wiener_plane(md_plan &P, const void *f, void *out, void *fpos, void *z, bool clamp, bool fwd_after,
                 int64_t nb, cudaStream_t st) {
    if (P.big && P.line_axis >= 0) {
        // 1D along the blur axis: forward (real input) x M in the last pass, inverse whose last
        // pass writes u0 / fpos -- 4 sub-transform passes
        const int H = P.d.height, W = P.d.width, ax = P.line_axis;
        const BigAxis &A = ax == 1 ? P.bigW : P.bigH;
        CU(big_axis<T>(A, z, H, W, ax, 0, f, nullptr, P.d_mult, 0, 1.0, nb, st));
        CU(big_axis_inv_wiener<T>(A, z, H, W, ax, 1.0 / (ax == 1 ? W : H), f, out, fpos, P.d.floor, clamp ? 1 : 0, nb,
                                  st));
        return MD_OK;
    }
    if (P.big) {
        const int H = P.d.height, W = P.d.width;
        // rows forward (real input) | columns: forward, x M and inverse of the inner digit fused
        // | rows inverse whose last pass writes u0 and fpos: 6 passes over the complex field
        CU(big_axis<T>(P.bigW, z, H, W, 1, 0, f, nullptr, nullptr, 0, 1.0, nb, st));
        CU(big_axis_filter<T>(P.bigH, z, H, W, 0, P.d_mult, 0, nb, st));
        CU(big_axis_inv_wiener<T>(P.bigW, z, H, W, 1, 1.0 / ((double)H * W), f, out, fpos, P.d.floor, clamp ? 1 : 0,
                                  nb, st));
        return MD_OK;
    }
    // two frames per complex field unless the FFT-path iteration needs z afterwards
    Fft2Args a = fft2_base<T>(P);
    a.pairs = fwd_after ? 0 : 1;
    a.nreal = nb;
    const int64_t nz = a.pairs ? (nb + 1) / 2 : nb;
    a.load = R_LOAD_REAL; a.ra = f; a.rb = nullptr; a.z = z; a.epi = R_EPI_NONE; a.fwd_after = 1;
    CU(launch_fft2_rows<T>(a, nz, st));
    a.filt = P.d_mult; a.conj_filt = 0; a.col_inv = 1;
    CU(launch_fft2_cols<T>(a, nz, st));
    a.load = R_LOAD_COMPLEX; a.inv = 1; a.epi = R_EPI_WIENER; a.fwd_after = fwd_after;
    a.oa = out; a.ob = fpos; a.f = f; a.floor = clamp ? P.d.floor : 0.0;
    CU(launch_fft2_rows<T>(a, nz, st));
    return MD_OK;
}

template <typename T>
int run_plane(md_plan &P, const void *f, void *u, int64_t nb, char *scr, cudaStream_t st) {
    const int64_t fb = P.frame_elems() * (int64_t)sizeof(T) * nb;
    void *FP = scr, *A = scr + fb, *B = scr + 2 * fb, *X = scr + 3 * fb, *Y = scr + 4 * fb;
    const int K = P.d.iterations;
    const bool wiener = P.d.init == MD_INIT_WIENER;
    const bool fftp = P.path == PATH_PLANE_FFT;
    void *z = X;   // complex field spans X and Y
    if (wiener) {
        int rc = wiener_plane<T>(P, f, K == 0 ? u : A, K == 0 ? nullptr : FP, z, true, fftp && K > 0, nb, st);
        prof_mark(st, PK_INIT);
        if (rc || K == 0) return rc;
    } else {
        if (K == 0) { CU(launch_clamp2<T>(f, u, nullptr, P.frame_elems() * nb, P.d.floor, st)); return MD_OK; }
        CU(launch_clamp2<T>(f, A, FP, P.frame_elems() * nb, P.d.floor, st));
        if (fftp) {
            Fft2Args a = fft2_base<T>(P);
            a.load = R_LOAD_REAL; a.ra = A; a.z = z; a.epi = R_EPI_NONE; a.fwd_after = 1;
            CU(launch_fft2_rows<T>(a, nb, st));
        }
        prof_mark(st, PK_INIT);
    }
    if (P.fused_plane) {
        FusedPlaneDesc fd{};
        fd.u0 = A; fd.fpos = FP; fd.u_out = u;
        fd.H = P.d.height; fd.W = P.d.width; fd.periodic = P.periodic; fd.iterations = K;
        fd.hb = P.hblur; fd.ha = P.hadj; fd.taps_blur = &P.htaps_blur; fd.taps_adj = &P.htaps_adj;
        fd.alpha = P.d.alpha; fd.eps_d2 = P.d.eps_data * P.d.eps_data; fd.eps_r2 = P.d.eps_reg * P.d.eps_reg;
        fd.has_d = P.has_d; fd.robust = P.robust; fd.lut = P.lut;
        CU(launch_fused_plane<T>(fd, nb, st));
        prof_mark(st, PK_ITER);
        return MD_OK;
    }
    void *cur = A;
    for (int k = 0; k < K; ++k) {
        const bool last = k == K - 1;
        void *dst = last ? u : (cur == A ? B : A);
        if (fftp) {
            Fft2Args a = fft2_base<T>(P);
            a.z = z;
            a.filt = P.d_hspec; a.conj_filt = 0; a.col_inv = 1;
            CU(launch_fft2_cols<T>(a, nb, st));                       // blur: x h
            a.load = R_LOAD_COMPLEX; a.inv = 1; a.epi = R_EPI_STAGE_A; a.f = FP; a.fwd_after = 1;
            CU(launch_fft2_rows<T>(a, nb, st));                       // b -> (p + iW), fwd
            a.conj_filt = 1;
            CU(launch_fft2_cols<T>(a, nb, st));                       // adjoint pair: x conj(h)
            a.epi = R_EPI_STAGE_B; a.u = cur; a.oa = dst; a.fwd_after = !last;
            if (P.has_d && fft2_dpre()) {
                // the TV divergence of u in one tiled pass, into dst: the update pass reads each
                // pixel's d before it writes u' there (same thread, same position)
                CU(launch_diffusion<T>(cur, dst, nb, P.d.height, P.d.width, P.d.eps_reg * P.d.eps_reg, st));
                a.dpre = dst;
            }
            CU(launch_fft2_rows<T>(a, nb, st));                       // update, fwd of u'
        } else if (P.fast_plane) {
            PlaneFastDesc s{};
            s.u = cur; s.f = FP; s.p = X; s.w = Y; s.u_out = dst;
            s.pw_pairs = 1;                                           // (p, W) pairs over X and Y
            s.H = P.d.height; s.W = P.d.width; s.periodic = P.periodic;
            s.hb = P.hblur; s.ha = P.hadj; s.taps_blur = &P.htaps_blur; s.taps_adj = &P.htaps_adj;
            s.alpha = P.d.alpha; s.eps_d2 = P.d.eps_data * P.d.eps_data; s.eps_r2 = P.d.eps_reg * P.d.eps_reg;
            s.has_d = P.has_d; s.lut = P.lut;
            CU(launch_plane_fast<T>(s, P.robust, nb, st));
        } else {
            StagePlaneArgs s{};
            s.u = cur; s.f = FP; s.p = X; s.w = Y; s.u_out = dst;
            s.H = P.d.height; s.W = P.d.width; s.periodic = P.periodic;
            s.blur = P.hblur; s.adj = P.hadj; s.blur_taps = P.d_ptaps_blur; s.adj_taps = P.d_ptaps_adj;
            s.alpha = P.d.alpha; s.eps_d2 = P.d.eps_data * P.d.eps_data; s.eps_r2 = P.d.eps_reg * P.d.eps_reg;
            s.floor = P.d.floor; s.has_d = P.has_d; s.floor_f = 0; s.general_weight = 0; s.lut = P.lut;
            CU(launch_stage_plane<T>(s, P.robust, nb, st));
        }
        prof_mark(st, PK_ITER);
        cur = dst;
    }
    return MD_OK;
}

template <typename T>
int run_chunk(md_plan &P, const void *f, void *u, int64_t nb, char *scr, cudaStream_t st) {
    return P.path == PATH_LINES ? run_lines<T>(P, f, u, nb, scr, st) : run_plane<T>(P, f, u, nb, scr, st);
}

constexpr int kHostStreams = 3;
inline size_t align_up(size_t b) { return (b + 255) & ~(size_t)255; }
inline int io_bytes(int t) { return t == MD_IO_F64 ? 8 : (t == MD_IO_F32 ? 4 : 1); }

template <typename T>
int run_typed(md_plan &P, const void *f, void *u, int64_t batch, cudaStream_t st) {
    if (lines_pipelined(P) && batch > auto_chunk(P, batch)) return run_lines_pipelined<T>(P, f, u, batch, st);
    const int64_t chunk = auto_chunk(P, batch);
    const size_t need = (size_t)scratch_fields(P) * P.frame_elems() * sizeof(T) * chunk;
    int rc = P.scratch.ensure(need);
    if (rc) return rc;
    const int64_t fbytes = P.frame_elems() * (int64_t)sizeof(T);
    for (int64_t b0 = 0; b0 < batch; b0 += chunk) {
        const int64_t nb = std::min(chunk, batch - b0);
        const void *fc = static_cast<const char *>(f) + b0 * fbytes;
        void *uc = static_cast<char *>(u) + b0 * fbytes;
        rc = P.path == PATH_LINES ? run_lines<T>(P, fc, uc, nb, (char *)P.scratch.p, st)
                                  : run_plane<T>(P, fc, uc, nb, (char *)P.scratch.p, st);
        if (rc) return rc;
    }
    return MD_OK;
}

}  // namespace

extern "C" {

int64_t md_plan_scratch_bytes(const md_plan *P, int64_t batch) {
    if (!P) return 0;
    return (int64_t)scratch_fields(*P) * P->frame_elems() * P->es * auto_chunk(*P, batch);
}

int32_t md_plan_set_chunk(md_plan *P, int64_t frames) {
    if (!P || frames < 0) return fail(MD_EINVAL, "bad chunk");
    std::lock_guard<std::recursive_mutex> lock(P->mu);
    P->chunk = frames;
    return MD_OK;
}

// the plan's description names the iteration kernel: keep it in step with the switch
static void describe_swap(std::string &d, const char *from, const char *to) {
    const size_t i = d.find(from);
    if (i != std::string::npos) d.replace(i, std::strlen(from), to);
}

int32_t md_plan_set_fused(md_plan *P, int32_t on) {
    if (!P) return fail(MD_EINVAL, "null plan");
    std::lock_guard<std::recursive_mutex> lock(P->mu);
    static const char *kFused = "fused cluster iteration kernel";
    if (P->path == PATH_PLANE_DIRECT) {
        if (on && !(P->fast_plane && !P->big &&
                    fused_plane_supported(P->d.height, P->d.width, P->hblur, P->hadj, P->htaps_blur, P->htaps_adj, P->d.dtype)))
            return fail(MD_EINVAL, "fused kernel not available for this plan");
        P->fused_plane = on != 0;
        if (on) describe_swap(P->describe, "direct taps (2 launches/iteration)", "direct taps, fused cluster iteration kernel");
        else describe_swap(P->describe, "direct taps, fused cluster iteration kernel", "direct taps (2 launches/iteration)");
        return MD_OK;
    }
    if (on && !(P->path == PATH_LINES && P->fast_lines && fused_lines_supported(P->d.dtype, P->n, P->m, 0,
                                                                         std::max(line_radius(P->lblur), line_radius(P->ladj)))))
        return fail(MD_EINVAL, "fused kernel not available for this plan");
    P->fused = on != 0;
    P->fused_clusters = !on ? 0 : (P->d.dtype == MD_F64 ? lines_fused_clusters<double>(*P) : lines_fused_clusters<float>(*P));
    if (P->path == PATH_LINES) {
        const char *per_it = P->fast_lines ? "k_wiener_lines + k_iter_lines_fast per iteration"
                                           : "k_wiener_lines + k_iter_lines per iteration";
        if (on) describe_swap(P->describe, per_it, kFused);
        else describe_swap(P->describe, kFused, per_it);
    }
    return MD_OK;
}

int32_t md_plan_is_fused(const md_plan *P) { return P && (P->fused || P->fused_plane) ? 1 : 0; }

int32_t md_plan_fused_geometry(const md_plan *P, int32_t *cluster_ctas, int32_t *resident_clusters,
                               int32_t *ctas_per_sm) {
    if (!P || !cluster_ctas || !resident_clusters || !ctas_per_sm) return fail(MD_EINVAL, "bad arguments");
    const bool on = P->fused && P->fused_clusters > 0;
    *cluster_ctas = on ? P->fused_geom[0] : 0;
    *resident_clusters = on ? P->fused_clusters : 0;
    *ctas_per_sm = on ? P->fused_geom[1] : 0;
    return MD_OK;
}

int32_t md_run(md_plan *P, const void *f, void *u, int64_t batch, void *stream) {
    if (!P || batch < 0) return fail(MD_EINVAL, "bad arguments");
    if (batch == 0) return MD_OK;                   // empty batch: nothing to read (pointers may be null)
    if (!f || !u) return fail(MD_EINVAL, "bad arguments");
    clear_stale_error();
    if (f == u) return fail(MD_EINVAL, "input and output must not alias");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    PlanUse use(P, st);
    return P->d.dtype == MD_F64 ? run_typed<double>(*P, f, u, batch, st) : run_typed<float>(*P, f, u, batch, st);
}

int32_t md_run_profile(md_plan *P, const void *f, void *u, int64_t batch, void *stream, double *ms_out) {
    if (!P || !ms_out) return fail(MD_EINVAL, "bad arguments");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    PlanUse use(P, st);
    Prof *pr = &g_prof_pool;
    pr->n = 0;
    cudaEventRecord(pr->get(0), st);
    g_prof = pr;
    int rc = md_run(P, f, u, batch, stream);
    g_prof = nullptr;
    if (rc == MD_OK) {
        cudaEventSynchronize(pr->ev[pr->n]);
        for (int k = 0; k < PK_KINDS; ++k) ms_out[k] = 0.0;
        for (int i = 1; i <= pr->n; ++i) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, pr->ev[i - 1], pr->ev[i]);
            ms_out[pr->kind[i]] += ms;
        }
        ms_out[PK_KINDS] = (double)pr->n;
    }
    return rc;
}

int32_t md_run_profile_groups(md_plan *P, const void *f, void *u, int64_t batch, void *stream, double *group_ms,
                              int32_t *group_kind, int32_t max_groups, int32_t *n_groups) {
    if (!P || !group_ms || !group_kind || !n_groups || max_groups < 1) return fail(MD_EINVAL, "bad arguments");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    PlanUse use(P, st);
    Prof *pr = &g_prof_pool;
    pr->n = 0;
    cudaEventRecord(pr->get(0), st);
    g_prof = pr;
    int rc = md_run(P, f, u, batch, stream);
    g_prof = nullptr;
    if (rc) return rc;
    cudaEventSynchronize(pr->ev[pr->n]);
    const int n = std::min<int>(pr->n, max_groups);
    for (int i = 1; i <= n; ++i) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, pr->ev[i - 1], pr->ev[i]);
        group_ms[i - 1] = ms;
        group_kind[i - 1] = pr->kind[i];
    }
    *n_groups = n;
    return MD_OK;
}

int32_t md_run_launch_count(const md_plan *P, int64_t batch) {
    if (!P || batch <= 0) return 0;
    const int64_t chunk = auto_chunk(*P, batch);
    const int64_t chunks = (batch + chunk - 1) / chunk;
    const int64_t sub = (chunk + 65534) / 65535;    // grid.y / grid.z splits
    const int K = P->d.iterations;
    int per = 0;
    const bool wiener = P->d.init == MD_INIT_WIENER;
    if (P->path == PATH_LINES) {
        per = 1;
        if (K > 0) per += P->fused ? 1 : K + (P->vert ? 1 : 0);
    } else {
        per = wiener ? (P->big ? (P->line_axis >= 0 ? 4 : 6) : 3) : 1;   // two-level Wiener: 6 (1D: 4) passes
        if (K > 0) {
            if (!wiener && P->path == PATH_PLANE_FFT) per += 1;
            per += P->fused_plane ? 1 : K * (P->path == PATH_PLANE_FFT ? 4 : 2);
        }
    }
    return (int32_t)(chunks * sub * per);
}

int32_t md_run_host_ex(md_plan *P, const void *f, int32_t in_type, void *u, int32_t out_type, int64_t batch,
                       void *stream) {
    if (!P || batch < 0) return fail(MD_EINVAL, "bad arguments");
    if (in_type != MD_IO_F64 && in_type != MD_IO_F32 && in_type != MD_IO_U8) return fail(MD_EINVAL, "bad input type");
    if (out_type != MD_IO_F64 && out_type != MD_IO_F32 && out_type != MD_IO_U8)
        return fail(MD_EINVAL, "bad output type");
    if (batch == 0) return MD_OK;
    if (!f || !u) return fail(MD_EINVAL, "bad arguments");
    clear_stale_error();
    cudaStream_t user = static_cast<cudaStream_t>(stream);
    PlanUse use(P, user);
    const int64_t fe = P->frame_elems();
    const int ib = io_bytes(in_type), ob = io_bytes(out_type);
    // pipeline: chunk c runs H2D -> convert -> pipeline -> convert -> D2H on internal stream
    // c % kHostStreams, so copies of one chunk overlap compute of the next
    const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(batch, std::max<int64_t>(1, (64ll << 20) / (fe * 8))));
    int rc = P->ensure_host_streams();
    if (rc) return rc;
    const size_t in_b = (size_t)fe * ib * chunk, tin_b = (size_t)fe * P->es * chunk, tout_b = tin_b,
                 out_b = (size_t)fe * ob * chunk;
    const size_t scr_b = (size_t)scratch_fields(*P) * fe * P->es * chunk;
    const size_t per = align_up(in_b) + align_up(tin_b) + align_up(tout_b) + align_up(out_b) + align_up(scr_b);
    const int nstreams = (int)std::min<int64_t>(kHostStreams, (batch + chunk - 1) / chunk);
    rc = P->stage.ensure(per * nstreams);      // one staging slot per stream actually used
    if (rc) return rc;
    // the host chunk size applies to this call only (restored on every exit path); on an error
    // the internal streams are drained before returning, so no copy into the caller's host
    // buffers is still in flight when the error comes back
    struct ChunkGuard {
        md_plan *P;
        int64_t saved;
        ~ChunkGuard() { P->chunk = saved; }
    } guard{P, P->chunk};
    auto body = [&]() -> int {
        CU(cudaEventRecord(P->ev_start, user));
        for (int s = 0; s < kHostStreams; ++s) CU(cudaStreamWaitEvent(P->hstream[s], P->ev_start, 0));
        P->chunk = chunk;
        for (int64_t b0 = 0, c = 0; b0 < batch; b0 += chunk, ++c) {
            const int64_t nb = std::min(chunk, batch - b0);
            const int s = (int)(c % kHostStreams);
            cudaStream_t st = P->hstream[s];
            char *base = (char *)P->stage.p + per * s;
            char *din = base, *dtin = din + align_up(in_b), *dtout = dtin + align_up(tin_b),
                 *dout = dtout + align_up(tout_b), *dscr = dout + align_up(out_b);
            CU(cudaMemcpyAsync(din, (const char *)f + b0 * fe * ib, nb * fe * ib, cudaMemcpyHostToDevice, st));
            const void *fin = din;
            if (in_type != (P->d.dtype == MD_F64 ? MD_IO_F64 : MD_IO_F32)) {
                CU(P->d.dtype == MD_F64 ? launch_convert_in<double>(din, in_type, dtin, nb * fe, st)
                                        : launch_convert_in<float>(din, in_type, dtin, nb * fe, st));
                fin = dtin;
            }
            const bool direct_out = out_type == (P->d.dtype == MD_F64 ? MD_IO_F64 : MD_IO_F32);
            void *uo = direct_out ? (void *)dout : (void *)dtout;
            const int r = P->d.dtype == MD_F64 ? run_chunk<double>(*P, fin, uo, nb, dscr, st)
                                               : run_chunk<float>(*P, fin, uo, nb, dscr, st);
            if (r) return r;
            if (!direct_out) {
                CU(P->d.dtype == MD_F64 ? launch_convert_out<double>(dtout, dout, out_type, nb * fe, st)
                                        : launch_convert_out<float>(dtout, dout, out_type, nb * fe, st));
            }
            CU(cudaMemcpyAsync((char *)u + b0 * fe * ob, dout, nb * fe * ob, cudaMemcpyDeviceToHost, st));
        }
        for (int s = 0; s < kHostStreams; ++s) {
            CU(cudaEventRecord(P->ev_done[s], P->hstream[s]));
            CU(cudaStreamWaitEvent(user, P->ev_done[s], 0));
        }
        return MD_OK;
    };
    rc = body();
    if (rc) {
        const std::string msg = g_err;                // keep the first error's message
        for (int s = 0; s < kHostStreams; ++s) cudaStreamSynchronize(P->hstream[s]);
        cudaGetLastError();
        g_err = msg;
        return rc;
    }
    CU(cudaStreamSynchronize(user));
    return MD_OK;
}

int32_t md_convert(const void *in, int32_t in_type, void *out, int32_t out_type, int64_t n, void *stream) {
    if (!in || !out || n < 0) return fail(MD_EINVAL, "bad arguments");
    if (in_type != MD_IO_F64 && in_type != MD_IO_F32 && in_type != MD_IO_U8) return fail(MD_EINVAL, "bad input type");
    if (out_type != MD_IO_F64 && out_type != MD_IO_F32 && out_type != MD_IO_U8)
        return fail(MD_EINVAL, "bad output type");
    if (out_type == MD_IO_U8 && in_type == MD_IO_U8) return fail(MD_EINVAL, "uint8 -> uint8 is not a conversion");
    if (n == 0) return MD_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (out_type == MD_IO_U8) {            // write_pgm quantisation of float results
        CU(in_type == MD_IO_F64 ? launch_convert_out<double>(in, out, MD_IO_U8, n, st)
                                : launch_convert_out<float>(in, out, MD_IO_U8, n, st));
        return MD_OK;
    }
    CU(out_type == MD_IO_F64 ? launch_convert_in<double>(in, in_type, out, n, st)
                             : launch_convert_in<float>(in, in_type, out, n, st));
    return MD_OK;
}

int32_t md_run_host(md_plan *P, const double *f, double *u, int64_t batch, void *stream) {
    return md_run_host_ex(P, f, MD_IO_F64, u, MD_IO_F64, batch, stream);
}

int32_t md_wiener(md_plan *P, const void *f, void *out, int64_t batch, void *stream) {
    if (!P || !f || !out || batch < 0) return fail(MD_EINVAL, "bad arguments");
    if (batch == 0) return MD_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    PlanUse use(P, st);
    if (P->path == PATH_LINES) {
        if (P->log2n < 0) return fail(MD_EINVAL, "the blur axis must have power-of-two extent");
        if (!P->d_mult) return fail(MD_EINVAL, "blur-axis length above the on-chip FFT limit");
        WienerLinesArgs a{};
        a.in = f; a.out = out; a.fpos = nullptr; a.n = P->n; a.log2n = P->log2n; a.m = P->m;
        a.in_vert = P->vert; a.out_vert = P->vert; a.clamp = 0; a.mult = P->d_mult; a.tw = P->d_tw_n;
        a.floor = P->d.floor;
        if (P->wiener_reg) {
            a.mult = P->d_mult_nat;
            CU(P->d.dtype == MD_F64 ? launch_wiener_reg<double>(a, batch, st) : launch_wiener_reg<float>(a, batch, st));
        } else {
            CU(P->d.dtype == MD_F64 ? launch_wiener_lines<double>(a, batch, st)
                                    : launch_wiener_lines<float>(a, batch, st));
        }
        return MD_OK;
    }
    if (!P->d_mult) return fail(MD_EINVAL, "2D Wiener needs power-of-two dimensions");
    const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(batch, (1ll << 30) / (P->frame_elems() * 2 * P->es)));
    int rc = P->scratch.ensure((size_t)P->frame_elems() * 2 * P->es * chunk);
    if (rc) return rc;
    for (int64_t b0 = 0; b0 < batch; b0 += chunk) {
        const int64_t nb = std::min(chunk, batch - b0);
        const int64_t off = b0 * P->frame_elems() * P->es;
        const void *fc = static_cast<const char *>(f) + off;
        void *oc = static_cast<char *>(out) + off;
        rc = P->d.dtype == MD_F64 ? wiener_plane<double>(*P, fc, oc, nullptr, P->scratch.p, false, false, nb, st)
                                  : wiener_plane<float>(*P, fc, oc, nullptr, P->scratch.p, false, false, nb, st);
        if (rc) return rc;
    }
    return MD_OK;
}

}  // extern "C"

namespace {

template <typename T>
int convolve_typed(md_plan &P, const void *in, void *out, int64_t batch, int which, cudaStream_t st) {
    const int64_t fe = P.frame_elems();
    if (P.path == PATH_LINES) {
        ConvLinesArgs a{};
        a.n = P.n; a.m = P.m; a.c = which ? P.ladj : P.lblur;
        a.taps = which ? P.d_taps_adj : P.d_taps_blur;
        if (!P.vert) {
            a.in = in; a.out = out;
            CU(launch_conv_lines<T>(a, batch, st));
            return MD_OK;
        }
        const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(batch, (1ll << 30) / (fe * 2 * (int64_t)sizeof(T))));
        int rc = P.scratch.ensure((size_t)fe * 2 * sizeof(T) * chunk);
        if (rc) return rc;
        char *A = (char *)P.scratch.p, *B = A + fe * sizeof(T) * chunk;
        for (int64_t b0 = 0; b0 < batch; b0 += chunk) {
            const int64_t nb = std::min(chunk, batch - b0);
            const int64_t off = b0 * fe * sizeof(T);
            CU(launch_transpose<T>(static_cast<const char *>(in) + off, A, nullptr, P.n, P.m, 0.0, 0, nb, st));
            a.in = A; a.out = B;
            CU(launch_conv_lines<T>(a, nb, st));
            CU(launch_transpose<T>(B, static_cast<char *>(out) + off, nullptr, P.m, P.n, 0.0, 0, nb, st));
        }
        return MD_OK;
    }
    if (P.path == PATH_PLANE_DIRECT) {
        ConvPlaneArgs a{};
        a.in = in; a.out = out; a.H = P.d.height; a.W = P.d.width; a.periodic = P.periodic;
        a.h = which ? P.hadj : P.hblur;
        a.taps = which ? P.d_ptaps_adj : P.d_ptaps_blur;
        CU(launch_conv_plane<T>(a, batch, st));
        return MD_OK;
    }
    const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(batch, (1ll << 30) / (fe * 2 * (int64_t)sizeof(T))));
    int rc = P.scratch.ensure((size_t)fe * 2 * sizeof(T) * chunk);
    if (rc) return rc;
    for (int64_t b0 = 0; b0 < batch; b0 += chunk) {
        const int64_t nb = std::min(chunk, batch - b0);
        const int64_t off = b0 * fe * sizeof(T);
        Fft2Args a = fft2_base<T>(P);
        a.z = P.scratch.p;
        a.load = R_LOAD_REAL; a.ra = static_cast<const char *>(in) + off; a.epi = R_EPI_NONE; a.fwd_after = 1;
        CU(launch_fft2_rows<T>(a, nb, st));
        a.filt = P.d_hspec; a.conj_filt = which; a.col_inv = 1;
        CU(launch_fft2_cols<T>(a, nb, st));
        a.load = R_LOAD_COMPLEX; a.inv = 1; a.epi = R_EPI_STORE_PAIR; a.fwd_after = 0;
        a.oa = static_cast<char *>(out) + off; a.ob = nullptr;
        CU(launch_fft2_rows<T>(a, nb, st));
    }
    return MD_OK;
}

template <typename T>
int adjoint_pair_typed(md_plan &P, const void *p, const void *q, void *op, void *oq, int64_t batch, cudaStream_t st) {
    if (P.path != PATH_PLANE_FFT) {
        int rc = convolve_typed<T>(P, p, op, batch, 1, st);
        if (rc) return rc;
        return convolve_typed<T>(P, q, oq, batch, 1, st);
    }
    const int64_t fe = P.frame_elems();
    const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(batch, (1ll << 30) / (fe * 2 * (int64_t)sizeof(T))));
    int rc = P.scratch.ensure((size_t)fe * 2 * sizeof(T) * chunk);
    if (rc) return rc;
    for (int64_t b0 = 0; b0 < batch; b0 += chunk) {
        const int64_t nb = std::min(chunk, batch - b0);
        const int64_t off = b0 * fe * sizeof(T);
        Fft2Args a = fft2_base<T>(P);
        a.z = P.scratch.p;
        a.load = R_LOAD_PAIR; a.ra = static_cast<const char *>(p) + off; a.rb = static_cast<const char *>(q) + off;
        a.epi = R_EPI_NONE; a.fwd_after = 1;
        CU(launch_fft2_rows<T>(a, nb, st));
        a.filt = P.d_hspec; a.conj_filt = 1; a.col_inv = 1;
        CU(launch_fft2_cols<T>(a, nb, st));
        a.load = R_LOAD_COMPLEX; a.inv = 1; a.epi = R_EPI_STORE_PAIR; a.fwd_after = 0;
        a.oa = static_cast<char *>(op) + off; a.ob = static_cast<char *>(oq) + off;
        CU(launch_fft2_rows<T>(a, nb, st));
    }
    return MD_OK;
}

}  // namespace

extern "C" {

int32_t md_convolve(md_plan *P, const void *in, void *out, int64_t batch, int32_t which, void *stream) {
    if (!P || !in || !out || batch < 0 || (which != 0 && which != 1)) return fail(MD_EINVAL, "bad arguments");
    if (batch == 0) return MD_OK;
    if (in == out) return fail(MD_EINVAL, "input and output must not alias");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    PlanUse use(P, st);
    return P->d.dtype == MD_F64 ? convolve_typed<double>(*P, in, out, batch, which, st)
                                : convolve_typed<float>(*P, in, out, batch, which, st);
}

int32_t md_adjoint_pair(md_plan *P, const void *p, const void *q, void *op, void *oq, int64_t batch, void *stream) {
    if (!P || !p || !q || !op || !oq || batch < 0) return fail(MD_EINVAL, "bad arguments");
    if (batch == 0) return MD_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    PlanUse use(P, st);
    return P->d.dtype == MD_F64 ? adjoint_pair_typed<double>(*P, p, q, op, oq, batch, st)
                                : adjoint_pair_typed<float>(*P, p, q, op, oq, batch, st);
}

// shared LUT for the plan-free step kernels (built once, never freed)
static std::mutex g_lut_mu;
static md_plan *g_lut_owner = nullptr;
static int lut_view(LutView *out) {
    std::lock_guard<std::mutex> lk(g_lut_mu);
    if (!g_lut_owner) {
        md_plan *P = new md_plan();
        const int rc = build_lut(P);
        if (rc) {
            delete P;
            return rc;
        }
        g_lut_owner = P;
    }
    *out = g_lut_owner->lut;
    return MD_OK;
}

int32_t md_robust_weight(int32_t dtype, const void *f, const void *b, void *out, int64_t n, double eps_data,
                         double floor, int32_t assume_floored, void *stream) {
    if (!f || !b || !out || n < 0) return fail(MD_EINVAL, "bad arguments");
    LutView L;
    int rc = lut_view(&L);
    if (rc) return rc;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const double e2 = eps_data * eps_data;
    CU(dtype == MD_F64 ? launch_robust_weight<double>(f, b, out, n, e2, floor, assume_floored, L, st)
                       : launch_robust_weight<float>(f, b, out, n, e2, floor, assume_floored, L, st));
    return MD_OK;
}

int32_t md_lut_r1(int32_t dtype, const void *x, void *out, int64_t n, void *stream) {
    if (!x || !out || n < 0) return fail(MD_EINVAL, "bad arguments");
    LutView L;
    int rc = lut_view(&L);
    if (rc) return rc;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    CU(dtype == MD_F64 ? launch_lut_r1<double>(x, out, n, L, st) : launch_lut_r1<float>(x, out, n, L, st));
    return MD_OK;
}

int32_t md_lut_table(double *host_out, int64_t count) {
    if (!host_out || count < kLutCount) return fail(MD_EINVAL, "need room for the whole table");
    LutView L;
    int rc = lut_view(&L);
    if (rc) return rc;
    CU(cudaMemcpy(host_out, L.t64, kLutCount * sizeof(double), cudaMemcpyDeviceToHost));
    return MD_OK;
}

int32_t md_diffusion(int32_t dtype, const void *u, void *out, int64_t batch, int32_t height, int32_t width,
                     double eps_reg, void *stream) {
    if (!u || !out || batch < 0 || height < 1 || width < 1) return fail(MD_EINVAL, "bad arguments");
    if (!(eps_reg > 0.0)) return fail(MD_EINVAL, "eps_reg must be positive");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    CU(dtype == MD_F64 ? launch_diffusion<double>(u, out, batch, height, width, eps_reg * eps_reg, st)
                       : launch_diffusion<float>(u, out, batch, height, width, eps_reg * eps_reg, st));
    return MD_OK;
}

int32_t md_rrrl_step(md_plan *P, const void *u, const void *f, const void *b, const void *w, const void *d,
                     void *out, int64_t batch, double alpha, void *stream) {
    if (!P || !u || !f || !b || !out || batch < 0) return fail(MD_EINVAL, "bad arguments");
    if (batch == 0) return MD_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    PlanUse use(P, st);
    const int64_t n = P->frame_elems() * batch;
    const size_t fb = (size_t)n * P->es;
    int rc = P->stage.ensure(4 * fb);
    if (rc) return rc;
    char *R = (char *)P->stage.p, *NUM = R + fb, *DEN = NUM + fb;
    const bool f64 = P->d.dtype == MD_F64;
    CU(f64 ? launch_ratio<double>(f, b, w, R, n, st) : launch_ratio<float>(f, b, w, R, n, st));
    rc = w ? md_adjoint_pair(P, R, w, NUM, DEN, batch, stream) : md_convolve(P, R, NUM, batch, 1, stream);
    if (rc) return rc;
    if (!d) alpha = 0.0;
    CU(f64 ? launch_combine<double>(u, NUM, w ? DEN : nullptr, d, out, n, alpha, st)
           : launch_combine<float>(u, NUM, w ? DEN : nullptr, d, out, n, alpha, st));
    return MD_OK;
}

// natural-order complex transforms of `lines` contiguous lines of length n, in place
// (FourierPlan.forward / inverse, fft.py:52-117): tables per (n, dtype) built once
int32_t md_fft(int32_t dtype, void *z, int32_t n, int64_t lines, int32_t inverse, void *stream) {
    if ((dtype != MD_F64 && dtype != MD_F32) || lines < 0 || n < 1 || n > (1 << 20) || !is_pow2(n))
        return fail(MD_EINVAL, "transform length must be a power of two in [1, 1048576]");
    if (lines == 0 || n == 1) return MD_OK;               // length 1: the identity both ways
    if (!z) return fail(MD_EINVAL, "bad arguments");
    clear_stale_error();
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    struct Tables { void *tw = nullptr; BigAxis ax{}; std::vector<void *> owned; };
    static std::mutex mu;
    static std::map<std::tuple<int, int, int>, Tables> cache;
    int dev = 0;
    cudaGetDevice(&dev);
    const bool single = n <= (dtype == MD_F64 ? fft_lines_max_single<double>() : fft_lines_max_single<float>());
    Tables *tb;
    {
        std::lock_guard<std::mutex> lock(mu);
        auto key = std::make_tuple(n, dtype, dev);
        auto it = cache.find(key);
        if (it == cache.end()) {
            Tables t;
            int rc = single ? build_twiddles(n, dtype, &t.tw) : build_big_axis(n, dtype, &t.ax, t.owned);
            if (rc) return rc;
            it = cache.emplace(key, std::move(t)).first;
        }
        tb = &it->second;
    }
    if (single) {
        CU(dtype == MD_F64 ? launch_fft_lines_nat<double>(z, n, lines, tb->tw, inverse ? 1 : 0, st)
                           : launch_fft_lines_nat<float>(z, n, lines, tb->tw, inverse ? 1 : 0, st));
        return MD_OK;
    }
    // two-level passes (N = N1 N2, factors up to 1024: the reference's 2^20 limit, fft.py:45) in
    // groups of lines whose element count keeps the passes' 32-bit in-frame offsets
    const int64_t per = std::max<int64_t>(1, ((1ll << 31) - 1) / n);
    const int es = dtype == MD_F64 ? 16 : 8;
    const size_t bytes = (size_t)std::min<int64_t>(lines, per) * n * es;
    void *tmp = nullptr;
    CU(cudaMallocAsync(&tmp, bytes, st));
    cudaError_t e = cudaSuccess;
    for (int64_t l0 = 0; l0 < lines && e == cudaSuccess; l0 += per) {
        const int64_t nl = std::min(per, lines - l0);
        void *zc = static_cast<char *>(z) + l0 * n * es;
        if (!inverse) {
            e = dtype == MD_F64 ? big_axis<double>(tb->ax, zc, (int)nl, n, 1, 0, nullptr, nullptr, nullptr, 0, 1.0, 1, st)
                                : big_axis<float>(tb->ax, zc, (int)nl, n, 1, 0, nullptr, nullptr, nullptr, 0, 1.0, 1, st);
            if (e == cudaSuccess)
                e = dtype == MD_F64 ? launch_fft_perm<double>(zc, tmp, tb->ax, nl, 1, st)
                                    : launch_fft_perm<float>(zc, tmp, tb->ax, nl, 1, st);
        } else {
            e = dtype == MD_F64 ? launch_fft_perm<double>(zc, tmp, tb->ax, nl, 0, st)
                                : launch_fft_perm<float>(zc, tmp, tb->ax, nl, 0, st);
            if (e == cudaSuccess)
                e = dtype == MD_F64
                        ? big_axis<double>(tb->ax, tmp, (int)nl, n, 1, 1, nullptr, nullptr, nullptr, 0, 1.0 / n, 1, st)
                        : big_axis<float>(tb->ax, tmp, (int)nl, n, 1, 1, nullptr, nullptr, nullptr, 0, 1.0 / n, 1, st);
        }
        if (e == cudaSuccess) e = cudaMemcpyAsync(zc, tmp, (size_t)nl * n * es, cudaMemcpyDeviceToDevice, st);
    }
    cudaFreeAsync(tmp, st);
    CU(e);
    return MD_OK;
}

int32_t md_min(int32_t dtype, const void *x, int64_t n, double *out_host, void *stream) {
    if (!x || n <= 0 || !out_host) return fail(MD_EINVAL, "bad arguments");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int nb = (int)std::min<int64_t>(1024, (n + 255) / 256);
    double *partial = nullptr;
    CU(cudaMallocAsync((void **)&partial, nb * sizeof(double), st));
    CU(dtype == MD_F64 ? launch_min<double>(x, n, partial, nb, st) : launch_min<float>(x, n, partial, nb, st));
    std::vector<double> h(nb);
    CU(cudaMemcpyAsync(h.data(), partial, nb * sizeof(double), cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    CU(cudaFreeAsync(partial, st));
    *out_host = *std::min_element(h.begin(), h.end());
    return MD_OK;
}

int32_t md_guard(int32_t dtype, void *x, int64_t n, void *stream) {
    if (!x || n < 0) return fail(MD_EINVAL, "bad arguments");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    CU(dtype == MD_F64 ? launch_guard<double>(x, n, st) : launch_guard<float>(x, n, st));
    return MD_OK;
}

}  // extern "C"

// ======================================================================== row slabs (c5)
// One image split into row slabs over ranks. The driver
// (paper_1212_2245_b200/slab.py) moves halo rows (NCCL send/recv) and transposes the
// spectrum (all-to-all); these entries are the per-rank compute.
namespace {

__global__ void k_copy_cols(const unsigned char *src, unsigned char *dst, int H, int W, int col0, int cols, int es) {
    const int64_t n = (int64_t)H * cols;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t y = i / cols, x = i - y * cols;
        const unsigned char *s = src + ((int64_t)y * W + col0 + x) * es;
        unsigned char *d = dst + i * es;
        for (int b = 0; b < es; ++b) d[b] = s[b];
    }
}

int slab_check(const md_plan *P) {
    if (!P) return fail(MD_EINVAL, "null plan");
    if (P->path != PATH_PLANE_DIRECT || !P->big || !P->fast_plane || P->line_axis >= 0)
        return fail(MD_EINVAL, "slab execution needs a 2D direct-tap plan built with MD_FLAG_BIG_FFT");
    return MD_OK;
}

}  // namespace

extern "C" {

int32_t md_slab_halo(const md_plan *P, int32_t *top, int32_t *bottom) {
    int rc = slab_check(P);
    if (rc) return rc;
    // stage A runs on rows [-adj.ht, S + adj.hb) and reads blur.ht / blur.hb more; TV needs 2
    *top = std::max(P->hadj.ht + P->hblur.ht, 2);
    *bottom = std::max(P->hadj.hb + P->hblur.hb, 2);
    return MD_OK;
}

int32_t md_slab_prepare(md_plan *P, int32_t col0, int32_t cols, void **mult_block) {
    int rc = slab_check(P);
    if (rc) return rc;
    if (col0 < 0 || cols < 1 || col0 + cols > P->d.width) return fail(MD_EINVAL, "bad column block");
    const int ces = P->d.dtype == MD_F64 ? 16 : 8;
    void *blk = nullptr;
    CU(cudaMalloc(&blk, (size_t)P->d.height * cols * ces));
    k_copy_cols<<<1024, 256>>>((const unsigned char *)P->d_mult, (unsigned char *)blk, P->d.height, P->d.width,
                               col0, cols, ces);
    CU(cudaGetLastError());
    CU(cudaDeviceSynchronize());
    P->owned.push_back(blk);
    *mult_block = blk;
    return MD_OK;
}

int32_t md_slab_rows_fft(md_plan *P, void *z, const void *real_in, int32_t rows, int32_t inv, double scale,
                         void *stream) {
    int rc = slab_check(P);
    if (rc) return rc;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    PlanUse use(P, st);
    const int W = P->d.width;
    CU(P->d.dtype == MD_F64 ? big_axis<double>(P->bigW, z, rows, W, 1, inv, real_in, nullptr, nullptr, 0, scale, 1, st)
                            : big_axis<float>(P->bigW, z, rows, W, 1, inv, real_in, nullptr, nullptr, 0, scale, 1, st));
    return MD_OK;
}

int32_t md_slab_cols_filter(md_plan *P, void *zc, int32_t cols, const void *mult_block, void *stream) {
    int rc = slab_check(P);
    if (rc) return rc;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    PlanUse use(P, st);
    const int H = P->d.height;
    CU(P->d.dtype == MD_F64 ? big_axis_filter<double>(P->bigH, zc, H, cols, 0, mult_block, 0, 1, st)
                            : big_axis_filter<float>(P->bigH, zc, H, cols, 0, mult_block, 0, 1, st));
    return MD_OK;
}

int32_t md_slab_wiener_epilogue(md_plan *P, const void *z, const void *f, void *u0, void *fpos, int32_t rows,
                                void *stream) {
    int rc = slab_check(P);
    if (rc) return rc;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    PlanUse use(P, st);
    const int64_t n = (int64_t)rows * P->d.width;
    const double scale = 1.0 / ((double)P->d.height * P->d.width);
    CU(P->d.dtype == MD_F64 ? launch_big_wiener_epilogue<double>(z, f, u0, fpos, n, scale, P->d.floor, 1, st)
                            : launch_big_wiener_epilogue<float>(z, f, u0, fpos, n, scale, P->d.floor, 1, st));
    return MD_OK;
}

int32_t md_slab_stage(md_plan *P, const void *u, const void *fpos, void *p, void *w, void *u_out, int32_t rows,
                      int32_t row0, int32_t a_begin, int32_t a_end, int32_t b_begin, int32_t b_end, void *stream) {
    int rc = slab_check(P);
    if (rc) return rc;
    if (a_begin < -P->hadj.ht || a_end > rows + P->hadj.hb || b_begin < 0 || b_end > rows)
        return fail(MD_EINVAL, "slab stage rows out of range");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    PlanUse use(P, st);
    PlaneFastDesc s{};
    s.u = u; s.f = fpos; s.p = p; s.w = w; s.u_out = u_out;     // all point at own row 0 of haloed buffers
    s.H = rows; s.W = P->d.width; s.periodic = P->periodic;
    s.slab = 1; s.gy0 = row0; s.Hg = P->d.height;
    s.a_begin = a_begin; s.a_end = a_end; s.b_begin = b_begin; s.b_end = b_end;
    int32_t top = 0, bot = 0;
    md_slab_halo(P, &top, &bot);                 // the haloed buffers' extent (slab.py SlabGeometry)
    s.halo_top = top; s.halo_bot = bot;
    s.hb = P->hblur; s.ha = P->hadj; s.taps_blur = &P->htaps_blur; s.taps_adj = &P->htaps_adj;
    s.alpha = P->d.alpha; s.eps_d2 = P->d.eps_data * P->d.eps_data; s.eps_r2 = P->d.eps_reg * P->d.eps_reg;
    s.has_d = P->has_d; s.lut = P->lut;
    CU(P->d.dtype == MD_F64 ? launch_plane_fast<double>(s, P->robust, 1, st)
                            : launch_plane_fast<float>(s, P->robust, 1, st));
    return MD_OK;
}

int32_t md_slab_iterate(md_plan *P, const void *u, const void *fpos, void *p, void *w, void *u_out, int32_t rows,
                        int32_t row0, void *stream) {
    if (!P) return fail(MD_EINVAL, "null plan");
    return md_slab_stage(P, u, fpos, p, w, u_out, rows, row0, -P->hadj.ht, rows + P->hadj.hb, 0, rows, stream);
}

int32_t md_slab_bands(const md_plan *P, int32_t *a_in, int32_t *b_in, int32_t *adj_top, int32_t *adj_bottom) {
    int rc = slab_check(P);
    if (rc) return rc;
    *adj_top = P->hadj.ht;
    *adj_bottom = P->hadj.hb;
    // stage A rows that read no halo u: [blur.ht, S - blur.hb); stage B rows whose p / W come from
    // those rows only (and whose TV stencil stays inside): [adj.ht + blur.ht, S - blur.hb - adj.hb)
    *a_in = std::max(P->hblur.ht, P->hblur.hb);
    *b_in = std::max(std::max(P->hadj.ht, P->hadj.hb) + *a_in, 2);
    return MD_OK;
}

}  // extern "C"
