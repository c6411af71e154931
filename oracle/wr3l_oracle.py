"""CPU oracle for the Wiener + RRRL deconvolution path -- TEST INFRASTRUCTURE ONLY.

What this is
    A plain NumPy float64 restatement of the reference package ``motiondeblur``
    (``/root/reference/pkg/src/motiondeblur``, arXiv:1212.2245) restricted to the hot
    path named by ``BASELINE.json`` ``north_star``: Wiener initialisation followed by
    robust regularised Richardson-Lucy (RRRL) iterations with a known PSF. Every
    function cites the reference ``file:line`` it follows.

Who may use it
    Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
    ``--impl reference`` legs, and only as the checker or the timed CPU baseline.
    The product package ``paper_1212_2245_b200`` never imports this module; its CUDA
    path fails loudly when the extension is missing.

How it is pinned
    ``tests/test_oracle_golden.py`` compares it against ``tests/golden/*.npz``, which
    ``oracle/gen_golden.py`` produced by running the reference package itself in the
    build container (``/root/reference`` is not present on the GPU box, so the
    fixtures are committed).

The FFT is deliberately the same radix-2 decimation-in-time scheme the reference uses
(bit-reversal gather, one butterfly sweep per stage, vectorised over trailing axes), so
that the CPU baseline timed from this module costs what the reference costs.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

GUARD = 1e-12                    # deconv.py:74  DIVISION_GUARD
RESUM_ROWS = 4096                # conv.py:35    _RESUM_INTERVAL


# --------------------------------------------------------------------------------------
# value types (core.py:138-257, restated as plain records)

@dataclass(frozen=True)
class OParams:
    """Same fields and defaults as ``DeconvParams`` (core.py:230-247)."""
    wiener_k: float = 0.006
    alpha: float = 0.003
    iterations: int = 5
    eps_data: float = 1.0
    eps_reg: float = 0.01
    floor: float = 0.1


@dataclass(frozen=True)
class OPsf:
    """kind in {"2d", "1d", "box"}; axis in {"v", "h", None} (core.py:83-93, 138-162).

    ``weights`` are already normalised; tap j reads x - (j - center) (core.py:146).
    """
    kind: str
    weights: np.ndarray
    center: object
    axis: str | None = None
    length: float | None = None

    @property
    def support(self):               # core.py:191-197
        if self.kind == "2d":
            return self.weights.shape
        n = self.weights.shape[0]
        return (n, 1) if self.axis == "v" else (1, n)


def box_weights(length: float) -> np.ndarray:
    """core.py:104-121 -- m taps of 1/m, or floor(L) taps of 1/L framed by two
    end taps of (L - floor L) / (2L)."""
    whole = math.floor(length)
    if length == whole:
        return np.full(whole, 1.0 / whole)
    end = (length - whole) / (2.0 * length)
    return np.concatenate(([end], np.full(whole, 1.0 / length), [end]))


def make_psf(kind, weights=None, center=None, axis=None, length=None) -> OPsf:
    """Normalising constructor mirroring core.py:164-189."""
    if kind == "box":
        w = box_weights(float(length))
        return OPsf("box", w, w.shape[0] // 2, axis, float(length))
    w = np.array(weights, dtype=np.float64)
    w = w / w.sum()
    if kind == "2d":
        w = np.atleast_2d(w)
        c = (w.shape[0] // 2, w.shape[1] // 2) if center is None else tuple(int(v) for v in center)
        return OPsf("2d", w, c)
    w = w.ravel()
    c = w.shape[0] // 2 if center is None else int(center)
    return OPsf("1d", w, c, axis)


def reflect(psf: OPsf) -> OPsf:
    """core.py:204-220 -- weights reversed, centre remapped to n-1-c."""
    if psf.kind == "2d":
        cy, cx = psf.center
        return OPsf("2d", psf.weights[::-1, ::-1].copy(),
                    (psf.weights.shape[0] - 1 - cy, psf.weights.shape[1] - 1 - cx))
    return OPsf(psf.kind, psf.weights[::-1].copy(), psf.weights.shape[0] - 1 - psf.center,
                psf.axis, psf.length)


def as_vertical(psf: OPsf) -> OPsf:
    """deconv.py:595-599."""
    if psf.axis != "h":
        return psf
    return OPsf(psf.kind, psf.weights, psf.center, "v", psf.length)


# --------------------------------------------------------------------------------------
# divergence table r1(s) = s - 1 - ln s   (deconv.py:81-139)

@dataclass(frozen=True)
class Lut:
    delta: float
    step: float
    upper: float
    direct_below: float
    table: np.ndarray = field(repr=False)
    slope: float
    intercept: float


def build_lut(delta=1.0 / 32.0, step=1.0 / 2048.0, upper=65.0, direct_below=0.5) -> Lut:
    """deconv.py:101-112."""
    count = int(round((upper - delta) / step)) + 1
    nodes = delta + step * np.arange(count)
    slope = 1.0 - 1.0 / upper
    return Lut(delta, step, upper, direct_below, nodes - 1.0 - np.log(nodes), slope,
               (upper - 1.0 - math.log(upper)) - slope * upper)


_LUT = None


def default_lut() -> Lut:
    global _LUT
    if _LUT is None:
        _LUT = build_lut()
    return _LUT


def r1(x: np.ndarray, lut: Lut | None = None) -> np.ndarray:
    """deconv.py:114-134 -- linear interpolation between table nodes, exact formula
    below ``direct_below``, linear continuation above ``upper``."""
    lut = default_lut() if lut is None else lut
    x = np.asarray(x, dtype=np.float64)
    t = np.minimum(x, lut.upper)
    t -= lut.delta
    t *= 1.0 / lut.step
    i = np.clip(t.astype(np.int64), 0, lut.table.shape[0] - 2)
    t -= i
    lo = lut.table[i]
    res = lut.table[i + 1]
    res -= lo
    res *= t
    res += lo
    above = x > lut.upper
    if above.any():
        res[above] = lut.slope * x[above] + lut.intercept
    below = x < lut.direct_below
    if below.any():
        xb = x[below]
        res[below] = xb - 1.0 - np.log(xb)
    return res


def robust_weight(f, b, eps_data=1.0, floor=0.1, lut=None, floored=False):
    """deconv.py:142-162 (and the public wrapper 165-180 without its checks)."""
    if floored:
        r = r1(b / f, lut)
        r *= f
    else:
        small = f < floor
        fs = np.where(small, 1.0, f)
        r = r1(b / fs, lut) * fs
        r = np.where(small, np.maximum(b - f, 0.0), r)
    r += eps_data * eps_data
    np.sqrt(r, out=r)
    np.divide(0.5, r, out=r)
    return r


def diffusion(u: np.ndarray, eps_reg: float) -> np.ndarray:
    """deconv.py:187-213 -- TV divergence with Neumann boundary; x fluxes first.
    (In-place NumPy so that the CPU baseline costs what the reference costs.)"""
    gx = u[:, 1:] - u[:, :-1]
    gy = u[1:, :] - u[:-1, :]
    gx2 = gx * gx
    gy2 = gy * gy
    g = np.zeros_like(u)
    g[:, 1:] += gx2
    g[:, :-1] += gx2
    g[1:, :] += gy2
    g[:-1, :] += gy2
    g *= 0.5
    g += eps_reg * eps_reg
    np.sqrt(g, out=g)
    np.divide(0.5, g, out=g)
    d = np.zeros_like(u)
    fx = g[:, 1:] + g[:, :-1]
    fx *= gx
    d[:, :-1] += fx
    d[:, 1:] -= fx
    fy = g[1:, :] + g[:-1, :]
    fy *= gy
    d[:-1, :] += fy
    d[1:, :] -= fy
    return d


def diffusion_energy(u: np.ndarray, eps_reg: float) -> float:
    """deconv.py:231-246."""
    gx2 = np.diff(u, axis=1) ** 2
    gy2 = np.diff(u, axis=0) ** 2
    q = np.zeros_like(u)
    q[:, 1:] += gx2
    q[:, :-1] += gx2
    q[1:, :] += gy2
    q[:-1, :] += gy2
    return float(np.sum(np.sqrt(0.5 * q + eps_reg * eps_reg)))


# --------------------------------------------------------------------------------------
# spatial convolution (conv.py:85-173)

def box_axis0(a: np.ndarray, length: float, center: int) -> np.ndarray:
    """conv.py:141-173 -- clamped sliding-window box along axis 0, as prefix-sum
    differences restarted every 4096 rows."""
    h = a.shape[0]
    whole = math.floor(length)
    frac = length != whole
    taps = whole + 2 if frac else whole
    out = np.empty_like(a)
    for r0 in range(0, h, RESUM_ROWS):
        r1_ = min(r0 + RESUM_ROWS, h)
        nk = r1_ - r0
        rows = np.clip(np.arange(r0 + center - taps + 1, r1_ + center), 0, h - 1)
        seg = a[rows]
        cs = np.zeros((seg.shape[0] + 1,) + a.shape[1:])
        np.cumsum(seg, axis=0, out=cs[1:])
        if frac:
            e = (length - whole) / (2.0 * length)
            blk = (cs[whole + 1:whole + 1 + nk] - cs[1:1 + nk]) * (1.0 / length)
            blk += e * seg[:nk]
            blk += e * seg[taps - 1:taps - 1 + nk]
        else:
            blk = (cs[whole:whole + nk] - cs[:nk]) * (1.0 / whole)
        out[r0:r1_] = blk
    return out


def box_filter(a: np.ndarray, length: float, center: int, axis: int = 0) -> np.ndarray:
    """conv.py:138-145."""
    if axis == 0:
        return box_axis0(a, length, center)
    return np.ascontiguousarray(box_axis0(np.ascontiguousarray(a.T), length, center).T)


def clamped_convolve(a: np.ndarray, psf: OPsf) -> np.ndarray:
    """conv.py:85-116 -- direct sum in tap order over an edge-replicated copy."""
    h, w = a.shape
    if psf.kind == "2d":
        k = psf.weights
        sy, sx = k.shape
        cy, cx = psf.center
        pad = np.pad(a, ((sy - 1 - cy, cy), (sx - 1 - cx, cx)), mode="edge")
        acc = np.zeros_like(a)
        for jy in range(sy):
            oy = sy - 1 - jy
            for jx in range(sx):
                if k[jy, jx] != 0.0:
                    ox = sx - 1 - jx
                    acc += k[jy, jx] * pad[oy:oy + h, ox:ox + w]
        return acc
    k = psf.weights
    s = k.shape[0]
    c = psf.center
    acc = np.zeros_like(a)
    if psf.axis == "v":
        pad = np.pad(a, ((s - 1 - c, c), (0, 0)), mode="edge")
        for j in range(s):
            if k[j] != 0.0:
                acc += k[j] * pad[s - 1 - j:s - 1 - j + h]
    else:
        pad = np.pad(a, ((0, 0), (s - 1 - c, c)), mode="edge")
        for j in range(s):
            if k[j] != 0.0:
                acc += k[j] * pad[:, s - 1 - j:s - 1 - j + w]
    return acc


def periodic_convolve(a: np.ndarray, psf: OPsf) -> np.ndarray:
    """Direct wrap-around convolution (the roll oracle of test_fft.py:16-28); equal to
    the FFT convolvers of deconv.py:329-376 up to rounding."""
    out = np.zeros_like(a)
    if psf.kind == "2d":
        cy, cx = psf.center
        for jy in range(psf.weights.shape[0]):
            for jx in range(psf.weights.shape[1]):
                if psf.weights[jy, jx] != 0.0:
                    out += psf.weights[jy, jx] * np.roll(a, (jy - cy, jx - cx), (0, 1))
        return out
    ax = 0 if psf.axis == "v" else 1
    for j in range(psf.weights.shape[0]):
        out += psf.weights[j] * np.roll(a, j - psf.center, ax)
    return out


# --------------------------------------------------------------------------------------
# radix-2 FFT (fft.py:52-117) and the real-pair filters (fft.py:160-280)

class Radix2:
    """Decimation-in-time radix-2 transform along axis 0 (fft.py:52-117).

    Forward is unnormalised, inverse scales by 1/n. Twiddles exp(-i pi k / half) are
    tabulated per stage (fft.py:77-85).
    """

    def __init__(self, n: int):
        if n < 1 or n & (n - 1) or n > (1 << 20):
            raise ValueError(f"transform length must be a power of two in [1, 2^20], got {n}")
        self.n = n
        bits = n.bit_length() - 1
        idx = np.arange(n)
        rev = np.zeros(n, dtype=np.intp)
        for b in range(bits):
            rev |= ((idx >> b) & 1) << (bits - 1 - b)
        self.perm = rev
        self.stages = []
        half = 1
        while half < n:
            self.stages.append(np.exp(-1j * np.pi * np.arange(half) / half))
            half <<= 1

    def _sweep(self, a, conj: bool):
        z = np.asarray(a, dtype=np.complex128)[self.perm]
        n = self.n
        tail = z.shape[1:]
        half = 1
        for tw in self.stages:
            w = (np.conj(tw) if conj else tw).reshape((half,) + (1,) * len(tail))
            v = z.reshape((n // (2 * half), 2, half) + tail)
            t = v[:, 1] * w
            v[:, 1] = v[:, 0] - t
            v[:, 0] += t
            half <<= 1
        return z

    def forward(self, a):
        return self._sweep(a, False)

    def inverse(self, a):
        z = self._sweep(a, True)
        z *= 1.0 / self.n
        return z


_PLANS: dict[int, Radix2] = {}


def plan(n: int) -> Radix2:
    p = _PLANS.get(n)
    if p is None:
        p = _PLANS[n] = Radix2(n)
    return p


def fft2(z, inverse=False):
    """fft.py:165-170 -- axis 1 (via transpose) then axis 0."""
    ph, pw = plan(z.shape[0]), plan(z.shape[1])
    if inverse:
        return ph.inverse(pw.inverse(z.T).T)
    return ph.forward(pw.forward(z.T).T)


def embed_1d(psf: OPsf, n: int) -> np.ndarray:
    """fft.py:192-201."""
    z = np.zeros(n)
    z[(np.arange(psf.weights.shape[0]) - psf.center) % n] = psf.weights
    return z


def embed_2d(psf: OPsf, shape) -> np.ndarray:
    """fft.py:204-221."""
    if psf.kind == "2d":
        w, (cy, cx) = psf.weights, psf.center
    elif psf.axis == "v":
        w, cy, cx = psf.weights[:, None], psf.center, 0
    else:
        w, cy, cx = psf.weights[None, :], 0, psf.center
    z = np.zeros(shape)
    z[np.ix_((np.arange(w.shape[0]) - cy) % shape[0], (np.arange(w.shape[1]) - cx) % shape[1])] = w
    return z


def spectrum_1d(psf: OPsf, n: int) -> np.ndarray:
    """fft.py:224-226."""
    return plan(n).forward(embed_1d(psf, n))


def spectrum_2d(psf: OPsf, shape) -> np.ndarray:
    """fft.py:229-233."""
    return fft2(embed_2d(psf, shape))


def column_filter(a: np.ndarray, filt: np.ndarray) -> np.ndarray:
    """fft.py:236-258 -- columns 2k / 2k+1 ride as real / imaginary part."""
    p = plan(a.shape[0])
    out = np.empty_like(a)
    npair = a.shape[1] // 2
    if npair:
        z = a[:, 0:2 * npair:2] + 1j * a[:, 1:2 * npair:2]
        z = p.inverse(p.forward(z) * filt[:, None])
        out[:, 0:2 * npair:2] = z.real
        out[:, 1:2 * npair:2] = z.imag
    if a.shape[1] % 2:
        out[:, -1] = p.inverse(p.forward(a[:, -1].astype(np.complex128)) * filt).real
    return out


def pair_filter(p_, q_, filt):
    """fft.py:261-271."""
    pl = plan(p_.shape[0])
    z = pl.inverse(pl.forward(p_ + 1j * q_) * filt[:, None])
    return z.real, z.imag


def pair_filter_2d(p_, q_, filt2d):
    """fft.py:274-280."""
    z = fft2(fft2(p_ + 1j * q_) * filt2d, inverse=True)
    return z.real, z.imag


def wiener_multiplier(hspec, k):
    """deconv.py:253-254."""
    return np.conj(hspec) / (hspec.real ** 2 + hspec.imag ** 2 + k)


def wiener_2d(f: np.ndarray, psf: OPsf, k: float) -> np.ndarray:
    """deconv.py:257-272 (unclamped)."""
    return fft2(fft2(f) * wiener_multiplier(spectrum_2d(psf, f.shape), k), inverse=True).real


def wiener_1d(f: np.ndarray, psf: OPsf, k: float) -> np.ndarray:
    """deconv.py:275-288 (unclamped; horizontal blur via transpose)."""
    a = f if psf.axis == "v" else np.ascontiguousarray(f.T)
    out = column_filter(a, wiener_multiplier(spectrum_1d(psf, a.shape[0]), k))
    return out if psf.axis == "v" else np.ascontiguousarray(out.T)


# --------------------------------------------------------------------------------------
# convolver realisations (deconv.py:295-403)

class SpatialConv:
    """deconv.py:295-307 -- clamped direct summation."""

    def __init__(self, psf):
        self.fwd, self.adj = psf, reflect(psf)

    def blur(self, a):
        return clamped_convolve(a, self.fwd)

    def adjoint(self, a):
        return clamped_convolve(a, self.adj)

    def adjoint_pair(self, p_, q_):
        return self.adjoint(p_), self.adjoint(q_)


class BoxConv:
    """deconv.py:310-326 -- adjoint centre taps-1-c."""

    def __init__(self, length, center, taps, axis=0):
        self.length, self.c, self.ca, self.axis = length, center, taps - 1 - center, axis

    def blur(self, a):
        return box_filter(a, self.length, self.c, self.axis)

    def adjoint(self, a):
        return box_filter(a, self.length, self.ca, self.axis)

    def adjoint_pair(self, p_, q_):
        return self.adjoint(p_), self.adjoint(q_)


class Fourier1DConv:
    """deconv.py:329-356."""

    def __init__(self, spec, axis=0):
        self.spec, self.conj, self.axis = spec, np.conj(spec), axis

    def _apply(self, a, filt):
        if self.axis == 0:
            return column_filter(a, filt)
        return np.ascontiguousarray(column_filter(np.ascontiguousarray(a.T), filt).T)

    def blur(self, a):
        return self._apply(a, self.spec)

    def adjoint(self, a):
        return self._apply(a, self.conj)

    def adjoint_pair(self, p_, q_):
        if self.axis == 0:
            return pair_filter(p_, q_, self.conj)
        rp, rq = pair_filter(np.ascontiguousarray(p_.T), np.ascontiguousarray(q_.T), self.conj)
        return np.ascontiguousarray(rp.T), np.ascontiguousarray(rq.T)


class Fourier2DConv:
    """deconv.py:359-376."""

    def __init__(self, spec):
        self.spec, self.conj = spec, np.conj(spec)

    def _apply(self, a, filt):
        return fft2(fft2(a) * filt, inverse=True).real

    def blur(self, a):
        return self._apply(a, self.spec)

    def adjoint(self, a):
        return self._apply(a, self.conj)

    def adjoint_pair(self, p_, q_):
        return pair_filter_2d(p_, q_, self.conj)


def make_convolver(psf: OPsf, shape, mode=None):
    """deconv.py:379-403."""
    if mode is None:
        mode = "box" if psf.kind == "box" else "spatial"
    if mode == "spatial":
        return SpatialConv(psf)
    if mode == "box":
        if psf.kind != "box":
            raise ValueError("box convolver requires a uniform-box PSF")
        return BoxConv(psf.length, psf.center, psf.weights.shape[0], 0 if psf.axis == "v" else 1)
    if mode == "fourier2d" or (mode == "fourier" and psf.kind == "2d"):
        return Fourier2DConv(spectrum_2d(psf, shape))
    if mode == "fourier":
        ax = 0 if psf.axis == "v" else 1
        return Fourier1DConv(spectrum_1d(psf, shape[ax]), ax)
    raise ValueError(f"unknown convolver mode {mode!r}")


# --------------------------------------------------------------------------------------
# RL / RRRL steps (deconv.py:415-559)

def blur_guarded(u, conv):
    """deconv.py:415-418."""
    return np.maximum(conv.blur(u), GUARD)


def combine(u, f, b, weight, diff, alpha, conv):
    """deconv.py:421-446."""
    ratio = f / b
    if weight is None:
        num, den = conv.adjoint(ratio), None
    else:
        ratio *= weight
        num, den = conv.adjoint_pair(ratio, weight)
    if diff is not None and alpha != 0.0:
        pos = np.maximum(diff, 0.0)
        pos *= alpha
        num += pos
        neg = np.minimum(diff, 0.0)
        neg *= alpha
        if den is None:
            den = 1.0 - neg
        else:
            den -= neg
    if den is None:
        return u * num
    np.maximum(den, GUARD, out=den)
    out = u * num
    out /= den
    return out


def rrrl_iteration(u, fpos, conv, params: OParams, lut=None, robust=True):
    """deconv.py:512-521."""
    b = blur_guarded(u, conv)
    w = robust_weight(fpos, b, params.eps_data, params.floor, lut, floored=True) if robust else None
    d = diffusion(u, params.eps_reg) if params.alpha > 0.0 else None
    return combine(u, fpos, b, w, d, params.alpha, conv)


def rl_step(u, f, conv):
    """deconv.py:449-460."""
    return combine(u, f, blur_guarded(u, conv), None, None, 0.0, conv)


def prepare_state(u, f, conv, params: OParams, robust=True, lut=None):
    """deconv.py:477-496 -> (blurred, weight|None, diffusion|None)."""
    b = blur_guarded(u, conv)
    w = robust_weight(f, b, params.eps_data, params.floor, lut) if robust else None
    d = diffusion(u, params.eps_reg) if params.alpha > 0.0 else None
    return b, w, d


def rrrl_step(u, f, state, conv, params: OParams):
    """deconv.py:499-509."""
    b, w, d = state
    return combine(u, f, b, w, d, params.alpha, conv)


def rl_deblur(f, psf: OPsf, iterations: int, mode=None, floor=0.1):
    """deconv.py:524-534."""
    conv = make_convolver(psf, f.shape, mode)
    fpos = np.maximum(f, floor)
    u = fpos.copy()
    for _ in range(iterations):
        u = rl_step(u, fpos, conv)
    return u


def rrrl_deblur(f, psf: OPsf, params: OParams, mode=None, lut=None):
    """deconv.py:537-559 -- horizontal 1D kernels run transposed."""
    tr = psf.axis == "h"
    a = np.ascontiguousarray(f.T) if tr else f
    p = as_vertical(psf) if tr else psf
    conv = make_convolver(p, a.shape, mode)
    fpos = np.maximum(a, params.floor)
    u = fpos.copy()
    for _ in range(params.iterations):
        u = rrrl_iteration(u, fpos, conv, params, lut)
    return np.ascontiguousarray(u.T) if tr else u


# --------------------------------------------------------------------------------------
# the combined pipeline (deconv.py:566-703)

def default_scenario(psf: OPsf) -> str:
    """deconv.py:574-579."""
    return {"box": "box", "1d": "fourier1d"}.get(psf.kind, "fourier2d")


def pipeline(f: np.ndarray, psf: OPsf, params: OParams, scenario: str | None = None,
             lut=None) -> np.ndarray:
    """DeblurPipeline.run (deconv.py:611-693) in one function: Wiener on the raw
    observation, clamp, then ``iterations`` RRRL steps with the scenario's convolver
    (box: clamped sliding window; fourier1d: per-column FFT; fourier2d: 2D FFT)."""
    scenario = default_scenario(psf) if scenario is None else scenario
    if scenario in ("box", "fourier1d") and psf.kind == "2d":
        raise ValueError(f"{scenario} requires a 1D PSF")
    if scenario == "box" and psf.kind != "box":
        raise ValueError("box scenario requires a uniform-box PSF")
    tr = scenario != "fourier2d" and psf.axis == "h"
    a = np.ascontiguousarray(f.T) if tr else np.asarray(f, dtype=np.float64)
    p = as_vertical(psf) if tr else psf
    if scenario == "fourier2d":
        hspec = spectrum_2d(p, a.shape)
        wien = fft2(fft2(a) * wiener_multiplier(hspec, params.wiener_k), inverse=True).real
        conv = Fourier2DConv(hspec)
    else:
        hspec = spectrum_1d(p, a.shape[0])
        wien = column_filter(a, wiener_multiplier(hspec, params.wiener_k))
        conv = (BoxConv(p.length, p.center, p.weights.shape[0]) if scenario == "box"
                else Fourier1DConv(hspec))
    u = np.maximum(wien, params.floor)
    fpos = np.maximum(a, params.floor)
    for _ in range(params.iterations):
        u = rrrl_iteration(u, fpos, conv, params, lut)
    return np.ascontiguousarray(u.T) if tr else u


def psnr(u: np.ndarray, g: np.ndarray) -> float:
    """Harness metric of SURVEY.md section 8(d): 10 log10(255^2 / MSE)."""
    mse = float(np.mean((np.asarray(u) - np.asarray(g)) ** 2))
    return math.inf if mse == 0.0 else 10.0 * math.log10(255.0 ** 2 / mse)
