"""TEST INFRASTRUCTURE: a NumPy stand-in for CudaSlabBackend (paper_1212_2245_b200/slab.py).

It computes each rank's share of the Wiener step and of one RRRL iteration in float64 NumPy,
following the reference algorithm (deconv.py:142-213, 253-254, 359-376, 421-446; the divergence
table via oracle/wr3l_oracle.r1), so the slab driver's communication logic (halo depth, periodic
neighbours, global Neumann rows, the two all-to-all transposes) can be checked on CPU with a
gloo process group against the oracle's whole-image pipeline.
"""

from __future__ import annotations

import numpy as np

from oracle import wr3l_oracle as O


def taps_of(weights: np.ndarray, center):
    sy, sx = weights.shape
    cy, cx = center
    blur, adj = [], []
    for jy in range(sy):
        for jx in range(sx):
            w = float(weights[jy, jx])
            if w != 0.0:
                blur.append((cy - jy, cx - jx, w))
                adj.append((jy - cy, jx - cx, w))
    return blur, adj


def extent(taps):
    dys = [t[0] for t in taps]
    return max(0, -min(dys)), max(0, max(dys))


class NumpySlabBackend:
    def __init__(self, weights, center, params: O.OParams, H: int, W: int):
        self.params, self.H, self.W = params, H, W
        self.blur, self.adj = taps_of(np.asarray(weights), center)
        bt, bb = extent(self.blur)
        at, ab = extent(self.adj)
        self.at, self.ab = at, ab
        self.halo = (max(at + bt, 2), max(ab + bb, 2))
        emb = O.embed_2d(O.OPsf("2d", np.asarray(weights), tuple(center)), (H, W))
        hs = np.fft.fft2(emb)
        self.M = np.conj(hs) / (hs.real ** 2 + hs.imag ** 2 + params.wiener_k)
        self.Mb = None

    def halo_rows(self):
        return self.halo

    def prepare(self, geo):
        self.Mb = self.M[:, geo.rank * geo.Wb:(geo.rank + 1) * geo.Wb]

    @staticmethod
    def _c(t):
        a = t.numpy()
        return a[..., 0] + 1j * a[..., 1]

    @staticmethod
    def _put(t, c):
        a = t.numpy()
        a[..., 0] = c.real
        a[..., 1] = c.imag

    def rows_fft(self, z, real_in, rows, inv, scale=1.0):
        if not inv:
            self._put(z, np.fft.fft(real_in.numpy(), axis=1))
        else:
            self._put(z, np.fft.ifft(self._c(z), axis=1) * self.W * scale)

    def cols_filter(self, zc, cols):
        c = np.fft.fft(self._c(zc), axis=0) * self.Mb
        self._put(zc, np.fft.ifft(c, axis=0) * self.H)

    def epilogue(self, z, f, u0, fpos, rows):
        u0.numpy()[:] = np.maximum(self._c(z).real / (self.H * self.W), self.params.floor)
        fpos.numpy()[:] = np.maximum(f.numpy(), self.params.floor)

    def _conv(self, src, taps, r0, r1):
        out = np.zeros((r1 - r0, src.shape[1]))
        for dy, dx, w in taps:
            out += w * np.roll(src[r0 + dy:r1 + dy], -dx, axis=1)
        return out

    def iterate(self, u_ext, fpos_ext, p_ext, w_ext, out_ext, geo):
        P = self.params
        u, fp, pp, ww, out = (t.numpy() for t in (u_ext, fpos_ext, p_ext, w_ext, out_ext))
        T, S = geo.top, geo.S
        a0, a1 = T - self.at, T + S + self.ab
        b = np.maximum(self._conv(u, self.blur, a0, a1), O.GUARD)
        fa = fp[a0:a1]
        wv = O.robust_weight(fa, b, P.eps_data, P.floor, floored=True)
        ww[a0:a1] = wv
        pp[a0:a1] = wv * (fa / b)
        num = self._conv(pp, self.adj, T, T + S)
        den = self._conv(ww, self.adj, T, T + S)
        # TV divergence on own rows; rows outside the global image are absent (Neumann)
        U = u[T - 2:T + S + 2]
        gidx = geo.row0 - 2 + np.arange(S + 4)
        valid = (gidx >= 0) & (gidx < geo.H)
        gx = np.diff(U, axis=1)
        gy = np.diff(U, axis=0)
        gy[~(valid[1:] & valid[:-1])] = 0.0
        q = np.zeros_like(U)
        q[:, :-1] += gx * gx
        q[:, 1:] += gx * gx
        q[:-1] += gy * gy
        q[1:] += gy * gy
        g = 0.5 / np.sqrt(0.5 * q + P.eps_reg ** 2)
        d = np.zeros_like(U)
        fx = (g[:, :-1] + g[:, 1:]) * gx
        d[:, :-1] += fx
        d[:, 1:] -= fx
        fy = (g[:-1] + g[1:]) * gy
        d[:-1] += fy
        d[1:] -= fy
        D = d[2:2 + S]
        nm = num + P.alpha * np.maximum(D, 0.0)
        dn = np.maximum(den - P.alpha * np.minimum(D, 0.0), O.GUARD)
        out[T:T + S] = u[T:T + S] * nm / dn
