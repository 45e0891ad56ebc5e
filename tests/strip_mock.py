"""CPU stand-in for paper_1409_7474_b200.strips.DeviceStrip -- TEST ONLY.

Implements the same phase interface (update / row / partition / finalize ...)
with the numpy oracle's arithmetic (oracle/lse_oracle.py) on one strip's rows,
so the strip driver and the communicators (LocalComm, DistComm over gloo) can
be exercised without a GPU.  State: b (+1/-1) of the local rows, padded to
whole word-rows; partials: the device's 64-byte layout with absolute sums.
"""
from __future__ import annotations

import contextlib
from types import SimpleNamespace

import numpy as np
import torch

import lse_oracle as O
from paper_1409_7474_b200.strips import PARTIAL_BYTES, WORD_ROWS


def _pack(a, b, na, nb, mism):
    buf = np.zeros(8, dtype=np.float64)
    buf[0], buf[2] = a, b
    ints = buf.view(np.int64)
    ints[4], ints[5], ints[6] = na, nb, mism
    return torch.from_numpy(buf.view(np.uint8).copy())


def _unpack(raw):
    q = np.ascontiguousarray(raw.numpy()).view(np.uint8).reshape(-1, PARTIAL_BYTES)
    f = q.copy().view(np.float64)
    i = q.copy().view(np.int64)
    return f[:, 0], f[:, 2], i[:, 4], i[:, 5], i[:, 6]


class MockStrip:
    def __init__(self, image_rows, win, seeds, params):
        self.win = win
        self.p = params
        self.inside_positive = int(seeds.inside_sign) > 0
        self.comm_device = torch.device("cpu")
        self.img = np.asarray(image_rows, dtype=np.float64)
        hr = (win.rows + WORD_ROWS - 1) // WORD_ROWS
        self.b = np.zeros((hr * WORD_ROWS, win.width), dtype=np.int32)
        inside = np.zeros((win.height, win.width), dtype=bool)
        for q in seeds.polygons:        # the strip sees only its rows; the count is global
            inside |= O.polygon_mask(np.asarray(q, dtype=np.float64), win.width, win.height)
        sgn = 1 if self.inside_positive else -1
        self.b[:win.rows] = np.where(inside[win.y_lo:win.y_hi], sgn, -sgn)
        self.w = O.gaussian_weights(params.sigma2, params.ts_reg)
        mp = params.model_params
        self.model = params.model.value
        self.g = (O.edge_function(self.img, mp.sigma1, mp.ts_pre, mp.edge_gain)
                  if self.model == "edge" else None)
        y0, y1 = win.own_rows
        self.own = slice(y0 - win.y_lo, y1 - win.y_lo)
        self.iteration = 0
        self.stop = False
        self.converged = False
        self.degenerate = False
        self.n_ckpt = 0
        self.equal_run = 0
        self.M = None
        self.coef = None
        self.need = False

    # communicator hooks
    def stream_context(self):
        return contextlib.nullcontext()

    def synchronize(self):
        pass

    def row(self, wr):
        return torch.from_numpy(self.b[wr * WORD_ROWS:(wr + 1) * WORD_ROWS])

    def image_range(self):
        return float(self.img.min()), float(self.img.max()), float(np.abs(self.img).max())

    def set_image_range(self, g):
        self.rng = g

    # phases
    def _phi(self):
        b = self.b[:self.win.rows].astype(np.float64)
        if self.iteration == 0:            # phi^0 is the rasterized +-1 field
            return b
        return O.convolve_same(b, self.w)

    def _sums(self, phi):
        own = phi[self.own]
        pos = own >= 0.0
        img = self.img[self.own]
        return _pack(float(img[pos].sum()), float(img[~pos].sum()), int(pos.sum()),
                     int((~pos).sum()), 0)

    def prepare(self):
        pos = self.b[:self.win.rows][self.own] > 0
        img = self.img[self.own]
        return _pack(float(img[pos].sum()), float(img[~pos].sum()), int(pos.sum()),
                     int((~pos).sum()), 0)

    def update(self):
        it = self.iteration + 1
        ckpt = it % self.p.conv_check_every == 0
        self.need = self.model != "edge" or ckpt
        self.ckpt = ckpt
        self.iteration = it
        if self.stop:
            return self.need
        self.iteration = it - 1
        phi = self._phi()
        self.iteration = it
        h = O.gradient_magnitude(phi)
        if self.model == "edge":
            v = self.g * h
        elif self.coef is None:
            v = np.zeros_like(phi)
            self.degenerate = True
        else:
            cp, cm = self.coef
            mn, mx, _ = self.rng
            if self.model == "zhang":
                m = 0.5 * (cp + cm)
                peak = max(abs(mx - m), abs(mn - m))
                data = self.p.model_params.nu * ((self.img - m) / peak) if peak else None
            else:
                D = lambda i: (cp - cm) * (2.0 * i - cp - cm)   # noqa: E731
                peak = max(abs(D(mx)), abs(D(mn)))
                data = D(self.img) / peak if peak else None
            if data is None:
                v = np.zeros_like(phi)
                self.degenerate = True
            else:
                v = data * h
        u = phi + self.p.dt * v
        self.b[:self.win.rows] = np.where(u > 0.0, 1, -1)
        return self.need

    def partition(self):
        if self.stop:
            return _pack(0.0, 0.0, 0, 0, 0)
        phi = self._phi()
        part = self._sums(phi)
        if self.ckpt:
            m = phi[self.own] > 0.0
            mism = 0 if self.M is None else int((m != self.M).sum())
            self.M = m
            q = part.numpy().view(np.int64)
            q[6] = mism
        return part

    # the one-pass protocol (lse_strip_fused): the partition of the current
    # state now, the update once the gathered partials fixed the coefficients
    # -- the device's speculative pass + fix / redo produce exactly that
    supports_fused = True

    def fused(self):
        part = self.partition()
        self._pending_update = True
        return part

    def finalize(self, gathered, absolute):
        self._finalize(gathered, absolute)
        if getattr(self, "_pending_update", False) and not absolute:
            self._pending_update = False
            self.update()

    def _finalize(self, gathered, absolute):
        if self.stop and not absolute:
            return
        a, b, na, nb, mism = _unpack(gathered)
        npos, nneg = int(na.sum()), int(nb.sum())
        # fixed rank order, as the device finalize
        sp = 0.0
        sn = 0.0
        for k in range(len(a)):
            sp += a[k]
            sn += b[k]
        self.coef = None if (npos == 0 or nneg == 0) else (sp / npos, sn / nneg)
        if absolute or not self.ckpt:
            return
        tot = int(mism.sum())
        if self.n_ckpt >= 1 and tot == 0:
            self.equal_run += 1
        else:
            self.equal_run = 0
        self.n_ckpt += 1
        if self.n_ckpt >= self.p.conv_window and self.equal_run >= self.p.conv_window - 1:
            self.converged = True
            self.stop = True
            self.conv_iter = self.iteration

    def sync(self):
        it = self.conv_iter if self.converged else self.iteration
        return SimpleNamespace(iteration=it, converged=int(self.converged),
                               degenerate=int(self.degenerate))

    def own_phi(self):
        return self._phi()[self.own]
