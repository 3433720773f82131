"""CPU emulation of the pencil pass kernels (TEST INFRASTRUCTURE ONLY).

Implements, in numpy, what each pencil ctap pass (PASS_PZ_*, PASS_PY_*,
PASS_PX_KIN; layouts in include/ctap.h and csrc/ctap_passes.cu) does to one
rank's buffers, with the oracle's phase factors, so the distributed schedule
of paper_1309_2451_b200.pencil runs under gloo on CPU against the oracle.
"""

import numpy as np
import scipy.fft as sfft

from paper_1309_2451_b200 import _lib


class EmulatedPencilRank:
    def __init__(self, layout, factors):
        self.L = layout
        self.f = factors  # oracle Factors on the GLOBAL grid

    # natural (xa, yb, nz) <-> z-chunked [b'][x][y][z']
    def _to_zc(self, a):
        L = self.L
        return a.reshape(L.xa, L.yb, L.Pc, L.zc).transpose(2, 0, 1, 3).reshape(-1)

    def _from_zc(self, buf):
        L = self.L
        return buf.reshape(L.Pc, L.xa, L.yb, L.zc).transpose(1, 2, 0, 3).reshape(L.xa, L.yb, L.n[2])

    def run_pass(self, kind, src, dst):
        L = self.L
        blk = (L.x_slice, L.y_slice)
        if kind == _lib.PASS_PZ_FIRST:
            a = sfft.fft(src.reshape(L.block_shape) * self.f.exp_v_half[blk], axis=2)
            dst[:] = self._to_zc(a)
        elif kind == _lib.PASS_PZ_MID:
            a = sfft.fft(sfft.ifft(self._from_zc(src), axis=2) * self.f.exp_v_full[blk], axis=2)
            dst[:] = self._to_zc(a)
        elif kind == _lib.PASS_PZ_LAST:
            dst[:] = (sfft.ifft(self._from_zc(src), axis=2) * self.f.exp_v_half[blk]).reshape(-1)
        elif kind == _lib.PASS_PY_FWD:   # Yb [b'][x][y'][z'] -> Xp [a'][x][y'][z']
            a = src.reshape(L.Pc, L.xa, L.yb, L.zc).transpose(1, 0, 2, 3).reshape(L.xa, L.n[1], L.zc)
            a = sfft.fft(a, axis=1)
            dst[:] = a.reshape(L.xa, L.Pr, L.yd, L.zc).transpose(1, 0, 2, 3).reshape(-1)
        elif kind == _lib.PASS_PY_INV:   # Xp -> Yb
            a = src.reshape(L.Pr, L.xa, L.yd, L.zc).transpose(1, 0, 2, 3).reshape(L.xa, L.n[1], L.zc)
            a = sfft.ifft(a, axis=1)
            dst[:] = a.reshape(L.xa, L.Pc, L.yb, L.zc).transpose(1, 0, 2, 3).reshape(-1)
        elif kind == _lib.PASS_PX_KIN:   # Xr natural (nx, yd, zc) of y block a, z chunk b
            ys = slice(L.a * L.yd, (L.a + 1) * L.yd)
            zs = slice(L.b * L.zc, (L.b + 1) * L.zc)
            a = src.reshape(L.n[0], L.yd, L.zc)
            dst[:] = sfft.ifft(sfft.fft(a, axis=0) * self.f.exp_k[:, ys, zs], axis=0).reshape(-1)
        else:
            raise ValueError(kind)
