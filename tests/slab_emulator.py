"""CPU emulation of the slab pass kernels (TEST INFRASTRUCTURE ONLY).

Implements, in numpy, what each ctap pass does to one rank's buffers in the
slab decomposition (layouts as in csrc/ctap_passes.cu), using the oracle's
phase factors, so the distributed schedule of paper_1309_2451_b200.slab can
be run under gloo on CPU and compared with the single-process oracle.
"""

import numpy as np
import scipy.fft as sfft

from paper_1309_2451_b200 import _lib


class EmulatedRank:
    def __init__(self, layout, factors):
        self.L = layout
        self.f = factors   # oracle Factors on the GLOBAL grid

    def run_pass(self, kind, src, dst):
        L = self.L
        nx, ny, nz = L.n
        nxl, nyl, P = L.nx_local, L.ny_local, L.P
        xs, ys = L.x_slice, L.y_slice
        if kind in (_lib.PASS_Z_FIRST, _lib.PASS_Z_MID, _lib.PASS_Z_LAST):
            a = src.reshape(nxl, ny, nz)
            if kind == _lib.PASS_Z_FIRST:
                a = sfft.fft(a * self.f.exp_v_half[xs], axis=2)
            elif kind == _lib.PASS_Z_MID:
                a = sfft.fft(sfft.ifft(a, axis=2) * self.f.exp_v_full[xs], axis=2)
            else:
                a = sfft.ifft(a, axis=2) * self.f.exp_v_half[xs]
            dst[:] = a.reshape(-1)
        elif kind == _lib.PASS_Y_FWD_TO_PEER:
            a = sfft.fft(src.reshape(nxl, ny, nz), axis=1)
            dst[:] = a.reshape(nxl, P, nyl, nz).transpose(1, 0, 2, 3).reshape(-1)
        elif kind == _lib.PASS_X_KIN:
            a = src.reshape(nx, nyl, nz)
            a = sfft.ifft(sfft.fft(a, axis=0) * self.f.exp_k[:, ys, :], axis=0)
            dst[:] = a.reshape(-1)
        elif kind == _lib.PASS_Y_INV_FROM_PEER:
            a = src.reshape(P, nxl, nyl, nz).transpose(1, 0, 2, 3).reshape(nxl, ny, nz)
            dst[:] = sfft.ifft(a, axis=1).reshape(-1)
        else:
            raise ValueError(kind)
