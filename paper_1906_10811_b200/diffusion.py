"""NEXT-2: the paper's own benchmark operator, 2D diffusion
u_t = nu (u_xx + u_yy), forward Euler -- thin owner of an ``aw_diffusion*``
(ctypes marshalling only; the step runs in aw_diffusion.cu)."""
from __future__ import annotations

import ctypes

import numpy as np

from . import _binding as B


class Diffusion:
    def __init__(self, shape, extent, space_order, nu, *, stream=None):
        if len(shape) != 2:
            raise B.AwError(B.AW_EUNSUPPORTED, "diffusion is 2D (PAPER.md:732-736)")
        self.shape = tuple(int(s) for s in shape)
        sh = (ctypes.c_int64 * 2)(*self.shape)
        ex = (ctypes.c_double * 2)(*[float(e) for e in extent])
        if stream is not None and not isinstance(stream, int):
            stream = B._torch_stream_handle(stream)
        h = ctypes.c_void_p()
        B.check(B.aw_diffusion_create(ctypes.byref(h), 2, ctypes.cast(sh, ctypes.c_void_p),
                                      ctypes.cast(ex, ctypes.c_void_p), int(space_order), float(nu), stream))
        self.handle = h

    def close(self):
        if getattr(self, "handle", None):
            B.aw_diffusion_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set(self, u=None):
        keep = []
        B.check(B.aw_diffusion_set(self.handle, B._ptr(u, keep=keep)))

    def run(self, nt, dt):
        B.check(B.aw_diffusion_run(self.handle, int(nt), float(dt)))

    def read(self, out=None):
        if out is None:
            out = np.zeros(self.shape, np.float32)
        B.check(B.aw_diffusion_read(self.handle, B._ptr(out)))
        return out

    def stats(self):
        st = B.aw_run_stats()
        B.check(B.aw_diffusion_stats(self.handle, ctypes.byref(st)))
        return {f: getattr(st, f) for f, _ in B.aw_run_stats._fields_}

    def set_option(self, option, value):
        B.check(B.aw_diffusion_set_option(self.handle, int(option), int(value)))
