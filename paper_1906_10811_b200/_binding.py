"""ctypes binding of libaw (include/aw.h) -- argument marshalling only.

Every function of the C ABI is exposed under the same name; ``Grid`` is a
thin owner of an ``aw_grid*`` that converts numpy arrays / torch tensors to
plain pointers.  There is no CPU fallback: importing this module without the
built ``libaw.so`` raises, and creating a grid without a CUDA device raises
``AwError(AW_ECUDA)``.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# AW_LIBRARY: development knob for same-box A/B runs of two builds (tools/ab_stream.py); the default
# and everything the tests, bench and smoke() load is the in-tree libaw.so
LIB_PATH = os.environ.get("AW_LIBRARY") or os.path.join(_HERE, "libaw.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -m paper_1906_10811_b200.build` "
        "(libaw has no CPU fallback)")

_lib = ctypes.CDLL(LIB_PATH)

# --- constants (include/aw.h) ---
AW_OK, AW_EINVAL, AW_ENOMEM, AW_ECUDA, AW_ENCCL, AW_ESTATE, AW_EUNSUPPORTED, AW_ENONFINITE = 0, -1, -2, -3, -4, -5, -6, -7
AW_GLOBAL, AW_LOCAL = 0, 1
AW_KERNEL_AUTO, AW_KERNEL_V1, AW_KERNEL_STREAM, AW_KERNEL_TILE2D = 0, 1, 2, 3
AW_OPT_KERNEL, AW_OPT_TIMING, AW_OPT_GRAPH_STEPS, AW_OPT_CHECK_FINITE, AW_OPT_CHECKPOINT_STEPS = 1, 2, 3, 4, 5
AW_OPT_TEMPORAL, AW_OPT_FWI_ACCUMULATE = 6, 7
AW_OPT_RESIDENT = 8
AW_RESIDENT_OFF, AW_RESIDENT_ON, AW_RESIDENT_AUTO = 0, 1, 2
AW_DIST_WORKSPACE = 1
STATUS_NAMES = {0: "AW_OK", -1: "AW_EINVAL", -2: "AW_ENOMEM", -3: "AW_ECUDA", -4: "AW_ENCCL",
                -5: "AW_ESTATE", -6: "AW_EUNSUPPORTED", -7: "AW_ENONFINITE"}


class aw_dist(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int), ("world", ctypes.c_int), ("device", ctypes.c_int),
                ("stream", ctypes.c_void_p), ("flags", ctypes.c_uint)]


class aw_run_stats(ctypes.Structure):
    _fields_ = [("ms_total", ctypes.c_double), ("ms_stencil", ctypes.c_double), ("n_stencil", ctypes.c_int64),
                ("launches", ctypes.c_int64), ("gpts", ctypes.c_double), ("points", ctypes.c_int64),
                ("kernel", ctypes.c_int), ("eta_tiles", ctypes.c_int), ("launches_total", ctypes.c_int64),
                ("fwi_steps", ctypes.c_int64), ("fwi_checkpoint", ctypes.c_int), ("timed_launches", ctypes.c_int64),
                ("ms_exchange", ctypes.c_double), ("exchange_waits", ctypes.c_int64),
                ("lib_device_bytes", ctypes.c_int64), ("workspace_bytes", ctypes.c_int64),
                ("resident", ctypes.c_int32)]


_P = ctypes.c_void_p
_I = ctypes.c_int
_I64 = ctypes.c_int64
_D = ctypes.c_double
_S = ctypes.c_int  # aw_status

_SIGS = {
    "aw_grid_create": (_S, [ctypes.POINTER(_P), _I, _P, _P, _P, _I, ctypes.POINTER(aw_dist)]),
    "aw_grid_destroy": (None, [_P]),
    "aw_local_extent": (_S, [_P, ctypes.POINTER(_I64), ctypes.POINTER(_I64)]),
    "aw_workspace_bytes": (ctypes.c_size_t, [_P]),
    "aw_bind_workspace": (_S, [_P, _P, ctypes.c_size_t]),
    "aw_set_model": (_S, [_P, _P, _P, _I]),
    "aw_add_sources": (_S, [_P, _I, _P, _I, _P]),
    "aw_add_receivers": (_S, [_P, _I, _P, _I]),
    "aw_set_wavefield": (_S, [_P, _P, _P, _I]),
    "aw_run": (_S, [_P, _I, _D]),
    "aw_reset": (_S, [_P]),
    "aw_steps_done": (_I64, [_P]),
    "aw_read_wavefield": (_S, [_P, _I, _P, _I]),
    "aw_read_receivers": (_S, [_P, _P]),
    "aw_debug_sparse": (_S, [_P, _I, _P, _P]),
    "aw_last_run_stats": (_S, [_P, ctypes.POINTER(aw_run_stats)]),
    "aw_set_option": (_S, [_P, _I, _I64]),
    "aw_critical_dt": (_D, [_I, _P, _I, _D]),
    "aw_last_error": (ctypes.c_char_p, []),
    "aw_abi_version": (_I, []),
    "aw_slab_partition": (_S, [_I64, _I, _I, _I, ctypes.POINTER(_I64), ctypes.POINTER(_I64)]),
    "aw_team_export_size": (ctypes.c_size_t, []),
    "aw_team_export": (_S, [_P, _P]),
    "aw_team_connect": (_S, [_P, _P]),
    "aw_team_connect_local": (_S, [ctypes.POINTER(_P), _I]),
    "aw_team_run": (_S, [ctypes.POINTER(_P), _I, _I, _D]),
    # NEXT-3: adjoint-state FWI gradient
    "aw_fwi_gradient": (_S, [_P, _I, _D, _P, _P, _I, _P, ctypes.POINTER(_D)]),
    # NEXT-2: the paper's diffusion operator
    "aw_diffusion_create": (_S, [ctypes.POINTER(_P), _I, _P, _P, _I, _D, _P]),
    "aw_diffusion_set": (_S, [_P, _P]),
    "aw_diffusion_run": (_S, [_P, _I, _D]),
    "aw_diffusion_read": (_S, [_P, _P]),
    "aw_diffusion_stats": (_S, [_P, ctypes.POINTER(aw_run_stats)]),
    "aw_diffusion_set_option": (_S, [_P, _I, _I64]),
    "aw_diffusion_destroy": (None, [_P]),
}
EXPORTED = tuple(_SIGS)

for _name, (_res, _args) in _SIGS.items():
    if os.environ.get("AW_LIBRARY") and not hasattr(_lib, _name):
        continue  # an older build under A/B measurement (tools/ab_stream.py) may lack newer calls
    _fn = getattr(_lib, _name)
    _fn.restype = _res
    _fn.argtypes = _args
    globals()[_name] = _fn


class AwError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


def check(status: int) -> int:
    if status != AW_OK:
        raise AwError(status, aw_last_error().decode(errors="replace"))
    return status


# --- array marshalling -------------------------------------------------------
def _ptr(a, dtype=np.float32, keep=None):
    """Pointer to the data of a numpy array / torch tensor (host or device) or None."""
    if a is None:
        return None
    if isinstance(a, int):
        return a
    if hasattr(a, "data_ptr"):  # torch.Tensor
        import torch
        want = {np.float32: torch.float32, np.float64: torch.float64}[dtype]
        if a.dtype != want or not a.is_contiguous():
            raise TypeError(f"tensor must be contiguous {want}")
        return a.data_ptr()
    arr = np.ascontiguousarray(a, dtype=dtype)
    if keep is not None:
        keep.append(arr)
    return arr.ctypes.data


def _out_ptr(a):
    """Pointer to a caller-provided OUTPUT buffer: it must already be C-contiguous float32 (the C side
    writes into it), so no temporary copy is ever made."""
    if hasattr(a, "data_ptr"):  # torch.Tensor
        import torch
        if a.dtype != torch.float32 or not a.is_contiguous():
            raise TypeError("output tensor must be a contiguous torch.float32 tensor")
        return a.data_ptr()
    if not isinstance(a, np.ndarray) or a.dtype != np.float32 or not a.flags["C_CONTIGUOUS"] \
            or not a.flags["WRITEABLE"]:
        raise TypeError("output array must be a writeable C-contiguous numpy.float32 array")
    return a.ctypes.data


def _torch_stream_handle(stream):
    """cudaStream_t for a torch stream; the legacy default stream maps to cudaStreamLegacy (0x1)."""
    h = stream.cuda_stream
    return h if h != 0 else 1


class Grid:
    """Owner of one ``aw_grid*`` (one slab / one GPU)."""

    def __init__(self, shape, extent, space_order, origin=None, *, rank=0, world=1, device=None, stream=None,
                 workspace=None):
        """workspace: None = the library allocates the grid arrays; "defer" = allocate nothing now
        (AW_DIST_WORKSPACE; call bind_workspace before set_model/run); a torch uint8 CUDA tensor =
        bind it right away (torch owns the device memory, include/aw.h aw_bind_workspace)."""
        self.ndim = len(shape)
        self.shape = tuple(int(s) for s in shape)
        sh = (ctypes.c_int64 * self.ndim)(*self.shape)
        ex = (ctypes.c_double * self.ndim)(*[float(e) for e in extent])
        org = None if origin is None else (ctypes.c_double * self.ndim)(*[float(o) for o in origin])
        if stream is not None and not isinstance(stream, int):
            stream = _torch_stream_handle(stream)
        flags = 0 if workspace is None else AW_DIST_WORKSPACE
        dist = aw_dist(rank, world, -1 if device is None else int(device), stream, flags)
        h = _P()
        check(aw_grid_create(ctypes.byref(h), self.ndim, ctypes.cast(sh, _P), ctypes.cast(ex, _P),
                             None if org is None else ctypes.cast(org, _P), int(space_order), ctypes.byref(dist)))
        self.handle = h
        self.space_order = space_order
        self.rank, self.world = rank, world
        z0, nz = _I64(), _I64()
        check(aw_local_extent(h, ctypes.byref(z0), ctypes.byref(nz)))
        self.z0, self.nz = z0.value, nz.value
        self.nr = 0
        self.ns = 0
        self.device = device
        self._ws = None
        if workspace is not None and not isinstance(workspace, str):
            self.bind_workspace(workspace)
        elif workspace not in (None, "defer"):
            raise ValueError("workspace must be None, 'defer' or a torch uint8 CUDA tensor")

    def workspace_bytes(self) -> int:
        """Bytes a caller workspace needs now (grid arrays + current sparse arenas)."""
        return int(aw_workspace_bytes(self.handle))

    def bind_workspace(self, ws=None, extra: int = 0):
        """Bind a torch uint8 CUDA tensor as the grid's device memory (allocated here with
        workspace_bytes() + extra bytes when ws is None).  The tensor is kept alive by the Grid."""
        import torch
        if ws is None:
            dev = torch.device("cuda", torch.cuda.current_device() if self.device is None else int(self.device))
            ws = torch.empty(self.workspace_bytes() + int(extra), dtype=torch.uint8, device=dev)
        if not (hasattr(ws, "data_ptr") and ws.dtype == torch.uint8 and ws.is_cuda and ws.is_contiguous()):
            raise TypeError("workspace must be a contiguous torch.uint8 CUDA tensor")
        check(aw_bind_workspace(self.handle, ws.data_ptr(), ws.numel()))
        self._ws = ws
        return ws

    # lifecycle
    def close(self):
        if getattr(self, "handle", None):
            aw_grid_destroy(self.handle)
            self.handle = None
        self._ws = None  # the library no longer references the workspace

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    @property
    def local_shape(self):
        return (self.nz,) + self.shape[1:]

    # calls
    def set_model(self, m, damp=None, layout=AW_GLOBAL):
        keep = []
        check(aw_set_model(self.handle, _ptr(m, keep=keep), _ptr(damp, keep=keep), layout))

    def add_sources(self, coords, wavelet):
        keep = []
        co = np.ascontiguousarray(coords, np.float64).reshape(-1, self.ndim)
        ns = co.shape[0]
        if hasattr(wavelet, "data_ptr"):
            nt_max = wavelet.shape[0]
        else:
            wavelet = np.ascontiguousarray(wavelet, np.float32).reshape(-1, max(ns, 1))
            nt_max = wavelet.shape[0]
        check(aw_add_sources(self.handle, ns, co.ctypes.data if ns else None, nt_max if ns else 0,
                             _ptr(wavelet, keep=keep) if ns else None))
        self.ns = ns

    def add_receivers(self, coords, nt_max):
        co = np.ascontiguousarray(coords, np.float64).reshape(-1, self.ndim)
        nr = co.shape[0]
        check(aw_add_receivers(self.handle, nr, co.ctypes.data if nr else None, int(nt_max) if nr else 0))
        self.nr = nr

    def set_wavefield(self, u_cur=None, u_prev=None, layout=AW_GLOBAL):
        keep = []
        check(aw_set_wavefield(self.handle, _ptr(u_cur, keep=keep), _ptr(u_prev, keep=keep), layout))

    def run(self, nt, dt):
        check(aw_run(self.handle, int(nt), float(dt)))

    def reset(self):
        check(aw_reset(self.handle))

    @property
    def steps_done(self):
        return int(aw_steps_done(self.handle))

    def read_wavefield(self, which=0, out=None, layout=AW_GLOBAL):
        if out is None:
            shp = self.shape if layout == AW_GLOBAL else self.local_shape
            out = np.zeros(shp, np.float32)
        check(aw_read_wavefield(self.handle, which, _out_ptr(out), layout))
        return out

    def read_receivers(self, out=None):
        if out is None:
            out = np.zeros((self.steps_done, self.nr), np.float32)
        if self.nr and self.steps_done:
            check(aw_read_receivers(self.handle, _out_ptr(out)))
        return out

    def debug_sparse(self, which):
        n = self.ns if which == 0 else self.nr
        nc = 1 << self.ndim
        corner = np.zeros((n, nc), np.int64)
        w = np.zeros((n, nc), np.float32)
        check(aw_debug_sparse(self.handle, which, corner.ctypes.data, w.ctypes.data))
        return corner, w

    def stats(self) -> dict:
        st = aw_run_stats()
        check(aw_last_run_stats(self.handle, ctypes.byref(st)))
        return {f: getattr(st, f) for f, _ in aw_run_stats._fields_}

    def set_option(self, option, value):
        check(aw_set_option(self.handle, int(option), int(value)))

    def fwi_gradient(self, nt, dt, d_obs, grad=None, residual=None, layout=AW_GLOBAL, want_residual=True):
        """NEXT-3: (grad, residual, J) of J = 1/2 sum (rec - d_obs)^2 (include/aw.h aw_fwi_gradient)."""
        keep = []
        if grad is None:
            grad = np.zeros(self.shape if layout == AW_GLOBAL else self.local_shape, np.float32)
        if residual is None and want_residual:
            residual = np.zeros((int(nt), self.nr), np.float32)
        J = _D(0.0)
        check(aw_fwi_gradient(self.handle, int(nt), float(dt), _ptr(d_obs, keep=keep), _out_ptr(grad), layout,
                              None if residual is None else _out_ptr(residual), ctypes.byref(J)))
        return grad, residual, J.value

    # team plumbing
    def team_export(self) -> bytes:
        n = aw_team_export_size()
        buf = (ctypes.c_char * n)()
        check(aw_team_export(self.handle, ctypes.cast(buf, _P)))
        return bytes(buf)

    def team_connect(self, all_records: bytes):
        buf = ctypes.create_string_buffer(all_records, len(all_records))
        check(aw_team_connect(self.handle, ctypes.cast(buf, _P)))


def critical_dt(spacing, space_order, vmax):
    sp = (ctypes.c_double * len(spacing))(*[float(s) for s in spacing])
    return aw_critical_dt(len(spacing), ctypes.cast(sp, _P), int(space_order), float(vmax))


def slab_partition(n0, world, rank, radius):
    """(z0, nz): the planes of axis 0 rank `rank` of `world` owns (host-only C call)."""
    z0, nz = _I64(), _I64()
    check(aw_slab_partition(int(n0), int(world), int(rank), int(radius), ctypes.byref(z0), ctypes.byref(nz)))
    return z0.value, nz.value


def team_connect_local(grids):
    arr = (_P * len(grids))(*[g.handle for g in grids])
    check(aw_team_connect_local(arr, len(grids)))


def team_run(grids, nt, dt):
    arr = (_P * len(grids))(*[g.handle for g in grids])
    check(aw_team_run(arr, len(grids), int(nt), float(dt)))
