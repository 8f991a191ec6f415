"""ctypes binding of include/fabf.h (argument marshalling only).

Names follow the C ABI: ``Plan`` wraps ``fabf_plan``/``fabf_destroy``;
``filter``, ``filter_diag``, ``bounds`` and ``filter_host`` wrap the entry points
of the same names.  Tensors are float32, contiguous; device tensors are passed
by ``data_ptr()`` with ``torch.cuda.current_stream()`` unless a stream is given.
"""
from __future__ import annotations

import ctypes
import os
import threading

_PKG = os.path.dirname(os.path.abspath(__file__))
library_path = os.environ.get("FABF_LIB") or os.path.join(_PKG, "libfabf.so")  # FABF_LIB: experiments

FLAG_LITERAL = 0x1
FLAG_CLAMP = 0x2
FLAG_DEBUG = 0x4
FLAG_FUSED = 0x8
CODE_IDENTITY = 0x1
CODE_GUARD = 0x2
CODE_SMALL_LAMBDA = 0x4
CODE_FALLBACK = 0x8
CODE_FAR_THETA = 0x10
MAX_N = 10

_STATUS = {0: "FABF_OK", 1: "FABF_ERR_INVALID_ARGUMENT", 2: "FABF_ERR_UNSUPPORTED",
           3: "FABF_ERR_CUDA", 4: "FABF_ERR_OUT_OF_MEMORY"}


class FabfError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"{_STATUS.get(status, status)}: {message}")
        self.status = status


class _Sharpen(ctypes.Structure):
    _fields_ = [("log_scale", ctypes.c_float), ("sigma_lo", ctypes.c_float), ("sigma_hi", ctypes.c_float),
                ("log_sat", ctypes.c_float)]


SHARPEN_DEFAULTS = dict(log_scale=1.0, sigma_lo=10.0, sigma_hi=40.0, log_sat=20.0)


class _Texture(ctypes.Structure):
    _fields_ = [("patch", ctypes.c_int), ("sigma_lo", ctypes.c_float), ("sigma_hi", ctypes.c_float),
                ("mrtv_sat", ctypes.c_float), ("eps", ctypes.c_float), ("second_scale", ctypes.c_float)]


TEXTURE_DEFAULTS = dict(patch=3, sigma_lo=8.0, sigma_hi=50.0, mrtv_sat=12.0, eps=1e-3, second_scale=0.8)


class _Diag(ctypes.Structure):
    _fields_ = [("alpha", ctypes.c_void_p), ("beta", ctypes.c_void_p), ("kappa", ctypes.c_void_p),
                ("t2n", ctypes.c_void_p), ("code", ctypes.c_void_p)]


_lock = threading.Lock()
_lib = None


def lib():
    """Load libfabf.so (raises if it has not been built -- no fallback)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(library_path):
                raise FabfError(2, f"{library_path} not built; run python -m paper_1811_02308_b200.build")
            L = ctypes.CDLL(library_path)
            P, i, u = ctypes.c_void_p, ctypes.c_int, ctypes.c_uint
            L.fabf_plan.argtypes = [ctypes.POINTER(P), i, i, i, u]
            L.fabf_filter.argtypes = [P, P, P, P, i, i, P, P]
            L.fabf_filter_diag.argtypes = [P, P, P, P, i, i, P, ctypes.POINTER(_Diag), P]
            L.fabf_bounds.argtypes = [P, P, i, P, P, P]
            L.fabf_filter_host.argtypes = [P, P, P, P, i, i, P, P]
            L.fabf_filter_profile.argtypes = [P, P, P, P, i, i, P, P, ctypes.POINTER(ctypes.c_float)]
            L.fabf_filter_events.argtypes = [P, P, P, P, i, i, P, P, ctypes.POINTER(ctypes.c_void_p)]
            L.fabf_last_fallback_count.argtypes = [P, ctypes.POINTER(ctypes.c_longlong)]
            if hasattr(L, "fabf_filter_sharpen"):
                L.fabf_sharpen_maps.argtypes = [P, P, i, ctypes.POINTER(_Sharpen), P, P, P]
                L.fabf_sharpen_maps.restype = ctypes.c_int
                L.fabf_filter_sharpen.argtypes = [P, P, i, i, ctypes.POINTER(_Sharpen), P, P]
                L.fabf_filter_sharpen.restype = ctypes.c_int
            if hasattr(L, "fabf_filter_texture"):
                L.fabf_texture_maps.argtypes = [P, P, ctypes.POINTER(_Texture), P, P, P]
                L.fabf_texture_maps.restype = ctypes.c_int
                L.fabf_filter_texture.argtypes = [P, P, i, i, ctypes.POINTER(_Texture), i, ctypes.POINTER(_Sharpen),
                                                  P, P, P, P]
                L.fabf_filter_texture.restype = ctypes.c_int
                L.fabf_filter_texture_map.argtypes = [P, P, P, ctypes.c_float, i, i, i, ctypes.POINTER(_Sharpen),
                                                      P, P, P, P]
                L.fabf_filter_texture_map.restype = ctypes.c_int
            if hasattr(L, "fabf_filter_gauss"):
                L.fabf_filter_gauss.argtypes = [P, P, P, P, i, i, P, P]
                L.fabf_filter_gauss.restype = ctypes.c_int
            if hasattr(L, "fabf_filter_mozerov"):
                L.fabf_filter_mozerov.argtypes = [P, P, P, P, i, P, P]
                L.fabf_filter_mozerov.restype = ctypes.c_int
            if hasattr(L, "fabf_filter_interleaved"):
                L.fabf_filter_interleaved.argtypes = [P, P, P, P, i, i, i, P, P]
                L.fabf_filter_interleaved.restype = ctypes.c_int
            if hasattr(L, "fabf_last_launch_count"):  # (absent from round-1 builds kept for A/B timing)
                L.fabf_last_launch_count.argtypes = [P, ctypes.POINTER(ctypes.c_int)]
                L.fabf_last_launch_count.restype = ctypes.c_int
            L.fabf_debug_status.argtypes = [P, ctypes.POINTER(ctypes.c_longlong), ctypes.POINTER(ctypes.c_longlong)]
            L.fabf_destroy.argtypes = [P]
            for fn in ("fabf_plan", "fabf_filter", "fabf_filter_diag", "fabf_bounds",
                       "fabf_filter_host", "fabf_last_fallback_count", "fabf_destroy",
                       "fabf_filter_profile", "fabf_filter_events", "fabf_debug_status"):
                getattr(L, fn).restype = ctypes.c_int
            L.fabf_status_string.argtypes = [i]
            L.fabf_status_string.restype = ctypes.c_char_p
            L.fabf_last_error_message.argtypes = []
            L.fabf_last_error_message.restype = ctypes.c_char_p
            L.fabf_version.argtypes = []
            L.fabf_version.restype = ctypes.c_int
            _lib = L
    return _lib


def version() -> int:
    return lib().fabf_version()


def _check(status: int):
    if status != 0:
        raise FabfError(status, lib().fabf_last_error_message().decode())


def _numel(shape):
    return shape[0] * shape[1] * shape[2]


def _dev_ptr(t, name, plan=None):
    """Device pointer of a contiguous float32 CUDA tensor holding exactly the
    plan's batch*height*width pixels (the C ABI reads and writes that many)."""
    import torch

    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise FabfError(1, f"{name} must be a CUDA tensor")
    if t.dtype != torch.float32 or not t.is_contiguous():
        raise FabfError(1, f"{name} must be contiguous float32")
    if plan is not None and t.numel() != _numel(plan.shape):
        raise FabfError(1, f"{name} has {t.numel()} elements, the plan {plan.shape} needs {_numel(plan.shape)}")
    return ctypes.c_void_p(t.data_ptr())


def _host_ptr(a, name, plan):
    """Host pointer of a contiguous float32 numpy array or CPU tensor with the
    plan's pixel count (other dtypes are refused, never reinterpreted)."""
    import numpy as np

    if hasattr(a, "data_ptr"):
        import torch

        if a.is_cuda or not a.is_contiguous() or a.dtype != torch.float32:
            raise FabfError(1, f"{name} must be a contiguous float32 host tensor")
        n, p = a.numel(), a.data_ptr()
    else:
        if not isinstance(a, np.ndarray) or not a.flags["C_CONTIGUOUS"] or a.dtype != np.float32:
            raise FabfError(1, f"{name} must be a contiguous float32 array")
        n, p = a.size, a.ctypes.data
    if n != _numel(plan.shape):
        raise FabfError(1, f"{name} has {n} elements, the plan {plan.shape} needs {_numel(plan.shape)}")
    return ctypes.c_void_p(p)


def _stream_ptr(stream):
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


class Plan:
    """fabf_plan / fabf_destroy for batch x height x width images."""

    def __init__(self, batch: int, height: int, width: int, flags: int = 0):
        self.shape = (int(batch), int(height), int(width))
        self.flags = int(flags)
        h = ctypes.c_void_p()
        _check(lib().fabf_plan(ctypes.byref(h), self.shape[0], self.shape[1], self.shape[2], self.flags))
        self._h = h

    @property
    def handle(self):
        return self._h

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib().fabf_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def last_fallback_count(self) -> int:
        c = ctypes.c_longlong(0)
        _check(lib().fabf_last_fallback_count(self._h, ctypes.byref(c)))
        return int(c.value)

    def last_launch_count(self) -> int:
        """Kernels the last filter call on this plan launched."""
        c = ctypes.c_int(0)
        _check(lib().fabf_last_launch_count(self._h, ctypes.byref(c)))
        return int(c.value)

    def debug_status(self):
        """FLAG_DEBUG plans: (violating pixels, first flat index or -1) of the last call."""
        c, f = ctypes.c_longlong(0), ctypes.c_longlong(0)
        _check(lib().fabf_debug_status(self._h, ctypes.byref(c), ctypes.byref(f)))
        return int(c.value), int(f.value)


def filter(plan: Plan, img, theta, sigma, rho: int, N: int, out=None, stream=None):
    """fabf_filter on device tensors; returns ``out``."""
    import torch

    if out is None:
        out = torch.empty_like(img)
    _check(lib().fabf_filter(plan.handle, _dev_ptr(img, "img", plan), _dev_ptr(theta, "theta", plan),
                             _dev_ptr(sigma, "sigma", plan), int(rho), int(N), _dev_ptr(out, "out", plan),
                             _stream_ptr(stream)))
    return out


def filter_diag(plan: Plan, img, theta, sigma, rho: int, N: int, out=None, stream=None):
    """fabf_filter_diag: returns (out, dict(alpha, beta, kappa, t2n, code))."""
    import torch

    if out is None:
        out = torch.empty_like(img)
    d = {k: torch.empty_like(img) for k in ("alpha", "beta", "kappa", "t2n")}
    d["code"] = torch.empty(img.shape, dtype=torch.uint8, device=img.device)
    diag = _Diag(*(ctypes.c_void_p(d[k].data_ptr()) for k in ("alpha", "beta", "kappa", "t2n", "code")))
    _check(lib().fabf_filter_diag(plan.handle, _dev_ptr(img, "img", plan), _dev_ptr(theta, "theta", plan),
                                  _dev_ptr(sigma, "sigma", plan), int(rho), int(N), _dev_ptr(out, "out", plan),
                                  ctypes.byref(diag), _stream_ptr(stream)))
    return out, d


def bounds(plan: Plan, img, rho: int, alpha=None, beta=None, stream=None):
    """fabf_bounds: (alpha, beta) = window (min, max)."""
    import torch

    alpha = torch.empty_like(img) if alpha is None else alpha
    beta = torch.empty_like(img) if beta is None else beta
    _check(lib().fabf_bounds(plan.handle, _dev_ptr(img, "img", plan), int(rho), _dev_ptr(alpha, "alpha", plan),
                             _dev_ptr(beta, "beta", plan), _stream_ptr(stream)))
    return alpha, beta


def filter_host(plan: Plan, img, theta, sigma, rho: int, N: int, out, stream=None):
    """fabf_filter_host on HOST buffers (numpy arrays or CPU tensors, ideally
    pinned); copies in, filters, copies out, synchronises."""
    def hp(a, name):
        return _host_ptr(a, name, plan)

    _check(lib().fabf_filter_host(plan.handle, hp(img, "img"), hp(theta, "theta"), hp(sigma, "sigma"),
                                  int(rho), int(N), hp(out, "out"), _stream_ptr(stream)))
    return out


def filter_events(plan: Plan, img, theta, sigma, rho: int, N: int, events, out=None, stream=None):
    """fabf_filter_events: the step with five caller-owned torch.cuda.Event
    (timing enabled, already created) recorded around its kernels; no sync."""
    import torch

    if out is None:
        out = torch.empty_like(img)
    if len(events) != 5:
        raise ValueError("five events")
    arr = (ctypes.c_void_p * 5)(*[ctypes.c_void_p(int(e.cuda_event)) for e in events])
    _check(lib().fabf_filter_events(plan.handle, _dev_ptr(img, "img", plan), _dev_ptr(theta, "theta", plan),
                                    _dev_ptr(sigma, "sigma", plan), int(rho), int(N), _dev_ptr(out, "out", plan),
                                    _stream_ptr(stream), arr))
    return out


def filter_profile(plan: Plan, img, theta, sigma, rho: int, N: int, out=None, stream=None):
    """fabf_filter_profile: returns (out, [ms bounds-rows, bounds-cols, filter, fallback])."""
    import torch

    if out is None:
        out = torch.empty_like(img)
    ms = (ctypes.c_float * 4)()
    _check(lib().fabf_filter_profile(plan.handle, _dev_ptr(img, "img", plan), _dev_ptr(theta, "theta", plan),
                                     _dev_ptr(sigma, "sigma", plan), int(rho), int(N), _dev_ptr(out, "out", plan),
                                     _stream_ptr(stream), ms))
    return out, [float(v) for v in ms]


def filter_interleaved(plan: Plan, img, theta, sigma, rho: int, N: int, out=None, stream=None):
    """fabf_filter_interleaved: colour / multi-channel images filtered channel by
    channel.  ``img``, ``theta``, ``sigma``: contiguous float32 CUDA
    tensors of shape (H, W, C) or (B, H, W, C); the plan's batch must be B * C
    planes.  Returns ``out`` (same shape)."""
    import torch

    if img.dim() not in (3, 4):
        raise FabfError(1, "img must be (H, W, C) or (B, H, W, C)")
    C = int(img.shape[-1])
    if out is None:
        out = torch.empty_like(img)

    def ptr(t, name):
        if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.float32 or not t.is_contiguous():
            raise FabfError(1, f"{name} must be a contiguous float32 CUDA tensor")
        if t.shape != img.shape or t.numel() != _numel(plan.shape):
            raise FabfError(1, f"{name} must have the image's shape and the plan's pixel count")
        return ctypes.c_void_p(t.data_ptr())

    _check(lib().fabf_filter_interleaved(plan.handle, ptr(img, "img"), ptr(theta, "theta"), ptr(sigma, "sigma"),
                                         C, int(rho), int(N), ptr(out, "out"), _stream_ptr(stream)))
    return out


def filter_mozerov(plan: Plan, img, theta, sigma, rho: int, out=None, stream=None):
    """fabf_filter_mozerov: the uniform-prior baseline on device tensors."""
    import torch

    if out is None:
        out = torch.empty_like(img)
    _check(lib().fabf_filter_mozerov(plan.handle, _dev_ptr(img, "img", plan), _dev_ptr(theta, "theta", plan),
                                     _dev_ptr(sigma, "sigma", plan), int(rho), _dev_ptr(out, "out", plan),
                                     _stream_ptr(stream)))
    return out


def _sharpen_params(kw):
    prm = dict(SHARPEN_DEFAULTS)
    prm.update(kw)
    return _Sharpen(*(float(prm[k]) for k in ("log_scale", "sigma_lo", "sigma_hi", "log_sat")))


def sharpen_maps(plan: Plan, img, rho: int, theta=None, sigma=None, stream=None, **params):
    """fabf_sharpen_maps: (theta, sigma) of the sharpening application."""
    import torch

    theta = torch.empty_like(img) if theta is None else theta
    sigma = torch.empty_like(img) if sigma is None else sigma
    prm = _sharpen_params(params)
    _check(lib().fabf_sharpen_maps(plan.handle, _dev_ptr(img, "img", plan), int(rho), ctypes.byref(prm),
                                   _dev_ptr(theta, "theta", plan), _dev_ptr(sigma, "sigma", plan),
                                   _stream_ptr(stream)))
    return theta, sigma


def filter_sharpen(plan: Plan, img, rho: int, N: int, out=None, stream=None, **params):
    """fabf_filter_sharpen: the sharpening application end to end on device tensors."""
    import torch

    out = torch.empty_like(img) if out is None else out
    prm = _sharpen_params(params)
    _check(lib().fabf_filter_sharpen(plan.handle, _dev_ptr(img, "img", plan), int(rho), int(N), ctypes.byref(prm),
                                     _dev_ptr(out, "out", plan), _stream_ptr(stream)))
    return out


def _texture_params(kw):
    prm = dict(TEXTURE_DEFAULTS)
    prm.update(kw or {})
    return _Texture(int(prm["patch"]), *(float(prm[k]) for k in ("sigma_lo", "sigma_hi", "mrtv_sat", "eps",
                                                                  "second_scale")))


def texture_maps(plan: Plan, img, sigma=None, mrtv=None, want_mrtv: bool = False, stream=None, **params):
    """fabf_texture_maps: the texture application's sigma map; returns
    (sigma, mrtv) -- mrtv is None unless asked for."""
    import torch

    sigma = torch.empty_like(img) if sigma is None else sigma
    if mrtv is None and want_mrtv:
        mrtv = torch.empty_like(img)
    prm = _texture_params(params)
    _check(lib().fabf_texture_maps(plan.handle, _dev_ptr(img, "img", plan), ctypes.byref(prm),
                                   _dev_ptr(sigma, "sigma", plan),
                                   None if mrtv is None else _dev_ptr(mrtv, "mrtv", plan), _stream_ptr(stream)))
    return sigma, mrtv


def filter_texture(plan: Plan, img, rho: int, N: int, texture=None, sharpen=None, rho_sharpen=None, out=None,
                   pass1=None, pass2=None, stream=None):
    """fabf_filter_texture: the three-pass texture-filtering application
    on device tensors; ``pass1`` / ``pass2`` (optional tensors) receive the
    intermediates."""
    import torch

    out = torch.empty_like(img) if out is None else out
    tp, sp = _texture_params(texture), _sharpen_params(sharpen or {})
    rs = int(rho if rho_sharpen is None else rho_sharpen)
    _check(lib().fabf_filter_texture(plan.handle, _dev_ptr(img, "img", plan), int(rho), int(N), ctypes.byref(tp), rs,
                                     ctypes.byref(sp), _dev_ptr(out, "out", plan),
                                     None if pass1 is None else _dev_ptr(pass1, "pass1", plan),
                                     None if pass2 is None else _dev_ptr(pass2, "pass2", plan), _stream_ptr(stream)))
    return out


def filter_texture_map(plan: Plan, img, sigma_map, rho: int, N: int, second_scale: float = 0.8, sharpen=None,
                       rho_sharpen=None, out=None, pass1=None, pass2=None, stream=None):
    """fabf_filter_texture_map: the three passes with the caller's sigma map (the
    paper's colour procedure: the map of the grey image for every channel plane)."""
    import torch

    out = torch.empty_like(img) if out is None else out
    sp = _sharpen_params(sharpen or {})
    rs = int(rho if rho_sharpen is None else rho_sharpen)
    _check(lib().fabf_filter_texture_map(plan.handle, _dev_ptr(img, "img", plan), _dev_ptr(sigma_map, "sigma_map", plan),
                                         float(second_scale), int(rho), int(N), rs, ctypes.byref(sp),
                                         _dev_ptr(out, "out", plan),
                                         None if pass1 is None else _dev_ptr(pass1, "pass1", plan),
                                         None if pass2 is None else _dev_ptr(pass2, "pass2", plan),
                                         _stream_ptr(stream)))
    return out


def filter_gauss(plan: Plan, img, theta, sigma, rho: int, N: int, out=None, stream=None):
    """fabf_filter_gauss: Algorithm 1 with the Gaussian spatial kernel of eq.(4)
    on [-3 rho, 3 rho]^2 (device tensors)."""
    import torch

    if out is None:
        out = torch.empty_like(img)
    _check(lib().fabf_filter_gauss(plan.handle, _dev_ptr(img, "img", plan), _dev_ptr(theta, "theta", plan),
                                   _dev_ptr(sigma, "sigma", plan), int(rho), int(N), _dev_ptr(out, "out", plan),
                                   _stream_ptr(stream)))
    return out
