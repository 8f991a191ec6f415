"""ctypes front end of the C oracle ``fabf_oracle.c`` (test infrastructure only).

Every function here is argument marshalling plus a thread pool over pixel ranges;
all arithmetic is in ``fabf_oracle.c``.  See that file's header for the paper
passages each routine follows (P:<line> = /root/reference/PAPER.md line).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from concurrent.futures import ThreadPoolExecutor

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "fabf_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

CODE_IDENTITY = 1
CODE_GUARD = 2
CODE_QUAD = 4
KAPPA_MAX = 1000.0

_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain C + libquadmath)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-O2", "-std=gnu11", "-fPIC", "-shared", "-o", tmp, _SRC, "-lquadmath", "-lm"]
        )
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_LIB)
            P = ctypes.c_void_p
            i, l, d = ctypes.c_int, ctypes.c_long, ctypes.c_double
            lib.fabfo_bounds.argtypes = [P, i, i, i, i, l, l, P, P]
            lib.fabfo_brute.argtypes = [P, P, P, i, i, i, i, l, l, P]
            lib.fabfo_fast.argtypes = [P, P, P, i, i, i, i, i, P, l, l, P, P, P, P, P]
            lib.fabfo_window.argtypes = [P, i, ctypes.c_float, ctypes.c_float, ctypes.c_float, i, i, P, P]
            lib.fabfo_hilbert_inverse.argtypes = [i, P]
            lib.fabfo_fit.argtypes = [P, i, P]
            lib.fabfo_stretch.argtypes = [P, i, d, d, P]
            lib.fabfo_integrals.argtypes = [d, d, i, P, i]
            lib.fabfo_literal.argtypes = [P, P, P, i, i, i, i, i, P]
            lib.fabfo_mozerov.argtypes = [P, P, P, i, i, i, i, l, l, P]
            lib.fabfo_fast_gauss.argtypes = [P, P, P, i, i, i, i, i, P, l, l, P, P, P, P, P]
            lib.fabfo_brute_gauss.argtypes = [P, P, P, i, i, i, i, l, l, P]
            lib.fabfo_window_w.argtypes = [P, P, i, ctypes.c_float, ctypes.c_float, ctypes.c_float, i, i, P, P]
            lib.fabfo_sharpen_maps.argtypes = [P, i, i, i, i, d, d, d, d, l, l, P, P]
            lib.fabfo_texture_maps.argtypes = [P, i, i, i, i, d, d, d, d, l, l, P, P]
            for fn in ("fabfo_bounds", "fabfo_brute", "fabfo_fast", "fabfo_window", "fabfo_literal", "fabfo_mozerov",
                       "fabfo_sharpen_maps", "fabfo_texture_maps", "fabfo_fast_gauss", "fabfo_brute_gauss", "fabfo_window_w",
                       "fabfo_hilbert_inverse", "fabfo_fit", "fabfo_stretch", "fabfo_integrals"):
                getattr(lib, fn).restype = ctypes.c_int
            _lib = lib
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _as3d(a):
    a = _f32(a)
    if a.ndim == 2:
        a = a[None]
    if a.ndim != 3:
        raise ValueError("expected H x W or B x H x W")
    return a


def _parallel(total: int, fn, threads: int | None, chunk: int = 4096):
    threads = threads or os.cpu_count() or 1
    ranges = [(s, min(total, s + chunk)) for s in range(0, total, chunk)]
    if threads <= 1 or len(ranges) <= 1:
        for r in ranges:
            fn(*r)
        return
    with ThreadPoolExecutor(max_workers=threads) as ex:
        for fut in [ex.submit(fn, *r) for r in ranges]:
            fut.result()


def bounds(img, rho: int, threads: int | None = None):
    """eq.(8) P:199-203 by exhaustive window scan -> (alpha, beta), float32."""
    lib = _load()
    f = _as3d(img)
    B, H, W = f.shape
    alpha = np.empty_like(f)
    beta = np.empty_like(f)

    def run(p0, p1):
        if lib.fabfo_bounds(_ptr(f), B, H, W, rho, p0, p1, _ptr(alpha), _ptr(beta)):
            raise ValueError("fabfo_bounds: invalid arguments")

    _parallel(f.size, run, threads)
    shp = np.shape(img)
    return alpha.reshape(shp), beta.reshape(shp)


def brute(img, theta, sigma, rho: int, threads: int | None = None, spatial: str = "box"):
    """eq.(1)-(3) P:54-67, fp64 -> g (float64).  ``spatial``: "box" (omega = 1 on
    the (2 rho + 1)^2 box, reading R1) or "gauss" (eq.(4): exp(-|j|^2 / 2 rho^2)
    on [-3 rho, 3 rho]^2)."""
    lib = _load()
    fn = {"box": lib.fabfo_brute, "gauss": lib.fabfo_brute_gauss}[spatial]
    f, th, sg = _as3d(img), _as3d(theta), _as3d(sigma)
    B, H, W = f.shape
    g = np.empty(f.shape, np.float64)

    def run(p0, p1):
        if fn(_ptr(f), _ptr(th), _ptr(sg), B, H, W, rho, p0, p1, _ptr(g)):
            raise ValueError("fabfo_brute: invalid arguments")

    _parallel(f.size, run, threads, chunk=2048)
    return g.reshape(np.shape(img))


def fast(img, theta, sigma, rho: int, N: int, pixels=None, threads: int | None = None, spatial: str = "box"):
    """Algorithm 1 / eq.(29) in __float128.

    Returns a dict of arrays: ``g_lit`` (eq.(29) as printed), ``g_guard`` (with the
    reading-R7 guard), ``kappa``, ``t2n`` (T2/n) and ``code``.  With ``pixels`` (flat
    indices into B*H*W) only those pixels are computed and the arrays follow that
    list; otherwise they have the image's shape.
    """
    lib = _load()
    fn = {"box": lib.fabfo_fast, "gauss": lib.fabfo_fast_gauss}[spatial]
    f, th, sg = _as3d(img), _as3d(theta), _as3d(sigma)
    B, H, W = f.shape
    if pixels is not None:
        idx = np.ascontiguousarray(pixels, dtype=np.int64).ravel()
        total = idx.size
    else:
        idx = None
        total = f.size
    out = {
        "g_lit": np.empty(total, np.float64),
        "g_guard": np.empty(total, np.float64),
        "kappa": np.empty(total, np.float64),
        "t2n": np.empty(total, np.float64),
        "code": np.empty(total, np.uint8),
    }

    def run(p0, p1):
        rc = fn(_ptr(f), _ptr(th), _ptr(sg), B, H, W, rho, N, _ptr(idx), p0, p1,
                            _ptr(out["g_lit"]), _ptr(out["g_guard"]), _ptr(out["kappa"]),
                            _ptr(out["t2n"]), _ptr(out["code"]))
        if rc:
            raise ValueError("fabfo_fast: invalid arguments")

    n = (2 * (3 * rho if spatial == "gauss" else rho) + 1) ** 2
    _parallel(total, run, threads, chunk=max(16, min(4096, 400000 // max(1, n * (N + 1)))))
    if pixels is None:
        shp = np.shape(img)
        out = {k: v.reshape(shp) for k, v in out.items()}
    return out


def fast_window(vals, f_center: float, theta: float, sigma: float, N: int, route: int = 0, weights=None):
    """g-hat for one explicit window (samples ``vals``): dict of scalars.

    ``route`` selects how eq.(22) is summed: 0 over the window's distinct values
    weighted by their counts (the histogram of eq.(5); what ``fast`` uses), 1
    sample by sample."""
    lib = _load()
    v = _f32(vals).ravel()
    o = np.empty(6, np.float64)
    code = ctypes.c_int(0)
    if weights is not None:  # omega(j) = weights[j] (the weighted histogram of eq.(5))
        wt = np.ascontiguousarray(weights, np.float64).ravel()
        if wt.size != v.size or lib.fabfo_window_w(_ptr(v), _ptr(wt), v.size, float(f_center), float(theta),
                                                   float(sigma), N, int(route), _ptr(o), ctypes.byref(code)):
            raise ValueError("fabfo_window_w: invalid arguments")
        return dict(g_lit=o[0], g_guard=o[1], kappa=o[2], t2n=o[3], lam=o[4], t0=o[5], code=code.value)
    if lib.fabfo_window(_ptr(v), v.size, float(f_center), float(theta), float(sigma), N, int(route), _ptr(o),
                        ctypes.byref(code)):
        raise ValueError("fabfo_window: invalid arguments")
    return dict(g_lit=o[0], g_guard=o[1], kappa=o[2], t2n=o[3], lam=o[4], t0=o[5], code=code.value)


def hilbert_inverse(N: int):
    """Theorem 1, eq.(19), as a float64 (N+1)x(N+1) array."""
    lib = _load()
    o = np.empty((N + 1, N + 1), np.float64)
    if lib.fabfo_hilbert_inverse(N, _ptr(o)):
        raise ValueError("N out of range")
    return o


def fit(mu, N: int):
    """c = A^{-1} mu (Algorithm 1 line 11) evaluated in __float128."""
    lib = _load()
    m = np.ascontiguousarray(mu, np.float64)
    c = np.empty(N + 1, np.float64)
    if lib.fabfo_fit(_ptr(m), N, _ptr(c)):
        raise ValueError("bad arguments")
    return c


def stretch(m, N: int, alpha: float, beta: float):
    """Prop.3 eq.(24) P:338-345 (binomial transform) in __float128."""
    lib = _load()
    mm = np.ascontiguousarray(m, np.float64)
    mu = np.empty(N + 1, np.float64)
    if lib.fabfo_stretch(_ptr(mm), N, alpha, beta, _ptr(mu)):
        raise ValueError("bad arguments")
    return mu


def integrals(lam: float, t0: float, K: int, method: int = 0):
    """I_0..I_K of eq.(28); method 0 auto, 1 eqs.(30)-(32), 2 quadrature.

    Returns (I, method_used)."""
    lib = _load()
    o = np.empty(K + 1, np.float64)
    used = lib.fabfo_integrals(lam, t0, K, _ptr(o), method)
    if used < 0:
        raise ValueError("bad arguments")
    return o, used


def literal(img, theta, sigma, rho: int, N: int, threads: int | None = None):
    """O3: Algorithm 1 as printed, plain fp64, the paper's [0,1] scaling,
    running-sum box moments, eq.(24), eq.(19), eqs.(30)-(32) for every lambda, no
    guard.  CONTEXT ONLY (not a parity target): how far the paper's own numerics
    drift from ``fast``.  Whole images; images of a batch run in parallel."""
    lib = _load()
    f, th, sg = _as3d(img), _as3d(theta), _as3d(sigma)
    B, H, W = f.shape
    g = np.empty(f.shape, np.float64)

    def run(b0, b1):
        for b in range(b0, b1):
            if lib.fabfo_literal(_ptr(f[b:b + 1]), _ptr(th[b:b + 1]), _ptr(sg[b:b + 1]), 1, H, W, rho, N,
                                 _ptr(g[b:b + 1])):
                raise ValueError("fabfo_literal: invalid arguments")

    _parallel(B, run, threads, chunk=1)
    return g.reshape(np.shape(img))


def mozerov(img, theta, sigma, rho: int, threads: int | None = None):
    """Mozerov & van de Weijer's uniform-prior filter as the paper compares it
    (P:128-141): eq.(29) at N = 0 on [f, 2 fbar - f] (Delta = 0) instead of
    [alpha, beta]; f where that interval is a point.  __float128 -> float64."""
    lib = _load()
    f, th, sg = _as3d(img), _as3d(theta), _as3d(sigma)
    B, H, W = f.shape
    g = np.empty(f.shape, np.float64)

    def run(p0, p1):
        if lib.fabfo_mozerov(_ptr(f), _ptr(th), _ptr(sg), B, H, W, rho, p0, p1, _ptr(g)):
            raise ValueError("fabfo_mozerov: invalid arguments")

    _parallel(f.size, run, threads, chunk=2048)
    return g.reshape(np.shape(img))


SHARPEN_DEFAULTS = dict(log_scale=1.0, sigma_lo=10.0, sigma_hi=40.0, log_sat=20.0)


def sharpen_maps(img, rho: int, log_scale=1.0, sigma_lo=10.0, sigma_hi=40.0, log_sat=20.0,
                 threads: int | None = None):
    """The sharpening application's maps: theta = 2f - fbar (box mean
    over Omega), sigma = sigma_hi - (sigma_hi - sigma_lo) min(|LoG f| / log_sat, 1)
    (reading R15).  Returns (theta, sigma) as float64."""
    lib = _load()
    f = _as3d(img)
    B, H, W = f.shape
    th = np.empty(f.shape, np.float64)
    sg = np.empty(f.shape, np.float64)

    def run(p0, p1):
        if lib.fabfo_sharpen_maps(_ptr(f), B, H, W, rho, float(log_scale), float(sigma_lo), float(sigma_hi),
                                  float(log_sat), p0, p1, _ptr(th), _ptr(sg)):
            raise ValueError("fabfo_sharpen_maps: invalid arguments")

    _parallel(f.size, run, threads, chunk=4096)
    return th.reshape(np.shape(img)), sg.reshape(np.shape(img))


TEXTURE_DEFAULTS = dict(patch=3, sigma_lo=8.0, sigma_hi=50.0, mrtv_sat=12.0, eps=1e-3, second_scale=0.8)


def texture_maps(img, patch=3, sigma_lo=8.0, sigma_hi=50.0, mrtv_sat=12.0, eps=1e-3, second_scale=0.8,
                 threads: int | None = None):
    """The texture-filtering application's maps (reading R19): mRTV over
    the box of half-width ``patch`` and sigma = sigma_hi - (sigma_hi - sigma_lo)
    min(mRTV / mrtv_sat, 1).  Returns (mrtv, sigma) as float64 (``second_scale``
    belongs to the pipeline and is ignored here)."""
    lib = _load()
    f = _as3d(img)
    B, H, W = f.shape
    m = np.empty(f.shape, np.float64)
    sg = np.empty(f.shape, np.float64)

    def run(p0, p1):
        if lib.fabfo_texture_maps(_ptr(f), B, H, W, int(patch), float(sigma_lo), float(sigma_hi), float(mrtv_sat),
                                  float(eps), p0, p1, _ptr(m), _ptr(sg)):
            raise ValueError("fabfo_texture_maps: invalid arguments")

    _parallel(f.size, run, threads, chunk=4096)
    return m.reshape(np.shape(img)), sg.reshape(np.shape(img))


def texture_pipeline(img, rho: int, N: int, texture=None, sharpen=None, rho_sharpen: int | None = None,
                     sigma=None, pass1=None, pass2=None, threads: int | None = None):
    """The three applications of Algorithm 1 of P:849-852: smoothing with
    theta = f and the mRTV sigma map, smoothing again with sigma scaled by
    ``second_scale`` (0.8 in the paper; the map is still the input image's), then
    the sharpening rule of P:620-630 on the result.  Each pass's output is the
    guarded g-hat rounded to fp32 (it is the next pass's fp32 input image, as on
    the device), the maps are rounded to fp32 likewise.  ``sigma`` / ``pass1`` /
    ``pass2`` replace the corresponding intermediate when given (stage-by-stage
    parity: the next stage is evaluated on the device's own intermediate).
    Returns a dict: sigma, pass1, pass2, theta3, sigma3, out."""
    tp = dict(TEXTURE_DEFAULTS)
    tp.update(texture or {})
    sp = dict(SHARPEN_DEFAULTS)
    sp.update(sharpen or {})
    rs = rho if rho_sharpen is None else int(rho_sharpen)
    f = _f32(img)
    if sigma is None:
        sigma = texture_maps(f, threads=threads, **tp)[1]
    sg = _f32(sigma)
    if pass1 is None:
        pass1 = fast(f, f, sg, rho, N, threads=threads)["g_guard"]
    g1 = _f32(pass1)
    sg2 = _f32(np.float32(tp["second_scale"]) * sg)
    if pass2 is None:
        pass2 = fast(g1, g1, sg2, rho, N, threads=threads)["g_guard"]
    g2 = _f32(pass2)
    th3, sg3 = sharpen_maps(g2, rs, threads=threads, **sp)
    out = fast(g2, _f32(th3), _f32(sg3), rs, N, threads=threads)["g_guard"]
    return dict(sigma=sg, pass1=g1, pass2=g2, theta3=th3, sigma3=sg3, out=out)
