"""Helpers shared by the GPU parity tests (test infrastructure)."""
from __future__ import annotations

import numpy as np

TOL_GREY = 0.05  # north_star: max |delta| <= 0.05 grey levels on a 0-255 scale
KAPPA_BAND = (990.0, 1010.0)  # guard decision taken within float rounding of the threshold


def grey_scale(img: np.ndarray) -> float:
    """Tolerance scale: 1 for 0-255 images, else (range / 255)."""
    span = float(img.max() - img.min())
    return 1.0 if img.min() >= 0 and img.max() <= 255 and span > 64 else max(span, 1e-30) / 255.0


def compare_guarded(gpu: np.ndarray, orc: dict, scale: float, tol: float = TOL_GREY):
    """Element-wise parity of the guarded output.  Where the oracle's kappa sits
    within rounding of the guard threshold either branch is a correct result."""
    g = np.asarray(gpu, np.float64).ravel()
    ref = orc["g_guard"].ravel()
    lit = orc["g_lit"].ravel()
    kap = orc["kappa"].ravel()
    err = np.abs(g - ref)
    band = (kap >= KAPPA_BAND[0]) & (kap <= KAPPA_BAND[1])
    err = np.where(band, np.minimum(err, np.abs(g - lit)), err)
    bad = err > tol * scale
    return float(err.max(initial=0.0)) / scale, int(bad.sum()), err / scale


def compare_literal(gpu: np.ndarray, orc: dict, scale: float, tol: float = TOL_GREY):
    """Literal eq.(29): compared where the oracle's kappa <= 1e3 (well-posed)."""
    g = np.asarray(gpu, np.float64).ravel()
    lit = orc["g_lit"].ravel()
    kap = orc["kappa"].ravel()
    ok = np.isfinite(kap) & (kap <= 1e3)
    err = np.where(ok, np.abs(g - lit), 0.0)
    return float(err.max(initial=0.0)) / scale, int((err > tol * scale).sum()), int((~ok).sum())


def psnr(a: np.ndarray, b: np.ndarray, peak: float = 255.0) -> float:
    mse = float(np.mean((np.asarray(a, np.float64) - np.asarray(b, np.float64)) ** 2))
    return float("inf") if mse == 0 else 10.0 * np.log10(peak * peak / mse)
